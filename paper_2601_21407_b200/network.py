"""Recurrent HH network (BASELINE config 5): layered cortex with delayed
spike delivery and per-step spike exchange across GPUs.

Reference: hhengine/cortex.py.  Host side (this module, NumPy): the config
and topology types and `build_network`, which draws exactly the reference's
RNG sequence (cortex.py:138-218) so a seed gives the same synapses.  Device
side (`CortexNetwork`, libhhb200.so): one step is

  hhb_cortex_input   drain ring row t % D, psp = psp*decay + arrived + background
                     (+ extra)                                   cortex.py:283-301
  hhb_forward        the HH step on the local neurons, spike bitmap cortex.py:303
  exchange           all-gather of the per-rank bitmap words (NCCL when the
                     population spans GPUs; identity on one GPU)
  hhb_spike_deliver  every set bit -> its synapse row -> ring[(t+d) % D][target]
                                                                 cortex.py:304-308

Delivery accumulates fixed-point integers (weights quantised to 2^-24 uA), so
the sum is independent of arrival order: bit-identical for any number of
ranks and any atomic ordering.  Each rank holds the synapses whose TARGET it
owns (re-partitioned from the reference's CSR-by-source), its slice of the
ring and its neurons' state; shard boundaries are multiples of 32 neurons so
bitmap words never straddle ranks.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _device as D
from . import _native as nat
from . import connectivity as conn
from .defaults import cortical_rs_params
from .dynamics import HHParams, _forward, _raise_if_bad, _table, init_state
from .errors import ConfigurationError, ExchangeError, NativeLibraryError, UsageError

W_FRAC_BITS = 24  # weight quantum 2^-24 uA


# ---------------------------------------------------------------------------
# specs and topology (cortex.py:28-218)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class PopulationSpec:
    name: str
    size: int
    offset: int

    def __post_init__(self):
        if self.size <= 0:
            raise ConfigurationError(f"population {self.name} is empty")


@dataclass(frozen=True)
class BackgroundSpec:
    """Independent external Poisson sources per neuron, Gaussian amplitudes."""

    rate_hz: float
    k_ext: np.ndarray
    w_mean: float
    w_std: float

    def __post_init__(self):
        if self.rate_hz < 0 or self.w_std < 0:
            raise ConfigurationError("background rate and w_std must be >= 0")


@dataclass
class CortexConfig:
    scale: float = 0.1
    recurrent_mean: float = 0.26
    recurrent_std: float = 0.026
    bg_mean: float = 0.17
    bg_std: float = 0.017
    bg_rate_hz: float = 8.0
    inh_factor: float = 4.0
    psp_tau_ms: float = 0.5
    dt: float = 0.1
    neuron: HHParams | None = None

    def resolved_neuron(self) -> HHParams:
        return self.neuron if self.neuron is not None else cortical_rs_params(dt=self.dt)


REST_CONFIG = CortexConfig()
THALAMIC_CONFIG = CortexConfig(bg_mean=0.22, bg_std=0.022, bg_rate_hz=4.0)


@dataclass
class NetworkTopology:
    """Synapses in CSR-by-source layout plus per-block bookkeeping."""

    populations: list
    syn_offsets: np.ndarray
    syn_target: np.ndarray
    syn_weight: np.ndarray
    syn_delay: np.ndarray
    block_stats: dict
    max_delay: int
    dt: float

    @property
    def n_neurons(self) -> int:
        return self.populations[-1].offset + self.populations[-1].size

    @property
    def n_synapses(self) -> int:
        return int(self.syn_target.size)

    def population(self, name: str) -> PopulationSpec:
        for p in self.populations:
            if p.name == name:
                return p
        raise UsageError(f"unknown population {name!r}")

    def pop_slice(self, name: str) -> slice:
        p = self.population(name)
        return slice(p.offset, p.offset + p.size)

    def pop_index(self) -> np.ndarray:
        """Population index of every neuron."""
        idx = np.empty(self.n_neurons, dtype=np.int32)
        for k, p in enumerate(self.populations):
            idx[p.offset:p.offset + p.size] = k
        return idx


def _lognormal_delays(rng, n, mean_ms, dt):
    """Rounded lognormal delays with std = DELAY_REL_STD * mean, >= 1 step
    (cortex.py:130-135); same RNG call as the reference."""
    s2 = math.log(1.0 + conn.DELAY_REL_STD ** 2)
    mu = math.log(mean_ms) - s2 / 2.0
    d = rng.lognormal(mu, math.sqrt(s2), size=n)
    return np.maximum(np.rint(d / dt).astype(np.int32), 1)


def build_network(scale: float, seed: int, config: CortexConfig | None = None) -> NetworkTopology:
    """Sample the sparse topology (cortex.py:138-218): per (pre, post) block a
    Binomial(N_pre*N_post, p) synapse count drawn without replacement,
    sign-constrained Gaussian weights, lognormal delays.  The draws happen in
    the reference's order, so a seed reproduces its network exactly."""
    if not (0.0 < scale <= 1.0):
        raise ConfigurationError("scale must lie in (0, 1]")
    cfg = config if config is not None else REST_CONFIG
    rng = np.random.default_rng(seed)
    sizes = np.rint(conn.FULL_SIZES * scale).astype(int)
    if (sizes <= 0).any():
        raise ConfigurationError(f"scale {scale} empties a population: {sizes}")
    offsets = np.concatenate([[0], np.cumsum(sizes)])
    pops = [PopulationSpec(nm, int(sz), int(off)) for nm, sz, off in zip(conn.POPULATIONS, sizes, offsets[:-1])]
    pre_l, post_l, w_l, d_l = [], [], [], []
    stats = {}
    for a, a_name in enumerate(conn.POPULATIONS):
        exc = conn.is_excitatory(a)
        wm = cfg.recurrent_mean if exc else -cfg.inh_factor * cfg.recurrent_mean
        ws = cfg.recurrent_std if exc else cfg.inh_factor * cfg.recurrent_std
        dm = conn.DELAY_MEAN_EXC_MS if exc else conn.DELAY_MEAN_INH_MS
        for b, b_name in enumerate(conn.POPULATIONS):
            p = conn.CONN_PROBS[b, a]
            pairs = sizes[a] * sizes[b]
            count = int(rng.binomial(pairs, p)) if p > 0 else 0
            stats[(a_name, b_name)] = {"count": count, "w_mean": wm, "w_std": ws, "p": float(p),
                                       "pairs": int(pairs)}
            if count == 0:
                continue
            ids = rng.choice(pairs, size=count, replace=False)
            src, dst = np.divmod(ids, sizes[b])
            w = rng.normal(wm, ws, size=count)
            w = np.maximum(w, 0.0) if exc else np.minimum(w, 0.0)
            pre_l.append(offsets[a] + src)
            post_l.append(offsets[b] + dst)
            w_l.append(w)
            d_l.append(_lognormal_delays(rng, count, dm, cfg.dt))
    n = int(offsets[-1])
    if pre_l:
        pre = np.concatenate(pre_l).astype(np.int64)
        post = np.concatenate(post_l).astype(np.int64)
        w = np.concatenate(w_l)
        d = np.concatenate(d_l)
    else:
        pre = post = np.zeros(0, dtype=np.int64)
        w, d = np.zeros(0), np.zeros(0, dtype=np.int32)
    order = np.argsort(pre, kind="stable")
    pre, post, w, d = pre[order], post[order], w[order], d[order]
    row = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row, pre + 1, 1)
    return NetworkTopology(pops, np.cumsum(row), post.astype(np.int32), w, d.astype(np.int32), stats,
                           int(d.max()) if d.size else 1, cfg.dt)


def make_background(config: CortexConfig) -> BackgroundSpec:
    return BackgroundSpec(config.bg_rate_hz, conn.K_EXT.astype(float), config.bg_mean, config.bg_std)


def background_lambda(topo: NetworkTopology, bg: BackgroundSpec, dt: float) -> np.ndarray:
    """Expected external events per neuron per step (cortex.py:290-295)."""
    lam = np.empty(topo.n_neurons)
    for k, p in enumerate(topo.populations):
        lam[p.offset:p.offset + p.size] = bg.k_ext[k] * bg.rate_hz * dt / 1000.0
    return lam


class HostBackground:
    """The reference's compound-Poisson background drawn on the host with its
    own RNG call sequence (cortex.py:225-232, 296), for parity runs against
    `run_network`: N ~ Poisson(lam); N*mu + sigma*sqrt(N)*z."""

    def __init__(self, topo, bg: BackgroundSpec, dt: float, rng: np.random.Generator):
        self.lam = background_lambda(topo, bg, dt)
        self.bg, self.rng, self.n = bg, rng, topo.n_neurons

    def sample(self) -> np.ndarray:
        k = self.rng.poisson(self.lam, size=self.n)
        out = k * self.bg.w_mean
        if self.bg.w_std > 0:
            out = out + self.bg.w_std * np.sqrt(k) * self.rng.standard_normal(self.n)
        return out


# ---------------------------------------------------------------------------
# sharding
# ---------------------------------------------------------------------------

def shard_range(n: int, rank: int, world: int) -> tuple:
    """[lo, hi) neurons of `rank`: contiguous, boundaries multiples of 32."""
    words = (n + 31) // 32
    per = (words + world - 1) // world
    lo = min(n, rank * per * 32)
    hi = min(n, (rank + 1) * per * 32)
    return lo, hi


def local_synapses(topo: NetworkTopology, lo: int, hi: int):
    """CSR over ALL sources of the synapses whose target lies in [lo, hi), with
    targets made local; the reference's per-source order is kept."""
    tgt = topo.syn_target.astype(np.int64)
    keep = (tgt >= lo) & (tgt < hi)
    src = np.repeat(np.arange(topo.n_neurons, dtype=np.int64), np.diff(topo.syn_offsets))[keep]
    counts = np.bincount(src, minlength=topo.n_neurons)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    return off, (tgt[keep] - lo).astype(np.int32), topo.syn_weight[keep], topo.syn_delay[keep]


def words_per_rank(n: int, world: int) -> int:
    return ((n + 31) // 32 + world - 1) // world


def allgather_exchange(n_global: int, group=None):
    """Bitmap all-gather over torch.distributed (NCCL between GPUs, gloo on CPU):
    every rank contributes words_per_rank words (its shard, zero padded) and
    receives the global bitmap.  4.8 KB per step at 38,586 neurons.  With a
    gloo group and device words the exchange is staged through host memory
    (gloo has no device all-gather): every step then synchronises the stream,
    which is what the CPU / one-GPU multi-process tests use."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    per = words_per_rank(n_global, world)
    total = (n_global + 31) // 32
    staged = dist.get_backend(group) == "gloo"
    buf = {}

    def exchange(local_words: torch.Tensor, gwords: torch.Tensor):
        dev = local_words.device
        out = buf.get(dev)
        if out is None:
            out = buf[dev] = torch.empty(per * world, dtype=torch.int32, device="cpu" if staged else dev)
        src = local_words[:per].contiguous()
        dist.all_gather_into_tensor(out, src.cpu() if staged else src, group=group)
        gwords[:total].copy_(out[:total])

    return exchange


class LibraryExchange:
    """The per-step spike-bitmap all-gather inside the C-ABI library
    (hhb_spk_exchange_*: ncclAllGather on the caller's stream over NVLink /
    NVSwitch), so CortexNetwork.advance() captures it into its CUDA graphs with
    the step kernels.  The communicator is the library's own (rank 0's NCCL
    unique id is broadcast over `group`, any torch.distributed backend).
    check() raises ExchangeError on an NCCL asynchronous error; wait() blocks
    until the stream's work is done or `timeout_s` passes, then aborts the
    communicator and raises ExchangeError (a dead peer cannot hang a rank)."""

    def __init__(self, n_global: int, group=None, timeout_s: float = 300.0, rank: int | None = None,
                 world: int | None = None):
        lib = nat.load()
        if not lib.hhb_spk_exchange_available():
            raise NativeLibraryError("NCCL (libnccl.so.2) is not loadable: no library spike exchange")
        if rank is None or world is None:
            import torch.distributed as dist
            rank, world = dist.get_rank(group), dist.get_world_size(group)
        else:
            dist = None
        self.rank, self.world = int(rank), int(world)
        self.per = words_per_rank(n_global, self.world)
        self.total = (n_global + 31) // 32
        self.timeout_s = float(timeout_s)
        uid = C.create_string_buffer(128)
        if self.rank == 0:
            nat.check(lib.hhb_spk_exchange_unique_id(uid, 128), "hhb_spk_exchange_unique_id")
        if self.world > 1:
            import torch.distributed as dist
            obj = [bytes(uid.raw)]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            uid = C.create_string_buffer(obj[0], 128)
        h = C.c_void_p()
        nat.check(lib.hhb_spk_exchange_init(uid, self.rank, self.world, self.per, C.byref(h)),
                  "hhb_spk_exchange_init")
        self.handle = h
        self._buf = {}

    def gathered_words(self) -> int:
        return self.per * self.world

    def __call__(self, local_words: torch.Tensor, gwords: torch.Tensor):
        """local_words: >= words_per_rank int32 (this rank's shard);
        gwords: >= world * words_per_rank int32 receives every rank's words."""
        if self.handle is None:
            raise ExchangeError("spike exchange used after close()")
        if gwords.numel() < self.per * self.world or local_words.numel() < self.per:
            raise UsageError("exchange buffers too small")
        nat.check(nat.load().hhb_spk_exchange_allgather(self.handle, local_words.data_ptr(), gwords.data_ptr(),
                                                        D.stream()), "hhb_spk_exchange_allgather")

    def check(self):
        if self.handle is None:
            return
        lib = nat.load()
        if lib.hhb_spk_exchange_status(self.handle) != 0:
            msg = lib.hhb_last_error().decode(errors="replace")
            self.abort()
            raise ExchangeError(msg)

    def wait(self, stream=None):
        """Block until the work queued on `stream` (default: current) is done,
        polling the NCCL status; abort + ExchangeError after timeout_s."""
        import time
        ev = torch.cuda.Event()
        ev.record(stream)
        t0 = time.monotonic()
        while not ev.query():
            self.check()
            if time.monotonic() - t0 > self.timeout_s:
                self.abort()
                raise ExchangeError(f"spike exchange did not complete within {self.timeout_s:.0f} s")
            time.sleep(1e-4)
        self.check()

    def abort(self):
        if self.handle is not None:
            nat.load().hhb_spk_exchange_abort(self.handle)
            self.handle = None

    def close(self):
        if self.handle is not None:
            nat.load().hhb_spk_exchange_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def quantise_weights(w: np.ndarray) -> np.ndarray:
    q = np.rint(np.asarray(w, dtype=np.float64) * (1 << W_FRAC_BITS))
    if np.abs(q).max(initial=0) >= 2 ** 31:
        raise ConfigurationError("synaptic weight too large for the fixed-point ring")
    return q.astype(np.int32)


# ---------------------------------------------------------------------------
# device network
# ---------------------------------------------------------------------------

class CortexNetwork:
    """Device-resident network state and step for one rank's neuron shard.

    exchange(local_words) -> global_words is the all-gather of the spike
    bitmap (identity when world == 1).  background: "host" uses a
    HostBackground (pass `host_bg`), "philox" draws the compound Poisson drive
    on the device keyed by (seed, global neuron, step) -- shard-invariant.
    """

    def __init__(self, topo: NetworkTopology, config: CortexConfig, device=None, dtype=np.float64,
                 rank: int = 0, world: int = 1, exchange=None, background: str = "philox",
                 host_bg: HostBackground | None = None, seed: int = 0):
        self.topo, self.config = topo, config
        self.dev = device or D.require_cuda()
        self.params = config.resolved_neuron().with_(dtype=dtype)
        self.dtype = np.dtype(dtype)
        self.td = D.torch_dtype(self.dtype)
        self.rank, self.world = rank, world
        self.n_global = topo.n_neurons
        self.lo, self.hi = shard_range(self.n_global, rank, world)
        self.n = self.hi - self.lo
        self.words_global = (self.n_global + 31) // 32
        self.word_lo = self.lo // 32
        self.exchange = exchange
        self.depth = topo.max_delay + 1
        off, tgt, w, d = local_synapses(topo, self.lo, self.hi)
        dev = self.dev
        self.off = torch.from_numpy(off).to(dev)
        self.tgt = torch.from_numpy(tgt).to(dev)
        self.w = torch.from_numpy(quantise_weights(w)).to(dev)
        self.delay = torch.from_numpy(d.astype(np.int32)).to(dev)
        st = init_state(self.params, (self.n,), device=dev)
        self.v, self.g = st.v.contiguous(), st.gates.contiguous()
        self.psp = torch.zeros(self.n, dtype=self.td, device=dev)
        self.ring = torch.zeros((self.depth, max(1, self.n)), dtype=torch.int64, device=dev)
        self.cur = torch.empty(max(1, self.n), dtype=self.td, device=dev)
        # padded to the same count on every rank for the all-gather
        self.words = torch.zeros(max(1, words_per_rank(self.n_global, world)), dtype=torch.int32, device=dev)
        # padded to world * words_per_rank: the all-gather writes every rank's words in place
        self.gwords = torch.zeros(max(self.words_global, words_per_rank(self.n_global, world) * world),
                                  dtype=torch.int32, device=dev)
        self.first_bad = torch.full((1,), D.INT64_MAX, dtype=torch.int64, device=dev)
        self.decay = math.exp(-config.dt / config.psp_tau_ms)
        self.bg_mode = background
        self.host_bg = host_bg
        bg = make_background(config)
        self.bg_spec = bg
        lam = background_lambda(topo, bg, config.dt)[self.lo:self.hi]
        self.lam = torch.from_numpy(np.ascontiguousarray(lam)).to(dev)
        self.seed = int(seed)
        self.bg_buf = torch.empty(max(1, self.n), dtype=self.td, device=dev)
        self.t = 0
        self.t_dev = torch.zeros(1, dtype=torch.int64, device=dev)   # step index for graph replay
        self._graphs = {}
        self.scratch = torch.empty(int(nat.load().hhb_spike_scratch(self.words_global * 32)), dtype=torch.int64,
                                   device=dev)

    THAL_SALT = 0x7468616C616D7573        # key of the thalamic Philox stream: seed ^ "thalamus"

    def set_thalamic(self, targets, weights, lam: float, t_on: int, t_off: int):
        """Thalamic drive drawn on the device (cortex.py:398-429): thalamic
        synapse k (targets[k], weights[k], the reference's _thalamic_setup
        table) fires at step t in [t_on, t_off) with probability lam, keyed
        by (seed, k, t) -- the same draws for any sharding and any of the
        eager / graph / persistent paths (hhb_thalamic_drive, hh_net).  Its
        current is added to that step's input only (not to the PSP), as
        step_network's extra_current."""
        targets = np.asarray(targets, dtype=np.int64)
        weights = np.asarray(weights, dtype=np.float64)
        if targets.shape != weights.shape or (targets.size and (targets.min() < 0 or targets.max() >= self.n_global)):
            raise UsageError("thalamic targets / weights must be matching arrays of global neuron ids")
        order = np.argsort(targets, kind="stable")
        goff = np.concatenate([[0], np.cumsum(np.bincount(targets, minlength=self.n_global))]).astype(np.int64)
        k0, k1 = int(goff[self.lo]), int(goff[self.hi])
        self.th_off = torch.from_numpy(goff[self.lo:self.hi + 1] - k0).to(self.dev)
        w = np.zeros(max(1, k1 - k0))
        w[:k1 - k0] = weights[order][k0:k1]
        self.th_w = torch.from_numpy(w).to(self.td).to(self.dev)
        thr = min(2 ** 32 - 1, int(math.floor(float(lam) * 2.0 ** 32)))
        self.thal = nat.Thalamic(self.th_off.data_ptr(), self.th_w.data_ptr(), k0, int(t_on), int(t_off), thr, 0,
                                 (self.seed ^ self.THAL_SALT) & (2 ** 64 - 1))
        self.thal_buf = torch.zeros(max(1, self.n), dtype=self.td, device=self.dev)
        self._graphs.clear()             # captured steps lack (or hold stale) thalamic launches

    def _thalamic(self, t_dev=None):
        nat.check(nat.load().hhb_thalamic_drive(D.code(self.dtype), self.n, self.t, D.ptr(t_dev), C.byref(self.thal),
                                                self.thal_buf.data_ptr(), D.stream()), "hhb_thalamic_drive")
        return self.thal_buf

    def _input(self, extra=None):
        lib = nat.load()
        mode = 0
        if self.bg_mode == "host":
            full = self.host_bg.sample()                    # advances the reference RNG for ALL neurons
            self.bg_buf.copy_(torch.from_numpy(np.ascontiguousarray(full[self.lo:self.hi])).to(self.td))
            mode = 1
        elif self.bg_mode == "philox" and self.bg_spec.rate_hz > 0:
            mode = 2
        ex = None if extra is None else D.to_dev(extra, self.dtype, self.dev)
        if getattr(self, "thal", None) is not None:
            th = self._thalamic()
            ex = th if ex is None else th + ex
        nat.check(lib.hhb_cortex_input(
            D.code(self.dtype), self.n, self.t, self.depth, self.ring.data_ptr(), self.psp.data_ptr(),
            self.decay, mode, self.bg_buf.data_ptr() if mode == 1 else None, self.lam.data_ptr(),
            self.bg_spec.w_mean,
            self.bg_spec.w_std, self.seed, self.lo, D.ptr(ex), self.cur.data_ptr(),
            float(1.0 / (1 << W_FRAC_BITS)), D.stream()), "hhb_cortex_input")

    def advance_local(self, extra=None) -> torch.Tensor:
        """Input + HH step of this rank's neurons; returns its bitmap words."""
        self._input(extra)
        _forward(self.params, self.v, self.g, self.cur[:self.n], 0, 1, 1, v_fin=self.v, g_fin=self.g,
                 bits=self.words.view(1, -1), step_base=self.t, first_bad=self.first_bad, reset_bad=False)
        return self.words

    def deliver(self, gwords: torch.Tensor):
        """Enqueue the synapses of every spiking source (global bitmap) whose
        target is local, then move to the next step."""
        nat.check(nat.load().hhb_spike_deliver_flat(
            self.words_global, gwords.data_ptr(), self.off.data_ptr(), self.tgt.data_ptr(),
            self.w.data_ptr(), self.delay.data_ptr(), self.t, None, self.depth, self.n, self.ring.data_ptr(),
            self.scratch.data_ptr(), D.stream()), "hhb_spike_deliver")
        self.t += 1

    def step(self, extra=None):
        """One network step (cortex.py:273-310); returns the global spike words."""
        words = self.advance_local(extra)
        if self.exchange is None:
            self.gwords[:self.words_global].copy_(words[:self.words_global])
        else:
            self.exchange(words, self.gwords)
        self.deliver(self.gwords)
        return self.gwords[:self.words_global]

    # ---------------------------------------------------------------- graphs
    def _step_dev(self):
        """One step whose step index lives in self.t_dev (capturable)."""
        lib = nat.load()
        mode = 2 if (self.bg_mode == "philox" and self.bg_spec.rate_hz > 0) else 0
        ex = self._thalamic(self.t_dev) if getattr(self, "thal", None) is not None else None
        nat.check(lib.hhb_cortex_input_dev(
            D.code(self.dtype), self.n, 0, self.t_dev.data_ptr(), self.depth, self.ring.data_ptr(),
            self.psp.data_ptr(), self.decay, mode, None, self.lam.data_ptr(), self.bg_spec.w_mean,
            self.bg_spec.w_std, self.seed, self.lo, D.ptr(ex), self.cur.data_ptr(),
            float(1.0 / (1 << W_FRAC_BITS)), D.stream()), "hhb_cortex_input_dev")
        _forward(self.params, self.v, self.g, self.cur[:self.n], 0, 1, 1, v_fin=self.v, g_fin=self.g,
                 bits=self.words.view(1, -1), step_base=0, first_bad=self.first_bad, reset_bad=False,
                 step_dev=self.t_dev)
        if isinstance(self.exchange, LibraryExchange):
            # the all-gather and the delivery in one C-ABI call (hhb_spk_step)
            nat.check(lib.hhb_spk_step(
                self.exchange.handle, self.words.data_ptr(), self.gwords.data_ptr(), self.words_global,
                self.off.data_ptr(), self.tgt.data_ptr(), self.w.data_ptr(), self.delay.data_ptr(), 0,
                self.t_dev.data_ptr(), self.depth, self.n, self.ring.data_ptr(), self.scratch.data_ptr(),
                D.stream()), "hhb_spk_step")
            nat.check(lib.hhb_cortex_tick(self.t_dev.data_ptr(), D.stream()), "hhb_cortex_tick")
            return self.gwords
        if self.exchange is None:
            gw = self.words            # one rank: the local bitmap is the global one (no copy)
        else:
            self.exchange(self.words, self.gwords)
            gw = self.gwords
        nat.check(lib.hhb_spike_deliver_flat(
            self.words_global, gw.data_ptr(), self.off.data_ptr(), self.tgt.data_ptr(),
            self.w.data_ptr(), self.delay.data_ptr(), 0, self.t_dev.data_ptr(), self.depth, self.n,
            self.ring.data_ptr(), self.scratch.data_ptr(), D.stream()), "hhb_spike_deliver_flat")
        nat.check(lib.hhb_cortex_tick(self.t_dev.data_ptr(), D.stream()), "hhb_cortex_tick")
        return gw

    def persistent_ok(self) -> bool:
        """Whether advance() runs the persistent kernel (hhb_cortex_run): one
        rank, float32 neurons, device (or no) background; HHB_NET_GRAPH=1
        forces the graph path."""
        import os
        return (self.exchange is None and self.world == 1 and self.dtype == np.float32 and self.n > 0
                and self.bg_mode != "host" and os.environ.get("HHB_NET_GRAPH", "0") in ("", "0"))

    def _tile_segments(self):
        """Sort every synapse row by target (delivery order does not change the
        int64 ring) and index, per row, the first synapse of each 256-neuron
        target tile: seg[s][k] for k = 0..tiles (hhb_cortex_run's layout)."""
        if getattr(self, "_seg", None) is None:
            dev = self.dev
            n_src = self.off.numel() - 1
            row = torch.repeat_interleave(torch.arange(n_src, device=dev), self.off[1:] - self.off[:-1])
            key = (row << 32) | self.tgt.long()
            del row
            key, perm = torch.sort(key, stable=True)
            # the arrays are replaced: graphs captured on the old pointers are stale
            self._graphs.clear()
            self.tgt = self.tgt[perm].contiguous()
            self.w = self.w[perm].contiguous()
            self.delay = self.delay[perm].contiguous()
            del perm
            tiles = (getattr(self, "n_pad", self.n) + 255) // 256    # replicas: padded populations
            q = (torch.arange(n_src, device=dev)[:, None] << 32) | (torch.arange(tiles + 1, device=dev) * 256)[None, :]
            self._seg = torch.searchsorted(key, q.reshape(-1)).reshape(n_src, tiles + 1).contiguous()
            self._tiles = tiles
        return self._seg, self._tiles

    def _advance_persistent(self, n_steps: int, record: torch.Tensor | None):
        """n_steps network steps in one cooperative launch (jit.cu hh_net)."""
        lib = nat.load()
        mode = 2 if (self.bg_mode == "philox" and self.bg_spec.rate_hz > 0) else 0
        W = self.words_global
        if record is not None:
            if (record.dtype != torch.int32 or not record.is_contiguous() or record.dim() != 2
                    or record.shape[0] < n_steps or record.shape[1] != W or record.device != self.v.device):
                raise UsageError(f"record must be a contiguous int32 [>= {n_steps}][{W}] tensor on {self.v.device}")
            bits, rec = record, 1
        else:
            if getattr(self, "_pingpong", None) is None:
                self._pingpong = torch.zeros((2, W), dtype=torch.int32, device=self.dev)
            bits, rec = self._pingpong, 0
        if getattr(self, "_barrier", None) is None:
            self._barrier = torch.zeros(1, dtype=torch.int32, device=self.dev)
        seg, tiles = self._tile_segments()
        P = _table(self.params)
        thal = getattr(self, "thal", None)
        rc = lib.hhb_cortex_run_ex(
            C.byref(P), self.n, n_steps, self.t, self.depth, self.ring.data_ptr(), self.psp.data_ptr(), self.decay,
            mode, self.lam.data_ptr(), self.bg_spec.w_mean, self.bg_spec.w_std, self.seed, self.lo,
            float(1.0 / (1 << W_FRAC_BITS)), self.v.data_ptr(), self.g.data_ptr() if self.g.numel() else None,
            self.n, bits.data_ptr(), rec, W, seg.data_ptr(), tiles, self.tgt.data_ptr(), self.w.data_ptr(),
            self.delay.data_ptr(), self.first_bad.data_ptr(), self._barrier.data_ptr(),
            D.ptr(getattr(self, "timing", None)), C.byref(thal) if thal is not None else None, D.stream())
        nat.check(rc, "hhb_cortex_run_ex")
        last = bits[n_steps - 1] if rec else bits[(n_steps - 1) & 1]
        self.words[:W].copy_(last[:W])
        self.t += n_steps
        self.t_dev.fill_(self.t)
        return record

    def advance(self, n_steps: int, steps_per_graph: int = 64, record: torch.Tensor | None = None,
                wait: bool = True):
        """Advance n_steps.  One rank with float32 neurons runs them in ONE
        persistent cooperative kernel (hhb_cortex_run: the phases of each step
        separated by grid barriers); otherwise a CUDA graph of
        `steps_per_graph` network steps (input, HH step, exchange, delivery,
        tick) is replayed, the per-step host work of `step()` (~5 launches)
        becoming one graph launch per steps_per_graph steps.  Both are
        bit-identical to `step()`.  record: optional int32
        [n_steps][words_global] device buffer receiving each step's global
        spike words.  Host-RNG background cannot run on the device (use
        step()).  With a LibraryExchange the call ends by waiting for the
        steps (NCCL error / timeout check) unless wait=False (then call
        exchange.wait() yourself)."""
        if self.bg_mode == "host":
            raise UsageError("advance(): the host background is drawn per step; use step()")
        if n_steps > 0 and self.persistent_ok() and not getattr(self, "_no_persist", False):
            try:
                return self._advance_persistent(n_steps, record)
            except NativeLibraryError as e:
                if "hh_net" not in str(e) and "unavailable" not in str(e):
                    raise
                self._no_persist = True          # too many tiles / no cooperative launch: graph path
        self.t_dev.fill_(self.t)
        S = max(1, min(int(steps_per_graph), n_steps)) if n_steps > 0 else 1
        done = 0
        rec_key = record is not None
        if n_steps >= S:
            key = (S, rec_key)
            if key not in self._graphs:
                buf = torch.empty((S, self.words_global), dtype=torch.int32, device=self.dev) if rec_key else None
                t0 = self.t_dev.clone()
                snap = (self.v.clone(), self.g.clone(), self.psp.clone(), self.ring.clone())
                self._step_dev()                  # warm-up outside capture (module load, allocations)
                self.t_dev.copy_(t0)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for k in range(S):
                        gw = self._step_dev()
                        if rec_key:
                            buf[k].copy_(gw[:self.words_global])
                # the capture did not run the steps; undo the warm-up step
                self.v.copy_(snap[0]); self.g.copy_(snap[1]); self.psp.copy_(snap[2]); self.ring.copy_(snap[3])
                self.t_dev.copy_(t0)
                self._graphs[key] = (g, buf)
            g, buf = self._graphs[key]
            while n_steps - done >= S:
                g.replay()
                if rec_key:
                    record[done:done + S].copy_(buf)
                done += S
        while done < n_steps:
            gw = self._step_dev()
            if rec_key:
                record[done].copy_(gw[:self.words_global])
            done += 1
        self.t += n_steps
        if wait and hasattr(self.exchange, "wait"):
            self.exchange.wait()        # NCCL async errors / a hung peer surface here (ExchangeError)
        return record

    def run(self, n_steps: int, record: bool = True):
        """Advance n_steps; returns (times_ms, neuron_ids) of the spikes of ALL
        neurons (the SpikeRecord arrays of cortex.py:422-438)."""
        rows = [] if record else None
        for _ in range(n_steps):
            g = self.step()
            if record:
                rows.append(g.clone())
        _raise_if_bad(self.first_bad)
        if not record:
            return None
        if n_steps == 0:
            return np.zeros(0), np.zeros(0, dtype=np.int64)
        t_idx, n_idx = spike_events(torch.stack(rows).contiguous(), self.n_global)
        return (t_idx + 1 + (self.t - n_steps)) * self.config.dt, n_idx


# ---------------------------------------------------------------------------
# the reference's step-level API (cortex.py:225-310) over the device network
# ---------------------------------------------------------------------------

def background_sample(lam_eff, mu: float, sigma: float, count, rng: np.random.Generator):
    """Compound-Poisson draw N mu + sigma sqrt(N) z, N ~ Poisson(lam_eff),
    with the reference's RNG call sequence (cortex.py:225-232): host NumPy, so a
    seeded run reproduces the reference's stream draw for draw."""
    n = rng.poisson(lam_eff, size=count)
    out = n * mu
    if sigma > 0:
        out = out + sigma * np.sqrt(n) * rng.standard_normal(count)
    return out


class SpikeBuffer:
    """Ring of per-step pending synaptic currents (cortex.py:238-256), on the
    device in int64 fixed point (weight quantum 2^-W_FRAC_BITS): sums commute,
    so any enqueue order gives the same ring.  `ring` (float64 numpy) is a
    read-only snapshot."""

    def __init__(self, depth: int, n_neurons: int, device=None, _ring: torch.Tensor | None = None):
        if depth < 1:
            raise ConfigurationError("ring depth must be >= 1")
        self.depth = depth
        dev = device or D.require_cuda()
        self._ring = _ring if _ring is not None else torch.zeros((depth, max(1, n_neurons)), dtype=torch.int64,
                                                                 device=dev)
        self.n = n_neurons

    @property
    def ring(self) -> np.ndarray:
        return self._ring[:, :self.n].cpu().numpy().astype(np.float64) / (1 << W_FRAC_BITS)

    def enqueue(self, t: int, targets, weights, delays):
        dev = self._ring.device
        tg = torch.as_tensor(np.asarray(targets, dtype=np.int64), device=dev)
        slots = (t + torch.as_tensor(np.asarray(delays, dtype=np.int64), device=dev)) % self.depth
        wq = torch.as_tensor(quantise_weights(np.asarray(weights, dtype=np.float64)).astype(np.int64), device=dev)
        self._ring.view(-1).index_add_(0, slots * self._ring.shape[1] + tg, wq)

    def drain(self, t: int) -> np.ndarray:
        row = self._ring[t % self.depth]
        arrived = row[:self.n].cpu().numpy().astype(np.float64) / (1 << W_FRAC_BITS)
        row.zero_()
        return arrived


class _OneShotBackground:
    """HostBackground stand-in feeding CortexNetwork one pre-drawn sample."""

    def __init__(self):
        self.value = None

    def sample(self):
        return self.value


class NetworkState:
    """The reference's NetworkState (cortex.py:259-264) backed by a device
    CortexNetwork: `neuron`, `psp` are host snapshots, `buffer` a view of the
    device ring, `t` the step counter."""

    def __init__(self, engine: "CortexNetwork"):
        self._engine = engine

    @property
    def t(self) -> int:
        return self._engine.t

    @property
    def neuron(self):
        from .dynamics import NeuronState
        e = self._engine
        return NeuronState(D.to_host(e.v, np.float64), D.to_host(e.g, np.float64))

    @property
    def psp(self) -> np.ndarray:
        return D.to_host(self._engine.psp, np.float64)

    @property
    def buffer(self) -> SpikeBuffer:
        e = self._engine
        return SpikeBuffer(e.depth, e.n, _ring=e.ring)


def init_network_state(topo: NetworkTopology, config: CortexConfig, device=None,
                       dtype=np.float64) -> NetworkState:
    """Rest state, zero PSP, empty ring (cortex.py:267-270); float64 neurons
    like the reference unless dtype says otherwise."""
    eng = CortexNetwork(topo, config, device=device, dtype=dtype, background="host", host_bg=_OneShotBackground())
    return NetworkState(eng)


def step_network(net: NetworkState, topo: NetworkTopology, background: BackgroundSpec | None,
                 config: CortexConfig, rng: np.random.Generator, params=None, workspace=None,
                 extra_current=0.0) -> np.ndarray:
    """One network step (cortex.py:273-310): drain the ring, decay the PSP,
    add the background (drawn from `rng` exactly as the reference does), the
    HH step, and the delivery of the new spikes -- on the device.  Returns the
    step's spikes (bool, n).  `params` replaces the neuron set of the state's
    config (the reference passes config.resolved_neuron()); `workspace` is
    accepted for signature compatibility (the device step needs none)."""
    eng = net._engine
    if params is not None:
        eng.params = params.with_(dtype=eng.dtype)
    n = topo.n_neurons
    if background is not None and background.rate_hz > 0:
        lam = background_lambda(topo, background, config.dt)
        eng.host_bg.value = background_sample(lam, background.w_mean, background.w_std, n, rng)
    else:
        eng.host_bg.value = np.zeros(n)
    extra = None
    if not (np.isscalar(extra_current) and extra_current == 0.0):
        extra = np.broadcast_to(np.asarray(extra_current, dtype=np.float64), (n,))
    words = eng.step(extra)
    bits = words[:eng.words_global].cpu().numpy().view(np.uint8)
    return np.unpackbits(bits, bitorder="little")[:n].astype(bool)


# ---------------------------------------------------------------------------
# run_network / SpikeRecord (cortex.py:319-464): the reference's driver and
# its output record, on the device network
# ---------------------------------------------------------------------------

@dataclass
class SpikeRecord:
    """Spike events plus per-population rate statistics (cortex.py:319-376)."""

    times_ms: np.ndarray
    neuron_ids: np.ndarray
    duration_ms: float
    warmup_ms: float
    topo: NetworkTopology

    def _mask(self, name: str, warm: bool = True):
        sl = self.topo.pop_slice(name)
        m = (self.neuron_ids >= sl.start) & (self.neuron_ids < sl.stop)
        if warm:
            m &= self.times_ms >= self.warmup_ms
        return sl, m

    def pop_rate(self, name: str) -> float:
        """Mean rate (Hz) per neuron over the post-warmup window."""
        sl, m = self._mask(name)
        window_s = (self.duration_ms - self.warmup_ms) / 1000.0
        return float(m.sum()) / (sl.stop - sl.start) / window_s

    def rate_quartiles(self, name: str):
        sl, m = self._mask(name)
        counts = np.bincount(self.neuron_ids[m] - sl.start, minlength=sl.stop - sl.start)
        window_s = (self.duration_ms - self.warmup_ms) / 1000.0
        return np.percentile(counts / window_s, [25, 50, 75])

    def isi_cv(self, name: str) -> float:
        """Mean ISI coefficient of variation over neurons with >= 3 spikes."""
        _, m = self._mask(name)
        ids, ts = self.neuron_ids[m], self.times_ms[m]
        cvs = []
        for nid in np.unique(ids):
            tt = np.sort(ts[ids == nid])
            if tt.size >= 3:
                isi = np.diff(tt)
                if isi.mean() > 0:
                    cvs.append(isi.std() / isi.mean())
        return float(np.mean(cvs)) if cvs else float("nan")

    def rate_histogram(self, name: str, bin_ms: float = 1.0):
        """(bin centers ms, rate Hz) over the full duration."""
        sl, m = self._mask(name, warm=False)
        edges = np.arange(0.0, self.duration_ms + bin_ms, bin_ms)
        hist, _ = np.histogram(self.times_ms[m], bins=edges)
        rate = hist / (sl.stop - sl.start) / (bin_ms / 1000.0)
        return 0.5 * (edges[:-1] + edges[1:]), rate

    def to_ndjson(self, path) -> None:
        """One event per line: {t_ms, pop, neuron} (cortex.py:369-376)."""
        import json
        pop_of = np.empty(self.topo.n_neurons, dtype=object)
        for p in self.topo.populations:
            pop_of[p.offset:p.offset + p.size] = p.name
        with open(path, "w") as f:
            for t, n in zip(self.times_ms, self.neuron_ids):
                f.write(json.dumps({"t_ms": round(float(t), 6), "pop": pop_of[n], "neuron": int(n)}) + "\n")


def _thalamic_setup(topo: NetworkTopology, thalamic: dict, duration_ms: float, dt: float, rng):
    """Thalamic targets/weights with the reference's RNG calls (cortex.py:401-423)."""
    if thalamic["t_on_ms"] + thalamic["duration_ms"] > duration_ms:
        raise UsageError("thalamic stimulus extends beyond the simulation")
    scale = topo.populations[0].size / conn.FULL_SIZES[0]
    n_thal = max(int(round(conn.N_THALAMUS * scale)), 1)
    tt, tw = [], []
    for pop_name, p in conn.THALAMIC_PROBS.items():
        sl = topo.pop_slice(pop_name)
        size = sl.stop - sl.start
        count = int(rng.binomial(n_thal * size, p))
        if count == 0:
            continue
        ids = rng.choice(n_thal * size, size=count, replace=False)
        tt.append(sl.start + (ids % size))
        tw.append(np.maximum(rng.normal(thalamic["weight"], thalamic.get("weight_std", 0.0), size=count), 0.0))
    targets = np.concatenate(tt) if tt else np.zeros(0, dtype=int)
    weights = np.concatenate(tw) if tw else np.zeros(0)
    lam = thalamic["rate_hz"] * dt / 1000.0
    lo = int(round(thalamic["t_on_ms"] / dt))
    hi = int(round((thalamic["t_on_ms"] + thalamic["duration_ms"]) / dt))
    return targets, weights, lam, lo, hi


def run_network(topo: NetworkTopology, config: CortexConfig, duration_ms: float, seed: int,
                warmup_ms: float = 0.0, thalamic: dict | None = None, background: str = "host",
                dtype=np.float64, device=None) -> SpikeRecord:
    """Simulate and collect spikes (cortex.py:379-438) on the device network.

    background="host" (default) draws the compound-Poisson background and the
    thalamic events from the reference's RNG stream (np.random.default_rng(seed),
    same call order), so a float64 run reproduces the reference raster;
    background="philox" draws the background and the thalamic events on the
    device (statistically the same processes, keyed by (seed, neuron, step)
    and (seed, synapse, step)) and runs every step in the persistent kernel
    (one GPU, float32) or 64-step CUDA graphs -- the throughput path."""
    rng = np.random.default_rng(seed)
    n_steps = int(round(duration_ms / config.dt))
    thal = None
    if thalamic is not None:
        thal = _thalamic_setup(topo, thalamic, duration_ms, config.dt, rng)
    if background == "host":
        hb = HostBackground(topo, make_background(config), config.dt, rng)
        net = CortexNetwork(topo, config, device=device, dtype=dtype, background="host", host_bg=hb)
    elif background == "philox":
        net = CortexNetwork(topo, config, device=device, dtype=dtype, background="philox", seed=seed)
    else:
        raise UsageError(f"unknown background {background!r}")
    rows = torch.empty((n_steps, net.words_global), dtype=torch.int32, device=net.dev)
    if background == "philox":
        # the thalamic events drawn on the device too (Philox keyed by (seed,
        # synapse, step)): every step in the persistent kernel / CUDA graphs
        if thal is not None:
            net.set_thalamic(thal[0], thal[1], thal[2], thal[3], thal[4])
        net.advance(n_steps, record=rows)
    else:
        for t in range(n_steps):
            extra = None
            if thal is not None and thal[3] <= t < thal[4] and thal[0].size:
                targets, weights, lam = thal[0], thal[1], thal[2]
                events = rng.random(targets.size) < lam
                if events.any():
                    extra = np.zeros(topo.n_neurons)
                    np.add.at(extra, targets[events], weights[events])
                    extra = extra[net.lo:net.hi]
            rows[t].copy_(net.step(extra))
    _raise_if_bad(net.first_bad)
    t_idx, n_idx = spike_events(rows, topo.n_neurons)
    return SpikeRecord((t_idx + 1) * config.dt, n_idx, duration_ms, warmup_ms, topo)


def spike_events(rows: torch.Tensor, n: int):
    """Device spike raster (int32 [steps][words]) -> (step, neuron) event
    arrays on the host, sorted by step then neuron (hhb_spike_event_counts /
    hhb_spike_events): only the events cross PCIe, not the raster."""
    lib = nat.load()
    T, W = rows.shape
    counts = torch.empty(max(1, T), dtype=torch.int64, device=rows.device)
    nat.check(lib.hhb_spike_event_counts(T, W, rows.data_ptr(), n, counts.data_ptr(), D.stream()), "spike events")
    ends = torch.cumsum(counts[:T], 0)
    total = int(ends[-1].item()) if T else 0
    offsets = ends - counts[:T]
    st = torch.empty(max(1, total), dtype=torch.int32, device=rows.device)
    nid = torch.empty(max(1, total), dtype=torch.int32, device=rows.device)
    nat.check(lib.hhb_spike_events(T, W, rows.data_ptr(), n, offsets.data_ptr(), st.data_ptr(), nid.data_ptr(),
                                   D.stream()), "spike events")
    return st[:total].cpu().numpy().astype(np.int64), nid[:total].cpu().numpy().astype(np.int64)


def rest_state_run(duration_ms: float, scale: float, seed: int, config: CortexConfig | None = None,
                   warmup_ms: float = 200.0, **kw) -> SpikeRecord:
    """Spontaneous-activity run with the rest-state parameter set (cortex.py:441-448)."""
    cfg = replace(config if config is not None else REST_CONFIG, scale=scale)
    topo = build_network(scale, seed, cfg)
    return run_network(topo, cfg, duration_ms, seed + 1, warmup_ms=warmup_ms, **kw)


def thalamic_stimulus_run(duration_ms: float, scale: float, seed: int, t_on_ms: float,
                          config: CortexConfig | None = None, warmup_ms: float = 200.0,
                          rate_hz: float | None = None, **kw) -> SpikeRecord:
    """Thalamic-transient run: weaker background, brief strong L4/L6 drive (cortex.py:451-464)."""
    cfg = replace(config if config is not None else THALAMIC_CONFIG, scale=scale)
    topo = build_network(scale, seed, cfg)
    thal = {"t_on_ms": t_on_ms, "duration_ms": conn.THALAMIC_DURATION_MS,
            "rate_hz": rate_hz if rate_hz is not None else conn.THALAMIC_RATE_HZ,
            "weight": cfg.bg_mean, "weight_std": cfg.bg_std}
    return run_network(topo, cfg, duration_ms, seed + 1, warmup_ms=warmup_ms, thalamic=thal, **kw)


class CortexReplicas:
    """`replicas` independent copies of one network on one GPU, stepped
    together ("replicas x speed"; SPEC's data-parallel batching):
    one input launch, one HH launch over replicas * n_pad neurons and one
    delivery launch per step for all of them, replayed as CUDA graphs.  Replica
    r draws the device background with seed + r and reproduces, bit for bit, a
    single `CortexNetwork(..., background="philox", seed=seed + r)` run.  The
    per-step cost of one network is launch-latency-bound; a batch fills the GPU."""

    def __init__(self, topo: NetworkTopology, config: CortexConfig, replicas: int, device=None,
                 dtype=np.float32, seed: int = 0):
        if replicas < 1:
            raise UsageError("replicas must be >= 1")
        self.topo, self.config, self.R = topo, config, int(replicas)
        self.dev = device or D.require_cuda()
        self.params = config.resolved_neuron().with_(dtype=dtype)
        self.dtype = np.dtype(dtype)
        self.td = D.torch_dtype(self.dtype)
        self.n = topo.n_neurons
        self.n_pad = (self.n + 31) // 32 * 32
        self.words = self.n_pad // 32
        self.depth = topo.max_delay + 1
        dev = self.dev
        off, tgt, w, d = local_synapses(topo, 0, self.n)
        self.off = torch.from_numpy(off).to(dev)
        self.tgt = torch.from_numpy(tgt).to(dev)
        self.w = torch.from_numpy(quantise_weights(w)).to(dev)
        self.delay = torch.from_numpy(d.astype(np.int32)).to(dev)
        NT = self.R * self.n_pad
        st = init_state(self.params, (NT,), device=dev)
        self.v, self.g = st.v.contiguous(), st.gates.contiguous()
        self.psp = torch.zeros(NT, dtype=self.td, device=dev)
        self.cur = torch.empty(NT, dtype=self.td, device=dev)
        self.ring = torch.zeros((self.R, self.depth, self.n_pad), dtype=torch.int64, device=dev)
        self.bits = torch.zeros(self.R * self.words, dtype=torch.int32, device=dev)
        lib = nat.load()
        self.scratch = torch.empty(self.R * int(lib.hhb_spike_scratch(self.n_pad)), dtype=torch.int64, device=dev)
        bg = make_background(config)
        self.bg = bg
        lam = np.zeros(self.n_pad)
        lam[:self.n] = background_lambda(topo, bg, config.dt)
        self.lam = torch.from_numpy(lam).to(dev)
        self.decay = math.exp(-config.dt / config.psp_tau_ms)
        self.seed = int(seed)
        self.first_bad = torch.full((1,), D.INT64_MAX, dtype=torch.int64, device=dev)
        self.t = 0
        self.t_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        self._graphs = {}

    def _phase(self, phase: int):
        nat.check(nat.load().hhb_cortex_step_batch(
            D.code(self.dtype), self.R, self.n_pad, self.words, self.t_dev.data_ptr(), self.depth,
            self.ring.data_ptr(), self.psp.data_ptr(), self.decay, self.lam.data_ptr(), self.bg.w_mean,
            self.bg.w_std, self.seed, self.cur.data_ptr(), float(1.0 / (1 << W_FRAC_BITS)), self.bits.data_ptr(),
            self.off.data_ptr(), self.tgt.data_ptr(), self.w.data_ptr(), self.delay.data_ptr(),
            self.scratch.data_ptr(), phase, D.stream()), "hhb_cortex_step_batch")

    def _step_dev(self):
        self._phase(0)
        _forward(self.params, self.v, self.g, self.cur, 0, 1, 1, v_fin=self.v, g_fin=self.g,
                 bits=self.bits.view(1, -1), step_base=0, first_bad=self.first_bad, reset_bad=False,
                 step_dev=self.t_dev)
        self._phase(1)
        nat.check(nat.load().hhb_cortex_tick(self.t_dev.data_ptr(), D.stream()), "hhb_cortex_tick")

    _tile_segments = CortexNetwork._tile_segments      # same attribute names (off, tgt, w, delay, n, dev)

    def persistent_ok(self) -> bool:
        """Replicas in the persistent kernel (groups of up to 16 per launch) are
        opt-in (HHB_NET_REPLICAS_PERSIST=1): a block stepping R replicas does R
        times the input, step and delivery work of its tile behind one barrier,
        and per replica-step that measured no better than the batched graph
        path, which fills the GPU with R x 38,586 neurons per launch (R = 4 at
        scale 0.5: 25.1 vs 25.3 µs per step over the same window)."""
        import os
        return (self.dtype == np.float32 and os.environ.get("HHB_NET_REPLICAS_PERSIST", "0") not in ("", "0")
                and os.environ.get("HHB_NET_GRAPH", "0") in ("", "0") and not getattr(self, "_no_persist", False))

    def _advance_persistent(self, n_steps: int, record: torch.Tensor | None):
        """All replicas n_steps in persistent launches of up to 16 replicas each
        (hhb_cortex_run_replicas): replica r is bit-identical to the graph path."""
        lib = nat.load()
        seg, tiles = self._tile_segments()
        Wd, R, npd = self.words, self.R, self.n_pad
        G = min(R, 16)
        mode = 2 if self.bg.rate_hz > 0 else 0
        if getattr(self, "_barrier", None) is None:
            self._barrier = torch.zeros(1, dtype=torch.int32, device=self.dev)
        P = _table(self.params)
        for r0 in range(0, R, G):
            g = min(G, R - r0)
            if record is not None:
                buf = torch.empty((n_steps, g, Wd), dtype=torch.int32, device=self.dev)
                rec = 1
            else:
                buf = torch.zeros((2, g, Wd), dtype=torch.int32, device=self.dev)
                rec = 0
            rc = lib.hhb_cortex_run_replicas(
                C.byref(P), g, npd, npd, n_steps, self.t, self.depth,
                self.ring[r0].data_ptr(), self.psp[r0 * npd:].data_ptr(), self.decay, mode, self.lam.data_ptr(),
                self.bg.w_mean, self.bg.w_std, self.seed + r0, 0, float(1.0 / (1 << W_FRAC_BITS)),
                self.v[r0 * npd:].data_ptr(), self.g[:, r0 * npd:].data_ptr() if self.g.numel() else None,
                R * npd, buf.data_ptr(), rec, Wd, seg.data_ptr(), tiles, self.tgt.data_ptr(), self.w.data_ptr(),
                self.delay.data_ptr(), self.first_bad.data_ptr(), self._barrier.data_ptr(),
                D.ptr(getattr(self, "timing", None)), D.stream())
            nat.check(rc, "hhb_cortex_run_replicas")
            if record is not None:
                record[:n_steps, r0:r0 + g].copy_(buf)
        self.t += n_steps
        self.t_dev.fill_(self.t)
        return record

    def advance(self, n_steps: int, steps_per_graph: int = 32, record: torch.Tensor | None = None):
        """Advance all replicas n_steps: float32 replicas in persistent
        launches (groups of <= 16 replicas), otherwise CUDA graphs of
        steps_per_graph steps.  record: optional int32
        [n_steps][replicas][n_pad/32] spike words."""
        if n_steps > 0 and self.persistent_ok():
            try:
                out = self._advance_persistent(n_steps, record)
                _raise_if_bad(self.first_bad)
                return out
            except NativeLibraryError as e:
                if "hh_net" not in str(e) and "unavailable" not in str(e):
                    raise
                self._no_persist = True
        self.t_dev.fill_(self.t)
        S = max(1, min(int(steps_per_graph), n_steps)) if n_steps > 0 else 1
        done, rec = 0, record is not None
        if n_steps >= S:
            key = (S, rec)
            if key not in self._graphs:
                buf = torch.empty((S, self.R * self.words), dtype=torch.int32, device=self.dev) if rec else None
                t0 = self.t_dev.clone()
                snap = (self.v.clone(), self.g.clone(), self.psp.clone(), self.ring.clone())
                self._step_dev()
                self.t_dev.copy_(t0)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for k in range(S):
                        self._step_dev()
                        if rec:
                            buf[k].copy_(self.bits)
                self.v.copy_(snap[0]); self.g.copy_(snap[1]); self.psp.copy_(snap[2]); self.ring.copy_(snap[3])
                self.t_dev.copy_(t0)
                self._graphs[key] = (g, buf)
            g, buf = self._graphs[key]
            while n_steps - done >= S:
                g.replay()
                if rec:
                    record[done:done + S].copy_(buf.view(S, self.R, self.words))
                done += S
        while done < n_steps:
            self._step_dev()
            if rec:
                record[done].copy_(self.bits.view(self.R, self.words))
            done += 1
        self.t += n_steps
        _raise_if_bad(self.first_bad)
        return record
