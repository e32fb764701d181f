"""CPU tests of the float32-contract machinery itself (tests/contract.py): the
per-neuron checks flag exactly the neurons that break them, and the
attribution explains a one-step spike shift across the horizon and a
reference-float32 disagreement, and leaves a genuine error unexplained."""

import numpy as np

from contract import attribute, check_against_oracle, neuron_failures
from oracle import hh_oracle as O
from paper_2601_21407_b200 import defaults as DF


def _run(n=6, T=2000, seed=0):
    p = DF.squid_axon_params(dt=0.02)
    rng = np.random.default_rng(seed)
    i = np.repeat(rng.uniform(5.0, 20.0, size=(1, n)), T + 2, 0)
    v, s = O.simulate(p, i)
    return p, i, v, s


def test_neuron_failures_flags_only_broken_neurons():
    p, i, v, s = _run()
    T = 2000
    v, s = v[:T], s[:T]
    fail, why = neuron_failures(v, s, v, s)
    assert not fail.any() and why == {}
    v2, s2 = v.copy(), s.copy()
    first = int(np.argmax(s[:, 1]))
    v2[first - 5, 1] += 1.0                      # pre-spike V violation
    j = int(np.flatnonzero(s[:, 2])[0])
    s2[j, 2], s2[j + 3, 2] = False, True          # a spike moved by 3 steps
    s2[:, 3] = False                              # count mismatch
    fail, why = neuron_failures(v2, s2, v, s)
    assert list(np.flatnonzero(fail)) == [1, 2, 3]
    assert "pre-spike V" in why[1] and "off by 3" in why[2] and "count" in why[3]


def test_attribution_categories():
    p, i, v_ext, s_ext = _run()
    T = 2000
    v, s = v_ext[:T], s_ext[:T]
    j = int(np.argmax(s.sum(0)))
    spikes = np.flatnonzero(s[:, j])
    assert spikes.size >= 2
    # a genuine error (a spike removed mid-run) is unexplained
    s_bad = s.copy()
    s_bad[spikes[1], j] = False
    rep = check_against_oracle(p, i[:T], v, s_bad, v, s)
    assert rep["failing"] == 1 and rep["unexplained"] == 1 and rep["listed"][0]["neuron"] == j
    # a window ending on a spike step, our spike one step later (past the
    # window): explained as a horizon-edge shift once both runs continue
    Tw = int(spikes[1]) + 1
    s_w = s[:Tw].copy()
    s_w[Tw - 1, j] = False
    s_ours_ext = s_ext[:Tw + 2].copy()
    s_ours_ext[Tw - 1, j], s_ours_ext[Tw, j] = False, True
    verdict = attribute(p, i[:Tw], [j], v[:Tw], s[:Tw],
                        ours_ext=lambda c: (v_ext[:Tw + 2, [j]], s_ours_ext[:, [j]]), i_ext=i[:Tw + 2])
    assert "horizon edge" in verdict[j], verdict[j]
