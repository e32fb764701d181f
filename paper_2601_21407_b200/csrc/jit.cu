// jit.cu -- runtime specialisation of the float kernels per channel table.
//
// The generic kernels in hh_kernels.cuh read the channel table from the
// kernel-parameter bank and branch on every rate kind and exponent at run
// time.  ncu on B200 (profiles/round1_fwd_generic.md) showed that this costs
// ~430 issued instructions per neuron-step for config 2 against 31 MUFU ops,
// plus instruction-cache misses from the 3-way unrolled code.  Here the same
// step is generated as CUDA source with every constant an immediate, every
// kind resolved and every power unrolled, compiled by NVRTC for sm_100a on
// first use of a table, and cached per (table, device) for the process.
//
// The generated module holds the forward kernel (1 and 4 neurons per thread)
// and the backward kernel; both call the same generated step function, so
// the backward's segment recompute reproduces the forward's checkpoints bit
// for bit.  NVRTC is loaded with dlopen and the driver API through
// cudaGetDriverEntryPoint, so the library still loads on hosts without a GPU.
// HHB_NO_JIT=1 forces the generic kernels.
#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <cctype>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "hh_host.cuh"

namespace hhb {
namespace jit {

// ------------------------------------------------------------ loaders
struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  bool ok = false;
  std::string why;
};

struct Driver {
  decltype(&cuModuleLoadData) load = nullptr;
  decltype(&cuModuleGetFunction) get = nullptr;
  decltype(&cuLaunchKernel) launch = nullptr;
  decltype(&cuLaunchCooperativeKernel) coop = nullptr;                        // optional
  decltype(&cuOccupancyMaxActiveBlocksPerMultiprocessor) occupancy = nullptr;  // optional
  decltype(&cuFuncSetAttribute) set_attr = nullptr;                           // optional
  decltype(&cuLaunchKernelEx) launch_ex = nullptr;                            // optional (PDL)
  bool ok = false;
  std::string why;
};

static std::mutex g_mu;
static Nvrtc g_nv;
static Driver g_drv;
static bool g_loaded = false;
static std::string g_status = "not initialised";

// cuLaunchKernel with the programmatic-stream-serialization attribute (pdl.cuh)
static CUresult launch_pdl_drv(CUfunction f, unsigned gx, unsigned bx, CUstream st, void** params) {
  if (!g_drv.launch_ex || !hhb::pdl_enabled()) return g_drv.launch(f, gx, 1, 1, bx, 1, 1, 0, st, params, nullptr);
  CUlaunchConfig cfg{};
  cfg.gridDimX = gx;
  cfg.gridDimY = cfg.gridDimZ = 1;
  cfg.blockDimX = bx;
  cfg.blockDimY = cfg.blockDimZ = 1;
  cfg.sharedMemBytes = 0;
  cfg.hStream = st;
  CUlaunchAttribute attr[1];
  attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
  attr[0].value.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return g_drv.launch_ex(&cfg, f, params, nullptr);
}

template <typename F>
static bool sym(void* h, const char* name, F& out) {
  out = reinterpret_cast<F>(dlsym(h, name));
  return out != nullptr;
}

static void load_libs() {
  if (g_loaded) return;
  g_loaded = true;
  const char* cands[] = {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12",
                         "/usr/local/cuda/lib64/libnvrtc.so", "libnvrtc.so"};
  void* h = nullptr;
  for (const char* c : cands) {
    h = dlopen(c, RTLD_NOW | RTLD_LOCAL);
    if (h) break;
  }
  if (!h) {
    g_nv.why = "libnvrtc.so.12 not found";
  } else {
    g_nv.ok = sym(h, "nvrtcCreateProgram", g_nv.create) && sym(h, "nvrtcCompileProgram", g_nv.compile) &&
              sym(h, "nvrtcGetCUBINSize", g_nv.cubin_size) && sym(h, "nvrtcGetCUBIN", g_nv.cubin) &&
              sym(h, "nvrtcGetProgramLogSize", g_nv.log_size) && sym(h, "nvrtcGetProgramLog", g_nv.log) &&
              sym(h, "nvrtcDestroyProgram", g_nv.destroy);
    if (!g_nv.ok) g_nv.why = "libnvrtc symbols missing";
  }
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  bool ok = true;
  ok = ok && cudaGetDriverEntryPoint("cuModuleLoadData", &p, cudaEnableDefault, &q) == cudaSuccess && p;
  g_drv.load = reinterpret_cast<decltype(g_drv.load)>(p);
  ok = ok && cudaGetDriverEntryPoint("cuModuleGetFunction", &p, cudaEnableDefault, &q) == cudaSuccess && p;
  g_drv.get = reinterpret_cast<decltype(g_drv.get)>(p);
  ok = ok && cudaGetDriverEntryPoint("cuLaunchKernel", &p, cudaEnableDefault, &q) == cudaSuccess && p;
  g_drv.launch = reinterpret_cast<decltype(g_drv.launch)>(p);
  if (cudaGetDriverEntryPoint("cuLaunchCooperativeKernel", &p, cudaEnableDefault, &q) == cudaSuccess && p)
    g_drv.coop = reinterpret_cast<decltype(g_drv.coop)>(p);
  if (cudaGetDriverEntryPoint("cuOccupancyMaxActiveBlocksPerMultiprocessor", &p, cudaEnableDefault, &q) ==
          cudaSuccess && p)
    g_drv.occupancy = reinterpret_cast<decltype(g_drv.occupancy)>(p);
  if (cudaGetDriverEntryPoint("cuFuncSetAttribute", &p, cudaEnableDefault, &q) == cudaSuccess && p)
    g_drv.set_attr = reinterpret_cast<decltype(g_drv.set_attr)>(p);
  if (cudaGetDriverEntryPoint("cuLaunchKernelEx", &p, cudaEnableDefault, &q) == cudaSuccess && p)
    g_drv.launch_ex = reinterpret_cast<decltype(g_drv.launch_ex)>(p);
  g_drv.ok = ok;
  if (!ok) g_drv.why = "driver entry points unavailable";
}

// ------------------------------------------------------------ codegen
static std::string fmt(const char* f, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  return buf;
}

// exact float literal (hex) of a double constant rounded to float
static std::string F(double x) {
  const float f = float(x);
  if (!std::isfinite(f)) return f > 0 ? "__int_as_float(0x7f800000)" : "__int_as_float(0xff800000)";
  char buf[64];
  snprintf(buf, sizeof buf, "%af", double(f));
  return std::string("(") + buf + ")";
}

// How a step variant treats the linoid's removable singularity:
//   kFast   -- direct formula only (the kernel proved no lane of the warp is
//              within |x/b| < 1/2 of any linoid's v0 this step)
//   kSeries -- direct formula with the Bernoulli series selected per lane
// Both give identical bits on lanes outside the series region, so which
// variant a warp ran never changes a neuron's result.
enum SeriesMode { kFast = 0, kSeries = 1 };

// One rate: value (and slope) of kind(a, v0, b) * scale at `v`.
static void emit_rate(std::string& o, const hhb_rate_t& r, double scale, const std::string& val,
                      const std::string* slope, SeriesMode mode) {
  const double A = r.a * scale, K2 = -kLog2e / r.b;
  o += "  {\n";
  if (r.kind == HHB_RATE_EXP && A > 0) {
    // a*2^y = 2^(y + log2 a): the amplitude rides in the exponent (one FMUL less)
    o += fmt("    %s = ex2f_(__fmaf_rn(v, %s, %s));\n", val.c_str(), F(K2).c_str(),
             F(-r.v0 * K2 + std::log2(A)).c_str());
    if (slope) o += fmt("    %s = __fmul_rn(%s, %s);\n", slope->c_str(), F(-1.0 / r.b).c_str(), val.c_str());
  } else if (r.kind == HHB_RATE_EXP || r.kind == HHB_RATE_SIGMOID) {
    o += fmt("    const float e = ex2f_(__fmaf_rn(v, %s, %s));\n", F(K2).c_str(), F(-r.v0 * K2).c_str());
    if (r.kind == HHB_RATE_EXP) {
      o += fmt("    %s = __fmul_rn(%s, e);\n", val.c_str(), F(A).c_str());
      if (slope) o += fmt("    %s = __fmul_rn(%s, %s);\n", slope->c_str(), F(-1.0 / r.b).c_str(), val.c_str());
    } else {
      o += "    const float q = rcpf_(__fadd_rn(1.0f, e));\n";
      o += fmt("    %s = __fmul_rn(%s, q);\n", val.c_str(), F(A).c_str());
      if (slope)
        o += fmt("    %s = __fmul_rn(__fmul_rn(%s, %s), __fsub_rn(1.0f, q));\n", slope->c_str(), val.c_str(),
                 F(1.0 / r.b).c_str());
    }
  } else {
    // linoid a*x/(1-exp(-x/b)); its Bernoulli series where |x/b| < 1/2
    o += fmt("    const float x = __fsub_rn(v, %s);\n", F(r.v0).c_str());
    o += fmt("    const float e = ex2f_(__fmul_rn(x, %s));\n", F(K2).c_str());
    o += "    const float den = __fsub_rn(1.0f, e);\n";
    o += "    const float rd = rcpf_(den);\n";
    o += fmt("    %s = __fmul_rn(__fmul_rn(%s, x), rd);\n", val.c_str(), F(A).c_str());
    if (slope)
      o += fmt("    %s = __fmul_rn(__fmul_rn(%s, __fsub_rn(den, __fmul_rn(__fmul_rn(x, %s), e))), "
               "__fmul_rn(rd, rd));\n",
               slope->c_str(), F(A).c_str(), F(1.0 / r.b).c_str());
    if (mode == kFast) {
      o += "  }\n";
      return;
    }
    o += fmt("    const bool sm = fabsf(x) < %s;\n", F(0.5 * std::fabs(r.b)).c_str());
    o += "    {\n";
    o += fmt("      const float u = __fmul_rn(x, %s);\n", F(1.0 / r.b).c_str());
    o += "      const float w = __fmul_rn(u, u);\n";
    o += "      float f = __fmaf_rn(w, -8.267195767195767e-07f, 3.3068783068783070e-05f);\n";
    o += "      f = __fmaf_rn(w, f, -1.3888888888888889e-03f);\n";
    o += "      f = __fmaf_rn(w, f, 8.3333333333333333e-02f);\n";
    o += "      f = __fmaf_rn(w, f, __fmaf_rn(u, 0.5f, 1.0f));\n";
    o += fmt("      %s = sm ? __fmul_rn(%s, f) : %s;\n", val.c_str(), F(r.a * r.b * scale).c_str(), val.c_str());
    if (slope) {
      o += "      float d = __fmaf_rn(w, 2.0876756987868099e-07f, -6.6137566137566138e-06f);\n";
      o += "      d = __fmaf_rn(w, d, 1.9841269841269841e-04f);\n";
      o += "      d = __fmaf_rn(w, d, -5.5555555555555556e-03f);\n";
      o += "      d = __fmaf_rn(w, d, 1.6666666666666667e-01f);\n";
      o += "      d = __fmaf_rn(u, d, 0.5f);\n";
      o += fmt("      %s = sm ? __fmul_rn(%s, d) : %s;\n", slope->c_str(), F(A).c_str(), slope->c_str());
    }
    o += "    }\n";
  }
  o += "  }\n";
}

static std::string pow_expr(const std::string& p, int k) {
  if (k == 0) return "1.0f";
  std::string e = p;
  for (int i = 1; i < k; ++i) e = "__fmul_rn(" + e + ", " + p + ")";
  return e;
}

struct Layout {
  int ng = 0;
  std::vector<int> first, last, chan;
  std::vector<int> leak_ch;
  double gl = 0, gle = 0;
};

static Layout layout_of(const hhb_params_t* P) {
  Layout L;
  L.ng = P->n_gates;
  L.first.assign(L.ng, 0);
  L.last.assign(L.ng, 0);
  L.chan.assign(L.ng, 0);
  for (int c = 0; c < P->n_channels; ++c) {
    const hhb_channel_t& C = P->channels[c];
    if (C.gate_count == 0) {
      L.leak_ch.push_back(c);
      L.gl += C.g_max;
      L.gle += C.g_max * C.e_rev;
      continue;
    }
    for (int g = C.gate_begin; g < C.gate_begin + C.gate_count; ++g) {
      L.first[g] = g == C.gate_begin;
      L.last[g] = g == C.gate_begin + C.gate_count - 1;
      L.chan[g] = c;
    }
  }
  return L;
}

// near_linoid(v): is v inside the series region |v - v0| < |b|/2 of any linoid rate?
static std::string emit_near_linoid(const hhb_params_t* P) {
  std::string o = "__device__ __forceinline__ bool near_linoid(const float v) {\n  bool n = false;\n";
  for (int g = 0; g < P->n_gates; ++g)
    for (const hhb_rate_t* r : {&P->gates[g].alpha, &P->gates[g].beta})
      if (r->kind == HHB_RATE_LINOID)
        o += fmt("  n = n || (fabsf(__fsub_rn(v, %s)) < %s);\n", F(r->v0).c_str(), F(0.5 * std::fabs(r->b)).c_str());
  return o + "  return n;\n}\n";
}

// step_fwd_<f|s>(v, p[], cur) -> v' ; p[] updated in place (hh_step, dynamics.py:472-528)
static std::string emit_forward_step(const hhb_params_t* P, const Layout& L, SeriesMode mode) {
  std::string o;
  const int NG = L.ng;
  o += fmt("__device__ __forceinline__ float step_fwd_%s(const float v, float (&p)[%d], const float cur) {\n",
           mode == kFast ? "f" : "s", NG > 0 ? NG : 1);
  o += L.leak_ch.empty() ? "  float ion = 0.0f;\n"
                         : fmt("  float ion = __fmaf_rn(%s, v, %s);\n", F(L.gl).c_str(), F(-L.gle).c_str());
  o += "  float eta = 1.0f;\n";
  for (int g = 0; g < NG; ++g) {
    const hhb_gate_t& G = P->gates[g];
    const hhb_channel_t& C = P->channels[L.chan[g]];
    o += fmt("  // gate %d (channel %d), exponent %d\n  {\n", g, L.chan[g], G.exponent);
    const std::string pg = fmt("p[%d]", g);
    o += "  const float pk = " + pow_expr(pg, G.exponent) + ";\n";
    o += L.first[g] ? "  eta = pk;\n" : "  eta = __fmul_rn(eta, pk);\n";
    o += "  float a, b;\n";
    emit_rate(o, G.alpha, P->rate_scale, "a", nullptr, mode);
    emit_rate(o, G.beta, P->rate_scale, "b", nullptr, mode);
    o += "  const float s = __fadd_rn(a, b);\n";
    o += "  const float pinf = __fmul_rn(a, rcpf_(s));\n";
    o += fmt("  const float dec = ex2f_(__fmul_rn(s, %s));\n", F(-P->dt * kLog2e).c_str());
    o += fmt("  const float pn = __fmaf_rn(__fsub_rn(%s, pinf), dec, pinf);\n", pg.c_str());
    o += fmt("  %s = (s == 0.0f) ? %s : pn;\n", pg.c_str(), pg.c_str());
    if (L.last[g])
      o += fmt("  ion = __fmaf_rn(__fmul_rn(eta, %s), __fsub_rn(v, %s), ion);\n", F(C.g_max).c_str(),
               F(C.e_rev).c_str());
    o += "  }\n";
  }
  o += fmt("  return __fmaf_rn(__fsub_rn(cur, ion), %s, v);\n}\n", F(P->dt / P->c_m).c_str());
  return o;
}

// ------------------------------------------------------------ merged step
// The MUFU pipe (16 ops/clk/SM) bounds the step above: config 2 needs 12 rate
// exps, 6 decay exps and 13 reciprocals per neuron-step.  The merged form
// spends fewer of them on the same arithmetic:
//  * rates whose slopes |b| are equal share one exponential: with
//    E = exp(-(v - vc)/b_g), a rate of slope +b_g needs c * E and one of slope
//    -b_g needs c' / E (c, c' constants); the reciprocal never materialises
//    because every rate is kept as a fraction n / d;
//  * a gate's two fractions merge: s = a + b = N / D and p_inf = a / s = A / N
//    with A = n_a d_b, N = A + n_b d_a, D = d_a d_b, and one reciprocal
//    r = 1 / (N D) serves both divisions (1/D = N r, 1/N = D r);
//  * -dt*log2(e) (and rate_scale) are folded into the numerators, so N / D is
//    the exp2 argument of the decay factor directly.
// Config 2: 8 shared exps + 6 decay exps + 6 reciprocals = 20 MUFU ops.
//
// The algebra is exact; what changes is rounding (a few ulp) and the range of
// the intermediates, so the host analyses the step in double over a voltage
// grid: one reciprocal per gate where N * D stays inside [2^-100, 2^100], two
// where only N and D do; the window [lo, hi] around v_rest where every
// intermediate is in range becomes a per-lane predicate.  Lanes outside it
// take the direct form (step_fwd_s), selected per lane, so a neuron's result
// depends only on its own state -- never on which warp-variant ran.
// A linoid's removable singularity: where |d| < 1/8 (|x/b| < ~0.13) the
// fraction is replaced per lane by (a b (1 + u/2 + u^2/12), 1), u = x/b,
// whose truncation error (u^4/720) is below float rounding there.
namespace mg {

constexpr double kRangeLo = 0x1p-100, kRangeHi = 0x1p100;
constexpr double kSingThr = 0.125;

struct Group {
  double b;       // signed slope of the first member; E = exp(-(v - vc) / b)
  double vc;
  int members = 0;
};

struct RatePlan {
  int kind;
  int group;
  int sigma;      // +1: e_r = c E ; -1: e_r = c / E
  double c;
  double Sa;      // a * rate_scale * (-dt log2 e)
  double v0, b;
  bool direct;    // single-member exp: value = sign(Sa) * ex2(v K2 + C + log2|Sa|)
  bool rational() const { return !(kind == HHB_RATE_EXP && sigma > 0); }
};

struct GatePlan {
  RatePlan a, b;
  bool one_rcp = true;
};

struct Plan {
  bool ok = false;
  std::string why;
  std::vector<Group> groups;
  std::vector<GatePlan> gates;
  double lo = 0, hi = 0;   // regular window
};

static bool inrange(double x) {
  const double a = std::fabs(x);
  return a >= kRangeLo && a <= kRangeHi && std::isfinite(x);
}

// exp argument of group g at v (what the kernel feeds ex2)
static double group_E(const Group& g, double v) { return std::exp(-(v - g.vc) / g.b); }

// emulate one rate at v in double, exactly as emitted: returns (n, d) of the
// selected fraction or the plain value (d = 1, plain = true); ok &= ranges
static void rate_nd(const RatePlan& r, const std::vector<Group>& G, double v, double& n, double& d, bool& ok) {
  const double E = group_E(G[r.group], v);
  ok = ok && inrange(E);
  const double x = v - r.v0;
  switch (r.kind) {
    case HHB_RATE_EXP:
      if (r.sigma > 0) { n = r.Sa * r.c * E; d = 1.0; }
      else { n = r.Sa * r.c; d = E; }
      break;
    case HHB_RATE_SIGMOID:
      if (r.sigma > 0) { n = r.Sa; d = r.c * E + 1.0; }
      else { n = r.Sa * E; d = E + r.c; }
      break;
    default: {  // linoid
      double thr;
      if (r.sigma > 0) { n = r.Sa * x; d = 1.0 - r.c * E; thr = kSingThr; }
      else { n = r.Sa * x * E; d = E - r.c; thr = kSingThr * r.c; }
      if (std::fabs(d) < thr) {
        const double u = x / r.b;
        n = r.Sa * r.b * (1.0 + u * (0.5 + u / 12.0));
        d = 1.0;
      }
    }
  }
  ok = ok && inrange(n) && inrange(d);
}

// reference value of a rate in double (dynamics.py:56-65), times Sa / a
static double rate_ref(const RatePlan& r, double v) {
  const double x = v - r.v0;
  const double e = std::exp(-x / r.b);
  const double a = r.Sa;
  if (r.kind == HHB_RATE_EXP) return a * e;
  if (r.kind == HHB_RATE_SIGMOID) return a / (1.0 + e);
  if (std::fabs(x / r.b) < 1e-6) return a * r.b;
  return a * x / (1.0 - e);
}

// is the merged gate computation valid at v (ranges + agreement with the
// direct formulas)?
static bool gate_ok(const GatePlan& g, const std::vector<Group>& G, double v, bool one_rcp) {
  bool ok = true;
  double na, da, nb, db;
  rate_nd(g.a, G, v, na, da, ok);
  rate_nd(g.b, G, v, nb, db, ok);
  const double A = na * db, N = nb * da + A, D = da * db;
  ok = ok && inrange(A) && inrange(N) && inrange(D);
  if (one_rcp) ok = ok && inrange(N * D) && inrange(1.0 / (N * D)) && inrange(N / (N * D)) && inrange(D / (N * D));
  else ok = ok && inrange(1.0 / N) && inrange(1.0 / D);
  if (!ok) return false;
  const double s = N / D, pinf = A / N;
  if (!(s < 0.0)) return false;   // scaled by -dt log2(e): the reference's s > 0 branch
  const double ra = rate_ref(g.a, v), rb = rate_ref(g.b, v);
  const double s_ref = ra + rb, pinf_ref = ra / s_ref;
  return std::fabs(s - s_ref) <= 1e-6 * std::fabs(s_ref) && std::fabs(pinf - pinf_ref) <= 1e-6 * std::fabs(pinf_ref) + 1e-12;
}

// largest [lo, hi] around v_rest (grid 1/64 mV, up to +-400 mV) where pred holds
template <typename F>
static void window(double vr, F pred, double& lo, double& hi) {
  const double h = 1.0 / 64;
  lo = hi = vr;
  if (!pred(vr)) { lo = hi = NAN; return; }
  for (double v = vr; v >= vr - 400.0 && pred(v); v -= h) lo = v;
  for (double v = vr; v <= vr + 400.0 && pred(v); v += h) hi = v;
}

static Plan plan_of(const hhb_params_t* P) {
  Plan M;
  const double S = P->rate_scale * (-P->dt * kLog2e);
  if (!(S < 0.0) || !std::isfinite(S)) { M.why = "rate_scale * dt must be positive"; return M; }
  // groups by |b|
  auto group_of = [&](const hhb_rate_t& r) -> int {
    for (size_t i = 0; i < M.groups.size(); ++i)
      if (std::fabs(M.groups[i].b) == std::fabs(r.b)) return int(i);
    Group g;
    g.b = r.b;
    g.vc = r.v0;
    M.groups.push_back(g);
    return int(M.groups.size() - 1);
  };
  for (int gi = 0; gi < P->n_gates; ++gi)
    for (const hhb_rate_t* r : {&P->gates[gi].alpha, &P->gates[gi].beta}) {
      if (r->a == 0.0 || !std::isfinite(r->a) || !std::isfinite(r->b) || !std::isfinite(r->v0)) {
        M.why = "zero or non-finite rate parameter";
        return M;
      }
      const int g = group_of(*r);
      Group& G = M.groups[g];
      ++G.members;
      // a linoid centres the group on its own singularity (smallest exp
      // argument, so the least rounding where 1 - e cancels)
      if (r->kind == HHB_RATE_LINOID && G.members == 1) G.vc = r->v0;
    }
  for (int gi = 0; gi < P->n_gates; ++gi) {
    GatePlan gp;
    for (int w = 0; w < 2; ++w) {
      const hhb_rate_t& r = w ? P->gates[gi].beta : P->gates[gi].alpha;
      RatePlan rp;
      rp.kind = r.kind;
      rp.group = group_of(r);
      const Group& G = M.groups[rp.group];
      rp.sigma = (r.b == G.b) ? 1 : -1;
      rp.c = rp.sigma > 0 ? std::exp((r.v0 - G.vc) / G.b) : std::exp((G.vc - r.v0) / G.b);
      rp.Sa = r.a * S;
      rp.v0 = r.v0;
      rp.b = r.b;
      rp.direct = r.kind == HHB_RATE_EXP && rp.sigma > 0 && G.members == 1;
      (w ? gp.b : gp.a) = rp;
    }
    M.gates.push_back(gp);
  }
  const double vr = P->v_rest;
  for (auto& g : M.gates) {
    double lo1, hi1;
    window(vr, [&](double v) { return gate_ok(g, M.groups, v, true); }, lo1, hi1);
    g.one_rcp = lo1 <= vr - 60.0 && hi1 >= vr + 140.0;
  }
  // One reciprocal per gate costs 4 issue slots and 1 MUFU op, two cost 2 and
  // 2.  With half of the gates on two reciprocals the first stream-specialised
  // forward sat at 0.80 of the MUFU peak, so every gate whose own window
  // allows it takes one (config 2: 1.60e11 -> 1.68e11 neuron-steps/s; before
  // the specialisation, issue-bound, half-and-half had won: 1.466e11 ->
  // 1.501e11).  The backward is far more issue-bound than MUFU-bound, so all
  // its gates take two (the window proven above holds for both: two
  // reciprocals only need N and D in range).  HHB_JIT_TWO_RCP=k moves the
  // last k forward gates to two.
  {
    int k = 0;
    if (const char* tr = getenv("HHB_JIT_TWO_RCP")) k = atoi(tr);
    for (int gi = int(M.gates.size()) - 1; gi >= 0 && k > 0; --gi, --k) M.gates[gi].one_rcp = false;
  }
  window(vr, [&](double v) {
    for (const auto& g : M.gates)
      if (!gate_ok(g, M.groups, v, g.one_rcp)) return false;
    return true;
  }, M.lo, M.hi);
  if (!(M.lo <= vr - 30.0 && M.hi >= vr + 100.0)) {
    M.why = "merged-form window too narrow";
    return M;
  }
  M.ok = true;
  return M;
}

static bool disabled() {
  const char* e = getenv("HHB_JIT_NOMERGE");
  return e && e[0] && e[0] != '0';
}

// shared exponentials (independent MUFU ops, issued back to back)
// poly: the first `poly` shared exponentials go to the FMA pipe (ex2p_, a
// degree-6 polynomial, 1.3 ulp -- below MUFU.EX2's ~2) instead of MUFU; the
// forward step only, where MUFU is the binding pipe (HHB_JIT_POLY_EXP)
static std::string emit_exps(const Plan& M, int poly = 0) {
  std::string o;
  std::vector<int> direct_only(M.groups.size(), 1);
  for (const auto& g : M.gates)
    for (const RatePlan* r : {&g.a, &g.b})
      if (!r->direct) direct_only[r->group] = 0;
  for (size_t i = 0; i < M.groups.size(); ++i) {
    if (direct_only[i]) continue;
    const double K2 = -kLog2e / M.groups[i].b;
    o += fmt("  const float E%d = %s(__fmaf_rn(v, %s, %s));\n", int(i), poly-- > 0 ? "ex2p_" : "ex2f_", F(K2).c_str(),
             F(-M.groups[i].vc * K2).c_str());
  }
  return o;
}

// symbolic float expression that knows when it is identically zero (the
// compiler may not fold x * 0.0f: x could be inf or NaN)
struct X {
  std::string e;
  bool zero = false;
};
static X Z() { return X{"0.0f", true}; }
static X V(const std::string& e) { return X{e, false}; }
static X mulx(const X& a, const X& b) { return (a.zero || b.zero) ? Z() : V("__fmul_rn(" + a.e + ", " + b.e + ")"); }
static X addx(const X& a, const X& b) {
  if (a.zero) return b;
  if (b.zero) return a;
  return V("__fadd_rn(" + a.e + ", " + b.e + ")");
}
static X fmax_(const X& a, const X& b, const X& c) {
  if (a.zero || b.zero) return c;
  if (c.zero) return mulx(a, b);
  return V("__fmaf_rn(" + a.e + ", " + b.e + ", " + c.e + ")");
}
static X negx(const X& a) { return a.zero ? a : V("(-" + a.e + ")"); }
// bind an expression to a named const (keeps the emitted source readable)
static X bind(std::string& o, const std::string& name, const X& x) {
  if (x.zero) return x;
  o += "  const float " + name + " = " + x.e + ";\n";
  return V(name);
}

// one rate of the backward: value (v) and V-slope (v1) as a plain number, or
// a fraction n / d with slopes n1, d1 (E' = -E / b_g)
struct RateX {
  bool rat;
  X v, v1, n, d, n1, d1;
};
static RateX emit_rate_bwd(std::string& o, const RatePlan& r, const std::vector<Group>& G, const char* nm) {
  RateX R;
  const double l2 = 1.0;   // slope scale (the decay term applies ln2 to s' itself)
  const std::string E = fmt("E%d", r.group);
  const double bg = G[r.group].b;
  const std::string w(nm);
  if (r.kind == HHB_RATE_EXP && r.sigma > 0) {
    R.rat = false;
    if (r.direct) {
      const double K2 = -kLog2e / r.b;
      R.v = bind(o, w + "v", V(std::string(r.Sa < 0 ? "(-" : "(") + fmt("ex2f_(__fmaf_rn(v, %s, %s)))", F(K2).c_str(),
                   F(-r.v0 * K2 + std::log2(std::fabs(r.Sa))).c_str())));
    } else {
      R.v = bind(o, w + "v", mulx(V(F(r.Sa * r.c)), V(E)));
    }
    R.v1 = bind(o, w + "v1", mulx(R.v, V(F(-l2 / r.b))));
    return R;
  }
  R.rat = true;
  switch (r.kind) {
    case HHB_RATE_EXP:  // sigma < 0: n = Sa c, d = E
      R.n = V(F(r.Sa * r.c));
      R.d = V(E);
      R.n1 = Z();
      R.d1 = bind(o, w + "d1", mulx(V(E), V(F(-l2 / bg))));
      break;
    case HHB_RATE_SIGMOID:
      if (r.sigma > 0) {
        R.n = V(F(r.Sa));
        R.d = bind(o, w + "d", V(fmt("__fmaf_rn(%s, %s, 1.0f)", F(r.c).c_str(), E.c_str())));
        R.n1 = Z();
        R.d1 = bind(o, w + "d1", V(fmt("__fmul_rn(%s, %s)", F(-l2 * r.c / bg).c_str(), E.c_str())));
      } else {
        R.n = bind(o, w + "n", mulx(V(F(r.Sa)), V(E)));
        R.d = bind(o, w + "d", V(fmt("__fadd_rn(%s, %s)", E.c_str(), F(r.c).c_str())));
        R.n1 = bind(o, w + "n1", mulx(R.n, V(F(-l2 / bg))));
        R.d1 = bind(o, w + "d1", mulx(V(E), V(F(-l2 / bg))));
      }
      break;
    default: {
      o += fmt("  const float %sx = __fsub_rn(v, %s);\n", nm, F(r.v0).c_str());
      std::string n0, d0, n10, d10;
      double thr;
      if (r.sigma > 0) {
        n0 = fmt("__fmul_rn(%s, %sx)", F(r.Sa).c_str(), nm);
        d0 = fmt("__fmaf_rn(%s, %s, 1.0f)", F(-r.c).c_str(), E.c_str());
        n10 = F(l2 * r.Sa);
        d10 = fmt("__fmul_rn(%s, %s)", F(l2 * r.c / bg).c_str(), E.c_str());
        thr = kSingThr;
      } else {
        n0 = fmt("__fmul_rn(__fmul_rn(%s, %sx), %s)", F(r.Sa).c_str(), nm, E.c_str());
        d0 = fmt("__fsub_rn(%s, %s)", E.c_str(), F(r.c).c_str());
        n10 = fmt("__fmul_rn(__fmaf_rn(%sx, %s, %s), %s)", nm, F(-l2 * r.Sa / bg).c_str(), F(l2 * r.Sa).c_str(),
                  E.c_str());
        d10 = fmt("__fmul_rn(%s, %s)", E.c_str(), F(-l2 / bg).c_str());
        thr = kSingThr * r.c;
      }
      o += fmt("  const float %sd0 = %s;\n", nm, d0.c_str());
      o += fmt("  const bool %ssg = fabsf(%sd0) < %s;\n", nm, nm, F(thr).c_str());
      o += fmt("  const float %sns = __fmaf_rn(%sx, __fmaf_rn(%sx, %s, %s), %s);\n", nm, nm, nm,
               F(r.Sa / (12.0 * r.b)).c_str(), F(0.5 * r.Sa).c_str(), F(r.Sa * r.b).c_str());
      o += fmt("  const float %sn = %ssg ? %sns : %s;\n", nm, nm, nm, n0.c_str());
      o += fmt("  const float %sd = %ssg ? 1.0f : %sd0;\n", nm, nm, nm);
      // slopes: d/dx of a b (1 + u/2 + u^2/12) = a (1/2 + u/6) in the series region
      o += fmt("  const float %sn1 = %ssg ? __fmaf_rn(%sx, %s, %s) : %s;\n", nm, nm, nm,
               F(l2 * r.Sa / (6.0 * r.b)).c_str(), F(l2 * 0.5 * r.Sa).c_str(), n10.c_str());
      o += fmt("  const float %sd1 = %ssg ? 0.0f : %s;\n", nm, nm, d10.c_str());
      R.n = V(w + "n");
      R.d = V(w + "d");
      R.n1 = V(w + "n1");
      R.d1 = V(w + "d1");
    }
  }
  return R;
}

// merged backward of one gate: emits s (scaled: the decay's exp2 argument),
// e, pinf, and term = dpinf/dV (1 - e) + (p - pinf) (-dt)(a' + b') e
// (adjoint.py:155-164); with s~ = -dt log2(e) s, (-dt)(a' + b') = ln2 s~'.
static std::string emit_gate_bwd(const GatePlan& gp, const std::vector<Group>& G, int g) {
  std::string o;
  const RateX a = emit_rate_bwd(o, gp.a, G, "a");
  const RateX b = emit_rate_bwd(o, gp.b, G, "b");
  X s, s1, pinf, dpinf;
  if (!a.rat && !b.rat) {
    s = bind(o, "s", addx(a.v, b.v));
    s1 = bind(o, "s1", addx(a.v1, b.v1));
    const X rs = bind(o, "rs", V("rcpf_(s)"));
    pinf = bind(o, "pinf", mulx(a.v, rs));
    dpinf = bind(o, "dpinf", mulx(fmax_(a.v1, b.v, negx(mulx(a.v, b.v1))), mulx(rs, rs)));
  } else {
    X A, A1, N, N1, D, D1;
    if (a.rat && b.rat) {
      A = bind(o, "A", mulx(a.n, b.d));
      A1 = bind(o, "A1", fmax_(a.n1, b.d, mulx(a.n, b.d1)));
      N = bind(o, "N", fmax_(b.n, a.d, A));
      N1 = bind(o, "N1", fmax_(b.n1, a.d, fmax_(b.n, a.d1, A1)));
      D = bind(o, "D", mulx(a.d, b.d));
      D1 = bind(o, "D1", fmax_(a.d1, b.d, mulx(a.d, b.d1)));
    } else if (a.rat) {
      A = a.n;
      A1 = a.n1;
      N = bind(o, "N", fmax_(b.v, a.d, a.n));
      N1 = bind(o, "N1", fmax_(b.v1, a.d, fmax_(b.v, a.d1, a.n1)));
      D = a.d;
      D1 = a.d1;
    } else {
      A = bind(o, "A", mulx(a.v, b.d));
      A1 = bind(o, "A1", fmax_(a.v1, b.d, mulx(a.v, b.d1)));
      N = bind(o, "N", addx(A, b.n));
      N1 = bind(o, "N1", addx(A1, b.n1));
      D = b.d;
      D1 = b.d1;
    }
    X iD, iN;
    static const bool bwd_one = getenv("HHB_JIT_BWD_ONE_RCP") && atoi(getenv("HHB_JIT_BWD_ONE_RCP")) > 0;
    if (bwd_one && gp.one_rcp) {   // default: the issue-bound backward takes two reciprocals (see plan_of)
      const X r = bind(o, "r", V("rcpf_(" + mulx(N, D).e + ")"));
      iD = bind(o, "iD", mulx(N, r));
      iN = bind(o, "iN", mulx(D, r));
    } else {
      iD = bind(o, "iD", V("rcpf_(" + D.e + ")"));
      iN = bind(o, "iN", V("rcpf_(" + N.e + ")"));
    }
    s = bind(o, "s", mulx(N, iD));
    pinf = bind(o, "pinf", mulx(A, iN));
    s1 = bind(o, "s1", mulx(fmax_(negx(s), D1, N1), iD));
    dpinf = bind(o, "dpinf", mulx(fmax_(negx(pinf), N1, A1), iN));
  }
  o += "  const float e = ex2f_(s);\n";
  // term = dpinf (1 - e) + (p - pinf) ln2 s1 e = e ((p - pinf) ln2 s1 - dpinf) + dpinf
  o += fmt("  const float term = __fmaf_rn(e, __fmaf_rn(__fsub_rn(p[%d], %s), %s, %s), %s);\n", g, pinf.e.c_str(),
           s1.zero ? "0.0f" : fmt("__fmul_rn(%s, %s)", s1.e.c_str(), F(std::log(2.0)).c_str()).c_str(), negx(dpinf).e.c_str(), dpinf.e.c_str());
  return o;
}

// step_fwd_m(v, p[], cur) -> v' : the merged-form step (regular lanes only)
static std::string emit_step(const hhb_params_t* P, const Layout& L, const Plan& M) {
  std::string o;
  const int NG = L.ng;
  o += fmt("__device__ __forceinline__ bool regular(const float v) { return fabsf(__fsub_rn(v, %s)) < %s; }\n",
           F(0.5 * (M.lo + M.hi)).c_str(), F(0.5 * (M.hi - M.lo)).c_str());
  o += fmt("__device__ __forceinline__ float step_fwd_m(const float v, float (&p)[%d], const float cur) {\n",
           NG > 0 ? NG : 1);
  const char* pe = getenv("HHB_JIT_POLY_EXP");
  o += emit_exps(M, pe ? atoi(pe) : 0);
  o += L.leak_ch.empty() ? "  float ion = 0.0f;\n"
                         : fmt("  float ion = __fmaf_rn(%s, v, %s);\n", F(L.gl).c_str(), F(-L.gle).c_str());
  o += "  float eta = 1.0f;\n";
  auto neg = [](double x, const std::string& e) { return x < 0 ? "(-" + e + ")" : e; };
  for (int g = 0; g < NG; ++g) {
    const hhb_gate_t& G = P->gates[g];
    const hhb_channel_t& C = P->channels[L.chan[g]];
    const GatePlan& gp = M.gates[g];
    o += fmt("  // gate %d (channel %d), exponent %d, %s reciprocal(s)\n  {\n", g, L.chan[g], G.exponent,
             gp.one_rcp ? "one" : "two");
    const std::string pg = fmt("p[%d]", g);
    o += "  const float pk = " + pow_expr(pg, G.exponent) + ";\n";
    o += L.first[g] ? "  eta = pk;\n" : "  eta = __fmul_rn(eta, pk);\n";
    // each rate -> plain value <w>v or fraction <w>n / <w>d
    for (int w = 0; w < 2; ++w) {
      const RatePlan& r = w ? gp.b : gp.a;
      const char* nm = w ? "b" : "a";
      const std::string E = fmt("E%d", r.group);
      if (r.kind == HHB_RATE_EXP && r.sigma > 0) {
        if (r.direct) {
          const double K2 = -kLog2e / r.b;
          o += fmt("  const float %sv = %s;\n", nm,
                   neg(r.Sa, fmt("ex2f_(__fmaf_rn(v, %s, %s))", F(K2).c_str(),
                                 F(-r.v0 * K2 + std::log2(std::fabs(r.Sa))).c_str())).c_str());
        } else {
          o += fmt("  const float %sv = __fmul_rn(%s, %s);\n", nm, F(r.Sa * r.c).c_str(), E.c_str());
        }
        continue;
      }
      switch (r.kind) {
        case HHB_RATE_EXP:  // sigma < 0
          o += fmt("  const float %sn = %s;\n  const float %sd = %s;\n", nm, F(r.Sa * r.c).c_str(), nm, E.c_str());
          break;
        case HHB_RATE_SIGMOID:
          if (r.sigma > 0)
            o += fmt("  const float %sn = %s;\n  const float %sd = __fmaf_rn(%s, %s, 1.0f);\n", nm, F(r.Sa).c_str(),
                     nm, F(r.c).c_str(), E.c_str());
          else
            o += fmt("  const float %sn = __fmul_rn(%s, %s);\n  const float %sd = __fadd_rn(%s, %s);\n", nm,
                     F(r.Sa).c_str(), E.c_str(), nm, E.c_str(), F(r.c).c_str());
          break;
        default: {
          o += fmt("  const float %sx = __fsub_rn(v, %s);\n", nm, F(r.v0).c_str());
          std::string n0, d0;
          double thr;
          if (r.sigma > 0) {
            n0 = fmt("__fmul_rn(%s, %sx)", F(r.Sa).c_str(), nm);
            d0 = fmt("__fmaf_rn(%s, %s, 1.0f)", F(-r.c).c_str(), E.c_str());
            thr = kSingThr;
          } else {
            n0 = fmt("__fmul_rn(__fmul_rn(%s, %sx), %s)", F(r.Sa).c_str(), nm, E.c_str());
            d0 = fmt("__fsub_rn(%s, %s)", E.c_str(), F(r.c).c_str());
            thr = kSingThr * r.c;
          }
          o += fmt("  const float %sd0 = %s;\n", nm, d0.c_str());
          o += fmt("  const bool %ssg = fabsf(%sd0) < %s;\n", nm, nm, F(thr).c_str());
          // a b (1 + u/2 + u^2/12), u = x / b, as a Horner form in x
          o += fmt("  const float %sns = __fmaf_rn(%sx, __fmaf_rn(%sx, %s, %s), %s);\n", nm, nm, nm,
                   F(r.Sa / (12.0 * r.b)).c_str(), F(0.5 * r.Sa).c_str(), F(r.Sa * r.b).c_str());
          o += fmt("  const float %sn = %ssg ? %sns : %s;\n", nm, nm, nm, n0.c_str());
          o += fmt("  const float %sd = %ssg ? 1.0f : %sd0;\n", nm, nm, nm);
        }
      }
    }
    const bool ra = gp.a.rational(), rb = gp.b.rational();
    if (!ra && !rb) {
      o += "  const float s = __fadd_rn(av, bv);\n";
      o += "  const float pinf = __fmul_rn(av, rcpf_(s));\n";
    } else {
      if (ra && rb) {
        o += "  const float A = __fmul_rn(an, bd);\n";
        o += "  const float N = __fmaf_rn(bn, ad, A);\n";
        o += "  const float D = __fmul_rn(ad, bd);\n";
      } else if (ra) {
        o += "  const float A = an;\n";
        o += "  const float N = __fmaf_rn(bv, ad, an);\n";
        o += "  const float D = ad;\n";
      } else {
        o += "  const float A = __fmul_rn(av, bd);\n";
        o += "  const float N = __fmaf_rn(av, bd, bn);\n";
        o += "  const float D = bd;\n";
      }
      if (gp.one_rcp) {
        o += "  const float r = rcpf_(__fmul_rn(N, D));\n";
        o += "  const float s = __fmul_rn(N, __fmul_rn(N, r));\n";
        o += "  const float pinf = __fmul_rn(A, __fmul_rn(D, r));\n";
      } else {
        o += "  const float s = __fmul_rn(N, rcpf_(D));\n";
        o += "  const float pinf = __fmul_rn(A, rcpf_(N));\n";
      }
    }
    // s is already -dt * log2(e) * (alpha + beta)
    o += "  const float dec = ex2f_(s);\n";
    o += fmt("  %s = __fmaf_rn(__fsub_rn(%s, pinf), dec, pinf);\n", pg.c_str(), pg.c_str());
    if (L.last[g])
      o += fmt("  ion = __fmaf_rn(eta, __fmaf_rn(v, %s, %s), ion);\n", F(C.g_max).c_str(),
               F(-C.g_max * C.e_rev).c_str());
    o += "  }\n";
  }
  o += fmt("  return __fmaf_rn(__fsub_rn(cur, ion), %s, v);\n}\n", F(P->dt / P->c_m).c_str());
  return o;
}


// Paired (f32x2) form of a merged step.  sm_100a issues FFMA2 / FMUL2 / FADD2:
// one warp instruction does the float op of two neurons (the FMA pipe's fp32
// rate is unchanged, the issue slots halve -- the merged steps are issue-bound,
// profiles/r2_fwdp.md, r2_bptt.md).  pair() rewrites the emitted scalar
// function into template <bool H> ...2(F2 ...): every float becomes an F2 (x =
// neuron j, y = neuron j + 1), selects become per-half sel2, MUFU ops stay one
// per half (H: the y half is a copy of x and its MUFU ops are skipped -- the
// one-neuron callers).  All callers, paired or not, run this one function, so
// every kernel reproduces the same states bit for bit (ptxas contracts
// FMUL2 + FADD2 into FFMA2 regardless of .rn; the scalar form would round
// differently).
static const char* kPairPrelude = R"(
struct __align__(8) F2 {
  float x, y;
  __device__ __forceinline__ F2() {}
  __device__ __forceinline__ F2(float a) : x(a), y(a) {}
  __device__ __forceinline__ F2(float a, float b) : x(a), y(b) {}
};
struct B2 { bool x, y; };
__device__ __forceinline__ float2 f2_(const F2 a) { return make_float2(a.x, a.y); }
__device__ __forceinline__ F2 F2_(const float2 a) { return F2(a.x, a.y); }
__device__ __forceinline__ F2 mul2(const F2 a, const F2 b) { return F2_(__fmul2_rn(f2_(a), f2_(b))); }
__device__ __forceinline__ F2 add2(const F2 a, const F2 b) { return F2_(__fadd2_rn(f2_(a), f2_(b))); }
__device__ __forceinline__ F2 sub2(const F2 a, const F2 b) { return F2_(__fadd2_rn(f2_(a), make_float2(-b.x, -b.y))); }
__device__ __forceinline__ F2 fma2(const F2 a, const F2 b, const F2 c) { return F2_(__ffma2_rn(f2_(a), f2_(b), f2_(c))); }
__device__ __forceinline__ F2 operator-(const F2 a) { return F2(-a.x, -a.y); }   // folds into operand modifiers
__device__ __forceinline__ F2 abs2(const F2 a) { return F2(fabsf(a.x), fabsf(a.y)); }
__device__ __forceinline__ B2 operator<(const F2 a, const float c) { return B2{a.x < c, a.y < c}; }
__device__ __forceinline__ F2 sel2(const B2 c, const F2 a, const F2 b) { return F2(c.x ? a.x : b.x, c.y ? a.y : b.y); }
// the y half's MUFU op is volatile: with duplicated halves (one-neuron callers)
// the compiler would merge the two and then copy x into y with a MOV on the chain
__device__ __forceinline__ float ex2y_(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcpy_(float x) { float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <bool H> __device__ __forceinline__ F2 ex2v(const F2 a) { const float x = ex2f_(a.x); return F2(x, H ? x : ex2y_(a.y)); }
template <bool H> __device__ __forceinline__ F2 rcpv(const F2 a) { const float x = rcpf_(a.x); return F2(x, H ? x : rcpy_(a.y)); }
__device__ __forceinline__ F2 ex2p2(const F2 x) {   // paired ex2p_ (same operations per half)
  const F2 t = add2(x, 12582912.0f);
  const F2 f = sub2(x, sub2(t, 12582912.0f));
  F2 p = fma2(0x1.41d332p-13f, f, 0x1.5f456ap-10f);
  p = fma2(p, f, 0x1.3b2dbcp-7f);
  p = fma2(p, f, 0x1.c6aed4p-5f);
  p = fma2(p, f, 0x1.ebfbdap-3f);
  p = fma2(p, f, 0x1.62e430p-1f);
  p = fma2(p, f, 1.0f);
  return F2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
            __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}
template <bool H> __device__ __forceinline__ F2 surrogate2(const Sur& s, const F2 u) {
  const float x = surrogate(s, u.x);
  return F2(x, H ? x : surrogate(s, u.y));
}
)";

static void replace_all(std::string& s, const std::string& a, const std::string& b) {
  for (size_t i = s.find(a); i != std::string::npos; i = s.find(a, i + b.size())) s.replace(i, a.size(), b);
}
static bool ident(char c) { return std::isalnum(static_cast<unsigned char>(c)) || c == '_'; }
// whole-word replacement (a is an identifier)
static void replace_word(std::string& s, const std::string& a, const std::string& b) {
  for (size_t i = s.find(a); i != std::string::npos;) {
    const bool l = i == 0 || !ident(s[i - 1]);
    const bool r = i + a.size() >= s.size() || !ident(s[i + a.size()]);
    if (l && r) {
      s.replace(i, a.size(), b);
      i = s.find(a, i + b.size());
    } else {
      i = s.find(a, i + a.size());
    }
  }
}
// "  const float x = c ? a : b;" -> "  const F2 x = sel2(c, a, b);" (the merged
// steps' only selects: one condition name, no nested ternaries)
static std::string pair_line(std::string ln) {
  const size_t q = ln.find(" ? ");
  if (q != std::string::npos) {
    const size_t eq = ln.rfind(" = ", q);
    const size_t c = ln.find(" : ", q);
    const size_t end = ln.rfind(';');
    if (eq == std::string::npos || c == std::string::npos || end == std::string::npos || end < c) return "#error pair";
    ln = ln.substr(0, eq + 3) + "sel2(" + ln.substr(eq + 3, q - eq - 3) + ", " + ln.substr(q + 3, c - q - 3) + ", " +
         ln.substr(c + 3, end - c - 3) + ")" + ln.substr(end);
  }
  return ln;
}
// scalar merged function (signature line + body) -> its paired template
static std::string pair(const std::string& fn, const std::string& name) {
  const size_t nl = fn.find('\n');
  std::string sig = fn.substr(0, nl), body = fn.substr(nl + 1);
  replace_word(sig, "float", "F2");
  replace_word(sig, name, name + "2");
  replace_all(sig, "__device__ __forceinline__", "template <bool H> __device__ __forceinline__");
  replace_word(body, "float", "F2");
  replace_word(body, "bool", "B2");
  replace_all(body, "__fmul_rn(", "mul2(");
  replace_all(body, "__fadd_rn(", "add2(");
  replace_all(body, "__fsub_rn(", "sub2(");
  replace_all(body, "__fmaf_rn(", "fma2(");
  replace_all(body, "ex2f_(", "ex2v<H>(");
  replace_all(body, "ex2p_(", "ex2p2(");
  replace_all(body, "rcpf_(", "rcpv<H>(");
  replace_all(body, "fabsf(", "abs2(");
  replace_all(body, "surrogate(", "surrogate2<H>(");
  std::string out = sig + "\n";
  size_t i = 0;
  while (i < body.size()) {
    size_t j = body.find('\n', i);
    if (j == std::string::npos) j = body.size();
    out += pair_line(body.substr(i, j - i)) + "\n";
    i = j + 1;
  }
  return out;
}
}  // namespace mg

// adjoint of step_fwd (hh_step_backward, adjoint.py:116-188).  The parameter-
// gradient terms (adjoint.py:144, :147) are accumulated straight into the
// caller's fp32 partials acc[] with FFMAs; per gated channel c the factor
// w_c = g_vp (v - E_c) is shared by its d_g_max term and the dp' chain rule of
// all its gates.  Merged variant: term = e ((p - pinf) ln2 s' - dpinf) + dpinf
// (s' the slope of the exp2 argument) costs 4 ops per gate.
static std::string emit_backward_step(const hhb_params_t* P, const Layout& L, SeriesMode mode,
                                      const mg::Plan* M = nullptr) {
  std::string o;
  const int NG = L.ng, NGX = NG > 0 ? NG : 1;
  const double dtcm = P->dt / P->c_m;
  o += fmt(
      "__device__ __forceinline__ float step_bwd_%s(const Sur& sur, const float v, const float (&p)[%d], "
      "const float cur, float& d_v, float (&d_p)[%d], const float d_spike, const bool has_s, "
      "float (&acc)[%d]) {\n",
      M ? "m" : (mode == kFast ? "f" : "s"), NGX, NGX, kSlots);
  if (M) o += mg::emit_exps(*M);
  o += L.leak_ch.empty() ? "  float ion = 0.0f;\n"
                         : fmt("  float ion = __fmaf_rn(%s, v, %s);\n", F(L.gl).c_str(), F(-L.gle).c_str());
  o += fmt("  float gsum = %s;\n", F(L.gl).c_str());
  o += fmt("  float pk[%d], eta_c[%d];\n", NGX, NGX);
  o += "  float eta = 1.0f;\n";
  for (int g = 0; g < NG; ++g) {
    const hhb_gate_t& G = P->gates[g];
    const hhb_channel_t& C = P->channels[L.chan[g]];
    o += fmt("  pk[%d] = %s;\n", g, pow_expr(fmt("p[%d]", g), G.exponent).c_str());
    o += L.first[g] ? fmt("  eta = pk[%d];\n", g) : fmt("  eta = __fmul_rn(eta, pk[%d]);\n", g);
    o += fmt("  eta_c[%d] = eta;\n", g);
    if (L.last[g]) {
      o += fmt("  ion = __fmaf_rn(__fmul_rn(eta, %s), __fsub_rn(v, %s), ion);\n", F(C.g_max).c_str(),
               F(C.e_rev).c_str());
      o += fmt("  gsum = __fmaf_rn(%s, eta, gsum);\n", F(C.g_max).c_str());
    }
  }
  o += "  const float dI = __fsub_rn(cur, ion);\n";
  o += fmt("  const float vn = __fmaf_rn(dI, %s, v);\n", F(dtcm).c_str());
  o += "  float g_vp = d_v;\n";
  o += fmt("  if (has_s) g_vp = __fmaf_rn(d_spike, surrogate(sur, __fsub_rn(vn, %s)), g_vp);\n",
           F(P->v_theta).c_str());
  o += "  acc[0] = __fmaf_rn(g_vp, dI, acc[0]);\n";
  // per gated channel: w_c = g_vp (v - E_c)
  for (int g = 0; g < NG; ++g) {
    if (!L.last[g]) continue;
    const hhb_channel_t& C = P->channels[L.chan[g]];
    o += fmt("  const float w%d = __fmul_rn(g_vp, __fsub_rn(v, %s));\n", L.chan[g], F(C.e_rev).c_str());
    o += fmt("  acc[%d] = __fmaf_rn(w%d, eta_c[%d], acc[%d]);\n", 1 + g, L.chan[g], g, 1 + g);
  }
  for (size_t j = 0; j < L.leak_ch.size(); ++j) {
    const int k = 1 + kMaxGates + int(j);
    o += fmt("  acc[%d] = __fmaf_rn(g_vp, __fsub_rn(v, %s), acc[%d]);\n", k,
             F(P->channels[L.leak_ch[j]].e_rev).c_str(), k);
  }
  o += fmt("  float dv_in = __fmul_rn(g_vp, __fmaf_rn(%s, gsum, 1.0f));\n", F(-dtcm).c_str());
  for (int g = 0; g < NG; ++g) {
    const hhb_gate_t& G = P->gates[g];
    const hhb_channel_t& C = P->channels[L.chan[g]];
    o += fmt("  // gate %d\n  {\n", g);
    if (M) {
      o += mg::emit_gate_bwd(M->gates[g], M->groups, g);
      o += fmt("  const float up = d_p[%d];\n", g);
      o += "  dv_in = __fmaf_rn(up, term, dv_in);\n";
      o += "  float dp = __fmul_rn(up, e);\n";
    } else {
      o += "  float a, b, da, db;\n";
      std::string sa = "da", sb = "db";
      emit_rate(o, G.alpha, P->rate_scale, "a", &sa, mode);
      emit_rate(o, G.beta, P->rate_scale, "b", &sb, mode);
      o += "  const float s = __fadd_rn(a, b);\n";
      o += "  const float rs = rcpf_(s);\n";
      o += fmt("  const float e = ex2f_(__fmul_rn(s, %s));\n", F(-P->dt * kLog2e).c_str());
      o += "  const float pinf = __fmul_rn(a, rs);\n";
      o += "  const float dpinf = __fmul_rn(__fsub_rn(__fmul_rn(da, b), __fmul_rn(a, db)), __fmul_rn(rs, rs));\n";
      o += fmt("  const float term = __fmaf_rn(dpinf, __fsub_rn(1.0f, e), __fmul_rn(__fsub_rn(p[%d], pinf), "
               "__fmul_rn(__fmul_rn(%s, __fadd_rn(da, db)), e)));\n",
               g, F(-P->dt).c_str());
      o += "  const bool pos = s > 0.0f;\n";
      o += fmt("  const float up = d_p[%d];\n", g);
      o += "  dv_in = pos ? __fmaf_rn(up, term, dv_in) : dv_in;\n";
      o += "  float dp = pos ? __fmul_rn(up, e) : up;\n";
    }
    if (G.exponent > 0) {
      // d eta / d p = k p^(k-1) prod(other gates of the channel), times the
      // constant -dt/c_m g_c of the membrane step, against w_c
      const double kc = -dtcm * C.g_max * double(G.exponent);
      std::string der = G.exponent > 1 ? pow_expr(fmt("p[%d]", g), G.exponent - 1) : "";
      const hhb_channel_t& CC = P->channels[L.chan[g]];
      for (int o2 = CC.gate_begin; o2 < CC.gate_begin + CC.gate_count; ++o2)
        if (o2 != g) der = der.empty() ? fmt("pk[%d]", o2) : fmt("__fmul_rn(%s, pk[%d])", der.c_str(), o2);
      const std::string dk = der.empty() ? F(kc) : fmt("__fmul_rn(%s, %s)", F(kc).c_str(), der.c_str());
      o += fmt("  dp = __fmaf_rn(w%d, %s, dp);\n", L.chan[g], dk.c_str());
    }
    o += fmt("  d_p[%d] = dp;\n  }\n", g);
  }
  o += "  d_v = dv_in;\n";
  o += fmt("  return __fmul_rn(g_vp, %s);\n}\n", F(dtcm).c_str());
  return o;
}


// Kernel bodies (parameterised by NG through the generated step functions).
static const char* kPrelude = R"(
#if HHB_CHECK
#define NET_CHK(c) do { if (!(c)) { printf("hhb check failed: %s (block %d thread %d)\n", #c, int(blockIdx.x), int(threadIdx.x)); __trap(); } } while (0)
#else
#define NET_CHK(c) do { } while (0)
#endif
typedef long long i64;
typedef unsigned int u32;
// programmatic dependent launch (pdl.cuh): wait for the predecessor grid before
// touching global memory, then let the successor's CTAs be scheduled
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
struct FwdArgs { i64 n, steps; const float* v_in; const float* g_in; i64 g_ld; float* v_fin; float* g_fin;
  const float* i_ext; i64 i_st, i_sn; float* v_out; i64 v_ld; u32* spk; i64 spk_ld; float* ckpt;
  i64 ck_every, ck_ld; i64 step_base; i64* first_bad; unsigned long long seed; i64 nbase;
  float* spk_val; i64 spkv_ld; const long long* step_dev; double* sq_part; unsigned short* spk_bf; i64 spkb_ld; };
struct PoissonTab { int size; float amp; float cdf[48]; };
// Philox-4x32-10 with the key schedule precomputed on the host (one kernel
// parameter per round key: LOP3 takes them straight from the constant bank)
struct Keys { u32 k[20]; };
__device__ __forceinline__ uint4 philox(const Keys& ks, i64 gj, i64 gq) {
  uint4 c = make_uint4(u32(gj), u32((unsigned long long)gj >> 32), u32(gq), u32((unsigned long long)gq >> 32));
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const u32 hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const u32 hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ ks.k[2 * r], lo1, hi0 ^ c.w ^ ks.k[2 * r + 1], lo0);
  }
  return c;
}
// guide-table inverse CDF in shared memory (hh_kernels.cuh PoissonSmem)
// guide-table Poisson draw (see hh_kernels.cuh PoissonSmem): each bucket holds
// amp*k0 and the three next CDF values as integer thresholds on the raw word,
// T(c) = ((floor(c 2^23) + 1) << 9) - 1, so u > c  <=>  w > T(c) exactly for
// the uniform u = (w >> 9) 2^-23: no int->float conversion per draw and
// bit-identical to the float compare of the generic kernels.
struct PoissonSmem {
  uint4 g4[256];
  int k0[256];
  float cdf[48];
  float amp;
  __device__ static u32 thr(float c) {
    return c >= 1.0f ? 0xFFFFFFFFu : ((u32(floorf(c * 8388608.0f)) + 1u) << 9) - 1u;
  }
  __device__ void fill(const PoissonTab& tab) {
    for (int k = threadIdx.x; k < 48; k += blockDim.x) cdf[k] = k < tab.size - 1 ? tab.cdf[k] : 2.0f;
    if (threadIdx.x == 0) amp = tab.amp;
    for (int b = threadIdx.x; b < 256; b += blockDim.x) {
      const float lo = float(b) * 0.00390625f;
      int k = 0;
      while (k < tab.size - 1 && tab.cdf[k] < lo) ++k;
      k0[b] = k;
      const float c0 = k < tab.size - 1 ? tab.cdf[k] : 2.0f;
      const float c1 = k + 1 < tab.size - 1 ? tab.cdf[k + 1] : 2.0f;
      const float c2 = k + 2 < tab.size - 1 ? tab.cdf[k + 2] : 2.0f;
      g4[b] = make_uint4(__float_as_uint(tab.amp * float(k)), thr(c0), thr(c1), thr(c2));
    }
  }
  __device__ __forceinline__ static float uniform(u32 w) { return __uint_as_float(0x3F800000u | (w >> 9)) - 1.0f; }
  __device__ __forceinline__ float draw(u32 w, bool& tail) const {
    const uint4 e = g4[w >> 24];
    float val = __uint_as_float(e.x);
    val = (w > e.y) ? val + amp : val;
    val = (w > e.z) ? val + amp : val;
    tail = w > e.w;
    return val;
  }
  __device__ float tail_draw(u32 w) const {
    const float u = uniform(w);
    int k = k0[w >> 24] + 3;
    while (u > cdf[k]) ++k;
    return amp * float(k);
  }
};
struct BwdArgs { i64 n, steps; const float* i_ext; i64 i_st, i_sn; const float* ckpt; i64 ck_every, ck_ld;
  float* seg; const float* seed_v; i64 sv_ld; const float* seed_s; i64 ss_ld; float* adj_v; float* adj_g;
  i64 ag_ld; float* d_i; i64 di_ld; double* partials; i64 step_base; i64* first_bad;
  unsigned short* di_hi; unsigned short* di_lo; i64 dh_ld; float* di_sum; i64 dh_grp, dh_pitch;
  const float* sv_scale; };
__device__ __forceinline__ void split_bf16(float x, unsigned short& hi, unsigned short& lo) {
  // round-to-nearest-even bf16 of x (cvt.rn.bf16x2.f32), then of the remainder
  // x - hi, which is exact in fp32; one packed cvt yields both halves
  u32 h;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(0.0f), "f"(x));
  const float r = __fsub_rn(x, __uint_as_float(h << 16));
  u32 pk;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pk) : "f"(r), "f"(x));
  hi = (unsigned short)(pk & 0xFFFFu);
  lo = (unsigned short)(pk >> 16);
}
struct Sur { int kind; float w, inv_w, k2, half_inv_w; };
#define LLMAX 0x7fffffffffffffffLL
__device__ __forceinline__ float ex2f_(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcpf_(float x) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
// 2^x on the FMA pipe: x = j + f (j = round(x) via the 1.5 * 2^23 shifter, |f| <= 1/2),
// a degree-6 polynomial for 2^f (max rel. error 7.9e-8 = 1.3 ulp over the interval;
// MUFU.EX2 is ~2 ulp), then j added to the exponent field.  For |x| < 126.
__device__ __forceinline__ float ex2p_(float x) {
  const float t = __fadd_rn(x, 12582912.0f);
  const float f = __fsub_rn(x, __fsub_rn(t, 12582912.0f));
  float p = __fmaf_rn(0x1.41d332p-13f, f, 0x1.5f456ap-10f);
  p = __fmaf_rn(p, f, 0x1.3b2dbcp-7f);
  p = __fmaf_rn(p, f, 0x1.c6aed4p-5f);
  p = __fmaf_rn(p, f, 0x1.ebfbdap-3f);
  p = __fmaf_rn(p, f, 0x1.62e430p-1f);
  p = __fmaf_rn(p, f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
__device__ __forceinline__ bool finitef_(float x) { return fabsf(x) < __int_as_float(0x7f800000); }
__device__ __forceinline__ float surrogate(const Sur& s, float u) {
  if (s.kind == 1) return (fabsf(u) <= s.w) ? s.half_inv_w : 0.0f;
  const float q = rcpf_(__fadd_rn(1.0f, ex2f_(__fmul_rn(u, s.k2))));
  return __fmul_rn(__fmul_rn(q, __fsub_rn(1.0f, q)), s.inv_w);
}
)";

static const char* kForwardBody = R"(
template <int VEC>
__device__ __forceinline__ void load_cur(const FwdArgs& a, i64 t, i64 n0, bool full, float (&c)[VEC]) {
  if (VEC == 4 && full && a.i_sn == 1) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(a.i_ext + t * a.i_st + n0));
    c[0] = q.x; c[1] = q.y; c[2] = q.z; c[3] = q.w;
  } else {
#pragma unroll
    for (int j = 0; j < VEC; ++j) c[j] = (n0 + j < a.n) ? __ldg(a.i_ext + t * a.i_st + (n0 + j) * a.i_sn) : 0.0f;
  }
}
template <int VEC>
__device__ __forceinline__ void store_vec(float* p, const float (&x)[VEC], bool full, i64 n0, i64 n) {
  if (VEC == 4 && full) { *reinterpret_cast<float4*>(p + n0) = make_float4(x[0], x[1], x[2], x[3]); }
  else {
#pragma unroll
    for (int j = 0; j < VEC; ++j) if (n0 + j < n) p[n0 + j] = x[j];
  }
}
template <int VEC, bool POIS>
struct Stimulus {
  __device__ __forceinline__ void at(const FwdArgs& a, const Keys& ks, const PoissonSmem& tab, i64 t, i64 n0,
                                     bool full, float (&c)[VEC]) {
    if (POIS) {
      const i64 gt = a.step_base + t;
      u32 w[VEC];
      if (VEC == 4) {  // host guarantees (nbase + n0) % 4 == 0
        const uint4 r = philox(ks, (a.nbase + n0) >> 2, gt);
        w[0] = r.x;
        w[VEC > 1 ? 1 : 0] = r.y;
        w[VEC > 2 ? 2 : 0] = r.z;
        w[VEC > 3 ? 3 : 0] = r.w;
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          const i64 gj = a.nbase + n0 + j;
          const uint4 r = philox(ks, gj >> 2, gt);
          const int i = int(gj & 3);
          w[j] = i == 0 ? r.x : i == 1 ? r.y : i == 2 ? r.z : r.w;
        }
      }
      bool tail[VEC], any_tail = false;
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        c[j] = tab.draw(w[j], tail[j]);
        any_tail = any_tail || tail[j];
      }
      if (__any_sync(0xffffffffu, any_tail)) {
#pragma unroll
        for (int j = 0; j < VEC; ++j)
          if (tail[j]) c[j] = tab.tail_draw(w[j]);
      }
    } else {
      load_cur<VEC>(a, t, n0, full, c);
    }
  }
};
// The module is specialised on which output streams the launch has (FF_VO V
// trace, FF_SO spike bitmap, FF_SVO spike values, FF_CK checkpoints) and on
// FF_AL: every stream neuron-contiguous and 16-byte aligned with n % 4 == 0,
// so a live thread always moves whole float4s (no per-step null checks, no
// per-neuron tails in the loop).
template <int VEC, bool POIS>
__device__ __forceinline__ void fwd_body(const FwdArgs& a_in, const PoissonTab& tab, const Keys& ks) {
  pdl_begin();
  FwdArgs a = a_in;
  if (a.step_dev != nullptr) a.step_base += *a.step_dev;
  const int lane = threadIdx.x & 31;
  const i64 tid = i64(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 n0 = tid * VEC;
  const bool full = n0 + VEC <= a.n;
  constexpr bool AL = FF_AL && VEC == 4;
  const bool live = n0 < a.n;                   // == full when AL
  Stimulus<VEC, POIS> stim;
  __shared__ PoissonSmem ps;
  if (POIS) {
    ps.fill(tab);
    __syncthreads();
  }
  float v[VEC];
  float p[VEC][NGX];
  u32 valid = 0;
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    const bool on = n0 + j < a.n;
    valid |= u32(on) << j;
    v[j] = on ? a.v_in[n0 + j] : -65.0f;
#pragma unroll
    for (int g = 0; g < NG; ++g) p[j][g] = on ? a.g_in[g * a.g_ld + n0 + j] : 0.5f;
  }
  i64 bad = LLMAX;
  int ck_count = 0;
  float sqf = 0.0f;
  double sqd = 0.0;
  // running pointers (one 64-bit add per step instead of t * ld)
  float* ckp = FF_CK ? a.ckpt + n0 : nullptr;
  const i64 sstride = (1 + NG) * a.ck_ld;
  const float* ip = POIS ? nullptr : a.i_ext + n0 * a.i_sn;
  const bool vec_in = VEC == 4 && (AL || (full && a.i_sn == 1));
  float* vo = FF_VO ? a.v_out + n0 : nullptr;
  u32* so = FF_SO ? a.spk + n0 / 32 : nullptr;
  float* svo = FF_SVO ? a.spk_val + n0 : nullptr;
  unsigned short* sbo = FF_SVB ? a.spk_bf + n0 : nullptr;
  const bool spk_writer = lane % (32 / VEC) == 0 && live;
  // loaded currents are prefetched FWD_PF (8) steps ahead with one neuron per
  // thread (small, latency-bound populations: one warp per SM, the step chain
  // is shorter than an HBM load) and one step ahead with four (throughput-
  // bound, registers are the limit); the drawn stimulus is made at the top of
  // its own step (no registers held across it)
  constexpr int PF = POIS ? 1 : (VEC == 1 ? FWD_PF : FWD_PF4);
  float cur[VEC];
  float pre[PF][VEC];
  auto load_in = [&](float (&c)[VEC]) {
    if (vec_in) {
      const float4 q = live ? __ldg(reinterpret_cast<const float4*>(ip)) : make_float4(0.f, 0.f, 0.f, 0.f);
      c[0] = q.x; c[VEC > 1 ? 1 : 0] = q.y; c[VEC > 2 ? 2 : 0] = q.z; c[VEC > 3 ? 3 : 0] = q.w;
    } else {
#pragma unroll
      for (int j = 0; j < VEC; ++j) c[j] = ((valid >> j) & 1u) ? __ldg(ip + j * a.i_sn) : 0.0f;
    }
    ip += a.i_st;
  };
  auto store4 = [&](float* q, const float (&x)[VEC]) {
    if (AL || (VEC == 4 && full)) {
      if (live) *reinterpret_cast<float4*>(q) = make_float4(x[0], x[VEC > 1 ? 1 : 0], x[VEC > 2 ? 2 : 0], x[VEC > 3 ? 3 : 0]);
    } else {
#pragma unroll
      for (int j = 0; j < VEC; ++j) if ((valid >> j) & 1u) q[j] = x[j];
    }
  };
  // PF > 1 (one neuron per thread): every prefetch is an unconditional load
  // (padding lanes read element 0, rows past the end re-read the last row) so
  // no select/phi copy of the loaded register is made -- such a copy waits for
  // the load and undoes the prefetch
  const float* ib1 = (n0 < a.n) ? a.i_ext + n0 * a.i_sn : a.i_ext;
  auto load_row = [&](i64 r, float (&c)[VEC]) {
    const float* q = ib1 + (r < a.steps ? r : a.steps - 1) * a.i_st;
    if (VEC == 1) {
      c[0] = __ldg(q);
    } else if (vec_in) {
      const float4 w = __ldg(reinterpret_cast<const float4*>(q));     // live lanes only (vec_in: n % 4 == 0 or full)
      c[0] = w.x; c[VEC > 1 ? 1 : 0] = w.y; c[VEC > 2 ? 2 : 0] = w.z; c[VEC > 3 ? 3 : 0] = w.w;
    } else {
#pragma unroll
      for (int j = 0; j < VEC; ++j) c[j] = __ldg(q + (((valid >> j) & 1u) ? j : 0) * a.i_sn);
    }
  };
  if (!POIS && a.steps > 0) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      if (PF > 1) load_row(k, pre[k]);
      else load_in(pre[k]);
    }
  }
  auto body = [&](const i64 t) {
    if (FF_CK && ck_count == 0) {      // state BEFORE step t
      store4(ckp, v);
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        float q[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) q[j] = p[j][g];
        store4(ckp + (1 + g) * a.ck_ld, q);
      }
      ckp += sstride;
      ck_count = int(a.ck_every);
    }
    --ck_count;
    float vn[VEC];
    step_all<VEC>(v, p, cur, vn);
    u32 nib = 0;
    bool fin = true;
#pragma unroll
    for (int j = 0; j < VEC; ++j) {
      nib |= u32((v[j] < THETA) && (vn[j] >= THETA)) << j;
      fin = fin && finitef_(vn[j]);
      v[j] = vn[j];
    }
    if (FF_L2) {   // fused MSE(V, 0) forward: fp32 partials, flushed to fp64 every 8 steps
#pragma unroll
      for (int j = 0; j < VEC; ++j) sqf = __fmaf_rn(((valid >> j) & 1u) ? v[j] : 0.0f, v[j], sqf);
      if ((t & 7) == 7) { sqd += double(sqf); sqf = 0.0f; }
    }
    nib &= valid;
    if (!fin && bad == LLMAX) {  // rare: locate the neuron (padding lanes never count)
#pragma unroll
      for (int j = 0; j < VEC; ++j)
        if (!finitef_(v[j]) && ((valid >> j) & 1u)) bad = a.step_base + t;
    }
    if (FF_VO) {
      store4(vo, v);
      vo += a.v_ld;
    }
    if (FF_SVO) {
      float f[VEC];
#pragma unroll
      for (int j = 0; j < VEC; ++j) f[j] = ((nib >> j) & 1u) ? 1.0f : 0.0f;
      store4(svo, f);
      svo += a.spkv_ld;
    }
    if (FF_SVB) {   // bf16 0/1 (0x3F80 = 1.0): the next layer's GEMM operand, written beside the fp32 flags
      if (VEC == 4 && AL) {           // AL: the host checked 8-byte alignment of every row (spkb_ld % 4 == 0)
        const u32 lo = ((nib & 1u) ? 0x3F80u : 0u) | ((nib & 2u) ? 0x3F800000u : 0u);
        const u32 hi = ((nib & 4u) ? 0x3F80u : 0u) | ((nib & 8u) ? 0x3F800000u : 0u);
        *reinterpret_cast<uint2*>(sbo) = make_uint2(lo, hi);
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j)
          if (n0 + j < a.n) sbo[j] = ((nib >> j) & 1u) ? (unsigned short)0x3F80 : (unsigned short)0;
      }
      sbo += a.spkb_ld;
    }
    if (FF_SO) {
      u32 w;
      if (VEC == 1) {
        w = __ballot_sync(0xffffffffu, nib != 0);
      } else {
        w = nib << (VEC * (lane % (32 / VEC)));
#pragma unroll
        for (int o = 1; o < 32 / VEC; o <<= 1) w |= __shfl_xor_sync(0xffffffffu, w, o);
      }
      if (spk_writer) *so = w;
      so += a.spk_ld;
    }
  };
  // unrolled PF times so that the prefetch registers rotate by name: step
  // t + k consumes pre[k] (loaded PF steps earlier) and refills it
  for (i64 tb = 0; tb < a.steps; tb += PF) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      const i64 t = tb + k;
      if (PF > 1 && t >= a.steps) break;
      if (POIS) {
        stim.at(a, ks, ps, t, n0, full, cur);
      } else {
#pragma unroll
        // (PF > 1: an explicit add copies the value out, so the refill can
        // land in pre[k]'s own register instead of a temporary moved back at
        // the end of the step -- that move would wait for the load)
        for (int j = 0; j < VEC; ++j) cur[j] = PF > 1 ? __fadd_rn(pre[k][j], 0.0f) : pre[k][j];
        if (PF > 1) load_row(t + PF, pre[k]);
        else if (t + PF < a.steps) load_in(pre[k]);
      }
      body(t);
    }
  }
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    if (n0 + j < a.n) {
      a.v_fin[n0 + j] = v[j];
#pragma unroll
      for (int g = 0; g < NG; ++g) a.g_fin[g * a.g_ld + n0 + j] = p[j][g];
    }
  }
  if (bad != LLMAX) atomicMin(reinterpret_cast<long long*>(a.first_bad), (long long)bad);
  if (FF_L2) {   // block partial: warp shuffle, then the warps in a fixed order
    __shared__ double red[8];
    double x = sqd + double(sqf);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) red[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      double y = 0.0;
      for (int w = 0; w < int(blockDim.x >> 5); ++w) y += red[w];
      a.sq_part[blockIdx.x] = y;
    }
  }
}
extern "C" __global__ void __launch_bounds__(256, FWD_MINB) hh_fwd_v1(const FwdArgs a, const PoissonTab t, const Keys k) { fwd_body<1, false>(a, t, k); }
extern "C" __global__ void __launch_bounds__(256, FWD_MINB) hh_fwd_v4(const FwdArgs a, const PoissonTab t, const Keys k) { fwd_body<4, false>(a, t, k); }
extern "C" __global__ void __launch_bounds__(256, FWD_MINB) hh_fwdp_v1(const FwdArgs a, const PoissonTab t, const Keys k) { fwd_body<1, true>(a, t, k); }
extern "C" __global__ void __launch_bounds__(256, FWD_MINB) hh_fwdp_v4(const FwdArgs a, const PoissonTab t, const Keys k) { fwd_body<4, true>(a, t, k); }

)";

// Persistent network kernel (BASELINE config 5, one rank): every network
// step of cortex.py:273-310 -- ring drain + PSP + Philox background, the HH
// step, spike bitmap, synapse delivery -- for `steps` steps in ONE cooperative
// launch.  Block b owns the 256-neuron tile b (state in registers for the
// whole launch) and is the only writer of its tile's ring columns: after the
// grid barrier that publishes a step's spike bitmap, every block lists the
// spiking sources and delivers, from each source's target-sorted synapse row,
// just the segment that lands in its tile (seg[source][tile], precomputed).
// One grid barrier per step; the ring drain of the next step needs only the
// block's own barrier.  The input arithmetic is that of k_cortex_input
// (cortex.cu, explicit roundings on both sides), the step the same step_fwd as
// the forward module, the ring int64 fixed point: rasters, state and ring are
// bit-identical to the per-step kernels.
static const char* kNetKernel = R"(
struct NetArgs { i64 n, steps, t0, depth; long long* ring; float* psp; const double* lam;
  float decay, mu, sigma, w_scale; int mode, rec; unsigned long long seed; i64 nbase;
  float* v; float* g; i64 g_ld; u32* bits; i64 words; const i64* seg; i64 tiles; const int* tgt; const int* w;
  const int* delay; i64* first_bad; unsigned* bar; unsigned long long* timing; i64 reps, ld;
  const i64* th_off; const float* th_w; i64 th_base, th_on, th_end; unsigned th_thr; unsigned long long th_seed; };
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long x;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(x));
  return x;
}
__device__ __forceinline__ uint4 philox_full(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const u32 hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const u32 hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}
// compound Poisson N mu + sigma sqrt(N) z (cortex.py:225-232), as cortex.cu bg_draw_f32
__device__ __forceinline__ float bg_draw(float L, float mu, float sigma, uint4 r) {
  const float u = __fmul_rn(__fadd_rn(__uint2float_rn(r.x), 0.5f), 2.3283064365386963e-10f);
  float p = __expf(-L), c = p;
  int k = 0;
  while (u > c && k < 64) {
    ++k;
    p = __fmul_rn(p, __fdividef(L, float(k)));
    c = __fadd_rn(c, p);
  }
  float add = __fmul_rn(float(k), mu);
  if (sigma > 0.0f && k > 0) {
    const float u1 = __fmul_rn(__fadd_rn(__uint2float_rn(r.y), 0.5f), 2.3283064365386963e-10f);
    const float u2 = __fmul_rn(__fadd_rn(__uint2float_rn(r.z), 0.5f), 2.3283064365386963e-10f);
    const float z = __fmul_rn(__fsqrt_rn(__fmul_rn(-2.0f, __logf(u1))), __cosf(__fmul_rn(6.283185307179586f, u2)));
    add = __fadd_rn(add, __fmul_rn(__fmul_rn(sigma, __fsqrt_rn(float(k))), z));
  }
  return add;
}
// thalamic current of neuron i at step t: cortex.cu thal_sum<float>, verbatim
__device__ __forceinline__ float thal_sum(const NetArgs& a, i64 i, i64 t) {
  const i64 k0 = a.th_off[i], k1 = a.th_off[i + 1];
  float s = 0.0f;
  for (i64 g = (a.th_base + k0) >> 2; 4 * g - a.th_base < k1; ++g) {
    const uint4 r = philox_full(make_uint4(u32(g), u32((unsigned long long)g >> 32), u32(t),
                                           u32((unsigned long long)t >> 32)),
                                make_uint2(u32(a.th_seed), u32(a.th_seed >> 32)));
    const u32 wd[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const i64 k = 4 * g + q - a.th_base;
      if (k >= k0 && k < k1 && wd[q] < a.th_thr) s = __fadd_rn(s, a.th_w[k]);
    }
  }
  return s;
}
// grid barrier on a monotonic arrival counter (zeroed by the host per launch);
// the launch is cooperative, so every block is resident.  (Measured against a
// barrier-free exchange of tagged 64-bit spike words, whose polling by every
// thread swamped L2: 9.3 vs 14.9 us per config-5 step.)
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // release-add (cumulative over the block's writes ordered by the bar.sync),
    // relaxed polling (an acquire load would invalidate L1 on every spin), one
    // acquire fence after
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned seen;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
    } while (seen < target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
// the same barrier split in two, so that work can run between the arrival and
// the wait: grid_arrive after the block's writes, grid_wait before reading the
// other blocks' writes
__device__ __forceinline__ void grid_arrive(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}
__device__ __forceinline__ void grid_wait(unsigned* bar, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned seen;
    do {
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(bar) : "memory");
    } while (seen < target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
#define NET_THREADS 256
// deliveries with delay >= 3 of one step, parked until the next step's barrier
// wait (they land in ring rows >= t + 3: nothing reads them sooner)
#ifndef NET_PEND
#define NET_PEND 2048
#endif
// exclusive block scan of one value per thread (warp shuffles + one smem pass)
__device__ __forceinline__ i64 block_scan(i64 x, i64* s_w, i64& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  i64 inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const i64 y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) s_w[wid] = inc;
  __syncthreads();
  i64 before = 0;
  total = 0;
#pragma unroll
  for (int k = 0; k < NET_THREADS / 32; ++k) {
    const i64 wv = s_w[k];
    if (k < wid) before += wv;
    total += wv;
  }
  __syncthreads();
  return before + inc - x;
}
// NET_REPS independent replicas of the network (CortexReplicas; 1 for one
// network) share the launch, the tiles and the barrier: replica r's neurons,
// PSP and ring live at r * ld (ring rows: r * depth * ld), its spike words at
// r * words of the step's bitmap block, its background key is seed + r.
#ifndef NET_REPS
#define NET_REPS 1
#endif
extern "C" __global__ void __launch_bounds__(NET_THREADS) hh_net(const NetArgs a) {
  constexpr int R = NET_REPS;
  // dynamic: step t's delay-1 deliveries into the tile, and ring row t + 1 of
  // the tile (cp.async prefetch), per replica
  extern __shared__ __align__(16) unsigned long long s_dyn[];
  unsigned long long (*s_next)[NET_THREADS] = reinterpret_cast<unsigned long long (*)[NET_THREADS]>(s_dyn);
  long long (*s_ahead)[NET_THREADS] = reinterpret_cast<long long (*)[NET_THREADS]>(s_dyn + R * NET_THREADS);
  // step t's delay-2 deliveries (ring row t + 2), shifted into s_next when step t + 1 starts
  unsigned long long (*s_next2)[NET_THREADS] =
      reinterpret_cast<unsigned long long (*)[NET_THREADS]>(s_dyn + 2 * R * NET_THREADS);
  __shared__ int s_poff[NET_PEND];                        // parked deliveries: ring offset, weight
  __shared__ int s_pw[NET_PEND];
  __shared__ int s_np;
  __shared__ int s_src[NET_CAP];                          // spiking sources, replica in bits 20+
  __shared__ int s_beg[NET_CAP];                          // (synapse indices < 2^31)
  __shared__ int s_pre[NET_CAP + 1];
  __shared__ i64 s_w[NET_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31;
  const unsigned nb = gridDim.x;
  unsigned phase = 0;
  const i64 tile = blockIdx.x;                    // host: gridDim.x == tiles
  const i64 i = tile * NET_THREADS + tid;
  const bool on = i < a.n;
  const i64 rring = a.depth * a.ld;               // one replica's ring
  // the tile's state lives in registers for the whole launch
  float vv[R], psp[R], pp[R][NGX];
  const float lam = (on && a.mode == 2) ? float(a.lam[i]) : 0.0f;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    vv[r] = on ? a.v[r * a.ld + i] : -65.0f;
    psp[r] = on ? a.psp[r * a.ld + i] : 0.0f;
#pragma unroll
    for (int q = 0; q < NGX; ++q) pp[r][q] = (on && q < NG) ? a.g[q * a.g_ld + r * a.ld + i] : 0.5f;
  }
  const i64 per = (a.words + NET_THREADS - 1) / NET_THREADS;
  const i64 w0 = tid * per, w1 = min(a.words, w0 + per);
  const i64 tlo = tile * NET_THREADS;             // this tile's neurons [tlo, tlo + NET_THREADS)
  // Ring row t + 1 of the tile is complete, except for step t's delay-1
  // synapses, once step t starts: it is read (and cleared) then, off the
  // critical path, and the delay-1 deliveries of step t go to s_next instead.
  // int64 sums commute: the drained values are those of the per-step kernels.
  // The row is copied asynchronously (cp.async: the thread does not wait for
  // it) and cleared when consumed, one step later.
  const int depth = int(a.depth);
  int row = int(a.t0 % a.depth);                  // ring row of step t (32-bit modular counter)
  // 16-byte pairs need an even row stride (and the tile's last pair whole)
  const bool pair = (a.ld & 1) == 0 && (a.n & 1) == 0 && !NET_NOPAIR;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    s_next[r][tid] = 0ull;
    s_next2[r][tid] = 0ull;
    s_ahead[r][tid] = (on && a.steps > 0) ? __ldcg(a.ring + r * rring + i64(row) * a.ld + i) : 0ll;
  }
  if (tid == 0) s_np = 0;
  unsigned long long* tm = a.timing ? a.timing + blockIdx.x * 4 : nullptr;
  for (i64 s = 0; s < a.steps; ++s) {
    const i64 t = a.t0 + s;
    u32* bw = a.bits + (a.rec ? s : (s & 1)) * (R * a.words);
    if (tm && tid == 0) tm[s * nb * 4 + 0] = gtimer();
    // ---- input + HH step of the tile (padding lanes run the step on a dummy state)
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();                                // (pairs: thread 2k copied entries 2k and 2k + 1)
    long long arr[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      arr[r] = (pair ? s_ahead[r][tid] : (on ? __ldcg(a.ring + r * rring + i64(row) * a.ld + i) : 0ll)) +
               (long long)s_next[r][tid];
      s_next[r][tid] = s_next2[r][tid];             // step t - 1's delay-2 deliveries: row t + 1
      s_next2[r][tid] = 0ull;                       // (both written after this block's barriers)
    }
    const int row1 = row + 1 == depth ? 0 : row + 1;
    NET_CHK(row >= 0 && row < depth && i64(row) == (t % a.depth));
    __syncwarp();                                   // lane 2k+1 has read s_ahead before lane 2k refills it
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (on) a.ring[r * rring + i64(row) * a.ld + i] = 0;   // row t consumed
      if (pair && (tid & 1) == 0 && i < a.n && s + 1 < a.steps) {
        // 16-byte L2-only async copy of this and the next neuron's entries
        const unsigned sa = unsigned(__cvta_generic_to_shared(&s_ahead[r][tid]));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa),
                     "l"(a.ring + r * rring + i64(row1) * a.ld + i)
                     : "memory");
      }
    }
    if (pair && (tid & 1) == 0 && i < a.n && s + 1 < a.steps) asm volatile("cp.async.commit_group;" ::: "memory");
    float cur[R], vn[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      cur[r] = 0.0f;
      if (on) {
        float x = __fadd_rn(__fmul_rn(psp[r], a.decay), __fmul_rn(float(double(arr[r])), a.w_scale));
        if (a.mode == 2) {
          const unsigned long long sd = a.seed + (unsigned long long)r;
          const uint4 rv = philox_full(make_uint4(u32(i + a.nbase), u32((unsigned long long)(i + a.nbase) >> 32),
                                                  u32(t), u32((unsigned long long)t >> 32)),
                                       make_uint2(u32(sd), u32(sd >> 32)));
          x = __fadd_rn(x, bg_draw(lam, a.mu, a.sigma, rv));
        }
        psp[r] = x;
        cur[r] = x;
        // thalamic drive (one replica): added to this step's current, not the PSP
        if (a.th_off != nullptr && t >= a.th_on && t < a.th_end) cur[r] = __fadd_rn(x, thal_sum(a, i, t));
      }
    }
    // the R replicas' neurons as one VEC = R group: their steps interleave
    // under one warp vote (step_all, as the 4-neurons-per-thread forward)
    step_all<R>(vv, pp, cur, vn);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float vo = vv[r];
      vv[r] = vn[r];
      const bool spk = on && (vo < THETA) && (vv[r] >= THETA);
      if (on && !finitef_(vv[r])) atomicMin(reinterpret_cast<long long*>(a.first_bad), (long long)t);
      const u32 word = __ballot_sync(0xffffffffu, spk);
      if (lane == 0 && (i >> 5) < a.words) bw[r * a.words + (i >> 5)] = word;
    }
    if (tm) {
      __syncthreads();
      if (tid == 0) tm[s * nb * 4 + 1] = gtimer();
    }
    grid_arrive(a.bar);
    // between arrival and wait: the previous step's parked (delay >= 3) deliveries
    {
      const int np = min(s_np, NET_PEND);
      for (int k = tid; k < np; k += NET_THREADS)
        atomicAdd(reinterpret_cast<unsigned long long*>(a.ring + s_poff[k]),
                  (unsigned long long)(long long)s_pw[k]);
    }
    grid_wait(a.bar, ++phase * nb);
    if (tid == 0) s_np = 0;                         // (read above, before grid_wait's bar.sync)
    if (tm && tid == 0) tm[s * nb * 4 + 2] = gtimer();
    // ---- delivery into this tile: list the spiking sources of every replica ...
    // this thread's (<= 8) words of every replica, loaded together (one L2 round trip)
    u32 wr[R][8];
    int cnt = 0;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        wr[r][k] = (w0 + k < w1) ? __ldcg(bw + r * a.words + w0 + k) : 0u;
        cnt += __popc(wr[r][k]);
      }
    i64 ns = 0;
    const i64 first = block_scan(cnt, s_w, ns);
    for (i64 r0 = 0; r0 < ns; r0 += NET_CAP) {
      const i64 m = min(i64(NET_CAP), ns - r0);
      if (cnt > 0 && first < r0 + m && first + cnt > r0) {
        i64 k = first;
        auto emit = [&](u32 x, i64 wi, int r) {
          while (x) {
            const int b = __ffs(int(x)) - 1;
            x &= x - 1;
            if (k >= r0 && k < r0 + m) s_src[k - r0] = int(wi * 32 + b) | (r << 20);
            NET_CHK(wi * 32 + b < a.n);                  // no spike bit past the population
            ++k;
          }
        };
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int q = 0; q < 8; ++q) emit(wr[r][q], w0 + q, r);
      }
      __syncthreads();
      // ... each source's segment of synapses with targets in the tile ...
      i64 lsum = 0;
      const i64 c0 = (m * tid) / NET_THREADS, c1 = (m * (tid + 1)) / NET_THREADS;
      for (i64 c = c0; c < c1; ++c) {
        const i64* sg = a.seg + i64(s_src[c] & 0xFFFFF) * (a.tiles + 1) + tile;
        const i64 beg = __ldg(sg), end = __ldg(sg + 1);
        s_beg[c] = int(beg);
        s_pre[c] = int(end - beg);                // length, turned into a prefix below
        lsum += end - beg;
      }
      i64 total = 0;
      i64 run = block_scan(lsum, s_w, total);
      for (i64 c = c0; c < c1; ++c) {
        const i64 l = s_pre[c];
        s_pre[c] = int(run);
        run += l;
      }
      if (tid == 0) s_pre[m] = int(total);
      __syncthreads();
      NET_CHK(m <= NET_CAP && s_pre[0] == 0 && s_pre[m] == int(total) && total >= 0);
      // ... and one thread per (source, synapse) pair, NET_UNROLL pairs in
      // flight per thread (their loads overlap)
#ifndef NET_UNROLL
#define NET_UNROLL 4
#endif
      for (i64 g0 = tid; g0 < total; g0 += NET_THREADS * NET_UNROLL) {
        int d[NET_UNROLL], tg[NET_UNROLL], wv[NET_UNROLL], rr[NET_UNROLL];
#pragma unroll
        for (int u = 0; u < NET_UNROLL; ++u) {
          const i64 gi = g0 + u * NET_THREADS;
          d[u] = 0;
          if (gi < total) {
            int lo = 0, hi = int(m);
            while (hi - lo > 1) {
              const int mid = (lo + hi) >> 1;
              if (s_pre[mid] <= gi) lo = mid;
              else hi = mid;
            }
            const i64 j = s_beg[lo] + (gi - s_pre[lo]);
            rr[u] = s_src[lo] >> 20;
            d[u] = __ldg(a.delay + j);
            tg[u] = __ldg(a.tgt + j);
            wv[u] = __ldg(a.w + j);
            NET_CHK(lo >= 0 && lo < m && s_pre[lo] <= gi && gi < s_pre[lo + 1]);
            NET_CHK(j >= s_beg[lo] && rr[u] >= 0 && rr[u] < R);
            NET_CHK(tg[u] >= tlo && tg[u] < tlo + NET_THREADS && tg[u] < a.n);    // the tile's own segment
            NET_CHK(d[u] >= 1 && d[u] < depth);
          }
        }
#pragma unroll
        for (int u = 0; u < NET_UNROLL; ++u) {
          if (d[u] == 0) continue;
          const unsigned long long wq = (unsigned long long)(long long)wv[u];
          if (d[u] == 1) {
            atomicAdd(&s_next[R == 1 ? 0 : rr[u]][tg[u] - tlo], wq);
          } else if (d[u] == 2) {
            atomicAdd(&s_next2[R == 1 ? 0 : rr[u]][tg[u] - tlo], wq);
          } else {
            const int q = row + d[u] >= depth ? row + d[u] - depth : row + d[u];   // (t + d) % depth, d < depth
            const i64 off = (R == 1 ? 0 : rr[u]) * rring + i64(q) * a.ld + tg[u];
            const int k = atomicAdd(&s_np, 1);
            if (k < NET_PEND && off <= 0x7fffffffLL) {   // parked until the next barrier wait
              s_poff[k] = int(off);
              s_pw[k] = wv[u];
            } else {
              atomicAdd(reinterpret_cast<unsigned long long*>(a.ring + off), wq);
            }
          }
        }
      }
      __syncthreads();
    }
    if (tm && tid == 0) tm[s * nb * 4 + 3] = gtimer();
    row = row1;
  }
  __syncthreads();
  {   // the last step's parked deliveries
    const int np = min(s_np, NET_PEND);
    for (int k = tid; k < np; k += NET_THREADS)
      atomicAdd(reinterpret_cast<unsigned long long*>(a.ring + s_poff[k]), (unsigned long long)(long long)s_pw[k]);
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (on && a.steps > 0) {   // the last step's delay-1 and delay-2 deliveries back into the ring
      long long* slot = a.ring + r * rring + ((a.t0 + a.steps) % a.depth) * a.ld + i;
      *slot = *slot + (long long)s_next[r][tid];
      long long* slot2 = a.ring + r * rring + ((a.t0 + a.steps + 1) % a.depth) * a.ld + i;
      *slot2 = *slot2 + (long long)s_next2[r][tid];
    }
    if (on) {
      a.v[r * a.ld + i] = vv[r];
      a.psp[r * a.ld + i] = psp[r];
#pragma unroll
      for (int q = 0; q < NG; ++q) a.g[q * a.g_ld + r * a.ld + i] = pp[r][q];
    }
  }
}
)";

static const char* kBwdKernel = R"(
__device__ __forceinline__ void load_state(const float* base, i64 ld, i64 i, float& v, float (&p)[NGX]) {
  v = base[i];
#pragma unroll
  for (int g = 0; g < NG; ++g) p[g] = base[(1 + g) * ld + i];
}
__device__ __forceinline__ void store_state(float* base, i64 ld, i64 i, float v, const float (&p)[NGX]) {
  base[i] = v;
#pragma unroll
  for (int g = 0; g < NG; ++g) base[(1 + g) * ld + i] = p[g];
}
// Reverse-sweep operand prefetch: each thread streams its own operands of
// step t (state row, current, seeds) into a DEPTH-deep shared-memory ring with
// 4-byte cp.async, DEPTH-1 steps ahead of the step it computes, so HBM latency
// hides behind compute without holding the operands in registers.  The module
// is specialised on which optional streams exist (BF_* below), so the sweep
// carries no run-time tests; every stream advances by a running pointer.
#define DEPTH 8   // power of two: slot wrap is a mask
// ring slots per step: v, p[NG], cur, then seed_v (unless BF_SPREV reads it
// from the previous step's state) and seed_s only when the launch has them --
// a smaller ring leaves room for more resident blocks
#define SV_SLOT (NG + 2)
#define SS_SLOT (NG + 2 + ((BF_SV && !BF_SPREV) ? 1 : 0))
#define NOPS (SS_SLOT + (BF_SS ? 1 : 0))
#define RING_STRIDE (NOPS * BWD_THREADS)
__device__ __forceinline__ void cpa4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((u32)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH - 1) : "memory"); }

// VEC neurons per thread (1 or 2; 2 when the host proved every stream 8-byte
// aligned and neuron-contiguous): a block always covers BWD_THREADS neurons, so
// the partial-sum layout (one slot row per block) is the same for both.
template <int VEC>
__device__ __forceinline__ void cpa(float* dst, const float* src) {
  if (VEC == 2)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((u32)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((u32)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
}

template <int VEC>
__device__ __forceinline__ void bwd_body(const Sur& sur, const BwdArgs& a) {
  pdl_begin();
  constexpr int TPB = BWD_THREADS / VEC;
  __shared__ __align__(16) float ring[DEPTH * RING_STRIDE];
  const i64 i0 = i64(blockIdx.x) * BWD_THREADS + i64(threadIdx.x) * VEC;
  bool on[VEC];
  i64 ii[VEC];
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    on[j] = i0 + j < a.n;
    ii[j] = on[j] ? i0 + j : 0;
  }
  const i64 ib0 = on[0] ? i0 : 0;      // VEC == 2: the host guarantees n even (both or neither on)
  double acc[SLOTS];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) acc[s] = 0.0;
  float accf[SLOTS];
  cb_zero(accf);
  int nf = 0;
  double csum[VEC];
  float csumf[VEC];
  i64 bad = -1;
  float d_v[VEC], d_p[VEC][NGX];
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    csum[j] = 0.0;
    csumf[j] = 0.0f;
    d_v[j] = on[j] ? a.adj_v[ii[j]] : 0.0f;
#pragma unroll
    for (int g = 0; g < NG; ++g) d_p[j][g] = on[j] ? a.adj_g[g * a.ag_ld + ii[j]] : 0.0f;
  }
  const i64 K = BF_K1 ? 1 : a.ck_every;
  const float svs = BF_SVS ? *a.sv_scale : 1.0f;
  const i64 sstride = (1 + NG) * a.ck_ld;
  i64 goff[NGX];
#pragma unroll
  for (int g = 0; g < NG; ++g) goff[g] = (1 + g) * a.ck_ld;
  const float* ib = a.i_ext + ib0 * a.i_sn;
  const float* svb = BF_SV ? a.seed_v + ib0 : nullptr;
  const float* ssb = BF_SS ? a.seed_s + ib0 : nullptr;
  float* const ring_t = ring + threadIdx.x * VEC;
  // K == 1: one stream over all steps; K > 1: one stream per recomputed segment
  const i64 nseg = BF_K1 ? 1 : (a.steps + K - 1) / K;
  for (i64 seg = nseg - 1; seg >= 0; --seg) {
    const i64 lo = BF_K1 ? 0 : seg * K;
    const i64 hi = BF_K1 ? a.steps : ((lo + K < a.steps) ? lo + K : a.steps);
    const float* ck = a.ckpt + seg * sstride;
    if (!BF_K1) {
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        float v, p[NGX];
        load_state(ck, a.ck_ld, ii[j], v, p);
        float* sp = a.seg + sstride;
        const float* ip = a.i_ext + ii[j] * a.i_sn + lo * a.i_st;
        for (i64 t = lo; t < hi - 1; ++t) {
          v = step_fwd(v, p, __ldg(ip));
          ip += a.i_st;
          if (on[j]) store_state(sp, a.ck_ld, ii[j], v, p);
          sp += sstride;
        }
      }
    }
    // issue pointers: operands of step tn (walk down from hi - 1)
    const float* rq = BF_K1 ? a.ckpt + (hi - 1) * sstride + ib0 : a.seg + (hi - 1 - lo) * sstride + ib0;
    const float* iq = ib + (hi - 1) * a.i_st;
    const float* vq = BF_SV ? svb + (hi - 1) * a.sv_ld : nullptr;
    const float* sq = BF_SS ? ssb + (hi - 1) * a.ss_ld : nullptr;
    i64 tn = hi - 1;
    int wslot = 0;
    auto issue = [&]() {
      float* r = ring_t + wslot * RING_STRIDE;
      const float* src = (!BF_K1 && tn == lo) ? ck + ib0 : rq;
      cpa<VEC>(r, src);
#pragma unroll
      for (int g = 0; g < NG; ++g) cpa<VEC>(r + (1 + g) * BWD_THREADS, src + goff[g]);
      cpa<VEC>(r + (NG + 1) * BWD_THREADS, iq);
      if (BF_SV && !BF_SPREV) cpa<VEC>(r + SV_SLOT * BWD_THREADS, vq);
      if (BF_SS) cpa<VEC>(r + SS_SLOT * BWD_THREADS, sq);
    };
    auto advance = [&]() {
      --tn;
      rq -= sstride;
      iq -= a.i_st;
      if (BF_SV) vq -= a.sv_ld;
      if (BF_SS) sq -= a.ss_ld;
      wslot = (wslot + 1) & (DEPTH - 1);
    };
#pragma unroll
    for (int k = 0; k < DEPTH - 1; ++k) {
      if (tn >= lo) issue();
      cpa_commit();
      advance();
    }
    float* dib = (BF_DI && on[0]) ? a.d_i + (hi - 1) * a.di_ld + ib0 : nullptr;
    const i64 scol = a.dh_grp > 0 ? (ib0 / a.dh_grp) * a.dh_pitch + ib0 % a.dh_grp : ib0;
    unsigned short* dhb = (BF_SPLIT && on[0]) ? a.di_hi + (hi - 1) * a.dh_ld + scol : nullptr;
    unsigned short* dlb = (BF_SPLIT && on[0]) ? a.di_lo + (hi - 1) * a.dh_ld + scol : nullptr;
    int rslot = 0;
    // BF_SPREV: the seed of step t is svs * V'(t), and V'(t) is the v of state
    // t + 1 -- loaded by the previous (later) step of this reverse sweep, so
    // only the final state's v is read here
    float vprev[VEC];
#pragma unroll
    for (int j = 0; j < VEC; ++j) vprev[j] = (BF_SPREV && on[j]) ? a.seed_v[(hi - 1) * a.sv_ld + ii[j]] : 0.0f;
    for (i64 t = hi - 1; t >= lo; --t) {
      if (tn >= lo) issue();
      cpa_commit();
      advance();
      cpa_wait();
      const float* r = ring_t + rslot * RING_STRIDE;
      NET_CHK(rslot == int((hi - 1 - t) & (DEPTH - 1)) && wslot == int((hi - 1 - tn) & (DEPTH - 1)));
      NET_CHK(tn == t - DEPTH && t >= lo && t < hi);
      rslot = (rslot + 1) & (DEPTH - 1);
      float di[VEC], v[VEC], p[VEC][NGX], cur[VEC], ds[VEC];
      bool reg = true;
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        v[j] = r[j];
#pragma unroll
        for (int g = 0; g < NG; ++g) p[j][g] = r[(1 + g) * BWD_THREADS + j];
        cur[j] = r[(NG + 1) * BWD_THREADS + j];
        if (BF_SPREV) {
          d_v[j] = __fmaf_rn(svs, vprev[j], d_v[j]);
          vprev[j] = v[j];
        } else if (BF_SV) {
          d_v[j] = BF_SVS ? __fmaf_rn(svs, r[SV_SLOT * BWD_THREADS + j], d_v[j])
                          : __fadd_rn(d_v[j], r[SV_SLOT * BWD_THREADS + j]);
        }
        ds[j] = BF_SS ? r[SS_SLOT * BWD_THREADS + j] : 0.0f;
#if HAS_MERGED
        reg = reg && regular(v[j]);
#endif
      }
#if HAS_MERGED
      // one warp vote per step for all VEC neurons of every lane
      if (__all_sync(0xffffffffu, reg)) {
#if BWD_PAIR
        if (VEC == 2) {   // both neurons per f32x2 op
          constexpr int k = VEC - 1;
          F2 q[NGX], dq[NGX], ac[SLOTS];
#pragma unroll
          for (int g = 0; g < NGX; ++g) {
            q[g] = F2(p[0][g], p[k][g]);
            dq[g] = F2(d_p[0][g], d_p[k][g]);
          }
#pragma unroll
          for (int s = 0; s < SLOTS; ++s) ac[s] = F2(accf[s], 0.0f);   // y: this step's second neuron
          F2 dv(d_v[0], d_v[k]);
          const F2 r = step_bwd_m2<false>(sur, F2(v[0], v[k]), q, F2(cur[0], cur[k]), dv, dq, F2(ds[0], ds[k]),
                                          BF_SS, ac);
          di[0] = r.x;
          di[k] = r.y;
          d_v[0] = dv.x;
          d_v[k] = dv.y;
#pragma unroll
          for (int g = 0; g < NGX; ++g) {
            d_p[0][g] = dq[g].x;
            d_p[k][g] = dq[g].y;
          }
#pragma unroll
          for (int s = 0; s < SLOTS; ++s) accf[s] = __fadd_rn(ac[s].x, ac[s].y);
        } else
#endif
        {
#pragma unroll
          for (int j = 0; j < VEC; ++j)
            di[j] = step_bwd_m(sur, v[j], p[j], cur[j], d_v[j], d_p[j], ds[j], BF_SS, accf);
        }
      } else {
#pragma unroll
        for (int j = 0; j < VEC; ++j)
          di[j] = step_bwd_irr(sur, v[j], p[j], cur[j], d_v[j], d_p[j], ds[j], BF_SS, accf);
      }
#else
#pragma unroll
      for (int j = 0; j < VEC; ++j) di[j] = step_bwd(sur, v[j], p[j], cur[j], d_v[j], d_p[j], ds[j], BF_SS, accf);
#endif
      if (BF_SUM) {
#pragma unroll
        for (int j = 0; j < VEC; ++j) csumf[j] = __fadd_rn(csumf[j], di[j]);
      }
      if (++nf == 8) {
        cb_flush(acc, accf);
        if (BF_SUM) {
#pragma unroll
          for (int j = 0; j < VEC; ++j) {
            csum[j] += double(csumf[j]);
            csumf[j] = 0.0f;
          }
        }
        nf = 0;
      }
      if (BF_DI && on[0]) {
        if (VEC == 2) *reinterpret_cast<float2*>(dib) = make_float2(di[0], di[VEC - 1]);
        else *dib = di[0];
        dib -= a.di_ld;
      }
      if (BF_SPLIT && on[0]) {
        unsigned short h[VEC], l[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) split_bf16(di[j], h[j], l[j]);
        if (VEC == 2) {
          *reinterpret_cast<u32*>(dhb) = u32(h[0]) | (u32(h[VEC - 1]) << 16);
          *reinterpret_cast<u32*>(dlb) = u32(l[0]) | (u32(l[VEC - 1]) << 16);
        } else {
          *dhb = h[0];
          *dlb = l[0];
        }
        dhb -= a.dh_ld;
        dlb -= a.dh_ld;
      }
      bool ok = true;
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        ok = ok && finitef_(d_v[j]);
#pragma unroll
        for (int g = 0; g < NG; ++g) ok = ok && finitef_(d_p[j][g]);
      }
      if (!ok && bad < 0 && on[0]) bad = a.step_base + t;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  cb_flush(acc, accf);
#pragma unroll
  for (int j = 0; j < VEC; ++j) {
    csum[j] += double(csumf[j]);
    if (on[j]) {
      a.adj_v[ii[j]] = d_v[j];
#pragma unroll
      for (int g = 0; g < NG; ++g) a.adj_g[g * a.ag_ld + ii[j]] = d_p[j][g];
      if (BF_SUM) a.di_sum[ii[j]] += float(csum[j]);
    }
  }
  if (bad >= 0) atomicMax(reinterpret_cast<long long*>(a.first_bad), (long long)bad);
  __shared__ double red[TPB / 32][SLOTS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    double x = on[0] ? acc[s] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) red[warp][s] = x;
  }
  __syncthreads();
  if (threadIdx.x < SLOTS) {
    double x = 0.0;
    for (int w = 0; w < TPB / 32; ++w) x += red[w][threadIdx.x];
    a.partials[i64(blockIdx.x) * SLOTS + threadIdx.x] = x;
  }
}
extern "C" __global__ void __launch_bounds__(BWD_THREADS, BWD_MINB) hh_bwd(const Sur sur, const BwdArgs a) {
  bwd_body<1>(sur, a);
}
extern "C" __global__ void __launch_bounds__(BWD_THREADS / 2, BWD2_MINB) hh_bwd2(const Sur sur, const BwdArgs a) {
  bwd_body<2>(sur, a);
}
)";

// kind >= 0: the backward module specialised on BF_* (kind = flags);
// kInspect: both (forward with the generic stream flags), for hhb_jit_source;
// otherwise the forward module specialised on FF_* (kind = -1 - flags).
// bwd_flags < 0: the forward module; >= 0: the backward module specialised
// on BF_* (which optional streams the launch has); -2: both, for inspection
enum { BF_SV = 1, BF_SS = 2, BF_DI = 4, BF_SPLIT = 8, BF_SUM = 16, BF_K1 = 32, BF_SVS = 64, BF_SPREV = 128 };
enum { FF_VO = 1, FF_SO = 2, FF_SVO = 4, FF_CK = 8, FF_AL = 16, FF_L2 = 32, FF_SVB = 64 };
constexpr int kInspect = -1000;
constexpr int kNet = -2000;   // the persistent network kernel (hh_net)
static int fwd_kind(int ff) { return -1 - ff; }
static std::string generate(const hhb_params_t* P, int bwd_flags = kInspect) {
  const Layout L = layout_of(P);
  // HHB_JIT_CHECK=1: device-side bounds / invariant checks that trap (the
  // substitute for compute-sanitizer, which this GPU pool does not allow)
  const char* chk = getenv("HHB_JIT_CHECK");
  std::string src = fmt("#define HHB_CHECK %d\n", chk && atoi(chk) > 0 ? 1 : 0);
  src += kPrelude;
  src += fmt("#define NG %d\n#define NGX %d\n#define SLOTS %d\n#define BWD_THREADS %d\n", L.ng,
             L.ng > 0 ? L.ng : 1, kSlots, kBwdThreads);
  src += fmt("#define THETA %s\n", F(P->v_theta).c_str());
  // occupancy knob for experiments: minimum resident 256-thread blocks per SM
  const char* mb = getenv("HHB_JIT_MINB");
  // merged step: 2 resident 256-thread blocks (<= 128 registers, no spills)
  // measured best for config 2 on B200 (profiles/r1_variants.md: 1.49e11 vs
  // 1.47e11 at 3 and 1.43e11 at 4, where 64 registers spill)
  src += fmt("#define FWD_MINB %d\n", mb ? atoi(mb) : 2);
  const char* pf = getenv("HHB_JIT_FWD_PF");
  src += fmt("#define FWD_PF %d\n", pf && atoi(pf) > 0 ? atoi(pf) : 8);
  const char* pf4 = getenv("HHB_JIT_FWD_PF4");
  // 4-neuron threads reading a current: 2 rows in flight (config-3 training
  // forward 128 -> 122 us, config 4 270 -> 261 us per hidden layer; 3-4: same)
  src += fmt("#define FWD_PF4 %d\n", pf4 && atoi(pf4) > 0 ? atoi(pf4) : 2);
  // one-neuron callers of the paired step: both halves' MUFU ops (0) or the x
  // half's only, the y half copied (1: a MOV after every MUFU op on the chain)
  const char* fh = getenv("HHB_JIT_FWD_HALF");
  src += fmt("#define FWD_HALF %d\n", fh && atoi(fh) > 0 ? 1 : 0);
  // 2-neuron BPTT: 8 resident 64-thread blocks (128 registers, no spills; the
  // operand ring holds only the launch's streams, 21.8 KB): 212 us vs 220 us
  // at 6 blocks for the config-3 step (profiles/r2_bptt.md)
  const char* bmb2 = getenv("HHB_JIT_BWD2_MINB");
  src += fmt("#define BWD2_MINB %d\n", bmb2 ? atoi(bmb2) : 8);
  const char* bmb = getenv("HHB_JIT_BWD_MINB");
  // 6 resident 128-thread blocks (<= 80 registers, no spills for up to 6 gates)
  // measured best at the config-3 shape: 259 us vs 276 us unconstrained
  src += fmt("#define BWD_MINB %d\n", bmb ? atoi(bmb) : 6);
  src += emit_near_linoid(P);
  src += emit_forward_step(P, L, kFast);
  src += emit_forward_step(P, L, kSeries);
  src += emit_backward_step(P, L, kFast);
  src += emit_backward_step(P, L, kSeries);
  const mg::Plan M = mg::disabled() ? mg::Plan{} : mg::plan_of(P);
  if (M.ok) {
    // merged form on every regular lane; one warp vote per step sends the
    // warp through the per-lane select only when some lane left the window
    {
      // regular(), then the paired merged step and its one-neuron wrapper
      const std::string st = mg::emit_step(P, L, M);
      const size_t k = st.find("__device__ __forceinline__ float step_fwd_m(");
      src += st.substr(0, k);
      src += mg::kPairPrelude;
      src += mg::pair(st.substr(k), "step_fwd_m");
      // the network kernel (one neuron per thread, its own module: nothing
      // else reproduces its states) keeps the scalar merged step
      src += fmt("#define FWD_PAIR %d\n", bwd_flags <= kNet ? 0 : 1);
      if (bwd_flags <= kNet) src += st.substr(k);
      else src += fmt(
          "__device__ __forceinline__ float step_fwd_m(const float v, float (&p)[%d], const float cur) {\n"
          "  F2 q[NGX];\n"
          "#pragma unroll\n  for (int g = 0; g < NGX; ++g) q[g] = F2(p[g]);\n"
          "  const F2 r = step_fwd_m2<FWD_HALF>(F2(v), q, F2(cur));\n"
          "#pragma unroll\n  for (int g = 0; g < NGX; ++g) p[g] = q[g].x;\n"
          "  return r.x;\n}\n",
          L.ng > 0 ? L.ng : 1);
    }
    src += R"(template <int VEC>
__device__ __forceinline__ void step_all(const float (&v)[VEC], float (&p)[VEC][NGX], const float (&cur)[VEC],
                                         float (&vn)[VEC]) {
  bool irr = false;
#pragma unroll
  for (int j = 0; j < VEC; ++j) irr = irr || !regular(v[j]);
  if (__any_sync(0xffffffffu, irr)) {
    if (FWD_PAIR && VEC % 2 == 0) {
      // merged form for both neurons of a pair, the series form per neuron
#pragma unroll
      for (int j = 0; j < VEC; j += 2) {
        const int k = VEC > 1 ? j + 1 : 0;
        F2 q[NGX];
#pragma unroll
        for (int g = 0; g < NGX; ++g) q[g] = F2(p[j][g], p[k][g]);
        const F2 r = step_fwd_m2<false>(F2(v[j], v[k]), q, F2(cur[j], cur[k]));
        const bool rj = regular(v[j]), rk = regular(v[k]);
        const float sj = step_fwd_s(v[j], p[j], cur[j]);
        const float sk = step_fwd_s(v[k], p[k], cur[k]);
        vn[j] = rj ? r.x : sj;
        vn[k] = rk ? r.y : sk;
#pragma unroll
        for (int g = 0; g < NGX; ++g) {
          p[j][g] = rj ? q[g].x : p[j][g];
          p[k][g] = rk ? q[g].y : p[k][g];
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < VEC; ++j) {
        float pm[NGX];
#pragma unroll
        for (int g = 0; g < NGX; ++g) pm[g] = p[j][g];
        const float vm = step_fwd_m(v[j], pm, cur[j]);
        const bool reg = regular(v[j]);
        const float vs = step_fwd_s(v[j], p[j], cur[j]);
        vn[j] = reg ? vm : vs;
#pragma unroll
        for (int g = 0; g < NGX; ++g) p[j][g] = reg ? pm[g] : p[j][g];
      }
    }
  } else if (FWD_PAIR && VEC % 2 == 0) {
    // two neurons per f32x2 op
#pragma unroll
    for (int j = 0; j < VEC; j += 2) {
      const int k = VEC > 1 ? j + 1 : 0;
      F2 q[NGX];
#pragma unroll
      for (int g = 0; g < NGX; ++g) q[g] = F2(p[j][g], p[k][g]);
      const F2 r = step_fwd_m2<false>(F2(v[j], v[k]), q, F2(cur[j], cur[k]));
      vn[j] = r.x;
      vn[k] = r.y;
#pragma unroll
      for (int g = 0; g < NGX; ++g) {
        p[j][g] = q[g].x;
        p[k][g] = q[g].y;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < VEC; ++j) vn[j] = step_fwd_m(v[j], p[j], cur[j]);
  }
}
)";
  } else {
    // one warp vote per step for all VEC neurons of every lane: the
    // branch-free variant unless a neuron sits in a linoid's series region
    src += "// merged form off: " + M.why + "\n";
    src += R"(template <int VEC>
__device__ __forceinline__ void step_all(const float (&v)[VEC], float (&p)[VEC][NGX], const float (&cur)[VEC],
                                         float (&vn)[VEC]) {
  bool near = false;
#pragma unroll
  for (int j = 0; j < VEC; ++j) near = near || near_linoid(v[j]);
  if (__any_sync(0xffffffffu, near)) {
#pragma unroll
    for (int j = 0; j < VEC; ++j) vn[j] = step_fwd_s(v[j], p[j], cur[j]);
  } else {
#pragma unroll
    for (int j = 0; j < VEC; ++j) vn[j] = step_fwd_f(v[j], p[j], cur[j]);
  }
}
)";
  }
  // one-neuron step (the backward's segment recompute): same dispatch, so it
  // reproduces the forward's states bit for bit
  src += fmt(
      "__device__ __forceinline__ float step_fwd(const float v, float (&p)[%d], const float cur) {\n"
      "  float vv[1] = {v}, cc[1] = {cur}, vn[1];\n"
      "  float pp[1][NGX];\n"
      "#pragma unroll\n  for (int g = 0; g < NGX; ++g) pp[0][g] = p[g];\n"
      "  step_all<1>(vv, pp, cc, vn);\n"
      "#pragma unroll\n  for (int g = 0; g < NGX; ++g) p[g] = pp[0][g];\n"
      "  return vn[0];\n}\n",
      L.ng > 0 ? L.ng : 1);
  // parameter-gradient contributions of one step: fp32 per step, added into
  // fp32 partials that are flushed into fp64 every 8 steps (fixed order, so
  // the sums do not depend on the checkpoint plan)
  {
    std::vector<int> used = {0};
    for (int g = 0; g < L.ng; ++g)
      if (L.last[g]) used.push_back(1 + g);
    for (size_t j = 0; j < L.leak_ch.size(); ++j) used.push_back(1 + kMaxGates + int(j));
    std::string add = "__device__ __forceinline__ void cb_add(float (&a)[SLOTS], const float (&c)[SLOTS]) {\n";
    std::string fl = "__device__ __forceinline__ void cb_flush(double (&d)[SLOTS], float (&a)[SLOTS]) {\n";
    std::string ze = "__device__ __forceinline__ void cb_zero(float (&a)[SLOTS]) {\n";
    std::string se = "__device__ __forceinline__ void cb_sel(bool q, float (&a)[SLOTS], const float (&c)[SLOTS]) {\n";
    std::string cp = "__device__ __forceinline__ void cb_copy(float (&a)[SLOTS], const float (&c)[SLOTS]) {\n";
    for (int k : used) {
      add += fmt("  a[%d] = __fadd_rn(a[%d], c[%d]);\n", k, k, k);
      fl += fmt("  d[%d] += double(a[%d]); a[%d] = 0.0f;\n", k, k, k);
      ze += fmt("  a[%d] = 0.0f;\n", k);
      se += fmt("  a[%d] = q ? c[%d] : a[%d];\n", k, k, k);
      cp += fmt("  a[%d] = c[%d];\n", k, k);
    }
    src += add + "}\n" + fl + "}\n" + ze + "}\n" + se + "}\n" + cp + "}\n";
  }
  const char* bwd_sig =
      "__device__ __forceinline__ float step_bwd(const Sur& sur, const float v, const float (&p)[NGX], "
      "const float cur, float& d_v, float (&d_p)[NGX], const float d_spike, const bool has_s, float (&cb)[SLOTS])";
  if (M.ok) {
    // the adjoint step stays scalar by default: paired, the BPTT kernel lost
    // ILP at its register budget (config 3: 203 -> 219 us, spills; DESIGN.md
    // section 8); HHB_JIT_BWD_PAIR=1 selects the paired form.  Either way the
    // segment recompute runs the forward's own (paired) step.
    const char* bp = getenv("HHB_JIT_BWD_PAIR");
    const bool bwd_pair = bp && atoi(bp) > 0;
    src += fmt("#define BWD_PAIR %d\n", bwd_pair ? 1 : 0);
    if (!bwd_pair) {
      src += emit_backward_step(P, L, kSeries, &M);
    } else {
      const std::string bm = emit_backward_step(P, L, kSeries, &M);
      src += mg::pair(bm, "step_bwd_m");
      src += fmt(
          "__device__ __forceinline__ float step_bwd_m(const Sur& sur, const float v, const float (&p)[%d], "
          "const float cur, float& d_v, float (&d_p)[%d], const float d_spike, const bool has_s, float (&acc)[SLOTS]) {\n"
          "  F2 q[NGX], dq[NGX], ac[SLOTS];\n"
          "#pragma unroll\n  for (int g = 0; g < NGX; ++g) { q[g] = F2(p[g]); dq[g] = F2(d_p[g]); }\n"
          "#pragma unroll\n  for (int s = 0; s < SLOTS; ++s) ac[s] = F2(acc[s]);\n"
          "  F2 dv(d_v);\n"
          "  const F2 r = step_bwd_m2<true>(sur, F2(v), q, F2(cur), dv, dq, F2(d_spike), has_s, ac);\n"
          "  d_v = dv.x;\n"
          "#pragma unroll\n  for (int g = 0; g < NGX; ++g) d_p[g] = dq[g].x;\n"
          "#pragma unroll\n  for (int s = 0; s < SLOTS; ++s) acc[s] = ac[s].x;\n"
          "  return r.x;\n}\n",
          L.ng > 0 ? L.ng : 1, L.ng > 0 ? L.ng : 1);
    }
    src += "#define HAS_MERGED 1\n";
    src += R"(// some lane of the warp left the merged form's window: both forms, per lane
__device__ __forceinline__ float step_bwd_irr(const Sur& sur, const float v, const float (&p)[NGX], const float cur,
                                           float& d_v, float (&d_p)[NGX], const float d_spike, const bool has_s,
                                           float (&cb)[SLOTS]) {
  float dvm = d_v, dpm[NGX], accm[SLOTS];
#pragma unroll
  for (int g = 0; g < NGX; ++g) dpm[g] = d_p[g];
  cb_copy(accm, cb);
  const float dim = step_bwd_m(sur, v, p, cur, dvm, dpm, d_spike, has_s, accm);
  const float dis = step_bwd_s(sur, v, p, cur, d_v, d_p, d_spike, has_s, cb);
  const bool reg = regular(v);
  d_v = reg ? dvm : d_v;
#pragma unroll
  for (int g = 0; g < NGX; ++g) d_p[g] = reg ? dpm[g] : d_p[g];
  cb_sel(reg, cb, accm);
  return reg ? dim : dis;
}
)";
    src += std::string(bwd_sig) + R"( {
  if (__all_sync(0xffffffffu, regular(v))) return step_bwd_m(sur, v, p, cur, d_v, d_p, d_spike, has_s, cb);
  // some lane left the window: both forms, selected per lane
  float dvm = d_v, dpm[NGX], accm[SLOTS];
#pragma unroll
  for (int g = 0; g < NGX; ++g) dpm[g] = d_p[g];
  cb_copy(accm, cb);
  const float dim = step_bwd_m(sur, v, p, cur, dvm, dpm, d_spike, has_s, accm);
  const float dis = step_bwd_s(sur, v, p, cur, d_v, d_p, d_spike, has_s, cb);
  const bool reg = regular(v);
  d_v = reg ? dvm : d_v;
#pragma unroll
  for (int g = 0; g < NGX; ++g) d_p[g] = reg ? dpm[g] : d_p[g];
  cb_sel(reg, cb, accm);
  return reg ? dim : dis;
}
)";
  } else {
    src += "#define HAS_MERGED 0\n";
    src += std::string(bwd_sig) + R"( {
  return __any_sync(0xffffffffu, near_linoid(v)) ? step_bwd_s(sur, v, p, cur, d_v, d_p, d_spike, has_s, cb)
                                                 : step_bwd_f(sur, v, p, cur, d_v, d_p, d_spike, has_s, cb);
}
)";
  }
  if (bwd_flags <= kNet) {
    src += fmt("#define NET_REPS %d\n", kNet - bwd_flags + 1);
    // spikes listed per delivery round (shared memory); HHB_NET_CAP lowers it (tests)
    const char* cap = getenv("HHB_NET_CAP");
    src += fmt("#define NET_CAP %d\n", cap && atoi(cap) > 0 && atoi(cap) < 2048 ? atoi(cap) : 2048);
    const char* nun = getenv("HHB_NET_UNROLL");
    const char* nop = getenv("HHB_NET_NOPAIR");   // tests: the odd-population (unpaired) ring path
    src += fmt("#define NET_UNROLL %d\n#define NET_NOPAIR %d\n", nun && atoi(nun) > 0 ? atoi(nun) : 4,
               nop && atoi(nop) > 0 ? 1 : 0);
    src += kNetKernel;
    return src;
  }
  if (bwd_flags < 0) {
    const int ff = bwd_flags == kInspect ? (FF_VO | FF_SO | FF_CK) : -1 - bwd_flags;
    src += fmt("#define FF_VO %d\n#define FF_SO %d\n#define FF_SVO %d\n#define FF_CK %d\n#define FF_AL %d\n"
               "#define FF_L2 %d\n#define FF_SVB %d\n",
               (ff & FF_VO) ? 1 : 0, (ff & FF_SO) ? 1 : 0, (ff & FF_SVO) ? 1 : 0, (ff & FF_CK) ? 1 : 0,
               (ff & FF_AL) ? 1 : 0, (ff & FF_L2) ? 1 : 0, (ff & FF_SVB) ? 1 : 0);
    src += kForwardBody;
  }
  if (bwd_flags >= 0 || bwd_flags == kInspect) {
    const int f = bwd_flags < 0 ? (BF_SV | BF_DI) : bwd_flags;
    src += fmt("#define BF_SV %d\n#define BF_SS %d\n#define BF_DI %d\n#define BF_SPLIT %d\n#define BF_SUM %d\n"
               "#define BF_K1 %d\n#define BF_SVS %d\n#define BF_SPREV %d\n",
               (f & BF_SV) ? 1 : 0, (f & BF_SS) ? 1 : 0, (f & BF_DI) ? 1 : 0, (f & BF_SPLIT) ? 1 : 0,
               (f & BF_SUM) ? 1 : 0, (f & BF_K1) ? 1 : 0, (f & BF_SVS) ? 1 : 0, (f & BF_SPREV) ? 1 : 0);
    src += kBwdKernel;
  }
  return src;
}

// ------------------------------------------------------------ cache
struct Module {
  CUfunction fwd1 = nullptr, fwd4 = nullptr, fwdp1 = nullptr, fwdp4 = nullptr, bwd = nullptr, bwd2 = nullptr;
  CUfunction net = nullptr;
  int net_blocks_per_sm = 0, net_smem = 0;
  bool ok = false;
};
static std::map<std::string, Module> g_cache;

static std::string key_of(const hhb_params_t* P, int dev) {
  hhb_params_t Q;
  memset(&Q, 0, sizeof Q);
  Q.n_gates = P->n_gates;
  Q.n_channels = P->n_channels;
  Q.c_m = P->c_m;
  Q.dt = P->dt;
  Q.v_theta = P->v_theta;
  Q.rate_scale = P->rate_scale;
  for (int g = 0; g < P->n_gates; ++g) {
    Q.gates[g].alpha = {P->gates[g].alpha.kind, 0, P->gates[g].alpha.a, P->gates[g].alpha.v0, P->gates[g].alpha.b};
    Q.gates[g].beta = {P->gates[g].beta.kind, 0, P->gates[g].beta.a, P->gates[g].beta.v0, P->gates[g].beta.b};
    Q.gates[g].exponent = P->gates[g].exponent;
    Q.gates[g].channel = P->gates[g].channel;
  }
  for (int c = 0; c < P->n_channels; ++c) Q.channels[c] = P->channels[c];
  std::string k(reinterpret_cast<const char*>(&Q), sizeof Q);
  k += std::to_string(dev);
  const char* mb = getenv("HHB_JIT_MINB");
  k += mb ? mb : "";
  k += mg::disabled() ? "nomerge" : "";
  const char* tr = getenv("HHB_JIT_TWO_RCP");
  k += tr ? std::string("r") + tr : "";
  const char* bmb = getenv("HHB_JIT_BWD_MINB");
  k += bmb ? std::string("b") + bmb : "";
  const char* bmb2 = getenv("HHB_JIT_BWD2_MINB");
  k += bmb2 ? std::string("c") + bmb2 : "";
  const char* pf = getenv("HHB_JIT_FWD_PF");
  k += pf ? std::string("p") + pf : "";
  const char* pf4 = getenv("HHB_JIT_FWD_PF4");
  k += pf4 ? std::string("q") + pf4 : "";
  const char* b1 = getenv("HHB_JIT_BWD_ONE_RCP");
  k += b1 ? std::string("o") + b1 : "";
  for (const char* e : {"HHB_NET_CAP", "HHB_NET_UNROLL", "HHB_NET_NOPAIR", "HHB_JIT_CHECK", "HHB_JIT_BWD_PAIR", "HHB_JIT_FWD_HALF", "HHB_JIT_POLY_EXP"}) {
    const char* x = getenv(e);
    k += x ? std::string("|") + e + x : "";
  }
  return k;
}

static bool disabled() {
  const char* e = getenv("HHB_NO_JIT");
  return e && e[0] && e[0] != '0';
}

static Module* get_module(const hhb_params_t* P, int bwd_flags) {
  if (disabled()) return nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_mu);
  load_libs();
  if (!g_nv.ok || !g_drv.ok) {
    g_status = "jit unavailable: " + (g_nv.ok ? g_drv.why : g_nv.why);
    return nullptr;
  }
  const std::string key = key_of(P, dev) + "|" + std::to_string(bwd_flags);
  auto it = g_cache.find(key);
  if (it != g_cache.end()) return it->second.ok ? &it->second : nullptr;
  Module& m = g_cache[key];
  const std::string src = generate(P, bwd_flags);
  nvrtcProgram prog;
  if (g_nv.create(&prog, src.c_str(), "hh_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    g_status = "nvrtcCreateProgram failed";
    return nullptr;
  }
  const char* opts[] = {"-arch=sm_100a", "--std=c++17", "-lineinfo", "-default-device"};
  const nvrtcResult rc = g_nv.compile(prog, 4, opts);
  if (rc != NVRTC_SUCCESS) {
    size_t n = 0;
    g_nv.log_size(prog, &n);
    std::string log(n, '\0');
    g_nv.log(prog, &log[0]);
    g_status = "nvrtc compile failed: " + log.substr(0, 2000);
    g_nv.destroy(&prog);
    return nullptr;
  }
  size_t n = 0;
  g_nv.cubin_size(prog, &n);
  std::vector<char> cubin(n);
  g_nv.cubin(prog, cubin.data());
  g_nv.destroy(&prog);
  CUmodule mod;
  bool loaded = g_drv.load(&mod, cubin.data()) == CUDA_SUCCESS;
  if (loaded && bwd_flags <= kNet) {
    // dynamic shared memory: s_next + s_ahead + s_next2, 3 x replicas x 256 x 8 bytes
    const int dyn = 3 * (kNet - bwd_flags + 1) * 256 * 8;
    loaded = g_drv.get(&m.net, mod, "hh_net") == CUDA_SUCCESS && g_drv.occupancy && g_drv.set_attr &&
             g_drv.set_attr(m.net, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, dyn) == CUDA_SUCCESS &&
             g_drv.occupancy(&m.net_blocks_per_sm, m.net, 256, size_t(dyn)) == CUDA_SUCCESS &&
             m.net_blocks_per_sm > 0;
    m.net_smem = dyn;
  } else if (loaded && bwd_flags < 0)
    loaded = g_drv.get(&m.fwd1, mod, "hh_fwd_v1") == CUDA_SUCCESS && g_drv.get(&m.fwd4, mod, "hh_fwd_v4") == CUDA_SUCCESS &&
             g_drv.get(&m.fwdp1, mod, "hh_fwdp_v1") == CUDA_SUCCESS &&
             g_drv.get(&m.fwdp4, mod, "hh_fwdp_v4") == CUDA_SUCCESS;
  if (loaded && bwd_flags >= 0)
    loaded = g_drv.get(&m.bwd, mod, "hh_bwd") == CUDA_SUCCESS && g_drv.get(&m.bwd2, mod, "hh_bwd2") == CUDA_SUCCESS;
  if (!loaded) {
    g_status = "cuModuleLoadData / cuModuleGetFunction failed";
    return nullptr;
  }
  m.ok = true;
  g_status = "ok";
  return &m;
}

}  // namespace jit

// Returns true when the JIT kernel was launched (rc holds its status).
bool jit_forward(const hhb_params_t* P, const FwdArgs<float>& a, const PoissonTab<float>* ptab, bool vec4,
                 cudaStream_t st, int& rc) {
  using namespace jit;
  const auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  const bool aligned = vec4 && a.n % 4 == 0 && (ptab || (a.i_sn == 1 && a.i_st % 4 == 0 && al16(a.i_ext))) &&
                       (!a.v_out || (a.v_ld % 4 == 0 && al16(a.v_out))) &&
                       (!a.spk_val || (a.spkv_ld % 4 == 0 && al16(a.spk_val))) &&
                       (!a.spk_bf || (a.spkb_ld % 4 == 0 && (reinterpret_cast<uintptr_t>(a.spk_bf) & 7u) == 0)) &&
                       (!a.ckpt || (a.ck_ld % 4 == 0 && al16(a.ckpt)));
  const int ff = (a.v_out ? FF_VO : 0) | (a.spk ? FF_SO : 0) | (a.spk_val ? FF_SVO : 0) | (a.ckpt ? FF_CK : 0) |
                 (aligned ? FF_AL : 0) | (a.sq_part ? FF_L2 : 0) | (a.spk_bf ? FF_SVB : 0);
  jit::Module* m = jit::get_module(P, fwd_kind(ff));
  if (!m) return false;
  const int VEC = vec4 ? 4 : 1;
  const int64_t threads = (a.n + VEC - 1) / VEC;
  const int tpb = fwd_block(threads);
  const int64_t blocks = (threads + tpb - 1) / tpb;
  FwdArgs<float> args = a;
  PoissonTab<float> tab = ptab ? *ptab : PoissonTab<float>{};
  // Philox-4x32-10 key schedule of a.seed (round r uses k + r * W)
  uint32_t keys[20];
  for (int r = 0; r < 10; ++r) {
    keys[2 * r] = uint32_t(a.seed) + uint32_t(r) * 0x9E3779B9u;
    keys[2 * r + 1] = uint32_t(a.seed >> 32) + uint32_t(r) * 0xBB67AE85u;
  }
  void* params[] = {&args, &tab, keys};
  CUfunction f = ptab ? (vec4 ? m->fwdp4 : m->fwdp1) : (vec4 ? m->fwd4 : m->fwd1);
  const CUresult r = jit::launch_pdl_drv(f, unsigned(blocks), unsigned(tpb), reinterpret_cast<CUstream>(st), params);
  rc = (r == CUDA_SUCCESS) ? HHB_OK : fail(HHB_ECUDA, "jit forward launch failed");
  return true;
}

bool jit_backward(const hhb_params_t* P, const DevSur<float>& sur, const BwdArgs<float>& a, cudaStream_t st,
                  int& rc) {
  using namespace jit;
  const int flags = (a.seed_v ? BF_SV : 0) | (a.seed_s ? BF_SS : 0) | (a.d_i ? BF_DI : 0) |
                    (a.di_hi ? BF_SPLIT : 0) | (a.di_sum ? BF_SUM : 0) | (a.ck_every == 1 ? BF_K1 : 0) |
                    (a.seed_v && a.sv_scale ? BF_SVS : 0) |
                    // the seed is the v-plane of the next checkpoint slot (fused MSE(V, 0) of the layer)
                    (a.seed_v && a.sv_scale && a.ck_every == 1 && !getenv("HHB_JIT_NO_SPREV") &&
                             a.seed_v == a.ckpt + (1 + P->n_gates) * a.ck_ld && a.sv_ld == (1 + P->n_gates) * a.ck_ld
                         ? BF_SPREV
                         : 0);
  jit::Module* m = jit::get_module(P, flags);
  if (!m) return false;
  const int64_t blocks = bwd_blocks(a.n);
  DevSur<float> s = sur;
  BwdArgs<float> args = a;
  void* params[] = {&s, &args};
  // two neurons per thread when every stream is neuron-contiguous and 8-byte
  // aligned for the pair (float2 / packed bf16x2 accesses)
  auto even = [](int64_t x) { return (x & 1) == 0; };
  auto al8 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 7) == 0; };
  const bool vec2 = !getenv("HHB_JIT_BWD_VEC1") && even(a.n) && a.i_sn == 1 && even(a.i_st) && even(a.ck_ld) &&
                    al8(a.i_ext) && al8(a.ckpt) && (a.ck_every == 1 || al8(a.seg)) &&
                    (!a.seed_v || (even(a.sv_ld) && al8(a.seed_v))) &&
                    (!a.seed_s || (even(a.ss_ld) && al8(a.seed_s))) && (!a.d_i || (even(a.di_ld) && al8(a.d_i))) &&
                    (!a.di_hi || (even(a.dh_ld) && (a.dh_grp == 0 || (even(a.dh_grp) && even(a.dh_pitch))) &&
                                  (reinterpret_cast<uintptr_t>(a.di_hi) & 3) == 0 &&
                                  (reinterpret_cast<uintptr_t>(a.di_lo) & 3) == 0));
  const CUresult r = jit::launch_pdl_drv(vec2 ? m->bwd2 : m->bwd, unsigned(blocks),
                                         unsigned(vec2 ? kBwdThreads / 2 : kBwdThreads), reinterpret_cast<CUstream>(st),
                                         params);
  rc = (r == CUDA_SUCCESS) ? HHB_OK : fail(HHB_ECUDA, "jit backward launch failed");
  return true;
}

// hh_net (kNetKernel): one cooperative launch for `steps` network steps.
// Returns false when the JIT or a cooperative launch is unavailable.
bool jit_cortex_run(const hhb_params_t* P, const CortexRunArgs& a, cudaStream_t st, int& rc) {
  using namespace jit;
  if (a.reps < 1 || a.reps > 16) {
    rc = fail(HHB_EINVAL, "hh_net: 1..16 replicas per launch");
    return true;
  }
  jit::Module* m = jit::get_module(P, kNet - int(a.reps - 1));
  if (!m || !g_drv.coop) return false;
  int dev = 0, sms = kNumSMs;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // one block per 256-neuron tile, all resident (cooperative launch)
  const int64_t tiles = (a.n + 255) / 256, most = int64_t(m->net_blocks_per_sm) * sms;
  if (cudaMemsetAsync(a.bar, 0, sizeof(unsigned), st) != cudaSuccess) {
    rc = fail(HHB_ECUDA, "barrier reset failed");
    return true;
  }
  if ((a.words + 255) / 256 > 8) {
    rc = fail(HHB_ENOTSUP, "hh_net: more than 65536 neurons (8 bitmap words per thread)");
    return true;
  }
  if (tiles > most || tiles != a.tiles) {
    rc = fail(HHB_ENOTSUP, "hh_net: the population needs more resident 256-neuron tiles than the GPU holds");
    return true;
  }
  const unsigned grid = unsigned(tiles);
  CortexRunArgs args = a;
  void* params[] = {&args};
  const CUresult r = g_drv.coop(m->net, grid, 1, 1, 256, 1, 1, unsigned(m->net_smem), reinterpret_cast<CUstream>(st),
                                params);
  rc = (r == CUDA_SUCCESS) ? HHB_OK : fail(HHB_ECUDA, "cooperative launch of hh_net failed");
  return true;
}

// compile-only (no device, no module load): the cubin of one generated module
// for sm_100a -- kind 0: forward + backward (inspection flags), 1: the
// persistent network kernel, 2: the network kernel for 4 replicas, >= 16: the
// backward module for BF_* flags kind - 16, < 0: the forward module for FF_*
// flags -1 - kind.  For CPU
// tests of the code generator and SASS inspection (cuobjdump / nvdisasm).
int jit_cubin(const hhb_params_t* P, int kind, std::vector<char>& cubin, std::string& log) {
  using namespace jit;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    load_libs();
  }
  if (!g_nv.ok) {
    log = g_nv.why;
    return HHB_ENOTSUP;
  }
  const int flags = kind == 0 ? kInspect : kind == 1 ? kNet : kind == 2 ? kNet - 3 : kind >= 16 ? kind - 16 : kind;
  const std::string src = generate(P, flags);
  nvrtcProgram prog;
  if (g_nv.create(&prog, src.c_str(), "hh_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    log = "nvrtcCreateProgram failed";
    return HHB_ECUDA;
  }
  const char* opts[] = {"-arch=sm_100a", "--std=c++17", "-lineinfo", "-default-device"};
  const nvrtcResult rc = g_nv.compile(prog, 4, opts);
  size_t n = 0;
  g_nv.log_size(prog, &n);
  log.assign(n, '\0');
  if (n) g_nv.log(prog, &log[0]);
  if (rc != NVRTC_SUCCESS) {
    g_nv.destroy(&prog);
    return HHB_ECUDA;
  }
  g_nv.cubin_size(prog, &n);
  cubin.resize(n);
  g_nv.cubin(prog, cubin.data());
  g_nv.destroy(&prog);
  return HHB_OK;
}

const char* jit_status() { return jit::g_status.c_str(); }

std::string jit_source(const hhb_params_t* P) { return jit::generate(P); }

}  // namespace hhb
