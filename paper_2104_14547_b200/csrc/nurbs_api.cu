// nurbs_api.cu — host side of the C ABI declared in include/nurbs.h: shape checks, the
// launch plan, checked mode, and the kernel launches on the caller's stream.
// Citations: P:n = reference/PAPER.md line n; R<k> = DESIGN.md §3 reading k.
#include <atomic>
#include <mutex>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled (driver entry point, no -lcuda)

#include "../../include/nurbs.h"
#include "nurbs_internal.cuh"
#include "nurbs_points.cuh"
#include "nurbs_points_plan.h"
#include "nurbs_knots.h"

using nb::Dir;
using nb::Params;
using nb::Plan;

namespace {

thread_local std::string g_detail;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_detail = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(NURBS_E_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

bool check_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* s = getenv("NURBS_CHECK");
    mode = (s && s[0] && s[0] != '0') ? 1 : 0;
  }
  return mode == 1;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Diagnostic switches, read once per process: NURBS_NO_TMA=1 forces the per-thread IO path,
// NURBS_TC=1 runs the tensor-core backward (nurbs_bwd_tc.cu) where it applies.
bool env_flag(const char* name) {
  const char* s = getenv(name);
  return s && s[0] && s[0] != '0';
}
std::atomic<int>& path_flags() {
  static std::atomic<int> f{(env_flag("NURBS_NO_TMA") ? NURBS_PATH_NO_TMA : 0) |
                           (env_flag("NURBS_TC") ? NURBS_PATH_TC : 0)};
  return f;
}
bool no_tma() { return (path_flags().load(std::memory_order_relaxed) & NURBS_PATH_NO_TMA) != 0; }
bool use_tc() { return (path_flags().load(std::memory_order_relaxed) & NURBS_PATH_TC) != 0; }

// Shape rules shared by surfaces and curves (one direction).
int check_dir(const char* name, int n, int p, int ns) {
  if (p < 1 || p > NURBS_MAX_DEGREE) return fail(NURBS_E_UNSUPPORTED, "%s: degree %d outside 1..%d", name, p, NURBS_MAX_DEGREE);
  if (n <= p) return fail(NURBS_E_ARG, "%s: control count %d must exceed degree %d", name, n, p);
  if (ns < 0) return fail(NURBS_E_ARG, "%s: negative sample count %d", name, ns);
  return NURBS_OK;
}

int check_surface_shape(const nurbs_shape* sh) {
  if (!sh) return fail(NURBS_E_ARG, "shape is NULL");
  if (sh->B < 0) return fail(NURBS_E_ARG, "negative batch %d", sh->B);
  if (sh->knots_batched != 0 && sh->knots_batched != 1) return fail(NURBS_E_ARG, "knots_batched must be 0 or 1");
  int st = check_dir("u", sh->n, sh->p, sh->n_u);
  if (st) return st;
  return check_dir("v", sh->m, sh->q, sh->n_v);
}

int check_curve_shape(const nurbs_shape* sh) {
  if (!sh) return fail(NURBS_E_ARG, "shape is NULL");
  if (sh->B < 0) return fail(NURBS_E_ARG, "negative batch %d", sh->B);
  if (sh->m != 1 || sh->q != 0) return fail(NURBS_E_ARG, "curve shape needs m = 1, q = 0 (got m=%d q=%d)", sh->m, sh->q);
  if (sh->knots_batched != 0 && sh->knots_batched != 1) return fail(NURBS_E_ARG, "knots_batched must be 0 or 1");
  return check_dir("u", sh->n, sh->p, sh->n_u);
}

// Internal directions. Surfaces: rows = u, cols = v. Curves: rows trivial, cols = the curve.
struct Geo {
  int B, P;
  Dir r, c;
};

Geo surface_geo(const nurbs_shape* sh, const float* U, const float* V, const float* u, const float* v) {
  Geo g{};
  g.B = sh->B;
  g.P = sh->p;
  g.r = Dir{sh->n, sh->p, sh->n_u, U, sh->knots_batched ? (long long)(sh->n + sh->p + 1) : 0LL, u, nullptr, nullptr, 0};
  g.c = Dir{sh->m, sh->q, sh->n_v, V, sh->knots_batched ? (long long)(sh->m + sh->q + 1) : 0LL, v, nullptr, nullptr, 0};
  return g;
}

Geo curve_geo(const nurbs_shape* sh, const float* U, const float* u) {
  Geo g{};
  g.B = sh->B;
  g.P = 0;
  g.r = Dir{1, 0, 1, nullptr, 0, nullptr, nullptr, nullptr, 0};
  g.c = Dir{sh->n, sh->p, sh->n_u, U, sh->knots_batched ? (long long)(sh->n + sh->p + 1) : 0LL, u, nullptr, nullptr, 0};
  return g;
}

// Point the directions at a caller's tables. In checked mode (NURBS_CHECK=1) the device
// header written by nurbs_tables is read back (synchronizes) and must match this call's shape:
// tables built for another n, degree or sample count would be read at wrong offsets.
int attach_tables(Geo& g, const void* tables, cudaStream_t st) {
  if (!tables) return NURBS_OK;
  const nb::TabLayout L = nb::tab_layout(g.P > 0 ? g.r.ns : 0, g.r.p, g.c.ns, g.c.p, g.r.n);
  const unsigned char* t = static_cast<const unsigned char*>(tables);
  if (check_mode()) {
    int h[10] = {};
    cudaError_t e = cudaMemcpyAsync(h, tables, sizeof(h), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "tables header read");
    const int want[10] = {(int)nb::kTabMagic, 1, g.P > 0 ? g.r.n : h[2], g.P > 0 ? g.r.p : h[3], g.P > 0 ? g.r.ns : 0,
                          L.np_r, g.c.n, g.c.p, g.c.ns, L.np_c};
    for (int k = 0; k < 10; ++k)
      if (h[k] != want[k])
        return fail(NURBS_E_TABLES, "tables header field %d is %d, this call needs %d (tables built for another shape)",
                    k, h[k], want[k]);
  }
  if (g.P > 0) {
    g.r.tspan = reinterpret_cast<const int*>(t + L.off_span_r);
    g.r.tN = reinterpret_cast<const float*>(t + L.off_N_r);
    g.r.tnp = L.np_r;
    g.r.tsfirst = L.nsf_r > 0 ? reinterpret_cast<const int*>(t + L.off_sfirst_r) : nullptr;
  }
  g.c.tspan = reinterpret_cast<const int*>(t + L.off_span_c);
  g.c.tN = reinterpret_cast<const float*>(t + L.off_N_c);
  g.c.tnp = L.np_c;
  return NURBS_OK;
}

// ---- 2-D TMA descriptor of a streamed [rows][n_v][3] fp32 tensor (out, dL/dS or the fit
// target), box = rps rows x 64 sample columns. Used when a stage's rows are not contiguous
// (n_v != 128); else (or if the driver entry point is unavailable) the kernels keep their
// bulk-copy paths.
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  // resolved once (thread-safe static initialisation); nullptr if the driver lacks it
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
    return f;
  }();
  return fn;
}

void set_io_map(nb::Params& prm, const float* base, long long rows, int nv, int rps) {
  prm.tmap = 0;
  if (!prm.bulk || nv < nb::kBoxCols || (nv == nb::kCB && prm.NCB == 1) || rows <= 0) return;
  // the descriptor is a pure function of (base, rows, nv, rps): a per-thread cache of recent
  // encodes keeps the driver call off the per-launch path of repeated calls
  struct Entry { const float* base; long long rows; int nv, rps; CUtensorMap map; };
  static thread_local Entry cache[4];
  static thread_local int next = 0;
  for (const Entry& c : cache)
    if (c.base == base && c.rows == rows && c.nv == nv && c.rps == rps) {
      prm.io_map = c.map;
      prm.tmap = 1;
      return;
    }
  PFN_cuTensorMapEncodeTiled_v12000 fn = tmap_encoder();
  if (!fn) return;
  const cuuint64_t dims[2] = {(cuuint64_t)nv * 3, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)nv * 12};
  const cuuint32_t box[2] = {3 * nb::kBoxCols, (cuuint32_t)rps};
  const cuuint32_t es[2] = {1, 1};
  if (fn(&prm.io_map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS) {
    prm.tmap = 1;
    cache[next] = Entry{base, rows, nv, rps, prm.io_map};
    next = (next + 1) & 3;
  }
}

// Checked mode: validate data on the device and synchronize.
int validate_geo(const Geo& g, const float* ctrl, cudaStream_t st) {
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(unsigned long long), st);
  if (e != cudaSuccess) return cuda_fail(e, "validate: cudaMallocAsync");
  e = cudaMemsetAsync(d, 0xff, sizeof(unsigned long long), st);
  if (e == cudaSuccess)
    e = nb::launch_validate(g.B, g.r, g.c, g.P > 0, reinterpret_cast<const float4*>(ctrl),
                            (long long)g.B * g.r.n * g.c.n, d, st);
  unsigned long long h = ~0ull;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(d, st);
  if (e != cudaSuccess) return cuda_fail(e, "validate");
  if (h == ~0ull) return NURBS_OK;
  const int code = (int)(h >> 48);
  const int which = (int)((h >> 40) & 0xff);
  const long long idx = (long long)(h & 0xffffffffffull);
  static const char* names[] = {"ctrl (weight <= 0 or non-finite)", "row-direction knots", "column-direction knots",
                                "row-direction samples", "column-direction samples"};
  return fail(code, "invalid %s at flat index %lld", which < 5 ? names[which] : "?", idx);
}

int launch(const Geo& g, bool bwd, const float* ctrl, float* out, const float* gout, float* gctrl, float* gR,
           float* gC, void* ws, size_t ws_bytes, cudaStream_t st) {
  const Plan pl = nb::make_plan(g.B, g.r.n, g.P, g.r.ns, g.c.n, g.c.ns, !bwd);
  const size_t grad_bytes = (size_t)g.B * g.r.n * g.c.n * 16;
  const int gR_per = g.r.n + g.r.p + 1, gC_per = g.c.n + g.c.p + 1;
  const int gR_items = g.r.kstride ? g.B : 1, gC_items = g.c.kstride ? g.B : 1;
  if (g.B == 0) return NURBS_OK;
  if (g.r.ns == 0 || g.c.ns == 0) {
    if (!bwd) return NURBS_OK;
    cudaError_t e = cudaMemsetAsync(gctrl, 0, grad_bytes, st);
    if (e == cudaSuccess && gR) e = cudaMemsetAsync(gR, 0, sizeof(float) * (size_t)gR_per * gR_items, st);
    if (e == cudaSuccess && gC) e = cudaMemsetAsync(gC, 0, sizeof(float) * (size_t)gC_per * gC_items, st);
    return e == cudaSuccess ? NURBS_OK : cuda_fail(e, "zero-fill");
  }
  if (pl.grid > 0x7fffffffLL) return fail(NURBS_E_ARG, "grid of %lld CTAs too large", pl.grid);
  if (bwd && pl.ws_bytes > 0) {
    if (!ws || ws_bytes < pl.ws_bytes)
      return fail(NURBS_E_WORKSPACE, "backward needs a %zu-byte workspace (got %zu at %p)", pl.ws_bytes, ws_bytes, ws);
  }
  Params prm{};
  prm.B = g.B;
  prm.r = g.r;
  prm.c = g.c;
  prm.ctrl = reinterpret_cast<const float4*>(ctrl);
  prm.out = out;
  prm.gout = gout;
  prm.gctrl = reinterpret_cast<float4*>(gctrl);
  prm.gR = gR;
  prm.gR_per = gR_per;
  prm.gR_items = gR_items;
  prm.gC = gC;
  prm.gC_per = gC_per;
  prm.gC_items = gC_items;
  prm.K = pl.K;
  prm.NRB = pl.NRB;
  prm.NCB = pl.NCB;
  prm.T_rows = pl.T_rows;
  prm.CBW = g.c.n < nb::kBandCols ? g.c.n : nb::kBandCols;
  prm.direct = pl.direct;
  const void* io = bwd ? static_cast<const void*>(gout) : static_cast<const void*>(out);
  prm.bulk = (g.c.ns % 4 == 0) && aligned16(io) ? 1 : 0;
  if (no_tma()) prm.bulk = 0;
  if (bwd && !pl.direct) {
    prm.slots = reinterpret_cast<float4*>(ws);
    prm.colband = reinterpret_cast<int2*>(static_cast<unsigned char*>(ws) + pl.slots_bytes);
  }
  set_io_map(prm, bwd ? gout : out, (long long)g.B * g.r.ns, g.c.ns, bwd ? nb::kRPS_B : nb::kRPS_F);
  cudaError_t e = cudaErrorNotSupported;
  if (bwd && use_tc() && nb::bwd_tc_supported(prm, g.P, g.c.p)) e = nb::launch_bwd_tc(prm, g.P, g.c.p, st);
  if (e == cudaErrorNotSupported) e = nb::launch_grid(prm, bwd ? 1 : 0, g.P, g.c.p, st);
  if (e != cudaSuccess) return cuda_fail(e, bwd ? "backward kernel launch" : "forward kernel launch");
  if (bwd && !pl.direct) {
    e = nb::launch_reduce(prm, g.P, st);
    if (e != cudaSuccess) return cuda_fail(e, "reduce kernel launch");
  }
  return NURBS_OK;
}

// Fused fitting step (NEXT-2): grid kernel with dL/dS = 2 (S - T) / N from the target, then
// the update kernel (tile reduce if needed, SGD on P and w, loss).
int launch_fit(const Geo& g, float* ctrl, const float* target, float lr, float* gctrl, float* loss, void* ws,
               size_t ws_bytes, cudaStream_t st) {
  const Plan pl = nb::make_plan(g.B, g.r.n, g.P, g.r.ns, g.c.n, g.c.ns);
  if (g.B == 0) return NURBS_OK;
  if (g.r.ns == 0 || g.c.ns == 0) {
    cudaError_t e = cudaMemsetAsync(gctrl, 0, (size_t)g.B * g.r.n * g.c.n * 16, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(loss, 0, sizeof(float), st);
    return e == cudaSuccess ? NURBS_OK : cuda_fail(e, "zero-fill");
  }
  if (pl.grid > 0x7fffffffLL) return fail(NURBS_E_ARG, "grid of %lld CTAs too large", pl.grid);
  if (!ws || ws_bytes < pl.fit_ws_bytes)
    return fail(NURBS_E_WORKSPACE, "fit step needs a %zu-byte workspace (got %zu at %p)", pl.fit_ws_bytes, ws_bytes, ws);
  Params prm{};
  prm.B = g.B;
  prm.r = g.r;
  prm.c = g.c;
  prm.ctrl = reinterpret_cast<const float4*>(ctrl);
  prm.gout = target;
  prm.gctrl = reinterpret_cast<float4*>(gctrl);
  prm.K = pl.K;
  prm.NRB = pl.NRB;
  prm.NCB = pl.NCB;
  prm.T_rows = pl.T_rows;
  prm.CBW = g.c.n < nb::kBandCols ? g.c.n : nb::kBandCols;
  prm.direct = pl.direct;
  prm.bulk = (g.c.ns % 4 == 0) && aligned16(target) ? 1 : 0;
  if (no_tma()) prm.bulk = 0;
  unsigned char* w = static_cast<unsigned char*>(ws);
  if (!pl.direct) {
    prm.slots = reinterpret_cast<float4*>(w);
    prm.colband = reinterpret_cast<int2*>(w + pl.slots_bytes);
  }
  prm.loss_parts = reinterpret_cast<float*>(w + pl.ws_bytes);
  prm.n_parts = (int)pl.grid;
  prm.loss = loss;
  prm.ctrl_mut = reinterpret_cast<float4*>(ctrl);
  prm.lr = lr;
  prm.fit_scale = (float)(2.0 / ((double)g.B * g.r.ns * g.c.ns));
  set_io_map(prm, target, (long long)g.B * g.r.ns, g.c.ns, nb::kRPS_B);
  cudaError_t e = nb::launch_grid(prm, 2, g.P, g.c.p, st);
  if (e != cudaSuccess) return cuda_fail(e, "fit kernel launch");
  e = nb::launch_fit_update(prm, g.P, st);
  if (e != cudaSuccess) return cuda_fail(e, "fit update kernel launch");
  return NURBS_OK;
}

int check_ptrs(bool bwd, const void* ctrl, const void* out, const void* gout, const void* gctrl) {
  if (!ctrl) return fail(NURBS_E_ARG, "ctrl is NULL");
  if (!bwd && !out) return fail(NURBS_E_ARG, "out is NULL");
  if (bwd && !gout) return fail(NURBS_E_ARG, "grad_out is NULL");
  if (bwd && !gctrl) return fail(NURBS_E_ARG, "grad_ctrl is NULL");
  if (!aligned16(ctrl)) return fail(NURBS_E_ARG, "ctrl must be 16-byte aligned (float4 control points)");
  if (bwd && !aligned16(gctrl)) return fail(NURBS_E_ARG, "grad_ctrl must be 16-byte aligned");
  return NURBS_OK;
}

// ---- true knot gradients (NEXT-4): workspace = the backward's + partials + assembly buffers
struct KnotWs {
  size_t hU, hV, cR, sR, cC, sC, tR, tC, xR, bytes;
};
KnotWs knot_ws(const Geo& g, const Plan& pl) {
  KnotWs w{};
  const size_t B = (size_t)g.B;
  size_t o = nb::align_up(pl.ws_bytes, 256);
  auto take = [&](size_t bytes) { const size_t at = o; o = nb::align_up(o + bytes, 256); return at; };
  // rows-direction units: the knot spans (span moments, grid mode 4) or the samples (mode 3)
  const bool spans = nb::kg_span_mode(g.r.ns, g.r.n, g.P);
  const size_t units = spans ? (size_t)(g.r.n - g.P) : (size_t)g.r.ns;
  w.hU = take(B * pl.NCB * units * (spans ? (g.P + 1) * (g.P + 1) : (g.P + 1)) * 4);
  w.hV = take(B * pl.NRB * g.c.ns * (g.c.p + 1) * 4);
  w.cR = take(B * units * 2 * g.P * 4);
  w.sR = take(B * units * 4);
  w.cC = take(B * g.c.ns * 2 * g.c.p * 4);
  w.sC = take(B * g.c.ns * 4);
  w.tR = take(B * (g.r.n + g.P + 1) * 4);
  w.tC = take(B * (g.c.n + g.c.p + 1) * 4);
  w.xR = take(spans && pl.NCB > nb::kKnotPartGroups ? B * nb::kKnotPartGroups * units * (g.P + 1) * (g.P + 1) * 4
                                                     : 0);  // group sums of the span moments
  w.bytes = o;
  return w;
}

// A helper stream per device for the column-direction knot assembly: the two directions'
// assembly chains (a few small, latency-bound kernels each, nurbs_knots.cu) are independent,
// so the v chain runs beside the u chain. Fork / join through events: the call stays
// asynchronous on the caller's stream and CUDA-graph capturable. The mutex keeps one call's
// event record / wait pairs together when several host threads share a device.
struct AsmSide {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
std::mutex g_asm_mu;
AsmSide g_asm[64];
cudaError_t asm_side(AsmSide*& out) {  // call with g_asm_mu held
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  AsmSide& a = g_asm[dev];
  if (!a.s) {
    if ((e = cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming)) != cudaSuccess) return e;
  }
  out = &a;
  return cudaSuccess;
}

int launch_knots(const Geo& g, const float* ctrl, const float* gout, float* gctrl, float* gR, float* gC, void* ws,
                 size_t ws_bytes, cudaStream_t st) {
  const Plan pl = nb::make_plan(g.B, g.r.n, g.P, g.r.ns, g.c.n, g.c.ns);
  if (g.B == 0) return NURBS_OK;
  const int gR_n = (g.r.n + g.r.p + 1) * (g.r.kstride ? g.B : 1);
  const int gC_n = (g.c.n + g.c.p + 1) * (g.c.kstride ? g.B : 1);
  if (g.r.ns == 0 || g.c.ns == 0) {  // no points: every gradient is zero
    cudaError_t e = cudaMemsetAsync(gctrl, 0, (size_t)g.B * g.r.n * g.c.n * 16, st);
    if (e == cudaSuccess && gR) e = cudaMemsetAsync(gR, 0, sizeof(float) * gR_n, st);
    if (e == cudaSuccess && gC) e = cudaMemsetAsync(gC, 0, sizeof(float) * gC_n, st);
    return e == cudaSuccess ? NURBS_OK : cuda_fail(e, "zero-fill");
  }
  if (pl.grid > 0x7fffffffLL) return fail(NURBS_E_ARG, "grid of %lld CTAs too large", pl.grid);
  const KnotWs W = knot_ws(g, pl);
  if (!ws || ws_bytes < W.bytes)
    return fail(NURBS_E_WORKSPACE, "backward with knot gradients needs a %zu-byte workspace (got %zu at %p)", W.bytes,
                ws_bytes, ws);
  unsigned char* w = static_cast<unsigned char*>(ws);
  Params prm{};
  prm.B = g.B;
  prm.r = g.r;
  prm.c = g.c;
  prm.ctrl = reinterpret_cast<const float4*>(ctrl);
  prm.gout = gout;
  prm.gctrl = reinterpret_cast<float4*>(gctrl);
  prm.K = pl.K;
  prm.NRB = pl.NRB;
  prm.NCB = pl.NCB;
  prm.T_rows = pl.T_rows;
  prm.CBW = g.c.n < nb::kBandCols ? g.c.n : nb::kBandCols;
  prm.direct = pl.direct;
  prm.bulk = (g.c.ns % 4 == 0) && aligned16(gout) ? 1 : 0;
  if (no_tma()) prm.bulk = 0;
  if (!pl.direct) {
    prm.slots = reinterpret_cast<float4*>(w);
    prm.colband = reinterpret_cast<int2*>(w + pl.slots_bytes);
  }
  prm.hU = reinterpret_cast<float*>(w + W.hU);
  prm.hV = reinterpret_cast<float*>(w + W.hV);
  set_io_map(prm, gout, (long long)g.B * g.r.ns, g.c.ns, nb::kRPS_B);
  const bool spans = nb::kg_span_mode(g.r.ns, g.r.n, g.P);
  cudaError_t e = nb::launch_grid(prm, spans ? 4 : 3, g.P, g.c.p, st);
  if (e != cudaSuccess) return cuda_fail(e, "backward (knot gradients) kernel launch");
  if (!pl.direct && (e = nb::launch_reduce(prm, g.P, st)) != cudaSuccess) return cuda_fail(e, "reduce kernel launch");
  const bool doR = g.P > 0 && gR;
  auto chain_v = [&](cudaStream_t sv) {
    nb::KnotDir d{g.B, g.c.n, g.c.p, g.c.ns, g.c.knots, g.c.kstride, g.c.s, g.c.tspan, prm.hV, pl.NRB, 0,
                  reinterpret_cast<float*>(w + W.cC), reinterpret_cast<int*>(w + W.sC), nullptr};
    return nb::launch_knot_grad(d, g.c.kstride != 0, reinterpret_cast<float*>(w + W.tC), gC, sv);
  };
  auto chain_u = [&](cudaStream_t su) {
    // units: the n - p knot spans (span moments, mode 4) or the samples (row sums, mode 3)
    nb::KnotDir d{g.B, g.r.n, g.P, spans ? g.r.n - g.P : g.r.ns, g.r.knots, g.r.kstride, g.r.s, g.r.tspan,
                  prm.hU, pl.NCB, spans ? 1 : 0, reinterpret_cast<float*>(w + W.cR), reinterpret_cast<int*>(w + W.sR),
                  reinterpret_cast<float*>(w + W.xR)};
    return nb::launch_knot_grad(d, g.r.kstride != 0, reinterpret_cast<float*>(w + W.tR), gR, su);
  };
  if (doR && gC) {  // both directions: the v chain on the helper stream, forked after the grid kernel
    std::lock_guard<std::mutex> lk(g_asm_mu);
    AsmSide* a = nullptr;
    if ((e = asm_side(a)) != cudaSuccess) return cuda_fail(e, "knot-gradient helper stream");
    if ((e = cudaEventRecord(a->fork, st)) != cudaSuccess) return cuda_fail(e, "knot-gradient fork");
    if ((e = cudaStreamWaitEvent(a->s, a->fork, 0)) != cudaSuccess) return cuda_fail(e, "knot-gradient fork");
    const cudaError_t ev = chain_v(a->s);
    // join even after a failed launch, so a capturing caller's graph is never left forked
    if ((e = cudaEventRecord(a->join, a->s)) != cudaSuccess) return cuda_fail(e, "knot-gradient join");
    const cudaError_t eu = chain_u(st);
    if ((e = cudaStreamWaitEvent(st, a->join, 0)) != cudaSuccess) return cuda_fail(e, "knot-gradient join");
    if (ev != cudaSuccess) return cuda_fail(ev, "knot-gradient kernels (v)");
    if (eu != cudaSuccess) return cuda_fail(eu, "knot-gradient kernels (u)");
    return NURBS_OK;
  }
  if (doR && (e = chain_u(st)) != cudaSuccess) return cuda_fail(e, "knot-gradient kernels (u)");
  if (gC && (e = chain_v(st)) != cudaSuccess) return cuda_fail(e, "knot-gradient kernels (v)");
  return NURBS_OK;
}

// ---- paired points (NEXT-1)
int check_points_shape(const nurbs_shape* sh) {
  if (!sh) return fail(NURBS_E_ARG, "shape is NULL");
  if (sh->B < 0) return fail(NURBS_E_ARG, "negative batch %d", sh->B);
  if (sh->knots_batched != 0 && sh->knots_batched != 1) return fail(NURBS_E_ARG, "knots_batched must be 0 or 1");
  if (sh->n_v != 1) return fail(NURBS_E_ARG, "paired points need n_v = 1 (n_u = points per surface), got n_v=%d", sh->n_v);
  int st = check_dir("u", sh->n, sh->p, sh->n_u);
  if (st) return st;
  return check_dir("v", sh->m, sh->q, 0);
}

nb::PtsParams points_params(const nurbs_shape* sh, const float* ctrl, const float* U, const float* V, const float* uv) {
  nb::PtsParams prm{};
  prm.B = sh->B;
  prm.n = sh->n;
  prm.m = sh->m;
  prm.N = sh->n_u;
  prm.U = U;
  prm.V = V;
  prm.ustride = sh->knots_batched ? (long long)(sh->n + sh->p + 1) : 0LL;
  prm.vstride = sh->knots_batched ? (long long)(sh->m + sh->q + 1) : 0LL;
  prm.uv = reinterpret_cast<const float2*>(uv);
  prm.ctrl = reinterpret_cast<const float4*>(ctrl);
  return prm;
}

int validate_points(const nurbs_shape* sh, const nb::PtsParams& prm, cudaStream_t st) {
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(unsigned long long), st);
  if (e != cudaSuccess) return cuda_fail(e, "validate_points: cudaMallocAsync");
  e = cudaMemsetAsync(d, 0xff, sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = nb::launch_points_validate(prm, sh->p, sh->q, d, st);
  unsigned long long h = ~0ull;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(d, st);
  if (e != cudaSuccess) return cuda_fail(e, "validate_points");
  if (h == ~0ull) return NURBS_OK;
  static const char* names[] = {"ctrl (weight <= 0 or non-finite)", "u knots", "v knots", "u of a point",
                                "v of a point"};
  const int which = (int)((h >> 40) & 0xff);
  return fail((int)(h >> 48), "invalid %s at flat index %lld", which < 5 ? names[which] : "?",
              (long long)(h & 0xffffffffffull));
}

int points_common(const nurbs_shape* sh, const float* ctrl, const float* U, const float* V, const float* uv, bool bwd) {
  if (!ctrl || !U || !V || !uv) return fail(NURBS_E_ARG, "NULL pointer");
  if (!aligned16(ctrl)) return fail(NURBS_E_ARG, "ctrl must be 16-byte aligned (float4 control points)");
  if ((reinterpret_cast<uintptr_t>(uv) & 7u) != 0) return fail(NURBS_E_ARG, "uv must be 8-byte aligned (float2 pairs)");
  const nb::PtsPlan pl = nb::pts_plan(sh->B, sh->n, sh->m, sh->p, sh->q, sh->n_u);
  if (!(bwd ? pl.fits_b : pl.fits_f))
    return fail(NURBS_E_UNSUPPORTED, "paired points: %d x %d net (degrees %d, %d) exceeds the in-smem cell reduction",
                sh->n, sh->m, sh->p, sh->q);
  return NURBS_OK;
}

}  // namespace

extern "C" {

size_t nurbs_surface_bwd_knots_workspace_bytes(const nurbs_shape* sh) {
  if (!sh || sh->B <= 0 || sh->n <= sh->p || sh->m <= sh->q || sh->n_u < 0 || sh->n_v < 0) return 0;
  Geo g = surface_geo(sh, nullptr, nullptr, nullptr, nullptr);
  return knot_ws(g, nb::make_plan(g.B, g.r.n, g.P, g.r.ns, g.c.n, g.c.ns)).bytes;
}

size_t nurbs_curve_bwd_knots_workspace_bytes(const nurbs_shape* sh) {
  if (!sh || sh->B <= 0 || sh->n <= sh->p || sh->n_u < 0) return 0;
  Geo g = curve_geo(sh, nullptr, nullptr);
  return knot_ws(g, nb::make_plan(g.B, g.r.n, g.P, g.r.ns, g.c.n, g.c.ns)).bytes;
}

int nurbs_surface_bwd_knots(const nurbs_shape* sh, const float* ctrl, const float* U, const float* V, const float* u,
                            const float* v, const void* tables, const float* grad_out, float* grad_ctrl, float* grad_U,
                            float* grad_V, void* workspace, size_t ws_bytes, void* stream) {
  g_detail.clear();
  int st = check_surface_shape(sh);
  if (st) return st;
  if (sh->B == 0) return NURBS_OK;
  if (!grad_ctrl) return fail(NURBS_E_ARG, "grad_ctrl is NULL");
  if (!U || !V || !u || !v) return fail(NURBS_E_ARG, "knot gradients need U, V, u and v");
  if (sh->n_u > 0 && sh->n_v > 0 && (st = check_ptrs(true, ctrl, nullptr, grad_out, grad_ctrl))) return st;
  if (tables && sh->knots_batched) return fail(NURBS_E_TABLES, "tables need shared knots (knots_batched = 0)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Geo g = surface_geo(sh, U, V, u, v);
  if (check_mode() && (st = validate_geo(g, ctrl, s))) return st;
  if ((st = attach_tables(g, tables, s))) return st;
  return launch_knots(g, ctrl, grad_out, grad_ctrl, grad_U, grad_V, workspace, ws_bytes, s);
}

int nurbs_curve_bwd_knots(const nurbs_shape* sh, const float* ctrl, const float* U, const float* u, const void* tables,
                          const float* grad_out, float* grad_ctrl, float* grad_U, void* workspace, size_t ws_bytes,
                          void* stream) {
  g_detail.clear();
  int st = check_curve_shape(sh);
  if (st) return st;
  if (sh->B == 0) return NURBS_OK;
  if (!grad_ctrl) return fail(NURBS_E_ARG, "grad_ctrl is NULL");
  if (!U || !u) return fail(NURBS_E_ARG, "knot gradients need U and u");
  if (sh->n_u > 0 && (st = check_ptrs(true, ctrl, nullptr, grad_out, grad_ctrl))) return st;
  if (tables && sh->knots_batched) return fail(NURBS_E_TABLES, "tables need shared knots (knots_batched = 0)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Geo g = curve_geo(sh, U, u);
  if (check_mode() && (st = validate_geo(g, ctrl, s))) return st;
  if ((st = attach_tables(g, tables, s))) return st;
  return launch_knots(g, ctrl, grad_out, grad_ctrl, nullptr, grad_U, workspace, ws_bytes, s);
}

size_t nurbs_surface_points_bwd_workspace_bytes(const nurbs_shape* sh) {
  if (!sh || sh->B <= 0 || sh->n_u <= 0 || sh->n <= sh->p || sh->m <= sh->q || sh->p < 1 || sh->q < 1) return 0;
  return nb::pts_plan(sh->B, sh->n, sh->m, sh->p, sh->q, sh->n_u).ws_bytes;
}

int nurbs_validate_points(const nurbs_shape* sh, const float* ctrl, const float* U, const float* V, const float* uv,
                          void* stream) {
  g_detail.clear();
  int st = check_points_shape(sh);
  if (st) return st;
  if (!ctrl || !U || !V || (!uv && sh->n_u > 0 && sh->B > 0)) return fail(NURBS_E_ARG, "NULL pointer");
  if (sh->B == 0) return NURBS_OK;
  return validate_points(sh, points_params(sh, ctrl, U, V, uv), static_cast<cudaStream_t>(stream));
}

int nurbs_surface_points_fwd(const nurbs_shape* sh, const float* ctrl, const float* U, const float* V,
                             const float* uv, float* out, void* stream) {
  g_detail.clear();
  int st = check_points_shape(sh);
  if (st) return st;
  if (sh->B == 0 || sh->n_u == 0) return NURBS_OK;
  if (!out) return fail(NURBS_E_ARG, "out is NULL");
  if ((st = points_common(sh, ctrl, U, V, uv, false))) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  nb::PtsParams prm = points_params(sh, ctrl, U, V, uv);
  if (check_mode() && (st = validate_points(sh, prm, s))) return st;
  const nb::PtsPlan pl = nb::pts_plan(sh->B, sh->n, sh->m, sh->p, sh->q, sh->n_u);
  if ((long long)sh->B * pl.nchunk_f > 0x7fffffffLL) return fail(NURBS_E_ARG, "too many points");
  prm.out = out;
  prm.chunk = pl.chunk_f;
  prm.nchunk = pl.nchunk_f;
  prm.ctrl_smem = pl.ctrl_smem;
  cudaError_t e = nb::launch_points(prm, false, sh->p, sh->q, pl.smem_f, s);
  return e == cudaSuccess ? NURBS_OK : cuda_fail(e, "paired forward kernel launch");
}

int nurbs_surface_points_bwd(const nurbs_shape* sh, const float* ctrl, const float* U, const float* V,
                             const float* uv, const float* grad_out, float* grad_ctrl, float* grad_U, float* grad_V,
                             void* workspace, size_t ws_bytes, void* stream) {
  g_detail.clear();
  int st = check_points_shape(sh);
  if (st) return st;
  if (sh->B == 0) return NURBS_OK;
  if (!grad_ctrl) return fail(NURBS_E_ARG, "grad_ctrl is NULL");
  if (!aligned16(grad_ctrl)) return fail(NURBS_E_ARG, "grad_ctrl must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int gU_n = (sh->n + sh->p + 1) * (sh->knots_batched ? sh->B : 1);
  const int gV_n = (sh->m + sh->q + 1) * (sh->knots_batched ? sh->B : 1);
  cudaError_t e = cudaSuccess;
  if (grad_U) e = cudaMemsetAsync(grad_U, 0, sizeof(float) * (size_t)gU_n, s);
  if (e == cudaSuccess && grad_V) e = cudaMemsetAsync(grad_V, 0, sizeof(float) * (size_t)gV_n, s);
  if (e != cudaSuccess) return cuda_fail(e, "knot-gradient zero-fill");
  if (sh->n_u == 0) {
    e = cudaMemsetAsync(grad_ctrl, 0, (size_t)sh->B * sh->n * sh->m * 16, s);
    return e == cudaSuccess ? NURBS_OK : cuda_fail(e, "zero-fill");
  }
  if (!grad_out) return fail(NURBS_E_ARG, "grad_out is NULL");
  if ((st = points_common(sh, ctrl, U, V, uv, true))) return st;
  nb::PtsParams prm = points_params(sh, ctrl, U, V, uv);
  if (check_mode() && (st = validate_points(sh, prm, s))) return st;
  const nb::PtsPlan pl = nb::pts_plan(sh->B, sh->n, sh->m, sh->p, sh->q, sh->n_u);
  if ((long long)sh->B * pl.nchunk_b > 0x7fffffffLL) return fail(NURBS_E_ARG, "too many points");
  if (pl.ws_bytes > 0 && (!workspace || ws_bytes < pl.ws_bytes))
    return fail(NURBS_E_WORKSPACE, "paired backward needs a %zu-byte workspace (got %zu at %p)", pl.ws_bytes, ws_bytes,
                workspace);
  prm.gout = grad_out;
  prm.gctrl = reinterpret_cast<float4*>(grad_ctrl);
  prm.chunk = pl.chunk_b;
  prm.nchunk = pl.nchunk_b;
  prm.slots = pl.nchunk_b > 1 ? reinterpret_cast<float4*>(workspace) : nullptr;
  prm.ctrl_smem = pl.ctrl_smem_b;
  e = nb::launch_points(prm, true, sh->p, sh->q, pl.smem_b, s);
  if (e != cudaSuccess) return cuda_fail(e, "paired backward kernel launch");
  if (pl.nchunk_b > 1) {
    e = nb::launch_points_reduce(prm, s);
    if (e != cudaSuccess) return cuda_fail(e, "paired reduce kernel launch");
  }
  return NURBS_OK;
}


int nurbs_abi_version(void) { return NURBS_ABI_VERSION; }

int nurbs_set_path_flags(int flags) { return path_flags().exchange(flags & (NURBS_PATH_NO_TMA | NURBS_PATH_TC)); }

int nurbs_sum_partials(const float* parts, int32_t n_parts, int64_t n, float* out, void* stream) {
  g_detail.clear();
  if (n_parts < 1 || n < 0) return fail(NURBS_E_ARG, "n_parts = %d, n = %lld", (int)n_parts, (long long)n);
  if (n == 0) return NURBS_OK;
  if (!parts || !out) return fail(NURBS_E_ARG, "NULL pointer");
  if (((n & 3) == 0) && (!aligned16(parts) || !aligned16(out)))
    return fail(NURBS_E_ARG, "parts and out must be 16-byte aligned");
  cudaError_t e = nb::launch_sum_partials(parts, n_parts, (long long)n, out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? NURBS_OK : cuda_fail(e, "sum_partials kernel launch");
}

const char* nurbs_strerror(int status) {
  switch (status) {
    case NURBS_OK: return "ok";
    case NURBS_E_ARG: return "invalid argument";
    case NURBS_E_UNSUPPORTED: return "unsupported degree";
    case NURBS_E_KNOTS: return "invalid knot vector";
    case NURBS_E_DOMAIN: return "parameter outside the knot domain";
    case NURBS_E_WEIGHT: return "invalid weight or non-finite control point";
    case NURBS_E_UNSORTED: return "parameters not sorted";
    case NURBS_E_CUDA: return "CUDA error";
    case NURBS_E_WORKSPACE: return "workspace missing or too small";
    case NURBS_E_TABLES: return "tables unusable for this call";
    default: return "unknown status";
  }
}

const char* nurbs_last_error_detail(void) { return g_detail.c_str(); }

size_t nurbs_tables_bytes(const nurbs_shape* sh) {
  if (!sh) return 0;
  if (sh->m == 1 && sh->q == 0) return nb::tab_layout(0, 0, sh->n_u, sh->p, 1).bytes;
  return nb::tab_layout(sh->n_u, sh->p, sh->n_v, sh->q, sh->n).bytes;
}

int nurbs_tables(const nurbs_shape* sh, const float* U, const float* V, const float* u, const float* v,
                 void* tables, void* stream) {
  g_detail.clear();
  const bool curve = sh && sh->m == 1 && sh->q == 0;
  int st = curve ? check_curve_shape(sh) : check_surface_shape(sh);
  if (st) return st;
  if (sh->knots_batched) return fail(NURBS_E_TABLES, "tables need shared knots (knots_batched = 0)");
  if (!tables || !U || !u || (!curve && (!V || !v))) return fail(NURBS_E_ARG, "NULL pointer");
  if (!aligned16(tables)) return fail(NURBS_E_ARG, "tables must be 16-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Geo g = curve ? curve_geo(sh, U, u) : surface_geo(sh, U, V, u, v);
  g.B = 1;
  // validate knots and samples (weights are not part of the tables)
  {
    unsigned long long* d = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(unsigned long long), s);
    if (e != cudaSuccess) return cuda_fail(e, "tables: cudaMallocAsync");
    e = cudaMemsetAsync(d, 0xff, sizeof(unsigned long long), s);
    if (e == cudaSuccess) e = nb::launch_validate(1, g.r, g.c, !curve, nullptr, 0, d, s);
    unsigned long long h = ~0ull;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFreeAsync(d, s);
    if (e != cudaSuccess) return cuda_fail(e, "tables: validate");
    if (h != ~0ull) return fail((int)(h >> 48), "tables: invalid knots or samples (flat index %lld)", (long long)(h & 0xffffffffffull));
  }
  Dir r = g.r;
  if (curve) r.ns = 0;
  const nb::TabLayout L = nb::tab_layout(r.ns, r.p, g.c.ns, g.c.p, r.n);
  cudaError_t e = nb::launch_tables(r, g.c, tables, L, s);
  if (e != cudaSuccess) return cuda_fail(e, "tables kernel launch");
  return NURBS_OK;
}

size_t nurbs_surface_bwd_workspace_bytes(const nurbs_shape* sh) {
  if (!sh || sh->B <= 0) return 0;
  return nb::make_plan(sh->B, sh->n, sh->p, sh->n_u, sh->m, sh->n_v).ws_bytes;
}

int nurbs_grid_plan(const nurbs_shape* sh, int32_t plan[6]) {
  g_detail.clear();
  if (!plan) return fail(NURBS_E_ARG, "plan is NULL");
  const bool curve = sh && sh->m == 1 && sh->q == 0;
  int st = curve ? check_curve_shape(sh) : check_surface_shape(sh);
  if (st) return st;
  Geo g = curve ? curve_geo(sh, nullptr, nullptr) : surface_geo(sh, nullptr, nullptr, nullptr, nullptr);
  const Plan pl = nb::make_plan(g.B, g.r.n, g.P, g.r.ns, g.c.n, g.c.ns);
  plan[0] = pl.K; plan[1] = pl.NRB; plan[2] = pl.NCB; plan[3] = pl.T_rows; plan[4] = pl.direct;
  plan[5] = pl.grid > 0x7fffffffLL ? 0x7fffffff : (int32_t)pl.grid;
  return NURBS_OK;
}

size_t nurbs_surface_fit_workspace_bytes(const nurbs_shape* sh) {
  if (!sh || sh->B <= 0) return 0;
  return nb::make_plan(sh->B, sh->n, sh->p, sh->n_u, sh->m, sh->n_v).fit_ws_bytes;
}

int nurbs_surface_fit_step(const nurbs_shape* sh, float* ctrl, const float* U, const float* V, const float* u,
                           const float* v, const void* tables, const float* target, float lr, float* grad_ctrl,
                           float* loss, void* workspace, size_t ws_bytes, void* stream) {
  g_detail.clear();
  int st = check_surface_shape(sh);
  if (st) return st;
  if (sh->B == 0) return NURBS_OK;
  if (!grad_ctrl || !loss) return fail(NURBS_E_ARG, "grad_ctrl and loss must not be NULL");
  if (sh->n_u > 0 && sh->n_v > 0 && (st = check_ptrs(true, ctrl, nullptr, target, grad_ctrl))) return st;
  if (!tables && (!U || !V || !u || !v)) return fail(NURBS_E_ARG, "NULL knots or samples");
  if (tables && sh->knots_batched) return fail(NURBS_E_TABLES, "tables need shared knots (knots_batched = 0)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Geo g = surface_geo(sh, U, V, u, v);
  if (check_mode() && (st = validate_geo(g, ctrl, s))) return st;
  if ((st = attach_tables(g, tables, s))) return st;
  return launch_fit(g, ctrl, target, lr, grad_ctrl, loss, workspace, ws_bytes, s);
}

int nurbs_surface_derivs(const nurbs_shape* sh, const float* ctrl, const float* U, const float* V, const float* u,
                         const float* v, float* out, float* out_u, float* out_v, float* normals, void* stream) {
  g_detail.clear();
  int st = check_surface_shape(sh);
  if (st) return st;
  if (sh->B == 0 || sh->n_u == 0 || sh->n_v == 0) return NURBS_OK;
  if (!ctrl || !U || !V || !u || !v || !out_u || !out_v) return fail(NURBS_E_ARG, "NULL pointer");
  if (!aligned16(ctrl)) return fail(NURBS_E_ARG, "ctrl must be 16-byte aligned (float4 control points)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Geo g = surface_geo(sh, U, V, u, v);
  if (check_mode() && (st = validate_geo(g, ctrl, s))) return st;
  const Plan pl = nb::make_plan(g.B, g.r.n, g.P, g.r.ns, g.c.n, g.c.ns);
  if (pl.grid > 0x7fffffffLL) return fail(NURBS_E_ARG, "grid of %lld CTAs too large", pl.grid);
  Params prm{};
  prm.B = g.B;
  prm.r = g.r;
  prm.c = g.c;
  prm.ctrl = reinterpret_cast<const float4*>(ctrl);
  prm.out = out;
  prm.K = pl.K;
  prm.NRB = pl.NRB;
  prm.NCB = pl.NCB;
  prm.T_rows = pl.T_rows;
  cudaError_t e = nb::launch_derivs(prm, g.P, g.c.p, out_u, out_v, normals, s);
  return e == cudaSuccess ? NURBS_OK : cuda_fail(e, "derivative kernel launch");
}

size_t nurbs_curve_bwd_workspace_bytes(const nurbs_shape* sh) {
  if (!sh || sh->B <= 0) return 0;
  return nb::make_plan(sh->B, 1, 0, 1, sh->n, sh->n_u).ws_bytes;
}

int nurbs_validate(const nurbs_shape* sh, const float* ctrl, const float* U, const float* V, const float* u,
                   const float* v, void* stream) {
  g_detail.clear();
  const bool curve = sh && sh->m == 1 && sh->q == 0;
  int st = curve ? check_curve_shape(sh) : check_surface_shape(sh);
  if (st) return st;
  if (!ctrl || !U || !u || (!curve && (!V || !v))) return fail(NURBS_E_ARG, "NULL pointer");
  Geo g = curve ? curve_geo(sh, U, u) : surface_geo(sh, U, V, u, v);
  return validate_geo(g, ctrl, static_cast<cudaStream_t>(stream));
}

int nurbs_surface_fwd(const nurbs_shape* sh, const float* ctrl, const float* U, const float* V, const float* u,
                      const float* v, const void* tables, float* out, void* stream) {
  g_detail.clear();
  int st = check_surface_shape(sh);
  if (st) return st;
  if (sh->B == 0 || sh->n_u == 0 || sh->n_v == 0) return NURBS_OK;  // nothing to evaluate
  if ((st = check_ptrs(false, ctrl, out, nullptr, nullptr))) return st;
  if (!tables && (!U || !V || !u || !v)) return fail(NURBS_E_ARG, "NULL knots or samples");
  if (tables && sh->knots_batched) return fail(NURBS_E_TABLES, "tables need shared knots (knots_batched = 0)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Geo g = surface_geo(sh, U, V, u, v);
  if (check_mode() && (st = validate_geo(g, ctrl, s))) return st;
  if ((st = attach_tables(g, tables, s))) return st;
  return launch(g, false, ctrl, out, nullptr, nullptr, nullptr, nullptr, nullptr, 0, s);
}

int nurbs_surface_bwd(const nurbs_shape* sh, const float* ctrl, const float* U, const float* V, const float* u,
                      const float* v, const void* tables, const float* grad_out, float* grad_ctrl, float* grad_U,
                      float* grad_V, void* workspace, size_t ws_bytes, void* stream) {
  g_detail.clear();
  int st = check_surface_shape(sh);
  if (st) return st;
  if (sh->B == 0) return NURBS_OK;
  if (sh->n_u == 0 || sh->n_v == 0) {  // no points: every gradient is zero
    if (!grad_ctrl) return fail(NURBS_E_ARG, "grad_ctrl is NULL");
    Geo g = surface_geo(sh, U, V, u, v);
    return launch(g, true, ctrl, nullptr, grad_out, grad_ctrl, grad_U, grad_V, workspace, ws_bytes,
                  static_cast<cudaStream_t>(stream));
  }
  if ((st = check_ptrs(true, ctrl, nullptr, grad_out, grad_ctrl))) return st;
  if (!tables && (!U || !V || !u || !v)) return fail(NURBS_E_ARG, "NULL knots or samples");
  if (tables && sh->knots_batched) return fail(NURBS_E_TABLES, "tables need shared knots (knots_batched = 0)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Geo g = surface_geo(sh, U, V, u, v);
  if (check_mode() && (st = validate_geo(g, ctrl, s))) return st;
  if ((st = attach_tables(g, tables, s))) return st;
  return launch(g, true, ctrl, nullptr, grad_out, grad_ctrl, grad_U, grad_V, workspace, ws_bytes, s);
}

int nurbs_curve_fwd(const nurbs_shape* sh, const float* ctrl, const float* U, const float* u, const void* tables,
                    float* out, void* stream) {
  g_detail.clear();
  int st = check_curve_shape(sh);
  if (st) return st;
  if (sh->B == 0 || sh->n_u == 0) return NURBS_OK;
  if ((st = check_ptrs(false, ctrl, out, nullptr, nullptr))) return st;
  if (!tables && (!U || !u)) return fail(NURBS_E_ARG, "NULL knots or samples");
  if (tables && sh->knots_batched) return fail(NURBS_E_TABLES, "tables need shared knots (knots_batched = 0)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Geo g = curve_geo(sh, U, u);
  if (check_mode() && (st = validate_geo(g, ctrl, s))) return st;
  if ((st = attach_tables(g, tables, s))) return st;
  return launch(g, false, ctrl, out, nullptr, nullptr, nullptr, nullptr, nullptr, 0, s);
}

int nurbs_curve_bwd(const nurbs_shape* sh, const float* ctrl, const float* U, const float* u, const void* tables,
                    const float* grad_out, float* grad_ctrl, float* grad_U, void* workspace, size_t ws_bytes,
                    void* stream) {
  g_detail.clear();
  int st = check_curve_shape(sh);
  if (st) return st;
  if (sh->B == 0) return NURBS_OK;
  if (sh->n_u == 0) {
    if (!grad_ctrl) return fail(NURBS_E_ARG, "grad_ctrl is NULL");
    Geo g = curve_geo(sh, U, u);
    return launch(g, true, ctrl, nullptr, grad_out, grad_ctrl, nullptr, grad_U, workspace, ws_bytes,
                  static_cast<cudaStream_t>(stream));
  }
  if ((st = check_ptrs(true, ctrl, nullptr, grad_out, grad_ctrl))) return st;
  if (!tables && (!U || !u)) return fail(NURBS_E_ARG, "NULL knots or samples");
  if (tables && sh->knots_batched) return fail(NURBS_E_TABLES, "tables need shared knots (knots_batched = 0)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Geo g = curve_geo(sh, U, u);
  if (check_mode() && (st = validate_geo(g, ctrl, s))) return st;
  if ((st = attach_tables(g, tables, s))) return st;
  return launch(g, true, ctrl, nullptr, grad_out, grad_ctrl, nullptr, grad_U, workspace, ws_bytes, s);
}

}  // extern "C"
