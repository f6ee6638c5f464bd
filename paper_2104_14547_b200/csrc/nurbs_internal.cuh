// nurbs_internal.cuh — structures shared by the sm_100a kernels (nurbs_kernels.cu) and the
// host C ABI (nurbs_api.cu). Not part of the public ABI (include/nurbs.h).
//
// Vocabulary: the kernels work on an internal "rows x cols" grid. For a surface, rows = the
// u direction (control count n, degree p, samples u) and cols = the v direction (m, q, v).
// A curve is the same grid with a trivial row direction (one control row, degree 0,
// one sample) and the curve along the columns.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda.h>  // CUtensorMap (the TMA descriptor type; no driver-library link needed)
#include <cuda_runtime.h>

namespace nb {

// Tuning knobs (compile-time; -D overrides are for experiments only).
#ifndef NB_RPS_F
#define NB_RPS_F 8
#endif
#ifndef NB_STAGES_F
#define NB_STAGES_F 2
#endif
#ifndef NB_RPS_B
#define NB_RPS_B 8
#endif
#ifndef NB_STAGES_B
#define NB_STAGES_B 3
#endif
#ifndef NB_HRING
#define NB_HRING 4
#endif
#ifndef NB_B2BATCH
#define NB_B2BATCH 4
#endif
#ifndef NB_ROWCHUNK
#define NB_ROWCHUNK 64
#endif
#ifndef NB_MINB_F
#define NB_MINB_F 7
#endif
#ifndef NB_MINB_B
#define NB_MINB_B 4
#endif

constexpr int kCB = 128;          // sample columns per CTA block = threads (one column each)
constexpr int kCompute = 128;     // threads per CTA (4 warps)
constexpr int kThreads = 128;
constexpr int kRPS_F = NB_RPS_F;         // forward: sample rows per TMA stage
constexpr int kStages_F = NB_STAGES_F;   //          stages in the ring
constexpr int kRPS_B = NB_RPS_B;         // backward: sample rows per TMA stage
constexpr int kStages_B = NB_STAGES_B;   //           stages in the ring (kStages_B-1 in flight)
constexpr int kRowChunk = NB_ROWCHUNK;   // rows whose span/basis are staged in smem at once
constexpr int kMaxQ = 5;          // max column degree (runtime q)
constexpr int kRMax = 16;         // max control rows in a row-block band
constexpr int kBandCols = 32;     // smem capacity (columns) of the staged control band
constexpr int kHRing = NB_HRING;         // completed-H rows buffered for B2 (power of 2)
constexpr int kB2Batch = NB_B2BATCH;     // B2 reduces completed rows in batches of this size
constexpr int kMinBlocks_F = NB_MINB_F;  // __launch_bounds__ min CTAs per SM (register budget)
constexpr int kMinBlocks_B = NB_MINB_B;

// One parametric direction.
struct Dir {
  int n;                    // control-point count
  int p;                    // degree (rows: template P; cols: runtime q)
  int ns;                   // number of samples
  const float* knots;       // [n+p+1] or batched
  long long kstride;        // floats between batch items' knot vectors (0 = shared)
  const float* s;           // samples [ns]
  const int* tspan;         // optional tables: span per sample
  const float* tN;          // optional tables: basis per sample, tnp floats each
  int tnp;
  const int* tsfirst;       // optional tables (rows): first sample with span >= s, at s - p
};

struct Params {
  int B;
  Dir r, c;
  const float4* ctrl;       // [B][r.n][c.n] (x,y,z,w)
  float* out;               // [B][r.ns][c.ns][3]
  const float* gout;        // [B][r.ns][c.ns][3]
  float4* gctrl;            // [B][r.n][c.n]
  float* gR; int gR_per; int gR_items;   // knot-gradient zero fill (rows direction)
  float* gC; int gC_per; int gC_items;   // (cols direction)
  int K;                    // knot spans per row block
  int NRB, NCB;             // row blocks, column blocks
  int T_rows;               // control rows of a row-block band = slot rows
  int CBW;                  // smem columns of the staged control band (min(m, kBandCols))
  int bulk;                 // 1: TMA bulk staging of out / grad_out
  int direct;               // 1: bwd writes grad_ctrl in-kernel (NRB == NCB == 1)
  float4* slots;            // [B][NRB][NCB][T_rows][c.n] partial dQ (direct == 0)
  int2* colband;            // [B][NCB] (j0, j1) column band of each column block
  // fused fitting step (NEXT-2)
  float fit_scale;          // 2 / (number of points): dL/dS = fit_scale (S - T)
  float* loss_parts;        // [grid] per-CTA sum of |S - T|^2
  float* loss;              // device scalar: mean |S - T|^2
  float4* ctrl_mut;         // ctrl updated in place: P -= lr dL/dP, w -= lr dL/dw (Eq.14)
  float lr;
  int n_parts;
  // true knot gradients (NEXT-4, mode 3)
  float* hU;                // mode 3: [B][NCB][r.ns][P+1] row sums of G . T_r; mode 4:
                            // [B][NCB][r.n-P][(P+1)^2] span moments X[r][r'] (nurbs_grid.cuh)
  float* hV;                // [B][NRB][c.ns][q+1]: sum over the band rows of Q[i][sv-q+h] . H[i][b]
  // 2-D TMA descriptor of the streamed tensor (out in the forward, dL/dS or the target in the
  // backward / fitting step) viewed as [B*n_u rows][n_v*3 floats], box = RPS rows x 192 floats
  // (64 sample columns): one stage of a 128-column block moves in two tensor copies instead of
  // one bulk copy per row. tmap == 0: per-row bulk copies (or one copy when rows are contiguous).
  int tmap;
  CUtensorMap io_map;       // 64-byte aligned; read through the kernel's __grid_constant__ params
};
constexpr int kBoxCols = 64;             // sample columns per tensor box (192 floats)

// Tables blob layout (nurbs_tables): header then five arrays, each 256-byte aligned; the
// last, sfirst_r[s - p] (s = p..n), is the first row sample whose knot span is >= s: a row
// block's sample range in two loads instead of a CTA-wide search.
struct TabLayout {
  size_t off_span_r, off_N_r, off_span_c, off_N_c, off_sfirst_r, bytes;
  int np_r, np_c, nsf_r;
};

inline int basis_stride(int p) { return (p + 1) <= 4 ? 4 : 8; }

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

inline TabLayout tab_layout(int ns_r, int p_r, int ns_c, int p_c, int n_r) {
  TabLayout L;
  L.np_r = basis_stride(p_r);
  L.np_c = basis_stride(p_c);
  L.nsf_r = (ns_r > 0 && p_r > 0 && n_r > p_r) ? n_r - p_r + 1 : 0;
  size_t o = 256;  // header
  L.off_span_r = o; o = align_up(o + sizeof(int) * (size_t)ns_r, 256);
  L.off_N_r = o;    o = align_up(o + sizeof(float) * (size_t)ns_r * L.np_r, 256);
  L.off_span_c = o; o = align_up(o + sizeof(int) * (size_t)ns_c, 256);
  L.off_N_c = o;    o = align_up(o + sizeof(float) * (size_t)ns_c * L.np_c, 256);
  L.off_sfirst_r = o; o = align_up(o + sizeof(int) * (size_t)L.nsf_r, 256);
  L.bytes = o;
  return L;
}

constexpr uint32_t kTabMagic = 0x4e524253u;  // "NRBS"

struct Plan {
  int K, NRB, NCB, T_rows, direct;
  long long grid;
  size_t slots_bytes, colband_bytes, ws_bytes;
  size_t fit_ws_bytes;      // workspace of the fused fitting step (adds the loss partials)
};

inline int plan_env(const char* name) {  // experiment overrides (NURBS_PLAN_K / _KF); 0 = off
  const char* e = getenv(name);
  return e ? atoi(e) : 0;
}
// The launch plan: K knot spans of u per row block (halving sequence from the largest K whose
// band fits kRMax rows), NCB column blocks of kCB samples. A pure function of the shape, so
// the backward's summation order (hence its bits) is too. Rules fitted to the round-2 plan
// sweep on one B200 (DESIGN.md §5 "Plan"): per-rank shapes of configs 4 and 5 at G = 1..8.
//  * backward: one tile per surface (no cross-tile reduce) whenever the surface fits one
//    tile and there are >= kDirectMinB surfaces; otherwise row blocks of <= kTileRows sample
//    rows, halved until the grid fills ~0.9 of one wave at kSlotsB CTAs per SM;
//  * forward (no reduction: only per-tile overhead): the K minimising
//    ceil(CTAs / slots) * (rows per tile + kTileCost), slots = CTAs resident per SM x SMs.
constexpr int kSMs = 148;                 // B200
constexpr int kSlotsB = 4, kSlotsF = 7, kSlotsF_tmap = 6;   // resident CTAs per SM (ptxas / smem)
constexpr int kDirectMinB = 128;          // direct backward from this many surfaces up
constexpr int kTileRows = 256;            // backward: sample rows per tile cap (tiled plans)
constexpr int kTileCost = 40;             // forward: per-tile overhead in sample-row units
inline Plan make_plan(int B, int n_r, int P, int ns_r, int n_c, int ns_c, bool fwd = false) {
  Plan pl{};
  const int spans = n_r - P;
  pl.NCB = (ns_c + kCB - 1) / kCB;
  int K = spans;
  if (K + P > kRMax) K = kRMax - P;
  if (K < 1) K = 1;
  const int Kmax = K;
  auto nrb = [&](int k) { return (spans + k - 1) / k; };
  auto ctas = [&](int k) { return (long long)B * nrb(k) * pl.NCB; };
  auto half = [](int k) { return (k + 1) / 2; };
  static const int kforce = plan_env("NURBS_PLAN_K"), kforce_f = plan_env("NURBS_PLAN_KF");
  const int kf = fwd ? kforce_f : kforce;
  if (kf > 0) {
    K = kf < K ? kf : K;
  } else if (fwd) {
    const bool tmap = ns_c >= 64 && !(ns_c == kCB && pl.NCB == 1);
    const long long slots = (long long)kSMs * (tmap ? kSlotsF_tmap : kSlotsF);
    double best = -1.0;
    for (int k = Kmax;; k = half(k)) {
      const double rows = (double)ns_r / nrb(k);
      const double t = (double)((ctas(k) + slots - 1) / slots) * (rows + kTileCost);
      if (best < 0.0 || t < best) { best = t; K = k; }
      if (k == 1) break;
    }
  } else if (!(K == spans && pl.NCB == 1 && B >= kDirectMinB)) {
    while (K > 1 && (long long)ns_r * K > (long long)kTileRows * spans) K = half(K);
    while (K > 1 && ctas(K) * 10 < 9LL * kSMs * kSlotsB) K = half(K);
  }
  pl.K = K;
  pl.NRB = (spans + K - 1) / K;
  pl.T_rows = (K + P < n_r) ? (K + P) : n_r;
  pl.direct = (pl.NRB == 1 && pl.NCB == 1) ? 1 : 0;
  pl.grid = (long long)B * pl.NRB * pl.NCB;
  if (pl.direct || B == 0 || ns_r == 0 || ns_c == 0) {
    pl.slots_bytes = pl.colband_bytes = pl.ws_bytes = 0;
  } else {
    pl.slots_bytes = align_up((size_t)B * pl.NRB * pl.NCB * pl.T_rows * (size_t)n_c * 16, 256);
    pl.colband_bytes = align_up((size_t)B * pl.NCB * sizeof(int2), 256);
    pl.ws_bytes = pl.slots_bytes + pl.colband_bytes;
  }
  pl.fit_ws_bytes = pl.ws_bytes + align_up((size_t)(pl.grid > 0 ? pl.grid : 1) * sizeof(float), 256);
  (void)ns_r;
  return pl;
}

// Knot-gradient mode of a surface shape (NEXT-4): span moments (grid mode 4) when the rows
// direction has at least kKgSpanRows sample rows per knot span on average (the per-span work
// then beats per-row dot products: config 5's 32 rows per span 0.335 -> 0.27 ms; config 4's
// 10 rows per span keep per-row weights, measured 0.368 vs 0.385 ms), else per-row (mode 3).
#ifndef NB_KG_SPAN_ROWS
#define NB_KG_SPAN_ROWS 16
#endif
constexpr int kKgSpanRows = NB_KG_SPAN_ROWS;
inline bool kg_span_mode(int ns_r, int n_r, int P) {
  return P > 0 && (long long)ns_r >= (long long)kKgSpanRows * (n_r - P);
}

// Launchers (nurbs_kernels.cu). Return cudaError_t of the launch.
cudaError_t launch_grid(const Params& prm, int mode, int P, int q, cudaStream_t st);  // mode 0 fwd, 1 bwd, 2 fit
cudaError_t launch_reduce(const Params& prm, int P, cudaStream_t st);
// fitting step: (reduce tile partials if needed) + SGD update of ctrl + loss = sum of the CTA partials
cudaError_t launch_fit_update(const Params& prm, int P, cudaStream_t st);
// NEXT-3 parametric derivatives (nurbs_derivs.cu): prm.out (nullable) receives S
cudaError_t launch_derivs(const Params& prm, int P, int q, float* out_u, float* out_v, float* normals,
                          cudaStream_t st);
cudaError_t launch_tables(const Dir& r, const Dir& c, void* tables, const TabLayout& L,
                          cudaStream_t st);
// status: device buffer of one unsigned long long, pre-set to ~0ull.
cudaError_t launch_validate(int B, const Dir& r, const Dir& c, int check_rows,
                            const float4* ctrl, long long n_ctrl,
                            unsigned long long* status, cudaStream_t st);
// tensor-core backward (nurbs_bwd_tc.cu): cudaErrorNotSupported for shapes it does not cover
bool bwd_tc_supported(const Params& prm, int P, int q);
cudaError_t launch_bwd_tc(const Params& prm, int P, int q, cudaStream_t st);
cudaError_t launch_sum_partials(const float* parts, int np, long long n, float* out, cudaStream_t st);
size_t grid_smem_bytes(bool bwd, int P, int q, int T_rows, int CBW, int kg = 0, bool tmap = false);

}  // namespace nb

namespace nb {
cudaError_t launch_grid_p0(const Params& prm, int mode, int q, cudaStream_t st);
cudaError_t launch_grid_p1(const Params& prm, int mode, int q, cudaStream_t st);
cudaError_t launch_grid_p2(const Params& prm, int mode, int q, cudaStream_t st);
cudaError_t launch_grid_p3(const Params& prm, int mode, int q, cudaStream_t st);
cudaError_t launch_grid_p4(const Params& prm, int mode, int q, cudaStream_t st);
cudaError_t launch_grid_p5(const Params& prm, int mode, int q, cudaStream_t st);
}  // namespace nb
