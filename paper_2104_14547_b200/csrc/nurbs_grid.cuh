// nurbs_grid.cuh — the fused grid kernel of the NURBS-Diff hot path (arXiv 2104.14547).
//
// Citations: P:n = reference/PAPER.md line n; R<k> = reading k of DESIGN.md §3.
//
// The grid case is evaluated as the separable banded product S' = N_u · Q · N_v^T (Eq.3
// P:110 with the homogeneous points of P:140, Q_ij = (w_ij P_ij, w_ij)):
//   F1  T[i][b]  = sum_h Nv[b][h] Q[i][sv(b)-q+h]            (per CTA column block, smem)
//   F2  S'[a][b] = sum_r Nu[a][r] T[su(a)-p+r][b]            (rolling register window)
//       S = S'_xyz / S'_w                                     (P:140 step 3)
// and the backward (Eq.8 P:215 / Eq.9 P:222 / J^T g of P:251) as its transpose:
//   G[a][b]  = (g/W, -(g.S)/W)              (homogeneous upstream)
//   B1 H[i][b]  = sum_a Nu[a][i-su(a)+p] G[a][b]   (rolling accumulators, flushed in order)
//   B2 dQ[i][j] = sum_b H[i][b] Nv[b][j-sv(b)+q]   (fixed b order)
//   dP = w dQ_xyz, dw = P.dQ_xyz + dQ_w
// Every reduction runs in a fixed order; there are no floating-point atomics, so results
// are bitwise repeatable (SPEC S:157's deterministic gather, instead of the paper's scatter
// of P:289).
//
// CTA = (surface s, row block rb, column block cb). A row block is K consecutive KNOT SPANS
// of the u direction (its sample rows are those whose span falls in [S0, S0+K)), so its
// control-row band [rb*K, S0+K-1] has at most K+p <= kRMax rows; a column block is 128
// consecutive SAMPLE columns (one compute thread each). Warp 4 is a TMA producer: it streams
// grad_out rows into a 3-stage smem ring (bwd) or drains the staged output rows to HBM with
// cp.async.bulk (fwd).
#pragma once
#include "nurbs_device.cuh"

namespace nb {

// ------------------------------------------------------------------------ the grid kernel
// One row of the walk (F2, and B1 in the backward) for one column: uniform across the CTA
// except for the column data. `nu` = basis of the row, `tw` = the T window (P+1 control rows
// [lo, lo+P] of this column), `io` = this thread's 3 floats of the output / dL/dS row.
template <int P, bool BWD, bool FIT, int KG>
__device__ __forceinline__ void walk_row(const float* __restrict__ nu, const float4 (&tw)[P + 1],
                                         float4 (&acc)[P + 1], float* io, bool valid, float fit_scale,
                                         float& lsum, float (&dots)[P + 1]) {
  float4 Sp = f4(0.f);
#pragma unroll
  for (int k = 0; k <= P; ++k) Sp = fma4v(nu[k], tw[k], Sp);
  const float rw = rcp_approx(Sp.w);
  if constexpr (!BWD) {
    const float2 oxy = up2(fmul2(pk2(Sp.x, Sp.y), pk2(rw, rw)));
    if (valid) {  // always true in TMA staging (columns >= cols land in the unused row tail)
      io[0] = oxy.x;
      io[1] = oxy.y;
      io[2] = Sp.z * rw;
    }
  } else {
    float gx, gy, gz;
    if constexpr (FIT) {
      // fused fitting step (NEXT-2): io holds the target T; L = mean |S - T|^2 over the
      // points, so g = dL/dS = fit_scale * (S - T) with fit_scale = 2 / (number of points)
      const float2 sxy = up2(fmul2(pk2(Sp.x, Sp.y), pk2(rw, rw)));
      const float sz = Sp.z * rw;
      const float dx = valid ? sxy.x - io[0] : 0.f;
      const float dy = valid ? sxy.y - io[1] : 0.f;
      const float dz = valid ? sz - io[2] : 0.f;
      lsum = fmaf(dx, dx, fmaf(dy, dy, fmaf(dz, dz, lsum)));
      gx = fit_scale * dx;
      gy = fit_scale * dy;
      gz = fit_scale * dz;
    } else {
      gx = valid ? io[0] : 0.f;
      gy = valid ? io[1] : 0.f;
      gz = valid ? io[2] : 0.f;
    }
    // G = (g/W, -(g.S)/W) with S = S'_xyz / W  (Eq.8/9 through the homogeneous point)
    const float2 gxy = up2(fmul2(pk2(gx, gy), pk2(rw, rw)));
    const float gzr = gz * rw;
    const float gS = fmaf(gxy.x, Sp.x, fmaf(gxy.y, Sp.y, gzr * Sp.z));
    const float4 G = make_float4(gxy.x, gxy.y, gzr, -gS * rw);
#pragma unroll
    for (int k = 0; k <= P; ++k) acc[k] = fma4v(nu[k], G, acc[k]);
    if constexpr (KG == 1) {  // NEXT-4: G . T_r, the row's weight of dN_r/dU
#pragma unroll
      for (int k = 0; k <= P; ++k) {
        const float2 t2 = up2(ffma2(pk2(G.z, G.w), pk2(tw[k].z, tw[k].w), fmul2(pk2(G.x, G.y), pk2(tw[k].x, tw[k].y))));
        dots[k] = t2.x + t2.y;
      }
    }
  }
}

// ---- B2 of the backward for a batch of completed control rows [i0, i0+nb) held in the H
// ring: dQ[i][j] = sum_b H[i][b] Nv[b][j - sv(b) + q] in ascending b, then the Eq.8/9
// epilogue (direct mode) or the tile partial (cross-tile reduce). Called by the 128 compute
// threads together (uniform), rarely (once per kB2Batch rows, outside the unrolled row loop).
struct B2Args {
  const float4* Hring;
  const float* Nv_s;
  const int* sv_s;
  const int* sst;
  const float4* ctrl_s;   // this surface's control net
  float4* gctrl_s;        // this surface's gradient (direct mode)
  float4* slots;          // this tile's partial slot [T_rows][m] (reduce mode)
  const float4* cband;    // the staged control band (rows from band_lo, columns from jlo)
  int m, cols, band_lo, sfirst, nspan;
  int cbw, jlo, ncol;     // band row stride, first column, columns staged
  int lps;                // lanes per knot span in the fast path (power of 2, nspan*lps <= 32)
  bool fast, direct, band_in_smem;
};

template <int Q>
__device__ __forceinline__ void b2_batch_fn(const B2Args& a, int i0, int nb) {
  constexpr int NQ = (Q + 1) <= 4 ? 4 : 8;
  __syncthreads();  // H rows of the batch written by every thread
  const int t = threadIdx.x, m = a.m;
  auto store_dq = [&](int i, int j, float4 a4) {
    if (a.direct) {  // dP = w dQ_xyz, dw = P.dQ_xyz + dQ_w
      const int jj = j - a.jlo;
      float4 c;
      if (a.band_in_smem && jj >= 0 && jj < a.ncol) c = a.cband[(size_t)(i - a.band_lo) * a.cbw + jj];
      else c = __ldg(a.ctrl_s + (size_t)i * m + j);
      a.gctrl_s[(size_t)i * m + j] =
          make_float4(c.w * a4.x, c.w * a4.y, c.w * a4.z, fmaf(c.x, a4.x, fmaf(c.y, a4.y, fmaf(c.z, a4.z, a4.w))));
    } else {
      a.slots[(size_t)(i - a.band_lo) * m + j] = a4;
    }
  };
  if (a.fast) {  // one warp per control row; lps lanes per knot span of the column block
    const int lane = t & 31;
    const int L = a.lps;
    const int k = lane / L, sub = lane - k * L;
    for (int rr = (t >> 5); rr < nb; rr += kCompute / 32) {
      const int i = i0 + rr;
      const float4* Hr = a.Hring + ((i - a.band_lo) & (kHRing - 1)) * kCB;
      float4 c[Q + 1];
#pragma unroll
      for (int h = 0; h <= Q; ++h) c[h] = f4(0.f);
      if (k < a.nspan) {  // span sfirst + k, columns [sst[k], sst[k+1]) strided over its lanes
        const int e = a.sst[k + 1];
        for (int bb = a.sst[k] + sub; bb < e; bb += L) {
          const float4 hv = Hr[bb];
          float nvv[NQ];
          const float4 q0 = *reinterpret_cast<const float4*>(a.Nv_s + bb * NQ);
          nvv[0] = q0.x; nvv[1] = q0.y; nvv[2] = q0.z; nvv[3] = q0.w;
          if constexpr (NQ == 8) {
            const float4 q1 = *reinterpret_cast<const float4*>(a.Nv_s + bb * NQ + 4);
            nvv[4] = q1.x; nvv[5] = q1.y; nvv[6] = q1.z; nvv[7] = q1.w;
          }
#pragma unroll
          for (int h = 0; h <= Q; ++h) c[h] = fma4v(nvv[h], hv, c[h]);
        }
      }
      for (int o = L >> 1; o > 0; o >>= 1) {  // sum the lanes of each span group (fixed order)
#pragma unroll
        for (int h = 0; h <= Q; ++h) {
          c[h].x += __shfl_xor_sync(0xffffffffu, c[h].x, o);
          c[h].y += __shfl_xor_sync(0xffffffffu, c[h].y, o);
          c[h].z += __shfl_xor_sync(0xffffffffu, c[h].z, o);
          c[h].w += __shfl_xor_sync(0xffffffffu, c[h].w, o);
        }
      }
      // lane jj collects column j = sfirst - q + jj: sum_h c[h] of span jj - h (group (jj-h)*L)
      float4 d = f4(0.f);
#pragma unroll
      for (int h = 0; h <= Q; ++h) {
        const int ks = lane - h;
        const int src = (ks >= 0 && ks < a.nspan) ? ks * L : 0;
        const float vx = __shfl_sync(0xffffffffu, c[h].x, src);
        const float vy = __shfl_sync(0xffffffffu, c[h].y, src);
        const float vz = __shfl_sync(0xffffffffu, c[h].z, src);
        const float vw = __shfl_sync(0xffffffffu, c[h].w, src);
        if (ks >= 0 && ks < a.nspan) d = make_float4(d.x + vx, d.y + vy, d.z + vz, d.w + vw);
      }
      if (lane < a.nspan + Q) store_dq(i, a.sfirst - Q + lane, d);
      if (a.direct)  // columns this block does not touch
        for (int j = lane; j < m; j += 32)
          if (j < a.sfirst - Q || j >= a.sfirst + a.nspan) store_dq(i, j, f4(0.f));
    }
  } else {  // many spans in one block (dense knots): one (row, column) task per thread
    const int jb0 = a.sfirst - Q;
    const int jb1 = a.sfirst + a.nspan - 1;
    const int nj = a.direct ? m : jb1 - jb0 + 1;
    const int jstart = a.direct ? 0 : jb0;
    for (int task = t; task < nb * nj; task += kCompute) {
      const int rr = task / nj;
      const int j = jstart + (task - rr * nj);
      const int i = i0 + rr;
      float4 a4 = f4(0.f);
      if (j >= jb0 && j <= jb1) {
        int blo = 0, bhi = a.cols;  // first b with sv >= j
        while (blo < bhi) {
          const int mid = (blo + bhi) >> 1;
          if (a.sv_s[mid] < j) blo = mid + 1; else bhi = mid;
        }
        int bend = blo, bh2 = a.cols;  // first b with sv > j + q
        while (bend < bh2) {
          const int mid = (bend + bh2) >> 1;
          if (a.sv_s[mid] <= j + Q) bend = mid + 1; else bh2 = mid;
        }
        const float4* Hr = a.Hring + ((i - a.band_lo) & (kHRing - 1)) * kCB;
        for (int bb = blo; bb < bend; ++bb) {
          const int h = j - a.sv_s[bb] + Q;  // in [0, Q] for sorted v; guarded for unsorted v
          if (h >= 0 && h <= Q) a4 = fma4v(a.Nv_s[bb * NQ + h], Hr[bb], a4);
        }
      }
      store_dq(i, j, a4);
    }
  }
  __syncthreads();  // ring slots free again
}

// IO: how the streamed tensor (out / dL/dS / target) moves: 0 per-thread global accesses,
// 1 TMA bulk copies (one per stage when rows are contiguous, else one per row), 2 2-D TMA
// tensor copies (two boxes per stage; rows need not be contiguous).
template <int P, int Q, bool BWD, int IO, bool FIT, int KG>
#ifndef NB_MINB_F_TMAP
#define NB_MINB_F_TMAP 6  // the tensor-map forward is shared-memory-limited to 6 CTAs: use their registers
#endif
__global__ void __launch_bounds__(kThreads, BWD ? kMinBlocks_B : (IO == 2 ? NB_MINB_F_TMAP : kMinBlocks_F))
    nurbs_grid_kernel(const __grid_constant__ Params prm) {
  constexpr bool BULK = IO >= 1;
  static_assert(!FIT || BWD, "the fitting step is a backward variant");
  static_assert(KG == 0 || (BWD && !FIT), "knot gradients extend the plain backward");
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int NP = (P + 1) <= 4 ? 4 : 8;  // floats per row-basis entry in smem
  constexpr int NQ = (Q + 1) <= 4 ? 4 : 8;  // floats per column-basis entry in smem
  constexpr int RPS = BWD ? kRPS_B : kRPS_F;      // sample rows per pipeline stage
  // stages per ring (the knot-gradient variant runs 2 so that, with its dot-product buffers,
  // four CTAs still fit an SM)
  constexpr int NST = BWD ? (KG != 0 ? 2 : kStages_B) : kStages_F;
  constexpr int SROW = kCB * 3;                    // floats of one staged sample row
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const Dir& R = prm.r;
  const Dir& C = prm.c;
  const int m = C.n;

  // ---- decode the tile
  int bid = blockIdx.x;
  const int cb = bid % prm.NCB;
  bid /= prm.NCB;
  const int rb = bid % prm.NRB;
  const int s = bid / prm.NRB;
  const int B0 = cb * kCB;
  const int cols = min(kCB, C.ns - B0);
  const int S0 = P + rb * prm.K;                 // first knot span of this row block
  const int S1 = min(S0 + prm.K, R.n);           // one past the last
  const int band_lo = S0 - P;                    // control-row band [band_lo, S1-1]
  const int band_rows = S1 - band_lo;            // <= T_rows
  const float* Uk = (P > 0) ? R.knots + (long long)s * R.kstride : nullptr;
  const float* Vk = C.tspan ? nullptr : C.knots + (long long)s * C.kstride;
  const float4* __restrict__ ctrl_s = prm.ctrl + (size_t)s * R.n * m;

  // ---- shared memory carve-up (sizes: grid_smem_bytes)
  float4* cband = reinterpret_cast<float4*>(smem);                                 // [T_rows][CBW]
  // [NST] slots of RPS rows: row-major [RPS][SROW], or with the tensor map two column halves
  // [2][RPS][3*kBoxCols] (each half is one dense TMA box); 128-byte aligned
  float* stage = reinterpret_cast<float*>(smem + (((size_t)prm.T_rows * prm.CBW * 16 + 127) & ~(size_t)127));
  float4* Hring = reinterpret_cast<float4*>(stage + NST * RPS * SROW);              // [kHRing][kCB] (bwd)
  // row span / basis tables of the current chunk; in the forward with the tensor-map IO (long,
  // strided row blocks) two buffers, the next chunk copied in with cp.async while this one is
  // walked (measured: config 5 forward 0.153 -> 0.146 ms; the backward lost 1 %, so it stays)
  constexpr bool RPF = IO == 2 && P > 0 && !BWD;
  constexpr int NRT = RPF ? 2 : 1;
  int* const su_b = reinterpret_cast<int*>(Hring + (BWD ? kHRing * kCB : 0));       // [NRT][kRowChunk]
  float* const Nu_b = reinterpret_cast<float*>(su_b + NRT * kRowChunk);            // [NRT][kRowChunk][NP]
  int* su_s = su_b;
  float* Nu_s = Nu_b;
  int* sv_s = reinterpret_cast<int*>(Nu_b + NRT * kRowChunk * NP);                 // [kCB]      (bwd)
  float* Nv_s = reinterpret_cast<float*>(sv_s + kCB);                              // [kCB][NQ]  (bwd)
  int* sst = reinterpret_cast<int*>(Nv_s + kCB * NQ);                              // [kCB+4]    (bwd)
  int* misc = BWD ? sst + kCB + 4 : sv_s;                                          // [4]
  uint64_t* bars = reinterpret_cast<uint64_t*>(misc + 4);                         // 8-byte aligned
  uint64_t* band_bar = bars;            // control band landed
  uint64_t* sfull = bars + 1;           // bwd: stage slot filled by TMA (count 1 + tx bytes)
  uint64_t* sempty = bars + 1 + NST;    // fwd: stage slot drained by TMA (count 1)
  int* scnt = reinterpret_cast<int*>(bars + 1 + 2 * NST);  // per slot: warps done with the stage
  // KG: [4 warps][kRowChunk][P+1], 16-byte aligned (the stage buffers behind it are read as float4)
  float* rowdot = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(scnt + NST + 2) + 15) & ~uintptr_t(15));
  // KG == 2 (span moments): per-warp lane rows [4][32][KXS], then the per-warp
  // span sums [4][kRMax][KNX], in the same place
  constexpr int KNX = (P + 1) * (P + 1), KXS = KNX | 1;  // odd row stride: conflict-free columns
  float* kxb = rowdot;
  float* kws = kxb + (kThreads / 32) * 32 * KXS;

  if (tid == 0) {
    mbar_init(band_bar, 1u);
    for (int i = 0; i < NST; ++i) {
      mbar_init(sfull + i, 1u);
      mbar_init(sempty + i, 1u);
      scnt[i] = 0;
    }
    fence_mbar_init();
  }

  // ---- sample rows of this row block: spans in [S0, S1)
  int a_lo = 0, a_hi = R.ns;
  if (prm.NRB > 1 && R.tsfirst) {  // tables: the row block's first / past-last sample, two loads
    if (rb > 0) a_lo = min(max(__ldg(R.tsfirst + (S0 - P)), 0), R.ns);
    if (rb < prm.NRB - 1) a_hi = min(max(__ldg(R.tsfirst + (S1 - P)), a_lo), R.ns);
  } else if (prm.NRB > 1) {
    int s_end = R.n - 1;  // last non-empty span (R3)
    if (P > 0 && !R.tspan)
      while (s_end > P && __ldg(Uk + s_end) == __ldg(Uk + s_end + 1)) --s_end;
    auto ge = [&](int S) {
      return [&, S](int a) -> bool {
        if (R.tspan) return __ldg(R.tspan + a) >= S;
        if (S > s_end) return false;
        return __ldg(R.s + a) >= __ldg(Uk + S);
      };
    };
    if (rb > 0) a_lo = cta_first_true(R.ns, ge(S0));
    if (rb < prm.NRB - 1) a_hi = cta_first_true(R.ns, ge(S1));
  }
  __syncthreads();  // mbarrier init visible
  const int nwalk = max(0, a_hi - a_lo);
  const int nstage = (nwalk + RPS - 1) / RPS;
  const bool row_pf = RPF && R.tspan != nullptr;
  auto prefetch_rows = [&](int r0) {  // chunk starting at walk row r0 -> buffer (r0 / kRowChunk) & 1
    const int cn = min(kRowChunk, nwalk - r0);
    if (tid < cn) {
      const int buf = (r0 / kRowChunk) & 1;
      const int a = a_lo + r0 + tid;
      cp_async4(su_b + buf * kRowChunk + tid, R.tspan + a);
#pragma unroll
      for (int k = 0; k < NP; k += 4) cp_async16(Nu_b + (buf * kRowChunk + tid) * NP + k, R.tN + (size_t)a * NP + k);
    }
    cp_async_commit();
  };
  if (row_pf && nwalk > 0) prefetch_rows(0);

  // ---- thread 0: the control band (rows [band_lo, S1), columns [jlo, jhi] of this column
  // block) into smem with TMA bulk copies.
  if (tid == 0) {
    auto cspan = [&](int bb) -> int {
      int sp = C.tspan ? __ldg(C.tspan + bb) : d_find_span(Vk, m, Q, __ldg(C.s + bb));
      return min(max(sp, Q), m - 1);
    };
    // spans of the first and last column (sorted v); max() keeps the band non-empty and
    // in bounds when v is not sorted (unchecked mode: wrong values, never out of bounds)
    const int jlo = cspan(B0) - Q;
    const int ncol = max(cspan(B0 + cols - 1), jlo + Q) - jlo + 1;
    const int use_smem = ncol <= prm.CBW;
    misc[0] = jlo;
    misc[1] = use_smem;
    misc[2] = ncol;
    if (use_smem) {
      const uint32_t rowb = (uint32_t)ncol * 16u;
      mbar_arrive_expect_tx(band_bar, rowb * band_rows);
      const float4* src = ctrl_s + (size_t)band_lo * m + jlo;
      if (ncol == m && ncol == prm.CBW) {
        bulk_g2s(cband, src, rowb * band_rows, band_bar);
      } else {
        for (int r = 0; r < band_rows; ++r) bulk_g2s(cband + r * prm.CBW, src + (size_t)r * m, rowb, band_bar);
      }
    } else {
      mbar_arrive(band_bar);
    }
  }

  // ---- TMA stage pipeline: slot = RPS whole sample rows (cols floats x 3). No producer warp:
  // the LAST warp to finish a stage (smem counter) issues the TMA for it — the next dL/dS
  // load into the freed slot (bwd) or the drain of the filled slot to HBM (fwd).
  const uint32_t rowbytes = (uint32_t)cols * 12u;
#ifdef NB_EXP_ROWCOPIES
  const bool one_copy = false;
#else
  const bool one_copy = (cols == C.ns) && cols == kCB;  // a stage is one contiguous span
#endif
  const size_t grow = (size_t)C.ns * 3;                 // floats between consecutive rows
  const size_t g0 = (((size_t)s * R.ns + a_lo) * C.ns + B0) * 3;  // row a_lo, column B0
  // tensor-map path: column halves h = 0, 1 of the block (64 sample columns each), rows of the
  // flattened [B*n_u] row index; a partial last stage falls back to per-row copies (a full box
  // would touch the next tile's rows)
  constexpr bool tm = IO == 2;
  constexpr int HROW = 3 * kBoxCols;                    // floats of one row of a half
  const int nh = cols > kBoxCols ? 2 : 1;               // halves holding columns of this block
  const uint32_t hb0 = (uint32_t)min(cols, kBoxCols) * 12u, hb1 = (uint32_t)max(0, cols - kBoxCols) * 12u;
  const int ty0 = s * R.ns + a_lo;                      // tensor row of walk row 0
  // this thread's 3 floats of a staged row, and the distance between staged rows
  const int io_off = tm ? (tid >> 6) * (RPS * HROW) + (tid & 63) * 3 : tid * 3;
  constexpr size_t io_stride = tm ? (size_t)HROW : (size_t)SROW;
  auto issue_load = [&](int k, int slot) {  // bwd, one thread: stage k of dL/dS into `slot`
    const int nr = min(RPS, nwalk - k * RPS);
    float* buf = stage + slot * (RPS * SROW);
    const float* src = prm.gout + g0 + (size_t)k * RPS * grow;
    if constexpr (tm) {
      if (nr == RPS) {
        mbar_arrive_expect_tx(sfull + slot, (uint32_t)nh * RPS * HROW * 4u);
        for (int h = 0; h < nh; ++h) tma_load_2d(buf + h * RPS * HROW, &prm.io_map, 3 * (B0 + h * kBoxCols), ty0 + k * RPS, sfull + slot);
      } else {
        mbar_arrive_expect_tx(sfull + slot, (hb0 + hb1) * nr);
        for (int rr = 0; rr < nr; ++rr) {
          bulk_g2s(buf + rr * HROW, src + (size_t)rr * grow, hb0, sfull + slot);
          if (hb1) bulk_g2s(buf + RPS * HROW + rr * HROW, src + (size_t)rr * grow + HROW, hb1, sfull + slot);
        }
      }
    } else {
      mbar_arrive_expect_tx(sfull + slot, rowbytes * nr);
      if (one_copy) {
        bulk_g2s(buf, src, rowbytes * nr, sfull + slot);
      } else {
        for (int rr = 0; rr < nr; ++rr) bulk_g2s(buf + rr * SROW, src + (size_t)rr * grow, rowbytes, sfull + slot);
      }
    }
  };
  auto issue_store = [&](int k, int slot) {  // fwd, one thread: drain stage k from `slot`
    const int nr = min(RPS, nwalk - k * RPS);
    const float* buf = stage + slot * (RPS * SROW);
    float* dst = prm.out + g0 + (size_t)k * RPS * grow;
    if constexpr (tm) {
      if (nr == RPS) {
        for (int h = 0; h < nh; ++h) tma_store_2d(&prm.io_map, 3 * (B0 + h * kBoxCols), ty0 + k * RPS, buf + h * RPS * HROW);
      } else {
        for (int rr = 0; rr < nr; ++rr) {
          bulk_s2g(dst + (size_t)rr * grow, buf + rr * HROW, hb0);
          if (hb1) bulk_s2g(dst + (size_t)rr * grow + HROW, buf + RPS * HROW + rr * HROW, hb1);
        }
      }
    } else {
      if (one_copy) {
        bulk_s2g(dst, buf, rowbytes * nr);
      } else {
        for (int rr = 0; rr < nr; ++rr) bulk_s2g(dst + (size_t)rr * grow, buf + rr * SROW, rowbytes);
      }
    }
    bulk_commit();
    bulk_wait_read_all();  // the slot may be rewritten once TMA has read it
    mbar_arrive(sempty + slot);
  };
  if (BWD && BULK && tid == 0)
    for (int k = 0; k < min(NST, nstage); ++k) issue_load(k, k);

  // ---- column span + basis (registers); the backward also needs them in smem for B2
  const bool valid = tid < cols;
  const int b = B0 + (valid ? tid : cols - 1);
  int sv;
  float nv[Q + 1];
  if (C.tspan) {
    sv = __ldg(C.tspan + b);
    const float* tn = C.tN + (size_t)b * C.tnp;
#pragma unroll
    for (int h = 0; h <= Q; ++h) nv[h] = __ldg(tn + h);
  } else {
    const float vb = __ldg(C.s + b);
    sv = d_find_span(Vk, m, Q, vb);
    d_basis<Q>(Vk, sv, vb, Q, nv);
  }
  sv = min(max(sv, Q), m - 1);

  // ---- F1 on demand: T(i) = sum_h Nv[h] Q[i][sv - q + h]  (P:140 homogeneous points)
  mbar_wait(band_bar, 0);
  const int jlo = misc[0];
  const bool band_in_smem = misc[1] != 0;
  // the block's spans lie in [jlo + Q, jlo + ncol - 1] when v is sorted; clamping keeps the
  // band reads and B2's column indices in bounds for unsorted v too (memory safety only)
  sv = min(max(sv, jlo + Q), jlo + misc[2] - 1);
  if constexpr (BWD) {
    sv_s[tid] = sv;
#pragma unroll
    for (int h = 0; h < NQ; ++h) Nv_s[tid * NQ + h] = h <= Q ? nv[h <= Q ? h : 0] : 0.f;
  }
  const float4* cb0 = cband + (sv - Q - jlo) - (size_t)band_lo * prm.CBW;  // smem band, row 0
  const float4* cg0 = ctrl_s + (sv - Q);                                     // global, row 0

  // ---- backward: knot spans present in this column block. B2 runs one warp per control row
  // with one lane per span when the block touches at most 32 - q consecutive spans.
  int sfirst = 0, nspan = 0;
  bool b2fast = false;
  if constexpr (BWD) {
    __syncthreads();  // sv_s / Nv_s complete
    sfirst = sv_s[0];
    nspan = sv_s[cols - 1] - sfirst + 1;
    b2fast = nspan + Q <= 32;
    if (b2fast) {
      for (int k = tid; k <= nspan; k += kThreads) {  // sst[k] = first b with sv(b) >= sfirst + k
        int lo2 = 0, hi2 = cols;
        while (lo2 < hi2) {
          const int mid = (lo2 + hi2) >> 1;
          if (sv_s[mid] < sfirst + k) lo2 = mid + 1; else hi2 = mid;
        }
        sst[k] = lo2;
      }
    }
  }
  B2Args b2a;
  if constexpr (BWD) {
    b2a.Hring = Hring; b2a.Nv_s = Nv_s; b2a.sv_s = sv_s; b2a.sst = sst;
    b2a.ctrl_s = ctrl_s; b2a.gctrl_s = prm.gctrl + (size_t)s * R.n * m;
    b2a.slots = prm.slots ? prm.slots + (((size_t)s * prm.NRB + rb) * prm.NCB + cb) * prm.T_rows * m : nullptr;
    b2a.cband = cband;
    b2a.m = m; b2a.cols = cols; b2a.band_lo = band_lo; b2a.sfirst = sfirst; b2a.nspan = nspan;
    b2a.cbw = prm.CBW; b2a.jlo = jlo; b2a.ncol = misc[2];
    int L = 32;
    while (L > 1 && nspan * L > 32) L >>= 1;
    b2a.lps = L;
    b2a.fast = b2fast; b2a.direct = prm.direct; b2a.band_in_smem = band_in_smem;
  }
  // One generic pointer + stride for both sources (the staged band in smem, or the net in
  // global memory when the block's columns do not fit the band): a uniform select once per
  // CTA instead of two predicated load paths in every unrolled window advance.
  const float4* tb0 = band_in_smem ? cb0 : cg0;
  const size_t tstride = band_in_smem ? (size_t)prm.CBW : (size_t)m;
  auto Trow = [&](int i) -> float4 {
    const float4* src = tb0 + (size_t)i * tstride;
    float4 a = f4(0.f);
#pragma unroll
    for (int h = 0; h <= Q; ++h) a = fma4v(nv[h], homog(src[h]), a);
    return a;
  };

  // ---- B2 (backward): batches of completed rows in the H ring -> dQ (b2_batch_fn)
#ifdef NB_EXP_NO_B2
  auto b2_batch = [&](int i0, int nb) { (void)i0; (void)nb; };
#elif defined(NB_EXP_B2_NOSYNC_WORK)
  auto b2_batch = [&](int i0, int nb) { __syncthreads(); __syncthreads(); (void)i0; (void)nb; };
#else
  auto b2_batch = [&](int i0, int nb) { b2_batch_fn<Q>(b2a, i0, nb); };
#endif
  int b2_next = band_lo;  // first completed control row not yet reduced by B2
  // row i complete (uniform across the CTA): H(i) -> ring. The fast variant never reduces
  // (the stage loop guarantees ring capacity); the checked one reduces a full ring.
  float hv[Q + 1];  // KG: this column's sum over control rows i of Q[i][sv-q+h] . H[i][b]
#pragma unroll
  for (int h = 0; h <= Q; ++h) hv[h] = 0.f;
  auto flush_fast = [&](int i, float4 hrow) {
    Hring[((i - band_lo) & (kHRing - 1)) * kCB + tid] = hrow;
    if constexpr (KG != 0) {
      const float4* src = tb0 + (size_t)i * tstride;
#pragma unroll
      for (int h = 0; h <= Q; ++h) {
        const float4 q4 = homog(src[h]);
        hv[h] = fmaf(q4.x, hrow.x, fmaf(q4.y, hrow.y, fmaf(q4.z, hrow.z, fmaf(q4.w, hrow.w, hv[h]))));
      }
    }
  };
  auto flush_checked = [&](int i, float4 h) {
    flush_fast(i, h);
    if (i + 1 - b2_next == kHRing) {
      b2_batch(b2_next, kHRing);
      b2_next += kHRing;
    }
  };

  // ---- walk the sample rows: rolling window of P+1 control rows [lo, lo+P]
  float4 tw[P + 1];
  float4 acc[P + 1];
  int lo = band_lo;
#pragma unroll
  for (int k = 0; k <= P; ++k) {
    tw[k] = Trow(band_lo + k);
    acc[k] = f4(0.f);
  }

  if constexpr (KG == 2) {  // start dot products of the first window (acc = 0) and the span sums
    for (int x = lane; x < 32 * KXS; x += 32) kxb[warp * 32 * KXS + x] = 0.f;
    for (int x = lane; x < kRMax * KNX; x += 32) kws[warp * kRMax * KNX + x] = 0.f;
    __syncwarp();
  }
  // TMA staging: columns >= cols use the unused row tail (the fit step still masks its loss)
  const bool vio = (BULK && !FIT && KG == 0) ? true : valid;
  // KG: the warp sums of G . T_r per walk row -> rowdot[warp][ci][r]. Each lane parks its
  // p+1 dot products of the stage's rows in a per-warp buffer (row stride 33 floats: the
  // column reads below are bank-conflict free); at the end of the stage lane l sums one
  // (row, r) pair over the 32 lanes in lane order (deterministic) — no per-row shuffles.
  // KG: the warp sums of G . T_r per walk row -> rowdot[warp][ci][r]. Each lane parks its
  // p+1 dot products of the stage's rows in a per-warp buffer (row stride 36 floats: 16-byte
  // rows, conflict-free float4 reads); every KGR rows, two lanes sum one (row, r) pair's 32
  // lane values — 16 each as four float4 in a fixed tree — and one xor shuffle joins the
  // halves (deterministic, all 32 lanes busy).
  constexpr int KGS = 36, KGR = 4;  // buffer row stride, rows per buffer fill
  float* kgb = rowdot + (kThreads / 32) * kRowChunk * (P + 1) + warp * (KGR * (P + 1) * KGS);
  auto kg_row = [&](int ci, const float (&d)[P + 1]) {
    if constexpr (KG == 1) {
      const int rr = ci % KGR;
#pragma unroll
      for (int k = 0; k <= P; ++k) kgb[(rr * (P + 1) + k) * KGS + lane] = d[k];
    }
  };
  auto kg_stage = [&](int ci0, int nr) {
    if constexpr (KG == 1) {
      __syncwarp();
      const int npair = nr * (P + 1), half = lane & 1;
      for (int base = 0; base < npair; base += 16) {  // uniform trip count (P > 3: two rounds)
        const int pr = base + (lane >> 1);
        float v = 0.f;
        if (pr < npair) {
          const float4* src = reinterpret_cast<const float4*>(kgb + pr * KGS + half * 16);
          const float4 a = src[0], b = src[1], c = src[2], d = src[3];
          v = (((a.x + a.y) + (a.z + a.w)) + ((b.x + b.y) + (b.z + b.w))) +
              (((c.x + c.y) + (c.z + c.w)) + ((d.x + d.y) + (d.z + d.w)));
        }
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        if (half == 0 && pr < npair) {
          const int rr = pr / (P + 1), k = pr - rr * (P + 1);
          rowdot[(warp * kRowChunk + ci0 + rr) * (P + 1) + k] = v;
        }
      }
      __syncwarp();
    }
  };
  // KG: rows [r0, r0 + cn) of the walk are complete in rowdot (after a barrier): warp sums in
  // warp order -> hU[s][cb][a][r] (fixed-order partial of the column block)
  auto kg_flush = [&](int r0, int cn) {
    if constexpr (KG == 1) {
      for (int x = tid; x < cn * (P + 1); x += kThreads) {
        const int row = x / (P + 1), k = x - row * (P + 1);
        float v = 0.f;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) v += rowdot[(w * kRowChunk + row) * (P + 1) + k];
        prm.hU[(((size_t)s * prm.NCB + cb) * R.ns + a_lo + r0 + row) * (P + 1) + k] = v;
      }
    }
  };
  // KG == 2: row-direction knot weights as span moments (NEXT-4). On a knot span
  // the window's T rows are fixed and B1's accumulator acc[r'] gains sum_a N_r'(u_a) G_ab over
  // the span's rows, so X[r][r'] = sum_b T_r(b) . (acc[r'] at span end - at span start) are the
  // moments the assembly needs (the knot derivative of N_r is a combination of the span's N_r').
  // Each lane keeps its start dot products in its kxb row; at the span end it replaces them by
  // end - start, and the warp sums the (p+1)^2 columns over its 32 lanes (lane pairs, fixed
  // order + one xor shuffle) into kws[warp][span - S0]. No per-row work (chosen for long spans).
  int kg_open = 0;  // rows processed in the current window (uniform)
  auto kdot = [](float4 a, float4 b) {
    const float2 t = up2(ffma2(pk2(a.z, a.w), pk2(b.z, b.w), fmul2(pk2(a.x, a.y), pk2(b.x, b.y))));
    return t.x + t.y;
  };
  auto kg_span_start = [&]() {  // the window just moved: start dot products (acc[p] = 0)
    if constexpr (KG == 2) {
      float* xr = kxb + (warp * 32 + lane) * KXS;
#pragma unroll
      for (int r = 0; r <= P; ++r)
#pragma unroll
        for (int q = 0; q < P; ++q) xr[r * (P + 1) + q] = kdot(tw[r], acc[q]);
    }
  };
  auto kg_span_end = [&](int span) {  // window [lo, lo+p] = knot span lo+p is complete
    if constexpr (KG == 2) {
      float* xw = kxb + warp * 32 * KXS;
      float* xr = xw + lane * KXS;
#pragma unroll
      for (int r = 0; r <= P; ++r) {
#pragma unroll
        for (int q = 0; q < P; ++q) xr[r * (P + 1) + q] = kdot(tw[r], acc[q]) - xr[r * (P + 1) + q];
        xr[r * (P + 1) + P] = kdot(tw[r], acc[P]);  // slot p starts every span at zero
      }
      __syncwarp();
      float* dst = kws + (warp * kRMax + (span - S0)) * KNX;
#pragma unroll
      for (int base = 0; base < KNX; base += 16) {  // lanes (v, half): v = base + lane/2
        const int v = base + (lane >> 1), half = lane & 1;
        float x = 0.f;
        if (v < KNX) {
          float y[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) y[j] = xw[(half * 16 + j) * KXS + v];
#pragma unroll
          for (int o = 8; o > 0; o >>= 1)  // fixed pairwise tree
#pragma unroll
            for (int j = 0; j < o; ++j) y[j] += y[j + o];
          x = y[0];
        }
        x += __shfl_xor_sync(0xffffffffu, x, 1);
        if (half == 0 && v < KNX) dst[v] += x;
      }
      __syncwarp();
      kg_open = 0;
    }
  };
  const float fit_scale = prm.fit_scale;
  float lsum = 0.f;  // FIT: this thread's sum of |S - T|^2
  // One row of the walk: advance the window to the row's span if it changed (uniform across
  // the CTA, rare: once per knot span), then F2 (+ B1). ci = row index in the smem tables.
  auto row_step = [&](int ci, float* io, auto flush, bool chg) {
    // the window only moves forward: a row whose span is below the window's (unsorted u,
    // unchecked mode) is evaluated with the current window — wrong values, never out of bounds
    const int target = chg ? su_s[ci] - P : lo;
    if (target > lo) {
      if constexpr (KG == 2) {
        if (kg_open) kg_span_end(lo + P);
      }
#ifndef NB_EXP_UNROLL_ADV
#pragma unroll 1  // keep the (rare) window advance compact: unrolling it bloats the row loop
#endif
      do {  // row lo is complete
        if constexpr (BWD) flush(lo, acc[0]);
#pragma unroll
        for (int k = 0; k < P; ++k) {
          tw[k] = tw[k + 1];
          if constexpr (BWD) acc[k] = acc[k + 1];
        }
        ++lo;
        tw[P] = Trow(lo + P);
        if constexpr (BWD) acc[P] = f4(0.f);
      } while (lo < target);
      kg_span_start();
    }
    if constexpr (KG == 2) kg_open = 1;
    const float* nup = Nu_s + ci * NP;
    float nu[NP];
    const float4 n0 = *reinterpret_cast<const float4*>(nup);
    nu[0] = n0.x; nu[1] = n0.y; nu[2] = n0.z; nu[3] = n0.w;
    if constexpr (NP == 8) {
      const float4 n1 = *reinterpret_cast<const float4*>(nup + 4);
      nu[4] = n1.x; nu[5] = n1.y; nu[6] = n1.z; nu[7] = n1.w;
    }
    float dots[P + 1];
    walk_row<P, BWD, FIT, KG>(nu, tw, acc, io, vio, fit_scale, lsum, dots);
    kg_row(ci, dots);
  };
  // rows [r0, r0+nr) of the walk: unrolled fast paths when the window does not move (no span
  // checks at all) or when the H ring cannot overflow
  auto run_rows = [&](int ci0, int nr, float* io0, size_t io_stride) {
    const int lo_end = max(lo, su_s[ci0 + nr - 1] - P);  // spans are non-decreasing
    if (nr == RPS && lo_end == lo) {
#pragma unroll
      for (int r = 0; r < RPS; ++r) {
        const float* nup = Nu_s + (ci0 + r) * NP;
        float nu[NP];
        const float4 n0 = *reinterpret_cast<const float4*>(nup);
        nu[0] = n0.x; nu[1] = n0.y; nu[2] = n0.z; nu[3] = n0.w;
        if constexpr (NP == 8) {
          const float4 n1 = *reinterpret_cast<const float4*>(nup + 4);
          nu[4] = n1.x; nu[5] = n1.y; nu[6] = n1.z; nu[7] = n1.w;
        }
        float dots[P + 1];
        walk_row<P, BWD, FIT, KG>(nu, tw, acc, io0 + r * io_stride, vio, fit_scale, lsum, dots);
        kg_row(ci0 + r, dots);
        if ((r + 1) % KGR == 0) kg_stage(ci0 + r + 1 - KGR, KGR);
      }
      if constexpr (KG == 2) kg_open = 1;
      return;
    }
    bool fast = nr == RPS;
    if constexpr (BWD) fast = fast && (lo_end - b2_next) <= kHRing;  // ring capacity
    if (fast) {
      // backward: the rows whose span differs from the previous row's, as one warp-uniform
      // mask (a ballot), so each unrolled row tests a bit instead of re-reading its span
      const int rl = min(lane, RPS - 1);
      const int sp = su_s[ci0 + rl] - P;
      const int pv = rl == 0 ? lo : su_s[ci0 + rl - 1] - P;
      const unsigned chg = BWD ? __ballot_sync(0xffffffffu, lane < RPS && sp != pv) : ~0u;
#pragma unroll
      for (int r = 0; r < RPS; ++r) {
        row_step(ci0 + r, io0 + r * io_stride, flush_fast, (chg >> r) & 1u);
        if ((r + 1) % KGR == 0) kg_stage(ci0 + r + 1 - KGR, KGR);
      }
    } else {
      for (int r = 0; r < nr; ++r) {
        row_step(ci0 + r, io0 + r * io_stride, flush_checked, true);
        if ((r + 1) % KGR == 0 || r == nr - 1) kg_stage(ci0 + r / KGR * KGR, r % KGR + 1);
      }
    }
    if constexpr (BWD) {
      while (lo - b2_next >= kB2Batch) {
        b2_batch(b2_next, kB2Batch);
        b2_next += kB2Batch;
      }
    }
  };

  // direct (non-TMA) path: this thread's element of row a_lo in out / grad_out
  float* gio = nullptr;
  if constexpr (!BULK) {
    gio = (BWD ? const_cast<float*>(prm.gout) : prm.out) + (((size_t)s * R.ns + a_lo) * C.ns + b) * 3;
  }

  int slot = 0, use = 0;
  for (int st = 0; st < nstage; ++st) {
    const int r0 = st * RPS;                  // walk index of the stage's first row
    const int nr = min(RPS, nwalk - r0);
    const int ci0 = r0 % kRowChunk;           // kRowChunk is a multiple of RPS
    if (ci0 == 0) {                           // stage span + basis of the next kRowChunk rows
      if (r0 > 0) __syncthreads();            // previous chunk fully consumed
      if (KG == 1 && r0 > 0) kg_flush(r0 - kRowChunk, kRowChunk);
      const int cn = min(kRowChunk, nwalk - r0);
      if (row_pf) {
        const int buf = (r0 / kRowChunk) & 1;
        su_s = su_b + buf * kRowChunk;
        Nu_s = Nu_b + buf * kRowChunk * NP;
        cp_async_wait_all();  // this thread's copies of the chunk have landed
        if (tid < cn) su_s[tid] = min(max(su_s[tid], S0), S1 - 1);  // memory safety (inconsistent inputs)
        __syncthreads();
        if (r0 + kRowChunk < nwalk) prefetch_rows(r0 + kRowChunk);  // into the other buffer
      } else if (tid < cn) {
        const int a = a_lo + r0 + tid;
        int su;
        float nu[P + 1];
        if constexpr (P == 0) {
          su = 0;
          nu[0] = 1.f;
        } else {
          if (R.tspan) {
            su = __ldg(R.tspan + a);
            const float* tn = R.tN + (size_t)a * R.tnp;
#pragma unroll
            for (int k = 0; k <= P; ++k) nu[k] = __ldg(tn + k);
          } else {
            const float ua = __ldg(R.s + a);
            su = d_find_span(Uk, R.n, P, ua);
            d_basis<P>(Uk, su, ua, P, nu);
          }
        }
        su_s[tid] = min(max(su, S0), S1 - 1);  // memory safety for inconsistent inputs
#pragma unroll
        for (int k = 0; k < NP; ++k) Nu_s[tid * NP + k] = (k <= P) ? nu[k <= P ? k : 0] : 0.f;
      }
      if (!row_pf) __syncthreads();
    }
    if constexpr (BULK) {
      float* sslot = stage + slot * (RPS * SROW);
      if constexpr (BWD) mbar_wait(sfull + slot, use & 1);
      else if (use > 0) mbar_wait(sempty + slot, (use - 1) & 1);
      run_rows(ci0, nr, sslot + io_off, io_stride);
      if constexpr (!BWD) fence_proxy_async();  // this thread's staged rows -> async proxy
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();  // release this warp's part of the stage
        const int done = atomicAdd(scnt + slot, 1);
        if (done == kThreads / 32 - 1) {  // last warp of this stage
          scnt[slot] = 0;
          __threadfence_block();  // acquire the other warps' parts
          if constexpr (BWD) {
            if (st + NST < nstage) issue_load(st + NST, slot);
          } else {
            issue_store(st, slot);
          }
        }
      }
    } else {
      run_rows(ci0, nr, gio + (size_t)r0 * grow, grow);
    }
    if (++slot == NST) { slot = 0; ++use; }
  }
  if constexpr (BULK && !BWD) bulk_wait_all();  // every store this thread issued has landed
  if constexpr (KG == 1) {
    __syncthreads();
    if (nwalk > 0) kg_flush((nstage - 1) * RPS / kRowChunk * kRowChunk, nwalk - (nstage - 1) * RPS / kRowChunk * kRowChunk);
  }
  if constexpr (KG == 2) {  // the last span's moments, then this tile's sums in warp order -> hU
    if (kg_open) kg_span_end(lo + P);
    __syncthreads();
    const int nsp = R.n - P;
    for (int x = tid; x < (S1 - S0) * KNX; x += kThreads) {
      const int sr = x / KNX, v = x - sr * KNX;
      float acc_x = 0.f;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) acc_x += kws[(w * kRMax + sr) * KNX + v];
      prm.hU[(((size_t)s * prm.NCB + cb) * nsp + (S0 - P + sr)) * KNX + v] = acc_x;
    }
  }

  if constexpr (BWD) {
    // ---- B1 epilogue: flush the last window and the rows never reached (zeros), in order
#pragma unroll
    for (int k = 0; k <= P; ++k) flush_checked(lo + k, acc[k]);
    for (int i = lo + P + 1; i < S1; ++i) flush_checked(i, f4(0.f));
    if (b2_next < S1) b2_batch(b2_next, S1 - b2_next);

    if constexpr (FIT) {  // per-CTA loss partial, fixed-order reduction
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
      float* lw = reinterpret_cast<float*>(su_s);  // the row tables are free now
      __syncthreads();
      if (lane == 0) lw[warp] = lsum;
      __syncthreads();
      if (tid == 0) prm.loss_parts[blockIdx.x] = (lw[0] + lw[1]) + (lw[2] + lw[3]);
    }
    if constexpr (KG != 0) {  // this tile's partial of hV[s][rb][b][h]
      if (valid)
#pragma unroll
        for (int h = 0; h <= Q; ++h) prm.hV[(((size_t)s * prm.NRB + rb) * C.ns + B0 + tid) * (Q + 1) + h] = hv[h];
    }
    if (!prm.direct && rb == 0 && tid == 0) prm.colband[(size_t)s * prm.NCB + cb] = make_int2(sfirst - Q, sfirst + nspan - 1);
    if (prm.direct && KG == 0) {  // knot gradients are zero by definition
      if (prm.gR && s < prm.gR_items)
        for (int x = tid; x < prm.gR_per; x += kThreads) prm.gR[(size_t)s * prm.gR_per + x] = 0.f;
      if (prm.gC && s < prm.gC_items)
        for (int x = tid; x < prm.gC_per; x += kThreads) prm.gC[(size_t)s * prm.gC_per + x] = 0.f;
    }
  }
}

template <int P, int Q, bool BWD, int IO, bool FIT, int KG = 0>
static cudaError_t launch_one(const Params& prm, cudaStream_t st) {
  const size_t smem = grid_smem_bytes(BWD, P, Q, prm.T_rows, prm.CBW, KG, IO == 2);
  // the dynamic shared-memory opt-in is per device (a benign race: setting it twice is harmless)
  static bool attr_set[64] = {};
  int dev = 0;
  cudaError_t e0 = cudaGetDevice(&dev);
  if (e0 != cudaSuccess) return e0;
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(nurbs_grid_kernel<P, Q, BWD, IO, FIT, KG>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  const unsigned grid = (unsigned)((long long)prm.B * prm.NRB * prm.NCB);
  nurbs_grid_kernel<P, Q, BWD, IO, FIT, KG><<<grid, kThreads, smem, st>>>(prm);
  return cudaGetLastError();
}

// mode: 0 forward, 1 backward, 2 fused fitting step (backward with dL/dS from a target),
// 3 backward with the knot-gradient partials (NEXT-4; per-row weights), 4 the same with
// span moments for the rows direction
template <int P, int Q, int IO>
static cudaError_t launch_pq_io(const Params& prm, int mode, cudaStream_t st) {
  if (mode == 4) return launch_one<P, Q, true, IO, false, 2>(prm, st);
  if (mode == 3) return launch_one<P, Q, true, IO, false, 1>(prm, st);
  if (mode == 2) return launch_one<P, Q, true, IO, true>(prm, st);
  if (mode == 1) return launch_one<P, Q, true, IO, false>(prm, st);
  return launch_one<P, Q, false, IO, false>(prm, st);
}
template <int P, int Q>
static cudaError_t launch_pq(const Params& prm, int mode, cudaStream_t st) {
  if (prm.bulk && prm.tmap) return launch_pq_io<P, Q, 2>(prm, mode, st);
  if (prm.bulk) return launch_pq_io<P, Q, 1>(prm, mode, st);
  return launch_pq_io<P, Q, 0>(prm, mode, st);
}

template <int P>
static cudaError_t launch_p(const Params& prm, int mode, int q, cudaStream_t st) {
#ifdef NB_EXPERIMENT_PQ33  // tuning experiments: only the bicubic kernels
  if constexpr (P == 3) {
    if (q == 3) return launch_pq<3, 3>(prm, mode, st);
  }
  return cudaErrorNotSupported;
#else
  switch (q) {
    case 1: return launch_pq<P, 1>(prm, mode, st);
    case 2: return launch_pq<P, 2>(prm, mode, st);
    case 3: return launch_pq<P, 3>(prm, mode, st);
    case 4: return launch_pq<P, 4>(prm, mode, st);
    case 5: return launch_pq<P, 5>(prm, mode, st);
    default: return cudaErrorInvalidValue;
  }
#endif
}

}  // namespace nb
