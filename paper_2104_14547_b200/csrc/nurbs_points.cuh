// nurbs_points.cuh — paired (scattered) parameter points, NEXT-1 of DESIGN.md §8.
//
// Citations: P:n = reference/PAPER.md line n; R<k> = reading k of DESIGN.md §3.
//
// Every point t of surface k carries its own (u, v) = uv[k][t] (S(u,v) over the whole domain,
// P:96-102; Alg.1's per-point span and basis). There is no grid structure to
// factor, so each point does FindSpan (binary search over smem knots), the A2.2
// triangle in registers, and the (p+1)(q+1) homogeneous sum itself:
//   T_r = sum_h Nv[h] Q[su-p+r][sv-q+h],  S' = sum_r Nu[r] T_r,  S = S'_xyz / S'_w.
// The A2.2 denominators right[r+1] + left[j-r] equal U[s+r+1] - U[s+r+1-j] (independent of
// u); their reciprocals are tabulated per span in smem once per CTA (R23), so the basis
// needs no division per point.
//
// Backward (Eq.8 P:215 / Eq.9 P:222 through G = (g/W, -(g.S)/W), as in the grid kernel):
//   dQ[i][j] = sum over points of Nu[i-su+p] Nv[j-sv+q] G,  dP = w dQ_xyz, dw = P.dQ_xyz + dQ_w.
// A point touches the (p+1)(q+1) control points of its knot CELL (su, sv). To make the sum
// deterministic without atomics, each CTA (surface, chunk of points) sorts its points by
// cell with a stable in-smem counting sort, then groups of kGrp lanes each own one cell:
// every lane accumulates its points' contributions to the cell's (p+1)(q+1) control points
// in registers, the group reduces them in a fixed butterfly order, and the group adds the
// cell's totals into its warp's private dQ copy in fixed group order. The warp copies are
// summed in warp order, the chunk partials (if a surface has several chunks) in chunk
// order. Every order is a function of the input only: results are bitwise repeatable.
#pragma once
#include "nurbs_device.cuh"

namespace nb {

constexpr int kPtsThreads = 256;                 // 8 warps
constexpr int kPtsWarps = kPtsThreads / 32;
#ifndef NB_KGRP
#define NB_KGRP 8
#endif
constexpr int kGrp = NB_KGRP;                    // lanes per cell in the backward
constexpr int kGrpPerWarp = 32 / kGrp;
constexpr int kGroups = kPtsWarps * kGrpPerWarp;

__host__ __device__ constexpr int tri(int p) { return p * (p + 1) / 2; }

struct PtsParams {
  int B, n, m, N;             // surfaces, control counts, points per surface
  const float* U;             // [n+p+1] or [B][n+p+1]
  const float* V;
  long long ustride, vstride; // floats between surfaces' knot vectors (0 = shared)
  const float2* uv;           // [B][N]
  const float4* ctrl;         // [B][n][m]
  float* out;                 // [B][N][3]
  const float* gout;          // [B][N][3]
  float4* gctrl;              // [B][n][m]
  int chunk, nchunk;          // points per CTA, CTAs per surface
  float4* slots;              // [B][nchunk][n*m] partial dQ (nchunk > 1)
  int ctrl_smem;              // fwd: stage the homogeneous net in smem
};

// ---- smem layout of the per-CTA knot data: U, V (for FindSpan), then one record per knot
// span and direction: rec[0..2p) = U[s-p+1 .. s+p] (the knots A2.2 reads) and
// rec[2p + tri(j-1) + r] = 1 / (U[s+r+1] - U[s+r+1-j]) (R23), padded to a float4 multiple.
__host__ __device__ constexpr int rec_len(int p) { return (2 * p + tri(p) + 3) / 4 * 4; }
struct PtsKnots {
  int offV, offRU, offRV, floats;
};
__host__ __device__ inline PtsKnots pts_knots(int n, int m, int p, int q) {
  PtsKnots k;
  k.offV = n + p + 1;
  k.offRU = (k.offV + m + q + 1 + 3) / 4 * 4;
  k.offRV = k.offRU + (n - p) * rec_len(p);
  k.floats = k.offRV + (m - q) * rec_len(q);
  return k;
}

// FindSpan (R2-R4) over knots in smem: the largest s in [p, n-1] with U[s] <= u,
// stepped down over empty intervals (only possible at u == U[n]); out-of-domain u is clamped
// (the checked mode rejects it). The walk starts from the uniform-knot guess
// p + floor((u - U[p]) (n-p) / (U[n] - U[p])) and moves until U[s] <= u < U[s+1], so the
// result is the exact A2.1 span for any knots (one or two compares for near-uniform ones).
// Plain fp32 comparisons: bit-exact with the oracle.
__device__ __forceinline__ int s_find_span(const float* U, int n, int p, float u, float u0, float scale) {
  const float t = fminf(fmaxf((u - u0) * scale, 0.f), (float)(n - p - 1));
  int s = p + (int)t;
  const float a = U[s], b = U[s + 1];
  if (a <= u && u < b) return s;  // the guess (exact for uniform knots away from the end)
  while (s < n - 1 && U[s + 1] <= u) ++s;
  while (s > p && U[s] > u) --s;
  while (s > p && U[s] == U[s + 1]) --s;
  return s;
}

// A2.2 (Eq.4) from a span record (registers or smem).
template <int P, typename R>
__device__ __forceinline__ void basis_rec(const R& rec, float u, float (&N)[P + 1]) {
  float left[P + 1], right[P + 1];
  N[0] = 1.f;
#pragma unroll
  for (int j = 1; j <= P; ++j) {
    left[j] = u - rec[P - j];         // u - U[s+1-j]
    right[j] = rec[P - 1 + j] - u;    // U[s+j] - u
    float saved = 0.f;
#pragma unroll
    for (int r = 0; r < j; ++r) {
      const float temp = N[r] * rec[2 * P + tri(j - 1) + r];
      N[r] = fmaf(right[r + 1], temp, saved);
      saved = left[j - r] * temp;
    }
    N[j] = saved;
  }
}

// The u and v bases of one point at once when p == q: the same A2.2 steps on (u, v) pairs
// with packed fp32x2 arithmetic (FADD2 / FMUL2 / FFMA2 round each lane like the scalar
// instructions, so the results are bitwise those of two basis_rec calls). r2[k] = (ru[k], rv[k]).
template <int P>
__device__ __forceinline__ void basis_rec2(const unsigned long long (&r2)[rec_len(P)], float u, float v,
                                           float (&Nu)[P + 1], float (&Nv)[P + 1]) {
  unsigned long long N[P + 1], left[P + 1], right[P + 1];
  const unsigned long long x = pk2(u, v);
  N[0] = pk2(1.f, 1.f);
#pragma unroll
  for (int j = 1; j <= P; ++j) {
    left[j] = fsub2(x, r2[P - j]);        // u - U[s+1-j]
    right[j] = fsub2(r2[P - 1 + j], x);   // U[s+j] - u
    unsigned long long saved = pk2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < j; ++r) {
      const unsigned long long temp = fmul2(N[r], r2[2 * P + tri(j - 1) + r]);
      N[r] = ffma2(right[r + 1], temp, saved);
      saved = fmul2(left[j - r], temp);
    }
    N[j] = saved;
  }
#pragma unroll
  for (int k = 0; k <= P; ++k) {
    const float2 t = up2(N[k]);
    Nu[k] = t.x;
    Nv[k] = t.y;
  }
}

template <int P>
__device__ __forceinline__ void load_rec(const float* src, float (&rec)[rec_len(P)]) {
#pragma unroll
  for (int k = 0; k < rec_len(P); k += 4) {
    const float4 v = *reinterpret_cast<const float4*>(src + k);
    rec[k] = v.x; rec[k + 1] = v.y; rec[k + 2] = v.z; rec[k + 3] = v.w;
  }
}

// Knots of surface s and the span records into smem (all threads; ends with a barrier).
template <int P, int Q>
__device__ __forceinline__ void pts_stage_knots(const PtsParams& prm, int s, float* ks) {
  const int n = prm.n, m = prm.m;
  const PtsKnots L = pts_knots(n, m, P, Q);
  const float* Uk = prm.U + (long long)s * prm.ustride;
  const float* Vk = prm.V + (long long)s * prm.vstride;
  for (int i = threadIdx.x; i < L.offV + m + Q + 1; i += blockDim.x)
    ks[i] = i < L.offV ? __ldg(Uk + i) : __ldg(Vk + i - L.offV);
  __syncthreads();
  constexpr int RU = rec_len(P), RV = rec_len(Q);
  const int nU = (n - P) * RU, nV = (m - Q) * RV;
  for (int e = threadIdx.x; e < nU + nV; e += blockDim.x) {
    const bool isU = e < nU;
    const int p = isU ? P : Q, R = isU ? RU : RV;
    const int k = isU ? e : e - nU;
    const int sp = k / R + p, idx = k - (k / R) * R;
    const float* K = isU ? ks : ks + L.offV;
    float val = 0.f;
    if (idx < 2 * p) {
      val = K[sp - p + 1 + idx];
    } else if (idx < 2 * p + tri(p)) {
      const int t = idx - 2 * p;
      int j = 1;
      while (tri(j) <= t) ++j;            // t = tri(j-1) + r
      const int r = t - tri(j - 1);
      const float d = K[sp + r + 1] - K[sp + r + 1 - j];
      val = d > 0.f ? 1.f / d : 0.f;      // empty spans are never selected
    }
    ks[(isU ? L.offRU : L.offRV) + k] = val;
  }
  __syncthreads();
}

// Pass 2 of the sorts: cstart[c] = exclusive prefix over cells of the NW per-row counts
// hist[w][c]; each count is replaced by its row's cursor (cell-major, then row order).
template <int NW>
__device__ __forceinline__ void pts_scan(int* hist, int* cstart, int C, int cnt) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int seg = (C + kPtsThreads - 1) / kPtsThreads;
  const int c0 = min(C, tid * seg), c1 = min(C, c0 + seg);
  int sum = 0;
  for (int ce = c0; ce < c1; ++ce)
#pragma unroll
    for (int w = 0; w < NW; ++w) sum += hist[w * (C + 1) + ce];
  int incl = sum;  // block-wide inclusive scan of the per-thread sums
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __shared__ int wsum[kPtsWarps];
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += wsum[w];
  int run = base + incl - sum;
  for (int ce = c0; ce < c1; ++ce) {
    cstart[ce] = run;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int h = hist[w * (C + 1) + ce];
      hist[w * (C + 1) + ce] = run;
      run += h;
    }
  }
  if (tid == kPtsThreads - 1) cstart[C] = cnt;
  __syncthreads();
}

// Passes 1-3 of the backward: STABLE in-smem counting sort of a chunk's cnt points by knot
// cell (su - p, sv - q). On return (after a barrier): cstart[c] .. cstart[c+1] index the
// points of cell c in sorted[], in (warp slice, position) order — a function of the input
// only (smem integer atomics from one warp execute in program order). hist
// [kPtsWarps][C+1] must be zero on entry. uv may be global or shared memory.
template <int P, int Q>
__device__ __forceinline__ void pts_sort(const float2* uv, int cnt, int n, int m, const float* Us, const float* Vs,
                                         int* hist, int* cstart, unsigned short* cell, unsigned short* sorted) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int Cv = m - Q, C = (n - P) * Cv;
  const float u0 = Us[P], su_scale = (float)(n - P) / (Us[n] - Us[P]);
  const float v0 = Vs[Q], sv_scale = (float)(m - Q) / (Vs[m] - Vs[Q]);
  // ---- pass 1: cell of every point; per-warp counts over the warp's contiguous slice
  const int per_warp = (cnt + kPtsWarps - 1) / kPtsWarps;
  const int w0 = warp * per_warp, w1 = min(cnt, w0 + per_warp);
  int* hw = hist + warp * (C + 1);
  float2 xn = (w0 + lane < w1) ? uv[w0 + lane] : make_float2(0.f, 0.f);
  for (int b = w0; b < w1; b += 32) {
    const int i = b + lane;
    const float2 x = xn;
    if (b + 32 + lane < w1) xn = uv[b + 32 + lane];  // next tile in flight
    int ce = C;  // sentinel for lanes past the slice
    if (i < w1) {
      const int su = s_find_span(Us, n, P, x.x, u0, su_scale);
      const int sv = s_find_span(Vs, m, Q, x.y, v0, sv_scale);
      ce = (su - P) * Cv + (sv - Q);
      cell[i] = (unsigned short)ce;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, ce);
    if (ce < C && lane == __ffs(peers) - 1) atomicAdd(hw + ce, __popc(peers));  // no return: RED
  }
  __syncthreads();
  pts_scan<kPtsWarps>(hist, cstart, C, cnt);
  // ---- pass 3: stable scatter (cell, warp, position in the warp's slice)
  for (int b = w0; b < w1; b += 32) {
    const int i = b + lane;
    const int ce = i < w1 ? (int)cell[i] : C;
    const unsigned peers = __match_any_sync(0xffffffffu, ce);
    const int leader = __ffs(peers) - 1;
    int pos = 0;
    if (ce < C && lane == leader) pos = atomicAdd(hw + ce, __popc(peers));
    pos = __shfl_sync(0xffffffffu, pos, leader) + __popc(peers & ((1u << lane) - 1u));
    if (ce < C) sorted[pos] = (unsigned short)i;
  }
  __syncthreads();
}

// Passes 1-3 of the forward: the same bucketing without the stability (every point's result
// is independent of the order): one count per cell, smem atomics, any order within a cell.
template <int P, int Q>
__device__ __forceinline__ void pts_bucket(const float2* uv, int cnt, int n, int m, const float* Us, const float* Vs,
                                           int* hist, int* cstart, unsigned short* cell, unsigned short* sorted) {
  const int tid = threadIdx.x;
  const int Cv = m - Q, C = (n - P) * Cv;
  const float u0 = Us[P], su_scale = (float)(n - P) / (Us[n] - Us[P]);
  const float v0 = Vs[Q], sv_scale = (float)(m - Q) / (Vs[m] - Vs[Q]);
  for (int i = tid; i < cnt; i += kPtsThreads) {
    const float2 x = uv[i];
    const int su = s_find_span(Us, n, P, x.x, u0, su_scale);
    const int sv = s_find_span(Vs, m, Q, x.y, v0, sv_scale);
    const int ce = (su - P) * Cv + (sv - Q);
    cell[i] = (unsigned short)ce;
    atomicAdd(hist + ce, 1);
  }
  __syncthreads();
  pts_scan<1>(hist, cstart, C, cnt);
  for (int i = tid; i < cnt; i += kPtsThreads) sorted[atomicAdd(hist + cell[i], 1)] = (unsigned short)i;
  __syncthreads();
}

// ------------------------------------------------------------------------ forward
// CTA = (surface, chunk of points). The chunk's (u, v) are staged in smem, bucketed by knot
// cell (pts_bucket), then groups of kGrpF lanes own cells: the cell's homogeneous control points
// and span records sit in registers, so each point costs its basis and 4(p+1)(q+1+1)
// register FMAs — no per-point gather of control points from smem (which would be
// bank-conflicted random 16-byte loads). Results go to an smem copy of the chunk's output,
// written to HBM coalesced at the end.
#ifndef NB_KGRPF
#define NB_KGRPF 4
#endif
constexpr int kGrpF = NB_KGRPF;
struct PtsFwdLayout {
  size_t uv, outs, cstart, hist, cell, sorted, knots, net, bytes;
};
__host__ __device__ inline PtsFwdLayout pts_fwd_layout(int n, int m, int p, int q, int chunk, bool net = false) {
  PtsFwdLayout L;
  const int C = (n - p) * (m - q);
  size_t o = 0;
  L.uv = o;     o += ((size_t)chunk * 8 + 15) & ~(size_t)15;
  L.outs = o;   o += (size_t)chunk * 12;
  o = (o + 15) & ~(size_t)15;
  L.cstart = o; o += (size_t)(C + 1) * 4;
  L.hist = o;   o += (size_t)(C + 1) * 4;
  L.cell = o;   o += (size_t)chunk * 2;
  L.sorted = o; o += (size_t)chunk * 2;
  o = (o + 15) & ~(size_t)15;
  L.knots = o;  o += (size_t)pts_knots(n, m, p, q).floats * 4;
  o = (o + 15) & ~(size_t)15;
  L.net = o;    o += net ? (size_t)n * m * 16 : 0;   // the homogeneous net (ctrl_smem)
  L.bytes = (o + 15) & ~(size_t)15;
  return L;
}

template <int P, int Q>
__global__ void __launch_bounds__(kPtsThreads, 2) nurbs_points_fwd_kernel(PtsParams prm) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int RU = rec_len(P), RV = rec_len(Q);
  constexpr int GPW = 32 / kGrpF, NG = kPtsWarps * GPW;
  const int s = blockIdx.x / prm.nchunk;
  const int c = blockIdx.x - s * prm.nchunk;
  const int n = prm.n, m = prm.m;
  const int Cv = m - Q, C = (n - P) * Cv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const PtsFwdLayout SL = pts_fwd_layout(n, m, P, Q, prm.chunk, prm.ctrl_smem != 0);
  const PtsKnots KL = pts_knots(n, m, P, Q);
  float2* uvs = reinterpret_cast<float2*>(smem + SL.uv);
  float* outs = reinterpret_cast<float*>(smem + SL.outs);
  int* cstart = reinterpret_cast<int*>(smem + SL.cstart);
  int* hist = reinterpret_cast<int*>(smem + SL.hist);
  unsigned short* cell = reinterpret_cast<unsigned short*>(smem + SL.cell);
  unsigned short* sorted = reinterpret_cast<unsigned short*>(smem + SL.sorted);
  float* ks = reinterpret_cast<float*>(smem + SL.knots);
  const int t0 = c * prm.chunk;
  const int cnt = min(prm.chunk, prm.N - t0);
  const float2* uv = prm.uv + (size_t)s * prm.N + t0;
  for (int i = tid; i < cnt; i += kPtsThreads) uvs[i] = __ldg(uv + i);
  for (int i = tid; i <= C; i += kPtsThreads) hist[i] = 0;
  const float4* ctrl_s = prm.ctrl + (size_t)s * n * m;
  float4* net = reinterpret_cast<float4*>(smem + SL.net);
  if (prm.ctrl_smem)  // the homogeneous net once per CTA: cells read it with smem broadcasts
    for (int i = tid; i < n * m; i += kPtsThreads) net[i] = homog(__ldg(ctrl_s + i));
  pts_stage_knots<P, Q>(prm, s, ks);  // ends with __syncthreads
  const float* Us = ks;
  const float* Vs = ks + KL.offV;
  pts_bucket<P, Q>(uvs, cnt, n, m, Us, Vs, hist, cstart, cell, sorted);

  const int grp = lane / kGrpF, gl = lane - grp * kGrpF;
  const int G = warp * GPW + grp;
  const int nsteps = (C - warp * GPW + NG - 1) / NG;
  for (int k = 0; k < nsteps; ++k) {
    const int ce = G + k * NG;
    const bool has = ce < C;
    const int beg = has ? cstart[ce] : 0, end = has ? cstart[ce + 1] : 0;
    if (end <= beg) continue;  // no shuffles below: groups may diverge freely
    const int cu = ce / Cv, cv = ce - cu * Cv;
    float4 Qc[P + 1][Q + 1];   // the cell's homogeneous control points
    if (prm.ctrl_smem) {
#pragma unroll
      for (int r = 0; r <= P; ++r)
#pragma unroll
        for (int h = 0; h <= Q; ++h) Qc[r][h] = net[(cu + r) * m + cv + h];
    } else {
#pragma unroll
      for (int r = 0; r <= P; ++r)
#pragma unroll
        for (int h = 0; h <= Q; ++h) Qc[r][h] = homog(__ldg(ctrl_s + (cu + r) * m + cv + h));
    }
    float ru[RU];  // u record in registers; the v record is read from smem (register budget)
    load_rec<P>(ks + KL.offRU + cu * RU, ru);
    const float* rv = ks + KL.offRV + cv * RV;
    for (int kk = beg + gl; kk < end; kk += kGrpF) {  // (packed u/v bases measured 2 % slower here)
      const int i = sorted[kk];
      const float2 x = uvs[i];
      float Nu[P + 1], Nv[Q + 1];
      basis_rec<P>(ru, x.x, Nu);
      basis_rec<Q>(rv, x.y, Nv);
      float4 Sp = f4(0.f);
#pragma unroll
      for (int r = 0; r <= P; ++r) {
        float4 T = f4(0.f);
#pragma unroll
        for (int h = 0; h <= Q; ++h) T = fma4v(Nv[h], Qc[r][h], T);
        Sp = fma4v(Nu[r], T, Sp);
      }
      const float rw = rcp_approx(Sp.w);
      outs[3 * i + 0] = Sp.x * rw;
      outs[3 * i + 1] = Sp.y * rw;
      outs[3 * i + 2] = Sp.z * rw;
    }
  }
  __syncthreads();
  float* out = prm.out + ((size_t)s * prm.N + t0) * 3;
  if ((reinterpret_cast<uintptr_t>(out) & 15u) == 0) {
    const int n4 = (cnt * 3) / 4;
    for (int i = tid; i < n4; i += kPtsThreads) reinterpret_cast<float4*>(out)[i] = reinterpret_cast<const float4*>(outs)[i];
    for (int i = 4 * n4 + tid; i < cnt * 3; i += kPtsThreads) out[i] = outs[i];
  } else {
    for (int i = tid; i < cnt * 3; i += kPtsThreads) out[i] = outs[i];
  }
}

// ------------------------------------------------------------------------ backward
// Reduce-scatter of NPAD floats over the kGrp lanes of a group, fixed butterfly order: at
// each level the lane with bit O set keeps the upper half and receives its partner's.
template <int O, int HALF, int NPAD>
__device__ __forceinline__ void grp_reduce_scatter(float (&acc)[NPAD], int gl) {
  if constexpr (O > 0) {
    const bool up = (gl & O) != 0;
#pragma unroll
    for (int e = 0; e < HALF; ++e) {
      const float send = up ? acc[e] : acc[e + HALF];
      const float keep = up ? acc[e + HALF] : acc[e];
      acc[e] = keep + __shfl_xor_sync(0xffffffffu, send, O);
    }
    grp_reduce_scatter<O / 2, HALF / 2, NPAD>(acc, gl);
  }
}

// smem carve-up (pts_bwd_smem_bytes mirrors it)
struct PtsBwdLayout {
  size_t dq, cstart, hist, cell, sorted, cq, knots, net, bytes;
};
__host__ __device__ inline PtsBwdLayout pts_bwd_layout(int n, int m, int p, int q, int chunk, bool net = false) {
  PtsBwdLayout L;
  const int C = (n - p) * (m - q);
  size_t o = 0;
  L.dq = o;     o += (size_t)kPtsWarps * n * m * 16;                 // per-warp dQ copies
  L.cq = o;     o += (size_t)kGroups * ((p + 1) * (q + 1) + 1) * 16;  // per-group cell net (+16 B: banks)
  L.cstart = o; o += (size_t)(C + 1) * 4;                            // cell start offsets
  L.hist = o;   o += (size_t)kPtsWarps * (C + 1) * 4;                // per-warp counts / cursors
  L.cell = o;   o += (size_t)chunk * 2;                              // cell of point i (uint16)
  L.sorted = o; o += (size_t)chunk * 2;                              // point index by cell
  o = (o + 15) & ~(size_t)15;
  L.knots = o;  o += (size_t)pts_knots(n, m, p, q).floats * 4;
  o = (o + 15) & ~(size_t)15;
  L.net = o;    o += net ? (size_t)n * m * 16 : 0;   // the homogeneous net (ctrl_smem)
  L.bytes = (o + 15) & ~(size_t)15;
  return L;
}

template <int P, int Q>
__global__ void __launch_bounds__(kPtsThreads, 2) nurbs_points_bwd_kernel(PtsParams prm) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NC = (P + 1) * (Q + 1);                 // control points of a cell
  constexpr int NV = NC * 4;                            // accumulator floats
  constexpr int NPAD = (NV + kGrp - 1) / kGrp * kGrp;   // padded for the group reduce-scatter
  constexpr int PER = NPAD / kGrp;                      // floats a lane owns after it
  const int s = blockIdx.x / prm.nchunk;
  const int c = blockIdx.x - s * prm.nchunk;
  const int n = prm.n, m = prm.m, nm = n * m;
  const int Cv = m - Q, C = (n - P) * Cv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const PtsBwdLayout SL = pts_bwd_layout(n, m, P, Q, prm.chunk, prm.ctrl_smem != 0);
  const PtsKnots KL = pts_knots(n, m, P, Q);
  float4* dqw = reinterpret_cast<float4*>(smem + SL.dq);
  float4* cq = reinterpret_cast<float4*>(smem + SL.cq);
  int* cstart = reinterpret_cast<int*>(smem + SL.cstart);
  int* hist = reinterpret_cast<int*>(smem + SL.hist);
  unsigned short* cell = reinterpret_cast<unsigned short*>(smem + SL.cell);
  unsigned short* sorted = reinterpret_cast<unsigned short*>(smem + SL.sorted);
  float* ks = reinterpret_cast<float*>(smem + SL.knots);

  for (int i = tid; i < kPtsWarps * nm; i += kPtsThreads) dqw[i] = f4(0.f);
  for (int i = tid; i < kPtsWarps * (C + 1); i += kPtsThreads) hist[i] = 0;
  float4* net = reinterpret_cast<float4*>(smem + SL.net);
  if (prm.ctrl_smem)  // the homogeneous net once per CTA
    for (int i = tid; i < nm; i += kPtsThreads) net[i] = homog(__ldg(prm.ctrl + (size_t)s * nm + i));
  pts_stage_knots<P, Q>(prm, s, ks);  // ends with __syncthreads
  const float* Us = ks;
  const float* Vs = ks + KL.offV;
  const int t0 = c * prm.chunk;
  const int cnt = min(prm.chunk, prm.N - t0);
  const float2* uv = prm.uv + (size_t)s * prm.N + t0;
  const float* g = prm.gout + ((size_t)s * prm.N + t0) * 3;
  const float4* ctrl_s = prm.ctrl + (size_t)s * nm;
#ifndef NB_PTS_NO_PREFETCH
  if (tid == 0 && cnt > 0) {  // the chunk's dL/dS into L2 while the points are sorted (pass 4 gathers it)
    // 16-byte granules inside [g, g + 3 cnt) only (a prefetch never touches bytes past the data)
    const uintptr_t a0 = (reinterpret_cast<uintptr_t>(g) + 15) & ~uintptr_t(15);
    const uintptr_t a1 = reinterpret_cast<uintptr_t>(g + 3 * (size_t)cnt) & ~uintptr_t(15);
    if (a1 > a0) prefetch_l2_bulk(reinterpret_cast<const void*>(a0), (uint32_t)(a1 - a0));
  }
#endif

  // ---- passes 1-3: stable counting sort of the chunk's points by knot cell
  pts_sort<P, Q>(uv, cnt, n, m, Us, Vs, hist, cstart, cell, sorted);

  // ---- pass 4: groups of kGrp lanes own cells; warp w's groups take cells w*4+g (+32 k)
  const int grp = lane / kGrp, gl = lane - grp * kGrp;
  const int G = warp * kGrpPerWarp + grp;
  float4* cqg = cq + G * (NC + 1);
  float4* dq = dqw + warp * nm;
  constexpr int RU = rec_len(P), RV = rec_len(Q);
  const int nsteps = (C - warp * kGrpPerWarp + kGroups - 1) / kGroups;
  for (int k = 0; k < nsteps; ++k) {
    const int ce = G + k * kGroups;
    const bool has = ce < C;
    const int beg = has ? cstart[ce] : 0, end = has ? cstart[ce + 1] : 0;
    const int cu = has ? ce / Cv : 0, cv = has ? ce - cu * Cv : 0;
    if (has && end > beg)  // the cell's homogeneous control points -> smem
      for (int e = gl; e < NC; e += kGrp) {
        const int r = e / (Q + 1), h = e - r * (Q + 1);
        cqg[e] = prm.ctrl_smem ? net[(cu + r) * m + cv + h] : homog(__ldg(ctrl_s + (cu + r) * m + cv + h));
      }
    __syncwarp();
    float ru[RU], rv[RV];  // the cell's span records, in registers for all its points
    load_rec<P>(ks + KL.offRU + cu * RU, ru);
    load_rec<Q>(ks + KL.offRV + cv * RV, rv);
    unsigned long long r2[RU];  // (u, v) record pairs for basis_rec2 (p == q)
#pragma unroll
    for (int k = 0; k < RU; ++k) r2[k] = pk2(ru[k], rv[k < RV ? k : 0]);
    float acc[NPAD];
#pragma unroll
    for (int e = 0; e < NPAD; ++e) acc[e] = 0.f;
    int kk = beg + gl;
    int in = kk < end ? sorted[kk] : 0;
    float2 xn = kk < end ? __ldg(uv + in) : make_float2(0.f, 0.f);
    float g0n = kk < end ? __ldg(g + 3 * in) : 0.f, g1n = kk < end ? __ldg(g + 3 * in + 1) : 0.f,
          g2n = kk < end ? __ldg(g + 3 * in + 2) : 0.f;
    for (; kk < end; kk += kGrp) {
      const float2 x = xn;
      const float g0 = g0n, g1 = g1n, g2 = g2n;
      if (kk + kGrp < end) {  // next point of this lane in flight
        in = sorted[kk + kGrp];
        xn = __ldg(uv + in);
        g0n = __ldg(g + 3 * in); g1n = __ldg(g + 3 * in + 1); g2n = __ldg(g + 3 * in + 2);
      }
      float Nu[P + 1], Nv[Q + 1];
#ifndef NB_PTS_NO_PACKED_BASIS
      if constexpr (P == Q) {
        basis_rec2<P>(r2, x.x, x.y, Nu, Nv);
      } else
#endif
      {
        basis_rec<P>(ru, x.x, Nu);
        basis_rec<Q>(rv, x.y, Nv);
      }
      float4 Sp = f4(0.f);
#pragma unroll
      for (int r = 0; r <= P; ++r) {
        float4 T = f4(0.f);
#pragma unroll
        for (int h = 0; h <= Q; ++h) T = fma4v(Nv[h], cqg[r * (Q + 1) + h], T);
        Sp = fma4v(Nu[r], T, Sp);
      }
      const float rw = rcp_approx(Sp.w);
      const float gx = g0 * rw, gy = g1 * rw, gz = g2 * rw;
      const float gS = fmaf(gx, Sp.x, fmaf(gy, Sp.y, gz * Sp.z));
      const float4 Gh = make_float4(gx, gy, gz, -gS * rw);   // G = (g/W, -(g.S)/W)
#pragma unroll
      for (int r = 0; r <= P; ++r) {
        const float4 Gu = make_float4(Nu[r] * Gh.x, Nu[r] * Gh.y, Nu[r] * Gh.z, Nu[r] * Gh.w);
#pragma unroll
        for (int h = 0; h <= Q; ++h) {
          float4 a = make_float4(acc[(r * (Q + 1) + h) * 4], acc[(r * (Q + 1) + h) * 4 + 1],
                                 acc[(r * (Q + 1) + h) * 4 + 2], acc[(r * (Q + 1) + h) * 4 + 3]);
          a = fma4v(Nv[h], Gu, a);
          acc[(r * (Q + 1) + h) * 4] = a.x;
          acc[(r * (Q + 1) + h) * 4 + 1] = a.y;
          acc[(r * (Q + 1) + h) * 4 + 2] = a.z;
          acc[(r * (Q + 1) + h) * 4 + 3] = a.w;
        }
      }
    }
    // group reduce-scatter (fixed butterfly): lane gl ends with acc[gl*PER .. gl*PER+PER)
    grp_reduce_scatter<kGrp / 2, NPAD / 2, NPAD>(acc, gl);
    // the cell's totals -> this warp's dQ copy, one group after another (fixed order)
#pragma unroll
    for (int gg = 0; gg < kGrpPerWarp; ++gg) {
      if (grp == gg && has && end > beg) {
#pragma unroll
        for (int e = 0; e < PER; ++e) {
          const int f = gl * PER + e;
          if (f < NV) {
            const int rh = f >> 2, comp = f & 3;
            const int r = rh / (Q + 1), h = rh - r * (Q + 1);
            float* dst = reinterpret_cast<float*>(dq + (cu + r) * m + cv + h) + comp;
            *dst += acc[e];
          }
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();

  // ---- pass 5: warp copies in warp order -> gradient (one chunk) or the chunk's partial
  float4* gctrl_s = prm.gctrl + (size_t)s * nm;
  float4* slot = prm.nchunk > 1 ? prm.slots + ((size_t)s * prm.nchunk + c) * nm : nullptr;
  for (int idx = tid; idx < nm; idx += kPtsThreads) {
    float4 d = dqw[idx];
    for (int w = 1; w < kPtsWarps; ++w) {
      const float4 e = dqw[w * nm + idx];
      d = make_float4(d.x + e.x, d.y + e.y, d.z + e.z, d.w + e.w);
    }
    if (slot) {
      slot[idx] = d;
    } else {
      const float4 cp = __ldg(ctrl_s + idx);  // dP = w dQ_xyz, dw = P.dQ_xyz + dQ_w
      gctrl_s[idx] = make_float4(cp.w * d.x, cp.w * d.y, cp.w * d.z,
                                 fmaf(cp.x, d.x, fmaf(cp.y, d.y, fmaf(cp.z, d.z, d.w))));
    }
  }
}


}  // namespace nb
