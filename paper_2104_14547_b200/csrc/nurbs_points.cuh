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
constexpr int kGrp = 8;                          // lanes per cell in the backward
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

// ---- smem layout of the per-CTA knot data: U, V, then the reciprocal tables (R23)
struct PtsKnots {
  int offV, offIU, offIV, floats;
};
__host__ __device__ inline PtsKnots pts_knots(int n, int m, int p, int q) {
  PtsKnots k;
  k.offV = n + p + 1;
  k.offIU = k.offV + m + q + 1;
  k.offIV = k.offIU + (n - p) * tri(p);
  k.floats = k.offIV + (m - q) * tri(q);
  return k;
}

// FindSpan (R2-R4) over knots in smem: largest s in [p, n-1] with U[s] <= u, stepped
// down over empty intervals (only possible at u == U[n]); out-of-domain u is clamped (the
// checked mode rejects it). Plain fp32 comparisons: bit-exact with the oracle.
__device__ __forceinline__ int s_find_span(const float* U, int n, int p, float u) {
  if (!(u >= U[p])) return p;
  int lo = p, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (U[mid] <= u) lo = mid; else hi = mid - 1;
  }
  while (lo > p && U[lo] == U[lo + 1]) --lo;
  return lo;
}

// A2.2 (Eq.4) with the tabulated reciprocal denominators of span s:
// inv[tri(j-1) + r] = 1 / (U[s+r+1] - U[s+r+1-j]).
template <int P>
__device__ __forceinline__ void basis_inv(const float* U, const float* inv, int s, float u, float (&N)[P + 1]) {
  float left[P + 1], right[P + 1];
  N[0] = 1.f;
#pragma unroll
  for (int j = 1; j <= P; ++j) {
    left[j] = u - U[s + 1 - j];
    right[j] = U[s + j] - u;
    float saved = 0.f;
#pragma unroll
    for (int r = 0; r < j; ++r) {
      const float temp = N[r] * inv[tri(j - 1) + r];
      N[r] = fmaf(right[r + 1], temp, saved);
      saved = left[j - r] * temp;
    }
    N[j] = saved;
  }
}

// Knots of surface s and the reciprocal tables into smem (all threads; ends with a barrier).
template <int P, int Q>
__device__ __forceinline__ void pts_stage_knots(const PtsParams& prm, int s, float* ks) {
  const int n = prm.n, m = prm.m;
  const PtsKnots L = pts_knots(n, m, P, Q);
  const float* Uk = prm.U + (long long)s * prm.ustride;
  const float* Vk = prm.V + (long long)s * prm.vstride;
  for (int i = threadIdx.x; i < L.offIU; i += blockDim.x)
    ks[i] = i < L.offV ? __ldg(Uk + i) : __ldg(Vk + i - L.offV);
  __syncthreads();
  const int nU = (n - P) * tri(P), nV = (m - Q) * tri(Q);
  for (int e = threadIdx.x; e < nU + nV; e += blockDim.x) {
    const bool isU = e < nU;
    const int p = isU ? P : Q;
    const int k = isU ? e : e - nU;
    const int t = tri(p);
    const int s_ = k / t + p, idx = k - (k / t) * t;
    int j = 1;
    while (tri(j) <= idx) ++j;             // idx = tri(j-1) + r
    const int r = idx - tri(j - 1);
    const float* K = isU ? ks : ks + L.offV;
    const float d = K[s_ + r + 1] - K[s_ + r + 1 - j];
    ks[(isU ? L.offIU : L.offIV) + k] = d > 0.f ? 1.f / d : 0.f;  // empty spans are never used
  }
  __syncthreads();
}

// ------------------------------------------------------------------------ forward
template <int P, int Q>
__global__ void __launch_bounds__(kPtsThreads) nurbs_points_fwd_kernel(PtsParams prm) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int s = blockIdx.x / prm.nchunk;
  const int c = blockIdx.x - s * prm.nchunk;
  const int n = prm.n, m = prm.m;
  const PtsKnots L = pts_knots(n, m, P, Q);
  float4* Qs = reinterpret_cast<float4*>(smem);                               // [n*m] (ctrl_smem)
  float* ks = reinterpret_cast<float*>(smem + (prm.ctrl_smem ? (size_t)n * m * 16 : 0));
  const float4* ctrl_s = prm.ctrl + (size_t)s * n * m;
  if (prm.ctrl_smem)
    for (int i = threadIdx.x; i < n * m; i += kPtsThreads) Qs[i] = homog(__ldg(ctrl_s + i));
  pts_stage_knots<P, Q>(prm, s, ks);
  const float* Us = ks;
  const float* Vs = ks + L.offV;
  const int t0 = c * prm.chunk;
  const int cnt = min(prm.chunk, prm.N - t0);
  const float2* uv = prm.uv + (size_t)s * prm.N + t0;
  float* out = prm.out + ((size_t)s * prm.N + t0) * 3;
  for (int i = threadIdx.x; i < cnt; i += kPtsThreads) {
    const float2 x = __ldg(uv + i);
    const int su = s_find_span(Us, n, P, x.x);
    const int sv = s_find_span(Vs, m, Q, x.y);
    float Nu[P + 1], Nv[Q + 1];
    basis_inv<P>(Us, ks + L.offIU + (su - P) * tri(P), su, x.x, Nu);
    basis_inv<Q>(Vs, ks + L.offIV + (sv - Q) * tri(Q), sv, x.y, Nv);
    float4 Sp = f4(0.f);
#pragma unroll
    for (int r = 0; r <= P; ++r) {
      const int row = (su - P + r) * m + (sv - Q);
      float4 T = f4(0.f);
      if (prm.ctrl_smem) {
#pragma unroll
        for (int h = 0; h <= Q; ++h) T = fma4v(Nv[h], Qs[row + h], T);
      } else {
#pragma unroll
        for (int h = 0; h <= Q; ++h) T = fma4v(Nv[h], homog(__ldg(ctrl_s + row + h)), T);
      }
      Sp = fma4v(Nu[r], T, Sp);
    }
    const float rw = 1.f / Sp.w;
    out[3 * i + 0] = Sp.x * rw;
    out[3 * i + 1] = Sp.y * rw;
    out[3 * i + 2] = Sp.z * rw;
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
  size_t dq, cstart, hist, cell, sorted, cq, knots, bytes;
};
__host__ __device__ inline PtsBwdLayout pts_bwd_layout(int n, int m, int p, int q, int chunk) {
  PtsBwdLayout L;
  const int C = (n - p) * (m - q);
  size_t o = 0;
  L.dq = o;     o += (size_t)kPtsWarps * n * m * 16;                 // per-warp dQ copies
  L.cq = o;     o += (size_t)kGroups * (p + 1) * (q + 1) * 16;      // per-group cell net
  L.cstart = o; o += (size_t)(C + 1) * 4;                            // cell start offsets
  L.hist = o;   o += (size_t)kPtsWarps * (C + 1) * 4;                // per-warp counts / cursors
  L.cell = o;   o += (size_t)chunk * 2;                              // cell of point i (uint16)
  L.sorted = o; o += (size_t)chunk * 2;                              // point index by cell
  o = (o + 15) & ~(size_t)15;
  L.knots = o;  o += (size_t)pts_knots(n, m, p, q).floats * 4;
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
  const PtsBwdLayout SL = pts_bwd_layout(n, m, P, Q, prm.chunk);
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
  pts_stage_knots<P, Q>(prm, s, ks);  // ends with __syncthreads
  const float* Us = ks;
  const float* Vs = ks + KL.offV;
  const int t0 = c * prm.chunk;
  const int cnt = min(prm.chunk, prm.N - t0);
  const float2* uv = prm.uv + (size_t)s * prm.N + t0;
  const float* g = prm.gout + ((size_t)s * prm.N + t0) * 3;
  const float4* ctrl_s = prm.ctrl + (size_t)s * nm;

  // ---- pass 1: cell of every point; per-warp counts over the warp's contiguous slice
  const int per_warp = (cnt + kPtsWarps - 1) / kPtsWarps;
  const int w0 = warp * per_warp, w1 = min(cnt, w0 + per_warp);
  int* hw = hist + warp * (C + 1);
  for (int b = w0; b < w1; b += 32) {
    const int i = b + lane;
    int ce = C;  // sentinel for lanes past the slice
    if (i < w1) {
      const float2 x = __ldg(uv + i);
      const int su = s_find_span(Us, n, P, x.x);
      const int sv = s_find_span(Vs, m, Q, x.y);
      ce = (su - P) * Cv + (sv - Q);
      cell[i] = (unsigned short)ce;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, ce);
    if (ce < C && lane == __ffs(peers) - 1) hw[ce] += __popc(peers);
  }
  __syncthreads();

  // ---- pass 2: cell starts (exclusive scan over cells) and per-warp cursors
  {
    const int seg = (C + kPtsThreads - 1) / kPtsThreads;
    const int c0 = min(C, tid * seg), c1 = min(C, c0 + seg);
    int sum = 0;
    for (int ce = c0; ce < c1; ++ce)
      for (int w = 0; w < kPtsWarps; ++w) sum += hist[w * (C + 1) + ce];
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
      for (int w = 0; w < kPtsWarps; ++w) {
        const int h = hist[w * (C + 1) + ce];
        hist[w * (C + 1) + ce] = run;
        run += h;
      }
    }
    if (tid == kPtsThreads - 1) cstart[C] = cnt;
  }
  __syncthreads();

  // ---- pass 3: stable scatter (cell, warp, position in the warp's slice)
  for (int b = w0; b < w1; b += 32) {
    const int i = b + lane;
    const int ce = i < w1 ? (int)cell[i] : C;
    const unsigned peers = __match_any_sync(0xffffffffu, ce);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (ce < C) sorted[hw[ce] + rank] = (unsigned short)i;
    __syncwarp();
    if (ce < C && lane == __ffs(peers) - 1) hw[ce] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();

  // ---- pass 4: groups of kGrp lanes own cells; warp w's groups take cells w*4+g (+32 k)
  const int grp = lane / kGrp, gl = lane - grp * kGrp;
  const int G = warp * kGrpPerWarp + grp;
  float4* cqg = cq + G * NC;
  float4* dq = dqw + warp * nm;
  const int nsteps = (C - warp * kGrpPerWarp + kGroups - 1) / kGroups;
  for (int k = 0; k < nsteps; ++k) {
    const int ce = G + k * kGroups;
    const bool has = ce < C;
    const int beg = has ? cstart[ce] : 0, end = has ? cstart[ce + 1] : 0;
    const int cu = has ? ce / Cv : 0, cv = has ? ce - cu * Cv : 0;
    const int su = cu + P, sv = cv + Q;
    if (has && end > beg)  // the cell's homogeneous control points -> smem
      for (int e = gl; e < NC; e += kGrp) {
        const int r = e / (Q + 1), h = e - r * (Q + 1);
        cqg[e] = homog(__ldg(ctrl_s + (cu + r) * m + cv + h));
      }
    __syncwarp();
    float acc[NPAD];
#pragma unroll
    for (int e = 0; e < NPAD; ++e) acc[e] = 0.f;
    const float* iU = ks + KL.offIU + cu * tri(P);
    const float* iV = ks + KL.offIV + cv * tri(Q);
    for (int kk = beg + gl; kk < end; kk += kGrp) {
      const int i = sorted[kk];
      const float2 x = __ldg(uv + i);
      float Nu[P + 1], Nv[Q + 1];
      basis_inv<P>(Us, iU, su, x.x, Nu);
      basis_inv<Q>(Vs, iV, sv, x.y, Nv);
      float4 Sp = f4(0.f);
#pragma unroll
      for (int r = 0; r <= P; ++r) {
        float4 T = f4(0.f);
#pragma unroll
        for (int h = 0; h <= Q; ++h) T = fma4v(Nv[h], cqg[r * (Q + 1) + h], T);
        Sp = fma4v(Nu[r], T, Sp);
      }
      const float rw = 1.f / Sp.w;
      const float gx = __ldg(g + 3 * i) * rw, gy = __ldg(g + 3 * i + 1) * rw, gz = __ldg(g + 3 * i + 2) * rw;
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
