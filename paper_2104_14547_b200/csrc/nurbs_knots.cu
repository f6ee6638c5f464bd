// nurbs_knots.cu — true knot gradients (NEXT-4 of DESIGN.md §8e). The paper defines the knot
// gradients as zero (§3.2.2); this extension differentiates the basis with respect to
// the knots. For one direction (rows = u shown; columns = v alike):
//   dL/dU_k = sum_a sum_r dN_r(u_a)/dU_k * h_r(a),   h_r(a) = sum_b G_ab . T_r(a, b)
// where G = (g/W, -(g.S)/W) is the backward's homogeneous upstream and T_r the F1 row; for
// the v direction h_h(b) = sum_i Q[i][sv(b)-q+h] . H[i][b] with H = N_u^T G (B1's output),
// written per (surface, row block, column). For the u direction the grid kernel writes span
// moments instead (nurbs_knot_spans_kernel below): on knot span s the derivative of each
// non-zero basis function is a degree-p polynomial, i.e. a combination of the span's p+1
// basis functions, dN_r/dU_k = sum_r' C[r][k][r'] N_r', so
//   sum_{a in s} dN_r(u_a)/dU_k h_r(a) = sum_r' C[r][k][r'] X[r][r'],
//   X[r][r'] = sum_{a in s} N_r'(u_a) h_r(a) = sum_b T_r(b) . (sum_{a in s} N_r'(u_a) G_ab).
// C comes from a (p+1) x (p+1) collocation solve on the span (fp64).
// dN_r/dU_k is forward-mode differentiation of the A2.2 triangle along each of the
// 2p knots U[s-p+1 .. s+p] it reads. Every sum runs in a fixed order (deterministic).
// Citations: P:n = reference/PAPER.md line n; R<k> = DESIGN.md §3 reading k.
#include <cuda_runtime.h>

#include "nurbs_device.cuh"
#include "nurbs_knots.h"

namespace nb {

// sum_r dN_r(u)/dU[s-p+1+t] * h[r] for one t in [0, 2p): the A2.2 triangle with dual numbers
// along knot t. kn = U[s-p+1 .. s+p].
template <int P>
__device__ __forceinline__ float d_basis_dknot_one(const float (&kn)[2 * P], float u, const float (&h)[P + 1],
                                                   int t) {
  float N[P + 1], D[P + 1], left[P + 1], right[P + 1], dl[P + 1], dr[P + 1];
  N[0] = 1.f;
  D[0] = 0.f;
#pragma unroll
  for (int j = 1; j <= P; ++j) {
    left[j] = u - kn[P - j];            // u - U[s+1-j]
    dl[j] = (P - j == t) ? -1.f : 0.f;
    right[j] = kn[P - 1 + j] - u;       // U[s+j] - u
    dr[j] = (P - 1 + j == t) ? 1.f : 0.f;
    float saved = 0.f, dsaved = 0.f;
#pragma unroll
    for (int r = 0; r < j; ++r) {
      const float den = right[r + 1] + left[j - r];
      const float dden = dr[r + 1] + dl[j - r];
      const float temp = N[r] / den;
      const float dtemp = (D[r] - temp * dden) / den;
      const float nN = fmaf(right[r + 1], temp, saved);
      const float nD = dsaved + dr[r + 1] * temp + right[r + 1] * dtemp;
      saved = left[j - r] * temp;
      dsaved = dl[j - r] * temp + left[j - r] * dtemp;
      N[r] = nN;
      D[r] = nD;
    }
    N[j] = saved;
    D[j] = dsaved;
  }
  float acc = 0.f;
#pragma unroll
  for (int r = 0; r <= P; ++r) acc = fmaf(D[r], h[r], acc);
  return acc;
}

// c[t] = sum_r dN_r(u)/dU[s-p+1+t] * h[r], t = 0..2p-1 (A2.2 with dual numbers, one pass per knot).
template <int P>
__device__ __forceinline__ void d_basis_dknots(const float* __restrict__ U, int s, float u, const float (&h)[P + 1],
                                               float (&c)[2 * P]) {
  float kn[2 * P];  // U[s-p+1 .. s+p]
#pragma unroll
  for (int t = 0; t < 2 * P; ++t) kn[t] = __ldg(U + s - P + 1 + t);
#pragma unroll
  for (int t = 0; t < 2 * P; ++t) c[t] = d_basis_dknot_one<P>(kn, u, h, t);
}

// Single-part weights (nparts == 1, e.g. the batch-summed weights of shared knots): one thread
// per (surface, sample, knot t) instead of per sample — the 2p dual passes run in parallel
// (the per-sample pass chain is what bounds this kernel's latency). Same arithmetic per t.
template <int P>
__global__ void nurbs_knot_rows_t_kernel(KnotDir d) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)d.B * d.ns * (2 * P)) return;
  const long long sa = idx / (2 * P);
  const int t = (int)(idx - sa * (2 * P));
  const int s = (int)(sa / d.ns), a = (int)(sa - (long long)s * d.ns);
  float h[P + 1];
  const float* src = d.part + ((size_t)s * d.ns + a) * (P + 1);
#pragma unroll
  for (int r = 0; r <= P; ++r) h[r] = __ldg(src + r);
  const float* Uk = d.knots + (long long)s * d.kstride;
  const float ua = __ldg(d.samples + a);
  int sp = d.tspan ? __ldg(d.tspan + a) : d_find_span(Uk, d.n, P, ua);
  sp = min(max(sp, P), d.n - 1);
  float kn[2 * P];
#pragma unroll
  for (int k = 0; k < 2 * P; ++k) kn[k] = __ldg(Uk + sp - P + 1 + k);
  d.contrib[(size_t)sa * (2 * P) + t] = d_basis_dknot_one<P>(kn, ua, h, t);
  if (t == 0) d.span[sa] = sp;
}

// Per (surface, sample): h = sum over the nparts partials (ascending), then the 2p knot
// contributions and the span.
template <int P>
__global__ void nurbs_knot_rows_kernel(KnotDir d) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)d.B * d.ns) return;
  const int s = (int)(idx / d.ns), a = (int)(idx - (long long)s * d.ns);
  float h[P + 1];
#pragma unroll
  for (int r = 0; r <= P; ++r) h[r] = 0.f;
  const size_t pstride = (size_t)d.ns * (P + 1);  // between consecutive parts
  const float* src = d.part + ((size_t)s * d.nparts * d.ns + a) * (P + 1);
  int pc = 0;
  for (; pc + 4 <= d.nparts; pc += 4) {  // four parts' loads in flight, added in part order
    float x[4][P + 1];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r <= P; ++r) x[j][r] = __ldg(src + (size_t)(pc + j) * pstride + r);
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int r = 0; r <= P; ++r) h[r] += x[j][r];
  }
  for (; pc < d.nparts; ++pc)
#pragma unroll
    for (int r = 0; r <= P; ++r) h[r] += __ldg(src + (size_t)pc * pstride + r);
  const float* Uk = d.knots + (long long)s * d.kstride;
  const float ua = __ldg(d.samples + a);
  int sp = d.tspan ? __ldg(d.tspan + a) : d_find_span(Uk, d.n, P, ua);
  sp = min(max(sp, P), d.n - 1);
  float c[2 * P];
  d_basis_dknots<P>(Uk, sp, ua, h, c);
#pragma unroll
  for (int t = 0; t < 2 * P; ++t) d.contrib[(size_t)idx * (2 * P) + t] = c[t];
  d.span[idx] = sp;
}

// out[s][g][e] = sum over the partials c of group g (parts [g*np/G, (g+1)*np/G), ascending)
// of part[s][c][e]: the span moments of the column blocks summed in G fixed groups, in
// parallel, before the per-(span, knot) threads add the G group sums (ascending g).
__global__ void nurbs_knot_partsum_kernel(const float* __restrict__ part, long long B, int nparts, int E, int G,
                                          float* __restrict__ out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * G * E) return;
  const long long sg = idx / E;
  const int e = (int)(idx - sg * E);
  const long long s = sg / G;
  const int g = (int)(sg - s * G);
  const int c0 = (int)((long long)nparts * g / G), c1 = (int)((long long)nparts * (g + 1) / G);
  const float* src = part + (size_t)s * nparts * E + e;
  float acc = 0.f;
  int c = c0;
  for (; c + 4 <= c1; c += 4) {  // four loads in flight, added in part order
    const float a0 = __ldg(src + (size_t)c * E), a1 = __ldg(src + (size_t)(c + 1) * E);
    const float a2 = __ldg(src + (size_t)(c + 2) * E), a3 = __ldg(src + (size_t)(c + 3) * E);
    acc += a0; acc += a1; acc += a2; acc += a3;
  }
  for (; c < c1; ++c) acc += __ldg(src + (size_t)c * E);
  out[idx] = acc;
}

// Rows direction from span moments (d.spans == 1, unit k = knot span s = p + k): one thread per
// (surface, span, knot t). X[r][r'] = sum over the nparts partials (ascending). With p+1
// Chebyshev points u_m of the span, A[m][r'] = N_r'(u_m) and Z A = X (Z: r x m, fp64 LU with
// partial pivoting of A^T), the span's contribution to knot U[s-p+1+t] is
//   sum_{r,r'} C[r][t][r'] X[r][r'] = sum_m sum_r dN_r(u_m)/dU_t Z[r][m]
// (C[r][t][.] = A^-1 applied to dN_r/dU_t at the points), i.e. p+1 dual-number A2.2 passes.
template <int P>
__global__ void nurbs_knot_spans_kernel(KnotDir d) {
  constexpr int NX = (P + 1) * (P + 1);
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)d.B * d.ns * (2 * P)) return;
  const long long sk = idx / (2 * P);
  const int t = (int)(idx - sk * (2 * P));
  const int sf = (int)(sk / d.ns), k = (int)(sk - (long long)sf * d.ns);
  const int sp = P + k;
  if (t == 0) d.span[sk] = sp;
  const float* Uk = d.knots + (long long)sf * d.kstride;
  const float ua = __ldg(Uk + sp), ub = __ldg(Uk + sp + 1);
  float res = 0.f;
  if (ub > ua) {  // empty spans hold no samples: no contribution
    float X[NX];
#pragma unroll
    for (int v = 0; v < NX; ++v) X[v] = 0.f;
    const float* src = d.part + ((size_t)sf * d.nparts * d.ns + k) * NX;
    for (int c = 0; c < d.nparts; ++c)
#pragma unroll
      for (int v = 0; v < NX; ++v) X[v] += __ldg(src + (size_t)c * d.ns * NX + v);
    float um[P + 1];
    double At[P + 1][P + 1];  // At[r'][m] = N_r'(u_m)
#pragma unroll
    for (int m = 0; m <= P; ++m) {
      const float c = 0.5f * (1.f - cospif((2.f * m + 1.f) / (2.f * (P + 1))));
      um[m] = fmaf(ub - ua, c, ua);
      float N[P + 1];
      d_basis<P>(Uk, sp, um[m], P, N);
#pragma unroll
      for (int r = 0; r <= P; ++r) At[r][m] = (double)N[r];
    }
    // Z A = X  <=>  A^T Z^T = X^T: LU of At (partial pivoting), then P+1 right-hand sides
    int piv[P + 1];
#pragma unroll
    for (int i = 0; i <= P; ++i) piv[i] = i;
#pragma unroll
    for (int c = 0; c <= P; ++c) {  // (fully unrolled: At stays in registers; swaps by selects)
      int pr = c;
      double best = fabs(At[c][c]);
#pragma unroll
      for (int i = c + 1; i <= P; ++i)
        if (fabs(At[i][c]) > best) { best = fabs(At[i][c]); pr = i; }
#pragma unroll
      for (int i = c + 1; i <= P; ++i) {
        if (i == pr) {
#pragma unroll
          for (int j = 0; j <= P; ++j) { const double tmp = At[c][j]; At[c][j] = At[i][j]; At[i][j] = tmp; }
          const int ti = piv[c]; piv[c] = piv[i]; piv[i] = ti;
        }
      }
      const double rinv = 1.0 / At[c][c];
#pragma unroll
      for (int i = c + 1; i <= P; ++i) {
        const double f = At[i][c] * rinv;
        At[i][c] = f;
#pragma unroll
        for (int j = c + 1; j <= P; ++j) At[i][j] -= f * At[c][j];
      }
    }
    float kn[2 * P];
#pragma unroll
    for (int q = 0; q < 2 * P; ++q) kn[q] = __ldg(Uk + sp - P + 1 + q);
    float Z[P + 1][P + 1];  // Z[r][m]
#pragma unroll
    for (int r = 0; r <= P; ++r) {  // solve At z = (X[r][0..P]) with the row permutation piv
      double y[P + 1];
#pragma unroll
      for (int i = 0; i <= P; ++i) {
        double xv = 0.0;
#pragma unroll
        for (int q = 0; q <= P; ++q)
          if (piv[i] == q) xv = (double)X[r * (P + 1) + q];
#pragma unroll
        for (int j = 0; j < i; ++j) xv -= At[i][j] * y[j];
        y[i] = xv;
      }
#pragma unroll
      for (int i = P; i >= 0; --i) {
        double a = y[i];
#pragma unroll
        for (int j = i + 1; j <= P; ++j) a -= At[i][j] * y[j];
        y[i] = a / At[i][i];
      }
#pragma unroll
      for (int m = 0; m <= P; ++m) Z[r][m] = (float)y[m];
    }
#pragma unroll
    for (int m = 0; m <= P; ++m) {
      float h[P + 1];
#pragma unroll
      for (int r = 0; r <= P; ++r) h[r] = Z[r][m];
      res += d_basis_dknot_one<P>(kn, um[m], h, t);
    }
  }
  d.contrib[(size_t)sk * (2 * P) + t] = res;
}

// Per (surface, knot k): sum over the samples whose span window holds k (spans are
// non-decreasing in the sorted samples, so the window is a contiguous range). One warp per
// (surface, knot): lane l sums samples lo+l, lo+l+32, ... in ascending order, then a fixed
// xor butterfly combines the lanes (deterministic).
__global__ void nurbs_knot_gather_kernel(KnotDir d, float* out /* [B][nk] */) {
  const int nk = d.n + d.p + 1;
  const long long idx = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (idx >= (long long)d.B * nk) return;  // warp-uniform
  const int s = (int)(idx / nk), k = (int)(idx - (long long)s * nk);
  const int p = d.p;
  const int* sp = d.span + (size_t)s * d.ns;
  // rows with span in [k - p, k + p - 1] contribute to knot k (t = k - (span - p + 1));
  // lo = the first of them. Units that are the knot spans themselves (span p + a at a) index
  // it directly; samples: a warp-wide search, 32 probes per round (one load latency per
  // 32x narrowing instead of one per halving)
  const int key = k - p;
  int lo = 0, hi = d.ns;
  if (d.spans) {
    lo = hi = min(max(key - p, 0), d.ns);
  }
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) / 32;
    const bool lt = sp[min(lo + step * lane, hi - 1)] < key;  // non-decreasing probes: a prefix
    const int c = __popc(__ballot_sync(0xffffffffu, lt));
    const int nlo = c == 0 ? lo : min(hi, lo + step * (c - 1) + 1);
    hi = c == 32 ? hi : min(hi, lo + step * c);
    lo = nlo;
  }
  if (hi > lo) {
    const bool lt = lo + lane < hi && sp[lo + lane] < key;
    lo += __popc(__ballot_sync(0xffffffffu, lt));
  }
  float acc = 0.f;
  for (int a = lo + lane; a < d.ns; a += 32) {
    const int spa = sp[a];
    if (spa > k + p - 1) break;
    const int t = k - (spa - p + 1);
    if (t >= 0 && t < 2 * p) acc += d.contrib[((size_t)s * d.ns + a) * (2 * p) + t];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[idx] = acc;
}

// Shared knots: out[k] = sum over surfaces (fixed partition + fixed tree) of per[s][k].
__global__ void __launch_bounds__(256) nurbs_knot_sum_kernel(const float* per, int B, int nk, float* out) {
  __shared__ float red[256];
  const int k = blockIdx.x;
  const int per_t = (B + 255) / 256;
  const int s0 = threadIdx.x * per_t, s1 = min(B, s0 + per_t);
  float a = 0.f;
  for (int s = s0; s < s1; ++s) a += per[(size_t)s * nk + k];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[k] = red[0];
}

// Shared knots: the knot derivative of a sample does not depend on the surface, so the
// per-surface weights h can be summed over the batch first (linearity):
//   dL/dU_k = sum_a sum_r dN_r(u_a)/dU_k * (sum_s sum_c part[s][c][a][r]).
// Two fixed-order levels: gpart[g][e] = sum over surfaces [g*B/G, (g+1)*B/G) (ascending) and
// parts c (ascending); hsum[e] = a fixed tree over the G groups. The per-sample kernels then
// run once, on one "surface" whose single part is hsum.
__global__ void nurbs_knot_hgroup_kernel(const float* __restrict__ part, int B, int nparts, int E, int G,
                                         float* __restrict__ gpart) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)E * G) return;
  const int g = (int)(idx / E), e = (int)(idx - (long long)g * E);
  const int s0 = (int)((long long)B * g / G), s1 = (int)((long long)B * (g + 1) / G);
  const int n = (s1 - s0) * nparts;  // the group's (surface, part) rows, contiguous in part[]
  const float* src = part + (size_t)s0 * nparts * E + e;
  float acc = 0.f;
  int i = 0;
  for (; i + 4 <= n; i += 4) {  // four independent loads in flight, added in order
    const float a0 = __ldg(src + (size_t)i * E), a1 = __ldg(src + (size_t)(i + 1) * E);
    const float a2 = __ldg(src + (size_t)(i + 2) * E), a3 = __ldg(src + (size_t)(i + 3) * E);
    acc += a0; acc += a1; acc += a2; acc += a3;
  }
  for (; i < n; ++i) acc += __ldg(src + (size_t)i * E);
  gpart[(size_t)g * E + e] = acc;
}

// hsum[e] = sum over g of gpart[g][e]: one block per element, thread t takes g = t, t+256, ...
// (ascending), then a fixed shared-memory tree.
__global__ void __launch_bounds__(256) nurbs_knot_htree_kernel(const float* __restrict__ gpart, int E, int G,
                                                               float* __restrict__ hsum) {
  __shared__ float red[256];
  const int e = blockIdx.x;
  float a = 0.f;
  for (int g = threadIdx.x; g < G; g += 256) a += gpart[(size_t)g * E + e];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) hsum[e] = red[0];
}

static cudaError_t launch_rows(const KnotDir& d, cudaStream_t st) {
  const long long rows = (long long)d.B * d.ns;
  if (d.spans) {
    const unsigned nbt = (unsigned)((rows * 2 * d.p + 127) / 128);
    switch (d.p) {
      case 1: nurbs_knot_spans_kernel<1><<<nbt, 128, 0, st>>>(d); break;
      case 2: nurbs_knot_spans_kernel<2><<<nbt, 128, 0, st>>>(d); break;
      case 3: nurbs_knot_spans_kernel<3><<<nbt, 128, 0, st>>>(d); break;
      case 4: nurbs_knot_spans_kernel<4><<<nbt, 128, 0, st>>>(d); break;
      case 5: nurbs_knot_spans_kernel<5><<<nbt, 128, 0, st>>>(d); break;
      default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
  }
  if (d.nparts == 1) {
    const unsigned nbt = (unsigned)((rows * 2 * d.p + 127) / 128);
    switch (d.p) {
      case 1: nurbs_knot_rows_t_kernel<1><<<nbt, 128, 0, st>>>(d); break;
      case 2: nurbs_knot_rows_t_kernel<2><<<nbt, 128, 0, st>>>(d); break;
      case 3: nurbs_knot_rows_t_kernel<3><<<nbt, 128, 0, st>>>(d); break;
      case 4: nurbs_knot_rows_t_kernel<4><<<nbt, 128, 0, st>>>(d); break;
      case 5: nurbs_knot_rows_t_kernel<5><<<nbt, 128, 0, st>>>(d); break;
      default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
  }
  const unsigned nbk = (unsigned)((rows + 127) / 128);
  switch (d.p) {
    case 1: nurbs_knot_rows_kernel<1><<<nbk, 128, 0, st>>>(d); break;
    case 2: nurbs_knot_rows_kernel<2><<<nbk, 128, 0, st>>>(d); break;
    case 3: nurbs_knot_rows_kernel<3><<<nbk, 128, 0, st>>>(d); break;
    case 4: nurbs_knot_rows_kernel<4><<<nbk, 128, 0, st>>>(d); break;
    case 5: nurbs_knot_rows_kernel<5><<<nbk, 128, 0, st>>>(d); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_knot_grad(const KnotDir& d, bool batched, float* tmp, float* out, cudaStream_t st) {
  if (d.B == 0) return cudaSuccess;
  if (!batched && d.B >= 16 && d.ns > 0) {
    // workspace (d.contrib holds B*ns*2p floats): [G][ns][p+1] group sums, [ns][p+1] batch
    // sum, then the one surface's [ns][2p] contributions
    const int E = d.ns * (d.spans ? (d.p + 1) * (d.p + 1) : d.p + 1);
    const long long cap = (long long)d.B * d.ns * 2 * d.p;
    long long G = (cap - (long long)d.ns * 2 * d.p - E) / E;
    G = G > 256 ? 256 : G;
    G = G > d.B ? d.B : G;
    if (G >= 1) {
      float* gpart = d.contrib;
      float* hsum = gpart + (size_t)G * E;
      const long long th = (long long)E * G;
      nurbs_knot_hgroup_kernel<<<(unsigned)((th + 255) / 256), 256, 0, st>>>(d.part, d.B, d.nparts, E, (int)G, gpart);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      nurbs_knot_htree_kernel<<<(unsigned)E, 256, 0, st>>>(gpart, E, (int)G, hsum);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      KnotDir d1 = d;
      d1.B = 1;
      d1.kstride = 0;
      d1.part = hsum;
      d1.nparts = 1;
      d1.contrib = hsum + E;
      if ((e = launch_rows(d1, st)) != cudaSuccess) return e;
      const int nk = d.n + d.p + 1;
      nurbs_knot_gather_kernel<<<(unsigned)((nk * 32LL + 127) / 128), 128, 0, st>>>(d1, out);
      return cudaGetLastError();
    }
  }
  const int nk = d.n + d.p + 1;
  if (d.ns > 0) {
    KnotDir dr = d;
    if (d.spans && d.nparts > kKnotPartGroups) {  // partials -> kKnotPartGroups group sums (d.xsum)
      const int E = d.ns * (d.p + 1) * (d.p + 1);
      const long long th = (long long)d.B * kKnotPartGroups * E;
      nurbs_knot_partsum_kernel<<<(unsigned)((th + 255) / 256), 256, 0, st>>>(d.part, d.B, d.nparts, E,
                                                                              kKnotPartGroups, d.xsum);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      dr.part = d.xsum;
      dr.nparts = kKnotPartGroups;
    }
    cudaError_t e = launch_rows(dr, st);
    if (e != cudaSuccess) return e;
  }
  float* dst = batched ? out : tmp;
  const long long items = (long long)d.B * nk;
  if (d.ns > 0) {
    nurbs_knot_gather_kernel<<<(unsigned)((items * 32 + 127) / 128), 128, 0, st>>>(d, dst);
  } else {
    cudaError_t e = cudaMemsetAsync(dst, 0, sizeof(float) * (size_t)items, st);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || batched) return e;
  nurbs_knot_sum_kernel<<<nk, 256, 0, st>>>(tmp, d.B, nk, out);
  return cudaGetLastError();
}

}  // namespace nb
