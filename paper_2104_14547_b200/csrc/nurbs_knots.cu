// nurbs_knots.cu — true knot gradients (NEXT-4 of DESIGN.md §8e). The paper defines the knot
// gradients as zero (§3.2.2); this extension differentiates the basis with respect to
// the knots. For one direction (rows = u shown; columns = v alike):
//   dL/dU_k = sum_a sum_r dN_r(u_a)/dU_k * h_r(a),   h_r(a) = sum_b G_ab . T_r(a, b)
// where G = (g/W, -(g.S)/W) is the backward's homogeneous upstream and T_r the F1 row
// (the grid kernel's mode 3 writes h per (surface, column block, row), nurbs_grid.cuh); for
// the v direction h_h(b) = sum_i Q[i][sv(b)-q+h] . H[i][b] with H = N_u^T G (B1's output).
// dN_r/dU_k is forward-mode differentiation of the A2.2 triangle along each of the
// 2p knots U[s-p+1 .. s+p] it reads. Every sum runs in a fixed order (deterministic).
// Citations: P:n = reference/PAPER.md line n; R<k> = DESIGN.md §3 reading k.
#include <cuda_runtime.h>

#include "nurbs_device.cuh"
#include "nurbs_knots.h"

namespace nb {

// c[t] = sum_r dN_r(u)/dU[s-p+1+t] * h[r], t = 0..2p-1 (A2.2 with dual numbers, one pass per knot).
template <int P>
__device__ __forceinline__ void d_basis_dknots(const float* __restrict__ U, int s, float u, const float (&h)[P + 1],
                                               float (&c)[2 * P]) {
  float kn[2 * P];  // U[s-p+1 .. s+p]
#pragma unroll
  for (int t = 0; t < 2 * P; ++t) kn[t] = __ldg(U + s - P + 1 + t);
#pragma unroll
  for (int t = 0; t < 2 * P; ++t) {
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
    c[t] = acc;
  }
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
  for (int c = 0; c < d.nparts; ++c) {
    const float* src = d.part + (((size_t)s * d.nparts + c) * d.ns + a) * (P + 1);
#pragma unroll
    for (int r = 0; r <= P; ++r) h[r] += src[r];
  }
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

// Per (surface, knot k): sum over the samples whose span window holds k (ascending samples;
// spans are non-decreasing in the sorted samples, so the window is a contiguous range).
__global__ void nurbs_knot_gather_kernel(KnotDir d, float* out /* [B][nk] */) {
  const int nk = d.n + d.p + 1;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)d.B * nk) return;
  const int s = (int)(idx / nk), k = (int)(idx - (long long)s * nk);
  const int p = d.p;
  const int* sp = d.span + (size_t)s * d.ns;
  // rows with span in [k - p, k + p - 1] contribute to knot k (t = k - (span - p + 1))
  int lo = 0, hi = d.ns;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (sp[mid] < k - p) lo = mid + 1; else hi = mid;
  }
  float acc = 0.f;
  for (int a = lo; a < d.ns && sp[a] <= k + p - 1; ++a) {
    const int t = k - (sp[a] - p + 1);
    if (t >= 0 && t < 2 * p) acc += d.contrib[((size_t)s * d.ns + a) * (2 * p) + t];
  }
  out[idx] = acc;
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

cudaError_t launch_knot_grad(const KnotDir& d, bool batched, float* tmp, float* out, cudaStream_t st) {
  if (d.B == 0) return cudaSuccess;
  const int nk = d.n + d.p + 1;
  const long long rows = (long long)d.B * d.ns;
  if (d.ns > 0) {
    const unsigned nbk = (unsigned)((rows + 127) / 128);
    switch (d.p) {
      case 1: nurbs_knot_rows_kernel<1><<<nbk, 128, 0, st>>>(d); break;
      case 2: nurbs_knot_rows_kernel<2><<<nbk, 128, 0, st>>>(d); break;
      case 3: nurbs_knot_rows_kernel<3><<<nbk, 128, 0, st>>>(d); break;
      case 4: nurbs_knot_rows_kernel<4><<<nbk, 128, 0, st>>>(d); break;
      case 5: nurbs_knot_rows_kernel<5><<<nbk, 128, 0, st>>>(d); break;
      default: return cudaErrorInvalidValue;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  float* dst = batched ? out : tmp;
  const long long items = (long long)d.B * nk;
  if (d.ns > 0) {
    nurbs_knot_gather_kernel<<<(unsigned)((items + 127) / 128), 128, 0, st>>>(d, dst);
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
