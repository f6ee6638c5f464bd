// nurbs_points.cu — paired-point plan, chunk-partial reduce, checked-mode validation and the
// launcher dispatch (NEXT-1; kernels in nurbs_points.cuh, instantiated in nurbs_points_p.cu).
// Citations: P:n = reference/PAPER.md line n; R<k> = DESIGN.md §3 reading k.
#include "nurbs_points.cuh"
#include "nurbs_points_plan.h"

namespace nb {

cudaError_t launch_points_p1(const PtsParams&, bool, int, size_t, cudaStream_t);
cudaError_t launch_points_p2(const PtsParams&, bool, int, size_t, cudaStream_t);
cudaError_t launch_points_p3(const PtsParams&, bool, int, size_t, cudaStream_t);
cudaError_t launch_points_p4(const PtsParams&, bool, int, size_t, cudaStream_t);
cudaError_t launch_points_p5(const PtsParams&, bool, int, size_t, cudaStream_t);

PtsPlan pts_plan(int B, int n, int m, int p, int q, int N) {
  PtsPlan pl{};
  const long long pts = (long long)B * N;
  const int ncell = (n - p) * (m - q);
  // forward: chunks of up to 4096 points (>= ~2 CTAs per SM when the batch is small)
  long long cf = (pts + 148LL * 2 - 1) / (148LL * 2);
  if (cf < 512) cf = 512;
  if (cf > 4096) cf = 4096;
  if (cf > N) cf = N > 0 ? N : 1;
  while (cf > 64 && pts_fwd_layout(n, m, p, q, (int)cf).bytes > kPtsSmemMax) cf = (cf + 1) / 2;
  pl.chunk_f = (int)cf;
  pl.nchunk_f = N > 0 ? (N + pl.chunk_f - 1) / pl.chunk_f : 0;
  // the homogeneous net in smem when it keeps two CTAs per SM
  pl.ctrl_smem = pts_fwd_layout(n, m, p, q, pl.chunk_f, true).bytes <= kPtsSmemMax / 2 + 8 * 1024 ? 1 : 0;
  pl.smem_f = pts_fwd_layout(n, m, p, q, pl.chunk_f, pl.ctrl_smem != 0).bytes;
  // backward: chunks of up to 8192 points (>= ~2 CTAs per SM when the batch is small), as
  // large as the smem budget allows
  long long cb = (pts + 148LL * 2 - 1) / (148LL * 2);
  if (cb < 512) cb = 512;
  if (cb > 8192) cb = 8192;
  if (cb > N) cb = N > 0 ? N : 1;
  while (cb > 64 && pts_bwd_layout(n, m, p, q, (int)cb).bytes > kPtsSmemMax) cb = (cb + 1) / 2;
  pl.chunk_b = (int)cb;
  pl.nchunk_b = N > 0 ? (N + pl.chunk_b - 1) / pl.chunk_b : 0;
  pl.ctrl_smem_b = pts_bwd_layout(n, m, p, q, pl.chunk_b, true).bytes <= kPtsSmemMax / 2 + 8 * 1024 ? 1 : 0;
  pl.smem_b = pts_bwd_layout(n, m, p, q, pl.chunk_b, pl.ctrl_smem_b != 0).bytes;
  pl.fits_f = ncell <= 65535 && pl.smem_f <= kPtsSmemMax;
  pl.fits_b = ncell <= 65535 && pl.smem_b <= kPtsSmemMax;
  pl.ws_bytes = pl.nchunk_b > 1 ? align_up((size_t)B * pl.nchunk_b * n * m * 16, 256) : 0;
  return pl;
}

// Chunk partials of each surface summed in chunk order, then the Eq.8/9 epilogue.
__global__ void nurbs_points_reduce_kernel(PtsParams prm) {
  const int nm = prm.n * prm.m;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)prm.B * nm) return;
  const long long s = idx / nm, j = idx - s * nm;
  const float4* sl = prm.slots + (size_t)s * prm.nchunk * nm + j;
  float4 d = sl[0];
  for (int c = 1; c < prm.nchunk; ++c) {
    const float4 e = sl[(size_t)c * nm];
    d = make_float4(d.x + e.x, d.y + e.y, d.z + e.z, d.w + e.w);
  }
  const float4 cp = __ldg(prm.ctrl + idx);
  prm.gctrl[idx] = make_float4(cp.w * d.x, cp.w * d.y, cp.w * d.z, fmaf(cp.x, d.x, fmaf(cp.y, d.y, fmaf(cp.z, d.z, d.w))));
}

// Checked mode: knots (non-decreasing, U[p] < U[n]), every (u, v) inside the domain, weights
// > 0 and finite control points. The smallest encoded (code, which, index) wins.
__global__ void nurbs_points_validate_kernel(PtsParams prm, int p, int q, unsigned long long* res) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nthr = (long long)gridDim.x * blockDim.x;
  auto rec = [&](int code, int which, long long i) {
    atomicMin(res, ((unsigned long long)code << 48) | ((unsigned long long)which << 40) |
                       ((unsigned long long)i & 0xffffffffffull));
  };
  const int nk = prm.ustride ? prm.B : 1;
  for (long long e = tid; e < (long long)nk * (prm.n + p); e += nthr) {  // U[k][i] <= U[k][i+1]
    const long long k = e / (prm.n + p), i = e - k * (prm.n + p);
    const float* Uk = prm.U + k * prm.ustride;
    if (!(Uk[i] <= Uk[i + 1])) rec(3, 1, e);
    if (i == 0 && !(Uk[p] < Uk[prm.n])) rec(3, 1, e);
  }
  const int nkv = prm.vstride ? prm.B : 1;
  for (long long e = tid; e < (long long)nkv * (prm.m + q); e += nthr) {
    const long long k = e / (prm.m + q), i = e - k * (prm.m + q);
    const float* Vk = prm.V + k * prm.vstride;
    if (!(Vk[i] <= Vk[i + 1])) rec(3, 2, e);
    if (i == 0 && !(Vk[q] < Vk[prm.m])) rec(3, 2, e);
  }
  for (long long e = tid; e < (long long)prm.B * prm.N; e += nthr) {
    const long long k = e / prm.N;
    const float* Uk = prm.U + k * prm.ustride;
    const float* Vk = prm.V + k * prm.vstride;
    const float2 x = prm.uv[e];
    if (!(x.x >= Uk[p] && x.x <= Uk[prm.n])) rec(4, 3, e);
    if (!(x.y >= Vk[q] && x.y <= Vk[prm.m])) rec(4, 4, e);
  }
  for (long long e = tid; e < (long long)prm.B * prm.n * prm.m; e += nthr) {
    const float4 c = prm.ctrl[e];
    if (!(c.w > 0.f) || !isfinite(c.w) || !isfinite(c.x) || !isfinite(c.y) || !isfinite(c.z)) rec(5, 0, e);
  }
}

cudaError_t launch_points(const PtsParams& prm, bool bwd, int p, int q, size_t smem, cudaStream_t st) {
  switch (p) {
    case 1: return launch_points_p1(prm, bwd, q, smem, st);
    case 2: return launch_points_p2(prm, bwd, q, smem, st);
    case 3: return launch_points_p3(prm, bwd, q, smem, st);
    case 4: return launch_points_p4(prm, bwd, q, smem, st);
    case 5: return launch_points_p5(prm, bwd, q, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_points_reduce(const PtsParams& prm, cudaStream_t st) {
  const long long total = (long long)prm.B * prm.n * prm.m;
  nurbs_points_reduce_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(prm);
  return cudaGetLastError();
}

cudaError_t launch_points_validate(const PtsParams& prm, int p, int q, unsigned long long* res, cudaStream_t st) {
  nurbs_points_validate_kernel<<<296, 256, 0, st>>>(prm, p, q, res);
  return cudaGetLastError();
}

}  // namespace nb
