// nurbs_points_p.cu — instantiations of the paired-point kernels (nurbs_points.cuh) for one
// u degree p = NB_P and every v degree q = 1..NURBS_MAX_DEGREE (one TU per p, built in parallel).
#include "nurbs_points.cuh"
#include "nurbs_points_plan.h"

#ifndef NB_P
#error "compile with -DNB_P=<p>"
#endif

namespace nb {

// The dynamic shared-memory opt-in (the plan's maximum, kPtsSmemMax) once per device and
// kernel, not on every launch (a benign race: setting it twice is harmless).
template <typename K>
static cudaError_t smem_optin(K k, bool (&done)[64]) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < 64 && done[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPtsSmemMax);
  if (e == cudaSuccess && dev >= 0 && dev < 64) done[dev] = true;
  return e;
}

template <int Q>
static cudaError_t launch_q(const PtsParams& prm, bool bwd, size_t smem, cudaStream_t st) {
  const unsigned grid = (unsigned)((long long)prm.B * prm.nchunk);
  if (bwd) {
    static bool done[64] = {};
    auto k = nurbs_points_bwd_kernel<NB_P, Q>;
    cudaError_t e = smem_optin(k, done);
    if (e != cudaSuccess) return e;
    k<<<grid, kPtsThreads, smem, st>>>(prm);
  } else {
    static bool done[64] = {};
    auto k = nurbs_points_fwd_kernel<NB_P, Q>;
    cudaError_t e = smem_optin(k, done);
    if (e != cudaSuccess) return e;
    k<<<grid, kPtsThreads, smem, st>>>(prm);
  }
  return cudaGetLastError();
}

#define NB_CAT2(a, b) a##b
#define NB_CAT(a, b) NB_CAT2(a, b)
cudaError_t NB_CAT(launch_points_p, NB_P)(const PtsParams& prm, bool bwd, int q, size_t smem, cudaStream_t st) {
  switch (q) {
    case 1: return launch_q<1>(prm, bwd, smem, st);
    case 2: return launch_q<2>(prm, bwd, smem, st);
    case 3: return launch_q<3>(prm, bwd, smem, st);
    case 4: return launch_q<4>(prm, bwd, smem, st);
    case 5: return launch_q<5>(prm, bwd, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace nb
