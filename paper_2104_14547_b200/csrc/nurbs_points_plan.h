// nurbs_points_plan.h — host-visible launch plan of the paired-point path (NEXT-1). The plan
// (chunk sizes, hence the summation order) is a pure function of the shape.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace nb {

struct PtsParams;
constexpr size_t kPtsSmemMax = 200 * 1024;

struct PtsPlan {
  int chunk_f, nchunk_f;   // forward: points per CTA, CTAs per surface
  int chunk_b, nchunk_b;   // backward
  size_t smem_f, smem_b;   // dynamic smem bytes
  int ctrl_smem;           // forward stages the homogeneous net in smem
  int ctrl_smem_b;         // backward stages the homogeneous net in smem
  bool fits_f, fits_b;     // smem within kPtsSmemMax (bwd also: cells <= 65535)
  size_t ws_bytes;         // backward chunk partials (nchunk_b > 1)
};

PtsPlan pts_plan(int B, int n, int m, int p, int q, int N);
cudaError_t launch_points(const PtsParams& prm, bool bwd, int p, int q, size_t smem, cudaStream_t st);
cudaError_t launch_points_reduce(const PtsParams& prm, cudaStream_t st);
cudaError_t launch_points_validate(const PtsParams& prm, int p, int q, unsigned long long* res, cudaStream_t st);

}  // namespace nb
