// nurbs_grid_p.cu — compiled once per row degree P (-DNB_P=0..5) so the 120 instantiations
// of nurbs_grid_kernel<P, Q, BWD, BULK> build in parallel.
#include "nurbs_grid.cuh"

#ifndef NB_P
#error "compile with -DNB_P=<row degree>"
#endif

namespace nb {
#define NB_CAT2(a, b) a##b
#define NB_CAT(a, b) NB_CAT2(a, b)
cudaError_t NB_CAT(launch_grid_p, NB_P)(const Params& prm, int mode, int q, cudaStream_t st) {
  return launch_p<NB_P>(prm, mode, q, st);
}
}  // namespace nb
