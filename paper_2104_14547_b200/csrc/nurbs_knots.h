// nurbs_knots.h — host-visible pieces of the knot-gradient assembly (NEXT-4, nurbs_knots.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

#define NURBS_MAXD 5

namespace nb {

struct KnotDir {             // one parametric direction
  int B, n, p, ns;           // surfaces, control count, degree, samples
  const float* knots;        // [n+p+1] or batched
  long long kstride;         // 0 = shared
  const float* samples;      // [ns], non-decreasing
  const int* tspan;          // optional span table
  const float* part;         // [B][nparts][ns][hlen] partial weights
  int nparts;
  int spans;                 // 0: units are samples, part = h [p+1] per sample;
                             // 1: units are the n-p knot spans (ns = n-p), part = span moments
                             //    X [(p+1)^2] per span (grid kernel mode 3, rows direction)
  float* contrib;            // [B][ns][2p] workspace
  int* span;                 // [B][ns] workspace
  float* xsum;               // spans with nparts > kKnotPartGroups: [B][groups][ns][(p+1)^2] workspace
};

// Span-moment partials are summed in this many fixed groups first (nurbs_knot_partsum_kernel);
// the workspace's xsum holds [B][kKnotPartGroups][ns][(p+1)^2].
constexpr int kKnotPartGroups = 8;

// dL/d(knots) of one direction into out ([B][nk] if batched, else [nk] via tmp [B][nk]).
cudaError_t launch_knot_grad(const KnotDir& d, bool batched, float* tmp, float* out, cudaStream_t st);

}  // namespace nb
