// nurbs_derivs.cu — NEXT-3: parametric derivatives S_u, S_v (Eq.7 P:196-209 and its v
// analogue) and unit normals (the offsetting input of §4.3) on the grid.
//
// Same decomposition as the grid kernel (CTA = surface x row block x 128-column block, one
// thread per sample column walking the rows with a rolling window of P+1 control rows), but
// the window carries two F1 products per control row: T = Q·Nv^T and T_v = Q·N'_v^T. Per
// point:  S' = sum Nu T,  S'_u = sum N'_u T,  S'_v = sum Nu T_v  (packed FFMA2), then the
// quotient rule S_u = (S'_u,xyz - S S'_u,w) / W (Eq.7) and n = (S_u x S_v)/|S_u x S_v|.
// Spans and bases (and their derivatives) are computed in-kernel; stores are direct.
#include <cuda_runtime.h>
#include <cstdint>

#include "nurbs_device.cuh"

#ifndef NB_DERIV_RU
#define NB_DERIV_RU 8
#endif

namespace nb {

// N and N' of the p+1 non-zero functions at span s: N' from the degree p-1 functions
// (differentiated Eq.4): N'_i = p N_{i,p-1}/(U[i+p]-U[i]) - p N_{i+1,p-1}/(U[i+p+1]-U[i+1]).
template <int MAXD>
__device__ __forceinline__ void d_basis_ders(const float* __restrict__ U, int s, float u, int p, float* N,
                                             float* dN) {
  float Nm[MAXD + 1];
  if (p > 0) d_basis<MAXD>(U, s, u, p - 1, Nm);
  d_basis<MAXD>(U, s, u, p, N);
#pragma unroll
  for (int r = 0; r <= MAXD; ++r) {
    float d = 0.f;
    if (r <= p && p > 0) {
      const int i = s - p + r;
      float a = 0.f, b = 0.f;
      if (r >= 1) {
        const float den = __ldg(U + i + p) - __ldg(U + i);
        a = den != 0.f ? Nm[r >= 1 ? r - 1 : 0] / den : 0.f;
      }
      if (r <= p - 1) {
        const float den = __ldg(U + i + p + 1) - __ldg(U + i + 1);
        b = den != 0.f ? Nm[r] / den : 0.f;
      }
      d = (float)p * (a - b);
    }
    dN[r] = d;
  }
}

template <int P, int Q>
__global__ void __launch_bounds__(kThreads) nurbs_derivs_kernel(const Params prm, float* out_u, float* out_v,
                                                               float* normals) {
  constexpr int NP = (P + 1) <= 4 ? 4 : 8;
  __shared__ int su_s[kRowChunk];
  __shared__ __align__(16) float Nu_s[kRowChunk * NP];
  __shared__ __align__(16) float Nud_s[kRowChunk * NP];
  const int tid = threadIdx.x;
  const Dir& R = prm.r;
  const Dir& C = prm.c;
  const int m = C.n;
  int bid = blockIdx.x;
  const int cb = bid % prm.NCB;
  bid /= prm.NCB;
  const int rb = bid % prm.NRB;
  const int s = bid / prm.NRB;
  const int B0 = cb * kCB;
  const int cols = min(kCB, C.ns - B0);
  const int S0 = P + rb * prm.K;
  const int S1 = min(S0 + prm.K, R.n);
  const int band_lo = S0 - P;
  const float* Uk = R.knots + (long long)s * R.kstride;
  const float* Vk = C.knots + (long long)s * C.kstride;
  const float4* __restrict__ ctrl_s = prm.ctrl + (size_t)s * R.n * m;

  int a_lo = 0, a_hi = R.ns;
  if (prm.NRB > 1) {
    int s_end = R.n - 1;
    while (s_end > P && __ldg(Uk + s_end) == __ldg(Uk + s_end + 1)) --s_end;
    auto ge = [&](int S) {
      return [&, S](int a) -> bool {
        if (S > s_end) return false;
        return __ldg(R.s + a) >= __ldg(Uk + S);
      };
    };
    if (rb > 0) a_lo = cta_first_true(R.ns, ge(S0));
    if (rb < prm.NRB - 1) a_hi = cta_first_true(R.ns, ge(S1));
  }
  const int nwalk = max(0, a_hi - a_lo);

  const bool valid = tid < cols;
  const int b = B0 + (valid ? tid : cols - 1);
  const float vb = __ldg(C.s + b);
  const int sv = min(max(d_find_span(Vk, m, Q, vb), Q), m - 1);
  float nv[kMaxQ + 1], nvd[kMaxQ + 1];
  d_basis_ders<kMaxQ>(Vk, sv, vb, Q, nv, nvd);

  // T(i) and T_v(i) of this column (F1 with N_v and N'_v)
  auto Trow2 = [&](int i, float4& t, float4& tv) {
    const float4* src = ctrl_s + (size_t)i * m + (sv - Q);
    t = f4(0.f);
    tv = f4(0.f);
#pragma unroll
    for (int h = 0; h <= Q; ++h) {
      const float4 c = homog(__ldg(src + h));
      t = fma4v(nv[h], c, t);
      tv = fma4v(nvd[h], c, tv);
    }
  };
  float4 tw[P + 1], tvw[P + 1];
  int lo = band_lo;
#pragma unroll
  for (int k = 0; k <= P; ++k) Trow2(band_lo + k, tw[k], tvw[k]);

  const size_t grow = (size_t)C.ns * 3;
  const size_t o0 = (((size_t)s * R.ns + a_lo) * C.ns + b) * 3;
  for (int c0 = 0; c0 < nwalk; c0 += kRowChunk) {
    const int cn = min(kRowChunk, nwalk - c0);
    __syncthreads();
    if (tid < cn) {
      const int a = a_lo + c0 + tid;
      const float ua = __ldg(R.s + a);
      const int su = min(max(d_find_span(Uk, R.n, P, ua), S0), S1 - 1);
      float nu[P + 1], nud[P + 1];
      d_basis_ders<P>(Uk, su, ua, P, nu, nud);
      su_s[tid] = su;
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        Nu_s[tid * NP + k] = k <= P ? nu[k <= P ? k : 0] : 0.f;
        Nud_s[tid * NP + k] = k <= P ? nud[k <= P ? k : 0] : 0.f;
      }
    }
    __syncthreads();
    // one row: S', S'_u, S'_v from the window (packed FFMA2), Eq.7 quotient rule, normal, stores
    auto row = [&](int i) {
      float4 Sp = f4(0.f), Su = f4(0.f), Sv = f4(0.f);
#pragma unroll
      for (int k = 0; k <= P; ++k) {
        const float nu = Nu_s[i * NP + k], nud = Nud_s[i * NP + k];
        Sp = fma4v(nu, tw[k], Sp);
        Su = fma4v(nud, tw[k], Su);
        Sv = fma4v(nu, tvw[k], Sv);
      }
      const float rw = 1.0f / Sp.w;
      const float sx = Sp.x * rw, sy = Sp.y * rw, sz = Sp.z * rw;
      // Eq.7: S_u = (NR_u w - NR w_u) / w^2 = (S'_u,xyz - S S'_u,w) / W
      const float ux = (Su.x - sx * Su.w) * rw, uy = (Su.y - sy * Su.w) * rw, uz = (Su.z - sz * Su.w) * rw;
      const float vx = (Sv.x - sx * Sv.w) * rw, vy = (Sv.y - sy * Sv.w) * rw, vz = (Sv.z - sz * Sv.w) * rw;
      if (valid) {
        const size_t o = o0 + (size_t)(c0 + i) * grow;
        if (prm.out) {
          prm.out[o] = sx;
          prm.out[o + 1] = sy;
          prm.out[o + 2] = sz;
        }
        out_u[o] = ux;
        out_u[o + 1] = uy;
        out_u[o + 2] = uz;
        out_v[o] = vx;
        out_v[o + 1] = vy;
        out_v[o + 2] = vz;
        if (normals) {  // n = S_u x S_v / |S_u x S_v| (offsetting input)
          const float nx = uy * vz - uz * vy, ny = uz * vx - ux * vz, nz = ux * vy - uy * vx;
          const float inv = rsqrtf(fmaf(nx, nx, fmaf(ny, ny, nz * nz)));
          normals[o] = nx * inv;
          normals[o + 1] = ny * inv;
          normals[o + 2] = nz * inv;
        }
      }
    };
    auto advance = [&](int target) {
      while (lo < target) {  // uniform: slide the window by one control row
#pragma unroll
        for (int k = 0; k < P; ++k) {
          tw[k] = tw[k + 1];
          tvw[k] = tvw[k + 1];
        }
        ++lo;
        Trow2(lo + P, tw[P], tvw[P]);
      }
    };
    constexpr int RU = NB_DERIV_RU;  // rows per unrolled run when the window does not move
    int i = 0;
    while (i < cn) {
      advance(su_s[i] - P);
      if (i + RU <= cn && su_s[i + RU - 1] - P == lo) {
#pragma unroll
        for (int r = 0; r < RU; ++r) row(i + r);
        i += RU;
      } else {
        row(i);
        ++i;
      }
    }
  }
}

template <int P, int Q>
static cudaError_t launch_derivs_pq(const Params& prm, float* ou, float* ov, float* nrm, cudaStream_t st) {
  nurbs_derivs_kernel<P, Q><<<(unsigned)((long long)prm.B * prm.NRB * prm.NCB), kThreads, 0, st>>>(prm, ou, ov, nrm);
  return cudaGetLastError();
}

template <int P>
static cudaError_t launch_derivs_p(const Params& prm, int q, float* ou, float* ov, float* nrm, cudaStream_t st) {
  switch (q) {
    case 1: return launch_derivs_pq<P, 1>(prm, ou, ov, nrm, st);
    case 2: return launch_derivs_pq<P, 2>(prm, ou, ov, nrm, st);
    case 3: return launch_derivs_pq<P, 3>(prm, ou, ov, nrm, st);
    case 4: return launch_derivs_pq<P, 4>(prm, ou, ov, nrm, st);
    case 5: return launch_derivs_pq<P, 5>(prm, ou, ov, nrm, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_derivs(const Params& prm, int P, int q, float* out_u, float* out_v, float* normals,
                          cudaStream_t st) {
  switch (P) {
    case 1: return launch_derivs_p<1>(prm, q, out_u, out_v, normals, st);
    case 2: return launch_derivs_p<2>(prm, q, out_u, out_v, normals, st);
    case 3: return launch_derivs_p<3>(prm, q, out_u, out_v, normals, st);
    case 4: return launch_derivs_p<4>(prm, q, out_u, out_v, normals, st);
    case 5: return launch_derivs_p<5>(prm, q, out_u, out_v, normals, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace nb
