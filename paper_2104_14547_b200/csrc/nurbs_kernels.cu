// nurbs_kernels.cu — sm_100a kernels of the NURBS-Diff hot path (arXiv 2104.14547).
//
// Citations: P:n = reference/PAPER.md line n; R<k> = reading k of DESIGN.md §3.
//
// The grid case is evaluated as the separable banded product S' = N_u · Q · N_v^T (Eq.3
// P:110 with the homogeneous points of P:140, Q_ij = (w_ij P_ij, w_ij)):
//   F1  T[i][b]  = sum_h Nv[b][h] Q[i][sv(b)-q+h]            (per CTA column block, smem)
//   F2  S'[a][b] = sum_r Nu[a][r] T[su(a)-p+r][b]            (rolling register window)
//       S = S'_xyz / S'_w                                     (P:140 step 3)
// and the backward (Eq.8 P:215 / Eq.9 P:222 / J^T g of P:251) as its transpose:
//   G[a][b]  = (g/W, -(g.S)/W)              (homogeneous upstream)
//   B1 H[i][b]  = sum_a Nu[a][i-su(a)+p] G[a][b]   (rolling accumulators, flushed in order)
//   B2 dQ[i][j] = sum_b H[i][b] Nv[b][j-sv(b)+q]   (fixed b order)
//   dP = w dQ_xyz, dw = P.dQ_xyz + dQ_w
// Every reduction runs in a fixed order; there are no floating-point atomics, so results
// are bitwise repeatable (SPEC S:157's deterministic gather, instead of the paper's scatter
// of P:289).
//
// CTA = (surface s, row block rb, column block cb). A row block is K consecutive KNOT SPANS
// of the u direction (its sample rows are those whose span falls in [S0, S0+K)), so its
// control-row band [rb*K, S0+K-1] has at most K+p <= kRMax rows; a column block is 128
// consecutive SAMPLE columns (one compute thread each). Warp 4 is a TMA producer: it streams
// grad_out rows into a 3-stage smem ring (bwd) or drains the staged output rows to HBM with
// cp.async.bulk (fwd).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "nurbs_internal.cuh"

namespace nb {

// ------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared, completion counted on an mbarrier (transaction bytes).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// TMA bulk copy shared -> global (bulk async-group completion).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bar_compute() {  // named barrier over the 128 compute threads
  asm volatile("bar.sync 1, %0;" ::"n"(kCompute) : "memory");
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float4 f4(float a) { return make_float4(a, a, a, a); }
__device__ __forceinline__ float4 fma4(float s, float4 a, float4 acc) {
  return make_float4(fmaf(s, a.x, acc.x), fmaf(s, a.y, acc.y), fmaf(s, a.z, acc.z), fmaf(s, a.w, acc.w));
}
// homogeneous point P^w = (w x, w y, w z, w)   (P:140 step 3)
__device__ __forceinline__ float4 homog(float4 c) { return make_float4(c.x * c.w, c.y * c.w, c.z * c.w, c.w); }

// ------------------------------------------------------------------------ FindSpan / basis
// FindSpan (R2-R4): largest s in [p, n-1] with U[s] <= u, stepped down over empty
// intervals (only possible at u == U[n]). Out-of-domain u is clamped (checked mode rejects
// it). Pure fp32 comparisons on the caller's fp32 knots, so spans are bit-exact with the
// oracle (which compares the same values in fp64).
__device__ __forceinline__ int d_find_span(const float* __restrict__ U, int n, int p, float u) {
  if (!(u >= __ldg(U + p))) return p;
  int lo = p, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(U + mid) <= u) lo = mid; else hi = mid - 1;
  }
  while (lo > p && __ldg(U + lo) == __ldg(U + lo + 1)) --lo;
  return lo;
}

// Cox-de Boor (Eq.4) on the p+1 non-zero functions, Piegl-Tiller A2.2 order.
// MAXD is the static array bound; p <= MAXD is the (possibly runtime) degree.
template <int MAXD>
__device__ __forceinline__ void d_basis(const float* __restrict__ U, int s, float u, int p, float* N) {
  float left[MAXD + 1], right[MAXD + 1];
  N[0] = 1.f;
#pragma unroll
  for (int j = 1; j <= MAXD; ++j) {
    if (j <= p) {
      left[j] = u - __ldg(U + s + 1 - j);
      right[j] = __ldg(U + s + j) - u;
      float saved = 0.f;
#pragma unroll
      for (int r = 0; r < j; ++r) {
        const float temp = N[r] / (right[r + 1] + left[j - r]);
        N[r] = fmaf(right[r + 1], temp, saved);
        saved = left[j - r] * temp;
      }
      N[j] = saved;
    } else {
      N[j] = 0.f;
    }
  }
}

// ------------------------------------------------------------------------ k-ary search
// First a in [0, ns] with pred(a) (pred monotone false..true, pred(ns) := true). Called by
// all kThreads threads of the CTA with identical arguments; ~2 rounds for ns = 8192.
template <typename Pred>
__device__ int cta_first_true(int ns, Pred pred) {
  int lo = 0, hi = ns;
  while (lo < hi) {
    const int step = (hi - lo + kThreads - 1) / kThreads;
    const int x = lo + (int)threadIdx.x * step;
    const bool f = (x < hi) && !pred(x);
    const int nf = __syncthreads_count(f);
    if (nf == 0) {
      hi = lo;
    } else {
      const int nlo = lo + (nf - 1) * step + 1;
      const int nhi = min(lo + nf * step, hi);
      lo = nlo;
      hi = nhi;
    }
  }
  return lo;
}

// Row span of sample a (tables or in-kernel).
template <int P>
__device__ __forceinline__ int row_span(const Dir& R, const float* Uk, int a) {
  if (P == 0) return 0;
  if (R.tspan) return __ldg(R.tspan + a);
  return d_find_span(Uk, R.n, P, __ldg(R.s + a));
}

// ------------------------------------------------------------------------ the grid kernel
template <int P, bool BWD>
__global__ void __launch_bounds__(kThreads, 4) nurbs_grid_kernel(const Params prm) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int NP = (P + 1) <= 4 ? 4 : 8;  // floats per row-basis entry in smem
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const Dir& R = prm.r;
  const Dir& C = prm.c;
  const int Q = C.p;
  const int NQ = (Q + 1) <= 4 ? 4 : 8;

  // ---- decode the tile
  int bid = blockIdx.x;
  const int cb = bid % prm.NCB;
  bid /= prm.NCB;
  const int rb = bid % prm.NRB;
  const int s = bid / prm.NRB;
  const int B0 = cb * kCB;
  const int cols = min(kCB, C.ns - B0);
  const int S0 = P + rb * prm.K;                 // first knot span of this row block
  const int S1 = min(S0 + prm.K, R.n);           // one past the last
  const int band_lo = S0 - P;                    // control-row band [band_lo, S1-1]
  const int band_rows = S1 - band_lo;            // <= T_rows
  const float* Uk = (P > 0) ? R.knots + (long long)s * R.kstride : nullptr;
  const float* Vk = C.tspan ? nullptr : C.knots + (long long)s * C.kstride;

  // ---- shared memory carve-up
  float4* T = reinterpret_cast<float4*>(smem);                       // [T_rows][kCB] (T, then H)
  float* stage = reinterpret_cast<float*>(T + (size_t)prm.T_rows * kCB);  // [kStages][kRPS*kCB*3]
  int* su_s = reinterpret_cast<int*>(stage + kStages * kRPS * kCB * 3);   // [kRowChunk]
  float* Nu_s = reinterpret_cast<float*>(su_s + kRowChunk);               // [kRowChunk][NP]
  int* sv_s = reinterpret_cast<int*>(Nu_s + kRowChunk * NP);              // [kCB]      (bwd)
  float* Nv_s = reinterpret_cast<float*>(sv_s + kCB);                     // [kCB][NQ]  (bwd)
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(Nv_s + (BWD ? kCB * NQ : 0)) + 7) & ~uintptr_t(7));
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;

  if (tid == 0 && prm.bulk) {
#pragma unroll
    for (int i = 0; i < kStages; ++i) {
      mbar_init(full + i, BWD ? 1u : (uint32_t)kCompute);
      mbar_init(empty + i, BWD ? (uint32_t)kCompute : 1u);
    }
    fence_mbar_init();
  }

  // ---- sample rows of this row block: spans in [S0, S1)   (all 160 threads)
  int a_lo = 0, a_hi = R.ns;
  if (prm.NRB > 1) {
    int s_end = R.n - 1;  // last non-empty span (R3)
    if (P > 0 && !R.tspan)
      while (s_end > P && __ldg(Uk + s_end) == __ldg(Uk + s_end + 1)) --s_end;
    auto ge = [&](int S) {
      return [&, S](int a) -> bool {
        if (R.tspan) return __ldg(R.tspan + a) >= S;
        if (S > s_end) return false;
        return __ldg(R.s + a) >= __ldg(Uk + S);
      };
    };
    if (rb > 0) a_lo = cta_first_true(R.ns, ge(S0));
    if (rb < prm.NRB - 1) a_hi = cta_first_true(R.ns, ge(S1));
  }
  __syncthreads();
  const int nwalk = max(0, a_hi - a_lo);
  const int nstage = (nwalk + kRPS - 1) / kRPS;
  const bool contig = (cols == C.ns);  // whole sample rows: consecutive rows are contiguous

  // ======================================================== producer warp (TMA bulk)
  if (warp == kCompute / 32) {
    if (prm.bulk && (tid & 31) == 0) {
      const uint32_t rowbytes = (uint32_t)cols * 12u;
      for (int k = 0; k < nstage; ++k) {
        const int slot = k % kStages, use = k / kStages;
        const int r0 = a_lo + k * kRPS;
        const int nr = min(kRPS, a_hi - r0);
        float* buf = stage + slot * (kRPS * kCB * 3);
        if (BWD) {
          if (use > 0) mbar_wait(empty + slot, (use - 1) & 1);
          mbar_arrive_expect_tx(full + slot, rowbytes * nr);
          const float* src = prm.gout + ((size_t)((size_t)s * R.ns + r0) * C.ns + B0) * 3;
          if (contig) {
            bulk_g2s(buf, src, rowbytes * nr, full + slot);
          } else {
            for (int rr = 0; rr < nr; ++rr)
              bulk_g2s(buf + rr * cols * 3, src + (size_t)rr * C.ns * 3, rowbytes, full + slot);
          }
        } else {
          mbar_wait(full + slot, use & 1);
          float* dst = prm.out + ((size_t)((size_t)s * R.ns + r0) * C.ns + B0) * 3;
          if (contig) {
            bulk_s2g(dst, buf, rowbytes * nr);
          } else {
            for (int rr = 0; rr < nr; ++rr) bulk_s2g(dst + (size_t)rr * C.ns * 3, buf + rr * cols * 3, rowbytes);
          }
          bulk_commit();
          bulk_wait_read_all();
          mbar_arrive(empty + slot);
        }
      }
      if (!BWD) bulk_wait_all();
    }
    return;
  }

  // ======================================================== compute warps (128 threads)
  const int t = tid;
  const bool valid = t < cols;
  const int b = B0 + (valid ? t : cols - 1);

  // ---- column span + basis (registers), shared with the B2 stage in smem
  int sv;
  float nv[kMaxQ + 1];
  if (C.tspan) {
    sv = __ldg(C.tspan + b);
    const float* tn = C.tN + (size_t)b * C.tnp;
#pragma unroll
    for (int h = 0; h <= kMaxQ; ++h) nv[h] = (h <= Q) ? __ldg(tn + h) : 0.f;
  } else {
    const float vb = __ldg(C.s + b);
    sv = d_find_span(Vk, C.n, Q, vb);
    d_basis<kMaxQ>(Vk, sv, vb, Q, nv);
  }
  sv = min(max(sv, Q), C.n - 1);
  if (BWD) {
    sv_s[t] = sv;
#pragma unroll
    for (int h = 0; h <= kMaxQ; ++h)
      if (h < NQ) Nv_s[t * NQ + h] = nv[h];
  }

  // ---- F1: T[r][t] = sum_h Nv[h] Q[band_lo + r][sv - q + h]
  const float4* __restrict__ ctrl_s = prm.ctrl + (size_t)s * R.n * C.n;
  {
    const float4* colp = ctrl_s + (sv - Q);
#pragma unroll 2
    for (int r = 0; r < band_rows; ++r) {
      const float4* rowp = colp + (size_t)(band_lo + r) * C.n;
      float4 acc = f4(0.f);
#pragma unroll
      for (int h = 0; h <= kMaxQ; ++h)
        if (h <= Q) acc = fma4(nv[h], homog(__ldg(rowp + h)), acc);
      T[r * kCB + t] = acc;
    }
  }

  // ---- walk the sample rows: rolling window of P+1 control rows [lo, lo+P]
  float4 tw[P + 1];
  float4 acc[P + 1];
  int lo = band_lo;
#pragma unroll
  for (int k = 0; k <= P; ++k) {
    tw[k] = T[k * kCB + t];
    acc[k] = f4(0.f);
  }

  const size_t gbase = (size_t)s * R.ns;  // row index base of this surface in out/gout
  for (int c0 = 0; c0 < nwalk; c0 += kRowChunk) {
    const int cn = min(kRowChunk, nwalk - c0);
    if (t < cn) {  // stage span + basis of rows a_lo+c0 .. +cn
      const int a = a_lo + c0 + t;
      int su;
      float nu[P + 1];
      if (P == 0) {
        su = 0;
        nu[0] = 1.f;
      } else if (R.tspan) {
        su = __ldg(R.tspan + a);
        const float* tn = R.tN + (size_t)a * R.tnp;
#pragma unroll
        for (int k = 0; k <= P; ++k) nu[k] = __ldg(tn + k);
      } else {
        const float ua = __ldg(R.s + a);
        su = d_find_span(Uk, R.n, P, ua);
        d_basis<P>(Uk, su, ua, P, nu);
      }
      su_s[t] = min(max(su, S0), S1 - 1);  // memory safety for inconsistent inputs
#pragma unroll
      for (int k = 0; k < NP; ++k) Nu_s[t * NP + k] = (k <= P) ? nu[k <= P ? k : 0] : 0.f;
    }
    bar_compute();

    for (int i = 0; i < cn; ++i) {
      const int ra = c0 + i;  // row index within the walk
      const int k_st = ra / kRPS;
      const int rr = ra - k_st * kRPS;
      const int slot = k_st % kStages;
      const int use = k_st / kStages;
      float* buf = stage + slot * (kRPS * kCB * 3) + rr * cols * 3;
      if (prm.bulk && rr == 0) {
        if (BWD) mbar_wait(full + slot, use & 1);
        else if (use > 0) mbar_wait(empty + slot, (use - 1) & 1);
      }
      // advance the window to the span of this row (uniform across the CTA)
      const int newlo = su_s[i] - P;
      while (lo < newlo) {
        if (BWD) T[(lo - band_lo) * kCB + t] = acc[0];  // row lo complete: H (aliases T)
#pragma unroll
        for (int k = 0; k < P; ++k) {
          tw[k] = tw[k + 1];
          if (BWD) acc[k] = acc[k + 1];
        }
        ++lo;
        tw[P] = T[(lo + P - band_lo) * kCB + t];
        if (BWD) acc[P] = f4(0.f);
      }
      float nu[NP];
      {
        const float4 n0 = *reinterpret_cast<const float4*>(Nu_s + i * NP);
        nu[0] = n0.x; nu[1] = n0.y; nu[2] = n0.z; nu[3] = n0.w;
        if constexpr (NP == 8) {
          const float4 n1 = *reinterpret_cast<const float4*>(Nu_s + i * NP + 4);
          nu[4] = n1.x; nu[5] = n1.y; nu[6] = n1.z; nu[7] = n1.w;
        }
      }
      float4 Sp = f4(0.f);
#pragma unroll
      for (int k = 0; k <= P; ++k) Sp = fma4(nu[k], tw[k], Sp);
      const float rw = rcp_approx(Sp.w);
      const size_t gidx = ((gbase + a_lo + ra) * C.ns + b) * 3;

      if (!BWD) {
        const float ox = Sp.x * rw, oy = Sp.y * rw, oz = Sp.z * rw;
        if (prm.bulk) {
          if (valid) {
            buf[t * 3 + 0] = ox;
            buf[t * 3 + 1] = oy;
            buf[t * 3 + 2] = oz;
          }
          if (rr == kRPS - 1 || ra == nwalk - 1) {
            fence_proxy_async();
            mbar_arrive(full + slot);
          }
        } else if (valid) {
          prm.out[gidx + 0] = ox;
          prm.out[gidx + 1] = oy;
          prm.out[gidx + 2] = oz;
        }
      } else {
        float gx = 0.f, gy = 0.f, gz = 0.f;
        if (prm.bulk) {
          if (valid) {
            gx = buf[t * 3 + 0];
            gy = buf[t * 3 + 1];
            gz = buf[t * 3 + 2];
          }
          if (rr == kRPS - 1 || ra == nwalk - 1) mbar_arrive(empty + slot);
        } else if (valid) {
          gx = __ldg(prm.gout + gidx + 0);
          gy = __ldg(prm.gout + gidx + 1);
          gz = __ldg(prm.gout + gidx + 2);
        }
        // G = (g/W, -(g.S)/W) with S = S'_xyz / W  (Eq.8/9 through the homogeneous point)
        const float gS = fmaf(gx, Sp.x, fmaf(gy, Sp.y, gz * Sp.z)) * rw;
        const float4 G = make_float4(gx * rw, gy * rw, gz * rw, -gS * rw);
#pragma unroll
        for (int k = 0; k <= P; ++k) acc[k] = fma4(nu[k], G, acc[k]);
      }
    }
    bar_compute();  // all rows of this chunk consumed before su_s/Nu_s are refilled
  }

  if constexpr (BWD) {
  // ---- B1 epilogue: flush the last window, zero the rows never reached
#pragma unroll
  for (int k = 0; k <= P; ++k) T[(lo + k - band_lo) * kCB + t] = acc[k];
  for (int r = lo + P + 1 - band_lo; r < band_rows; ++r) T[r * kCB + t] = f4(0.f);
  bar_compute();

  // ---- B2: dQ[i][j] = sum_b H[i-band_lo][b] Nv[b][j - sv(b) + q], b ascending
  const int j0 = sv_s[0] - Q;
  const int j1 = sv_s[cols - 1];
  const int nj = j1 - j0 + 1;
  float4* gctrl_s = prm.gctrl + (size_t)s * R.n * C.n;
  const int ntask = prm.direct ? R.n * C.n : band_rows * nj;
  for (int task = t; task < ntask; task += kCompute) {
    int r, j;
    if (prm.direct) {
      r = task / C.n;  // band_lo == 0 and band_rows == R.n in direct mode
      j = task - r * C.n;
    } else {
      r = task / nj;
      j = j0 + (task - r * nj);
    }
    float4 a4 = f4(0.f);
    if (j >= j0 && j <= j1) {
      int blo = 0, bhi = cols;  // first b with sv >= j
      while (blo < bhi) {
        const int mid = (blo + bhi) >> 1;
        if (sv_s[mid] < j) blo = mid + 1; else bhi = mid;
      }
      int bend = blo, bh2 = cols;  // first b with sv > j + q
      while (bend < bh2) {
        const int mid = (bend + bh2) >> 1;
        if (sv_s[mid] <= j + Q) bend = mid + 1; else bh2 = mid;
      }
      const float4* Hr = T + r * kCB;
      for (int bb = blo; bb < bend; ++bb) a4 = fma4(Nv_s[bb * NQ + (j - sv_s[bb] + Q)], Hr[bb], a4);
    }
    if (prm.direct) {
      // epilogue (Eq.8/9): dP = w dQ_xyz, dw = P.dQ_xyz + dQ_w
      const float4 c = __ldg(ctrl_s + (size_t)r * C.n + j);
      gctrl_s[(size_t)r * C.n + j] =
          make_float4(c.w * a4.x, c.w * a4.y, c.w * a4.z, fmaf(c.x, a4.x, fmaf(c.y, a4.y, fmaf(c.z, a4.z, a4.w))));
    } else {
      prm.slots[((((size_t)s * prm.NRB + rb) * prm.NCB + cb) * prm.T_rows + r) * C.n + j] = a4;
    }
  }
  if (!prm.direct && rb == 0 && t == 0) prm.colband[(size_t)s * prm.NCB + cb] = make_int2(j0, j1);
  if (prm.direct) {  // knot gradients are zero by definition
    if (prm.gR && s < prm.gR_items)
      for (int x = t; x < prm.gR_per; x += kCompute) prm.gR[(size_t)s * prm.gR_per + x] = 0.f;
    if (prm.gC && s < prm.gC_items)
      for (int x = t; x < prm.gC_per; x += kCompute) prm.gC[(size_t)s * prm.gC_per + x] = 0.f;
  }
  }  // BWD
}

// ------------------------------------------------------------------------ cross-tile reduce
// dQ_ij = sum over row blocks rb (ascending) and column blocks cb (ascending) whose bands
// contain (i, j) of the tile partials; then the Eq.8/9 epilogue. One thread per control point.
__global__ void __launch_bounds__(256) nurbs_reduce_kernel(const Params prm, int P) {
  const long long total = (long long)prm.B * prm.r.n * prm.c.n;
  const long long gsz = (long long)gridDim.x * blockDim.x;
  const long long idx0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (prm.gR)
    for (long long x = idx0; x < (long long)prm.gR_items * prm.gR_per; x += gsz) prm.gR[x] = 0.f;
  if (prm.gC)
    for (long long x = idx0; x < (long long)prm.gC_items * prm.gC_per; x += gsz) prm.gC[x] = 0.f;
  for (long long idx = idx0; idx < total; idx += gsz) {
    const int m = prm.c.n;
    const int j = (int)(idx % m);
    const long long t2 = idx / m;
    const int i = (int)(t2 % prm.r.n);
    const int s = (int)(t2 / prm.r.n);
    const int K = prm.K;
    const int rb_hi = min(prm.NRB - 1, i / K);
    const int x = i - K - P + 1;
    const int rb_lo = x <= 0 ? 0 : (x + K - 1) / K;
    const int2* cbands = prm.colband + (size_t)s * prm.NCB;
    int lo = 0, hi = prm.NCB;  // first cb with j1 >= j
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (cbands[mid].y < j) lo = mid + 1; else hi = mid;
    }
    float4 a4 = f4(0.f);
    for (int rb = rb_lo; rb <= rb_hi; ++rb) {
      const int r = i - rb * K;
      for (int cb = lo; cb < prm.NCB && cbands[cb].x <= j; ++cb) {
        const float4 v = prm.slots[((((size_t)s * prm.NRB + rb) * prm.NCB + cb) * prm.T_rows + r) * m + j];
        a4.x += v.x; a4.y += v.y; a4.z += v.z; a4.w += v.w;
      }
    }
    const float4 c = __ldg(prm.ctrl + idx);
    prm.gctrl[idx] =
        make_float4(c.w * a4.x, c.w * a4.y, c.w * a4.z, fmaf(c.x, a4.x, fmaf(c.y, a4.y, fmaf(c.z, a4.z, a4.w))));
  }
}

// ------------------------------------------------------------------------ tables
__global__ void nurbs_tables_kernel(Dir R, Dir C, unsigned char* tab, TabLayout L) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx == 0) {
    int* h = reinterpret_cast<int*>(tab);
    h[0] = (int)kTabMagic; h[1] = 1;
    h[2] = R.n; h[3] = R.p; h[4] = R.ns; h[5] = L.np_r;
    h[6] = C.n; h[7] = C.p; h[8] = C.ns; h[9] = L.np_c;
  }
  const Dir& D = idx < R.ns ? R : C;
  const int a = idx < R.ns ? idx : idx - R.ns;
  if (idx >= R.ns + C.ns) return;
  int* span = reinterpret_cast<int*>(tab + (idx < R.ns ? L.off_span_r : L.off_span_c));
  float* N = reinterpret_cast<float*>(tab + (idx < R.ns ? L.off_N_r : L.off_N_c));
  const int np = idx < R.ns ? L.np_r : L.np_c;
  const float x = __ldg(D.s + a);
  float nb_[kMaxQ + 1];
  int sp = 0;
  if (D.p == 0) {
    nb_[0] = 1.f;
  } else {
    sp = d_find_span(D.knots, D.n, D.p, x);
    d_basis<kMaxQ>(D.knots, sp, x, D.p, nb_);
  }
  span[a] = sp;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (k < np) N[(size_t)a * np + k] = (k <= D.p && k <= kMaxQ) ? nb_[k <= kMaxQ ? k : 0] : 0.f;
}

// ------------------------------------------------------------------------ validation
// status = min over violations of (code << 48 | which << 40 | index).
__device__ __forceinline__ void report(unsigned long long* st, int code, int which, long long index) {
  const unsigned long long key =
      ((unsigned long long)code << 48) | ((unsigned long long)which << 40) | ((unsigned long long)index & 0xffffffffffull);
  atomicMin(st, key);
}

__global__ void nurbs_validate_kernel(int B, Dir R, Dir C, int check_rows, const float4* ctrl, long long n_ctrl,
                                      unsigned long long* st) {
  const long long gsz = (long long)gridDim.x * blockDim.x;
  const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int items_r = R.kstride ? B : 1, items_c = C.kstride ? B : 1;
  // weights and finiteness (code 5 = NURBS_E_WEIGHT), which = 0
  for (long long x = i0; x < n_ctrl; x += gsz) {
    const float4 c = ctrl[x];
    if (!(c.w > 0.f) || !isfinite(c.w) || !isfinite(c.x) || !isfinite(c.y) || !isfinite(c.z)) report(st, 5, 0, x);
  }
  for (int d = 0; d < 2; ++d) {
    const Dir& D = d == 0 ? R : C;
    if (d == 0 && !check_rows) continue;
    const int items = d == 0 ? items_r : items_c;
    const int nk = D.n + D.p + 1;
    // knots non-decreasing, finite, non-empty domain (code 3 = NURBS_E_KNOTS), which = 1 + d
    for (long long x = i0; x < (long long)items * nk; x += gsz) {
      const int it = (int)(x / nk), k = (int)(x % nk);
      const float* Uk = D.knots + (long long)it * D.kstride;
      if (!isfinite(Uk[k])) report(st, 3, 1 + d, x);
      if (k + 1 < nk && !(Uk[k] <= Uk[k + 1])) report(st, 3, 1 + d, x);
      if (k == 0 && !(Uk[D.p] < Uk[D.n])) report(st, 3, 1 + d, x);
    }
    // samples sorted (code 6) and inside every item's domain (code 4), which = 3 + d
    for (long long x = i0; x < (long long)items * D.ns; x += gsz) {
      const int it = (int)(x / D.ns), a = (int)(x % D.ns);
      const float* Uk = D.knots + (long long)it * D.kstride;
      const float u = D.s[a];
      if (it == 0 && a + 1 < D.ns && !(u <= D.s[a + 1])) report(st, 6, 3 + d, a);
      if (!(u >= Uk[D.p] && u <= Uk[D.n])) report(st, 4, 3 + d, a);
    }
  }
}

// ------------------------------------------------------------------------ launchers
size_t grid_smem_bytes(bool bwd, int P, int q, int T_rows) {
  const int NP = (P + 1) <= 4 ? 4 : 8;
  const int NQ = (q + 1) <= 4 ? 4 : 8;
  size_t b = (size_t)T_rows * kCB * 16 + (size_t)kStages * kRPS * kCB * 3 * 4 + kRowChunk * 4 +
             (size_t)kRowChunk * NP * 4;
  if (bwd) b += kCB * 4 + (size_t)kCB * NQ * 4;
  b = (b + 7) / 8 * 8 + 2 * kStages * 8;
  return b;
}

template <int P, bool BWD>
static cudaError_t launch_one(const Params& prm, cudaStream_t st) {
  const size_t smem = grid_smem_bytes(BWD, P, prm.c.p, prm.T_rows);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(nurbs_grid_kernel<P, BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         96 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  nurbs_grid_kernel<P, BWD><<<(unsigned)((long long)prm.B * prm.NRB * prm.NCB), kThreads, smem, st>>>(prm);
  return cudaGetLastError();
}

cudaError_t launch_grid(const Params& prm, bool bwd, int P, int q, cudaStream_t st) {
  (void)q;
#define NB_CASE(PP)                                                                   \
  case PP:                                                                            \
    return bwd ? launch_one<PP, true>(prm, st) : launch_one<PP, false>(prm, st);
  switch (P) {
    NB_CASE(0)
    NB_CASE(1)
    NB_CASE(2)
    NB_CASE(3)
    NB_CASE(4)
    NB_CASE(5)
    default:
      return cudaErrorInvalidValue;
  }
#undef NB_CASE
}

cudaError_t launch_reduce(const Params& prm, int P, cudaStream_t st) {
  const long long total = (long long)prm.B * prm.r.n * prm.c.n;
  long long blocks = (total + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 32) blocks = 148 * 32;
  nurbs_reduce_kernel<<<(unsigned)blocks, 256, 0, st>>>(prm, P);
  return cudaGetLastError();
}

cudaError_t launch_tables(const Dir& r, const Dir& c, void* tables, const TabLayout& L, cudaStream_t st) {
  const int total = r.ns + c.ns;
  const int blocks = total > 0 ? (total + 255) / 256 : 1;
  nurbs_tables_kernel<<<blocks, 256, 0, st>>>(r, c, static_cast<unsigned char*>(tables), L);
  return cudaGetLastError();
}

cudaError_t launch_validate(int B, const Dir& r, const Dir& c, int check_rows, const float4* ctrl,
                            long long n_ctrl, unsigned long long* status, cudaStream_t st) {
  nurbs_validate_kernel<<<148 * 4, 256, 0, st>>>(B, r, c, check_rows, ctrl, n_ctrl, status);
  return cudaGetLastError();
}

}  // namespace nb
