// nurbs_device.cuh — device helpers shared by the sm_100a kernels: PTX wrappers (mbarrier,
// cp.async.bulk TMA, proxy fences), FindSpan / Cox-de Boor, the CTA k-ary search.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

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
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity), "r"(0x989680u)  // suspend-time hint (ns): sleep until the phase flips
      : "memory");
}
// TMA bulk copy global -> shared, completion counted on an mbarrier (transaction bytes).
// Bulk prefetch of [p, p + bytes) into L2 (p 16-byte aligned, bytes a multiple of 16).
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
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
// Ampere-style cp.async (LDGSTS): small global -> shared copies completing asynchronously
// (the next row chunk's span / basis tables, prefetched one chunk ahead).
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// 2-D tensor TMA (cp.async.bulk.tensor): box {x = innermost element, y = row} of the tensor
// described by `map` (a __grid_constant__ kernel parameter), dense in smem.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {  // at most N most recent bulk groups still reading smem
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
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
// Packed fp32x2 (sm_100 FFMA2 / FMUL2): a float4 is two 64-bit register pairs (x,y), (z,w);
// a scalar factor is broadcast by ptxas into the .F32 operand form (no packing moves).
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(a), "f"(b));
  return d;
}
__device__ __forceinline__ float2 up2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long fmul2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ unsigned long long fsub2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// acc + s * a on float4 as two FFMA2 (same rounding as four fmaf).
__device__ __forceinline__ float4 fma4v(float s, float4 a, float4 acc) {
  const unsigned long long ss = pk2(s, s);
  const float2 lo = up2(ffma2(ss, pk2(a.x, a.y), pk2(acc.x, acc.y)));
  const float2 hi = up2(ffma2(ss, pk2(a.z, a.w), pk2(acc.z, acc.w)));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
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
__device__ __forceinline__ int cta_first_true(int ns, Pred pred) {
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

}  // namespace nb
