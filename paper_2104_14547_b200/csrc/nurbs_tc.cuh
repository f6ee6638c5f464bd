// nurbs_tc.cuh — PTX wrappers for the 5th-generation tensor cores (tcgen05) and tensor
// memory (TMEM) on sm_100a: allocation, the kind::tf32 MMA with A in TMEM and B in shared
// memory, commit to an mbarrier, TMEM <-> register moves, the ordering fences, and the
// shared-memory matrix / instruction descriptors.
//
// Layouts (PTX ISA "tcgen05 matrix descriptors", CUTLASS cute/arch/mma_sm100_desc.hpp):
//  * TMEM address = (lane << 16) | column; a warp w may only touch lanes 32*(w%4) .. +31.
//  * D (fp32 accumulator) of an M = 128, cta_group::1 MMA: row m -> lane m, column n -> col n.
//  * A from TMEM (kind::tf32): A[m][k] at lane m, column a_col + k (8 columns per MMA, K = 8).
//  * B from shared memory, K-major, no swizzle ("interleave"): 8-row x 16-byte core matrices;
//    element (n, k) of a tf32 matrix at byte (n%8)*16 + (n/8)*SBO + (k/4)*LBO + (k%4)*4.
#pragma once
#include <cstdint>

#include "nurbs_device.cuh"

namespace nb {
namespace tc {

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// mbarrier wait without a suspend-time hint (the hardware's default, short, time limit): the
// MMA issuer and the compute warps react to a completed phase at once instead of sleeping.
__device__ __forceinline__ void mbar_wait_spin(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT_S:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_S;\n"
      "bra LAB_WAIT_S;\n"
      "DONE_S:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem desc], kind::tf32, fp32 accumulate; `acc` = 0 overwrites D.
__device__ __forceinline__ void mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}
// Arrive (once) on `bar` when every tcgen05.mma issued so far by this thread has completed.
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Instruction descriptor: kind::tf32, D fp32, A and B tf32 K-major, M x N (CUTLASS
// UMMA::InstrDescriptor: c_format bits 4-5, a/b_format bits 7-9 / 10-12, N>>3 at 17, M>>4 at 24).
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// Shared-memory matrix descriptor, K-major, no swizzle (version 1 = sm_100).
__device__ __forceinline__ uint64_t sdesc(const void* p, uint32_t lbo, uint32_t sbo) {
  const uint32_t a = smem_u32(p);
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// Byte offset of element (n, k) in a K-major no-swizzle tf32 operand with LBO = 128 (the two
// 16-byte K halves of an MMA step are adjacent core matrices) and SBO = (K/4) * 128.
__device__ __forceinline__ uint32_t kmaj_off(int n, int k, int K) {
  return (uint32_t)((n & 7) * 16 + (n >> 3) * (K / 4) * 128 + (k >> 2) * 128 + (k & 3) * 4);
}

// The tf32 head of x: its top 19 bits (sign, exponent, 10 mantissa bits), i.e. x truncated
// toward zero, which the tensor core reads exactly; x - hi is then exact in fp32 and holds the
// next 13 bits, of which the tensor core reads the top 11 (3xTF32: ~2^-21 relative per
// product). One LOP3 (cvt.rna.tf32.f32 is a 4-instruction sequence on sm_100a).
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
// (x0 - h0, x1 - h1) as one packed FFMA2: the two tails of a pair of splits.
__device__ __forceinline__ float2 tf32_lo2(float x0, float x1, float h0, float h1) {
  return up2(ffma2(pk2(h0, h1), pk2(-1.f, -1.f), pk2(x0, x1)));
}

// TMEM <-> registers, 32 lanes x 32 bits x N columns (thread t of the warp <-> lane base + t).
__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}

}  // namespace tc
}  // namespace nb
