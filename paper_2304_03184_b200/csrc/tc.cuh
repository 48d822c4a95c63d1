// tcgen05 / TMEM / mbarrier primitives (inline PTX, sm_100a) and the fused
// tiny-MLP layer step used by every network kernel.
//
// Operand layout in shared memory (UMMA canonical K-major, SWIZZLE_NONE):
// an R x K fp16 matrix is stored as core matrices of 8 rows x 8 halves
// (128 contiguous bytes, row r at +16 r), ordered [r/8][k/8]:
//   byte(r, k) = (r/8) * (K/8) * 128 + (k/8) * 128 + (r%8) * 16 + (k%8) * 2
// so LBO (next core matrix along K) = 128 B and SBO (next 8-row group) = K*16 B.
// Activations (A, M=128 samples) and weights (B, N x K, i.e. W row-major) share it.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__host__ __device__ constexpr uint32_t core_offset(int r, int k, int K) {
  return (uint32_t)((r >> 3) * (K >> 3) * 128 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

// smem matrix descriptor (tcgen05 "shared memory descriptor", version 1)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (Blackwell)
  // base_offset = 0, lbo_mode = 0, layout = SWIZZLE_NONE (0)
  return d;
}

// instruction descriptor: kind::f16, A/B = F16, D = F32, both K-major, M=128
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4)                          // c_format = F32
         | (0u << 7) | (0u << 10)           // a/b format = F16
         | (0u << 15) | (0u << 16)          // K-major A and B
         | ((uint32_t)(N >> 3) << 17)       // n_dim
         | ((uint32_t)(M >> 4) << 24);      // m_dim
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// Wait for the phase with a suspend-time hint: the waiting warps sleep until the phase
// completes instead of polling, so a slot waiting on its MMAs leaves the issue slots to
// the slot running its epilogue (polling warps took 39 % of the DeformNet kernel's stall
// samples and stretched the other slot's epilogue)
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, 0x989680;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
  }
}

// named barrier over `count` threads
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_free(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// 16 consecutive fp32 columns
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// A operand from TMEM ("TS" form): D[128 x N] (+)= A_tmem[128 x K] * B_smem[N x K]^T.
// A row r = TMEM lane r; column c holds fp16 elements (2c, 2c+1) (low half = even k).
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Split-fp16 layer ("fp32" precision mode): with A = Ah + Al and B = Bh + Bl
// (hi/lo fp16 halves), D = Ah.Bh + Ah.Bl + Al.Bh accumulated in fp32 TMEM — three
// kind::f16 MMA chains, ~22 significant bits per operand (the dropped Al.Bl term is
// 2^-22 relative). A halves in TMEM (TS form), B halves in smem. Issued by a whole
// (converged) warp from one elected lane, the three chains and the commit in one asm
// block: the operands stay in uniform registers and the MMAs go out back to back.
// Issued from one divergent thread, each MMA cost ~14 instructions of convergence
// loops and R2UR broadcasts, and the issue stream stalled behind the other slot's
// epilogue warps (DeformNet fp32 mode 118 -> 96 us).
#define CF_MMA_STEP(ACC)                                              \
  "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [ta], tb, %5, " ACC ";\n\t" \
  "add.u32 ta, ta, 8;\n\tadd.s64 tb, tb, 16;\n\t"
#define CF_CHAIN2(ACC) CF_MMA_STEP(ACC) CF_MMA_STEP("pt")
#define CF_CHAIN4(ACC) CF_CHAIN2(ACC) CF_CHAIN2("pt")
#define CF_CHAIN8(ACC) CF_CHAIN4(ACC) CF_CHAIN4("pt")
#define CF_SPLIT_ASM(CHAIN)                                                                          \
  "{\n\t.reg .pred e, pf, pt;\n\t.reg .b32 ta;\n\t.reg .b64 tb;\n\t"                              \
  "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 pf, 0, 0;\n\tsetp.eq.b32 pt, 0, 0;\n\t"                 \
  "mov.b32 ta, %1;\n\tmov.b64 tb, %3;\n\t" CHAIN("pf")                                             \
  "mov.b32 ta, %1;\n\tmov.b64 tb, %4;\n\t" CHAIN("pt")                                             \
  "mov.b32 ta, %2;\n\tmov.b64 tb, %3;\n\t" CHAIN("pt")                                             \
  "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n\t}\n"
template <int K>
__device__ __forceinline__ void issue_split_warp(uint32_t tmem_d, uint32_t a_hi, uint32_t a_lo, const uint8_t* b_hi,
                                                 const uint8_t* b_lo, int N, uint64_t* bar) {
  const uint64_t dh = sdesc(smem_u32(b_hi), 128, (uint32_t)K * 16), dl = sdesc(smem_u32(b_lo), 128, (uint32_t)K * 16);
  const uint32_t idesc = idesc_f16(128, N), b = smem_u32(bar);
  if constexpr (K == 32)
    asm volatile(CF_SPLIT_ASM(CF_CHAIN2)::"r"(tmem_d), "r"(a_hi), "r"(a_lo), "l"(dh), "l"(dl), "r"(idesc), "r"(b)
                 : "memory");
  else if constexpr (K == 64)
    asm volatile(CF_SPLIT_ASM(CF_CHAIN4)::"r"(tmem_d), "r"(a_hi), "r"(a_lo), "l"(dh), "l"(dl), "r"(idesc), "r"(b)
                 : "memory");
  else {
    static_assert(K == 128, "K = 32, 64 or 128");
    asm volatile(CF_SPLIT_ASM(CF_CHAIN8)::"r"(tmem_d), "r"(a_hi), "r"(a_lo), "l"(dh), "l"(dl), "r"(idesc), "r"(b)
                 : "memory");
  }
}

// (a, b) -> packed fp16x2 hi = fp16(x) and lo = fp16(x - hi) (low halves = a)
__device__ __forceinline__ void split_f16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// ReLU fused into the split, 5 instructions per pair: hi = fp16x2 of relu(a, b) rounded
// toward zero (so x - hi >= 0 for x > 0), lo = fp16x2 of relu(x - hi) with x - hi from
// the mixed-precision f32 += f16 add (FHADD) on the negated hi halves; for x <= 0 both
// halves are 0. hi + lo carries relu(x) to ~2^-21 relative (lo < one fp16 ulp of hi).
__device__ __forceinline__ void split_relu_rz(float a, float b, uint32_t& hi, uint32_t& lo) {
  asm("cvt.rz.relu.f16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(b), "f"(a));
  const uint32_t nh = hi ^ 0x80008000u;
  float la, lb;
  asm("add.f32.f16 %0, %1, %2;" : "=f"(la) : "h"((unsigned short)(nh & 0xffffu)), "f"(a));
  asm("add.f32.f16 %0, %1, %2;" : "=f"(lb) : "h"((unsigned short)(nh >> 16)), "f"(b));
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(lb), "f"(la));
}

// 32 fp32 columns without the wait (issue several, then tmem_wait_ld once)
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// store 32 / 8 consecutive 32-bit columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
      "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
      "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// relu(a), relu(b) -> packed fp16x2 (low half = a), one instruction
__device__ __forceinline__ uint32_t relu_f16x2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

// write 8 fp16 (k = k0..k0+7) of row r into a canonical K-major operand buffer
__device__ __forceinline__ void st_row8(uint8_t* buf, int r, int k0, int K, const float* v) {
  __half2 h[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
  *reinterpret_cast<uint4*>(buf + core_offset(r, k0, K)) = *reinterpret_cast<uint4*>(h);
}

// Whole-warp issue: the calling warp is converged, one elected lane issues. The
// operands stay warp-uniform (uniform registers, no per-MMA convergence loop), so the
// issue stream is a few instructions per MMA even while other warps of the CTA run
// their epilogues. Commit from the same elected lane (tcgen05.commit tracks the MMAs
// of the executing thread).
__device__ __forceinline__ void mma_ts_elect(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_ss_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}
// a layer (TS: A from TMEM / SS: A from a canonical smem buffer) + commit, by one warp
__device__ __forceinline__ void layer_ts_warp(uint32_t tmem_d, uint32_t tmem_a, const uint8_t* b_buf, int K, int N,
                                              uint64_t* bar) {
  const uint64_t b0 = sdesc(smem_u32(b_buf), 128, (uint32_t)K * 16);
  const uint32_t idesc = idesc_f16(128, N);
  for (int ks = 0; ks < K / 16; ++ks)
    mma_ts_elect(tmem_d, tmem_a + (uint32_t)(ks * 8), b0 + (uint64_t)(ks * 16), idesc, ks > 0 ? 1u : 0u);
  commit_elect(bar);
}
__device__ __forceinline__ void layer_ss_warp(uint32_t tmem_d, const uint8_t* a_buf, const uint8_t* b_buf, int K,
                                              int N, uint64_t* bar) {
  const uint64_t a0 = sdesc(smem_u32(a_buf), 128, (uint32_t)K * 16), b0 = sdesc(smem_u32(b_buf), 128, (uint32_t)K * 16);
  const uint32_t idesc = idesc_f16(128, N);
  for (int ks = 0; ks < K / 16; ++ks)
    mma_ss_elect(tmem_d, a0 + (uint64_t)(ks * 16), b0 + (uint64_t)(ks * 16), idesc, ks > 0 ? 1u : 0u);
  commit_elect(bar);
}

}  // namespace tc
