// attn_sm100.cuh — paged prefill attention on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// One work item = (request i, kv head kh, M-tile of TQ = 128/g suffix tokens).  The g q-heads
// sharing kv head kh are packed as rows (row = token * g + head) so one 128-row tcgen05 tile
// covers TQ tokens x g heads (GQA packing).  KV tiles are 128 keys = 8 pages of 16 tokens,
// each page a [16][128] bf16 block of the caller's [C][Hkv][16][d] cache, fetched by TMA
// (two 64-column boxes per page, 128-byte swizzle).  Per KV tile:
//   S = Q K^T      tcgen05.mma kind::f16, A = Q (smem, K-major), B = K tile (smem, K-major),
//                  D in TMEM (fp32, 128 lanes x 128 columns, double buffered)
//   softmax        one warpgroup per Q tile, one TMEM lane (= one row) per thread: causal mask, running max with
//                  a lazy rescale (O is rescaled in TMEM only when the max grows by > 2^8), exp2,
//                  P written back as packed bf16 over the first 64 columns of its S in TMEM
//   O += P V       A = P (TMEM), B = V tile (smem, MN-major), D = O in TMEM
// K and V stream through separate smem rings (K is released right after QK, V after its
// last PV).  Two M-tiles share each CTA (see "work decomposition"): a KV tile both need is
// loaded once.  Warp roles (persistent CTA per SM, 384 threads): warp 0 = TMA producer for K,
// warp 3 = TMA producer for V, warp 1 = MMA issuer (warp-uniform, one elected lane), warp 2 =
// TMEM allocator, then TMA producer for Q, warps 4-11 = softmax + epilogue.  Hand-offs are mbarriers; MMA completion is signalled with
// tcgen05.commit; tcgen05.mma from one thread execute in order, which orders the reuse of S.
// Softmax runs on two warpgroups (warps 4-7 and 8-11) that split each tile's key columns.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include "il_internal.cuh"

namespace il {
namespace sm100 {

// IL_CHECKS builds (scripts/gpu_checks.sh; the pool refuses compute-sanitizer): every global index
// the attention kernels form is checked against its buffer's extent, a violation traps
#ifdef IL_CHECKS
#define IL_CHECK(cond) do { if (!(cond)) { printf("IL_CHECK failed %s:%d %s\n", __FILE__, __LINE__, #cond); __trap(); } } while (0)
#else
#define IL_CHECK(cond) do { } while (0)
#endif

#ifdef IL_ATTN_TRACE
// debug build only (build.py --trace): per-tile clock64 stamps of each role in CTA 0
__device__ unsigned long long g_trace[16][4096];
__device__ unsigned int g_trace_item[1024][4];
#define IL_TRACE(slot, idx) \
  do { if (blockIdx.x == 0 && phase == IL_TRACE_PHASE && (idx) < 4096) g_trace[slot][idx] = clock64(); } while (0)
#ifndef IL_TRACE_PHASE
#define IL_TRACE_PHASE 1
#endif
#else
#define IL_TRACE(slot, idx) do { } while (0)
#endif

constexpr uint32_t BM = 128;             // rows per M-tile
constexpr uint32_t BN = 128;             // keys per KV tile (= 8 pages) = one softmax step
constexpr uint32_t CB = 16384;           // one 64-column block of a 128-row bf16 tile
constexpr uint32_t KCB = CB;             // one 64-column block of a 128-key K/V tile
#ifndef IL_NSTK
#define IL_NSTK 3
#endif
#ifndef IL_NSTV
#define IL_NSTV 2
#endif
constexpr uint32_t NSTK = IL_NSTK, NSTV = IL_NSTV;   // K and V ring depths
// smem (per head dim DH, NCB = DH / 64 column blocks): Q pair [0, 2 QTILE), K ring at OFF_K
// (K[s] = OFF_K + s KVTILE), V ring at OFF_V, barriers at OFF_BAR; QTILE = KVTILE = NCB x 16 KB
__host__ __device__ constexpr uint32_t smem_bytes(uint32_t DH) { return (2 + NSTK + NSTV) * (DH / 64) * CB + 256; }
constexpr uint32_t NBAR = 16 + 2 * NSTK + 2 * NSTV;
constexpr int THREADS = 384;
// Softmax warpgroup x owns Q tile x (thread = one full 128-key row, no max exchange); the two
// tiles' softmaxes run concurrently, so one's row max / bookkeeping overlaps the other's
// exponentials.  (Round-1 history: both warpgroups splitting every tile's key columns with a
// row-max exchange through smem was 8% slower, git 11b8cd7.)
// IL_P_SPLIT = 1: P is released in two 64-key halves, so the first half's PV MMAs overlap the
// second half's exponentials.
#ifndef IL_P_SPLIT
#define IL_P_SPLIT 1
#endif
#ifndef IL_SETMAXNREG
#define IL_SETMAXNREG 1
#endif
#ifndef IL_REG_PROD
#define IL_REG_PROD 56
#endif
#ifndef IL_REG_SM
#define IL_REG_SM 224
#endif
// setmaxnreg.inc only completes when the CTA's pool (168 x 384 registers at launch) holds the
// requested registers: 4 warps x IL_REG_PROD + 8 x IL_REG_SM must not exceed 12 x 168, or the
// softmax warps wait forever
static_assert(4 * IL_REG_PROD + 8 * IL_REG_SM <= 12 * 168, "setmaxnreg split exceeds the register pool");
// producers / MMA issuer need few registers; the softmax warps hold a 128-column row
#if IL_SETMAXNREG
#define IL_REGS_DEC() asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(IL_REG_PROD))
#define IL_REGS_INC() asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(IL_REG_SM))
#else
#define IL_REGS_DEC() do { } while (0)
#define IL_REGS_INC() do { } while (0)
#endif

// Q_*, S_FULL, P_*, PV_DONE, O_* are per Q tile (stream) x: index + x
enum Bar : uint32_t { Q_FULL = 0, Q_FREE = 2, K_FULL = 4, K_FREE = K_FULL + NSTK, V_FULL = K_FREE + NSTK,
                      V_FREE = V_FULL + NSTV, S_FULL = V_FREE + NSTV, P_FULL = S_FULL + 2, PV_DONE = P_FULL + 2,
                      O_FULL = PV_DONE + 2, O_FREE = O_FULL + 2, P_HALF = O_FREE + 2 };
static_assert(P_HALF + 2 == NBAR, "barrier map");

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// try_wait with a suspend-time hint: the waiting warp sleeps until the phase completes (or the
// hint expires) instead of spinning and taking issue slots from the softmax warps on its SMSP.
#ifndef IL_WAIT_HINT_NS
#define IL_WAIT_HINT_NS 1000000
#endif
// A wait that has not completed after ~2^34 cycles (~9 s) traps (a launch error the host
// reports) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  long long t0 = 0;
  do {
    if (t0 == 0) t0 = clock64();
#ifdef IL_CHECKS
    else if (clock64() - t0 > (1ll << 32)) {
      printf("mbar_wait timeout: block %d thread %d bar smem+0x%x parity %u\n", blockIdx.x, threadIdx.x, bar, parity);
      __trap();
    }
#else
    else if (clock64() - t0 > (1ll << 34)) __trap();
#endif
#if IL_WAIT_HINT_NS > 0
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity), "n"(IL_WAIT_HINT_NS)
        : "memory");
#else
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
#endif
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
// L2 prefetch of a TMA box (no smem, no barrier): warms L2 for a later tma_load_3d
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"((uint64_t)map), "r"(c0), "r"(c1),
               "r"(c2)
               : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"((uint64_t)map), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// Warp-uniform variants: every lane of the warp executes them, one elected lane issues (keeps
// the operands in uniform registers: no per-instruction waterfall).
template <uint32_t IDESC>
__device__ __forceinline__ void mma_ss_w(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{ .reg .pred e, q; setp.ne.b32 q, %3, 0; elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, q; }" ::"r"(d_tmem), "l"(a), "l"(b), "r"(acc),
      "n"(IDESC)
      : "memory");
}
template <uint32_t IDESC>
__device__ __forceinline__ void mma_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t acc) {
  asm volatile(
      "{ .reg .pred e, q; setp.ne.b32 q, %3, 0; elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %4, q; }" ::"r"(d_tmem), "r"(a_tmem), "l"(b), "r"(acc),
      "n"(IDESC)
      : "memory");
}
__device__ __forceinline__ void commit_w(uint32_t bar) {
  asm volatile(
      "{ .reg .pred e; elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0]; }" ::"r"(bar)
      : "memory");
}
// A operand from TMEM (lane = row, 32-bit column = 2 consecutive bf16 along K)
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// 32 lanes x 32 consecutive fp32 columns: thread t of the warp gets its lane's 32 columns
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,"
      "%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  const uint32_t* r = reinterpret_cast<const uint32_t*>(v);
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st32u(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x for a PAIR on the FMA pipe (exp2 emulation, offloads the MUFU unit) with packed fp32x2 ops: magic-number
// rounding to j, cubic in f = x - j, 2^j added to the exponent field by one IMAD per element).
#ifndef IL_EXP_EMU_PAIRS
#define IL_EXP_EMU_PAIRS 0                           // bit (j/2) % 8 set: that pair emulated (0x4A, 3 of 8, was best with split softmax)
#endif
__device__ __forceinline__ void ex2_poly2(float x0, float x1, float& y0, float& y1) {
  x0 = fmaxf(x0, -125.f);
  x1 = fmaxf(x1, -125.f);
  uint32_t t0, t1, p0, p1;
  asm("{ .reg .b64 x, t, j, f, p, c, m, nm, k3, k2, k1, one;\n\t"
      "mov.b64 x, {%4, %5};\n\t"
      "mov.b64 m, {0f4B400000, 0f4B400000};\n\t"            // 1.5 * 2^23
      "mov.b64 nm, {0fCB400000, 0fCB400000};\n\t"
      "add.rn.f32x2 t, x, m;\n\t"                           // t = x + M (rounds x to an integer)
      "add.rn.f32x2 j, t, nm;\n\t"                          // j = t - M
      "mov.b64 c, {0fBF800000, 0fBF800000};\n\t"
      "fma.rn.f32x2 f, j, c, x;\n\t"                        // f = x - j in [-0.5, 0.5]
      "mov.b64 k3, {0f3D61FBB0, 0f3D61FBB0};\n\t"           // minimax cubic for 2^f on [-1/2, 1/2]
      "mov.b64 k2, {0f3E786F0F, 0f3E786F0F};\n\t"           // (relative error 7.5e-5)
      "mov.b64 k1, {0f3F31798D, 0f3F31798D};\n\t"
      "mov.b64 one, {0f3F7FFB49, 0f3F7FFB49};\n\t"
      "fma.rn.f32x2 p, f, k3, k2;\n\t"
      "fma.rn.f32x2 p, p, f, k1;\n\t"
      "fma.rn.f32x2 p, p, f, one;\n\t"
      "mov.b64 {%0, %1}, t;\n\t"
      "mov.b64 {%2, %3}, p; }"
      : "=r"(t0), "=r"(t1), "=r"(p0), "=r"(p1) : "f"(x0), "f"(x1));
  // the low mantissa bits of t hold j + 2^22 (mod 2^9); (t << 23) = j << 23 (mod 2^32)
  y0 = __uint_as_float(p0 + (t0 << 23));
  y1 = __uint_as_float(p1 + (t1 << 23));
}

// packed fp32x2 (FFMA2 / FADD2 on sm_100a): two elements per instruction
__device__ __forceinline__ void ffma2(float& o0, float& o1, float a0, float a1, float s, float m) {
  asm("{ .reg .b64 x, y, z, w; mov.b64 x, {%2, %3}; mov.b64 y, {%4, %4}; mov.b64 z, {%5, %5};\n\t"
      "fma.rn.f32x2 w, x, y, z; mov.b64 {%0, %1}, w; }"
      : "=f"(o0), "=f"(o1) : "f"(a0), "f"(a1), "f"(s), "f"(m));
}
__device__ __forceinline__ void fadd2(float& s0, float& s1, float a0, float a1) {
  asm("{ .reg .b64 x, y, w; mov.b64 x, {%0, %1}; mov.b64 y, {%2, %3};\n\t"
      "add.rn.f32x2 w, x, y; mov.b64 {%0, %1}, w; }"
      : "+f"(s0), "+f"(s1) : "f"(a0), "f"(a1));
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));   // low half = a
  return r;
}

// 256-bit global load / store (LDG.256 / STG.256 on sm_100a): a thread's 256-byte output row in
// 8 accesses instead of 16 -- the rows of a warp lie in 8-32 different lines, so every access is
// one L1 wavefront per lane group and halving their number halves the epilogue's LSU time
__device__ __forceinline__ void st_v8(void* p, const uint32_t (&v)[8]) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]),
               "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void ld_v8(const void* p, uint32_t (&v)[8]) {
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "l"(p));
}
// the same load as a plain (non-volatile) asm: the compiler may hoist and batch it, for data
// written by an earlier kernel (the phase-2 epilogue's partial rows)
__device__ __forceinline__ void ld_v8_nv(const void* p, uint32_t (&v)[8]) {
  asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
      : "l"(p));
}
// 32 fp32 values x inv -> 32 bf16 at p (64 bytes: two 256-bit stores)
__device__ __forceinline__ void store_row32(__nv_bfloat16* p, const float (&ov)[32], float inv) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint32_t w[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) w[e] = pack_bf16(ov[16 * h + 2 * e] * inv, ov[16 * h + 2 * e + 1] * inv);
    st_v8(p + 16 * h, w);
  }
}

// UMMA shared-memory descriptor (sm100): start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46),
// version 1 [46,48), layout SWIZZLE_128B = 2 [61,64).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor kind::f16: D f32 [4,6)=1, A bf16 [7,10)=1, B bf16 [10,13)=1,
// A major [15] (0 = K), B major [16] (1 = MN), N >> 3 [17,23), M >> 4 [24,29)
template <uint32_t DH>   // P V: A = P (K-major), B = V (MN-major), N = head dim
constexpr uint32_t IDESC_PV_T = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((DH >> 3) << 17) | ((BM >> 4) << 24);
constexpr uint32_t IDESC_QK = (1u << 4) | (1u << 7) | (1u << 10) | ((BN >> 3) << 17) | ((BM >> 4) << 24);

// ------------------------------------------------------------------ work decomposition
// M-tile t = (request i, tile mt of TQ tokens).  A work item is a PAIR of consecutive M-tiles
// (A = 2u, B = 2u+1) with one kv head.  Their KV tile sequences usually start with the same
// pages (the instruction and often the demonstrations, P:182 / PAIR rule 1), counted by nsh
// (k_pair_scan); a shared KV tile is loaded once and feeds both Q tiles.
struct Tile {
  uint32_t i, mt, P, S, r0, ntok, kv0, n_kv, nblk;
  bool valid;
};
// Cascade: NC = the leading 128-key KV tiles every request of the batch reads
// from the same cached pages (the instruction).  Phase 1 runs them once over DENSE
// M-tiles of all suffix rows of the batch (no padding between requests, no mask: every suffix
// position lies past the shared prefix).  Phase 2 runs FIRST: each request's own M-tiles over KV
// tiles NC.. (the causal part), leaving (O / l in `out`, m + log2 l in attn_ml); phase 1 starts
// each row from that partial (its items are long, so the extra load is amortised) and writes
// the result.  NC = 0: phase 2 alone is the whole attention.
__device__ __forceinline__ Tile decode_tile(const Ctx& c, const int32_t* __restrict__ cu_q,
                                            const int32_t* __restrict__ prefix_len, uint32_t t, uint32_t TQ,
                                            uint32_t phase, uint32_t NC) {
  Tile T;
  if (phase != 2) {                                     // phase 1 (or 3: phase 1 running first)
    T.valid = t < c.sc->n_dense;
    const uint32_t tot = c.sc->q_total;
    T.i = 0; T.mt = t; T.P = 0; T.r0 = 0; T.S = tot;
    T.ntok = T.valid ? min(TQ, tot - t * TQ) : 0;
    T.kv0 = 0; T.n_kv = T.valid ? NC : 0; T.nblk = 8 * NC;
    return T;
  }
  T.valid = t < c.sc->n_tiles;
  if (!T.valid) { T.i = T.mt = T.P = T.S = T.r0 = T.ntok = T.kv0 = T.n_kv = T.nblk = 0; return T; }
  const uint32_t i = c.tile_req[t];
  T.i = i;
  T.mt = t - c.tile_off[i];
  T.P = (uint32_t)prefix_len[i];
  T.r0 = (uint32_t)cu_q[i];
  T.S = (uint32_t)cu_q[i + 1] - T.r0;
  T.ntok = min(TQ, T.S - T.mt * TQ);
  T.kv0 = NC;
  T.n_kv = (T.P + T.mt * TQ + T.ntok - 1) / BN + 1 - NC;
  T.nblk = cdiv(T.P + T.S, BS);
  return T;
}
struct Pair {
  Tile a, b;
  uint32_t kh, nsh, nload;
};
__device__ __forceinline__ Pair decode_pair(const Ctx& c, const int32_t* __restrict__ cu_q,
                                            const int32_t* __restrict__ prefix_len, uint32_t w, uint32_t Hkv,
                                            uint32_t TQ, uint32_t phase, uint32_t NC) {
  Pair p;
  const uint32_t u = w / Hkv;
  p.kh = w % Hkv;
  p.a = decode_tile(c, cu_q, prefix_len, 2 * u, TQ, phase, NC);
  p.b = decode_tile(c, cu_q, prefix_len, 2 * u + 1, TQ, phase, NC);
  p.nsh = p.b.valid ? (phase != 2 ? NC : c.pair_nsh[u]) : 0;
  p.nload = p.a.n_kv + (p.b.valid ? p.b.n_kv - p.nsh : 0);
  return p;
}
// Load order: the nsh shared tiles (targets A and B), then the rest of A and of B interleaved
// (A, B, A, B, ...), then the longer remainder.  Returns the KV tile index, the request whose
// pages it reads, and the target mask (bit 0 = A, bit 1 = B).
__device__ __forceinline__ void load_info(const Pair& p, uint32_t l, uint32_t& n, uint32_t& req, uint32_t& tgt) {
  if (l < p.nsh) { n = l; req = p.a.i; tgt = 3; return; }
  const uint32_t ra = p.a.n_kv - p.nsh, rb = p.b.valid ? p.b.n_kv - p.nsh : 0;
  const uint32_t x = l - p.nsh, m = min(ra, rb);
  if (x < 2 * m) {
    const uint32_t j = x >> 1;
    if ((x & 1) == 0) { n = p.nsh + j; req = p.a.i; tgt = 1; } else { n = p.nsh + j; req = p.b.i; tgt = 2; }
    return;
  }
  const uint32_t j = m + (x - 2 * m);
  if (ra > rb) { n = p.nsh + j; req = p.a.i; tgt = 1; } else { n = p.nsh + j; req = p.b.i; tgt = 2; }
}

// One KV tile load of the CTA's load sequence: absolute KV tile kvt of request req (its block
// table row, nblk blocks), kv head kh, target mask tgt (bit x = Q tile / stream x), and per
// target stream whether this is the first / last load of the stream's current item and that
// item's index among the stream's items (barrier parities).
struct Load {
  uint32_t kvt, req, nblk, kh, tgt, first, last;
  uint32_t ix[2];
};
// The CTA's load sequence, walked identically by the K producer, the V producer and the MMA
// issuer.  Pair mode (phase 1): items are pairs (A, B) of one kv head and a KV tile both need is
// loaded once (load_info order).  Stream mode (phase 2, short items that share few tiles): the
// A tiles and the B tiles of the CTA's items are two independent streams whose loads alternate
// (A, B, A, B, ..., then the rest of the longer one), so one stream's item boundary (final PV,
// epilogue, next Q) never waits for the other stream's item to end.
struct LoadSeq {
  const Ctx* c;
  const int32_t* cu_q;
  const int32_t* prefix_len;
  uint32_t Hkv, TQ, phase, NC, n_items, stride;
  bool streams;
  uint32_t w, l, it, seen0, seen1;                     // pair mode
  Pair pr;
  uint32_t sw[2], sl[2], six[2], lastx;                 // stream mode
  Tile st[2];
  bool act[2];

  template <uint32_t X>
  __device__ __forceinline__ void seek() {
    while (sw[X] < n_items) {
      st[X] = decode_tile(*c, cu_q, prefix_len, 2 * (sw[X] / Hkv) + X, TQ, phase, NC);
      if (st[X].valid && st[X].n_kv > 0) break;
      sw[X] += stride;
    }
    act[X] = sw[X] < n_items;
    sl[X] = 0;
  }
  template <uint32_t X>
  __device__ __forceinline__ void stream_load(Load& L) {
    lastx = X;
    const Tile& T = st[X];
    L.kvt = T.kv0 + sl[X]; L.req = T.i; L.nblk = T.nblk; L.kh = sw[X] % Hkv; L.tgt = 1u << X;
    L.first = sl[X] == 0 ? L.tgt : 0u;
    L.last = sl[X] + 1 == T.n_kv ? L.tgt : 0u;
    L.ix[0] = six[0]; L.ix[1] = six[1];
    if (++sl[X] == T.n_kv) { ++six[X]; sw[X] += stride; seek<X>(); }
  }
  __device__ __forceinline__ void init(const Ctx* c_, const int32_t* cu_q_, const int32_t* prefix_len_, uint32_t Hkv_,
                                       uint32_t TQ_, uint32_t phase_, uint32_t NC_, uint32_t n_items_, bool streams_) {
    c = c_; cu_q = cu_q_; prefix_len = prefix_len_; Hkv = Hkv_; TQ = TQ_; phase = phase_; NC = NC_;
    n_items = n_items_; stride = gridDim.x; streams = streams_;
    if (streams) {
      sw[0] = sw[1] = blockIdx.x; six[0] = six[1] = 0;
      seek<0>(); seek<1>();
      lastx = 1;
    } else {
      w = blockIdx.x; l = 0; it = 0; seen0 = seen1 = 0;
      if (w < n_items) pr = decode_pair(*c, cu_q, prefix_len, w, Hkv, TQ, phase, NC);
    }
  }
  __device__ __forceinline__ bool next(Load& L) {
    if (streams) {
      // alternate A, B, A, B, ...; an exhausted stream leaves its turns to the other
      const bool pick1 = lastx == 0 ? act[1] : !act[0];
      if (pick1 ? !act[1] : !act[0]) return false;
      if (pick1) stream_load<1>(L); else stream_load<0>(L);
      return true;
    }
    if (w >= n_items) return false;
    uint32_t n, req, tgt;
    load_info(pr, l, n, req, tgt);
    L.kvt = pr.a.kv0 + n; L.req = req; L.nblk = req == pr.a.i ? pr.a.nblk : pr.b.nblk; L.kh = pr.kh; L.tgt = tgt;
    L.first = L.last = 0;
    if (tgt & 1u) { L.first |= seen0 == 0 ? 1u : 0u; L.last |= seen0 + 1 == pr.a.n_kv ? 1u : 0u; ++seen0; }
    if (tgt & 2u) { L.first |= seen1 == 0 ? 2u : 0u; L.last |= seen1 + 1 == pr.b.n_kv ? 2u : 0u; ++seen1; }
    L.ix[0] = L.ix[1] = it;    // (an invalid B tile only occurs in the CTA's last items)
    if (++l == pr.nload) {
      w += stride; ++it; l = 0; seen0 = seen1 = 0;
      if (w < n_items) pr = decode_pair(*c, cu_q, prefix_len, w, Hkv, TQ, phase, NC);
    }
    return true;
  }
  // a stream that has no further loads
  __device__ __forceinline__ bool done(uint32_t x) const { return streams && !act[x]; }
};
#ifndef IL_Q_PREFETCH
#define IL_Q_PREFETCH 1
#endif
#ifndef IL_KV_PREFETCH
#define IL_KV_PREFETCH 0      // (measured: 1 / 2 / 3 items ahead = 0.966 / 0.994 / 0.999 ms vs 0.886 off)
#endif
#ifndef IL_STREAMS
#define IL_STREAMS 0
#endif

template <uint32_t DH>
__global__ void __launch_bounds__(THREADS, 1)
    k_attn_sm100(Ctx c, uint32_t B, const int32_t* __restrict__ cu_q, const int32_t* __restrict__ prefix_len,
                 const int32_t* __restrict__ block_table, __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                 float scale_log2, uint32_t g, uint32_t TQ, uint32_t phase, const __grid_constant__ CUtensorMap tm_q,
                 const __grid_constant__ CUtensorMap tm_o,
                 const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v) {
  // head dim DH = 128 or 64: one 64-column (128-byte swizzle atom) block of Q / K / V per 64 dims
  constexpr uint32_t D = DH, NCB = DH / 64;
  constexpr uint32_t QTILE = NCB * CB, KVTILE = NCB * KCB;
  constexpr uint32_t OFF_QA = 0, OFF_K = 2 * QTILE, OFF_V = OFF_K + NSTK * KVTILE, OFF_BAR = OFF_V + NSTV * KVTILE;
    static_assert(DH == 64 || DH == 128, "head dim");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((smem_u32(smem) & 1023) != 0) __trap();          // swizzle atoms need 1024-byte alignment
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + OFF_BAR;
  auto bar = [&](uint32_t idx) { return bar0 + 8 * idx; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + NBAR * 8);

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t Hq = c.cfg.n_q_heads, Hkv = c.cfg.n_kv_heads;
  const uint32_t NC = c.sc->shared_blk / 8;
  // (phase 1 with NC = 0 has nothing to do: every item would have zero KV tiles)
  // phase: 2 = each request's own M-tiles over KV tiles NC.. (leaves a partial when NC > 0);
  // 1 = dense M-tiles over the NC shared tiles, continuing phase 2's partial; 3 = the same dense
  // pass running FIRST and leaving the partial (O / l in `out`, m + log2 l in attn_ml) that the
  // phase-2 kernel k_attn_p2 merges in its epilogue
  const uint32_t n_items = phase != 2 ? (NC ? cdiv(c.sc->n_dense, 2) * Hkv : 0u) : cdiv(c.sc->n_tiles, 2) * Hkv;
  const bool cascade = NC > 0;                          // phase 2 leaves a partial that phase 1 merges
  const bool streams = IL_STREAMS && phase == 2;

  if (threadIdx.x == 0) {
    for (uint32_t x = 0; x < 2; ++x) { mbar_init(bar(Q_FULL + x), 1); mbar_init(bar(Q_FREE + x), 1); }
    for (uint32_t s = 0; s < NSTK; ++s) { mbar_init(bar(K_FULL + s), 1); mbar_init(bar(K_FREE + s), 1); }
    static_assert(K_FREE == K_FULL + NSTK && V_FULL == K_FREE + NSTK && V_FREE == V_FULL + NSTV, "barrier map");
    for (uint32_t s = 0; s < NSTV; ++s) { mbar_init(bar(V_FULL + s), 1); mbar_init(bar(V_FREE + s), 1); }
    for (int x = 0; x < 2; ++x) {
      mbar_init(bar(S_FULL + x), 1); mbar_init(bar(P_FULL + x), 128);
      mbar_init(bar(PV_DONE + x), 1); mbar_init(bar(P_HALF + x), 128);
      mbar_init(bar(O_FULL + x), 1); mbar_init(bar(O_FREE + x), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm_q) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm_k) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm_v) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: S_A [0,128), S_B [128,256) (the P of a tile overwrites the first 64 columns
  // of its S as packed bf16), O_A [256,384), O_B [384,512).

  if (warp == 2) {
    // ============ Q producer, lane x = Q tile (stream) x: the tile of the stream's next item
    // loads as soon as the last QK of its current item has read Q (K / V run ahead independently)
    IL_REGS_DEC();
    if (lane < 2) {
      // Q rows live in HBM (the whole batch's Q exceeds L2): the stream's NEXT Q tile is
      // prefetched into L2 when the current one is loaded, so the load at the item boundary hits L2
      const uint32_t x = lane, qbytes = 2 * D * g * TQ;
      auto seek = [&](uint32_t& w, Tile& T) {
        for (; w < n_items; w += gridDim.x) {
          T = decode_tile(c, cu_q, prefix_len, 2 * (w / Hkv) + x, TQ, phase, NC);
          if (T.valid) break;
        }
      };
      uint32_t w = blockIdx.x, ix = 0;
      Tile T;
      seek(w, T);
      while (w < n_items) {
        uint32_t wn = w + gridDim.x;
        Tile Tn;
        seek(wn, Tn);
        if (ix >= 1) mbar_wait(bar(Q_FREE + x), (ix - 1) & 1);
        mbar_expect_tx(bar(Q_FULL + x), qbytes);
        const int row = (int)(T.r0 + T.mt * TQ), hq = (int)((w % Hkv) * g);
#pragma unroll
        for (uint32_t h = 0; h < NCB; ++h)
          tma_load_3d(sbase + OFF_QA + x * QTILE + h * CB, &tm_q, (int)(64 * h), hq, row, bar(Q_FULL + x));
        if (IL_Q_PREFETCH && wn < n_items) {
          const int rown = (int)(Tn.r0 + Tn.mt * TQ), hqn = (int)((wn % Hkv) * g);
#pragma unroll
          for (uint32_t h = 0; h < NCB; ++h) {
            tma_prefetch_3d(&tm_q, (int)(64 * h), hqn, rown);
            if (phase == 1) tma_prefetch_3d(&tm_o, (int)(64 * h), hqn, rown);   // the next item's partial
          }
          // phase 2 (profiling knob, off): the K / V pages of an item IL_KV_PREFETCH items ahead into
          // L2.  Slower at every distance: the loads are not what the MMA issuer waits for
          if (IL_KV_PREFETCH && phase == 2) {          // (IL_KV_PREFETCH = items ahead)
            uint32_t wp = wn;
            Tile Tp = Tn;
            for (int a = 1; a < IL_KV_PREFETCH && wp < n_items; ++a) { wp += gridDim.x; seek(wp, Tp); }
            const int32_t* btn = block_table + (size_t)Tp.i * c.max_blocks;
            const uint32_t khn = wp % Hkv;
            if (wp < n_items)
            for (uint32_t blk = Tp.kv0 * 8; blk < min(Tp.nblk, (Tp.kv0 + Tp.n_kv) * 8); ++blk) {
              const int row = (int)(((uint32_t)__ldg(btn + blk) * Hkv + khn) * BS);
#pragma unroll
              for (uint32_t h = 0; h < NCB; ++h) {
                tma_prefetch_2d(&tm_k, (int)(64 * h), row);
                tma_prefetch_2d(&tm_v, (int)(64 * h), row);
              }
            }
          }
        }
        ++ix;
        w = wn;
        T = Tn;
      }
    }
    __syncwarp();
  } else if (warp == 0 || warp == 3) {
    // ============ TMA producers: warp 0 = K tiles, warp 3 = V tiles ============
    IL_REGS_DEC();
    const bool is_k = warp == 0;
    const CUtensorMap* tm = is_k ? &tm_k : &tm_v;
    const uint32_t nst = is_k ? NSTK : NSTV;
    const uint32_t full0 = is_k ? K_FULL : V_FULL, free0 = is_k ? K_FREE : V_FREE;
    const uint32_t ring = sbase + (is_k ? OFF_K : OFF_V);
    LoadSeq seq;
    seq.init(&c, cu_q, prefix_len, Hkv, TQ, phase, NC, n_items, streams);
    Load L;
    for (uint32_t lc = 0; seq.next(L); ++lc) {
      const int32_t* bt = block_table + (size_t)L.req * c.max_blocks;
      IL_CHECK(L.req < B && L.kvt * 8 < c.max_blocks + 8);
      const uint32_t blk = L.kvt * 8 + (lane & 7);
      const int32_t page = blk < L.nblk ? __ldg(bt + blk) : __ldg(bt);
      const uint32_t s = lc % nst, u = lc / nst;
      if (lane == 0) {
        if (lc >= nst) mbar_wait(bar(free0 + s), (u - 1) & 1);
        IL_TRACE(is_k ? 0 : 1, lc & 4095);
#ifdef IL_NO_KV_TMA
        mbar_arrive(bar(full0 + s));                   // profiling variant: no K / V loads
#else
        mbar_expect_tx(bar(full0 + s), KVTILE);
#endif
      }
      __syncwarp();
#ifdef IL_NO_KV_TMA
      if (false) {
#else
      if (lane < 8 * NCB) {                            // lane = (page, 64-column block)
#endif
        const uint32_t p = lane & 7, h = lane >> 3;
        const int row = (int)(((uint32_t)page * Hkv + L.kh) * BS);
        tma_load_2d(ring + s * KVTILE + h * KCB + p * 2048, tm, (int)(64 * h), row, bar(full0 + s));
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer: warp-uniform loop, one elected lane issues ==============
    // Per Q tile x: S_x = Q_x K^T, then (after the softmax) O_x += P_x V.  S_x is single
    // buffered, so PV of a tile is issued right before the next QK of the same Q tile
    // (tcgen05 ops from one thread execute in order); the two Q tiles' chains interleave on
    // the tensor pipe.
    IL_REGS_DEC();
    const uint64_t dq0 = sdesc(sbase + OFF_QA, 16, 1024);
    const uint64_t dk0 = sdesc(sbase + OFF_K, 16, 1024), dv0 = sdesc(sbase + OFF_V, KCB, 1024);
    uint32_t cnt[2] = {0, 0};
    uint32_t vus = 0;                                 // 2-bit PV-user counters per load (lc % 8)
    // pending PV per Q tile: flag, load counter, tile count, last tile of its item
    uint32_t pn[2] = {0, 0}, pl[2] = {0, 0}, pc[2] = {0, 0}, pf[2] = {0, 0}, pix[2] = {0, 0};
    bool fst[2] = {true, true}, ordy[2] = {true, true};
    auto pv_one = [&](const uint32_t x) {
      const uint32_t vs = pl[x] % NSTV;
      if (!ordy[x]) { mbar_wait(bar(O_FREE + x), (pix[x] - 1) & 1); ordy[x] = true; }   // epilogue of the previous item
      mbar_wait(bar((IL_P_SPLIT ? P_HALF : P_FULL) + x), pc[x] & 1);
      mbar_wait(bar(V_FULL + vs), (pl[x] / NSTV) & 1);
      if (lane == 0) IL_TRACE(3, (2 * pl[x] + x) & 4095);
      tc_fence_after();
      const uint64_t dv = dv0 + (uint64_t)((vs * KVTILE) >> 4);
      const uint32_t o_tmem = tmem + 256 + 128 * x, p_tmem = tmem + 128 * x;
      // K = 128 keys in 8 steps of 16 (V tile rows; 16 keys = 2 swizzle atoms = 2048 B)
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k) {
        // IL_P_SPLIT: keys 0-63 of P are released first; their MMAs run while the softmax
        // computes keys 64-127
        if (IL_P_SPLIT && k == 4) { mbar_wait(bar(P_FULL + x), pc[x] & 1); tc_fence_after(); }
        mma_ts_w<IDESC_PV_T<DH>>(o_tmem, p_tmem + 8 * k, dv + (uint64_t)((k * 2048) >> 4), (fst[x] && k == 0) ? 0u : 1u);
      }
      fst[x] = false;
      commit_w(bar(PV_DONE + x));
      if (pf[x]) commit_w(bar(O_FULL + x));          // the item's last PV of this tile: epilogue may start
      const uint32_t sh = 2 * (pl[x] & 7);
      vus -= 1u << sh;
      if (((vus >> sh) & 3u) == 0) commit_w(bar(V_FREE + vs));
      pn[x] = 0;
    };
    LoadSeq seq;
    seq.init(&c, cu_q, prefix_len, Hkv, TQ, phase, NC, n_items, streams);
    Load L;
    for (uint32_t lc = 0; seq.next(L); ++lc) {
#pragma unroll
      for (uint32_t x = 0; x < 2; ++x)                 // a tile whose item has no more loads here drains its PV
        if (!((L.tgt >> x) & 1u) && pn[x] && pf[x] && (!streams || seq.done(x))) pv_one(x);
      const uint32_t ks = lc % NSTK;
      mbar_wait(bar(K_FULL + ks), (lc / NSTK) & 1);
      if (lane == 0) IL_TRACE(2, lc & 4095);
      tc_fence_after();
      const uint32_t sh = 2 * (lc & 7);
      vus = (vus & ~(3u << sh)) | ((uint32_t)__popc(L.tgt) << sh);
      const uint64_t dk = dk0 + (uint64_t)((ks * KVTILE) >> 4);
#pragma unroll
      for (uint32_t x = 0; x < 2; ++x) {
        if (!((L.tgt >> x) & 1u)) continue;
        if (pn[x]) pv_one(x);                          // frees the S/P columns this QK overwrites
        if ((L.first >> x) & 1u) {                     // a new item of this Q tile
          mbar_wait(bar(Q_FULL + x), L.ix[x] & 1);
          if (lane == 0 && x == 0) IL_TRACE(13, L.ix[0] & 4095);
          tc_fence_after();
          fst[x] = phase != 1;                         // phase 1 accumulates onto the partial
          ordy[x] = L.ix[x] == 0;
          pix[x] = L.ix[x];
        }
        const uint64_t dq = dq0 + (uint64_t)((x * QTILE) >> 4);
#pragma unroll
        for (uint32_t k = 0; k < D / 16; ++k)
          mma_ss_w<IDESC_QK>(tmem + 128 * x, dq + (uint64_t)(((k >> 2) * CB + (k & 3) * 32) >> 4),
                             dk + (uint64_t)(((k >> 2) * KCB + (k & 3) * 32) >> 4), k ? 1u : 0u);
        commit_w(bar(S_FULL + x));
        pn[x] = 1; pl[x] = lc; pc[x] = cnt[x]++; pf[x] = (L.last >> x) & 1u;
        if (pf[x]) commit_w(bar(Q_FREE + x));          // the item's last QK of this tile has read Q
      }
      commit_w(bar(K_FREE + ks));
    }
#pragma unroll
    for (uint32_t x = 0; x < 2; ++x)
      if (pn[x]) pv_one(x);
  } else if (warp >= 4) {
    // ====== softmax + epilogue, one warpgroup per Q tile: thread = row r of tile xo ======
    IL_REGS_INC();
    const uint32_t sm_t = threadIdx.x - 128, xo = sm_t >> 7, r = sm_t & 127, q4 = warp & 3;
    const uint32_t lane_addr = (32 * q4) << 16;
    const uint32_t s_tmem = tmem + lane_addr + 128 * xo, o_tmem = tmem + lane_addr + 256 + 128 * xo;
    uint32_t it = 0, cnt = 0;
    const uint32_t t = r / g, hh = r % g;
    // items are decoded one ahead (the decode's dependent loads stay off the item boundary)
    auto seek = [&](uint32_t& w, Tile& T) {
      for (; w < n_items; w += gridDim.x) {
        T = decode_tile(c, cu_q, prefix_len, 2 * (w / Hkv) + xo, TQ, phase, NC);
        if (T.valid) break;                            // (uniform over the warpgroup)
      }
    };
    uint32_t w = blockIdx.x;
    Tile T;
    seek(w, T);
    while (w < n_items) {
      const uint32_t kh = w % Hkv;
      const bool valid = (r < g * TQ) && (t < T.ntok);
      const uint32_t pos_q = T.P + T.mt * TQ + min(t, T.ntok - 1);
      const size_t orow = (size_t)(T.r0 + T.mt * TQ + t) * Hq + kh * g + hh;
      float m_used = -INFINITY, l = 0.f;
      if (phase == 1) {
        // continue phase 2's partial (m + log2 l, O / l) of these rows: state (m + log2 l, 1, O / l).
        // Warp-uniform (tcgen05.st is .aligned); padding rows store zeros.
        if (r == 0 && xo == 0) IL_TRACE(12, it & 4095);
        // (the rows were prefetched into L2 by the Q producer one item ahead)
        if (valid) { m_used = c.attn_ml[orow]; l = 1.f; }
        uint32_t raw[D / 16][8];
#pragma unroll
        for (int j = 0; j < (int)(D / 16); ++j) {
          if (valid) ld_v8(out + orow * D + 16 * j, raw[j]);
          else {
#pragma unroll
            for (int e = 0; e < 8; ++e) raw[j][e] = 0u;
          }
        }
#pragma unroll
        for (int q = 0; q < (int)(D / 32); ++q) {
          float ov[32];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const uint32_t u = raw[2 * q + (j >> 3)][j & 7];
            ov[2 * j] = __uint_as_float(u << 16);
            ov[2 * j + 1] = __uint_as_float(u & 0xFFFF0000u);
          }
          tmem_st32(o_tmem + 32 * q, ov);
        }
        tmem_wait_st();
        if (r == 0 && xo == 0) IL_TRACE(14, it & 4095);
      }
      for (uint32_t n = 0; n < T.n_kv; ++n) {        // this tile's KV tiles in load order
        mbar_wait(bar(S_FULL + xo), cnt & 1);
        if (r == 0) IL_TRACE(4 + 2 * xo, cnt & 4095);
        tc_fence_after();
#ifdef IL_NO_SOFTMAX
        {   // profiling variant: P = 0 without touching S (the MMA / TMA pipeline alone)
          uint32_t z[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) z[j] = 0u;
          tmem_st32u(s_tmem, z);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(bar(P_HALF + xo));
          tmem_st32u(s_tmem + 32, z);
          tmem_wait_st();
          tc_fence_before();
          if (r == 0) IL_TRACE(5 + 2 * xo, cnt & 4095);
          mbar_arrive(bar(P_FULL + xo));
          ++cnt;
          continue;
        }
#endif
        const uint32_t key0 = (T.kv0 + n) * BN;
        float a[128];
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_ld32(s_tmem + 32 * q, *reinterpret_cast<float(*)[32]>(&a[32 * q]));
        tmem_wait_ld();
        if (r == 0 && xo == 0) IL_TRACE(8, cnt & 4095);
        // causal mask: keys key0 + j with j >= nv are in this row's future.  Per 32-key chunk: all
        // valid (no work), all masked (constant), or the one boundary chunk (per-element select)
        // causal mask: keys key0 + j with j >= nv are in this row's future; 32-key chunks valid
        // for the whole warp need no select (warp-uniform branches)
        const int nv = (int)pos_q - (int)key0 + 1;
        if (phase == 2 && __any_sync(~0u, nv < (int)BN)) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (__all_sync(~0u, 32 * q + 32 <= nv)) continue;
#pragma unroll
            for (int j = 0; j < 32; ++j) a[32 * q + j] = 32 * q + j < nv ? a[32 * q + j] : -INFINITY;
          }
        }
        float mxa[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) mxa[q] = a[q];
#pragma unroll
        for (int j = 8; j < 128; ++j) mxa[j & 7] = fmaxf(mxa[j & 7], a[j]);
        const float mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                               fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
        if (r == 0 && xo == 0) IL_TRACE(9, cnt & 4095);
        const float mx2 = mx * scale_log2;
        bool need = false;
        float factor = 1.f;
        if (m_used == -INFINITY) {
          m_used = mx2;
        } else if (mx2 > m_used + 8.f) {
          need = true;
          factor = ex2(m_used - mx2);
          m_used = mx2;
          l *= factor;
        }
        if (__any_sync(~0u, need)) {
          // lazy rescale of this row's O once the previous tile's PV has landed
          mbar_wait(bar(PV_DONE + xo), (cnt - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int q = 0; q < (int)(D / 32); ++q) {
            float ov[32];
            tmem_ld32(o_tmem + 32 * q, ov);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) ov[j] *= factor;
            tmem_st32(o_tmem + 32 * q, ov);
          }
          tmem_wait_st();
        }
        // a fully masked row (no key yet) keeps p = 0: exp2(-inf - 0)
        const float negm = m_used == -INFINITY ? 0.f : -m_used;
        float rsa[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t pk[32];
#pragma unroll
          for (int jj = 0; jj < 64; jj += 2) {
            const int j = 64 * h + jj;
            float x0, x1;
            ffma2(x0, x1, a[j], a[j + 1], scale_log2, negm);
            float p0, p1;
            if ((IL_EXP_EMU_PAIRS >> ((j >> 1) & 7)) & 1) {
              ex2_poly2(x0, x1, p0, p1);
            } else {
              p0 = ex2(x0);
              p1 = ex2(x1);
            }
            fadd2(rsa[(j >> 1) & 2], rsa[((j >> 1) & 2) + 1], p0, p1);
            pk[jj >> 1] = pack_bf16(p0, p1);
          }
          // P (bf16 pairs) of keys [64h, 64h + 64) -> TMEM columns [32h, 32h + 32) of this S
          tmem_st32u(s_tmem + 32 * h, pk);
          if (IL_P_SPLIT && h == 0) {                    // first half of P -> its PV MMAs may start
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(bar(P_HALF + xo));
          }
        }
        l += (rsa[0] + rsa[1]) + (rsa[2] + rsa[3]);
        if (r == 0 && xo == 0) IL_TRACE(10, cnt & 4095);
        tmem_wait_st();
        if (r == 0 && xo == 0) IL_TRACE(11, cnt & 4095);
        tc_fence_before();
        if (r == 0) IL_TRACE(5 + 2 * xo, cnt & 4095);
        mbar_arrive(bar(P_FULL + xo));
        ++cnt;
      }
      uint32_t wn = w + gridDim.x;                     // decode the next item while the last PV runs
      Tile Tn;
      seek(wn, Tn);
      // epilogue: O / l -> bf16 row of `out`, natural-log LSE (or the phase-2 partial)
      mbar_wait(bar(O_FULL + xo), it & 1);
      tc_fence_after();
      {
        const float inv = 1.f / l;
#pragma unroll
        for (int q = 0; q < (int)(D / 32); ++q) {
          float ov[32];
          tmem_ld32(o_tmem + 32 * q, ov);
          tmem_wait_ld();
          if (valid) {
            IL_CHECK(orow < (size_t)c.sc->q_total * Hq);
            store_row32(out + orow * D + 32 * q, ov, inv);
          }
        }
        if (valid) {
          if ((phase == 2 && cascade) || phase == 3) c.attn_ml[orow] = m_used + __log2f(l);
          else if (lse) lse[orow] = (m_used + __log2f(l)) * 0.69314718055994531f;
        }
      }
      tc_fence_before();
      if (r == 0 && xo == 0) IL_TRACE(15, it & 4095);  // epilogue done
      mbar_arrive(bar(O_FREE + xo));
      ++it;
      w = wn;
      T = Tn;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// k_pair_scan: for every pair of consecutive M-tiles, how many leading KV tiles read the same
// 8 pages for both (one warp per pair).
__global__ void __launch_bounds__(256) k_pair_scan(Ctx c, const int32_t* __restrict__ cu_q,
                                                   const int32_t* __restrict__ prefix_len,
                                                   const int32_t* __restrict__ block_table, uint32_t TQ) {
  const uint32_t lane = threadIdx.x & 31, nt = c.sc->n_tiles, NC = c.sc->shared_blk / 8;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < cdiv(nt, 2);
       u += (gridDim.x * blockDim.x) >> 5) {
  const Tile A = decode_tile(c, cu_q, prefix_len, 2 * u, TQ, 2, NC);
  const Tile Bt = decode_tile(c, cu_q, prefix_len, 2 * u + 1, TQ, 2, NC);
  uint32_t nsh = 0;
  if (Bt.valid) {
    const uint32_t ntile = min(A.n_kv, Bt.n_kv);
    const int32_t* ba = block_table + (size_t)A.i * c.max_blocks;
    const int32_t* bb = block_table + (size_t)Bt.i * c.max_blocks;
    // tile n is shared iff its 8 page ids agree (blocks past a request's end read page bt[0])
    uint32_t n = 0;
    for (; n < ntile; n += 4) {
      const uint32_t tn = n + (lane >> 3), blk = (NC + tn) * 8 + (lane & 7);
      bool eq = true;
      if (tn < ntile) {
        const int32_t pa = blk < A.nblk ? ba[blk] : ba[0], pb = blk < Bt.nblk ? bb[blk] : bb[0];
        eq = pa == pb;
      }
      const uint32_t bad = __ballot_sync(~0u, !eq);
      if (bad) { n += (__ffs(bad) - 1) >> 3; break; }
    }
    nsh = min(n, ntile);
  }
  if (lane == 0) c.pair_nsh[u] = nsh;
  }
}

// k_shared_scan: blocks every request shares with request 0 (same page ids, within both hit
// ranges); sc->shared_blk starts at request 0's hit count (k_tile_scan).  Warp per request.
__global__ void __launch_bounds__(256) k_shared_scan(Ctx c, uint32_t B, const int32_t* __restrict__ prefix_len,
                                                     const int32_t* __restrict__ block_table) {
  const uint32_t lane = threadIdx.x & 31;
  const int32_t* b0 = block_table;
  for (uint32_t i = 1 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < B; i += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t lim = min((uint32_t)prefix_len[i] / BS, *(volatile uint32_t*)&c.sc->shared_blk);
    const int32_t* bi = block_table + (size_t)i * c.max_blocks;
    uint32_t n = 0;
    for (; n < lim; n += 32) {
      const uint32_t b = n + lane;
      const bool ne = b < lim && bi[b] != b0[b];
      const uint32_t bad = __ballot_sync(~0u, ne);
      if (bad) { n += __ffs(bad) - 1; break; }
    }
    // n = blocks shared with request 0 (<= lim).  Also when every block up to lim matched, a
    // request whose hits end before the current bound lowers it to its own hit count: otherwise
    // its M-tiles would start inside the shared range (zero phase-2 KV tiles: a hang)
    n = min(n, lim);
    if (lane == 0 && n < *(volatile uint32_t*)&c.sc->shared_blk) atomicMin(&c.sc->shared_blk, n);
  }
}

}  // namespace sm100
}  // namespace il

#include "attn_p2.cuh"
#include "attn_dense2.cuh"

namespace il {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// decode: one row per request (cu_q = 0, 1, .., B; il_decode_attn): each request's own keys run on
// CUDA cores (k_decode_own, decode_dev.cuh) instead of tensor phase 2; phase 1 is unchanged.
static inline il_status attn_sm100_launch(Ctx* c, uint32_t B, const int32_t* cu_q, const int32_t* prefix_len,
                                          const int32_t* block_table, const il_bf16* q, il_bf16* k_pages,
                                          il_bf16* v_pages, il_bf16* out, float* lse, float scale, cudaStream_t st,
                                          bool decode = false) {
  using namespace sm100;
  const uint32_t Hq = c->cfg.n_q_heads, Hkv = c->cfg.n_kv_heads, g = Hq / Hkv, TQ = BM / g, D = c->cfg.head_dim;
  auto enc = encode_fn();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable"); return IL_ERR_CUDA; }
  CUtensorMap tq, to, tk, tv;
  for (int which = 0; which < 2; ++which) {            // Q, and `out` (same geometry: L2 prefetch only)
    cuuint64_t dims[3] = {D, Hq, decode ? (cuuint64_t)B : (cuuint64_t)c->cfg.max_suffix_tokens};
    cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)Hq * D * 2};
    cuuint32_t box[3] = {64, g, TQ};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(which ? &to : &tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, which ? (void*)out : (void*)q, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { set_error("tensor map (q / out) encode failed"); return IL_ERR_CUDA; }
  }
  for (int which = 0; which < 2; ++which) {
    cuuint64_t dims[2] = {D, (cuuint64_t)c->cfg.kv_pages * Hkv * BS};
    cuuint64_t strides[1] = {(cuuint64_t)D * 2};
    cuuint32_t box[2] = {64, BS};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(which ? &tv : &tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, which ? (void*)v_pages : (void*)k_pages,
                     dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { set_error("tensor map (kv) encode failed"); return IL_ERR_CUDA; }
  }
  const char* ce = getenv("IL_CASCADE");
  const bool cascade = !(ce && ce[0] == '0');
  // phase 2 on the 64-key double-buffered-S kernel (attn_p2.cuh); IL_P2=0 keeps it on
  // k_attn_sm100 (the round-2 path, A / B comparisons)
  const char* pe = getenv("IL_P2");
  const bool p2 = !(pe && pe[0] == '0');
  // IL_DENSE_P2=1: the dense pass on k_attn_p2<DH, true> (64-key double-buffered S, shared K / V
  // rings) instead of k_attn_sm100 phase 3 -- measured slower, 644 vs 512 us
  const char* pd = getenv("IL_DENSE_P2");
  const bool dense_old = !(pd && pd[0] == '1');
  // IL_DENSE2=1: the dense pass on the CTA-pair kernel (attn_dense2.cuh; head dim 128)
  const char* pd2 = getenv("IL_DENSE2");
  const bool dense2 = pd2 && pd2[0] == '1' && D == 128;
  k_tile_scan<<<1, 1024, 0, st>>>(*c, B, cu_q, prefix_len, TQ, cascade ? 1u : 0u);
  if (cascade && B > 1) k_shared_scan<<<c->num_sms * 2, 256, 0, st>>>(*c, B, prefix_len, block_table);
  if (!decode && !p2) k_pair_scan<<<c->num_sms * 4, 256, 0, st>>>(*c, cu_q, prefix_len, block_table, TQ);
  const int grid = c->attn_ctas ? c->attn_ctas : c->num_sms;   // (il_set_sm_split)
  if (decode) {
    const uint32_t G2 = g <= 1 ? 1 : g <= 2 ? 2 : g <= 4 ? 4 : 8;
    const dim3 dg(B * Hkv), db(DEC_WARPS * 32);
    const float sl2 = scale * 1.4426950408889634f;
    const __nv_bfloat16 *qq = (const __nv_bfloat16*)q, *kp = (const __nv_bfloat16*)k_pages,
                        *vp = (const __nv_bfloat16*)v_pages;
    __nv_bfloat16* oo = (__nv_bfloat16*)out;
#define IL_DEC(DD, GG) k_decode_own<DD, GG><<<dg, db, 0, st>>>(*c, B, prefix_len, block_table, qq, kp, vp, oo, lse, sl2)
    if (D == 128) {
      if (G2 == 1) IL_DEC(128, 1); else if (G2 == 2) IL_DEC(128, 2); else if (G2 == 4) IL_DEC(128, 4); else IL_DEC(128, 8);
    } else {
      if (G2 == 1) IL_DEC(64, 1); else if (G2 == 2) IL_DEC(64, 2); else if (G2 == 4) IL_DEC(64, 4); else IL_DEC(64, 8);
    }
#undef IL_DEC
    IL_LAUNCH_CHECK("k_decode_own");
  }
  // phase order: with k_attn_p2, the dense pass over the shared prefix runs first (phase 3) and
  // k_attn_p2 merges its partial in the epilogue; otherwise (decode, IL_P2=0) each request's own
  // part runs first and the dense pass continues it (phase 1)
  const bool p1_first = p2 && !decode;
  for (uint32_t phase : {p1_first ? 3u : 2u, p1_first ? 2u : 1u}) {
    if (phase == 2 && decode) continue;
    if ((phase == 1 || phase == 3) && !cascade) continue;
    if (phase == 3 && dense2) {
      d2::k_attn_dense2<128><<<grid & ~1, THREADS, d2::SMEM, st>>>(*c, block_table, (__nv_bfloat16*)out,
                                                                 scale * 1.4426950408889634f, g, TQ, tq, tk, tv);
      IL_LAUNCH_CHECK("k_attn_dense2");
      continue;
    }
    // phase 2, and (IL_DENSE_P2=1) the dense pass too, on k_attn_p2
    if ((phase == 2 && p2) || (phase == 3 && !dense_old)) {
      const float sl2 = scale * 1.4426950408889634f;
      __nv_bfloat16* o16 = (__nv_bfloat16*)out;
      if (D == 128) {
        if (phase == 3) p2::k_attn_p2<128, true><<<grid, p2::THREADS2, p2::smem_bytes2<128>, st>>>(*c, B, block_table, o16, lse, sl2, g, TQ, tq, to, tk, tv);
        else p2::k_attn_p2<128, false><<<grid, p2::THREADS2, p2::smem_bytes2<128>, st>>>(*c, B, block_table, o16, lse, sl2, g, TQ, tq, to, tk, tv);
      } else {
        if (phase == 3) p2::k_attn_p2<64, true><<<grid, p2::THREADS2, p2::smem_bytes2<64>, st>>>(*c, B, block_table, o16, lse, sl2, g, TQ, tq, to, tk, tv);
        else p2::k_attn_p2<64, false><<<grid, p2::THREADS2, p2::smem_bytes2<64>, st>>>(*c, B, block_table, o16, lse, sl2, g, TQ, tq, to, tk, tv);
      }
      IL_LAUNCH_CHECK("k_attn_p2");
      continue;
    }
    if (D == 128)
      k_attn_sm100<128><<<grid, THREADS, smem_bytes(128), st>>>(*c, B, cu_q, prefix_len, block_table,
          (__nv_bfloat16*)out, lse, scale * 1.4426950408889634f, g, TQ, phase, tq, to, tk, tv);
    else
      k_attn_sm100<64><<<grid, THREADS, smem_bytes(64), st>>>(*c, B, cu_q, prefix_len, block_table,
          (__nv_bfloat16*)out, lse, scale * 1.4426950408889634f, g, TQ, phase, tq, to, tk, tv);
    IL_LAUNCH_CHECK("k_attn_sm100");
  }
  // k_tile_scan, k_shared_scan (cascade, B > 1), k_pair_scan (old phase 2) or k_decode_own, the two phases
  c->launches += 1 + (cascade && B > 1 ? 1 : 0) + (decode || !p2 ? 1 : 0) + (decode ? 0u : 1u) + (cascade ? 1 : 0);
  return IL_OK;
}

}  // namespace il
