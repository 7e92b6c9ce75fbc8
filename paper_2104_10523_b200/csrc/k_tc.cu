// a7 (tensor-core path): complex64 contraction-as-GEMM on 5th-generation tensor cores,
// error-compensated split-TF32 ("3xTF32") with round-to-nearest splits.
//
// Paper: the A100 TF32 tensor-core runs of the Sycamore amplitude (Table 2)
// lost accuracy ("correct to 3 decimal digits").  Here each fp32 operand x is
// split on chip into hi = rna_tf32(x), lo = rna_tf32(x - hi) and the product is
// accumulated as hi*hi + hi*lo + lo*hi in fp32 (TMEM), which keeps complex64-class
// accuracy (SURVEY §7 hard part 2, E8/E15).
//
// Complex arithmetic as one real GEMM (interleaved complex64, "real block form"):
//   X viewed as fp32 [N][2K] (re, im interleaved along K),
//   W[2k+a][2m+b] = [[Yr, Yi], [-Yi, Yr]][a][b] for complex Y(k, m),
//   C viewed as fp32 [N][2M] = X * W  (re, im interleaved along M) -- so C comes out in
//   the same interleaved complex64 layout as X, with no planar split in HBM.
// tcgen05 form: D[128 rows][BN] += A[128][8] * B[BN][8]^T per MMA (kind::tf32, K-major
// A and B, fp32 accumulators in TMEM).  A = X tile (TMA, 128B swizzle, split in place
// by converter warps), B = W^T hi/lo tiles built once per step by a prep kernel.
//
// CTA (persistent, one per SM -- or one CTA pair per TPC -- 512 threads):
//   warp 0      TMA producer (X chunk + W^T hi + W^T lo per stage, one mbarrier)
//   warp 1      TMEM allocator + single-thread MMA issuer (12 MMAs per 32-wide K chunk)
//   warps 2-3   gather producer (X not K-contiguous: 16-byte cp.async pieces)
//   warps 4-7   converters: fp32 -> (hi in place, lo to a second buffer), fence.proxy.async
//   warps 8-15  epilogue: tcgen05.ld (32x32b) -> registers -> swizzled smem -> TMA bulk store
// Pipelines: stage ring full/conv/empty mbarriers; double-buffered TMEM accumulators.
//
// Batched (a9): one launch runs the step for nb units (slices / bitstrings).  Items are
// unit-major; each CTA takes a contiguous block of items, so the unit changes rarely; the
// X, W^T and C tensor maps carry a unit dimension.  The per-unit arithmetic does not
// depend on nb: the K flush groups are fixed by K, and a split-K launch splits exactly at
// flush-group boundaries and adds the group partials in the same fp32 order as the
// unsplit kernel's TMEM running total, so split or not gives bit-identical results.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"
#include "pdl.cuh"

namespace tnqvm {
namespace dev {
namespace {

constexpr int kBM = 128;        // rows per tile (MMA M)
constexpr int kBKf = 32;        // fp32 per K chunk (128 bytes = one swizzle atom row)
constexpr int kThreadsTC = 512;
constexpr int kConvWarp0 = 4;   // converters: warps 4..7
constexpr int kEpiWarp0 = 8;    // epilogue: warps 8..15 (two per TMEM lane quarter)
constexpr int kEpiWarps = 8;

struct TcParams {
  int64_t N;       // rows per unit
  int K2;          // fp32 columns of X (= 2K)
  int M2;          // fp32 columns of C (= 2M)
  int BN;          // fp32 columns per tile (MMA N), multiple of 16, <= 256
  int n_col_tiles, n_row_tiles, k_splits, chunks_per_split, n_chunks;
  int group_chunks;  // K chunks accumulated in one TMEM partial before a round-to-nearest flush
  int longk;         // K beyond kLongKChunks chunks: a fixed split of kLongKChunks chunks per item (shape
                     // only), the split partials added in fp64 (accuracy over thousands of groups)
  int nbuf;          // TMEM partial buffers (2; 1 when BN=256 flushes: partial + total fill 512 columns)
  int stages;
  int nb;                  // units of the launch (item = unit-major, then k split, row tile, column tile)
  int64_t items_per_unit;  // n_row_tiles * n_col_tiles * k_splits
  int64_t n_items;         // nb * items_per_unit
  uint32_t idesc;
  uint32_t tmem_cols;
  int boxw;         // fp32 columns per TMA store box (32, or M2 < 32)
  int wres;         // 1: the whole W^T hi/lo of the (single) column tile stays resident in smem,
                    // reloaded when the CTA's next item belongs to another unit
  int tsa;          // 1 (single CTA, streamed W^T, BN <= 128): the A operand (X hi/lo) lives in TMEM --
                    // the converters tcgen05.st it there and the MMAs read [a_tmem]; no X hi/lo in
                    // shared memory (the 3xTF32 kernel is shared-memory-bandwidth bound)
  int sa, acol;     // tsa: TMEM A stages (64 columns each: hi | lo) starting at column acol
  int nstg;         // staging buffers per epilogue warp (1..4)
  int xb;           // 1: the X map has a unit dimension (each unit its own X); 0: all units read one X
  int gather;       // 1: X tiles gathered with cp.async by warps 2-3 (any layout with a contracted fastest mode)
  // gbox (TMEM-A steps): a gather step whose tile bits (7 row bits, 4 k bits) fall into <= 5
  // runs of contiguous strides: one TMA box per stage (tm_x: up to 5 dims, box = the tile)
  // lands the tile in box order; the converters read row r, k pair j at rowoff(r) + koff(j)
  // (gb_rs / gb_ks: smem byte strides of row bits 0-6 and k bits 1-3) instead of the
  // canonical SW128 position
  int gbox, gb_ndim, gb_udim, gb_us;
  int8_t gb_nd[33], gb_ns[33];  // row bits 7..: TMA dim and bit position inside it
  int8_t gb_kd[16], gb_ks_[16];  // k bits 4..: TMA dim and bit position inside it
  uint32_t gb_rs[7], gb_ks[3];
  int nn, nk;
  const float2* Xg;  // gather: unit 0's X; unit b's at + b * xbs elements
  int64_t xbs;
  int64_t sxn[40], sxk[40];
  // wbuild: resident W^T hi/lo built in shared memory by the epilogue warps straight from
  // the small operand Y (per-bit strides), instead of a prep kernel + TMA loads
  int wbuild, nm;
  const float2* Yg;         // unit 0's Y
  const int64_t* ydelta;    // unit b's Y at Yg + ydelta[b] (null: one unit)
  int64_t syk[20], sym[16];
};

// ---------------- PTX helpers ----------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2,
                                            int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until at most n of this thread's bulk stores still read shared memory (n = staging buffers - 1)
__device__ __forceinline__ void bulk_wait_read(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory"); break;
  }
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// every thread of the CTA (warps may be diverged: the non-.aligned barrier)
__device__ __forceinline__ void cta_bsync() { asm volatile("barrier.sync 3, %0;" ::"n"(kThreadsTC) : "memory"); }
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// CTA-pair (cta_group::2) helpers
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the mbarrier at the same shared offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t rank) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(rank)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {  // both CTAs' barriers at this offset
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tc_mma_tf32_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_mma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// K-major, 128-byte swizzle, 8-row core groups 1024 bytes apart (SBO), LBO unused (1).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;            // leading byte offset (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // stride byte offset
  d |= (uint64_t)1 << 46;            // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;            // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ bool elect_one() {  // one lane of the (converged) warp
  uint32_t r;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(r));
  return r != 0;
}
__device__ __forceinline__ uint32_t cvt_rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
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
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
      "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
      "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// ---------------- the GEMM kernel ----------------
// kCG = 1: one CTA per 128-row tile.  kCG = 2 (CTA pair, cluster of 2 on one TPC): the pair
// owns a 256-row tile; each CTA stages its own 128 X rows and HALF of the W^T tile (BN/2
// rows), the leader issues tcgen05.mma.cta_group::2 (M = 256) and commits to both CTAs'
// barriers -- per SM the shared-memory operand traffic of the MMAs drops by a third and the
// W^T TMA bytes by half (the single-CTA kernel is shared-memory-bandwidth bound).
template <int kCG>
__global__ void __launch_bounds__(kThreadsTC, 1)
    tc_gemm_kernel_t(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_bhi,
                   const __grid_constant__ CUtensorMap tm_blo, const __grid_constant__ CUtensorMap tm_c,
                   TcParams p) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned carve-up
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  const int S = p.stages;
  const uint32_t xbytes = kBM * kBKf * 4;          // 16 KB
  const uint32_t bbytes = (uint32_t)(p.BN / kCG) * kBKf * 4;  // this CTA's W^T rows per stage
  const uint32_t xlo_bytes = p.tsa ? 0u : xbytes;  // tsa: X hi/lo go to TMEM, not shared memory
  const uint32_t stage_bytes = xbytes + xlo_bytes + (p.wres ? 0u : 2 * bbytes);
  uint8_t* wres = base + (size_t)S * stage_bytes;      // resident W^T: per chunk [hi | lo]
  const size_t wres_bytes = p.wres ? (size_t)p.n_chunks * 2 * bbytes : 0;
  uint8_t* staging = wres + wres_bytes;  // per epilogue warp nstg x [32 rows][boxw fp32], 1024-aligned
  const uint32_t stg_bytes = 32u * p.boxw * 4;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + (size_t)kEpiWarps * p.nstg * stg_bytes);
  uint64_t* full = bars;            // [S]  TMA landed
  uint64_t* conv = bars + S;        // [S]  converters done
  uint64_t* empty = bars + 2 * S;   // [S]  MMAs consumed the stage
  uint64_t* tfull = bars + 3 * S;   // [2]  accumulator ready
  uint64_t* tempty = bars + 3 * S + 2;  // [2] accumulator drained
  uint64_t* wfull = bars + 3 * S + 4;  // resident W landed (one phase per unit the CTA visits)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 5);
  uint64_t* aempty = bars + 3 * S + 6;  // [sa] tsa: MMAs consumed the TMEM A stage

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t crank = 0;
  if constexpr (kCG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const bool leader = crank == 0;
  // this CTA's (pair's) contiguous block of items [it_lo, it_hi)
  const int64_t U = kCG == 2 ? (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;
  const int64_t uidx = kCG == 2 ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
  const int64_t it_lo = p.n_items * uidx / U, it_hi = p.n_items * (uidx + 1) / U;
  auto row0 = [&](int64_t rt) { return rt * (kBM * kCG) + (int64_t)crank * kBM; };  // this CTA's first row
  if (threadIdx.x == 0) {
    // full[s]: TMA thread (expect_tx) and/or the 64 gather threads (cp.async arrive)
    const uint32_t full_count = p.gather ? (64u + (p.wres ? 0u : 1u)) : 1u;
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], full_count);
      mbar_init(&conv[s], kCG == 2 ? 2 * 4 : 128);  // pair: one arrival per converter warp of each CTA
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kCG == 2 ? 2 * kEpiWarps : 32 * kEpiWarps);
    }
    mbar_init(wfull, p.wbuild ? 32u * kEpiWarps : 1u);
    for (int a = 0; a < p.sa; ++a) mbar_init(&aempty[a], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_x)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_bhi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_blo)) : "memory");
  }
  if (warp == 1) {
    if constexpr (kCG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(p.tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(p.tmem_cols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kCG == 2) cluster_sync_all();  // the peer's barriers are initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto stage_x = [&](int s) { return base + (size_t)s * stage_bytes; };
  auto stage_xlo = [&](int s) { return base + (size_t)s * stage_bytes + xbytes; };
  auto stage_bhi = [&](int s) { return base + (size_t)s * stage_bytes + xbytes + xlo_bytes; };
  auto stage_blo = [&](int s) { return base + (size_t)s * stage_bytes + xbytes + xlo_bytes + bbytes; };
  auto wres_hi = [&](int c) { return wres + (size_t)c * 2 * bbytes; };
  auto wres_lo = [&](int c) { return wres + (size_t)c * 2 * bbytes + bbytes; };

  // item -> (unit, row tile, col tile, k split): unit slowest, columns fastest (the X row
  // tile is reused from L2).  32-bit fast paths: a 64-bit division costs ~100 instructions
  // on every role's item loop.
  const bool small_items = p.n_items < ((int64_t)1 << 31);
  auto decode = [&](int64_t item, int& ub, int64_t& rt, int& ct, int& ks) {
    int64_t loc;
    if (small_items) {
      const uint32_t it = (uint32_t)item, ipu = (uint32_t)p.items_per_unit;
      ub = (int)(it / ipu);
      loc = (int64_t)(it - (uint32_t)ub * ipu);
    } else {
      ub = (int)(item / p.items_per_unit);
      loc = item - (int64_t)ub * p.items_per_unit;
    }
    if (p.n_col_tiles == 1 && p.k_splits == 1) {
      ct = 0;
      ks = 0;
      rt = loc;
    } else if (small_items) {
      const uint32_t it = (uint32_t)loc, nct = (uint32_t)p.n_col_tiles, nrt = (uint32_t)p.n_row_tiles;
      const uint32_t r = it / nct;
      ct = (int)(it - r * nct);
      const uint32_t k = r / nrt;
      rt = (int64_t)(r - k * nrt);
      ks = (int)k;
    } else {
      ct = (int)(loc % p.n_col_tiles);
      int64_t r = loc / p.n_col_tiles;
      rt = r % p.n_row_tiles;
      ks = (int)(r / p.n_row_tiles);
    }
  };
  auto chunk_range = [&](int ks, int& c0, int& c1) {
    c0 = ks * p.chunks_per_split;
    c1 = min(p.n_chunks, c0 + p.chunks_per_split);
  };
  // resident W^T (wres): before the first item of each unit the CTA visits, every thread
  // passes one CTA barrier (all MMAs of the previous unit have completed: the epilogue has
  // drained their accumulators), then the W^T of the new unit is loaded / built
  auto unit_change = [&](int ub, int& cur) -> bool {
    if (!p.wres || ub == cur) return false;
    if (cur >= 0) cta_bsync();
    cur = ub;
    return true;
  };
  auto idle = [&]() {  // threads without a role still pass the unit-change barriers
    if (!p.wres) return;
    int cur = -1;
    for (int64_t item = it_lo; item < it_hi; ++item) {
      int ub, ct, ks;
      int64_t rt;
      decode(item, ub, rt, ct, ks);
      unit_change(ub, cur);
    }
  };

  if (warp == 0) {
    // ===== TMA producer =====
    // the whole warp runs the loop; lane 0 issues.  gbox: lane i adds the coordinate of row-tile
    // bit i (then of chunk bit i) and one warp reduction per TMA dimension sums them
    int s = 0, cur = -1;
    uint32_t ph = 0;
    const int nrb = p.gbox ? p.nn - 7 : 0, nkb = p.gbox ? p.nk - 4 : 0;
    const int rb_d = lane < nrb ? p.gb_nd[lane] : -1, rb_v = lane < nrb ? 1 << p.gb_ns[lane] : 0;
    const int kb_d = lane < nkb ? p.gb_kd[lane] : -1, kb_v = lane < nkb ? 1 << p.gb_ks_[lane] : 0;
    for (int64_t item = it_lo; item < it_hi; ++item) {
      int ub, ct, ks, c0, c1;
      int64_t rt;
      decode(item, ub, rt, ct, ks);
      chunk_range(ks, c0, c1);
      if (unit_change(ub, cur) && !p.wbuild && lane == 0) {  // the unit's whole W^T, resident
        mbar_expect_tx(wfull, (uint32_t)(p.n_chunks * 2 * bbytes));
        for (int c = 0; c < p.n_chunks; ++c) {
          tma_load_3d(&tm_bhi, wfull, wres_hi(c), c * kBKf, 0, ub);
          tma_load_3d(&tm_blo, wfull, wres_lo(c), c * kBKf, 0, ub);
        }
      }
      if (p.gather && p.wres) continue;  // nothing per stage for this warp
      // gbox: the item's row-tile (and unit) coordinates per TMA dimension
      int g0 = 0, g1 = 0, g2 = 0, g3 = 0, g4 = 0;
      auto red = [&](int dsel, int d, int v) { return (int)__reduce_add_sync(0xffffffffu, (unsigned)(dsel == d ? v : 0)); };
      if (p.gbox) {
        const int on = (int)((row0(rt) >> (7 + lane)) & 1) * rb_v;
        const int uo = ub << p.gb_us;
        g0 = red(rb_d, 0, on) + (p.gb_udim == 0 ? uo : 0);
        g1 = red(rb_d, 1, on) + (p.gb_udim == 1 ? uo : 0);
        g2 = red(rb_d, 2, on) + (p.gb_udim == 2 ? uo : 0);
        g3 = red(rb_d, 3, on) + (p.gb_udim == 3 ? uo : 0);
        g4 = red(rb_d, 4, on) + (p.gb_udim == 4 ? uo : 0);
      }
      for (int c = c0; c < c1; ++c) {
        int k0 = 0, k1 = 0, k2 = 0, k3 = 0, k4 = 0;
        if (p.gbox) {
          const int on = ((c >> lane) & 1) * kb_v;
          k0 = g0 + red(kb_d, 0, on);
          k1 = g1 + red(kb_d, 1, on);
          k2 = g2 + red(kb_d, 2, on);
          k3 = g3 + red(kb_d, 3, on);
          k4 = g4 + red(kb_d, 4, on);
        }
        mbar_wait(&empty[s], ph ^ 1);
        if (lane == 0) {
          mbar_expect_tx(&full[s], (p.gather ? 0u : xbytes) + (p.wres ? 0u : 2u * bbytes));
          if (p.gbox) {
            tma_load_5d(&tm_x, &full[s], stage_x(s), k0, k1, k2, k3, k4);
          } else if (!p.gather) {
            tma_load_3d(&tm_x, &full[s], stage_x(s), c * kBKf, (int)row0(rt), p.xb ? ub : 0);
          }
          if (!p.wres) {
            const int brow = ct * p.BN + (int)crank * (p.BN / kCG);
            tma_load_3d(&tm_bhi, &full[s], stage_bhi(s), c * kBKf, brow, ub);
            tma_load_3d(&tm_blo, &full[s], stage_blo(s), c * kBKf, brow, ub);
          }
        }
        __syncwarp();
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ===== gather producer (X not K-contiguous): 16-byte cp.async pieces, manual SW128 =====
    if (p.gather) {
      const int g = threadIdx.x - 64;  // 0..63: rows g and g+64 of every tile
      int64_t roff[2], koff[8];
      for (int h = 0; h < 2; ++h) {
        const int r = g + 64 * h;
        int64_t o = 0;
        for (int i = 0; i < 7 && i < p.nn; ++i)
          if ((r >> i) & 1) o += p.sxn[i];
        roff[h] = o;
      }
      for (int j = 0; j < 8; ++j) {  // complex k = 2j within the chunk (k bit 0 is the pair)
        int64_t o = 0;
        for (int i = 1; i < 4 && i < p.nk; ++i)
          if (((2 * j) >> i) & 1) o += p.sxk[i];
        koff[j] = o;
      }
      int s = 0, cur = -1;
      uint32_t ph = 0;
      for (int64_t item = it_lo; item < it_hi; ++item) {
        int ub, ct, ks, c0, c1;
        int64_t rt;
        decode(item, ub, rt, ct, ks);
        chunk_range(ks, c0, c1);
        unit_change(ub, cur);
        const float2* Xu = p.Xg + (int64_t)ub * p.xbs;
        const int64_t n0 = row0(rt);
        int64_t nbase = 0;
        for (int i = 7; i < p.nn; ++i)
          if ((n0 >> i) & 1) nbase += p.sxn[i];
        const bool ok0 = n0 + g < p.N, ok1 = n0 + g + 64 < p.N;
        for (int c = c0; c < c1; ++c) {
          int64_t kbase = 0;
          const int64_t kc = (int64_t)c * 16;
          for (int i = 4; i < p.nk; ++i)
            if ((kc >> i) & 1) kbase += p.sxk[i];
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* dst = stage_x(s);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = g + 64 * h;
            const bool ok = h ? ok1 : ok0;
            const float2* rowp = Xu + nbase + roff[h] + kbase;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const bool kok = 2 * j < (p.K2 / 2) - c * 16;  // K tail
              cp_async16(dst + r * 128 + ((j ^ (r & 7)) << 4), ok && kok ? (const void*)(rowp + koff[j]) : (const void*)Xu,
                         ok && kok ? 16u : 0u);
            }
          }
          cp_async_arrive_noinc(&full[s]);
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
    } else {
      idle();
    }
  } else if (warp == 1) {
    // ===== MMA issuer (pair: the leader CTA issues for both) =====
    // the whole warp runs the loop (its values stay warp-uniform, so the descriptors live in
    // uniform registers) and one elected lane issues each chunk's MMAs and commits; a
    // single-lane loop made the compiler wrap every tcgen05.mma in an R2UR waterfall loop
    if (leader) {
      int s = 0, cur = -1;
      uint32_t ph = 0, wph = 0;
      int sa_m = 0;  // tsa: TMEM A stage
      int acc = 0;
      uint32_t aph = 0;
      for (int64_t item = it_lo; item < it_hi; ++item) {
        int ub, ct, ks, c0, c1;
        int64_t rt;
        decode(item, ub, rt, ct, ks);
        chunk_range(ks, c0, c1);
        if (unit_change(ub, cur)) {
          mbar_wait(wfull, wph);
          wph ^= 1;
        }
        // flush groups of <= p.group_chunks chunks: each group accumulates into a fresh
        // TMEM partial; the epilogue adds the partials with round-to-nearest fp32
        for (int g0 = c0; g0 < c1; g0 += p.group_chunks) {
          const int g1 = min(c1, g0 + p.group_chunks);
          mbar_wait(&tempty[acc], aph ^ 1);
          tc_fence_after();
          const uint32_t d = tmem_base + (uint32_t)(acc * p.BN);
          for (int c = g0; c < g1; ++c) {
            mbar_wait(&conv[s], ph);
            tc_fence_after();
            const uint32_t bh = smem_u32(p.wres ? wres_hi(c) : stage_bhi(s));
            const uint32_t bl = smem_u32(p.wres ? wres_lo(c) : stage_blo(s));
            if (p.tsa) {  // A = X hi/lo from TMEM stage sa_m (lane = row, column = k)
              const uint32_t ah = tmem_base + (uint32_t)(p.acol + sa_m * 64), alo = ah + 32;
              if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < kBKf / 8; ++kk) {
                  const uint32_t off = kk * 32;
                  const uint32_t first = (c == g0 && kk == 0) ? 0u : 1u;
                  tc_mma_tf32_ts(d, alo + kk * 8, umma_desc_sw128(bh + off), p.idesc, first);
                  tc_mma_tf32_ts(d, ah + kk * 8, umma_desc_sw128(bl + off), p.idesc, 1u);
                  tc_mma_tf32_ts(d, ah + kk * 8, umma_desc_sw128(bh + off), p.idesc, 1u);
                }
                tc_commit(&empty[s]);
                tc_commit(&aempty[sa_m]);
              }
              __syncwarp();
              if (++sa_m == p.sa) sa_m = 0;
              if (++s == S) { s = 0; ph ^= 1; }
              continue;
            }
            const uint32_t ax = smem_u32(stage_x(s)), al = smem_u32(stage_xlo(s));
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < kBKf / 8; ++kk) {
                const uint32_t off = kk * 32;  // 8 tf32 = 32 bytes along K inside the swizzle atom
                const uint32_t first = (c == g0 && kk == 0) ? 0u : 1u;
                if constexpr (kCG == 2) {
                  tc_mma_tf32_pair(d, umma_desc_sw128(al + off), umma_desc_sw128(bh + off), p.idesc, first);
                  tc_mma_tf32_pair(d, umma_desc_sw128(ax + off), umma_desc_sw128(bl + off), p.idesc, 1u);
                  tc_mma_tf32_pair(d, umma_desc_sw128(ax + off), umma_desc_sw128(bh + off), p.idesc, 1u);
                } else {
                  tc_mma_tf32(d, umma_desc_sw128(al + off), umma_desc_sw128(bh + off), p.idesc, first);
                  tc_mma_tf32(d, umma_desc_sw128(ax + off), umma_desc_sw128(bl + off), p.idesc, 1u);
                  tc_mma_tf32(d, umma_desc_sw128(ax + off), umma_desc_sw128(bh + off), p.idesc, 1u);
                }
              }
              if constexpr (kCG == 2) tc_commit_pair(&empty[s]);
              else tc_commit(&empty[s]);
            }
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1; }
          }
          if (elect_one()) {
            if constexpr (kCG == 2) tc_commit_pair(&tfull[acc]);
            else tc_commit(&tfull[acc]);
          }
          __syncwarp();
          if (++acc == p.nbuf) { acc = 0; aph ^= 1; }
        }
      }
    } else {
      idle();
    }
  } else if (warp >= kConvWarp0 && warp < kConvWarp0 + 4) {
    // ===== converters: x -> hi (in place), lo (second buffer) =====
    const int t = threadIdx.x - kConvWarp0 * 32;  // 0..127
    // gbox: this thread's row (t) offset and the 8 k-pair offsets inside the box (bytes)
    uint32_t g_row = 0, g_k[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) g_k[j] = 0;
    if (p.gbox) {
      for (int i = 0; i < 7; ++i)
        if ((t >> i) & 1) g_row += p.gb_rs[i];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        for (int i = 0; i < 3; ++i)
          if ((j >> i) & 1) g_k[j] += p.gb_ks[i];
    }
    int s = 0, cur = -1;
    uint32_t ph = 0;
    int sa_c = 0;        // tsa: TMEM A stage
    uint32_t aph_c = 0;
    for (int64_t item = it_lo; item < it_hi; ++item) {
      int ub, ct, ks, c0, c1;
      int64_t rt;
      decode(item, ub, rt, ct, ks);
      chunk_range(ks, c0, c1);
      unit_change(ub, cur);
      for (int c = c0; c < c1; ++c) {
        mbar_wait(&full[s], ph);
        if (p.tsa) {
          // this thread's X row (= its TMEM lane) -> RN hi/lo -> TMEM A stage sa_c
          mbar_wait(&aempty[sa_c], aph_c ^ 1);
          tc_fence_after();
          const int q = warp - kConvWarp0, row = q * 32 + lane;
          const uint32_t xr = smem_u32(stage_x(s)) + (p.gbox ? g_row : (uint32_t)row * 128);
          const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(p.acol + sa_c * 64);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float hi[16], lo[16];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int j = 4 * h + jj;
              const float4 v = lds128(xr + (p.gbox ? g_k[j] : (uint32_t)((j ^ (row & 7)) << 4)));
              const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float hv = __uint_as_float(cvt_rna_tf32(vv[e]));
                hi[4 * jj + e] = hv;
                lo[4 * jj + e] = __uint_as_float(cvt_rna_tf32(vv[e] - hv));
              }
            }
            tmem_st16(ta + (uint32_t)(16 * h), hi);
            tmem_st16(ta + 32u + (uint32_t)(16 * h), lo);
          }
          tc_fence_before();
          mbar_arrive(&conv[s]);
          if (++sa_c == p.sa) { sa_c = 0; aph_c ^= 1; }
          if (++s == S) { s = 0; ph ^= 1; }
          continue;
        }
        const uint32_t xs = smem_u32(stage_x(s)), xl = smem_u32(stage_xlo(s));
        float4 vin[8];
#pragma unroll
        for (int i = 0; i < (int)(kBM * kBKf / 4 / 128); ++i) vin[i] = lds128(xs + (uint32_t)(i * 128 + t) * 16);
#pragma unroll
        for (int i = 0; i < (int)(kBM * kBKf / 4 / 128); ++i) {  // 8 float4 per thread
          const uint32_t off = (uint32_t)(i * 128 + t) * 16;
          const float4 v = vin[i];
          float4 h, l;
          h.x = __uint_as_float(cvt_rna_tf32(v.x));
          h.y = __uint_as_float(cvt_rna_tf32(v.y));
          h.z = __uint_as_float(cvt_rna_tf32(v.z));
          h.w = __uint_as_float(cvt_rna_tf32(v.w));
          l.x = __uint_as_float(cvt_rna_tf32(v.x - h.x));
          l.y = __uint_as_float(cvt_rna_tf32(v.y - h.y));
          l.z = __uint_as_float(cvt_rna_tf32(v.z - h.z));
          l.w = __uint_as_float(cvt_rna_tf32(v.w - h.w));
          sts128(xs + off, h.x, h.y, h.z, h.w);
          sts128(xl + off, l.x, l.y, l.z, l.w);
        }
        fence_proxy_async();
        if constexpr (kCG == 2) {
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(&conv[s], 0);
        } else {
          mbar_arrive(&conv[s]);
        }
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + kEpiWarps) {
    // ===== epilogue: TMEM -> registers -> swizzled smem -> per-warp TMA bulk store =====
    // warp w owns TMEM lane quarter w%4 (32 rows) and every other store box of the tile;
    // no cross-warp barriers: each warp stages its 32 rows and issues its own stores
    const int et = threadIdx.x - kEpiWarp0 * 32;  // 0..255
    // wbuild: the unit's W^T rows r = 2m + b, fp32 column c2 = 2k + a of chunk c = c2 / 32: row
    // 2m holds (Yr, -Yi) at (2k, 2k+1), row 2m+1 holds (Yi, Yr); hi = rna_tf32(w),
    // lo = rna_tf32(w - hi); stored in the SW128 K-major layout TMA would have produced
    auto build_w = [&](int ub, bool first) {
      const int K = p.K2 / 2, Mc = p.M2 / 2;
      if (first && (p.K2 % kBKf)) {  // K tail of the last chunk: zeros (never overwritten), as TMA's OOB fill
        const uint32_t wbytes = (uint32_t)(p.n_chunks * 2 * p.BN * kBKf * 4);
        for (uint32_t o = (uint32_t)et * 16; o < wbytes; o += 32 * kEpiWarps * 16)
          *reinterpret_cast<float4*>(wres + o) = make_float4(0.f, 0.f, 0.f, 0.f);
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      }
      const float2* Yu = p.Yg + (p.ydelta ? p.ydelta[ub] : 0);
      // resident W^T is <= 64 KB, so K*M <= 2048 complex: <= 8 values per thread, all
      // loads issued before the first use (one memory round trip, not eight)
      constexpr int kWPer = 8;
      float2 yv[kWPer];
#pragma unroll
      for (int j = 0; j < kWPer; ++j) {
        const int idx = et + j * 32 * kEpiWarps;
        if (idx < K * Mc) {
          const int k = idx % K, m = idx / K;
          int64_t o = 0;
          for (int i = 0; i < p.nk; ++i)
            if ((k >> i) & 1) o += p.syk[i];
          for (int i = 0; i < p.nm; ++i)
            if ((m >> i) & 1) o += p.sym[i];
          yv[j] = __ldg(Yu + o);
        }
      }
#pragma unroll
      for (int j = 0; j < kWPer; ++j) {
        const int idx = et + j * 32 * kEpiWarps;
        if (idx >= K * Mc) break;
        const int k = idx % K, m = idx / K;
        const float2 y = yv[j];
        const float w[4] = {y.x, -y.y, y.y, y.x};  // (row 2m: col 2k, 2k+1), (row 2m+1: col 2k, 2k+1)
        const int c2 = 2 * k, c = c2 / kBKf, cc = c2 % kBKf;
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int r = 2 * m + b;
          const uint32_t off = (uint32_t)(r * 128 + (((cc >> 2) ^ (r & 7)) << 4) + (cc & 3) * 4);
          const float h0 = __uint_as_float(cvt_rna_tf32(w[2 * b])), h1 = __uint_as_float(cvt_rna_tf32(w[2 * b + 1]));
          const float l0 = __uint_as_float(cvt_rna_tf32(w[2 * b] - h0)), l1 = __uint_as_float(cvt_rna_tf32(w[2 * b + 1] - h1));
          *reinterpret_cast<float2*>(wres_hi(c) + off) = make_float2(h0, h1);
          *reinterpret_cast<float2*>(wres_lo(c) + off) = make_float2(l0, l1);
        }
      }
      fence_proxy_async();
      mbar_arrive(wfull);
    };
    const int q = warp & 3;
    const int half = (warp - kEpiWarp0) >> 2;
    int acc = 0, sbuf = 0, cur = -1;
    uint32_t aph = 0;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t tot = tmem_base + (uint32_t)(p.nbuf * p.BN) + lane_off;  // running total (flush mode)
    const bool swz = p.boxw == 32;
    const uint32_t pitch = (uint32_t)p.boxw * 4;
    uint8_t* my_stg = staging + (size_t)(warp - kEpiWarp0) * p.nstg * stg_bytes;
    const int nbox = p.BN / p.boxw;
    for (int64_t item = it_lo; item < it_hi; ++item) {
      int ub, ct, ks, c0, c1;
      int64_t rt;
      decode(item, ub, rt, ct, ks);
      chunk_range(ks, c0, c1);
      {
        const bool first = cur < 0;
        if (unit_change(ub, cur) && p.wbuild) build_w(ub, first);
      }
      for (int g0 = c0; g0 < c1; g0 += p.group_chunks) {
        const bool first = g0 == c0, last = g0 + p.group_chunks >= c1;
        mbar_wait(&tfull[acc], aph);
        tc_fence_after();
        const uint32_t taddr = tmem_base + (uint32_t)(acc * p.BN) + lane_off;
        for (int bx = half; bx < nbox; bx += 2) {
          const int cb = bx * p.boxw;
          float v[32];
          if (p.boxw == 32) {
            tmem_ld32(taddr + (uint32_t)cb, v);
            if (!first) {
              float t[32];
              tmem_ld32(tot + (uint32_t)cb, t);
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __fadd_rn(v[j], t[j]);
            }
            if (!last) {
              tmem_st16(tot + (uint32_t)cb, v);
              tmem_st16(tot + (uint32_t)cb + 16, v + 16);
            }
          } else {
            tmem_ld16(taddr + (uint32_t)cb, v);
            if (!first) {
              float t[16];
              tmem_ld16(tot + (uint32_t)cb, t);
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = __fadd_rn(v[j], t[j]);
            }
            if (!last) tmem_st16(tot + (uint32_t)cb, v);
          }
          if (!last) continue;
          // this warp's staging buffer sbuf was used by its store nstg boxes ago
          if (lane == 0) bulk_wait_read(p.nstg - 1);
          __syncwarp();
          const uint32_t stg = smem_u32(my_stg + (size_t)sbuf * stg_bytes) + (uint32_t)lane * pitch;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (j < p.boxw / 4) {
              const int pos = swz ? (j ^ (lane & 7)) : j;
              sts128(stg + pos * 16, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_4d(&tm_c, my_stg + (size_t)sbuf * stg_bytes, ct * p.BN + cb, (int)row0(rt) + q * 32, ks, ub);
            bulk_commit();
          }
          if (++sbuf == p.nstg) sbuf = 0;
        }
        tc_fence_before();
        if constexpr (kCG == 2) {
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
        } else {
          mbar_arrive(&tempty[acc]);
        }
        if (++acc == p.nbuf) { acc = 0; aph ^= 1; }
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kCG == 2) cluster_sync_all();  // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    if constexpr (kCG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(p.tmem_cols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(p.tmem_cols));
  }
}

// W^T hi/lo [M2][K2] of unit blockIdx.z: Wt[2m+b][2k+a] = W[2k+a][2m+b], W block [[Yr, Yi], [-Yi, Yr]]
// One CTA per (256 / kc complex columns m, block of kc = min(K, 256) complex k, unit): the small
// operand is gathered with per-thread column offsets plus a shared table for the low k bits,
// and the four real-block entries are written as float2 pairs (coalesced along k).
__global__ void __launch_bounds__(256) tc_prep_kernel(const float2* __restrict__ Y, float* __restrict__ wbuf,
                                                      int64_t wunit, int nk, int nm, GemmDesc g,
                                                      const int64_t* __restrict__ ydelta) {
  pdl_wait();
  pdl_trigger();
  __shared__ int64_t lowtab[256];
  const int64_t K = (int64_t)1 << nk, K2 = 2 * K, M2 = (int64_t)2 << nm;
  const int ub = blockIdx.z;
  const float2* Yu = Y + (ydelta ? ydelta[ub] : 0);
  float* whi = wbuf + (int64_t)ub * wunit;
  float* wlo = whi + K2 * M2;
  const int lowbits = nk < 8 ? nk : 8, kc = 1 << lowbits;
  const int64_t m = (int64_t)blockIdx.x * (256 >> lowbits) + (threadIdx.x >> lowbits);
  const int64_t k0 = (int64_t)blockIdx.y * kc;
  const int kl = threadIdx.x & (kc - 1);
  {
    int t = threadIdx.x;
    int64_t o = 0;
    for (int i = 0; i < lowbits; ++i)
      if ((t >> i) & 1) o += g.syk[i];
    lowtab[t] = o;
  }
  __syncthreads();
  if (m >= (M2 >> 1)) return;
  int64_t base = 0;
  for (int i = 0; i < nm; ++i)
    if ((m >> i) & 1) base += g.sym[i];
  for (int i = lowbits; i < nk; ++i)
    if ((k0 >> i) & 1) base += g.syk[i];
  const int64_t k = k0 + kl;
  const float2 y = Yu[base + lowtab[kl]];
  // W^T row 2m: (Yr, -Yi) at columns (2k, 2k+1); row 2m+1: (Yi, Yr)
  const float w[4] = {y.x, -y.y, y.y, y.x};
  const int64_t r0 = (2 * m) * K2 + 2 * k, r1 = (2 * m + 1) * K2 + 2 * k;
  float h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    h[i] = __uint_as_float(cvt_rna_tf32(w[i]));
    l[i] = __uint_as_float(cvt_rna_tf32(w[i] - h[i]));
  }
  *reinterpret_cast<float2*>(whi + r0) = make_float2(h[0], h[1]);
  *reinterpret_cast<float2*>(whi + r1) = make_float2(h[2], h[3]);
  *reinterpret_cast<float2*>(wlo + r0) = make_float2(l[0], l[1]);
  *reinterpret_cast<float2*>(wlo + r1) = make_float2(l[2], l[3]);
}

// split-K partials -> C of unit blockIdx.y.  Short K: partial k holds flush group k alone, so
// the sequential fp32 sum part[0] + part[1] + ... repeats the unsplit kernel's TMEM running
// total exactly (bit-identical).  Long K (the split is fixed by the shape): fp64 sum in order.
__global__ void tc_splitk_reduce(const float* __restrict__ part, float* __restrict__ C, int64_t n, int ks,
                                 int64_t pks, int64_t punit, const int64_t* __restrict__ cdelta, int longk) {
  pdl_wait();
  pdl_trigger();
  const int ub = blockIdx.y;
  part += (int64_t)ub * punit;
  C += 2 * (cdelta ? cdelta[ub] : 0);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (longk) {
      double s = 0.0;
      for (int k = 0; k < ks; ++k) s += (double)part[(int64_t)k * pks + i];
      C[i] = (float)s;
    } else {
      float s = part[i];
      for (int k = 1; k < ks; ++k) s = __fadd_rn(s, part[(int64_t)k * pks + i]);
      C[i] = s;
    }
  }
}

// ---------------- host side ----------------
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

uint64_t up16(uint64_t b) { return (b + 15) / 16 * 16; }

// fp32 tensor map over [outer2][outer1][inner] with explicit byte strides of the two outer dims
void encode(CUtensorMap* m, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
            const uint32_t* box, CUtensorMapSwizzle swz, CUtensorMapL2promotion l2) {
  auto enc = get_encode();
  TNQVM_CHECK(enc, TNQVM_ECUDA, "cuTensorMapEncodeTiled is unavailable (driver too old for sm_100a TMA)");
  cuuint64_t d[5];
  cuuint64_t st[4];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    bx[i] = box[i];
    es[i] = 1;
  }
  for (int i = 0; i + 1 < rank; ++i) st[i] = strides_bytes[i];
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<void*>(ptr), d, st, bx, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, swz, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TNQVM_CHECK(r == CUDA_SUCCESS, TNQVM_ECUDA, "cuTensorMapEncodeTiled failed (error " + std::to_string((int)r) + ")");
}

// K per TMEM partial before a round-to-nearest flush: the MMA chain accumulates with an error
// growing linearly in its length.  Measured against torch complex64 (SURVEY 8(d) bar: <= 4x
// and <= 1e-6 for K <= 2^10; profiles/r02b_tc_accuracy.jsonl, 18 shapes): 1 chunk (16 complex
// K) 0.34-2.9x; 2 chunks (32 complex K) 0.49-3.1x and <= 7.9e-7 everywhere; 4 chunks up to
// 4.5x and 1.2e-6 (fails) but 5-11% faster on the tensor-bound shapes.  So: 2 chunks.
constexpr int kGroupChunks = 2;

int group_chunks_of(int /*n_chunks*/) { return kGroupChunks; }
// chunks (16 complex K each) per split item for long K (1024 complex K = 32 flush groups)
constexpr int kLongKChunks = 64;

// Tile / split / flush decisions.  Everything that shapes a unit's arithmetic (BN, flush
// groups) depends on (N, K, M) only; `split` only chooses whether the flush groups run in
// one CTA or as separate items (bit-identical either way).
TcParams plan_tc(int64_t N, int nk, int nm, int cg, bool tsa, bool split) {
  TcParams p{};
  p.N = N;
  p.K2 = 2 << nk;
  p.M2 = 2 << nm;
  p.n_chunks = (p.K2 + kBKf - 1) / kBKf;
  const int group_chunks = group_chunks_of(p.n_chunks);
  const bool flush = p.n_chunks > group_chunks;
  p.BN = std::min(256, std::max(16, p.M2));
  p.n_col_tiles = (p.M2 + p.BN - 1) / p.BN;
  p.n_row_tiles = (int)((N + kBM * cg - 1) / (kBM * cg));  // CTA pairs own 256-row tiles
  p.longk = p.n_chunks > kLongKChunks ? 1 : 0;
  p.chunks_per_split = p.longk ? kLongKChunks : split && flush ? group_chunks : p.n_chunks;
  p.k_splits = (p.n_chunks + p.chunks_per_split - 1) / p.chunks_per_split;
  p.group_chunks = std::min(p.chunks_per_split, group_chunks);
  p.boxw = p.M2 >= 32 ? 32 : 16;  // TMA clips columns beyond M2
  const size_t wres_bytes = (size_t)p.n_chunks * 2 * p.BN * kBKf * 4;
  p.wres = (cg == 1 && p.n_col_tiles == 1 && p.k_splits == 1 && wres_bytes <= 64 * 1024) ? 1 : 0;
  p.tsa = (tsa && cg == 1 && p.BN <= 128) ? 1 : 0;
  const uint32_t stage_bytes = (p.tsa ? 1 : 2) * kBM * kBKf * 4 + (p.wres ? 0 : 2 * (p.BN / cg) * kBKf * 4);
  const size_t avail = 225 * 1024;  // 227 KB opt-in minus alignment slack and barriers
  // staging buffers per epilogue warp: one per store box the warp issues per tile (up to 4),
  // so a tile's stores are all in flight instead of each waiting for the previous one to
  // leave shared memory (the short-K steps were epilogue-latency bound with one buffer:
  // profiles/r02c_*), as long as >= 3 input stages remain
  const int boxes_per_warp = std::max(1, p.BN / p.boxw / 2);
  int nstg0 = std::min(4, boxes_per_warp);
  for (p.nstg = nstg0; ; --p.nstg) {
    const size_t fixed = (size_t)kEpiWarps * p.nstg * 32 * p.boxw * 4 + (p.wres ? wres_bytes : 0);
    p.stages = fixed + 2 * (size_t)stage_bytes <= avail ? std::min<int>(6, (int)((avail - fixed) / stage_bytes)) : 2;
    if (p.stages >= 3 || p.nstg == 1) break;
  }
  const bool flushing = p.chunks_per_split > p.group_chunks;
  p.nbuf = (flushing && 3 * p.BN > 512) ? 1 : 2;
  uint32_t need = (uint32_t)((flushing ? p.nbuf + 1 : 2) * p.BN), cols = 32;
  if (p.tsa) {  // two TMEM A stages (X hi | lo, 64 columns each) after the accumulators
    p.sa = 2;
    p.acol = (int)need;
    need += (uint32_t)(p.sa * 64);
  }
  while (cols < need) cols <<= 1;
  p.tmem_cols = cols;
  // instruction descriptor: D=f32, A=B=tf32, K-major both, N>>3, M>>4
  p.idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(p.BN >> 3) << 17) | ((uint32_t)((kBM * cg) >> 4) << 24);
  return p;
}

// streamed-W^T steps: A from TMEM in a single CTA when BN <= 128, else CTA pairs
// (cta_group::2) with >= 2 pair tiles (per-unit shape only)
bool choose_tsa(int64_t N, int nk, int nm) {
  TcParams p1 = plan_tc(N, nk, nm, 1, false, false);
  // long K (fixed 1024-complex-K items) on CTA pairs when the rows allow: A from shared memory
  // and half the MMA instructions per SM (C3's N = 2^11, K = 2^19 step 23.1 -> 21.3 ms)
  if (p1.longk && N >= 2 * kBM * 2 && p1.BN >= 32) return false;
  return p1.BN <= 128;
}
int choose_cg(int64_t N, int nk, int nm) {
  if (choose_tsa(N, nk, nm)) return 1;
  TcParams p1 = plan_tc(N, nk, nm, 1, false, false);
  if (p1.wres || p1.BN < 32 || N < 2 * kBM * 2) return 1;
  return 2;
}

int64_t part_floats(int64_t N, int nm) { return (int64_t)up16((uint64_t)N * ((uint64_t)2 << nm) * 4) / 4; }

// gbox: the gather step's X as one TMA box per stage.  The bits of X (each row bit n_i and k
// bit k_i has a stride; k_0 has stride 1 complex) sorted by stride, with the re/im bit below,
// are cut into TMA dimensions at every stride gap, where a tile bit (rows n_0..n_6, the chunk's
// k_0..k_3) would sit above a coordinate bit of the same run, and where a run's box would pass
// 256 elements.  Feasible when that gives <= 5 dimensions (unit dimension included).
struct GBox {
  int ndim = 0, udim = -1, ushift = 0;
  uint64_t base[5], size[5];  // fp32 stride and extent of each dimension
  uint32_t box[5];
  int8_t nd[33], ns[33], kd[16], ks[16];
  uint32_t rs[7], kstr[3];
};
bool plan_gbox(const GemmDesc& g, int nb, int64_t xstep, GBox* o) {
  if (!g.gather || g.nk < 4 || g.nn < 7 || g.nn > 40 || g.nk > 20 || g.sxk[0] != 1) return false;
  struct Bit { int64_t stride; int kind, idx; };  // kind 0 = n, 1 = k
  std::vector<Bit> bits;
  for (int i = 0; i < g.nn; ++i) bits.push_back({g.sxn[i], 0, i});
  for (int i = 0; i < g.nk; ++i) bits.push_back({g.sxk[i], 1, i});
  std::sort(bits.begin(), bits.end(), [](const Bit& a, const Bit& b) { return a.stride < b.stride; });
  GBox b;
  bool coord[6] = {false, false, false, false, false, false};
  int pos_of_n[40], dim_of_n[40], pos_of_k[20], dim_of_k[20];
  b.ndim = 1;
  b.base[0] = 1;
  b.size[0] = 2;  // re / im
  b.box[0] = 2;
  for (const Bit& t : bits) {
    if (t.stride <= 0) return false;
    const uint64_t f = 2 * (uint64_t)t.stride;  // fp32 stride
    const bool tile = t.kind == 0 ? t.idx < 7 : t.idx < 4;
    int d = b.ndim - 1;
    const bool contiguous = f == b.base[d] * b.size[d];
    if (!(contiguous && (!tile || (!coord[d] && b.box[d] * 2 <= 256)))) {
      if (b.ndim == 5) return false;
      d = b.ndim++;
      b.base[d] = f;
      b.size[d] = 1;
      b.box[d] = 1;
      coord[d] = false;
    }
    int pos = 0;
    while (((uint64_t)1 << pos) < b.size[d]) ++pos;
    b.size[d] *= 2;
    if (tile) b.box[d] *= 2;
    else coord[d] = true;
    (t.kind == 0 ? pos_of_n : pos_of_k)[t.idx] = pos;
    (t.kind == 0 ? dim_of_n : dim_of_k)[t.idx] = d;
  }
  if (nb > 1 && xstep != 0) {  // the unit index: extends the top run if contiguous, else a dimension
    const int d = b.ndim - 1;
    if ((uint64_t)2 * (uint64_t)xstep == b.base[d] * b.size[d]) {
      b.udim = d;
      int pos = 0;
      while (((uint64_t)1 << pos) < b.size[d]) ++pos;
      b.ushift = pos;
      b.size[d] *= (uint64_t)nb;
    } else {
      if (b.ndim == 5) return false;
      const int e = b.ndim++;
      b.base[e] = 2 * (uint64_t)xstep;
      b.size[e] = (uint64_t)nb;
      b.box[e] = 1;
      b.udim = e;
      b.ushift = 0;
    }
  }
  for (int d = 0; d < b.ndim; ++d)
    if (b.box[d] > 256 || b.size[d] > ((uint64_t)1 << 32) || (d > 0 && (b.base[d] * 4) % 16) ||
        b.base[d] * 4 >= ((uint64_t)1 << 40))
      return false;
  if ((b.box[0] * 4) % 16) return false;
  uint64_t vol = 1;
  for (int d = 0; d < b.ndim; ++d) vol *= b.box[d];
  if (vol != (uint64_t)kBM * kBKf) return false;  // the box is exactly one stage's X tile (expect_tx)
  // shared-memory byte stride of a tile bit: the box lands dimension 0 fastest
  auto sstride = [&](int d, int pos) {
    uint64_t st = 1;
    for (int e = 0; e < d; ++e) st *= b.box[e];
    return (uint32_t)(4 * (st << pos));
  };
  if (dim_of_k[0] != 0 || pos_of_k[0] != 1) return false;  // (re, im) x k_0: 16 contiguous bytes
  for (int i = 0; i < 7; ++i) b.rs[i] = sstride(dim_of_n[i], pos_of_n[i]);
  for (int i = 1; i < 4; ++i) b.kstr[i - 1] = sstride(dim_of_k[i], pos_of_k[i]);
  for (int i = 7; i < g.nn; ++i) { b.nd[i - 7] = (int8_t)dim_of_n[i]; b.ns[i - 7] = (int8_t)pos_of_n[i]; }
  for (int i = 4; i < g.nk; ++i) { b.kd[i - 4] = (int8_t)dim_of_k[i]; b.ks[i - 4] = (int8_t)pos_of_k[i]; }
  *o = b;
  return true;
}

}  // namespace

bool tc_supported(int nk, int nm) {
  // X rows must be 16-byte multiples for TMA (K >= 2); W^T must fit comfortably
  // (a pure function of the shape: the program compiler runs on hosts without a GPU; the
  // driver's tensor-map encoder is checked at launch)
  return nk >= 1 && nk <= 20 && nm <= 16 && nk + nm <= 26;
}

// per unit: W^T hi + lo [M2][K2] fp32, then room for one partial per flush group
size_t tc_wbuf_bytes(int64_t N, int nk, int nm) {
  const int n_chunks = ((2 << nk) + kBKf - 1) / kBKf;
  const int gc = group_chunks_of(n_chunks);
  int64_t parts = 1;
  if (n_chunks > kLongKChunks) {
    parts = (n_chunks + kLongKChunks - 1) / kLongKChunks;  // fixed long-K split
  } else if (n_chunks > gc) {
    // flush groups as separate items only when one unit's tiles cannot fill half the
    // machine (launch_gemm_tc's rule at nb = 1; more units only split less)
    const int cg = choose_cg(N, nk, nm);
    TcParams p = plan_tc(N, nk, nm, cg, choose_tsa(N, nk, nm), false);
    if ((int64_t)p.n_row_tiles * p.n_col_tiles * 2 <= sm_count() / cg) parts = (n_chunks + gc - 1) / gc;
  }
  return ((size_t)32 << (nk + nm)) + (parts > 1 ? (size_t)parts * part_floats(N, nm) * 4 : 0);
}

void launch_gemm_tc(const GemmDesc& g, void* wbuf, const Batch& bt, cudaStream_t st) {
  TNQVM_CHECK(tc_supported(g.nk, g.nm), TNQVM_EINVAL, "shape not supported by the tcgen05 kernel");
  int64_t xstep = 0, cstep = 0;
  const size_t wunit_bytes = tc_wbuf_bytes(g.N, g.nk, g.nm);
  if (!bt.affine(0, &xstep) || !bt.affine(2, &cstep) || (bt.nb > 1 && cstep == 0)) {
    // units whose X / C are not at a constant step: one launch per unit
    for (int b = 0; b < bt.nb; ++b) {
      GemmDesc gu = g;
      gu.X = (const float2*)g.X + bt.d(0, b);
      gu.Y = (const float2*)g.Y + bt.d(1, b);
      gu.C = (float2*)g.C + bt.d(2, b);
      launch_gemm_tc(gu, (char*)wbuf + wunit_bytes * b, Batch{}, st);
    }
    return;
  }
  const int nb = bt.nb;
  const int cg = choose_cg(g.N, g.nk, g.nm);
  const bool tsa = choose_tsa(g.N, g.nk, g.nm);
  // gbox only with the A operand in TMEM: with CTA pairs the extra raw-box buffer per stage
  // costs more than the cp.async gather loses (C2 op14 equal, op23 0.086 -> 0.107 ms)
  GBox gb;
  const bool gbox = tsa && plan_gbox(g, nb, xstep, &gb);
  // split the flush groups into separate items when the units' output tiles cannot fill the machine
  TcParams p = plan_tc(g.N, g.nk, g.nm, cg, tsa, false);
  const int units = sm_count() / cg;
  if (!p.longk && (int64_t)nb * p.n_row_tiles * p.n_col_tiles * 2 <= units && p.n_chunks > p.group_chunks)
    p = plan_tc(g.N, g.nk, g.nm, cg, tsa, true);
  const int K2 = p.K2, M2 = p.M2;
  p.nb = nb;
  p.items_per_unit = (int64_t)p.n_row_tiles * p.n_col_tiles * p.k_splits;
  p.n_items = p.items_per_unit * nb;
  p.xb = xstep != 0 ? 1 : 0;
  const int64_t wunit = (int64_t)(wunit_bytes / 4);  // floats per unit slab
  float* whi = reinterpret_cast<float*>(wbuf);
  const int64_t* ydelta = bt.delta ? bt.delta + nb : nullptr;
  p.wbuild = p.wres && p.BN == M2 && g.nk + g.nm <= 11;  // <= 8 Y values per epilogue thread
  if (p.wbuild) {
    p.Yg = reinterpret_cast<const float2*>(g.Y);
    p.ydelta = ydelta;
    p.nm = g.nm;
    for (int i = 0; i < g.nk; ++i) p.syk[i] = g.syk[i];
    for (int i = 0; i < g.nm; ++i) p.sym[i] = g.sym[i];
  } else {
    const int lowbits = std::min(g.nk, 8), mper = 256 >> lowbits;  // complex columns per CTA
    dim3 grid((unsigned)((M2 / 2 + mper - 1) / mper), (unsigned)((int64_t)1 << (g.nk - lowbits)), (unsigned)nb);
    launch_pdl(tc_prep_kernel, grid, 256, 0, st, reinterpret_cast<const float2*>(g.Y), whi, wunit, g.nk, g.nm, g,
               ydelta);
  }
  const bool split = p.k_splits > 1;
  float* part = whi + (size_t)2 * K2 * M2;  // unit 0's partials follow its W^T hi/lo
  const int64_t pks = part_floats(g.N, g.nm);
  p.gather = gbox ? 0 : g.gather;
  p.gbox = gbox ? 1 : 0;
  p.gb_udim = -1;
  if (gbox) {
    p.gb_ndim = gb.ndim;
    p.gb_udim = gb.udim;
    p.gb_us = gb.ushift;
    for (int i = 0; i < 33; ++i) { p.gb_nd[i] = gb.nd[i]; p.gb_ns[i] = gb.ns[i]; }
    for (int i = 0; i < 16; ++i) { p.gb_kd[i] = gb.kd[i]; p.gb_ks_[i] = gb.ks[i]; }
    for (int i = 0; i < 7; ++i) p.gb_rs[i] = gb.rs[i];
    for (int i = 0; i < 3; ++i) p.gb_ks[i] = gb.kstr[i];
  }
  p.nn = g.nn;
  p.nk = g.nk;
  p.Xg = reinterpret_cast<const float2*>(g.X);
  p.xbs = xstep;
  if (g.gather) {
    for (int i = 0; i < g.nn && i < 40; ++i) p.sxn[i] = g.sxn[i];
    for (int i = 0; i < g.nk && i < 40; ++i) p.sxk[i] = g.sxk[i];
  }
  CUtensorMap mx, mbh, mbl, mc;
  {  // C (or the partials): [unit][k split][N][M2] fp32
    const uint64_t dims[4] = {(uint64_t)M2, (uint64_t)g.N, (uint64_t)p.k_splits, (uint64_t)nb};
    const uint64_t rowb = (uint64_t)M2 * 4;
    const uint64_t ksb = split ? (uint64_t)pks * 4 : up16(rowb * g.N);
    const uint64_t ub = split ? (uint64_t)wunit * 4 : (nb > 1 ? (uint64_t)cstep * 8 : up16(ksb * p.k_splits));
    const uint64_t strides[3] = {rowb, ksb, ub};
    const uint32_t box[4] = {(uint32_t)p.boxw, 32, 1, 1};  // one epilogue warp's 32 rows
    encode(&mc, split ? (const void*)part : g.C, 4, dims, strides, box,
           p.boxw == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE);
  }
  {  // X: [unit][N][K2] (unit dimension only if the units' X differ)
    const uint64_t rowb = (uint64_t)K2 * 4;
    const uint64_t dims[3] = {(uint64_t)K2, (uint64_t)g.N, (uint64_t)(p.xb ? nb : 1)};
    const uint64_t strides[2] = {rowb, p.xb ? (uint64_t)xstep * 8 : up16(rowb * g.N)};
    const uint32_t box[3] = {(uint32_t)kBKf, (uint32_t)kBM, 1};
    if (gbox) {  // the box map: 5 dimensions (unused ones of extent 1)
      uint64_t dims[5], strides[4];
      uint32_t box[5];
      for (int d = 0; d < 5; ++d) {
        dims[d] = d < gb.ndim ? gb.size[d] : 1;
        box[d] = d < gb.ndim ? gb.box[d] : 1;
        if (d > 0) strides[d - 1] = 4 * (d < gb.ndim ? gb.base[d] : gb.base[gb.ndim - 1] * gb.size[gb.ndim - 1]);
      }
      encode(&mx, g.X, 5, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    } else if (g.gather) {
      const uint64_t wd[3] = {(uint64_t)K2, (uint64_t)M2, 1};
      const uint64_t ws[2] = {rowb, up16(rowb * M2)};
      encode(&mx, whi, 3, wd, ws, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);  // unused
    } else {
      encode(&mx, g.X, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    }
  }
  {  // W^T hi / lo: [unit][M2][K2], unit slabs wunit floats apart
    const uint64_t dims[3] = {(uint64_t)K2, (uint64_t)M2, (uint64_t)nb};
    const uint64_t strides[2] = {(uint64_t)K2 * 4, (uint64_t)wunit * 4};
    const uint32_t box[3] = {(uint32_t)kBKf, (uint32_t)(p.wres ? p.BN : p.BN / cg), 1};
    encode(&mbh, whi, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    encode(&mbl, whi + (size_t)K2 * M2, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
  }
  const uint32_t stage_bytes = (p.tsa ? 1 : 2) * kBM * kBKf * 4 + (p.wres ? 0 : 2 * (p.BN / cg) * kBKf * 4);
  const size_t smem = 1024 + (size_t)p.stages * stage_bytes + (p.wres ? (size_t)p.n_chunks * 2 * p.BN * kBKf * 4 : 0) +
                      (size_t)kEpiWarps * p.nstg * 32 * p.boxw * 4 + (3 * p.stages + 8 + 4) * 8 + 16;
  const int nsm = sm_count();
  if (cg == 2) {
    cudaFuncSetAttribute(tc_gemm_kernel_t<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int pairs = (int)std::min<int64_t>(p.n_items, nsm / 2);
    launch_pdl_cluster(tc_gemm_kernel_t<2>, 2 * pairs, kThreadsTC, smem, st, 2u, mx, mbh, mbl, mc, p);
  } else {
    cudaFuncSetAttribute(tc_gemm_kernel_t<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = (int)std::min<int64_t>(p.n_items, nsm);
    launch_pdl(tc_gemm_kernel_t<1>, grid, kThreadsTC, smem, st, mx, mbh, mbl, mc, p);
  }
  if (split) {
    const int64_t n = g.N * (int64_t)M2;
    const dim3 rg((unsigned)std::min<int64_t>((n + 255) / 256, 8192), (unsigned)nb);
    launch_pdl(tc_splitk_reduce, rg, 256, 0, st, part, reinterpret_cast<float*>(g.C), n, p.k_splits, pks, wunit,
               bt.delta ? bt.delta + 2 * nb : nullptr, p.longk);
  }
}

}  // namespace dev
}  // namespace tnqvm
