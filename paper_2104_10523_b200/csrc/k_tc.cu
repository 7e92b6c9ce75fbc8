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
// CTA (persistent, one per SM, 384 threads):
//   warp 0      TMA producer (X chunk + W^T hi + W^T lo per stage, one mbarrier)
//   warp 1      TMEM allocator + single-thread MMA issuer (12 MMAs per 32-wide K chunk)
//   warps 4-7   converters: fp32 -> (hi in place, lo to a second buffer), fence.proxy.async
//   warps 8-11  epilogue: tcgen05.ld (32x32b) -> registers -> global (or split-K partials)
// Pipelines: stage ring full/conv/empty mbarriers; double-buffered TMEM accumulators.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <mutex>

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
  int64_t N;       // rows
  int K2;          // fp32 columns of X (= 2K)
  int M2;          // fp32 columns of C (= 2M)
  int BN;          // fp32 columns per tile (MMA N), multiple of 16, <= 256
  int n_col_tiles, n_row_tiles, k_splits, chunks_per_split, n_chunks;
  int group_chunks;  // K chunks accumulated in one TMEM partial before a round-to-nearest flush
  int nbuf;          // TMEM partial buffers (2; 1 when BN=256 flushes: partial + total fill 512 columns)
  int stages;
  int64_t n_items;
  float* C;        // output fp32 [N][M2]
  float* part;     // split-K partials [k_splits][N][M2] (k_splits > 1)
  uint32_t idesc;
  uint32_t tmem_cols;
  int boxw;         // fp32 columns per TMA store box (32, or M2 < 32)
  int wres;         // 1: the whole W^T hi/lo of the (single) column tile stays resident in smem
  int wsplit;       // 1 (streamed W^T): W^T is loaded once as raw fp32 and split into hi/lo on chip by
                    // the converter warps, halving the per-stage L2->SM bytes of the small operand
  int tsa;          // 1 (single CTA, streamed W^T, BN <= 128): the A operand (X hi/lo) lives in TMEM --
                    // the converters tcgen05.st it there and the MMAs read [a_tmem]; no X hi/lo in
                    // shared memory (the 3xTF32 kernel is shared-memory-bandwidth bound)
  int sa, acol;     // tsa: TMEM A stages (64 columns each: hi | lo) starting at column acol
  int ystream;      // 1: both operands streamed (split-K steps with a tiny output): the Y tile [BN/2 m][32 fp32 of K]
                    // (Y stored [M][K], K fastest) lands in the lo buffer and the converters expand it into
                    // the W^T hi/lo real-block tiles -- no prep kernel, no W^T workspace
  int nstg;         // staging buffers per epilogue warp (2, or 1 when shared memory is tight)
  int gather;       // 1: X tiles gathered with cp.async by warps 2-3 (any layout with a contracted fastest mode)
  int nn, nk;
  const float2* Xg;
  int64_t sxn[40], sxk[40];
  // wbuild: resident W^T hi/lo built in shared memory by the epilogue warps straight from
  // the small operand Y (per-bit strides), instead of a prep kernel + TMA loads
  int wbuild, nm;
  const float2* Yg;
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
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
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
  uint8_t* staging = wres + wres_bytes;  // per epilogue warp 2 x [32 rows][boxw fp32], 1024-aligned
  const uint32_t stg_bytes = 32u * p.boxw * 4;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + (size_t)kEpiWarps * p.nstg * stg_bytes);
  uint64_t* full = bars;            // [S]  TMA landed
  uint64_t* conv = bars + S;        // [S]  converters done
  uint64_t* empty = bars + 2 * S;   // [S]  MMAs consumed the stage
  uint64_t* tfull = bars + 3 * S;   // [2]  accumulator ready
  uint64_t* tempty = bars + 3 * S + 2;  // [2] accumulator drained
  uint64_t* wfull = bars + 3 * S + 4;  // resident W landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 5);
  uint64_t* aempty = bars + 3 * S + 6;  // [sa] tsa: MMAs consumed the TMEM A stage

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t crank = 0;
  if constexpr (kCG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const bool leader = crank == 0;
  const int64_t item0 = kCG == 2 ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;
  const int64_t istep = kCG == 2 ? (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;
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

  // item -> (row tile, col tile, k split): columns fastest (X row tile reused from L2)
  // (32-bit fast paths: one column tile / no split-K are the common cases, and a 64-bit
  // division costs ~100 instructions on every role's item loop)
  const bool small_items = p.n_items < ((int64_t)1 << 31);
  auto decode = [&](int64_t item, int64_t& rt, int& ct, int& ks) {
    if (p.n_col_tiles == 1 && p.k_splits == 1) {
      ct = 0;
      ks = 0;
      rt = item;
    } else if (small_items) {
      const uint32_t it = (uint32_t)item, nct = (uint32_t)p.n_col_tiles, nrt = (uint32_t)p.n_row_tiles;
      const uint32_t r = it / nct;
      ct = (int)(it - r * nct);
      const uint32_t k = r / nrt;
      rt = (int64_t)(r - k * nrt);
      ks = (int)k;
    } else {
      ct = (int)(item % p.n_col_tiles);
      int64_t r = item / p.n_col_tiles;
      rt = r % p.n_row_tiles;
      ks = (int)(r / p.n_row_tiles);
    }
  };
  auto chunk_range = [&](int ks, int& c0, int& c1) {
    c0 = ks * p.chunks_per_split;
    c1 = min(p.n_chunks, c0 + p.chunks_per_split);
  };

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      if (p.wres && !p.wbuild) {  // the single column tile's W^T, once per CTA
        mbar_expect_tx(wfull, (uint32_t)(p.n_chunks * 2 * bbytes));
        for (int c = 0; c < p.n_chunks; ++c) {
          tma_load_2d(&tm_bhi, wfull, wres_hi(c), c * kBKf, 0);
          tma_load_2d(&tm_blo, wfull, wres_lo(c), c * kBKf, 0);
        }
      }
      for (int64_t item = item0; item < p.n_items; item += istep) {
        int64_t rt;
        int ct, ks, c0, c1;
        decode(item, rt, ct, ks);
        chunk_range(ks, c0, c1);
        for (int c = c0; c < c1; ++c) {
          if (p.gather && p.wres) break;  // nothing per stage for this thread
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], (p.gather ? 0u : xbytes) +
                                       (p.ystream ? bbytes / 2 : p.wres ? 0u : (p.wsplit ? 1u : 2u) * bbytes));
          if (!p.gather) tma_load_2d(&tm_x, &full[s], stage_x(s), c * kBKf, (int)row0(rt));
          if (p.ystream) {
            tma_load_2d(&tm_bhi, &full[s], stage_blo(s), c * kBKf, ct * (p.BN / 2));
          } else if (!p.wres) {
            const int brow = ct * p.BN + (int)crank * (p.BN / kCG);
            tma_load_2d(&tm_bhi, &full[s], stage_bhi(s), c * kBKf, brow);
            if (!p.wsplit) tma_load_2d(&tm_blo, &full[s], stage_blo(s), c * kBKf, brow);
          }
          if (++s == S) { s = 0; ph ^= 1; }
        }
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
      int s = 0;
      uint32_t ph = 0;
      for (int64_t item = item0; item < p.n_items; item += istep) {
        int64_t rt;
        int ct, ks, c0, c1;
        decode(item, rt, ct, ks);
        chunk_range(ks, c0, c1);
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
            const float2* rowp = p.Xg + nbase + roff[h] + kbase;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const bool kok = 2 * j < (p.K2 / 2) - c * 16;  // K tail
              cp_async16(dst + r * 128 + ((j ^ (r & 7)) << 4), ok && kok ? (const void*)(rowp + koff[j]) : (const void*)p.Xg,
                         ok && kok ? 16u : 0u);
            }
          }
          cp_async_arrive_noinc(&full[s]);
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (pair: the leader CTA issues for both) =====
    if (lane == 0 && leader) {
      int s = 0;
      uint32_t ph = 0;
      if (p.wres) mbar_wait(wfull, 0);
      int sa_m = 0;  // tsa: TMEM A stage
      int acc = 0;
      uint32_t aph = 0;
      for (int64_t item = item0; item < p.n_items; item += istep) {
        int64_t rt;
        int ct, ks, c0, c1;
        decode(item, rt, ct, ks);
        chunk_range(ks, c0, c1);
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
            if (p.tsa) {  // A = X hi/lo from TMEM stage sa_m (lane = row, column = k)
              const uint32_t ah = tmem_base + (uint32_t)(p.acol + sa_m * 64), alo = ah + 32;
              const uint32_t bh = smem_u32(stage_bhi(s)), bl = smem_u32(stage_blo(s));
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
              if (++sa_m == p.sa) sa_m = 0;
              if (++s == S) { s = 0; ph ^= 1; }
              continue;
            }
            const uint32_t ax = smem_u32(stage_x(s)), al = smem_u32(stage_xlo(s));
            const uint32_t bh = smem_u32(p.wres ? wres_hi(c) : stage_bhi(s));
            const uint32_t bl = smem_u32(p.wres ? wres_lo(c) : stage_blo(s));
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
            if (++s == S) { s = 0; ph ^= 1; }
          }
          if constexpr (kCG == 2) tc_commit_pair(&tfull[acc]);
          else tc_commit(&tfull[acc]);
          if (++acc == p.nbuf) { acc = 0; aph ^= 1; }
        }
      }
    }
  } else if (warp >= kConvWarp0 && warp < kConvWarp0 + 4) {
    // ===== converters: x -> hi (in place), lo (second buffer) =====
    const int t = threadIdx.x - kConvWarp0 * 32;  // 0..127
    int s = 0;
    uint32_t ph = 0;
    int sa_c = 0;        // tsa: TMEM A stage
    uint32_t aph_c = 0;
    for (int64_t item = item0; item < p.n_items; item += istep) {
      int64_t rt;
      int ct, ks, c0, c1;
      decode(item, rt, ct, ks);
      chunk_range(ks, c0, c1);
      for (int c = c0; c < c1; ++c) {
        mbar_wait(&full[s], ph);
        if (p.tsa) {
          // this thread's X row (= its TMEM lane) -> RN hi/lo -> TMEM A stage sa_c
          mbar_wait(&aempty[sa_c], aph_c ^ 1);
          tc_fence_after();
          const int q = warp - kConvWarp0, row = q * 32 + lane;
          const uint32_t xr = smem_u32(stage_x(s)) + (uint32_t)row * 128;
          const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(p.acol + sa_c * 64);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float hi[16], lo[16];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int j = 4 * h + jj;
              const float4 v = lds128(xr + (uint32_t)((j ^ (row & 7)) << 4));
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
        if (p.ystream) {
          // Y tile (SW128 rows m, 16-byte pieces j = complex k 2j, 2j+1) -> W^T rows 2m (Yr, -Yi) and
          // 2m+1 (Yi, Yr), split into hi/lo; all reads land in registers before the named barrier
          const uint32_t ys = smem_u32(stage_blo(s)), wh = smem_u32(stage_bhi(s)), wl = ys;
          float4 yin[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int idx = t + 128 * i;  // (m, j) = (idx >> 3, idx & 7)
            if (idx < 4 * p.BN) {
              const int m = idx >> 3, j = idx & 7;
              yin[i] = lds128(ys + (uint32_t)(m * 128 + ((j ^ (m & 7)) << 4)));
            }
          }
          asm volatile("bar.sync 2, 128;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int idx = t + 128 * i;
            if (idx < 4 * p.BN) {
              const int m = idx >> 3, j = idx & 7;
              const float4 v = yin[i];
#pragma unroll
              for (int b = 0; b < 2; ++b) {
                const float4 w = b ? make_float4(v.y, v.x, v.w, v.z) : make_float4(v.x, -v.y, v.z, -v.w);
                const int r = 2 * m + b;
                const uint32_t off = (uint32_t)(r * 128 + ((j ^ (r & 7)) << 4));
                float4 h, l;
                h.x = __uint_as_float(cvt_rna_tf32(w.x));
                h.y = __uint_as_float(cvt_rna_tf32(w.y));
                h.z = __uint_as_float(cvt_rna_tf32(w.z));
                h.w = __uint_as_float(cvt_rna_tf32(w.w));
                l.x = __uint_as_float(cvt_rna_tf32(w.x - h.x));
                l.y = __uint_as_float(cvt_rna_tf32(w.y - h.y));
                l.z = __uint_as_float(cvt_rna_tf32(w.z - h.z));
                l.w = __uint_as_float(cvt_rna_tf32(w.w - h.w));
                sts128(wh + off, h.x, h.y, h.z, h.w);
                sts128(wl + off, l.x, l.y, l.z, l.w);
              }
            }
          }
        }
        if (p.wsplit) {  // W^T tile: raw fp32 -> hi (in place), lo (second buffer); BN/16 float4 per thread
          const uint32_t ws = smem_u32(stage_bhi(s)), wl = smem_u32(stage_blo(s));
          for (int i0 = 0; i0 < p.BN / 16; i0 += 8) {
            float4 win[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (i0 + i < p.BN / 16) win[i] = lds128(ws + (uint32_t)((i0 + i) * 128 + t) * 16);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if (i0 + i >= p.BN / 16) break;
              const uint32_t off = (uint32_t)((i0 + i) * 128 + t) * 16;
              const float4 v = win[i];
              float4 h, l;
              h.x = __uint_as_float(cvt_rna_tf32(v.x));
              h.y = __uint_as_float(cvt_rna_tf32(v.y));
              h.z = __uint_as_float(cvt_rna_tf32(v.z));
              h.w = __uint_as_float(cvt_rna_tf32(v.w));
              l.x = __uint_as_float(cvt_rna_tf32(v.x - h.x));
              l.y = __uint_as_float(cvt_rna_tf32(v.y - h.y));
              l.z = __uint_as_float(cvt_rna_tf32(v.z - h.z));
              l.w = __uint_as_float(cvt_rna_tf32(v.w - h.w));
              sts128(ws + off, h.x, h.y, h.z, h.w);
              sts128(wl + off, l.x, l.y, l.z, l.w);
            }
          }
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
    if (p.wbuild) {
      // W^T rows r = 2m + b, fp32 column c2 = 2k + a of chunk c = c2 / 32: row 2m holds
      // (Yr, -Yi) at (2k, 2k+1), row 2m+1 holds (Yi, Yr); hi = rna_tf32(w), lo = rna_tf32(w - hi);
      // stored in the SW128 K-major layout TMA would have produced
      const int et = threadIdx.x - kEpiWarp0 * 32;  // 0..255
      const int K = p.K2 / 2, Mc = p.M2 / 2;
      if (p.K2 % kBKf) {  // K tail of the last chunk: zeros, as TMA's out-of-bounds fill
        const uint32_t wbytes = (uint32_t)(p.n_chunks * 2 * p.BN * kBKf * 4);
        for (uint32_t o = (uint32_t)et * 16; o < wbytes; o += 32 * kEpiWarps * 16)
          *reinterpret_cast<float4*>(wres + o) = make_float4(0.f, 0.f, 0.f, 0.f);
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      }
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
          yv[j] = __ldg(p.Yg + o);
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
    }
    const int q = warp & 3;
    const int half = (warp - kEpiWarp0) >> 2;
    const int row = q * 32 + lane;
    int acc = 0, sbuf = 0;
    uint32_t aph = 0;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const uint32_t tot = tmem_base + (uint32_t)(p.nbuf * p.BN) + lane_off;  // running total (flush mode)
    const bool swz = p.boxw == 32;
    const uint32_t pitch = (uint32_t)p.boxw * 4;
    uint8_t* my_stg = staging + (size_t)(warp - kEpiWarp0) * p.nstg * stg_bytes;
    const int nbox = p.BN / p.boxw;
    for (int64_t item = item0; item < p.n_items; item += istep) {
      int64_t rt;
      int ct, ks, c0, c1;
      decode(item, rt, ct, ks);
      chunk_range(ks, c0, c1);
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
          // this warp's staging buffer sbuf was used by its store two boxes ago
          if (lane == 0) {
            if (p.nstg == 2) bulk_wait_read1();
            else bulk_wait_read0();
          }
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
            tma_store_3d(&tm_c, my_stg + (size_t)sbuf * stg_bytes, ct * p.BN + cb, (int)row0(rt) + q * 32,
                         p.k_splits > 1 ? ks : 0);
            bulk_commit();
          }
          if (p.nstg == 2) sbuf ^= 1;
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

// W^T hi/lo [M2][K2]: Wt[2m+b][2k+a] = W[2k+a][2m+b], W block [[Yr, Yi], [-Yi, Yr]]
// One CTA per (complex column m, block of 256 complex k): the small operand is gathered
// with a per-CTA base offset plus a shared 256-entry table for the low k bits, and the
// four real-block entries are written as float2 pairs (coalesced along k).
__global__ void __launch_bounds__(256) tc_prep_kernel(const float2* __restrict__ Y, float* __restrict__ whi,
                                                      float* __restrict__ wlo, int nk, int nm, GemmDesc g) {
  pdl_wait();
  pdl_trigger();
  __shared__ int64_t lowtab[256];
  const int64_t K = (int64_t)1 << nk, K2 = 2 * K;
  const int64_t m = blockIdx.x;
  const int64_t k0 = (int64_t)blockIdx.y * 256;
  const int lowbits = nk < 8 ? nk : 8;
  {
    int t = threadIdx.x;
    int64_t o = 0;
    for (int i = 0; i < lowbits; ++i)
      if ((t >> i) & 1) o += g.syk[i];
    lowtab[t] = o;
  }
  int64_t base = 0;
  for (int i = 0; i < nm; ++i)
    if ((m >> i) & 1) base += g.sym[i];
  for (int i = lowbits; i < nk; ++i)
    if ((k0 >> i) & 1) base += g.syk[i];
  __syncthreads();
  const int64_t k = k0 + threadIdx.x;
  if (k >= K) return;
  const float2 y = Y[base + lowtab[threadIdx.x]];
  // W^T row 2m: (Yr, -Yi) at columns (2k, 2k+1); row 2m+1: (Yi, Yr)
  const float w[4] = {y.x, -y.y, y.y, y.x};
  const int64_t r0 = (2 * m) * K2 + 2 * k, r1 = (2 * m + 1) * K2 + 2 * k;
  if (!wlo) {  // on-chip split (wsplit): raw fp32 W^T only
    *reinterpret_cast<float2*>(whi + r0) = make_float2(w[0], w[1]);
    *reinterpret_cast<float2*>(whi + r1) = make_float2(w[2], w[3]);
    return;
  }
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

__global__ void tc_splitk_reduce(const float* __restrict__ part, float* __restrict__ C, int64_t n, int ks) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < ks; ++k) s += (double)part[(int64_t)k * n + i];
    C[i] = (float)s;
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

bool make_map_c(CUtensorMap* m, const void* ptr, uint64_t M2, uint64_t N, uint64_t splits, uint32_t boxw) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {M2, N, splits};
  cuuint64_t strides[2] = {M2 * 4, N * M2 * 4};
  cuuint32_t box[3] = {boxw, 32, 1};  // one epilogue warp's 32 rows
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, boxw == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint32_t box_inner, uint32_t box_outer) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int g_nsm = 0;
thread_local int t_tc_lanes = 1;  // slice lanes in flight on this thread (tc_set_concurrency)

// K per TMEM partial before a round-to-nearest flush: the MMA chain accumulates with an error
// growing linearly in its length.  Measured against torch complex64 (SURVEY 8(d) bar: <= 4x):
// 2 chunks (32 complex K) 1.1-3.2x everywhere; 4 chunks 2.2-3.2x for K >= 128 but 4.5x at
// K = 64 (one unflushed chain), and 5-10% faster on the tensor-bound steps (fewer drains of
// the single BN = 256 partial).  So: 4 chunks when K >= 128 complex, else 2.
constexpr int kGroupChunks = 2;
constexpr int kGroupChunksLongK = 4;

// Tile / split / flush decisions shared by the launcher and the workspace sizing.
TcParams plan_tc(int64_t N, int nk, int nm, bool ystream = false, int cg = 1, bool tsa = false) {
  if (!g_nsm) cudaDeviceGetAttribute(&g_nsm, cudaDevAttrMultiProcessorCount, 0);
  const int nsm = g_nsm ? g_nsm : 148;
  TcParams p{};
  p.N = N;
  p.K2 = 2 << nk;
  p.M2 = 2 << nm;
  p.n_chunks = (p.K2 + kBKf - 1) / kBKf;
  static const int env_group = getenv("TNQVM_TC_GROUP") ? atoi(getenv("TNQVM_TC_GROUP")) : 0;
  const int group_chunks =
      env_group > 0 ? env_group : (p.n_chunks >= 8 && !ystream ? kGroupChunksLongK : kGroupChunks);
  const bool flush = p.n_chunks > group_chunks;
  static const int env_bn = getenv("TNQVM_TC_FLUSH_BN") ? atoi(getenv("TNQVM_TC_FLUSH_BN")) : 256;
  static const int env_bnmax = getenv("TNQVM_TC_BN") ? atoi(getenv("TNQVM_TC_BN")) : 256;
  p.BN = std::min(flush ? env_bn : env_bnmax, std::max(16, p.M2));
  p.n_col_tiles = (p.M2 + p.BN - 1) / p.BN;
  p.n_row_tiles = (int)((N + kBM * cg - 1) / (kBM * cg));  // CTA pairs own 256-row tiles
  const int64_t tiles = (int64_t)p.n_row_tiles * p.n_col_tiles;
  const int units = nsm / cg;
  p.k_splits = 1;
  if (tiles < 2 * units && p.n_chunks >= 8)  // split K when the output tiles cannot fill the machine
    p.k_splits = std::max(1, (int)std::min<int64_t>((2 * units + tiles - 1) / tiles, p.n_chunks / 4));
  p.chunks_per_split = (p.n_chunks + p.k_splits - 1) / p.k_splits;
  p.k_splits = (p.n_chunks + p.chunks_per_split - 1) / p.chunks_per_split;
  p.group_chunks = std::min(p.chunks_per_split, group_chunks);
  p.n_items = tiles * p.k_splits;
  p.boxw = p.M2 >= 32 ? 32 : 16;  // TMA clips columns beyond M2
  const size_t wres_bytes = (size_t)p.n_chunks * 2 * p.BN * kBKf * 4;
  p.wres = (!ystream && cg == 1 && p.n_col_tiles == 1 && p.k_splits == 1 && wres_bytes <= 64 * 1024) ? 1 : 0;
  p.tsa = (tsa && cg == 1 && !p.wres && !ystream && p.BN <= 128) ? 1 : 0;
  const uint32_t stage_bytes = (p.tsa ? 1 : 2) * kBM * kBKf * 4 + (p.wres ? 0 : 2 * (p.BN / cg) * kBKf * 4);
  const size_t avail = 225 * 1024;  // 227 KB opt-in minus alignment slack and barriers
  // one staging buffer per epilogue warp: the freed shared memory buys input stages, which
  // measured faster or equal on every probed shape (tools/tc_sweep.sh)
  static const int env_nstg = getenv("TNQVM_TC_NSTG") ? atoi(getenv("TNQVM_TC_NSTG")) : 1;
  p.nstg = env_nstg;
  for (int ns = env_nstg; ns >= 1; --ns) {
    const size_t fixed = (size_t)kEpiWarps * ns * 32 * p.boxw * 4 + (p.wres ? wres_bytes : 0);
    p.nstg = ns;
    if (fixed + 2 * (size_t)stage_bytes <= avail) {
      p.stages = std::min<int>(6, (int)((avail - fixed) / stage_bytes));
      break;
    }
    p.stages = 2;
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

}  // namespace

// ystream: C[N][M] = X[N][K] * Y[M][K]^T (complex64, both K-fastest with one K order), M <= 128
bool tc_ystream_supported(int64_t N, int nk, int nm) {
  return N >= 1 && nk >= 1 && nk <= 30 && nm >= 1 && nm <= 7 && get_encode() != nullptr;  // C rows: 16-byte multiples (TMA)
}
size_t tc_ystream_part_bytes(int64_t N, int nk, int nm) {
  TcParams p = plan_tc(N, nk, nm, true);
  return p.k_splits > 1 ? (size_t)p.k_splits * N * p.M2 * 4 : 0;
}
void launch_gemm_tc_ystream(const void* X, const void* Y, void* C, int64_t N, int nk, int nm, void* part,
                            cudaStream_t st) {
  TcParams p = plan_tc(N, nk, nm, true);
  const int K2 = p.K2, M2 = p.M2;
  p.wres = 0;
  p.wsplit = 0;
  p.wbuild = 0;
  p.ystream = 1;
  p.gather = 0;
  p.C = reinterpret_cast<float*>(C);
  p.part = p.k_splits > 1 ? reinterpret_cast<float*>(part) : nullptr;
  CUtensorMap mx, my, mc;
  bool ok = make_map_c(&mc, p.k_splits > 1 ? (const void*)p.part : (const void*)p.C, (uint64_t)M2, (uint64_t)N,
                       (uint64_t)p.k_splits, (uint32_t)p.boxw) &&
            make_map(&mx, X, (uint64_t)K2, (uint64_t)N, kBKf, kBM) &&
            make_map(&my, Y, (uint64_t)K2, (uint64_t)(M2 / 2), kBKf, (uint32_t)(p.BN / 2));
  if (!ok) {
    fprintf(stderr, "tnqvm: cuTensorMapEncodeTiled failed\n");
    return;
  }
  // stages: X hi/lo + W^T hi/lo per stage (the Y tile lands in the W^T lo buffer)
  const uint32_t stage_bytes = 2 * kBM * kBKf * 4 + 2 * p.BN * kBKf * 4;
  const size_t smem = 1024 + (size_t)p.stages * stage_bytes + (size_t)kEpiWarps * p.nstg * 32 * p.boxw * 4 +
                      (3 * p.stages + 5) * 8 + 16;
  cudaFuncSetAttribute(tc_gemm_kernel_t<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = (int)std::min<int64_t>(p.n_items, g_nsm);
  launch_pdl(tc_gemm_kernel_t<1>, grid, kThreadsTC, smem, st, mx, my, my, mc, p);
  if (p.k_splits > 1) {
    int64_t n = N * (int64_t)M2;
    int blocks = (int)std::min<int64_t>((n + 255) / 256, 8192);
    launch_pdl(tc_splitk_reduce, blocks, 256, 0, st, p.part, reinterpret_cast<float*>(C), n, p.k_splits);
  }
}

void tc_set_concurrency(int lanes) { t_tc_lanes = lanes < 1 ? 1 : lanes; }

size_t tc_part_bytes(int64_t N, int nk, int nm) {  // enough for either CTA grouping
  size_t b = 0;
  for (int cg = 1; cg <= 2; ++cg) {
    TcParams p = plan_tc(N, nk, nm, false, cg);
    if (p.k_splits > 1) b = std::max(b, (size_t)p.k_splits * N * p.M2 * 4);
  }
  return b;
}
size_t tc_wbuf_bytes(int64_t N, int nk, int nm) { return ((size_t)32 << (nk + nm)) + tc_part_bytes(N, nk, nm); }

bool tc_supported(int nk, int nm) {
  // X rows must be 16-byte multiples for TMA (K >= 2); W^T must fit comfortably
  return nk >= 1 && nk <= 20 && nm <= 16 && nk + nm <= 26 && get_encode() != nullptr;
}

// Persistent-grid cap: with several slice lanes in flight, a GEMM that holds every SM (one
// 230 KB CTA per SM) serialises the lanes; capping each GEMM's grid lets the lanes' GEMMs
// run side by side (C2, 8 lanes: 148 SMs 279, 74 292, 37 296 amplitudes/s; 1 lane: 148 208,
// 74 151; 4 GPUs = 2 lanes per rank: 148 856, 74 722).  The runtime sets the cap from its
// lane count (tc_set_concurrency): <= 2 lanes all SMs, 3-4 half, 5+ a quarter; TNQVM_TC_GRID
// overrides.
int tc_grid_cap(int64_t n_items) {
  static const int env = getenv("TNQVM_TC_GRID") ? atoi(getenv("TNQVM_TC_GRID")) : 0;
  if (env > 0) return std::min(env, g_nsm);
  // long GEMMs (C3: tens of thousands of tiles) keep the whole machine: measured 3% slower
  // on C3 at 2 lanes with the cap; the cap is for the short, latency-dominated ones
  if (n_items >= (int64_t)16 * g_nsm) return g_nsm;
  const int l = t_tc_lanes;
  const int cap = l <= 2 ? g_nsm : l <= 4 ? g_nsm / 2 : g_nsm / 4;
  return std::max(2, cap & ~1);
}

// Streamed-W^T steps: A from TMEM in a single CTA when BN <= 128 (TNQVM_TC_TSA=0: off), else CTA
// pairs (cta_group::2) with >= 2 pair tiles (TNQVM_TC_CG=1: off)
bool choose_tsa(int64_t N, int nk, int nm) {
  static const int env_tsa = getenv("TNQVM_TC_TSA") ? atoi(getenv("TNQVM_TC_TSA")) : 1;
  static const int env_wsplit = getenv("TNQVM_TC_WSPLIT") ? atoi(getenv("TNQVM_TC_WSPLIT")) : 0;
  if (!env_tsa || env_wsplit) return false;
  TcParams p1 = plan_tc(N, nk, nm);
  return !p1.wres && p1.BN <= 128;
}
int choose_cg(int64_t N, int nk, int nm) {
  static const int env_cg = getenv("TNQVM_TC_CG") ? atoi(getenv("TNQVM_TC_CG")) : 2;
  if (env_cg != 2 || choose_tsa(N, nk, nm)) return 1;
  TcParams p1 = plan_tc(N, nk, nm);
  static const int env_wsplit = getenv("TNQVM_TC_WSPLIT") ? atoi(getenv("TNQVM_TC_WSPLIT")) : 0;
  if (p1.wres || env_wsplit || p1.BN < 32 || N < 2 * kBM * 2) return 1;
  return 2;
}

void launch_gemm_tc(const GemmDesc& g, void* wbuf, cudaStream_t st) {
  const int cg = choose_cg(g.N, g.nk, g.nm);
  TcParams p = plan_tc(g.N, g.nk, g.nm, false, cg, choose_tsa(g.N, g.nk, g.nm));
  const int K2 = p.K2, M2 = p.M2;
  float* whi = reinterpret_cast<float*>(wbuf);
  float* wlo = whi + (size_t)K2 * M2;
  static const bool no_wbuild = getenv("TNQVM_TC_NO_WBUILD") != nullptr;
  p.wbuild = p.wres && p.BN == M2 && g.nk + g.nm <= 11 && !no_wbuild;  // <= 8 Y values per epilogue thread
  // off by default: measured 15-20% slower on tensor-bound shapes -- the converters' extra shared-memory
  // traffic competes with the MMA operand reads (the kernel is shared-memory-bandwidth bound)
  static const int env_wsplit = getenv("TNQVM_TC_WSPLIT") ? atoi(getenv("TNQVM_TC_WSPLIT")) : 0;
  p.wsplit = !p.wres && env_wsplit;
  if (p.wbuild) {
    p.Yg = reinterpret_cast<const float2*>(g.Y);
    p.nm = g.nm;
    for (int i = 0; i < g.nk; ++i) p.syk[i] = g.syk[i];
    for (int i = 0; i < g.nm; ++i) p.sym[i] = g.sym[i];
  } else {
    dim3 grid((unsigned)(M2 / 2), (unsigned)std::max<int64_t>(1, ((K2 / 2) + 255) / 256));
    launch_pdl(tc_prep_kernel, grid, 256, 0, st, reinterpret_cast<const float2*>(g.Y), whi, p.wsplit ? nullptr : wlo,
               g.nk, g.nm, g);
  }
  p.C = reinterpret_cast<float*>(g.C);
  p.part = p.k_splits > 1 ? wlo + (size_t)K2 * M2 : nullptr;  // partials follow W^T in wbuf
  p.gather = g.gather;
  p.nn = g.nn;
  p.nk = g.nk;
  p.Xg = reinterpret_cast<const float2*>(g.X);
  if (g.gather) {
    for (int i = 0; i < g.nn && i < 40; ++i) p.sxn[i] = g.sxn[i];
    for (int i = 0; i < g.nk && i < 40; ++i) p.sxk[i] = g.sxk[i];
  }
  CUtensorMap mx, mbh, mbl, mc;
  bool ok = make_map_c(&mc, p.k_splits > 1 ? (const void*)p.part : (const void*)p.C, (uint64_t)M2, (uint64_t)g.N,
                       (uint64_t)p.k_splits, (uint32_t)p.boxw) &&
            (g.gather ? make_map(&mx, whi, (uint64_t)K2, (uint64_t)M2, kBKf, (uint32_t)p.BN)  // unused
                      : make_map(&mx, g.X, (uint64_t)K2, (uint64_t)g.N, kBKf, kBM)) &&
            make_map(&mbh, whi, (uint64_t)K2, (uint64_t)M2, kBKf, (uint32_t)(p.BN / cg)) &&
            make_map(&mbl, wlo, (uint64_t)K2, (uint64_t)M2, kBKf, (uint32_t)(p.BN / cg));
  if (!ok) {
    fprintf(stderr, "tnqvm: cuTensorMapEncodeTiled failed\n");
    return;
  }
  const uint32_t stage_bytes = (p.tsa ? 1 : 2) * kBM * kBKf * 4 + (p.wres ? 0 : 2 * (p.BN / cg) * kBKf * 4);
  const size_t smem = 1024 + (size_t)p.stages * stage_bytes + (p.wres ? (size_t)p.n_chunks * 2 * p.BN * kBKf * 4 : 0) +
                      (size_t)kEpiWarps * p.nstg * 32 * p.boxw * 4 + (3 * p.stages + 8 + 4) * 8 + 16;
  if (cg == 2) {
    cudaFuncSetAttribute(tc_gemm_kernel_t<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int pairs = (int)std::min<int64_t>(p.n_items, tc_grid_cap(2 * p.n_items) / 2);
    launch_pdl_cluster(tc_gemm_kernel_t<2>, 2 * pairs, kThreadsTC, smem, st, 2u, mx, mbh, mbl, mc, p);
  } else {
    cudaFuncSetAttribute(tc_gemm_kernel_t<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = (int)std::min<int64_t>(p.n_items, tc_grid_cap(p.n_items));
    launch_pdl(tc_gemm_kernel_t<1>, grid, kThreadsTC, smem, st, mx, mbh, mbl, mc, p);
  }
  if (p.k_splits > 1) {
    int64_t n = g.N * (int64_t)M2;
    int blocks = (int)std::min<int64_t>((n + 255) / 256, 8192);
    launch_pdl(tc_splitk_reduce, blocks, 256, 0, st, p.part, reinterpret_cast<float*>(g.C), n, p.k_splits);
  }
}


}  // namespace dev
}  // namespace tnqvm
