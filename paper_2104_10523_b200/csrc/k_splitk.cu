// a7 (split-K, any layout): the last steps of a sliced contraction are a
// huge K contracted into a tiny output (N*M <= 16 amplitudes / open-qubit values).  The two
// operands are produced by earlier steps in whatever order of the contracted modes suited
// those steps; reordering one of them to match the other would cost a full read + write of
// a multi-GB tensor.  This kernel reads both in their stored layouts instead:
//   * the K index is split into a 9-bit tile index t (X's 5 fastest contracted modes plus
//     Y's fastest ones) and a rest index r;
//   * per tile, X is read straight into registers (thread owns t = tid, tid + 256) and Y is
//     read in Y's own fastest-mode order and scattered into shared memory at position t --
//     both streams are coalesced, the transpose happens on chip;
//   * fp32 products are summed per thread over <= 64 terms, then in fp64; one CTA per
//     contiguous range of r (fixed grid: deterministic), partials reduced in fp64.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "kernels.hpp"
#include "pdl.cuh"

namespace tnqvm {
namespace dev {
namespace {

template <typename T> struct C2;
template <> struct C2<float> { using t = float2; };
template <> struct C2<double> { using t = double2; };

constexpr int kThr = 256;
constexpr int kTileBits = 9;  // T = 512 K values per tile, 2 per thread
constexpr int kFlush = 32;    // tiles per fp32 partial (64 terms per thread)

struct SplitKDesc {
  const void* X;
  const void* Y;
  void* C;
  int u, nr;
  int64_t xt[kTileBits], yt[kTileBits];  // strides of tile bit j
  int32_t yv2t[kTileBits];               // v bit i (Y-coalesced order) -> tile bit
  int64_t xr[48], yr[48];                // strides of rest bits
  int64_t dxr[48], dyr[48];              // r -> r + 1 with carry out of bit j: offset += d*r[j]
  int64_t xn[64], ym[64], cn[64], cm[64];
  int xvec;     // big kernel, complex64: X tile pairs (v, v + 1) are adjacent 16-byte-aligned elements
  int blocked;  // big kernel: register-blocked outputs (complex128)
  const int64_t* delta;  // batch: unit b's X / Y / C at + delta[{xsel, 1 - xsel, 2} * nb + b] elements (blockIdx.y = b)
  int nb, xsel;          // xsel = 1: the caller's Y is the kernel's X (operands swapped)
};
constexpr int kMaxCtas = 1024;
// unit blockIdx.y's operands and partial slab
template <typename V>
__device__ __forceinline__ void unit_ptrs(const SplitKDesc& d, const V*& X, const V*& Y, V*& C, int64_t& poff,
                                          int NP) {
  const int b = blockIdx.y;
  X = reinterpret_cast<const V*>(d.X) + (d.delta ? d.delta[d.xsel * d.nb + b] : 0);
  Y = reinterpret_cast<const V*>(d.Y) + (d.delta ? d.delta[(1 - d.xsel) * d.nb + b] : 0);
  C = reinterpret_cast<V*>(d.C) + (d.delta ? d.delta[2 * d.nb + b] : 0);
  poff = (int64_t)b * kMaxCtas * NP;
}

// Larger outputs (16 < N*M <= 4096, N, M <= 64): 32-value K tiles of every X row and Y row
// are staged in padded shared memory through a cp.async ring (each operand gathered in its
// own fastest-mode order, per-bit strides); each thread owns a PN x PM register block of
// outputs (rows tn + TN*i, columns tm + TM*j), so a shared-memory value feeds PM or PN
// complex multiply-adds.  complex128 is shared-memory-bandwidth bound with one output per
// thread (32 B of operands per complex MAC), so it takes 2 x 2 register blocks and, when
// the blocks need fewer than 256 threads, KG thread groups that split each K tile
// (k = kg, kg + KG, ...) and are summed in a fixed order in shared memory at the end.
// (complex64 keeps one output per thread: its steps are bound by the latency of the
// scattered operand gathers, and the blocked variant measured slower on C2.)
constexpr int kBigBits = 5;
struct BigBlock { int PN, PM, TN, TM, KG; };
__host__ __device__ inline BigBlock big_block(int N, int M, int threads, bool blocked) {
  if (!blocked) {  // TM = min(M, 16), TN = min(N, threads / TM)
    BigBlock b{1, 1, 1, M < 16 ? M : 16, 1};
    b.TN = N < threads / b.TM ? N : threads / b.TM;
    b.PN = N / b.TN;
    b.PM = M / b.TM;
    return b;
  }
  BigBlock b{1, 1, N, M, 1};
  while (b.PN * b.PM < 4 || b.TN * b.TM > threads) {
    const int lim = b.TN * b.TM > threads ? 4 : 2;
    const bool grow_n = b.PN < lim && 2 * b.PN <= N && (N / b.PN >= M / b.PM || !(b.PM < lim && 2 * b.PM <= M));
    if (grow_n) b.PN *= 2;
    else if (b.PM < lim && 2 * b.PM <= M) b.PM *= 2;
    else break;
    b.TN = N / b.PN;
    b.TM = M / b.PM;
  }
  b.KG = threads / (b.TN * b.TM);
  if (b.KG < 1) b.KG = 1;
  if (b.KG > (1 << kBigBits)) b.KG = 1 << kBigBits;
  return b;
}
template <typename T>
__host__ __device__ constexpr int big_stages() { return sizeof(T) == 4 ? 4 : 2; }
// k = 0, STEP, 2 STEP, ... < KT of one staged tile: a[i] = pa[i][k], b[j] = pb[j][k],
// complex multiply-add into the PN x PM register block (fp32 FMAs in a fixed order)
template <typename T, int kBigP, int KT, int STEP>
__device__ __forceinline__ void tile_mac(const typename C2<T>::t* const (&pa)[kBigP],
                                         const typename C2<T>::t* const (&pb)[kBigP], int PN, int PM,
                                         T (&re)[kBigP][kBigP], T (&im)[kBigP][kBigP]) {
  using V = typename C2<T>::t;
#pragma unroll
  for (int k = 0; k < KT; k += STEP) {
    V a[kBigP], b[kBigP];
#pragma unroll
    for (int i = 0; i < kBigP; ++i)
      if (i < PN) a[i] = pa[i][k];
#pragma unroll
    for (int j = 0; j < kBigP; ++j)
      if (j < PM) b[j] = pb[j][k];
#pragma unroll
    for (int i = 0; i < kBigP; ++i)
#pragma unroll
      for (int j = 0; j < kBigP; ++j)
        if (i < PN && j < PM) {
          re[i][j] = fma(a[i].x, b[j].x, fma(-a[i].y, b[j].y, re[i][j]));
          im[i][j] = fma(a[i].x, b[j].y, fma(a[i].y, b[j].x, im[i][j]));
        }
  }
}

template <typename T, int kBigP>  // kBigP: max register block per dimension (1, 2, 4)
__global__ void __launch_bounds__(kThr, kBigP >= 4 ? 1 : kBigP == 1 ? 3 : 2) splitk_big_kernel(SplitKDesc d, int nn, int nm,
                                                                              double2* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  using V = typename C2<T>::t;
  constexpr int kBigStages = big_stages<T>();
  // complex64 rows are padded to an even length so 16-byte copies land aligned
  constexpr int KT = 1 << kBigBits, PADW = sizeof(T) == 4 ? KT + 2 : KT + 1, PER = (128 * KT) / kThr;
  const int N = 1 << nn, M = 1 << nm, NP = N * M, rows = N + M;
  extern __shared__ __align__(16) unsigned char sks_raw[];
  V* sm = reinterpret_cast<V*>(sks_raw);  // [kBigStages][rows][PADW]: X rows then Y rows
  const V* X;
  const V* Y;
  V* Cu;
  int64_t poff;
  unit_ptrs<V>(d, X, Y, Cu, poff, NP);
  part += poff;
  (void)Cu;
  const int tid = threadIdx.x;
  const int v = tid & (KT - 1);  // this thread's tile position in load order (fixed: 256 % KT == 0)
  const int Tn = 1 << d.u;
  int64_t xo = 0, yo = 0;
  int ypos = 0;
  for (int i = 0; i < d.u; ++i)
    if ((v >> i) & 1) {
      xo += d.xt[i];
      yo += d.yt[d.yv2t[i]];
      ypos |= 1 << d.yv2t[i];
    }
  const bool vok = v < Tn;
  // vectorised X gather (d.xvec): thread copies tile positions v2, v2 + 1 of X rows
  // tid / 16 + 16 i as one 16-byte cp.async (half the L1 requests of the 8-byte gather,
  // which ncu shows as the limiter: L1/TEX 70% busy at 20% of DRAM bandwidth)
  const int v2 = 2 * (tid & (KT / 2 - 1));
  int64_t xo2 = 0;
  for (int i = 0; i < d.u; ++i)
    if ((v2 >> i) & 1) xo2 += d.xt[i];
  const bool v2ok = v2 < Tn;
  const int64_t ntile = (int64_t)1 << d.nr;
  const int64_t r0 = ntile * blockIdx.x / gridDim.x, r1 = ntile * (blockIdx.x + 1) / gridDim.x;
  // kBigStages-deep cp.async ring: tile r + kBigStages - 1 is in flight while tile r is
  // multiplied; `nxt` / (bx, by) track the next tile to issue (carry-delta offsets)
  int64_t nxt = r0, bx = 0, by = 0;
  for (int i = 0; i < d.nr; ++i)
    if ((r0 >> i) & 1) { bx += d.xr[i]; by += d.yr[i]; }
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
  auto issue = [&]() {
    if (nxt < r1) {
      const int stg = (int)((nxt - r0) % kBigStages);
      const uint32_t sb = sbase + (uint32_t)((size_t)stg * rows * PADW * sizeof(V));
      if (sizeof(V) == 8 && d.xvec) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // N <= 64 rows, 16 per pass
          const int row = (tid >> 4) + 16 * i;
          if (v2ok && row < N) {
            const V* src = X + d.xn[row] + bx + xo2;
            const uint32_t dst = sb + (uint32_t)((row * PADW + v2) * sizeof(V));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // M <= 64 rows, 8 per pass
          const int yr = (tid >> 5) + 8 * i;
          if (vok && yr < M) {
            const V* src = Y + d.ym[yr] + by + yo;
            const uint32_t dst = sb + (uint32_t)(((N + yr) * PADW + ypos) * sizeof(V));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
          }
        }
      } else
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int row = (tid + i * kThr) / KT;
        if (vok && row < rows) {
          const V* src = row < N ? X + d.xn[row] + bx + xo : Y + d.ym[row - N] + by + yo;
          const uint32_t dst = sb + (uint32_t)((row * PADW + (row < N ? v : ypos)) * sizeof(V));
          if (sizeof(V) == 8)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
          else
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        }
      }
      ++nxt;
      if (nxt < r1) {
        const int j = __ffsll((unsigned long long)nxt) - 1;
        bx += d.dxr[j];
        by += d.dyr[j];
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // tile positions v >= Tn (K < KT) stay zero: clear every stage once
  for (int e = tid; e < kBigStages * rows * PADW; e += kThr) {
    V z;
    z.x = 0;
    z.y = 0;
    sm[e] = z;
  }
  __syncthreads();
  for (int s = 0; s < kBigStages - 1; ++s) issue();
  // output block of this thread and its K group
  const BigBlock bb = big_block(N, M, kThr, sizeof(T) == 8 || d.blocked);
  const int TM = bb.TM, TN = bb.TN, PN = bb.PN, PM = bb.PM, KG = bb.KG;
  const int og = tid % (TN * TM), kg = tid / (TN * TM);
  const bool act = kg < KG;
  const int tn = og / TM, tm = og % TM;
  double dr[kBigP][kBigP], di[kBigP][kBigP];
#pragma unroll
  for (int i = 0; i < kBigP; ++i)
#pragma unroll
    for (int j = 0; j < kBigP; ++j) dr[i][j] = di[i][j] = 0.0;
  for (int64_t r = r0; r < r1; ++r) {
    asm volatile("cp.async.wait_group %0;" ::"n"(kBigStages - 2) : "memory");
    __syncthreads();  // tile r landed for every thread; the stage issued next was consumed
    issue();
    const V* sb = sm + (size_t)((r - r0) % kBigStages) * rows * PADW;
    if (act) {
      T re[kBigP][kBigP], im[kBigP][kBigP];
#pragma unroll
      for (int i = 0; i < kBigP; ++i)
#pragma unroll
        for (int j = 0; j < kBigP; ++j) re[i][j] = im[i][j] = 0;
      if (KG == 1 || (sizeof(T) == 4 && (KG == 2 || KG == 4 || KG == 8))) {  // (complex128: register-bound)
        // K groups of 1, 2, 4 or 8: the thread's k = kg, kg + KG, ... of the tile with a
        // compile-time trip count, so every shared-memory operand load is a fixed offset
        // from a per-thread row pointer (the generic loop below spends about as many
        // integer instructions on addresses and loop control as on the FMAs; ncu: this
        // kernel is L1/TEX- and issue-bound, not DRAM-bound).  Same summation order.
        const V* pa[kBigP];
        const V* pb[kBigP];
#pragma unroll
        for (int i = 0; i < kBigP; ++i) {
          pa[i] = sb + (tn + TN * (i < PN ? i : 0)) * PADW + kg;
          pb[i] = sb + (N + tm + TM * (i < PM ? i : 0)) * PADW + kg;
        }
        if (KG == 1) tile_mac<T, kBigP, KT, 1>(pa, pb, PN, PM, re, im);
        else if (sizeof(T) == 4) {
          if (KG == 2) tile_mac<T, kBigP, KT, 2>(pa, pb, PN, PM, re, im);
          else if (KG == 4) tile_mac<T, kBigP, KT, 4>(pa, pb, PN, PM, re, im);
          else tile_mac<T, kBigP, KT, 8>(pa, pb, PN, PM, re, im);
        }
      } else
#pragma unroll 4
      for (int k = kg; k < KT; k += KG) {
        V a[kBigP], b[kBigP];
#pragma unroll
        for (int i = 0; i < kBigP; ++i)
          if (i < PN) a[i] = sb[(tn + TN * i) * PADW + k];
#pragma unroll
        for (int j = 0; j < kBigP; ++j)
          if (j < PM) b[j] = sb[(N + tm + TM * j) * PADW + k];
#pragma unroll
        for (int i = 0; i < kBigP; ++i)
#pragma unroll
          for (int j = 0; j < kBigP; ++j)
            if (i < PN && j < PM) {
              re[i][j] = fma(a[i].x, b[j].x, fma(-a[i].y, b[j].y, re[i][j]));
              im[i][j] = fma(a[i].x, b[j].y, fma(a[i].y, b[j].x, im[i][j]));
            }
      }
#pragma unroll
      for (int i = 0; i < kBigP; ++i)
#pragma unroll
        for (int j = 0; j < kBigP; ++j) {
          dr[i][j] += (double)re[i][j];
          di[i][j] += (double)im[i][j];
        }
    }
  }
  if (KG > 1) {
    // K groups -> one partial per output: fp64 staging in shared memory, summed in kg order
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    double2* red = reinterpret_cast<double2*>(sks_raw);  // [KG][TN*TM][PN*PM]
    const int OG = TN * TM, Q = PN * PM;
    if (act)
#pragma unroll
      for (int i = 0; i < kBigP; ++i)
#pragma unroll
        for (int j = 0; j < kBigP; ++j)
          if (i < PN && j < PM) red[((size_t)kg * OG + og) * Q + i * PM + j] = make_double2(dr[i][j], di[i][j]);
    __syncthreads();
    for (int e = tid; e < OG * Q; e += kThr) {
      double2 a = red[e];
      for (int g = 1; g < KG; ++g) {
        const double2 v = red[(size_t)g * OG * Q + e];
        a.x += v.x;
        a.y += v.y;
      }
      const int o = e / Q, q = e % Q, i = q / PM, j = q % PM;
      const int pp = (o / TM + TN * i) * M + (o % TM) + TM * j;
      part[(int64_t)blockIdx.x * NP + pp] = a;
    }
    return;
  }
  if (act)
#pragma unroll
    for (int i = 0; i < kBigP; ++i)
#pragma unroll
      for (int j = 0; j < kBigP; ++j)
        if (i < PN && j < PM) {
          const int pp = (tn + TN * i) * M + tm + TM * j;
          part[(int64_t)blockIdx.x * NP + pp] = make_double2(dr[i][j], di[i][j]);
        }
}

template <typename T>
__global__ void __launch_bounds__(kThr) splitk_big_final(SplitKDesc d, int nm, int NP, const double2* __restrict__ part_in,
                                                         int G) {
  pdl_wait();
  pdl_trigger();
  // one CTA per pair: strided fp64 partial sums, then a fixed-shape tree (deterministic)
  using V = typename C2<T>::t;
  __shared__ double2 red[kThr];
  const int p = blockIdx.x;
  const V* Xu;
  const V* Yu;
  V* Cu;
  int64_t poff;
  unit_ptrs<V>(d, Xu, Yu, Cu, poff, NP);
  const double2* part = part_in + poff;
  double2 acc = make_double2(0.0, 0.0);
  for (int g = threadIdx.x; g < G; g += kThr) {
    const double2 v = part[(int64_t)g * NP + p];
    acc.x += v.x;
    acc.y += v.y;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kThr / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      red[threadIdx.x].x += red[threadIdx.x + s].x;
      red[threadIdx.x].y += red[threadIdx.x + s].y;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    V v;
    v.x = (T)red[0].x;
    v.y = (T)red[0].y;
    Cu[d.cn[p >> nm] + d.cm[p & ((1 << nm) - 1)]] = v;
  }
}

// CTA b walks the contiguous rest range [b*R/G, (b+1)*R/G) with incremental (carry-delta)
// offsets; complex64 partial sums are kept in fp32 registers for kFlush tiles and then
// added into per-thread fp64 slots in shared memory (complex128: fp64 registers).
template <typename T, int NN, int MM>
constexpr int sks_min_blocks() { return NN <= 4 && NN * MM * sizeof(T) <= 32 ? 3 : 1; }

template <typename T, int NN, int MM>
__global__ void __launch_bounds__(kThr, (sks_min_blocks<T, NN, MM>())) splitk_strided_kernel(SplitKDesc d, double2* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  using V = typename C2<T>::t;
  constexpr int NP = NN * MM;
  constexpr bool kF32 = sizeof(T) == 4;
  extern __shared__ __align__(16) unsigned char sks_raw[];
  auto ys = reinterpret_cast<V(*)[MM][1 << kTileBits]>(sks_raw);  // [2][MM][T]
  double* sacc = reinterpret_cast<double*>(sks_raw + 2 * MM * (1 << kTileBits) * sizeof(V));  // [2*NP][kThr]
  const V* X;
  const V* Y;
  V* Cu;
  int64_t poff;
  unit_ptrs<V>(d, X, Y, Cu, poff, NP);
  part += poff;
  (void)Cu;
  const int Tn = 1 << d.u;
  const int tid = threadIdx.x;
  // per-thread tile offsets (fixed over tiles)
  int64_t xo[2], yo[2];
  int yti[2];
  bool tv[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int t = tid + kThr * j;
    tv[j] = t < Tn;
    int64_t a = 0, b = 0;
    int ti = 0;
    for (int i = 0; i < d.u; ++i) {
      if ((t >> i) & 1) {
        a += d.xt[i];
        b += d.yt[d.yv2t[i]];
        ti |= 1 << d.yv2t[i];
      }
    }
    xo[j] = a;
    yo[j] = b;
    yti[j] = ti;
  }
  if (kF32)
    for (int p = 0; p < 2 * NP; ++p) sacc[p * kThr + tid] = 0.0;

  T re[NP], im[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) re[p] = im[p] = 0;
  const int64_t ntile = (int64_t)1 << d.nr;
  const int64_t r0 = ntile * blockIdx.x / gridDim.x, r1 = ntile * (blockIdx.x + 1) / gridDim.x;
  int64_t bx = 0, by = 0;
  for (int i = 0; i < d.nr; ++i)
    if ((r0 >> i) & 1) { bx += d.xr[i]; by += d.yr[i]; }
  // register prefetch of the next tile while the current one is multiplied; the Y tile is
  // double-buffered in shared memory so one barrier per tile suffices
  V xv[NN][2], yl[MM][2];
  auto load = [&](bool in) {
#pragma unroll
    for (int m = 0; m < MM; ++m)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (in && tv[j]) yl[m][j] = __ldcs(Y + d.ym[m] + by + yo[j]);
        else { yl[m][j].x = 0; yl[m][j].y = 0; }
      }
#pragma unroll
    for (int n = 0; n < NN; ++n)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (in && tv[j]) xv[n][j] = __ldcs(X + d.xn[n] + bx + xo[j]);
        else { xv[n][j].x = 0; xv[n][j].y = 0; }
      }
  };
  load(r0 < r1);
  int buf = 0, cnt = 0;
  for (int64_t r = r0; r < r1; ++r, buf ^= 1) {
    // Y tile -> shared memory (loaded coalesced in Y's order, stored at tile position)
#pragma unroll
    for (int m = 0; m < MM; ++m)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (tv[j]) ys[buf][m][yti[j]] = yl[m][j];
    V xc[NN][2];
#pragma unroll
    for (int n = 0; n < NN; ++n) { xc[n][0] = xv[n][0]; xc[n][1] = xv[n][1]; }
    __syncthreads();
    if (r + 1 < r1) {
      const int j = __ffsll((unsigned long long)(r + 1)) - 1;
      bx += d.dxr[j];
      by += d.dyr[j];
    }
    load(r + 1 < r1);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int t = tid + kThr * j;
      V yv[MM];
#pragma unroll
      for (int m = 0; m < MM; ++m) {
        if (tv[j]) yv[m] = ys[buf][m][t];
        else { yv[m].x = 0; yv[m].y = 0; }
      }
#pragma unroll
      for (int n = 0; n < NN; ++n)
#pragma unroll
        for (int m = 0; m < MM; ++m) {
          const V a = xc[n][j], b = yv[m];
          re[n * MM + m] = fma(a.x, b.x, fma(-a.y, b.y, re[n * MM + m]));
          im[n * MM + m] = fma(a.x, b.y, fma(a.y, b.x, im[n * MM + m]));
        }
    }
    if (kF32 && ++cnt == kFlush) {
      cnt = 0;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        sacc[(2 * p) * kThr + tid] += (double)re[p];
        sacc[(2 * p + 1) * kThr + tid] += (double)im[p];
        re[p] = im[p] = 0;
      }
    }
  }
  __shared__ double sred[kThr / 32][NP][2];
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    double a = (double)re[p], b = (double)im[p];
    if (kF32) {
      a += sacc[(2 * p) * kThr + tid];
      b += sacc[(2 * p + 1) * kThr + tid];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (lane == 0) { sred[warp][p][0] = a; sred[warp][p][1] = b; }
  }
  __syncthreads();
  if (tid < NP) {
    double a = 0, b = 0;
    for (int w = 0; w < kThr / 32; ++w) { a += sred[w][tid][0]; b += sred[w][tid][1]; }
    part[(int64_t)blockIdx.x * NP + tid] = make_double2(a, b);
  }
}

// fp64 sum of the G partials of every pair: thread t takes partials t, t + 256, ... (all
// loads in flight at once), then a fixed-shape shared-memory tree -- deterministic.
constexpr int kFinThr = 256;
template <typename T, int NN, int MM>
__global__ void __launch_bounds__(kFinThr) splitk_strided_final(SplitKDesc d, const double2* __restrict__ part_in, int G) {
  pdl_wait();
  pdl_trigger();
  using V = typename C2<T>::t;
  constexpr int NP = NN * MM;
  const V* Xu;
  const V* Yu;
  V* Cu;
  int64_t poff;
  unit_ptrs<V>(d, Xu, Yu, Cu, poff, NP);
  const double2* part = part_in + poff;
  __shared__ double2 red[kFinThr];
  double2 acc[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) acc[p] = make_double2(0.0, 0.0);
  for (int g = threadIdx.x; g < G; g += kFinThr)
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const double2 v = part[(int64_t)g * NP + p];
      acc[p].x += v.x;
      acc[p].y += v.y;
    }
  for (int p = 0; p < NP; ++p) {
    red[threadIdx.x] = acc[p];
    __syncthreads();
    for (int s = kFinThr / 2; s > 0; s >>= 1) {
      if ((int)threadIdx.x < s) {
        red[threadIdx.x].x += red[threadIdx.x + s].x;
        red[threadIdx.x].y += red[threadIdx.x + s].y;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      V v;
      v.x = (T)red[0].x;
      v.y = (T)red[0].y;
      Cu[d.cn[p / MM] + d.cm[p % MM]] = v;
    }
    __syncthreads();
  }
}

int grid_ctas() {
  return std::min(sm_count() * 4, kMaxCtas);
}

template <typename T, int NN, int MM>
void go(const SplitKDesc& d, void* scratch, cudaStream_t st) {
  using V = typename C2<T>::t;
  const int64_t ntile = (int64_t)1 << d.nr;
  const int smem = (int)(2 * MM * (1 << kTileBits) * sizeof(V) + (sizeof(T) == 4 ? 2 * NN * MM * kThr * 8 : 0));
  // persistent grid: every CTA resident (fixed per device: deterministic summation order)
  cudaFuncSetAttribute(splitk_strided_kernel<T, NN, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, splitk_strided_kernel<T, NN, MM>, kThr, smem);
  const int G0 = std::max(1, std::min(grid_ctas(), std::max(1, per_sm) * grid_ctas() / 4));
  const int G = (int)std::min<int64_t>(ntile, G0);
  launch_pdl(splitk_strided_kernel<T, NN, MM>, dim3(G, d.nb), kThr, smem, st, d, (double2*)scratch);
  launch_pdl(splitk_strided_final<T, NN, MM>, dim3(1, d.nb), kFinThr, 0, st, d, (const double2*)scratch, G);
}

template <typename T>
void dispatch(int nn, int nm, const SplitKDesc& d, void* scratch, cudaStream_t st) {
#define TNQVM_SKS(a, b) \
  if (nn == a && nm == b) return go<T, 1 << a, 1 << b>(d, scratch, st);
  TNQVM_SKS(0, 0) TNQVM_SKS(1, 0) TNQVM_SKS(1, 1) TNQVM_SKS(2, 0) TNQVM_SKS(2, 1) TNQVM_SKS(3, 0)
  TNQVM_SKS(2, 2) TNQVM_SKS(3, 1) TNQVM_SKS(4, 0)
#undef TNQVM_SKS
}

template <typename T, int P>
void go_big_p(const SplitKDesc& d, int nn, int nm, void* scratch, cudaStream_t st) {
  using V = typename C2<T>::t;
  const int rows = (1 << nn) + (1 << nm), NP = 1 << (nn + nm);
  const BigBlock bb = big_block(1 << nn, 1 << nm, kThr, sizeof(T) == 8 || d.blocked);
  const int padw = (1 << kBigBits) + (sizeof(T) == 4 ? 2 : 1);
  const int smem = std::max((int)(big_stages<T>() * rows * padw * sizeof(V)),
                            bb.KG > 1 ? (int)(kThr * bb.PN * bb.PM * sizeof(double2)) : 0);
  // one resident wave of CTAs (the grid size depends only on the shape and the device)
  const int maxsm = (int)(big_stages<T>() * 128 * ((1 << kBigBits) + 2) * sizeof(V));
  cudaFuncSetAttribute(splitk_big_kernel<T, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
  const int nsm = sm_count();
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, splitk_big_kernel<T, P>, kThr, smem);
  const int G0 = std::max(1, std::min(kMaxCtas, std::max(1, per_sm) * nsm));
  const int G = (int)std::min<int64_t>((int64_t)1 << d.nr, G0);
  launch_pdl(splitk_big_kernel<T, P>, dim3(G, d.nb), kThr, smem, st, d, nn, nm, (double2*)scratch);
  launch_pdl(splitk_big_final<T>, dim3(NP, d.nb), kThr, 0, st, d, nm, NP, (const double2*)scratch, G);
}

template <typename T>
void go_big(const SplitKDesc& d, int nn, int nm, void* scratch, cudaStream_t st) {
  // the same block shape the kernel derives
  const BigBlock bb = big_block(1 << nn, 1 << nm, kThr, sizeof(T) == 8 || d.blocked);
  const int P = std::max(bb.PN, bb.PM);
  if (P <= 1) go_big_p<T, 1>(d, nn, nm, scratch, st);
  else if (P <= 2) go_big_p<T, 2>(d, nn, nm, scratch, st);
  else go_big_p<T, 4>(d, nn, nm, scratch, st);
}


// complex64 split-K with lanes over the output rows ("lane" kernel): for steps whose larger
// operand X has a contracted mode of stride 1 (and possibly of stride 2), lane n of a warp
// reads its own X row straight from global memory Q = 2 or 4 complex at a time (16 / 32
// contiguous bytes), and the smaller operand Y is staged per warp block in warp-private shared
// memory (cp.async), where the lanes of an r-group read the same words (broadcast).  Per
// complex MAC this moves ~1/16 of the shared-memory wavefronts of splitk_big_kernel, which ncu
// showed shared-memory bound.  Every warp works alone on a contiguous range of rest indices
// (no CTA barriers in the loop) with the next block's X words and Y tile in flight while it
// multiplies the current block.
// Rest index r = the contracted modes other than X's Q-modes, ordered by X stride; a warp
// block = RB consecutive r; r-group g of the warp takes r = g + gpw * j, j < kLaneRpg.
// fp32 sums over <= 4 blocks, then fp64; lane, warp and CTA partials reduced in a fixed order
// (deterministic, independent of the batch).
struct LaneDesc {
  const void* X;
  const void* Y;
  const int64_t* delta;
  int nb, xsel;
  int nn, nm, qb, lrb, nrh;
  int64_t xn[32], ym[16], yq[4];
  int64_t xlo[8], ylo[8];      // strides of the low (in-block) rest bits
  int64_t xhs[48], yhs[48];    // strides of the high rest bits (block index)
  int64_t dxh[48], dyh[48];    // block -> block + 1 with carry out of bit j: offset += d[j]
};
constexpr int kLaneThr = 256, kLaneWarps = kLaneThr / 32, kLaneRpg = 2, kLanePf = 4;
constexpr int kLaneTileMax = 128;  // Y tile complex per warp block: RB * Q * M

template <int M>
__global__ void __launch_bounds__(kLaneThr, M >= 16 ? 1 : 2) splitk_lane_kernel(LaneDesc L, double2* __restrict__ part) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.y;
  const float2* X = reinterpret_cast<const float2*>(L.X) + (L.delta ? L.delta[L.xsel * L.nb + b] : 0);
  const float2* Y = reinterpret_cast<const float2*>(L.Y) + (L.delta ? L.delta[(1 - L.xsel) * L.nb + b] : 0);
  const int N = 1 << L.nn, Q = 1 << L.qb, RB = 1 << L.lrb, NP = N * M;
  part += (int64_t)b * kMaxCtas * NP;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = lane & (N - 1), gpw = 32 >> L.nn, g = lane >> L.nn;
  const int tile = RB * Q * M;  // complex per warp block
  extern __shared__ __align__(16) unsigned char lane_smem[];
  float2* ysm = reinterpret_cast<float2*>(lane_smem) + (size_t)warp * 2 * tile;  // this warp's [2][RB][Q][M]
  // this lane's in-block offsets (r = g + gpw * j) and its cp.async elements of a Y tile
  int64_t xlow[kLaneRpg];
#pragma unroll
  for (int j = 0; j < kLaneRpg; ++j) {
    const int i = g + gpw * j;
    int64_t a = 0;
    for (int t = 0; t < L.lrb; ++t)
      if ((i >> t) & 1) a += L.xlo[t];
    xlow[j] = a;
  }
  const int64_t NBW = (int64_t)1 << L.nrh;  // warp blocks per unit
  const int64_t W = (int64_t)gridDim.x * kLaneWarps, w = (int64_t)blockIdx.x * kLaneWarps + warp;
  const int64_t b0 = NBW * w / W, b1 = NBW * (w + 1) / W;
  int64_t xh = 0, yh = 0;
  for (int j = 0; j < L.nrh; ++j)
    if ((b0 >> j) & 1) { xh += L.xhs[j]; yh += L.yhs[j]; }
  const float2* Xn = X + L.xn[n];
  // this lane's Y tile elements e = lane + 32 t (tile = RB * Q * M <= kLaneTileMax): their
  // in-block offsets, fixed over blocks
  int64_t yoe[kLaneTileMax / 32];
#pragma unroll
  for (int t = 0; t < kLaneTileMax / 32; ++t) {
    const int e = lane + 32 * t;
    const int m = e & (M - 1), q = (e / M) & (Q - 1), i = e / (M * Q);
    int64_t o = L.yq[q] + L.ym[m];
    for (int u = 0; u < L.lrb; ++u)
      if ((i >> u) & 1) o += L.ylo[u];
    yoe[t] = o;
  }
  auto stage = [&](int buf, int64_t yoff) {  // Y[block][i][q][m] -> ysm[buf] (warp-private)
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(ysm + (size_t)buf * tile) + (uint32_t)lane * 8;
    const float2* yb = Y + yoff;
#pragma unroll
    for (int t = 0; t < kLaneTileMax / 32; ++t)
      if (32 * t < tile)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sb + (uint32_t)t * 256), "l"(yb + yoe[t])
                     : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto loadx = [&](int64_t off, float4 (&xv)[kLaneRpg][2]) {
#pragma unroll
    for (int j = 0; j < kLaneRpg; ++j) {
      const float4* src = reinterpret_cast<const float4*>(Xn + off + xlow[j]);
      xv[j][0] = __ldcs(src);
      if (Q == 4) xv[j][1] = __ldcs(src + 1);
    }
  };
  float ar[M], ai[M];
  double dr[M], di[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    dr[m] = di[m] = 0.0;
    ar[m] = ai[m] = 0.f;
  }
  float4 xc[kLaneRpg][2], xn2[kLaneRpg][2];
  if (b0 < b1) {
    stage(0, yh);
    loadx(xh, xc);
  }
  // X words of block bl + kLanePf are prefetched into L2 (no registers held)
  int64_t xpf = 0;
  for (int j = 0; j < L.nrh; ++j)
    if (((b0 + kLanePf) >> j) & 1) xpf += L.xhs[j];
  int nf = 0;
  for (int64_t bl = b0; bl < b1; ++bl) {
    const int buf = (int)((bl - b0) & 1);
    if (bl + kLanePf < b1) {
#pragma unroll
      for (int j = 0; j < kLaneRpg; ++j)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(Xn + xpf + xlow[j]));
      const int jj = __ffsll((unsigned long long)(bl + kLanePf + 1)) - 1;
      xpf += L.dxh[jj];
    }
    if (bl + 1 < b1) {  // next block: offsets by carry delta, its Y tile and X words in flight
      const int j = __ffsll((unsigned long long)(bl + 1)) - 1;
      xh += L.dxh[j];
      yh += L.dyh[j];
      stage(buf ^ 1, yh);
      loadx(xh, xn2);
    } else {
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    const float2* yb = ysm + (size_t)buf * tile;
#pragma unroll
    for (int j = 0; j < kLaneRpg; ++j) {
      const int i = g + gpw * j;
      const float2 xq[4] = {make_float2(xc[j][0].x, xc[j][0].y), make_float2(xc[j][0].z, xc[j][0].w),
                            make_float2(xc[j][1].x, xc[j][1].y), make_float2(xc[j][1].z, xc[j][1].w)};
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < Q) {
          const float4* yr = reinterpret_cast<const float4*>(yb + ((size_t)i * Q + q) * M);
          const float2 x = xq[q];
          if (M == 1) {
            const float2 y = yb[(size_t)i * Q + q];
            ar[0] = fmaf(x.x, y.x, fmaf(-x.y, y.y, ar[0]));
            ai[0] = fmaf(x.x, y.y, fmaf(x.y, y.x, ai[0]));
          } else {
#pragma unroll
            for (int m2 = 0; m2 < M / 2; ++m2) {
              const float4 y = yr[m2];
              ar[2 * m2] = fmaf(x.x, y.x, fmaf(-x.y, y.y, ar[2 * m2]));
              ai[2 * m2] = fmaf(x.x, y.y, fmaf(x.y, y.x, ai[2 * m2]));
              ar[2 * m2 + 1] = fmaf(x.x, y.z, fmaf(-x.y, y.w, ar[2 * m2 + 1]));
              ai[2 * m2 + 1] = fmaf(x.x, y.w, fmaf(x.y, y.z, ai[2 * m2 + 1]));
            }
          }
        }
    }
    if (++nf == 4 || bl + 1 == b1) {  // fp32 over <= 4 blocks (<= 32 terms), then fp64
      nf = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) {
        dr[m] += (double)ar[m];
        di[m] += (double)ai[m];
        ar[m] = ai[m] = 0.f;
      }
    }
    __syncwarp();  // the tile staged next reuses this buffer
#pragma unroll
    for (int j = 0; j < kLaneRpg; ++j) {
      xc[j][0] = xn2[j][0];
      xc[j][1] = xn2[j][1];
    }
  }
  // lanes of one row n (the r-groups of the warp): xor tree over the group bits
#pragma unroll
  for (int m = 0; m < M; ++m)
    for (int o = N; o < 32; o <<= 1) {
      dr[m] += __shfl_xor_sync(0xffffffffu, dr[m], o);
      di[m] += __shfl_xor_sync(0xffffffffu, di[m], o);
    }
  __syncthreads();
  double2* red = reinterpret_cast<double2*>(lane_smem);  // [m][warp][n] (conflict-free writes)
  if (lane < N)
#pragma unroll
    for (int m = 0; m < M; ++m) red[((size_t)m * kLaneWarps + warp) * N + n] = make_double2(dr[m], di[m]);
  __syncthreads();
  for (int p = tid; p < NP; p += kLaneThr) {
    const int pn = p / M, pm = p % M;
    double2 a = red[((size_t)pm * kLaneWarps) * N + pn];
    for (int v = 1; v < kLaneWarps; ++v) {
      const double2 t = red[((size_t)pm * kLaneWarps + v) * N + pn];
      a.x += t.x;
      a.y += t.y;
    }
    part[(int64_t)blockIdx.x * NP + p] = a;
  }
}

// the lane kernel's block shape: RB = r-groups per warp x kLaneRpg rest indices per warp block
int lane_lrb(int nn, int /*nm*/, int /*qb*/) { return (5 - nn) + 1; }
size_t lane_smem_bytes(int nn, int nm, int qb, int lrb) {
  const size_t tiles = (size_t)kLaneWarps * 2 * ((size_t)1 << (lrb + qb + nm)) * 8;
  const size_t red = (size_t)kLaneWarps * ((size_t)1 << (nn + nm)) * 16;
  return std::max(tiles, red);
}

template <int M>
void go_lane(const LaneDesc& L, const SplitKDesc& d, void* scratch, cudaStream_t st) {
  const int smem = (int)lane_smem_bytes(L.nn, L.nm, L.qb, L.lrb);
  cudaFuncSetAttribute(splitk_lane_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, splitk_lane_kernel<M>, kLaneThr, smem);
  // one resident wave per unit (the grid depends only on the shape and the device)
  const int G = (int)std::min<int64_t>((int64_t)1 << L.nrh, std::min(kMaxCtas, std::max(1, per_sm) * sm_count()));
  launch_pdl(splitk_lane_kernel<M>, dim3(G, L.nb), kLaneThr, smem, st, L, (double2*)scratch);
  const int NP = 1 << (L.nn + L.nm);
  launch_pdl(splitk_big_final<float>, dim3(NP, L.nb), kThr, 0, st, d, L.nm, NP, (const double2*)scratch, G);
}

}  // namespace

size_t splitk_strided_scratch_bytes(int nn, int nm) {
  return sizeof(double2) * (size_t)kMaxCtas * ((size_t)1 << (nn + nm));
}

bool splitk_strided_supported(int nn, int nk, int nm) {
  return nn <= 6 && nm <= 6 && nk >= 1 && nk - kBigBits <= 48;
}

void launch_splitk_strided(int dtype, const StridedSplitK& s0, void* scratch, const Batch& bt, cudaStream_t st) {
  // the operand with fewer free modes is the one staged in shared memory (Y)
  StridedSplitK s = s0;
  const bool swap = s0.nm > s0.nn;
  if (swap) {
    s.X = s0.Y; s.Y = s0.X; s.nn = s0.nm; s.nm = s0.nn;
    for (int i = 0; i < 6; ++i) { s.sxn[i] = s0.sym[i]; s.scn[i] = s0.scm[i]; s.sym[i] = s0.sxn[i]; s.scm[i] = s0.scn[i]; }
    for (int i = 0; i < s0.nk; ++i) { s.sxk[i] = s0.syk[i]; s.syk[i] = s0.sxk[i]; }
  }
  SplitKDesc d{};
  d.X = s.X;
  d.Y = s.Y;
  d.C = s.C;
  d.nb = bt.nb;
  d.delta = bt.delta;
  const int xi = swap ? 1 : 0;  // Batch operand index of the kernel's X
  d.xsel = xi;
  const int nk = s.nk;
  const bool big = s.nn + s.nm > 4;
  // tile bits: X's 5 fastest contracted modes, then Y's 4 fastest ones, then X's next ones
  // (big outputs: 64-value tiles, X's 3 fastest then Y's 3 fastest)
  std::vector<int> U;
  auto in_u = [&](int k) { return std::find(U.begin(), U.end(), k) != U.end(); };
  const int u = std::min(nk, big ? kBigBits : kTileBits);
  const int ux = big ? 3 : 5, uy = big ? 2 : 4;
  std::vector<int> xorder(nk), yorder(nk);
  for (int k = 0; k < nk; ++k) xorder[k] = yorder[k] = k;
  std::sort(xorder.begin(), xorder.end(), [&](int a, int b) { return s.sxk[a] < s.sxk[b]; });
  std::sort(yorder.begin(), yorder.end(), [&](int a, int b) { return s.syk[a] < s.syk[b]; });
  for (int i = 0; i < std::min(nk, ux); ++i) U.push_back(xorder[i]);
  for (int i = 0; i < nk && (int)U.size() < u && i < uy; ++i)
    if (!in_u(yorder[i])) U.push_back(yorder[i]);
  for (int i = 0; i < nk && (int)U.size() < u; ++i)
    if (!in_u(xorder[i])) U.push_back(xorder[i]);
  d.u = u;
  for (int j = 0; j < u; ++j) { d.xt[j] = s.sxk[U[j]]; d.yt[j] = s.syk[U[j]]; }
  std::vector<int> v2t(u);
  for (int j = 0; j < u; ++j) v2t[j] = j;
  std::sort(v2t.begin(), v2t.end(), [&](int a, int b) { return d.yt[a] < d.yt[b]; });
  for (int i = 0; i < u; ++i) d.yv2t[i] = v2t[i];
  d.nr = 0;
  for (int k = 0; k < nk; ++k)
    if (!in_u(k)) { d.xr[d.nr] = s.sxk[k]; d.yr[d.nr] = s.syk[k]; ++d.nr; }
  int64_t sx = 0, sy = 0;
  for (int j = 0; j < d.nr; ++j) {
    d.dxr[j] = d.xr[j] - sx;
    d.dyr[j] = d.yr[j] - sy;
    sx += d.xr[j];
    sy += d.yr[j];
  }
  for (int n = 0; n < (1 << s.nn); ++n) {
    int64_t a = 0, c = 0;
    for (int i = 0; i < s.nn; ++i)
      if ((n >> i) & 1) { a += s.sxn[i]; c += s.scn[i]; }
    d.xn[n] = a;
    d.cn[n] = c;
  }
  for (int m = 0; m < (1 << s.nm); ++m) {
    int64_t a = 0, c = 0;
    for (int i = 0; i < s.nm; ++i)
      if ((m >> i) & 1) { a += s.sym[i]; c += s.scm[i]; }
    d.ym[m] = a;
    d.cm[m] = c;
  }
  // complex64, X rows <= 32, M <= 16, X's stride-1 mode contracted: the lane kernel
  if (dtype == 0 && big && s.nn <= 5 && s.nm <= 4 && nk >= 2) {
    int k1 = -1, k2 = -1;
    for (int k = 0; k < nk; ++k) {
      if (s.sxk[k] == 1) k1 = k;
      if (s.sxk[k] == 2) k2 = k;
    }
    const int qb = k1 < 0 ? 0 : (k2 >= 0 ? 2 : 1);
    bool ok = qb > 0 && ((uintptr_t)s.X & 15) == 0 && bt.all_even(xi);
    std::vector<int> rest;
    for (int k = 0; k < nk; ++k)
      if (k != k1 && !(qb == 2 && k == k2)) rest.push_back(k);
    std::sort(rest.begin(), rest.end(), [&](int a, int b) { return s.sxk[a] < s.sxk[b]; });
    for (int k : rest) ok = ok && (s.sxk[k] % 2 == 0);
    for (int n = 0; ok && n < (1 << s.nn); ++n) ok = (d.xn[n] % 2) == 0;
    const int lrb = lane_lrb(s.nn, s.nm, qb);
    if (ok && (int)rest.size() >= lrb && (int)rest.size() - lrb <= 48 &&
        (1 << (lrb + qb + s.nm)) <= kLaneTileMax && (1 << (lrb + qb + s.nm)) >= 32) {
      LaneDesc L{};
      L.X = s.X;
      L.Y = s.Y;
      L.delta = bt.delta;
      L.nb = bt.nb;
      L.xsel = xi;
      L.nn = s.nn;
      L.nm = s.nm;
      L.qb = qb;
      L.lrb = lrb;
      L.nrh = (int)rest.size() - lrb;
      for (int n = 0; n < (1 << s.nn); ++n) L.xn[n] = d.xn[n];
      for (int m = 0; m < (1 << s.nm); ++m) L.ym[m] = d.ym[m];
      L.yq[0] = 0;
      L.yq[1] = s.syk[k1];
      if (qb == 2) { L.yq[2] = s.syk[k2]; L.yq[3] = s.syk[k1] + s.syk[k2]; }
      for (int j = 0; j < lrb; ++j) { L.xlo[j] = s.sxk[rest[j]]; L.ylo[j] = s.syk[rest[j]]; }
      int64_t sx = 0, sy = 0;
      for (int j = 0; j < L.nrh; ++j) {
        L.xhs[j] = s.sxk[rest[lrb + j]];
        L.yhs[j] = s.syk[rest[lrb + j]];
        L.dxh[j] = L.xhs[j] - sx;
        L.dyh[j] = L.yhs[j] - sy;
        sx += L.xhs[j];
        sy += L.yhs[j];
      }
      switch (s.nm) {
        case 0: return go_lane<1>(L, d, scratch, st);
        case 1: return go_lane<2>(L, d, scratch, st);
        case 2: return go_lane<4>(L, d, scratch, st);
        case 3: return go_lane<8>(L, d, scratch, st);
        default: return go_lane<16>(L, d, scratch, st);
      }
    }
  }
  if (big) {
    // 16-byte X copies: tile bit 0 is X's unit-stride mode and every other X offset is even
    // (so pair starts are 16-byte aligned); TNQVM_SPLITK_XVEC=0 disables
    bool xv = dtype == 0 && u >= 2 && d.xt[0] == 1 && ((uintptr_t)d.X & 15) == 0 && bt.all_even(xi);
    for (int j = 1; xv && j < u; ++j) xv = (d.xt[j] & 1) == 0;
    for (int j = 0; xv && j < d.nr; ++j) xv = (d.xr[j] & 1) == 0;
    for (int n = 0; xv && n < (1 << s.nn); ++n) xv = (d.xn[n] & 1) == 0;
    d.xvec = xv ? 1 : 0;
    d.blocked = 0;  // complex128 always blocks (big_block); complex64 one output per thread
    if (dtype == 0) go_big<float>(d, s.nn, s.nm, scratch, st);
    else go_big<double>(d, s.nn, s.nm, scratch, st);
    return;
  }
  if (dtype == 0) dispatch<float>(s.nn, s.nm, d, scratch, st);
  else dispatch<double>(s.nn, s.nm, d, scratch, st);
}

}  // namespace dev
}  // namespace tnqvm
