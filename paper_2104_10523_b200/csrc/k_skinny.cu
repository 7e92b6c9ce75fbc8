// a7 (streaming path for skinny steps, K*M <= 64): the most common large step of sliced
// random-circuit contraction plans is a big tensor contracted with a gate-sized one on
// a few modes (SURVEY E3 step histograms).  These are HBM-bound (AI <= 8 flop/B):
// the kernel reads the big operand X once in its stored layout (no permute), keeps the
// small operand Y in shared memory, accumulates the M outputs of each X index in
// registers (two-level for K > 16) and writes C in any layout.  Thread t of a CTA owns
// n = base + t, so the 8 lowest n bits (X's fastest free modes) map to consecutive lanes
// and both the X reads and the C writes coalesce; per-thread offsets are split into a
// once-per-thread low part and a per-iteration high part.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.hpp"
#include "pdl.cuh"

namespace tnqvm {
namespace dev {
namespace {

template <typename T> struct C2;
template <> struct C2<float> { using t = float2; };
template <> struct C2<double> { using t = double2; };

constexpr int kSkThreads = 256;

template <typename T, int MM>
__global__ void __launch_bounds__(kSkThreads, 2) skinny_kernel(SkinnyDesc d, const int64_t* __restrict__ delta, int nb) {
  pdl_wait();
  pdl_trigger();
  using V = typename C2<T>::t;
  __shared__ V Ys[512];       // [k][m], K*M <= 512
  __shared__ int64_t xk[64];  // X offset of k
  __shared__ int64_t cm[64];  // C offset of m
  const int K = 1 << d.nk;
  const int ub = blockIdx.y;  // unit of the batch
  const V* __restrict__ X = reinterpret_cast<const V*>(d.X) + (delta ? delta[ub] : 0);
  const V* __restrict__ Y = reinterpret_cast<const V*>(d.Y) + (delta ? delta[nb + ub] : 0);
  V* __restrict__ C = reinterpret_cast<V*>(d.C) + (delta ? delta[2 * nb + ub] : 0);
  for (int t = threadIdx.x; t < K * MM; t += kSkThreads) {
    const int k = t / MM, m = t % MM;
    int64_t o = 0;
    for (int i = 0; i < d.nk; ++i)
      if ((k >> i) & 1) o += d.syk[i];
    for (int i = 0; i < d.nm; ++i)
      if ((m >> i) & 1) o += d.sym[i];
    Ys[t] = Y[o];
  }
  for (int k = threadIdx.x; k < K; k += kSkThreads) {
    int64_t o = 0;
    for (int i = 0; i < d.nk; ++i)
      if ((k >> i) & 1) o += d.sxk[i];
    xk[k] = o;
  }
  for (int m = threadIdx.x; m < MM; m += kSkThreads) {
    int64_t o = 0;
    for (int i = 0; i < d.nm; ++i)
      if ((m >> i) & 1) o += d.scm[i];
    cm[m] = o;
  }
  // low-bit offsets of this thread (n bits 0..7)
  const int lowb = d.nn < 8 ? d.nn : 8;
  int64_t xlo = 0, clo = 0;
  for (int i = 0; i < lowb; ++i)
    if ((threadIdx.x >> i) & 1) { xlo += d.sxn[i]; clo += d.scn[i]; }
  __syncthreads();
  const int64_t N = (int64_t)1 << d.nn;
  const int64_t step = (int64_t)gridDim.x * kSkThreads;
  for (int64_t base = (int64_t)blockIdx.x * kSkThreads; base < N; base += step) {
    if (base + threadIdx.x >= N) break;
    int64_t xo = xlo, co = clo;
    for (int i = lowb; i < d.nn; ++i)
      if ((base >> i) & 1) { xo += d.sxn[i]; co += d.scn[i]; }
    T ar[MM], ai[MM];
#pragma unroll
    for (int m = 0; m < MM; ++m) ar[m] = ai[m] = 0;
    // K in blocks of 8: the block's X values are loaded first (16 loads in flight per
    // thread), then multiplied into all M outputs; blocks are summed separately (two-level)
    for (int k0 = 0; k0 < K; k0 += 8) {
      const int kb = min(8, K - k0);
      V xs[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < kb) xs[j] = __ldcs(X + xo + xk[k0 + j]);
      T br[MM], bi[MM];
#pragma unroll
      for (int m = 0; m < MM; ++m) br[m] = bi[m] = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < kb) {
          const V x = xs[j];
#pragma unroll
          for (int m = 0; m < MM; ++m) {
            const V y = Ys[(k0 + j) * MM + m];
            br[m] = fma(x.x, y.x, fma(-x.y, y.y, br[m]));
            bi[m] = fma(x.x, y.y, fma(x.y, y.x, bi[m]));
          }
        }
      }
#pragma unroll
      for (int m = 0; m < MM; ++m) { ar[m] += br[m]; ai[m] += bi[m]; }
    }
#pragma unroll
    for (int m = 0; m < MM; ++m) {
      V c;
      c.x = ar[m];
      c.y = ai[m];
      __stcs(C + co + cm[m], c);
    }
  }
}

// complex64 with n bit 0 of stride 1 in both X and C: thread t owns the adjacent pair
// (2t, 2t + 1), so every X read and C write is a 16-byte vector (twice the bytes in flight
// per thread of skinny_kernel).
template <int MM>
__global__ void __launch_bounds__(kSkThreads, 2) skinny_pair_kernel(SkinnyDesc d, const int64_t* __restrict__ delta, int nb) {
  pdl_wait();
  pdl_trigger();
  __shared__ float2 Ys[512];
  __shared__ int64_t xk[64];
  __shared__ int64_t cm[64];
  const int K = 1 << d.nk;
  const int ub = blockIdx.y;  // unit of the batch
  const float2* __restrict__ Y = reinterpret_cast<const float2*>(d.Y) + (delta ? delta[nb + ub] : 0);
  const float* __restrict__ X = reinterpret_cast<const float*>(d.X) + 2 * (delta ? delta[ub] : 0);
  float* __restrict__ C = reinterpret_cast<float*>(d.C) + 2 * (delta ? delta[2 * nb + ub] : 0);
  for (int t = threadIdx.x; t < K * MM; t += kSkThreads) {
    const int k = t / MM, m = t % MM;
    int64_t o = 0;
    for (int i = 0; i < d.nk; ++i)
      if ((k >> i) & 1) o += d.syk[i];
    for (int i = 0; i < d.nm; ++i)
      if ((m >> i) & 1) o += d.sym[i];
    Ys[t] = Y[o];
  }
  for (int k = threadIdx.x; k < K; k += kSkThreads) {
    int64_t o = 0;
    for (int i = 0; i < d.nk; ++i)
      if ((k >> i) & 1) o += d.sxk[i];
    xk[k] = o;
  }
  for (int m = threadIdx.x; m < MM; m += kSkThreads) {
    int64_t o = 0;
    for (int i = 0; i < d.nm; ++i)
      if ((m >> i) & 1) o += d.scm[i];
    cm[m] = o;
  }
  // pair index p = n >> 1: its bits i >= 0 are n bits i + 1
  const int np = d.nn - 1;
  const int lowb = np < 8 ? np : 8;
  int64_t xlo = 0, clo = 0;
  for (int i = 0; i < lowb; ++i)
    if ((threadIdx.x >> i) & 1) { xlo += d.sxn[i + 1]; clo += d.scn[i + 1]; }
  __syncthreads();
  const int64_t NP = (int64_t)1 << np;
  const int64_t step = (int64_t)gridDim.x * kSkThreads;
  for (int64_t base = (int64_t)blockIdx.x * kSkThreads; base < NP; base += step) {
    if (base + threadIdx.x >= NP) break;
    int64_t xo = xlo, co = clo;
    for (int i = lowb; i < np; ++i)
      if ((base >> i) & 1) { xo += d.sxn[i + 1]; co += d.scn[i + 1]; }
    float ar[2][MM], ai[2][MM];
#pragma unroll
    for (int m = 0; m < MM; ++m) ar[0][m] = ai[0][m] = ar[1][m] = ai[1][m] = 0;
    for (int k0 = 0; k0 < K; k0 += 8) {
      const int kb = min(8, K - k0);
      float4 xs[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < kb) xs[j] = __ldcs(reinterpret_cast<const float4*>(X + 2 * (xo + xk[k0 + j])));
      float br[2][MM], bi[2][MM];
#pragma unroll
      for (int m = 0; m < MM; ++m) br[0][m] = bi[0][m] = br[1][m] = bi[1][m] = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < kb) {
          const float4 x = xs[j];
#pragma unroll
          for (int m = 0; m < MM; ++m) {
            const float2 y = Ys[(k0 + j) * MM + m];
            br[0][m] = fmaf(x.x, y.x, fmaf(-x.y, y.y, br[0][m]));
            bi[0][m] = fmaf(x.x, y.y, fmaf(x.y, y.x, bi[0][m]));
            br[1][m] = fmaf(x.z, y.x, fmaf(-x.w, y.y, br[1][m]));
            bi[1][m] = fmaf(x.z, y.y, fmaf(x.w, y.x, bi[1][m]));
          }
        }
      }
#pragma unroll
      for (int m = 0; m < MM; ++m) {
        ar[0][m] += br[0][m];
        ai[0][m] += bi[0][m];
        ar[1][m] += br[1][m];
        ai[1][m] += bi[1][m];
      }
    }
#pragma unroll
    for (int m = 0; m < MM; ++m)
      __stcs(reinterpret_cast<float4*>(C + 2 * (co + cm[m])), make_float4(ar[0][m], ai[0][m], ar[1][m], ai[1][m]));
  }
}

template <typename T>
void launch_t(const SkinnyDesc& d, const Batch& bt, cudaStream_t st) {
  const int nsm = sm_count();
  const int64_t N = (int64_t)1 << d.nn;
  // each thread computes whole outputs: any grid gives the same values; ~16 CTAs per SM in total
  const int64_t blocks =
      std::max<int64_t>(1, std::min<int64_t>((N + kSkThreads - 1) / kSkThreads, (int64_t)nsm * 16 / bt.nb + 1));
  const dim3 grid((unsigned)blocks, (unsigned)bt.nb);
  switch (1 << d.nm) {
#define TNQVM_SKC(m) \
  case m:            \
    launch_pdl(skinny_kernel<T, m>, grid, kSkThreads, 0, st, d, bt.delta, bt.nb); \
    break;
    TNQVM_SKC(1) TNQVM_SKC(2) TNQVM_SKC(4) TNQVM_SKC(8) TNQVM_SKC(16) TNQVM_SKC(32)
#undef TNQVM_SKC
    default: break;
  }
}

}  // namespace

void launch_skinny(int dtype, const SkinnyDesc& d, const Batch& bt, cudaStream_t st) {
  // pair path: n bit 0 contiguous in X and C; every other X / C offset even (16-byte
  // aligned) in every unit -- the same per-thread arithmetic as the scalar kernel
  bool pair = dtype == 0 && d.nn >= 2 && d.sxn[0] == 1 && d.scn[0] == 1 && d.nm <= 3 &&
              ((reinterpret_cast<uintptr_t>(d.X) | reinterpret_cast<uintptr_t>(d.C)) & 15) == 0 && bt.all_even(0) &&
              bt.all_even(2);
  for (int i = 1; pair && i < d.nn; ++i) pair = (d.sxn[i] % 2 == 0) && (d.scn[i] % 2 == 0);
  for (int i = 0; pair && i < d.nk; ++i) pair = d.sxk[i] % 2 == 0;
  for (int i = 0; pair && i < d.nm; ++i) pair = d.scm[i] % 2 == 0;
  if (pair) {
    const int nsm = sm_count();
    const int64_t NP = (int64_t)1 << (d.nn - 1);
    const int64_t blocks =
        std::max<int64_t>(1, std::min<int64_t>((NP + kSkThreads - 1) / kSkThreads, (int64_t)nsm * 16 / bt.nb + 1));
    const dim3 grid((unsigned)blocks, (unsigned)bt.nb);
    switch (1 << d.nm) {
      case 1: launch_pdl(skinny_pair_kernel<1>, grid, kSkThreads, 0, st, d, bt.delta, bt.nb); return;
      case 2: launch_pdl(skinny_pair_kernel<2>, grid, kSkThreads, 0, st, d, bt.delta, bt.nb); return;
      case 4: launch_pdl(skinny_pair_kernel<4>, grid, kSkThreads, 0, st, d, bt.delta, bt.nb); return;
      case 8: launch_pdl(skinny_pair_kernel<8>, grid, kSkThreads, 0, st, d, bt.delta, bt.nb); return;
      default: break;
    }
  }
  if (dtype == 0) launch_t<float>(d, bt, st);
  else launch_t<double>(d, bt, st);
}

}  // namespace dev
}  // namespace tnqvm
