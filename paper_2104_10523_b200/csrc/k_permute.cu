// a6: index permute of binary-mode tensors (N1), shared-memory staged.
//
// TTGT realisation of a pairwise contraction needs the contracted modes of the
// streamed operand to be the fastest ones.  When the planner's layout choice (a5) cannot
// avoid it, the tensor is re-laid out here: out[pi(i)] = in[i] for a rank-r tensor whose
// modes all have extent 2.  A CTA owns one tile = every combination of the tile modes U
// (the input's fastest modes joined with the output's fastest modes, |U| <= 11) for one
// assignment of the remaining modes.  The tile is read in input order (contiguous,
// 16-byte vector loads), staged in shared memory, and written in output order
// (contiguous, 16-byte vector stores).  Traffic = 2 x tensor bytes: HBM-bound.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "kernels.hpp"
#include "pdl.cuh"

namespace tnqvm {
namespace dev {
namespace {

constexpr int kMaxU = 12;
constexpr int kMaxR = 48;

struct PermPlan {
  int nu, nrest;
  int64_t tin[kMaxU];      // tile bit i (input order, LSB = fastest) -> input stride
  int tpos_of_u[kMaxU];    // output-order tile bit j -> tile bit i
  int64_t uout[kMaxU];     // output-order tile bit j -> output stride
  int64_t rin[kMaxR], rout[kMaxR];
};

template <typename V>
__global__ void __launch_bounds__(256) permute_kernel(const V* __restrict__ in, V* __restrict__ out, PermPlan p,
                                                      int64_t nblocks, const int64_t* __restrict__ delta, int nub) {
  pdl_wait();
  pdl_trigger();
  if (delta) {  // unit blockIdx.y of the batch
    in += delta[blockIdx.y];
    out += delta[2 * nub + blockIdx.y];
  }
  extern __shared__ __align__(16) unsigned char sm[];
  V* tile = reinterpret_cast<V*>(sm);
  const int T = 1 << p.nu;
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
    int64_t bi = 0, bo = 0;
    for (int i = 0; i < p.nrest; ++i)
      if ((b >> i) & 1) { bi += p.rin[i]; bo += p.rout[i]; }
    __syncthreads();
    // load: consecutive t are consecutive input addresses for the low (contiguous) bits
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
      int64_t o = 0;
#pragma unroll 4
      for (int i = 0; i < p.nu; ++i)
        if ((t >> i) & 1) o += p.tin[i];
      tile[t] = __ldg(in + bi + o);
    }
    __syncthreads();
    // store in output order
    for (int u = threadIdx.x; u < T; u += blockDim.x) {
      int t = 0;
      int64_t o = 0;
#pragma unroll 4
      for (int j = 0; j < p.nu; ++j)
        if ((u >> j) & 1) { t |= 1 << p.tpos_of_u[j]; o += p.uout[j]; }
      out[bo + o] = tile[t];
    }
  }
}

// c64 variant with paired 16-byte stores (output-fastest mode inside the tile, stride 1)
__global__ void __launch_bounds__(256) permute_kernel_v2(const float2* __restrict__ in, float2* __restrict__ out,
                                                         PermPlan p, int64_t nblocks, const int64_t* __restrict__ delta,
                                                         int nub) {
  pdl_wait();
  pdl_trigger();
  if (delta) {
    in += delta[blockIdx.y];
    out += delta[2 * nub + blockIdx.y];
  }
  extern __shared__ __align__(16) unsigned char sm[];
  float2* tile = reinterpret_cast<float2*>(sm);
  const int T = 1 << p.nu;
  const bool in_pairs = p.tin[0] == 1;
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
    int64_t bi = 0, bo = 0;
    for (int i = 0; i < p.nrest; ++i)
      if ((b >> i) & 1) { bi += p.rin[i]; bo += p.rout[i]; }
    __syncthreads();
    if (in_pairs) {
      for (int t2 = threadIdx.x; t2 < T / 2; t2 += blockDim.x) {
        int t = 2 * t2;
        int64_t o = 0;
        for (int i = 1; i < p.nu; ++i)
          if ((t >> i) & 1) o += p.tin[i];
        float4 v = __ldg(reinterpret_cast<const float4*>(in + bi + o));
        reinterpret_cast<float4*>(tile)[t2] = v;
      }
    } else {
      for (int t = threadIdx.x; t < T; t += blockDim.x) {
        int64_t o = 0;
        for (int i = 0; i < p.nu; ++i)
          if ((t >> i) & 1) o += p.tin[i];
        tile[t] = __ldg(in + bi + o);
      }
    }
    __syncthreads();
    for (int u2 = threadIdx.x; u2 < T / 2; u2 += blockDim.x) {
      int u = 2 * u2;
      int t = 0;
      int64_t o = 0;
      for (int j = 1; j < p.nu; ++j)
        if ((u >> j) & 1) { t |= 1 << p.tpos_of_u[j]; o += p.uout[j]; }
      float2 a = tile[t], c = tile[t | (1 << p.tpos_of_u[0])];
      *reinterpret_cast<float4*>(out + bo + o) = make_float4(a.x, a.y, c.x, c.y);
    }
  }
}

// Register-precomputed variant: every thread moves J 16-byte units per tile, with its
// load / store offsets and tile indices computed once (they split into a per-thread part
// and a per-iteration part); J independent 16-byte loads in flight per thread.
// PAIR = true: complex64, a 16-byte unit is two elements (input pair along the input's
// fastest mode, output pair along the output's fastest mode).
template <typename E, bool PAIR, int J>
__global__ void __launch_bounds__(256) permute_kernel_v3(const E* __restrict__ in_e, E* __restrict__ out_e, PermPlan p,
                                                         int64_t nblocks, const int64_t* __restrict__ delta, int nub) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char sm[];
  using S = typename std::conditional<PAIR, float2, E>::type;  // smem element (one complex)
  S* tile = reinterpret_cast<S*>(sm);
  const S* in = reinterpret_cast<const S*>(in_e) + (delta ? delta[blockIdx.y] : 0);
  S* out = reinterpret_cast<S*>(out_e) + (delta ? delta[2 * nub + blockIdx.y] : 0);
  const int sh = PAIR ? 1 : 0;
  int64_t in_off[J], out_off[J];
  int ta[J];
  const int tb = PAIR ? (1 << p.tpos_of_u[0]) : 0;
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const int t = (threadIdx.x + 256 * j) << sh;
    int64_t o = 0;
    for (int i = sh; i < p.nu; ++i)
      if ((t >> i) & 1) o += p.tin[i];
    in_off[j] = o;
    int tt = 0;
    int64_t oo = 0;
    for (int i = sh; i < p.nu; ++i)
      if ((t >> i) & 1) { tt |= 1 << p.tpos_of_u[i]; oo += p.uout[i]; }
    ta[j] = tt;
    out_off[j] = oo;
  }
  for (int64_t b = blockIdx.x; b < nblocks; b += gridDim.x) {
    int64_t bi = 0, bo = 0;
    for (int i = 0; i < p.nrest; ++i)
      if ((b >> i) & 1) { bi += p.rin[i]; bo += p.rout[i]; }
    E v[J];
#pragma unroll
    for (int j = 0; j < J; ++j) v[j] = __ldcs(reinterpret_cast<const E*>(in + bi + in_off[j]));
    __syncthreads();
    // 16-byte units of the tile are XOR-swizzled inside 128-byte rows (unit u at u ^ h(u),
    // h = the XOR of u's 3-bit groups above the row): the output-order reads jump by large
    // powers of two in the input-order tile and hit one bank group unswizzled (ncu: 31.6 M of
    // 35.9 M shared wavefronts conflicted, profiles/r02c_*); the linear stores stay
    // conflict-free (h is constant within a row)
    auto swz = [](int u) { return u ^ (((u >> 3) ^ (u >> 6) ^ (u >> 9)) & 7); };
#pragma unroll
    for (int j = 0; j < J; ++j) reinterpret_cast<E*>(tile)[swz(threadIdx.x + 256 * j)] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (PAIR) {
        const int t0 = ta[j], t1 = ta[j] | tb;
        const float2 x0 = reinterpret_cast<const float2*>(tile)[(swz(t0 >> 1) << 1) | (t0 & 1)];
        const float2 x1 = reinterpret_cast<const float2*>(tile)[(swz(t1 >> 1) << 1) | (t1 & 1)];
        __stcs(reinterpret_cast<float4*>(out + bo + out_off[j]), make_float4(x0.x, x0.y, x1.x, x1.y));
      } else {
        __stcs(reinterpret_cast<E*>(out + bo + out_off[j]), reinterpret_cast<const E*>(tile)[swz(ta[j])]);
      }
    }
  }
}

}  // namespace

void launch_permute(int dtype, const void* in, void* out, int rank, const int* perm, const Batch& bt,
                    cudaStream_t st) {
  if (rank <= 0) {
    const size_t es = dtype == 0 ? 8 : 16;
    for (int b = 0; b < bt.nb; ++b)
      cudaMemcpyAsync((char*)out + es * bt.d(2, b), (const char*)in + es * bt.d(0, b), es, cudaMemcpyDeviceToDevice, st);
    return;
  }
  std::vector<int> inv(rank);
  for (int i = 0; i < rank; ++i) inv[perm[i]] = i;
  auto in_stride = [&](int j) { return (int64_t)1 << (rank - 1 - j); };
  auto out_stride = [&](int j) { return (int64_t)1 << (rank - 1 - inv[j]); };
  const int target = std::min(rank, dtype == 0 ? 11 : 10);
  std::vector<char> inU(rank, 0);
  int nu = 0;
  for (int s = 0; nu < target && s < rank; ++s) {
    int a = rank - 1 - s;           // input's s-th fastest mode
    int b = perm[rank - 1 - s];     // input mode that is the output's s-th fastest
    if (!inU[a] && nu < target) { inU[a] = 1; ++nu; }
    if (!inU[b] && nu < target) { inU[b] = 1; ++nu; }
  }
  PermPlan p{};
  p.nu = nu;
  std::vector<int> U;  // input modes in U, fastest input first
  for (int j = rank - 1; j >= 0; --j)
    if (inU[j]) U.push_back(j);
  for (int i = 0; i < nu; ++i) p.tin[i] = in_stride(U[i]);
  std::vector<int> byout(nu);
  for (int i = 0; i < nu; ++i) byout[i] = i;
  std::sort(byout.begin(), byout.end(), [&](int x, int y) { return out_stride(U[x]) < out_stride(U[y]); });
  for (int j = 0; j < nu; ++j) {
    p.tpos_of_u[j] = byout[j];
    p.uout[j] = out_stride(U[byout[j]]);
  }
  int nr = 0;
  for (int j = rank - 1; j >= 0; --j)
    if (!inU[j]) {
      p.rin[nr] = in_stride(j);
      p.rout[nr] = out_stride(j);
      ++nr;
    }
  p.nrest = nr;
  int64_t nblocks = (int64_t)1 << nr;
  const int nsm = sm_count();
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(nblocks, (int64_t)nsm * 16 / bt.nb + 1));
  const dim3 g((unsigned)grid, (unsigned)bt.nb);
  size_t smem = (size_t)(dtype == 0 ? 8 : 16) << nu;
  // 16-byte units per tile: 2^(nu-1) (c64 pairs) or 2^nu (c128); 4 per thread at full tiles
  const int units = dtype == 0 ? (1 << (nu - 1)) : (1 << nu);
  // (16-byte paths need every unit's tensors 16-byte aligned: per-slice pools and leaves are)
  const bool al = bt.all_even(0) && bt.all_even(2);
  if (nu >= 2 && units == 1024 && p.uout[0] == 1 && p.tin[0] == 1 && dtype == 0 && al) {
    launch_pdl(permute_kernel_v3<float4, true, 4>, g, 256, smem, st, (const float4*)in, (float4*)out, p, nblocks,
               bt.delta, bt.nb);
  } else if (units == 1024 && dtype == 1) {
    launch_pdl(permute_kernel_v3<double2, false, 4>, g, 256, smem, st, (const double2*)in, (double2*)out, p, nblocks,
               bt.delta, bt.nb);
  } else if (dtype == 0) {
    if (nu >= 2 && p.uout[0] == 1 && al)
      launch_pdl(permute_kernel_v2, g, 256, smem, st, (const float2*)in, (float2*)out, p, nblocks, bt.delta, bt.nb);
    else
      launch_pdl(permute_kernel<float2>, g, 256, smem, st, (const float2*)in, (float2*)out, p, nblocks, bt.delta,
                 bt.nb);
  } else {
    launch_pdl(permute_kernel<double2>, g, 256, smem, st, (const double2*)in, (double2*)out, p, nblocks, bt.delta,
               bt.nb);
  }
}

// ---- accumulate final contraction results into the complex128 group slots (a9) ----
namespace {
template <typename V>
__global__ void accum_kernel(const V* __restrict__ src, double2* __restrict__ dst, int64_t n,
                             const UnitDesc* __restrict__ units, const int64_t* __restrict__ delta, int nb) {
  pdl_wait();
  pdl_trigger();
  // one thread per output element walks the units in order: a slot's units are added in
  // ascending unit (slice) order, exactly as one launch per slice would
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    for (int b = 0; b < nb; ++b) {
      const V v = src[(delta ? delta[b] : 0) + j];
      double2* d = dst + (int64_t)units[b].slot * n + j;
      d->x += (double)v.x;
      d->y += (double)v.y;
    }
  }
}
}  // namespace

void launch_accum(int dtype, const void* src, void* dst, int64_t n, const UnitDesc* units, const Batch& bt,
                  cudaStream_t st) {
  if (n <= 0) return;
  unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 4096);
  if (dtype == 0)
    launch_pdl(accum_kernel<float2>, g, 256, 0, st, (const float2*)src, (double2*)dst, n, units, bt.delta, bt.nb);
  else
    launch_pdl(accum_kernel<double2>, g, 256, 0, st, (const double2*)src, (double2*)dst, n, units, bt.delta, bt.nb);
}

}  // namespace dev
}  // namespace tnqvm
