// a7 (tensor-core path, complex128): contraction-as-GEMM on FP64 DMMA
// (mma.sync.aligned.m8n8k4.row.col.f64), the double-precision tensor-core path used for
// the doubled (noisy) networks where complex128 is required.
//
// Same real-block form as the complex64 kernel: X viewed as fp64 [N][2K] (interleaved
// complex128), W[2K][2M] = real block of Y built by a prep kernel, C = X * W viewed as
// fp64 [N][2M] (interleaved complex128).  CTA tile 64 rows x 64 real columns, K chunk 16,
// 8 warps each owning a 32x16 sub-tile (4 x 2 m8n8 accumulators); operands staged in
// padded shared memory (conflict-free fragment loads), double-buffered via cp.async.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.hpp"
#include "pdl.cuh"

namespace tnqvm {
namespace dev {
namespace {

constexpr int DB_M = 64, DB_N = 64, DB_K = 16;
constexpr int A_LD = DB_K + 4;   // doubles per A row in smem (bank-conflict-free fragments)
constexpr int B_LD = DB_N + 4;   // doubles per W row in smem

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// W[2K][2M] (fp64 row-major) from complex128 Y gathered with bit strides
__global__ void __launch_bounds__(256) dmma_prep_kernel(const double2* __restrict__ Y, double* __restrict__ W,
                                                        GemmDesc g, const int64_t* __restrict__ delta, int nb,
                                                        int64_t wstride) {
  pdl_wait();
  pdl_trigger();
  if (delta) {  // unit blockIdx.z: its Y, its W slab
    Y += delta[nb + blockIdx.z];
    W += (int64_t)blockIdx.z * wstride;
  }
  const int64_t K = (int64_t)1 << g.nk, M = (int64_t)1 << g.nm, M2 = 2 * M;
  const int64_t k = blockIdx.x;
  const int64_t m = (int64_t)blockIdx.y * 256 + threadIdx.x;
  if (k >= K || m >= M) return;
  int64_t o = 0;
  for (int i = 0; i < g.nk; ++i)
    if ((k >> i) & 1) o += g.syk[i];
  for (int i = 0; i < g.nm; ++i)
    if ((m >> i) & 1) o += g.sym[i];
  const double2 y = Y[o];
  // W[2k][2m] = Yr, W[2k][2m+1] = Yi, W[2k+1][2m] = -Yi, W[2k+1][2m+1] = Yr
  *reinterpret_cast<double2*>(W + (2 * k) * M2 + 2 * m) = make_double2(y.x, y.y);
  *reinterpret_cast<double2*>(W + (2 * k + 1) * M2 + 2 * m) = make_double2(-y.y, y.x);
}

__global__ void __launch_bounds__(256) dmma_gemm_kernel(const double* __restrict__ X, const double* __restrict__ W,
                                                        double* __restrict__ Cout, int64_t N, int K2, int M2,
                                                        int kchunk, int splits, const int64_t* __restrict__ delta, int nb,
    int64_t wstride, int64_t pstride) {
  pdl_wait();
  pdl_trigger();
  // blockIdx.z = unit * splits + split; split-K: split z covers K range [z*kchunk, (z+1)*kchunk),
  // partials land in slab z of the unit's partial area (pstride > 0), else in the unit's C
  const int ub = blockIdx.z / splits, zs = blockIdx.z % splits;
  if (delta) {
    X += 2 * delta[ub];
    W += (int64_t)ub * wstride;
    Cout += pstride ? (int64_t)ub * pstride : 2 * delta[2 * nb + ub];
  }
  const int kbeg = zs * kchunk;
  const int kend = min(K2, kbeg + kchunk);
  double* __restrict__ C = Cout + (size_t)zs * (size_t)N * M2;
  __shared__ __align__(16) double As[2][DB_M * A_LD];
  __shared__ __align__(16) double Bs[2][DB_K * B_LD];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n0 = (int64_t)blockIdx.x * DB_M;
  const int m0 = blockIdx.y * DB_N;
  const int wr = (warp >> 2) * 32;  // warp row offset in tile (0 / 32)
  const int wc = (warp & 3) * 16;   // warp col offset (0,16,32,48)
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  auto load = [&](int buf, int kc) {
    // A: 64 rows x 16 k  (1024 doubles, 4 per thread)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = tid + i * 256;
      int r = e >> 4, kk = e & 15;
      int64_t n = n0 + r;
      int k = kc + kk;
      bool ok = n < N && k < kend;
      cp_async8(&As[buf][r * A_LD + kk], ok ? X + n * K2 + k : X, ok);
    }
    // W: 16 k x 64 cols
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = tid + i * 256;
      int kk = e >> 6, c = e & 63;
      int k = kc + kk, col = m0 + c;
      bool ok = k < kend && col < M2;
      cp_async8(&Bs[buf][kk * B_LD + c], ok ? W + (int64_t)k * M2 + col : W, ok);
    }
    cp_async_commit();
  };

  const int nk = (kend - kbeg + DB_K - 1) / DB_K;
  load(0, kbeg);
  for (int c = 0; c < nk; ++c) {
    const int buf = c & 1;
    if (c + 1 < nk) {
      load(buf ^ 1, kbeg + (c + 1) * DB_K);
      cp_async_wait1();
    } else {
      cp_async_wait0();
    }
    __syncthreads();
    const double* A = As[buf];
    const double* Bm = Bs[buf];
#pragma unroll
    for (int ks = 0; ks < DB_K; ks += 4) {
      double a[4], b[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = A[(wr + i * 8 + (lane >> 2)) * A_LD + ks + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 2; ++j) b[j] = Bm[(ks + (lane & 3)) * B_LD + wc + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    __syncthreads();
  }
  // epilogue: D fragment c0 = D[lane/4][2*(lane%4)], c1 = D[lane/4][2*(lane%4)+1]
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t n = n0 + wr + i * 8 + (lane >> 2);
    if (n >= N) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int col = m0 + wc + j * 8 + 2 * (lane & 3);
      if (col + 1 < M2) {
        *reinterpret_cast<double2*>(C + n * M2 + col) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else if (col < M2) {
        C[n * M2 + col] = acc[i][j][0];
      }
    }
  }
}


// Larger tile for the FP64-bound steps: CTA 128 rows x TN real columns (TN = 64: 8 warps in a
// 4 x 2 grid each owning 32 x 32, 4 x 4 m8n8 accumulators -- 16 DMMAs per 8 fragment loads;
// TN = 32 for narrow outputs (M <= 16 complex, C5's low-K steps wasted half of a 64-column
// tile): 8 x 1 warps of 16 x 32), K chunk 16, 3-stage cp.async ring with 16-byte copies,
// dynamic shared memory.  Every output element sums its K in the same order in both tiles.
constexpr int D2_M = 128, D2_K = 16, D2_S = 3;
constexpr int D2_ALD = D2_K + 4;
template <int TN>
constexpr int d2_smem() { return D2_S * (D2_M * D2_ALD + D2_K * (TN + 4)) * 8; }
__device__ __forceinline__ void cp_async16z(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
template <int D2_N>
__global__ void __launch_bounds__(256, 2) dmma_gemm2_kernel(const double* __restrict__ X, const double* __restrict__ W,
                                                           double* __restrict__ Cout, int64_t N, int K2, int M2,
                                                           int kchunk, int splits, const int64_t* __restrict__ delta, int nb,
    int64_t wstride, int64_t pstride) {
  pdl_wait();
  pdl_trigger();
  const int ub = blockIdx.z / splits, zs = blockIdx.z % splits;
  if (delta) {
    X += 2 * delta[ub];
    W += (int64_t)ub * wstride;
    Cout += pstride ? (int64_t)ub * pstride : 2 * delta[2 * nb + ub];
  }
  const int kbeg = zs * kchunk;
  const int kend = min(K2, kbeg + kchunk);
  double* __restrict__ C = Cout + (size_t)zs * (size_t)N * M2;
  extern __shared__ __align__(16) double d2s[];
  double* As = d2s;                          // [S][128][ALD]
  double* Bs = d2s + D2_S * D2_M * D2_ALD;   // [S][16][BLD]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n0 = (int64_t)blockIdx.x * D2_M;
  const int m0 = blockIdx.y * D2_N;
  constexpr int D2_BLD = D2_N + 4;
  constexpr int WN = D2_N / 32, FM = 2 * WN;  // warps along columns; row fragments per warp (32 / 16 rows)
  const int wr = (warp / WN) * (8 * FM);     // 64-col: 0, 32, 64, 96; 32-col: 0, 16, ..., 112
  const int wc = (warp % WN) * 32;
  double acc[FM][4][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  auto load = [&](int stg, int kc) {
    double* A = As + stg * D2_M * D2_ALD;
    double* B = Bs + stg * D2_K * D2_BLD;
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // A: 128 rows x 8 pairs
      const int e = tid + i * 256;
      const int r = e >> 3, kk = (e & 7) * 2;
      const int64_t n = n0 + r;
      const int k = kc + kk;
      const bool ok = n < N && k < kend;  // K2 even: a pair never straddles kend
      cp_async16z(&A[r * D2_ALD + kk], ok ? X + n * K2 + k : X, ok);
    }
#pragma unroll
    for (int i = 0; i < D2_N / 32; ++i) {  // W: 16 k x D2_N/2 pairs
      const int e = tid + i * 256;
      const int kk = e / (D2_N / 2), c = (e % (D2_N / 2)) * 2;
      const int k = kc + kk, col = m0 + c;
      const bool ok = k < kend && col < M2;  // M2 even
      cp_async16z(&B[kk * D2_BLD + c], ok ? W + (int64_t)k * M2 + col : W, ok);
    }
  };
  const int nk = (kend - kbeg + D2_K - 1) / D2_K;
#pragma unroll
  for (int s0 = 0; s0 < D2_S - 1; ++s0) {
    if (s0 < nk) load(s0, kbeg + s0 * D2_K);
    cp_async_commit();
  }
  for (int c = 0; c < nk; ++c) {
    asm volatile("cp.async.wait_group %0;" ::"n"(D2_S - 2) : "memory");
    __syncthreads();  // chunk c landed everywhere; the stage refilled below was consumed
    if (c + D2_S - 1 < nk) load((c + D2_S - 1) % D2_S, kbeg + (c + D2_S - 1) * D2_K);
    cp_async_commit();
    const double* A = As + (c % D2_S) * D2_M * D2_ALD;
    const double* Bm = Bs + (c % D2_S) * D2_K * D2_BLD;
#pragma unroll
    for (int ks = 0; ks < D2_K; ks += 4) {
      double a[FM], b[4];
#pragma unroll
      for (int i = 0; i < FM; ++i) a[i] = A[(wr + i * 8 + (lane >> 2)) * D2_ALD + ks + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bm[(ks + (lane & 3)) * D2_BLD + wc + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
#pragma unroll
  for (int i = 0; i < FM; ++i) {
    const int64_t n = n0 + wr + i * 8 + (lane >> 2);
    if (n >= N) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = m0 + wc + j * 8 + 2 * (lane & 3);
      if (col + 1 < M2) {
        *reinterpret_cast<double2*>(C + n * M2 + col) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else if (col < M2) {
        C[n * M2 + col] = acc[i][j][0];
      }
    }
  }
}

__global__ void dmma_splitk_reduce(const double* __restrict__ part, double* __restrict__ C, int64_t n, int splits,
                                   const int64_t* __restrict__ delta, int nb, int64_t pstride) {
  pdl_wait();
  pdl_trigger();
  if (delta) {  // unit blockIdx.y
    part += (int64_t)blockIdx.y * pstride;
    C += 2 * delta[2 * nb + blockIdx.y];
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += part[(int64_t)z * n + i];
    C[i] = s;
  }
}

// split-K from the per-unit shape only (the summation order of a slice never depends on
// how many units share the launch)
int dmma_splits(int64_t N, int nk, int nm, int* kchunk) {
  const int nsm = 148;  // fixed: the partition must not depend on the device either
  const int64_t K2 = (int64_t)2 << nk, M2 = (int64_t)2 << nm;
  const int64_t tiles = ((N + DB_M - 1) / DB_M) * ((M2 + DB_N - 1) / DB_N);
  int splits = 1;
  if (tiles < 2 * nsm && K2 / DB_K >= 16)
    splits = (int)std::max<int64_t>(1, std::min<int64_t>((2 * nsm + tiles - 1) / tiles, K2 / DB_K / 8));
  int64_t kc = (K2 + splits - 1) / splits;
  kc = (kc + DB_K - 1) / DB_K * DB_K;
  splits = (int)((K2 + kc - 1) / kc);
  *kchunk = (int)kc;
  return splits;
}

}  // namespace

size_t dmma_wbuf_bytes(int64_t N, int nk, int nm) {
  int kc;
  int splits = dmma_splits(N, nk, nm, &kc);
  size_t part = splits > 1 ? (size_t)splits * (size_t)N * ((size_t)2 << nm) * 8 : 0;
  return ((size_t)32 << (nk + nm)) + part;  // fp64 W [2K][2M] + split-K partials
}

bool dmma_supported(int nk, int nm) { return nk + nm <= 28 && nm <= 20 && nk <= 26; }

void launch_gemm_dmma(const GemmDesc& g, void* wbuf, const Batch& bt, cudaStream_t st) {
  const int64_t K = (int64_t)1 << g.nk, M = (int64_t)1 << g.nm;
  const int nb = bt.nb;
  double* W = reinterpret_cast<double*>(wbuf);
  const int64_t wunit = (int64_t)(dmma_wbuf_bytes(g.N, g.nk, g.nm) / 8);  // doubles per unit slab
  dim3 pg((unsigned)K, (unsigned)((M + 255) / 256), (unsigned)nb);
  launch_pdl(dmma_prep_kernel, pg, 256, 0, st, reinterpret_cast<const double2*>(g.Y), W, g, bt.delta, nb, wunit);
  const int K2 = (int)(2 * K), M2 = (int)(2 * M);
  int kchunk;
  const int splits = dmma_splits(g.N, g.nk, g.nm, &kchunk);
  // partials follow W in the unit's slab
  double* out = splits > 1 ? W + (size_t)K2 * M2 : reinterpret_cast<double*>(g.C);
  const int64_t pstride = splits > 1 ? wunit : 0;
  // the 128 x 64 tile when the launch is large enough to fill the machine with it (same
  // per-element summation order as the 64 x 64 tile: bit-identical)
  // the 128-row tiles when the launch is large enough to fill the machine with them (same
  // per-element summation order as the 64 x 64 tile: bit-identical); 32 real columns when
  // the output is that narrow
  const bool narrow = M2 <= 32;
  const int tn = narrow ? 32 : 64;
  const bool big =
      (M2 >= 64 || narrow) && ((g.N + D2_M - 1) / D2_M) * ((M2 + tn - 1) / tn) * splits * nb >= 2 * sm_count();
  if (big) {
    dim3 grid((unsigned)((g.N + D2_M - 1) / D2_M), (unsigned)((M2 + tn - 1) / tn), (unsigned)(splits * nb));
    if (narrow) {
      cudaFuncSetAttribute(dmma_gemm2_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, d2_smem<32>());
      launch_pdl(dmma_gemm2_kernel<32>, grid, 256, (size_t)d2_smem<32>(), st, reinterpret_cast<const double*>(g.X), W,
                 out, g.N, K2, M2, kchunk, splits, bt.delta, nb, wunit, pstride);
    } else {
      cudaFuncSetAttribute(dmma_gemm2_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, d2_smem<64>());
      launch_pdl(dmma_gemm2_kernel<64>, grid, 256, (size_t)d2_smem<64>(), st, reinterpret_cast<const double*>(g.X), W,
                 out, g.N, K2, M2, kchunk, splits, bt.delta, nb, wunit, pstride);
    }
  } else {
    dim3 grid((unsigned)((g.N + DB_M - 1) / DB_M), (unsigned)((M2 + DB_N - 1) / DB_N), (unsigned)(splits * nb));
    launch_pdl(dmma_gemm_kernel, grid, 256, 0, st, reinterpret_cast<const double*>(g.X), W, out, g.N, K2, M2, kchunk,
               splits, bt.delta, nb, wunit, pstride);
  }
  if (splits > 1) {
    const int64_t n = g.N * (int64_t)M2;
    const dim3 rg((unsigned)std::min<int64_t>((n + 255) / 256, 8192), (unsigned)nb);
    launch_pdl(dmma_splitk_reduce, rg, 256, 0, st, out, reinterpret_cast<double*>(g.C), n, splits, bt.delta, nb,
               pstride);
  }
}

}  // namespace dev
}  // namespace tnqvm
