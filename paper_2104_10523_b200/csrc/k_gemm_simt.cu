// a7 (SIMT path): streaming complex contraction-as-GEMM for low-arithmetic-intensity steps.
//
// A pairwise contraction step of the plan is C[n][m] = sum_k X[n][k] Y(k, m)
// with X the big operand (row-major, contracted modes contiguous) and Y the small one.
// When K*M is small the step is HBM-bound far below the FP32 ridge: the kernel streams
// X tiles through shared memory with 16-byte coalesced loads, keeps Y (gathered from any
// layout with bit strides) resident in shared memory, accumulates complex products in
// registers (exact fp32 / fp64 FMA), and writes C tiles back through shared memory with
// coalesced 16-byte stores.  Grid = a multiple of the SM count, persistent over row tiles.
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.hpp"
#include "pdl.cuh"

namespace tnqvm {
namespace dev {
namespace {

template <typename T> struct C2;
template <> struct C2<float> { using t = float2; };
template <> struct C2<double> { using t = double2; };

constexpr int kThreads = 256;

// MPT: output columns per thread.  G = column groups, R32 = 32-row slabs per tile.
template <typename T, int MPT>
__global__ void __launch_bounds__(kThreads) gemm_simt_kernel(GemmDesc g, int mtile, int G, int R32) {
  pdl_wait();
  pdl_trigger();
  using V = typename C2<T>::t;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = 1 << g.nk, M = 1 << g.nm;
  const int TR = 32 * R32;
  const int KP = K + 1;  // padded row stride of the X tile
  V* Ws = reinterpret_cast<V*>(smem_raw);              // [K][mtile]
  V* Xs = Ws + (size_t)K * mtile;                       // [TR][KP]
  V* Cs = Xs + (size_t)TR * KP;                         // [TR][mtile]
  const V* __restrict__ X = reinterpret_cast<const V*>(g.X);
  const V* __restrict__ Y = reinterpret_cast<const V*>(g.Y);
  V* __restrict__ C = reinterpret_cast<V*>(g.C);
  const int m0 = blockIdx.y * mtile;

  // gather the small operand once per CTA
  for (int t = threadIdx.x; t < K * mtile; t += kThreads) {
    int k = t / mtile, m = m0 + t % mtile;
    int64_t o = 0;
    for (int i = 0; i < g.nk; ++i)
      if ((k >> i) & 1) o += g.syk[i];
    for (int i = 0; i < g.nm; ++i)
      if ((m >> i) & 1) o += g.sym[i];
    Ws[t] = Y[o];
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = (warp % R32) * 32 + lane;
  const int grp = warp / R32;
  const int64_t ntiles = (g.N + TR - 1) / TR;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * TR;
    const int rows = (int)((g.N - r0) < (int64_t)TR ? (g.N - r0) : (int64_t)TR);
    __syncthreads();
    // X tile: rows*K contiguous complex values
    const V* src = X + r0 * K;
    const int64_t nval = (int64_t)rows * K;
    if (sizeof(V) == 8 && (K % 2 == 0)) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
      for (int64_t t = threadIdx.x; t < nval / 2; t += kThreads) {
        float4 v = __ldg(s4 + t);
        int64_t e = 2 * t;
        int r = (int)(e / K), k = (int)(e % K);
        V* d = Xs + (size_t)r * KP + k;
        reinterpret_cast<float2*>(d)[0] = make_float2(v.x, v.y);
        reinterpret_cast<float2*>(d)[1] = make_float2(v.z, v.w);
      }
    } else {
      for (int64_t t = threadIdx.x; t < nval; t += kThreads) {
        int r = (int)(t / K), k = (int)(t % K);
        Xs[(size_t)r * KP + k] = src[t];
      }
    }
    __syncthreads();
    T acc_re[MPT], acc_im[MPT];
#pragma unroll
    for (int i = 0; i < MPT; ++i) { acc_re[i] = 0; acc_im[i] = 0; }
    if (row < rows) {
      const V* xr = Xs + (size_t)row * KP;
      for (int k = 0; k < K; ++k) {
        V x = xr[k];
        const V* wk = Ws + (size_t)k * mtile + grp;
#pragma unroll
        for (int i = 0; i < MPT; ++i) {
          V w = wk[i * G];
          acc_re[i] = fma(x.x, w.x, acc_re[i]);
          acc_re[i] = fma(-x.y, w.y, acc_re[i]);
          acc_im[i] = fma(x.x, w.y, acc_im[i]);
          acc_im[i] = fma(x.y, w.x, acc_im[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < MPT; ++i) {
        V c;
        c.x = acc_re[i];
        c.y = acc_im[i];
        Cs[(size_t)row * mtile + grp + i * G] = c;
      }
    }
    __syncthreads();
    // coalesced store of the C tile (rows x mtile, row stride M in global)
    if (mtile == M) {
      V* dst = C + r0 * M;
      const int64_t n = (int64_t)rows * M;
      if (sizeof(V) == 8 && (n % 2 == 0)) {
        float4* d4 = reinterpret_cast<float4*>(dst);
        const float4* s4 = reinterpret_cast<const float4*>(Cs);
        for (int64_t t = threadIdx.x; t < n / 2; t += kThreads) d4[t] = s4[t];
      } else {
        for (int64_t t = threadIdx.x; t < n; t += kThreads) dst[t] = Cs[t];
      }
    } else {
      for (int t = threadIdx.x; t < rows * mtile; t += kThreads) {
        int r = t / mtile, m = t % mtile;
        C[(r0 + r) * M + m0 + m] = Cs[t];
      }
    }
  }
}

// Classic register-blocked tiled GEMM for the remaining shapes (large K or M): 64x64
// complex output tile per CTA, K chunks of 16 staged in shared memory, 4x4 complex
// micro-tile per thread.
constexpr int TB_N = 64, TB_M = 64, TB_K = 16;

template <typename T>
__global__ void __launch_bounds__(256) gemm_tiled_kernel(GemmDesc g) {
  pdl_wait();
  pdl_trigger();
  using V = typename C2<T>::t;
  __shared__ V Xs[TB_K][TB_N + 1];
  __shared__ V Ws[TB_K][TB_M];
  __shared__ int64_t offm[TB_M];
  const int64_t K = (int64_t)1 << g.nk, M = (int64_t)1 << g.nm;
  const V* __restrict__ X = reinterpret_cast<const V*>(g.X);
  const V* __restrict__ Y = reinterpret_cast<const V*>(g.Y);
  V* __restrict__ C = reinterpret_cast<V*>(g.C);
  const int64_t n0 = (int64_t)blockIdx.x * TB_N, m0 = (int64_t)blockIdx.y * TB_M;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  if (tid < TB_M) {
    int64_t m = m0 + tid, o = 0;
    for (int i = 0; i < g.nm; ++i)
      if ((m >> i) & 1) o += g.sym[i];
    offm[tid] = o;
  }
  T cr[4][4], ci[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) { cr[i][j] = 0; ci[i][j] = 0; }
  for (int64_t kc = 0; kc < K; kc += TB_K) {
    __syncthreads();
    {  // X tile: 64 rows x 16 k
      int r = tid / 4, kk0 = (tid % 4) * 4;
      int64_t n = n0 + r;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int64_t k = kc + kk0 + i;
        V v;
        v.x = 0; v.y = 0;
        if (n < g.N && k < K) v = X[n * K + k];
        Xs[kk0 + i][r] = v;
      }
    }
    {  // W tile: 16 k x 64 m, gathered from Y's layout
      int kk = tid / 16, mm0 = (tid % 16) * 4;
      int64_t k = kc + kk, ok = 0;
      for (int i = 0; i < g.nk; ++i)
        if ((k >> i) & 1) ok += g.syk[i];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        V v;
        v.x = 0; v.y = 0;
        if (k < K && m0 + mm0 + j < M) v = Y[ok + offm[mm0 + j]];
        Ws[kk][mm0 + j] = v;
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < TB_K; ++kk) {
      V a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Xs[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Ws[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          cr[i][j] = fma(a[i].x, b[j].x, cr[i][j]);
          cr[i][j] = fma(-a[i].y, b[j].y, cr[i][j]);
          ci[i][j] = fma(a[i].x, b[j].y, ci[i][j]);
          ci[i][j] = fma(a[i].y, b[j].x, ci[i][j]);
        }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t n = n0 + ty * 4 + i;
    if (n >= g.N) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t m = m0 + tx * 4 + j;
      if (m < M) {
        V v;
        v.x = cr[i][j];
        v.y = ci[i][j];
        C[n * M + m] = v;
      }
    }
  }
}

template <typename T>
void launch_t(const GemmDesc& g, cudaStream_t st) {
  using V = typename C2<T>::t;
  const int K = 1 << g.nk, M = 1 << g.nm;
  if (g.nk > 8 || g.nm > 8) {
    dim3 grid((unsigned)((g.N + TB_N - 1) / TB_N), (unsigned)((M + TB_M - 1) / TB_M));
    launch_pdl(gemm_tiled_kernel<T>, grid, 256, 0, st, g);
    return;
  }
  // tile M so that W fits in ~48 KB
  const int wcap = (int)(49152 / sizeof(V));
  int mtile = M;
  while ((int64_t)K * mtile > wcap && mtile > 1) mtile >>= 1;
  mtile = std::min(mtile, 256);
  int G = std::min(8, mtile);
  int R32 = 8 / G;
  int MPT = mtile / G;
  int TR = 32 * R32;
  size_t smem = sizeof(V) * ((size_t)K * mtile + (size_t)TR * (K + 1) + (size_t)TR * mtile);
  const int nsm = sm_count();
  int64_t ntiles = (g.N + TR - 1) / TR;
  int per_sm = (int)std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / std::max<size_t>(smem, 1)));
  int64_t gx = std::min<int64_t>(ntiles, (int64_t)nsm * per_sm / std::max(1, M / mtile) + 1);
  gx = std::max<int64_t>(gx, 1);
  dim3 grid((unsigned)gx, (unsigned)(M / mtile));
#define TNQVM_SIMT_CASE(P)                                                                      \
  case P:                                                                                       \
    cudaFuncSetAttribute(gemm_simt_kernel<T, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                         (int)smem);                                                            \
    launch_pdl(gemm_simt_kernel<T, P>, grid, kThreads, smem, st, g, mtile, G, R32);                      \
    break;
  switch (MPT) {
    TNQVM_SIMT_CASE(1)
    TNQVM_SIMT_CASE(2)
    TNQVM_SIMT_CASE(4)
    TNQVM_SIMT_CASE(8)
    TNQVM_SIMT_CASE(16)
    TNQVM_SIMT_CASE(32)
    default: break;
  }
#undef TNQVM_SIMT_CASE
}

// ---- split-K: C[n][m] = sum_k X[n][k] Y[m][k], tiny N*M, huge K ----
// K chunk per partial: enough chunks for 4 CTAs per SM (a fixed function of K and the SM
// count, so the summation order is fixed), at least 1024 (one UNR x 256-thread sweep)
constexpr int64_t kChunkMin = 1 << 10;
inline int64_t chunk_of(int64_t K) {
  const int64_t target = (int64_t)148 * 4;  // fixed partition (deterministic on any device)
  int64_t c = kChunkMin;
  while (c * 2 * target <= K) c <<= 1;
  return c;
}

// One CTA per K chunk computes every (n, m) pair (N*M <= 16): X and Y are each read
// once, UNR independent loads per operand row in flight per thread, fp32 partial sums per
// thread (<= 128 terms) combined in fp64 across threads and chunks.
template <typename T, int NN, int MM>
__global__ void __launch_bounds__(kThreads) splitk_partial_t(const typename C2<T>::t* __restrict__ X,
                                                             const typename C2<T>::t* __restrict__ Y,
                                                             double2* __restrict__ part, int64_t K, int64_t kChunk) {
  pdl_wait();
  pdl_trigger();
  using V = typename C2<T>::t;
  constexpr int NP = NN * MM, UNR = 4;
  const int64_t nchunks = (K + kChunk - 1) / kChunk;
  double dre[NP], dim_[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) dre[p] = dim_[p] = 0.0;
  // persistent CTAs walk chunks b, b+G, ... (fixed order: deterministic)
  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
  const int64_t k0 = chunk * kChunk, k1 = (K < k0 + kChunk) ? K : k0 + kChunk;
  T re[NP], im[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) re[p] = im[p] = 0;
  for (int64_t kb = k0 + threadIdx.x; kb < k1; kb += (int64_t)kThreads * UNR) {
    V xv[UNR][NN], yv[UNR][MM];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t k = kb + (int64_t)u * kThreads;
      const bool ok = k < k1;
#pragma unroll
      for (int i = 0; i < NN; ++i) {
        if (ok) xv[u][i] = __ldcs(X + i * K + k);
        else { xv[u][i].x = 0; xv[u][i].y = 0; }
      }
#pragma unroll
      for (int i = 0; i < MM; ++i) {
        if (ok) yv[u][i] = __ldcs(Y + i * K + k);
        else { yv[u][i].x = 0; yv[u][i].y = 0; }
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int n = 0; n < NN; ++n)
#pragma unroll
        for (int m = 0; m < MM; ++m) {
          const V a = xv[u][n], b = yv[u][m];
          re[n * MM + m] = fma(a.x, b.x, fma(-a.y, b.y, re[n * MM + m]));
          im[n * MM + m] = fma(a.x, b.y, fma(a.y, b.x, im[n * MM + m]));
        }
  }
#pragma unroll
  for (int p = 0; p < NP; ++p) { dre[p] += (double)re[p]; dim_[p] += (double)im[p]; }
  }
  __shared__ double sred[kThreads / 32][NP][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    double r = dre[p], i = dim_[p];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      r += __shfl_xor_sync(0xffffffffu, r, o);
      i += __shfl_xor_sync(0xffffffffu, i, o);
    }
    if (lane == 0) { sred[warp][p][0] = r; sred[warp][p][1] = i; }
  }
  __syncthreads();
  if (threadIdx.x < NP) {
    double r = 0, i = 0;
    for (int w = 0; w < kThreads / 32; ++w) { r += sred[w][threadIdx.x][0]; i += sred[w][threadIdx.x][1]; }
    part[(int64_t)blockIdx.x * NP + threadIdx.x] = make_double2(r, i);
  }
}

// General split-K (16 < N*M <= 256, N + M <= 64): per K tile of 64 the CTA stages the N
// rows of X and M rows of Y in shared memory (coalesced along K); thread t owns pair t.
constexpr int kGenKT = 64;
template <typename T>
__global__ void __launch_bounds__(kThreads) splitk_general(const typename C2<T>::t* __restrict__ X,
                                                           const typename C2<T>::t* __restrict__ Y,
                                                           double2* __restrict__ part, int N, int M, int64_t K,
                                                           int64_t kChunk) {
  pdl_wait();
  pdl_trigger();
  using V = typename C2<T>::t;
  constexpr int kPad = kGenKT + 1;  // odd row pitch: the M (and N) rows read at the same kk hit distinct banks
  constexpr int kPer = (64 * kGenKT) / kThreads;  // loads per thread per tile at N + M = 64
  extern __shared__ __align__(16) unsigned char smraw[];
  V* xs = reinterpret_cast<V*>(smraw);   // [N][kPad]
  V* ys = xs + N * kPad;                 // [M][kPad]
  const int NM = N * M, t = threadIdx.x;
  const int n = t / M, m = t % M;
  const int nel = (N + M) * kGenKT;
  // this CTA's tiles: chunks b, b + G, ... each split into 64-wide K tiles; the next tile is
  // prefetched into registers while the current one is multiplied from shared memory
  const int64_t nchunks = (K + kChunk - 1) / kChunk;
  V pre[kPer];
  int64_t chunk = blockIdx.x, kt = chunk * kChunk;
  auto fetch = [&](int64_t c, int64_t k) {
    const int64_t k1 = (K < (c + 1) * kChunk) ? K : (c + 1) * kChunk;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = t + i * kThreads;
      const int r = e / kGenKT, kk = e % kGenKT;
      V v;
      v.x = 0;
      v.y = 0;
      if (c < nchunks && e < nel && k + kk < k1)
        v = r < N ? __ldcs(X + (int64_t)r * K + k + kk) : __ldcs(Y + (int64_t)(r - N) * K + k + kk);
      pre[i] = v;
    }
  };
  fetch(chunk, kt);
  double dr = 0, di = 0;
  while (chunk < nchunks) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = t + i * kThreads;
      if (e < nel) xs[(e / kGenKT) * kPad + e % kGenKT] = pre[i];  // rows 0..N-1 then the M rows of Y
    }
    __syncthreads();
    int64_t nk = kt + kGenKT, nc = chunk;
    if (nk >= ((K < (chunk + 1) * kChunk) ? K : (chunk + 1) * kChunk)) {
      nc = chunk + gridDim.x;
      nk = nc * kChunk;
    }
    fetch(nc, nk);
    if (t < NM) {
      const V* xr = xs + n * kPad;
      const V* yr = ys + m * kPad;
      T re = 0, im = 0;
#pragma unroll 8
      for (int kk = 0; kk < kGenKT; ++kk) {
        const V a = xr[kk], b = yr[kk];
        re = fma(a.x, b.x, fma(-a.y, b.y, re));
        im = fma(a.x, b.y, fma(a.y, b.x, im));
      }
      dr += (double)re;
      di += (double)im;
    }
    __syncthreads();
    chunk = nc;
    kt = nk;
  }
  if (t < NM) part[(int64_t)blockIdx.x * NM + t] = make_double2(dr, di);
}

template <typename T>
__global__ void splitk_final(const double2* __restrict__ part, typename C2<T>::t* __restrict__ C,
                             int64_t NM, int64_t chunks) {
  pdl_wait();
  pdl_trigger();
  for (int64_t p = blockIdx.x * blockDim.x + threadIdx.x; p < NM; p += (int64_t)gridDim.x * blockDim.x) {
    double re = 0, im = 0;
    for (int64_t c = 0; c < chunks; ++c) {
      re += part[c * NM + p].x;
      im += part[c * NM + p].y;
    }
    typename C2<T>::t v;
    v.x = (T)re;
    v.y = (T)im;
    C[p] = v;
  }
}

}  // namespace

void launch_gemm_simt(int dtype, const GemmDesc& g0, const Batch& bt, cudaStream_t st) {
  if (g0.N <= 0) return;
  const size_t es = dtype == 0 ? 8 : 16;
  for (int b = 0; b < bt.nb; ++b) {  // fallback path: one launch per unit
    GemmDesc g = g0;
    g.X = (const char*)g0.X + es * bt.d(0, b);
    g.Y = (const char*)g0.Y + es * bt.d(1, b);
    g.C = (char*)g0.C + es * bt.d(2, b);
    if (dtype == 0) launch_t<float>(g, st);
    else launch_t<double>(g, st);
  }
}

size_t splitk_scratch_bytes(int dtype, int64_t N, int64_t M, int64_t K) {
  (void)dtype;
  int64_t chunks = (K + chunk_of(K) - 1) / chunk_of(K);
  return sizeof(double2) * (size_t)chunks * (size_t)(N * M);
}

void launch_splitk_one(int dtype, const void* X, const void* Y, void* C, int64_t N, int64_t M, int64_t K,
                       void* scratch, cudaStream_t st);
void launch_splitk(int dtype, const void* X, const void* Y, void* C, int64_t N, int64_t M, int64_t K,
                   void* scratch, const Batch& bt, cudaStream_t st) {
  const size_t es = dtype == 0 ? 8 : 16;
  const size_t sb = splitk_scratch_bytes(dtype, N, M, K);
  for (int b = 0; b < bt.nb; ++b)  // one launch pair per unit, each with its own partial slab
    launch_splitk_one(dtype, (const char*)X + es * bt.d(0, b), (const char*)Y + es * bt.d(1, b),
                      (char*)C + es * bt.d(2, b), N, M, K, (char*)scratch + sb * b, st);
}
void launch_splitk_one(int dtype, const void* X, const void* Y, void* C, int64_t N, int64_t M, int64_t K,
                       void* scratch, cudaStream_t st) {
  const int64_t kChunk = chunk_of(K);
  int64_t chunks = std::min<int64_t>((K + kChunk - 1) / kChunk, (int64_t)148 * 4);  // = CTAs (partials)
  dim3 grid((unsigned)chunks);
  auto go = [&](auto tag) {
    using T = decltype(tag);
    using V = typename C2<T>::t;
    const V* x = (const V*)X;
    const V* y = (const V*)Y;
    double2* pp = (double2*)scratch;
#define TNQVM_SK(n, m) \
    if (N == n && M == m) launch_pdl(splitk_partial_t<T, n, m>, grid, kThreads, 0, st, x, y, pp, K, kChunk);
    TNQVM_SK(1, 1) TNQVM_SK(2, 1) TNQVM_SK(1, 2) TNQVM_SK(2, 2) TNQVM_SK(4, 1) TNQVM_SK(1, 4) TNQVM_SK(4, 2)
    TNQVM_SK(2, 4) TNQVM_SK(4, 4) TNQVM_SK(8, 1) TNQVM_SK(1, 8) TNQVM_SK(8, 2) TNQVM_SK(2, 8) TNQVM_SK(16, 1)
    TNQVM_SK(1, 16)
#undef TNQVM_SK
    if (N * M > 16) {
      const size_t smem = sizeof(V) * (size_t)(N + M) * (kGenKT + 1);
      cudaFuncSetAttribute(splitk_general<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      launch_pdl(splitk_general<T>, grid, kThreads, smem, st, x, y, pp, (int)N, (int)M, K, kChunk);
    }
    launch_pdl(splitk_final<T>, (unsigned)std::max<int64_t>(1, (N * M + 255) / 256), 256, 0, st, 
        (const double2*)scratch, (V*)C, N * M, chunks);
  };
  if (dtype == 0) go(float{});
  else go(double{});
}

}  // namespace dev
}  // namespace tnqvm
