// a8: fused small-tensor path (N4).
//
// "Small gate tensors are contracted internally to form larger tensors": the
// many tiny early (and late) pairwise contractions of a plan run inside ONE kernel, one
// CTA per independent subtree (or per slice / per expectation term of a batch), with
// the step list executed in order and a CTA barrier between steps.  Intermediates read
// only by later steps of the same task live in the CTA's shared-memory arena (placed by the
// program compiler, SmallStepDesc::smem); the others in L1/L2-resident scratch; the K-offset
// tables live in shared memory; complex
// accumulation in registers; per-step output bits are decoded with stride tables so any
// operand / output layout is read and written directly (no permutes on this path).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.hpp"
#include "kernels.hpp"
#include "pdl.cuh"

namespace tnqvm {
namespace dev {
namespace {

template <typename T> struct C2;
template <> struct C2<float> { using t = float2; };
template <> struct C2<double> { using t = double2; };

__device__ __forceinline__ uint64_t pext64(uint64_t x, uint64_t mask) {
  uint64_t r = 0;
  int o = 0;
  while (mask) {
    int b = __ffsll((long long)mask) - 1;
    r |= ((x >> b) & 1ULL) << o;
    ++o;
    mask &= mask - 1;
  }
  return r;
}

template <typename T, int NT>
__global__ void __launch_bounds__(NT) small_kernel(const SmallStepDesc* __restrict__ steps,
                                                    const SmallTask* __restrict__ tasks,
                                                    const LeafDesc* __restrict__ leaves,
                                                    const typename C2<T>::t* __restrict__ leafbuf,
                                                    typename C2<T>::t* __restrict__ arena,
                                                    double2* __restrict__ result,
                                                    const UnitDesc* __restrict__ units) {
  pdl_wait();
  pdl_trigger();
  using V = typename C2<T>::t;
  __shared__ int32_t tabA[1 << SMALL_MAXK];
  __shared__ int32_t tabB[1 << SMALL_MAXK];
  // the task's step descriptors are staged in shared memory kDescChunk at a time (one
  // cooperative burst instead of a chain of dependent global loads per step), and the
  // operand base pointers of the chunk are resolved in parallel (one thread per step)
  constexpr int kDescChunk = 12;
  __shared__ __align__(16) SmallStepDesc sd[kDescChunk];
  __shared__ const V* sA[kDescChunk];
  __shared__ const V* sB[kDescChunk];
  __shared__ V* sC[kDescChunk];
  __shared__ V red[256];
  extern __shared__ __align__(16) unsigned char small_dyn[];
  V* sarena = reinterpret_cast<V*>(small_dyn);  // task-internal tensors (generic pointers below)
  const SmallTask task = tasks[blockIdx.x];
  const UnitDesc unit = units[blockIdx.y];
  const uint64_t slice = task.slice + unit.slice;
  const int64_t lbase = task.leaf_base + unit.leaf_base;
  const V* last = nullptr;
  int last_n = 0;
  for (int s0 = task.begin; s0 < task.end; s0 += kDescChunk) {
    const int nsd = min(kDescChunk, task.end - s0);
    {
      const uint64_t* src = reinterpret_cast<const uint64_t*>(steps + s0);
      uint64_t* dst = reinterpret_cast<uint64_t*>(sd);
      const int nw = nsd * (int)(sizeof(SmallStepDesc) / 8);
      for (int w = threadIdx.x; w < nw; w += blockDim.x) dst[w] = src[w];
    }
    __syncthreads();
    if ((int)threadIdx.x < nsd) {
      const SmallStepDesc& d = sd[threadIdx.x];
      sA[threadIdx.x] = d.a_leaf >= 0
                            ? leafbuf + lbase + leaves[d.a_leaf].off +
                                  (int64_t)pext64(slice, leaves[d.a_leaf].mask) * leaves[d.a_leaf].subsize
                        : (d.smem & 1) ? sarena + d.a_off
                                       : arena + task.arena_base + d.a_off + (d.a_dep ? unit.dep_shift : unit.inv_shift);
      sB[threadIdx.x] = d.b_leaf >= 0
                            ? leafbuf + lbase + leaves[d.b_leaf].off +
                                  (int64_t)pext64(slice, leaves[d.b_leaf].mask) * leaves[d.b_leaf].subsize
                        : (d.smem & 2) ? sarena + d.b_off
                                       : arena + task.arena_base + d.b_off + (d.b_dep ? unit.dep_shift : unit.inv_shift);
      sC[threadIdx.x] = (d.smem & 4) ? sarena + d.c_off
                                     : arena + task.arena_base + d.c_off + (d.c_dep ? unit.dep_shift : unit.inv_shift);
    }
    __syncthreads();
  for (int si = 0; si < nsd; ++si) {
    const SmallStepDesc& d = sd[si];
    const V* A = sA[si];
    const V* B = sB[si];
    V* Cp = sC[si];
    const int nk = d.nk, nc = d.nc;
    const int K = 1 << nk;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
      int32_t oa = 0, ob = 0;
      for (int i = 0; i < nk; ++i)
        if ((k >> i) & 1) { oa += d.sa_k[i]; ob += d.sb_k[i]; }
      tabA[k] = oa;
      tabB[k] = ob;
    }
    __syncthreads();
    const int64_t NC = (int64_t)1 << nc;
    // G threads per output when the outputs cannot occupy the CTA (G, NC powers of two):
    // thread g of output j sums k = g, g + G, ... (two-level, 64-term blocks), then the G
    // partial sums are combined by a fixed tree (warp shuffles, then shared memory)
    const int G = NC >= (int64_t)blockDim.x ? 1 : min((int)(blockDim.x / NC), K);
    const int64_t nthr = NC * G;
    for (int64_t t = threadIdx.x; t < ((nthr + blockDim.x - 1) / blockDim.x) * blockDim.x; t += blockDim.x) {
      const bool act = t < nthr;
      const int64_t j = t / G;
      const int g = (int)(t % G);
      T re = 0, im = 0;
      if (act) {
        int64_t oa = 0, ob = 0;
        for (int i = 0; i < nc; ++i)
          if ((j >> i) & 1) { oa += d.sa_c[i]; ob += d.sb_c[i]; }
        for (int k0 = g; k0 < K; k0 += 64 * G) {
          T br = 0, bi = 0;
          const int k1 = min(K, k0 + 64 * G);
          for (int k = k0; k < k1; k += G) {
            V a = A[oa + tabA[k]];
            V b = B[ob + tabB[k]];
            br = fma(a.x, b.x, br);
            br = fma(-a.y, b.y, br);
            bi = fma(a.x, b.y, bi);
            bi = fma(a.y, b.x, bi);
          }
          re += br;
          im += bi;
        }
      }
      if (G > 1) {  // G <= blockDim and t's group never straddles an iteration (G | blockDim)
        const int gw = min(G, 32);
        for (int o = gw / 2; o > 0; o >>= 1) {
          re += __shfl_xor_sync(0xffffffffu, re, o);
          im += __shfl_xor_sync(0xffffffffu, im, o);
        }
        if (G > 32) {
          if ((threadIdx.x & 31) == 0) {
            red[threadIdx.x >> 5].x = re;
            red[threadIdx.x >> 5].y = im;
          }
          __syncthreads();
          if (act && g == 0) {
            re = 0;
            im = 0;
            const int w0 = (int)(threadIdx.x >> 5);
            for (int w = 0; w < G / 32; ++w) {
              re += red[w0 + w].x;
              im += red[w0 + w].y;
            }
          }
          __syncthreads();
        }
      }
      if (act && g == 0) {
        V c;
        c.x = re;
        c.y = im;
        Cp[j] = c;
      }
    }
    __syncthreads();
    last = Cp;
    last_n = (int)NC;
  }
  }
  if (task.result_slot >= 0 && last) {
    double2* r = result + (int64_t)(task.result_slot + unit.slot) * task.rlen;
    for (int j = threadIdx.x; j < last_n && j < task.rlen; j += blockDim.x) {
      V v = last[j];
      double vr = (double)v.x, vi = (double)v.y;
      r[j].x += task.scale_re * vr - task.scale_im * vi;
      r[j].y += task.scale_re * vi + task.scale_im * vr;
    }
  }
}

// One strided contraction step spread over the whole GPU (one output element per thread):
// used for steps too large for a single CTA but too skinny (K*M small) or too
// layout-constrained for the GEMM kernels.  Reads and writes any layout directly.
template <typename T>
__global__ void __launch_bounds__(256) strided_kernel(const SmallStepDesc* __restrict__ dp,
                                                      const LeafDesc* __restrict__ leaves,
                                                      const typename C2<T>::t* __restrict__ leafbuf,
                                                      typename C2<T>::t* __restrict__ arena,
                                                      const UnitDesc* __restrict__ units) {
  pdl_wait();
  pdl_trigger();
  using V = typename C2<T>::t;
  __shared__ int32_t tabA[1 << SMALL_MAXK];
  __shared__ int32_t tabB[1 << SMALL_MAXK];
  __shared__ __align__(16) SmallStepDesc d;
  for (int w = threadIdx.x; w < (int)(sizeof(SmallStepDesc) / 8); w += blockDim.x)
    reinterpret_cast<uint64_t*>(&d)[w] = reinterpret_cast<const uint64_t*>(dp)[w];
  __syncthreads();
  const UnitDesc unit = units[blockIdx.y];
  const uint64_t slice = unit.slice;
  const V* A = d.a_leaf >= 0 ? leafbuf + unit.leaf_base + leaves[d.a_leaf].off +
                                   (int64_t)pext64(slice, leaves[d.a_leaf].mask) * leaves[d.a_leaf].subsize
                             : arena + d.a_off + (d.a_dep ? unit.dep_shift : unit.inv_shift);
  const V* B = d.b_leaf >= 0 ? leafbuf + unit.leaf_base + leaves[d.b_leaf].off +
                                   (int64_t)pext64(slice, leaves[d.b_leaf].mask) * leaves[d.b_leaf].subsize
                             : arena + d.b_off + (d.b_dep ? unit.dep_shift : unit.inv_shift);
  V* Cp = arena + d.c_off + (d.c_dep ? unit.dep_shift : unit.inv_shift);
  const int K = 1 << d.nk;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    int32_t oa = 0, ob = 0;
    for (int i = 0; i < d.nk; ++i)
      if ((k >> i) & 1) { oa += d.sa_k[i]; ob += d.sb_k[i]; }
    tabA[k] = oa;
    tabB[k] = ob;
  }
  __syncthreads();
  const int64_t NC = (int64_t)1 << d.nc;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < NC; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t oa = 0, ob = 0;
    for (int i = 0; i < d.nc; ++i)
      if ((j >> i) & 1) { oa += d.sa_c[i]; ob += d.sb_c[i]; }
    T re = 0, im = 0;
    for (int k0 = 0; k0 < K; k0 += 64) {
      T br = 0, bi = 0;
      const int k1 = min(K, k0 + 64);
      for (int k = k0; k < k1; ++k) {
        V a = A[oa + tabA[k]];
        V b = B[ob + tabB[k]];
        br = fma(a.x, b.x, br);
        br = fma(-a.y, b.y, br);
        bi = fma(a.x, b.y, bi);
        bi = fma(a.y, b.x, bi);
      }
      re += br;
      im += bi;
    }
    V c;
    c.x = re;
    c.y = im;
    Cp[j] = c;
  }
}

}  // namespace

void launch_strided(int dtype, const SmallStepDesc* step, int nc, const LeafDesc* leaves, const void* leafbuf,
                    void* arena, const UnitDesc* units, int nb, cudaStream_t st) {
  const int nsm = sm_count();
  // a full wave over all units (each unit's outputs are independent: any grid)
  const int64_t want = std::max<int64_t>(1, (int64_t)nsm * 8 / std::max(1, nb));
  const int64_t blocks = std::min<int64_t>(((int64_t)1 << nc) / 256 + 1, want);
  const dim3 grid((unsigned)blocks, (unsigned)nb);
  if (dtype == 0)
    launch_pdl(strided_kernel<float>, grid, 256, 0, st, step, leaves, (const float2*)leafbuf, (float2*)arena, units);
  else
    launch_pdl(strided_kernel<double>, grid, 256, 0, st, step, leaves, (const double2*)leafbuf, (double2*)arena,
               units);
}

void launch_small(int dtype, const SmallStepDesc* steps, const SmallTask* tasks, int ntasks,
                  const LeafDesc* leaves, const void* leafbuf, void* arena, void* result,
                  const UnitDesc* units, int nb, cudaStream_t st, int threads, int64_t smem_elems) {
  if (ntasks <= 0 || nb <= 0) return;
  // threads per task CTA (256 | 512 | 1024): a task is one dependent chain of steps, so a
  // wider CTA shortens each step's serial loop over its outputs but pays more for every
  // CTA barrier.  Measured on B200: the amplitude programs' batches (C2, 2^13-2^16-MAC
  // tasks) gain 20% of their time at 512; the expectation batches (C4, many short tasks)
  // lose 0-7% above 256.
  const int nt = threads >= 1024 ? 1024 : threads >= 512 ? 512 : 256;
  const dim3 grid((unsigned)ntasks, (unsigned)nb);
  const size_t dyn = (size_t)smem_elems * (dtype == 0 ? 8 : 16);
  TNQVM_CHECK(dyn <= (size_t)SMALL_SMEM_BYTES, TNQVM_EINVAL, "small-task shared arena too large");
  if (dtype == 0) {
    auto k = nt == 1024 ? small_kernel<float, 1024> : nt == 512 ? small_kernel<float, 512> : small_kernel<float, 256>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMALL_SMEM_BYTES);
    launch_pdl(k, grid, nt, dyn, st, steps, tasks, leaves, (const float2*)leafbuf, (float2*)arena,
               (double2*)result, units);
  } else {
    auto k = nt == 1024 ? small_kernel<double, 1024> : nt == 512 ? small_kernel<double, 512> : small_kernel<double, 256>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMALL_SMEM_BYTES);
    launch_pdl(k, grid, nt, dyn, st, steps, tasks, leaves, (const double2*)leafbuf, (double2*)arena,
               (double2*)result, units);
  }
}

}  // namespace dev
}  // namespace tnqvm
