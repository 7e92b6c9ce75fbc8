// NEXT-2: partial expectation values of wave-function slices (Table 1 "expectation value
// by state vector slicing"; workflow steps 4-5).
//
// For each region r (one projected bitstring p of the sliced-out qubits) the evaluation
// left the group slots of the partial state vector psi_p over the open qubits; here
//   psi[x]  = sum_g slots[r][g][x]                 (group order: the amplitude finalisation)
//   v[r][j] = sum_x conj(psi[x]) (-1)^{popc(x & zy_j)} psi[x ^ flip_j]
// so that <psi_p| P_j |psi_p> = (-i)^{nY_j} v[r][j] (Y = -i (-1)^{x_q} on the flipped bit,
// Z = (-1)^{x_q}).  One CTA per (term, region); each thread sums its x's in complex128, then a
// fixed-shape tree -- deterministic.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"
#include "pdl.cuh"

namespace tnqvm {
namespace dev {
namespace {

constexpr int kWfThr = 256;

__device__ __forceinline__ double2 psi_at(const double2* __restrict__ s, int64_t rlen, int64_t x) {
  double2 a = s[x];
  for (int g = 1; g < 8; ++g) {
    const double2 b = s[(int64_t)g * rlen + x];
    a.x += b.x;
    a.y += b.y;
  }
  return a;
}

__global__ void __launch_bounds__(kWfThr) wf_partial_kernel(const double2* __restrict__ slots, int64_t rlen,
                                                             const WfTerm* __restrict__ terms, int nterms,
                                                             double2* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.x, r = blockIdx.y;
  const WfTerm t = terms[j];
  const double2* s = slots + (int64_t)r * 8 * rlen;
  double re = 0, im = 0;
  for (int64_t x = threadIdx.x; x < rlen; x += kWfThr) {
    const double2 a = psi_at(s, rlen, x);
    const double2 b = psi_at(s, rlen, x ^ (int64_t)t.flip);
    const double sg = (__popcll((unsigned long long)(x & (int64_t)t.zy)) & 1) ? -1.0 : 1.0;
    // conj(a) * b
    re += sg * (a.x * b.x + a.y * b.y);
    im += sg * (a.x * b.y - a.y * b.x);
  }
  __shared__ double sr[kWfThr], si[kWfThr];
  sr[threadIdx.x] = re;
  si[threadIdx.x] = im;
  __syncthreads();
  for (int w = kWfThr / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      sr[threadIdx.x] += sr[threadIdx.x + w];
      si[threadIdx.x] += si[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[(int64_t)r * nterms + j] = make_double2(sr[0], si[0]);
}

}  // namespace

void launch_wf_partial(const void* slots, int64_t rlen, int nregions, const WfTerm* terms, int nterms, void* out,
                       cudaStream_t st) {
  if (nterms <= 0 || nregions <= 0) return;
  launch_pdl(wf_partial_kernel, dim3((unsigned)nterms, (unsigned)nregions), kWfThr, 0, st,
             (const double2*)slots, rlen, terms, nterms, (double2*)out);
}

}  // namespace dev
}  // namespace tnqvm
