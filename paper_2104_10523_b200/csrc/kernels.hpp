// Host-callable launchers of the sm_100a kernels (implemented in k_*.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tnqvm {
namespace dev {

constexpr int SMALL_MAXC = 16;  // output bits of a fused small step
constexpr int SMALL_MAXK = 12;  // contracted bits of a fused small step (K table in shared memory)

// a8: one pairwise contraction inside the fused small-tensor path.
// C[j] = sum_k A[offA(j) + tabAk[k]] * B[offB(j) + tabBk[k]],
// offA(j) = sum_i bit_i(j) * sa_c[i] (bit 0 = fastest axis of C), likewise for B and k.
struct SmallStepDesc {
  int32_t a_leaf, b_leaf;       // leaf index, or -1 = arena tensor
  int64_t a_off, b_off, c_off;  // element offsets into the arena (ignored for leaves)
  int32_t nc, nk;               // log2 |C|, log2 |K|
  int8_t a_dep, b_dep, c_dep, pad_;  // arena operand is per-slice: add the lane's dep_base
  int64_t sa_c[32], sb_c[32];  // up to 32 output bits (strided steps); small steps use <= SMALL_MAXC
  int32_t sa_k[SMALL_MAXK], sb_k[SMALL_MAXK];
};

// Leaf placement: leaf buffer offset of slice s = off + pext(s, mask) * subsize.
struct LeafDesc {
  int64_t off;
  int64_t subsize;
  uint64_t mask;
};

// One CTA runs steps [begin, end) in order; `unit` selects the slice / term of a batch.
struct SmallTask {
  int32_t begin, end;
  int64_t arena_base;   // added to every arena offset of this task (per-unit scratch)
  uint64_t slice;       // slice id used for leaf offsets
  int64_t leaf_base;    // added to every leaf offset (per-unit leaf set)
  int32_t result_slot;  // >= 0: accumulate C of the last step into result[slot * rlen ...]
  int32_t rlen;
  double scale_re, scale_im;
};

// dep_base: element offset added to per-slice (x_dep) arena operands -- the runtime lane's pool.
// threads: CTA width per task (256, 512 or 1024).
void launch_small(int dtype, const SmallStepDesc* steps, const SmallTask* tasks, int ntasks,
                  const LeafDesc* leaves, const void* leafbuf, void* arena, void* result,
                  uint64_t slice, cudaStream_t st, int64_t dep_base, int threads = 256);

// One contraction step over the whole GPU, any operand/output layout (descriptor in
// device memory; nc = log2 |C| <= 32, nk <= SMALL_MAXK).
void launch_strided(int dtype, const SmallStepDesc* step, int nc, const LeafDesc* leaves, const void* leafbuf,
                    void* arena, uint64_t slice, cudaStream_t st, int64_t dep_base);

// Skinny step (K*M <= 512, M <= 32, K <= 64): C(n, m) = sum_k X(n, k) Y(k, m) with X, Y, C in ANY layout
// (bit strides per index bit; bit 0 = fastest).  One thread per n, all M outputs in
// registers, Y staged in shared memory -- streams X at HBM rate without a permute.
struct SkinnyDesc {
  const void* X;
  const void* Y;
  void* C;
  int nn, nk, nm;
  int64_t sxn[40], scn[40];
  int64_t sxk[6], syk[6], sym[6], scm[6];
};
void launch_skinny(int dtype, const SkinnyDesc& d, cudaStream_t st);

// a7 (SIMT path): C[n][m] = sum_k X[n][k] * Y(k, m); X row-major N x K (K contiguous),
// Y gathered with bit strides (k bit i -> syk[i], m bit i -> sym[i]); C row-major N x M.
struct GemmDesc {
  const void* X;
  const void* Y;
  void* C;
  int64_t N;
  int32_t nk, nm;  // K = 2^nk, M = 2^nm
  int64_t syk[40];
  int64_t sym[40];
  // tensor-core gather mode (X not K-contiguous; its fastest mode is contracted): X element
  // (n, k) at sum_bits(n) sxn + sum_bits(k) sxk, complex units, k bit 0 stride 1
  int32_t gather, nn;
  int64_t sxn[40];
  int64_t sxk[40];
};
void launch_gemm_simt(int dtype, const GemmDesc& g, cudaStream_t st);
// split-K for tiny outputs: C[n][m] = sum_k X[n][k] Y[m][k] with both K-contiguous
// (Y row-major M x K), deterministic two-pass reduction in `scratch` (>= 2*chunks*N*M reals of dtype... see impl)
size_t splitk_scratch_bytes(int dtype, int64_t N, int64_t M, int64_t K);
void launch_splitk(int dtype, const void* X, const void* Y, void* C, int64_t N, int64_t M, int64_t K,
                   void* scratch, cudaStream_t st);

// split-K with both operands in ANY layout (N, M <= 64): C(n, m) = sum_k X(n, k) Y(m, k),
// element offsets = sums of per-bit strides (bit 0 = fastest; k bits in X's order, fastest
// first).  Two launches (persistent partials + fp64 final), `scratch` >= splitk_strided_scratch_bytes.
struct StridedSplitK {
  const void* X;
  const void* Y;
  void* C;
  int nn, nk, nm;
  int64_t sxn[6], scn[6], sym[6], scm[6];
  int64_t sxk[64], syk[64];
};
bool splitk_strided_supported(int nn, int nk, int nm);
size_t splitk_strided_scratch_bytes(int nn, int nm);
void launch_splitk_strided(int dtype, const StridedSplitK& s, void* scratch, cudaStream_t st);

// a7 (tensor-core path, complex64 via 3xTF32 tcgen05): same contract as launch_gemm_simt.
// W (the small operand expanded to real block form, hi/lo split) is built by a prep kernel
// into `wbuf` (tc_wbuf_bytes).  Returns false if the shape is unsupported.
size_t tc_wbuf_bytes(int64_t N, int nk, int nm);  // W^T hi/lo + split-K partials
bool tc_supported(int nk, int nm);
void launch_gemm_tc(const GemmDesc& g, void* wbuf, cudaStream_t st);
// number of slice lanes the caller keeps in flight on this thread (caps the GEMM grid)
void tc_set_concurrency(int lanes);
// Split-K steps with a tiny output and two large operands (C3's last contraction): both
// X [N][K] and Y [M][K] (K fastest, one K order) streamed by TMA; the converter warps build
// the W^T hi/lo tiles from Y on chip.  `part` holds the split-K partials (tc_ystream_part_bytes).
bool tc_ystream_supported(int64_t N, int nk, int nm);
size_t tc_ystream_part_bytes(int64_t N, int nk, int nm);
void launch_gemm_tc_ystream(const void* X, const void* Y, void* C, int64_t N, int nk, int nm, void* part,
                            cudaStream_t st);
// complex128 via FP64 DMMA (mma.sync m8n8k4), same contract.
bool dmma_supported(int nk, int nm);
size_t dmma_wbuf_bytes(int64_t N, int nk, int nm);  // W + split-K partials
void launch_gemm_dmma(const GemmDesc& g, void* wbuf, cudaStream_t st);

// a6: index permute of a rank-r binary-mode tensor: out mode i <- in mode perm[i]
// (modes numbered slowest-first).
void launch_permute(int dtype, const void* in, void* out, int rank, const int* perm, cudaStream_t st);

// accumulate: dst[j] (complex128) += scale * src[j] for j < n (src in dtype)
void launch_accum(int dtype, const void* src, void* dst, int64_t n, double sre, double sim, cudaStream_t st);

}  // namespace dev
}  // namespace tnqvm
