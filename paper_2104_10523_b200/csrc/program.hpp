// a5: compiled device program of a plan (layouts, kernel classes, arena offsets, launch list).
#pragma once

#include <cstdint>
#include <vector>

#include "kernels.hpp"
#include "plan.hpp"

namespace tnqvm {

enum OpKind : int { OP_SMALL = 0, OP_GEMM = 1, OP_SPLITK = 2, OP_PERMUTE = 3, OP_ACCUM = 4, OP_STRIDED = 5, OP_SKINNY = 6 };
enum StepClass : int { CLS_SMALL = 0, CLS_GEMM = 1, CLS_SPLITK = 2, CLS_STRIDED = 3, CLS_SKINNY = 4 };
enum GemmMethod : int { GM_SIMT = 0, GM_TC = 1, GM_DMMA = 2 };

struct Ten {
  int rank = 0;
  std::vector<int> layout;  // wire ids slowest -> fastest (sliced wires excluded)
  bool leaf = false;
  int leaf_index = -1;
  bool decided = false;
  bool dep = false;         // value depends on the slice id
  int64_t off = 0;          // arena offset (elements), intermediates only
  int64_t size() const { return (int64_t)1 << rank; }
};

struct Op {
  OpKind kind;
  bool dep;
  // OP_SMALL (task range); OP_STRIDED: task_begin = descriptor index in small_steps
  int task_begin = 0, task_end = 0;  // range in Program::tasks
  // OP_GEMM / OP_SPLITK / OP_PERMUTE / OP_ACCUM
  int x = -1, y = -1, c = -1;        // tensor ids (permute: x -> c; accum: x)
  int method = GM_SIMT;
  int nk = 0, nm = 0;
  int64_t N = 0;
  std::vector<int64_t> syk, sym;     // Y strides for k bits / m bits (LSB first)
  std::vector<int> perm;             // OP_PERMUTE
  int nn = 0;                        // OP_SKINNY / gather GEMM: bits of the streamed operand's free index
  int gather = 0;                    // OP_GEMM (TC): X gathered (not K-contiguous)
  std::vector<int> rd, wr;           // tensor ids read / written (runtime stream dependencies)
  std::vector<int64_t> sxn, scn, sxk, scm;  // OP_SKINNY strides (bit 0 = fastest)
  double flops = 0, bytes = 0;       // algorithmic cost of this op
};

struct Program {
  uint64_t uid = 0;   // unique per compiled program (cache keys)
  int dtype = 0;
  int esize = 8;
  std::vector<Ten> tens;                  // leaves first, then step outputs, then permute temps
  std::vector<std::vector<int>> leaf_full_layout;  // sliced wires (slice-digit order) + per-slice layout
  std::vector<dev::LeafDesc> leaves;      // device leaf placement
  int64_t leaf_elems = 0;
  std::vector<dev::SmallStepDesc> small_steps;
  std::vector<dev::SmallTask> tasks;
  int64_t small_smem_elems = 0;           // shared-memory arena of a small-task CTA (task-internal tensors)
  std::vector<Op> ops;                    // invariant ops first, then per-slice ops
  int64_t arena_elems = 0;                // inv_elems + dep_elems (one lane)
  int64_t inv_elems = 0, dep_elems = 0;   // slice-invariant pool, per-slice pool (per lane)
  int final_tensor = -1;                  // -1: the network is a bare scalar
  int64_t result_len = 1;
  bool final_dep = false;
  int n_sliced = 0;
  std::vector<int> sliced;                // wire ids
  double flops_per_slice = 0, bytes_per_slice = 0, flops_invariant = 0, bytes_invariant = 0;
  size_t scratch_bytes = 0;               // split-K partials (per unit)
  size_t wbuf_bytes = 0;                  // tensor-core W operand + partials (per unit)
  // device copies (owned; freed in program_free)
  void* d_small_steps = nullptr;
  void* d_tasks = nullptr;
  void* d_leaves = nullptr;
  int device = -1;
  // captured CUDA graphs of whole evaluations (runtime.cu), keyed by the context, its
  // device buffers and the unit set they were captured for; destroyed with the program
  struct Graph {
    std::vector<const void*> key;
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0, gemm_launches = 0;
    double gemm_bytes = 0, gemm_flops = 0;
  };
  std::vector<Graph> graphs;
};

// Build the program for plan p on a device (host work + small device uploads).
Program* compile_program(const tnqvm_plan& p, int device);

// Pack the leaves of network `net` (same structure as the plan) into the program's host
// leaf layout, cast to the device dtype (round to nearest).  out: leaf_elems * esize bytes.
void pack_leaves(const Program& prog, const Network& net, void* out);

}  // namespace tnqvm
