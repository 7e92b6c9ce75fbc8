/*
 * tnqvm.h -- C-ABI of libtnqvm: the B200-native sliced tensor-network
 * contraction path of arXiv:2104.10523 (TNQVM on ExaTN), §3.1 and §3.3.
 *
 * The calls follow the paper's statement of the problem:
 *   tnqvm_circuit_create / tnqvm_apply_gate   -- the circuit (§3.1)
 *   tnqvm_apply_kraus                         -- Kraus channels, Eq.(3)
 *   tnqvm_plan_create                         -- contraction sequence + index slicing
 *   tnqvm_amplitude                           -- <b|U|0>, Eq.(1); noisy: <b|rho|b>
 *   tnqvm_amplitudes                          -- marginal wave-function slice, -1 = open (§4.4)
 *   tnqvm_expectation                         -- sum_j c_j <P_j>, Eq.(2); noisy: Tr(H rho)
 *
 * Conventions:
 *   - qubit 0 is the most significant bit of a state index; bits[q] is qubit q;
 *   - a gate / Kraus matrix is row-major 2^k x 2^k in the basis |q[0] q[1]>, q[0] the MSB;
 *   - amplitudes() output index j has its MSB at the lowest-numbered open qubit;
 *     for a noisy circuit it is the 2^k x 2^k block rho[ket, bra], row-major, ket-major;
 *   - complex numbers cross the ABI as tnqvm_c128 (two doubles, re then im).
 *
 * Ownership: every input is copied at call time; the library never retains a
 * caller pointer.  Outputs go to caller-owned HOST buffers.  Handles are freed by
 * their *_destroy call.  A plan snapshots the circuit revision; using it after the
 * circuit changed returns TNQVM_ESTATE.  Calls on one ctx are serialised by the
 * caller; separate ctxs are independent.  Calls are host-synchronous (results are
 * in caller memory on return) and stream-ordered on the ctx's CUDA stream.
 * No C++ exception crosses this boundary.
 *
 * Errors: 0 = OK, negative = TNQVM_E*; tnqvm_last_error() returns a thread-local
 * message for the last failing call on this thread.
 *
 * Device work (the GPU path) never falls back to the CPU: a ctx on a machine
 * without a usable sm_100 device fails with TNQVM_ECUDA.
 */
#ifndef TNQVM_H
#define TNQVM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TNQVM_OK           0
#define TNQVM_EINVAL      -1  /* bad argument: qubit out of range/duplicated, k not in {1,2}, m<1,
                                 Pauli char not in IXYZ, bit not in {0,1,-1}, open pattern differs
                                 from the plan, amplitude() on a plan with open qubits, NULL pointer */
#define TNQVM_ENOTUNITARY -2  /* max|U^dagger U - I| > 1e-10 */
#define TNQVM_ENOTCPTP    -3  /* max|sum_k K^dagger K - I| > 1e-10 */
#define TNQVM_EINFEASIBLE -4  /* max_slice_bytes below what slicing every bond can reach */
#define TNQVM_ENOMEM      -5  /* host or device allocation failure */
#define TNQVM_ECUDA       -6  /* CUDA error / no usable device */
#define TNQVM_ENCCL       -7  /* NCCL error */
#define TNQVM_ESTATE      -8  /* stale plan (circuit changed) or wrong ctx/plan kind */

typedef struct tnqvm_ctx tnqvm_ctx;
typedef struct tnqvm_circuit tnqvm_circuit;
typedef struct tnqvm_plan tnqvm_plan;

typedef struct { double re, im; } tnqvm_c128;

typedef enum { TNQVM_C64 = 0, TNQVM_C128 = 1 } tnqvm_dtype;

/* One operator string term c * prod_i P_{qubits[i]}: Pauli 'I','X','Y','Z' (Eq.(2)),
 * or the projectors '0' = |0><0| and '1' = |1><1| (marginal probabilities for bit-string
 * sampling, Table 1 "direct unbiased bit-string sampling"). */
typedef struct {
  double coeff;
  int32_t nops;
  const int32_t* qubits;
  const char* paulis;
} tnqvm_pauli_term;

/* Planner options; tnqvm_plan_opts_default() fills the defaults. */
typedef struct {
  uint64_t seed;              /* planner RNG seed (deterministic per seed)                       */
  int32_t restarts;           /* greedy + random restarts ("heuristics"); default 64      */
  int32_t threads;            /* host threads for restarts (result independent of this); 0=auto */
  double time_cap_s;          /* stop starting new restarts after this wall time; <=0: no cap    */
  tnqvm_dtype dtype;          /* device precision                                               */
  int32_t cancel_conjugates;  /* expectation: drop U U^dagger pairs outside the light cone */
  uint64_t min_slices;        /* slice at least this many ways (multi-GPU balance)               */
  int32_t cost_model;         /* planner objective: 0 = multiply-add count (the paper's flop count,
                                 P:L134); 1 = B200 time model, per step max(MACs, beta x elements
                                 moved for tensors > 2^21 elements) (R18). Default 1. */
  int32_t partition;          /* 1: every other restart builds its tree by recursive balanced min-cut
                                 bisection of the network (the paper's graph-partitioning search,
                                 P:L134) in addition to the greedy restarts; all refined alike.
                                 Default 1. */
} tnqvm_plan_opts;

/* Summary numbers of a plan (exact integers as decimal strings live in the JSON). */
typedef struct {
  int32_t n_leaves, n_steps, n_wires, n_open, n_sliced;
  uint64_t n_slices;
  double log2_macs_unsliced;   /* complex multiply-adds, all slices */
  double log2_macs_sliced;
  double log2_max_intermediate;
  double flops_sliced;         /* 8 real flops per complex MAC x sliced MACs */
  double bytes_sliced;         /* algorithmic bytes sum sizeof*(|A|+|B|+|C|) over steps x slices */
  int32_t noisy;               /* 1: doubled network (Kraus) */
  int32_t dtype;
} tnqvm_plan_info;

/* Per-call device statistics of the last evaluation on a ctx. */
typedef struct {
  double ms_total;             /* device time of the slice loop + reduction (CUDA events) */
  double ms_gemm;              /* summed device time of the dominant contraction kernel class */
  int64_t gemm_launches;
  int64_t kernel_launches;     /* all kernels launched by the library during the call */
  double gemm_bytes;           /* algorithmic bytes of the timed GEMM launches */
  double gemm_flops;           /* useful real flops of the timed GEMM launches */
  double flops;                /* algorithmic real flops of the call */
  double bytes;                /* algorithmic bytes of the call */
  uint64_t h2d_bytes, d2h_bytes;
  double host_ms;              /* host time from the call's entry to the end of enqueueing */
  int32_t graph;               /* 1: the evaluation was replayed from a captured CUDA graph */
  int32_t pad_;
} tnqvm_stats;

int tnqvm_version(void);
const char* tnqvm_last_error(void);
void tnqvm_plan_opts_default(tnqvm_plan_opts* opts);

/* ---- circuits (host only) ------------------------------------------------ */
int tnqvm_circuit_create(int32_t nq, tnqvm_circuit** out);             /* state |0...0> */
void tnqvm_circuit_destroy(tnqvm_circuit* c);
/* U: 2^k x 2^k row-major; qubits: k distinct indices; k in {1,2}. */
int tnqvm_apply_gate(tnqvm_circuit* c, const tnqvm_c128* U, const int32_t* qubits, int32_t k);
/* K: m consecutive 2^k x 2^k row-major Kraus operators with sum_k K^dagger K = I. */
int tnqvm_apply_kraus(tnqvm_circuit* c, const tnqvm_c128* K, int32_t m, const int32_t* qubits, int32_t k);

/* ---- plans (host only) --------------------------------------------------- */
/* Builds the network (absorbing 1-qubit gates and boundary vectors in complex128),
 * searches a pairwise contraction sequence and slices bonds until every
 * intermediate fits max_slice_bytes.  out_qubits (n_out of them,
 * strictly increasing) stay open; amplitudes() then needs bits[q] == -1 exactly at
 * them.  For a noisy circuit the network is the doubled (ket/bra) network with
 * Kraus tensors.  opts may be NULL (defaults).  Host-only: needs no GPU. */
int tnqvm_plan_create(const tnqvm_circuit* c, const int32_t* out_qubits, int32_t n_out,
                      uint64_t max_slice_bytes, const tnqvm_plan_opts* opts, tnqvm_plan** out);
/* Canonical plan JSON (sorted keys, integers and strings only): byte-identical for the
 * same (op-list structure, out_qubits, budget, opts) on any machine / thread count. */
int tnqvm_plan_json(const tnqvm_plan* p, char* buf, size_t cap, size_t* len);
int tnqvm_plan_get_info(const tnqvm_plan* p, tnqvm_plan_info* info);
/* Builder inspection hook (host only): the network handed to the planner, with leaf
 * values for bitstring `bits` (NULL: the planning values), as JSON
 * {"scalar":[re,im],"open":[wire ids],"leaves":[{"wires":[...],"data":[re,im,...]}]};
 * leaf data row-major with the first listed wire slowest. */
int tnqvm_network_export(const tnqvm_plan* p, const int8_t* bits, char* buf, size_t cap, size_t* len);
/* Slice ids owned by `rank` of `world` (8 fixed contiguous groups, group g -> rank g % world;
 * SURVEY §8(e)); writes up to cap ids into out and the total count into *n.  Host only. */
int tnqvm_plan_rank_slices(const tnqvm_plan* p, int rank, int world, uint64_t* out, uint64_t cap, uint64_t* n);
/* Kernel classes of the plan's launch list (host only: compiles the device program
 * without uploading it): counts[c] = ops of class c (TNQVM_K_*, TNQVM_K_NCLASS entries). */
int tnqvm_plan_kernel_classes(const tnqvm_plan* p, int64_t* counts);
/* Inspection hook (host only): the compiled launch list as JSON {"ops":[{"class","dep","x",
 * "y","c","N","nk","nm","gather","bytes","flops"}],"tensors":[{"rank","leaf","dep","layout"}],
 * "inv_elems","dep_elems","leaf_elems"} (layout: wire ids slowest first; ops in launch order). */
int tnqvm_plan_program_json(const tnqvm_plan* p, char* buf, size_t cap, size_t* len);
void tnqvm_plan_destroy(tnqvm_plan* p);
/* Planner test hook (host only): plan an abstract network of binary wires.  Leaf i has
 * leaf_ranks[i] wire ids taken consecutively from leaf_wires; `open` lists open wires;
 * budget in elements.  Writes {"macs_sliced","macs_unsliced","log2_max","sliced","steps"}
 * as JSON into buf (same conventions as tnqvm_plan_json). */
int tnqvm_plan_raw_network(const int32_t* leaf_ranks, const int32_t* leaf_wires, int32_t nleaves,
                           const int32_t* open, int32_t nopen, uint64_t budget_elems,
                           const tnqvm_plan_opts* opts, char* buf, size_t cap, size_t* len);

/* ---- device context ------------------------------------------------------ */
/* rank/world: this process's share of the slice groups; world>1 takes
 * nccl_id (128 bytes from tnqvm_nccl_unique_id on rank 0, broadcast by the caller) and
 * sums the group slots over the ranks with one ncclAllReduce per call.  world>1 with
 * nccl_id == NULL is an EMULATED rank: it evaluates only its own groups and skips the
 * collective (tnqvm_ctx_group_slots then returns its partial slots) -- the multi-rank
 * partition can be checked on one GPU.
 * cuda_stream: the cudaStream_t all work is ordered on; NULL = the legacy default stream.  alloc/free_: optional
 * device allocator callbacks (e.g. the torch caching allocator) or NULL (cudaMalloc). */
int tnqvm_ctx_create(int device, int rank, int world, const void* nccl_id, void* cuda_stream,
                     void* (*alloc)(size_t bytes, void* ud), void (*free_)(void* ptr, void* ud),
                     void* alloc_ud, tnqvm_ctx** out);
void tnqvm_ctx_destroy(tnqvm_ctx* ctx);
int tnqvm_nccl_unique_id(void* out128);
int tnqvm_ctx_last_stats(const tnqvm_ctx* ctx, tnqvm_stats* out);
/* Instrumentation switch: 1 = record CUDA events around every launched op, summed per
 * kernel class (tnqvm_ctx_class_stats; tnqvm_stats.ms_gemm = the GEMM + skinny classes).
 * A timed evaluation runs its slices on one stream so that classes do not overlap. */
int tnqvm_ctx_set_timing(tnqvm_ctx* ctx, int on);

/* Kernel classes of the launch list. */
enum {
  TNQVM_K_SMALL = 0,   /* fused small-step batch, one CTA per task (a8) */
  TNQVM_K_STRIDED,     /* one whole-GPU strided step */
  TNQVM_K_SKINNY,      /* streaming skinny step, any layout */
  TNQVM_K_GEMM_TC,     /* complex64 3xTF32 tcgen05 GEMM (+ W prep) (a7) */
  TNQVM_K_GEMM_DMMA,   /* complex128 FP64 DMMA GEMM (+ W prep) */
  TNQVM_K_GEMM_SIMT,   /* SIMT GEMM */
  TNQVM_K_SPLITK,      /* split-K for tiny outputs (partials + fp64 final) */
  TNQVM_K_PERMUTE,     /* index permute (a6) */
  TNQVM_K_ACCUM,       /* slice accumulation into the complex128 group slot */
  TNQVM_K_NCLASS
};
typedef struct {
  double ms;           /* summed CUDA-event time of the class's ops in the last timed call */
  double bytes;        /* algorithmic bytes of those ops (sizeof * (|A| + |B| + |C|)) */
  double flops;        /* useful real flops (8 per complex MAC) */
  int64_t launches;    /* ops of the class (an op may be 1-2 kernels) */
  double roof_ms;      /* sum over the ops of max(bytes / HBM peak, flops / compute peak) */
  double roof_hbm_ms;  /* the part of roof_ms spent by ops whose bound is HBM */
} tnqvm_class_stats;
/* Per-class statistics of the last evaluation made with timing on.  cls < TNQVM_K_NCLASS. */
int tnqvm_ctx_class_stats(const tnqvm_ctx* ctx, int cls, tnqvm_class_stats* out);
/* Peaks the per-op roofline times of tnqvm_class_stats use: HBM GB/s, complex64 useful
 * TFLOP/s (3xTF32: TF32 peak / 3) and complex128 TFLOP/s (FP64).  Defaults: 6551, 268, 45. */
int tnqvm_ctx_set_roofline(tnqvm_ctx* ctx, double hbm_gbs, double c64_tflops, double c128_tflops);

/* ---- evaluation (device) ------------------------------------------------- */
/* bits: nq entries in {0,1}.  Pure: <b|U|0>.  Noisy: <b|rho|b> (imag ~ 0). */
int tnqvm_amplitude(tnqvm_ctx* ctx, tnqvm_plan* p, const int8_t* bits, tnqvm_c128* out);
/* Plan selection by measured cost (NEXT-1; the planner's objective ranks candidate plans
 * poorly): plans the amplitude network of c (no open qubits) once per seed in
 * seeds[0..n_seeds) with the other options of opts (NULL: defaults), evaluates each on this
 * context's GPU with tnqvm_amplitude_batch over the nb x nq row-major bitstrings (one warm-up
 * call, then reps timed calls; device time = the calls' CUDA-event span) and returns the
 * fastest plan in *best (caller-owned; tnqvm_plan_destroy).  ms_out (NULL or n_seeds
 * entries) receives each candidate's best call time in ms.  The other candidates are freed.
 * Errors: EINVAL (NULL, n_seeds / nb / reps < 1, a bad bitstring, a multi-rank context --
 * tune on one GPU and share the seed), plus those of planning and evaluation. */
int tnqvm_plan_autotune(tnqvm_ctx* ctx, const tnqvm_circuit* c, uint64_t max_slice_bytes, const tnqvm_plan_opts* opts,
                        const uint64_t* seeds, int32_t n_seeds, const int8_t* bits, int32_t nb, int32_t reps,
                        tnqvm_plan** best, double* ms_out);
/* Many bitstrings of one plan without open qubits (the "many amplitudes of one circuit"
 * use of Eq.(1)): bits is nb x nq row-major (row i = bitstring i, each
 * entry 0|1), out receives nb values (caller-owned, host).  The same values as nb
 * tnqvm_amplitude calls; the host preparation of bitstring i overlaps the device work of
 * bitstring i - 1.  nb = 0 is a no-op.  Errors: EINVAL (NULL, nb < 0, a bad entry in any
 * row -- nothing is evaluated then, open qubits in the plan), plus those of
 * tnqvm_amplitude.  Stats of the call: ms_total spans the whole batch on the device. */
int tnqvm_amplitude_batch(tnqvm_ctx* ctx, tnqvm_plan* p, const int8_t* bits, int32_t nb, tnqvm_c128* out);
/* bits: -1 exactly at the plan's out_qubits.  out: 2^k (pure) or 4^k (noisy block). */
int tnqvm_amplitudes(tnqvm_ctx* ctx, tnqvm_plan* p, const int8_t* bits, tnqvm_c128* out);
/* Sum_j c_j <P_j> (pure) or Tr(H rho) (noisy) via the bra-ket network of each term
 * (Eq.(2), Table 1 "expectation value by conjugate").  out_per_term (nterms) may be NULL. */
int tnqvm_expectation(tnqvm_ctx* ctx, const tnqvm_circuit* c, const tnqvm_pauli_term* terms,
                      int32_t nterms, uint64_t max_slice_bytes, const tnqvm_plan_opts* opts,
                      tnqvm_c128* out_total, tnqvm_c128* out_per_term);
/* Expectation value by wave-function slicing (Table 1 "expectation value by state vector
 * slicing"; the five-step workflow of P:L190-199).  rank_max open qubits O are kept
 * (every qubit a term acts on with X or Y -- more than rank_max of them is EINVAL -- then the
 * lowest-numbered others); the other nq - |O| qubits are projected to each of their
 * 2^(nq - |O|) bitstrings p (8 fixed contiguous groups of p; group g on rank g % world).
 * For each p the partial state vector psi_p over O is contracted (max_slice_bytes budget,
 * opts) and the partial expectation <psi_p|P_j|psi_p> computed on the device; Z factors on
 * projected qubits enter as (-1)^{p_q}.  Results: sum_j c_j <P_j> and the per-term values
 * (out_per_term may be NULL).  Pure circuits only (a Kraus op: EINVAL); terms use IXYZ. */
int tnqvm_expectation_wfslice(tnqvm_ctx* ctx, const tnqvm_circuit* c, const tnqvm_pauli_term* terms,
                              int32_t nterms, int32_t rank_max, uint64_t max_slice_bytes,
                              const tnqvm_plan_opts* opts, tnqvm_c128* out_total, tnqvm_c128* out_per_term);
/* Direct unbiased bit-string sampling (Table 1): nshots bitstrings of the circuit's
 * output distribution (|<b|U|0>|^2, or <b|rho|b> for a noisy circuit).  Qubits are sampled
 * in the order 0..nq-1, `block` (1..8) at a time; the probability of each extension of a
 * shot's sampled prefix is a marginal -- the bra-ket network closed with projectors
 * |b_q><b_q| on the sampled qubits and the identity (trace) on the rest, contracted like an
 * expectation term (light-cone cancellation applies).  uniforms: nshots caller-drawn values
 * in [0, 1), one per shot (the method's randomness is an input).  Decision: the lexicographic
 * inverse CDF (qubit 0 most significant) -- take the first extension a whose cumulative mass
 * m + P(prefix a) exceeds u.  out_bits: nshots x nq (row-major, 0/1); out_probs (nshots, may
 * be NULL): the probability of each sampled bitstring. */
int tnqvm_sample(tnqvm_ctx* ctx, const tnqvm_circuit* c, const double* uniforms, int32_t nshots, int32_t block,
                 uint64_t max_slice_bytes, const tnqvm_plan_opts* opts, int8_t* out_bits, double* out_probs);
/* Parity hook: value of each listed slice (ids in [0, n_slices)) for bitstring bits
 * (out_per_slice: n x 2^k).  rank/world of the ctx play no part. */
int tnqvm_eval_slices(tnqvm_ctx* ctx, tnqvm_plan* p, const int8_t* bits, const uint64_t* slice_ids,
                      int32_t n, tnqvm_c128* out_per_slice);
/* The 8 x 2^k complex128 group slots of the last amplitude / amplitudes call on this ctx
 * (group g's partial sum in slot g, after the cross-rank reduction; an
 * emulated rank -- world > 1 without a communicator -- holds only its own groups' slots,
 * zeros elsewhere).  Writes min(cap, *n) values into out (host), the total count into *n.
 * The host sums the slots in group order to form the result. */
int tnqvm_ctx_group_slots(const tnqvm_ctx* ctx, tnqvm_c128* out, int64_t cap, int64_t* n);

/* ---- kernel-level entry points (benchmarks / parity of single kernels) --- */
/* These two are stream-ordered and return without host synchronisation: inputs and
 * outputs are device buffers on the ctx stream (the caller synchronises before reading). */
/* N1: out[perm-layout] = in; in is a rank-r binary-mode complex tensor (dtype) in device
 * memory; perm[i] = input mode that becomes output mode i (modes numbered slowest-first). */
int tnqvm_permute_device(tnqvm_ctx* ctx, int dtype, const void* in, void* out, int32_t rank,
                         const int32_t* perm);
/* N2/N3: C[n][m] = sum_k X[n][k] * Y[k][m] (row-major complex, device memory);
 * method: 0 = auto, 1 = SIMT FMA, 2 = tensor core (c64: 3xTF32 tcgen05; c128: DMMA),
 * 3 = strided split-K (N, M powers of two <= 64; K >= 2; ctx workspace).  Other methods: EINVAL. */
int tnqvm_gemm_device(tnqvm_ctx* ctx, int dtype, int method, const void* X, const void* Y, void* C,
                      int64_t N, int64_t K, int64_t M);
/* N2 with X in any binary-mode layout (the program's "gather" steps: X's fastest mode is
 * contracted but its other contracted modes are not): X element (n, k) at
 * sum_i bit_i(n) sxn[i] + sum_i bit_i(k) sxk[i] complex elements (bit 0 = least significant),
 * N = 2^nn, K = 2^nk, M = 2^nm; Y row-major K x M, C row-major N x M (device memory).
 * dtype 0 (complex64) runs the tcgen05 kernel's gather producer and requires sxk[0] == 1;
 * EINVAL otherwise or for nn > 40, nk > 20, nm > 16. */
int tnqvm_gemm_gather_device(tnqvm_ctx* ctx, int dtype, const void* X, const void* Y, void* C, int32_t nn,
                             int32_t nk, int32_t nm, const int64_t* sxn, const int64_t* sxk);

#ifdef __cplusplus
}
#endif
#endif /* TNQVM_H */
