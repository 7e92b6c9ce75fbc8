// a3/a4: contraction-order planner (greedy + random restarts) and index slicer.
#pragma once

#include <array>
#include <string>
#include <vector>

#include "builder.hpp"

namespace tnqvm {

struct PlanOpts {
  uint64_t seed = 0;
  int restarts = 64;
  int threads = 0;
  double time_cap_s = 0.0;
  uint64_t min_slices = 1;
  int reconf_k = 8;        // subtree reconfiguration frontier size (0 = off)
  int reconf_passes = 4;
  int reconf_k2 = 11;      // deeper reconfiguration of the best `refine_top` restarts
  int refine_top = 4;
  // objective: 0 = multiply-add count (the paper's flop count); 1 = B200 time model
  // per step max(MACs, beta * elements moved), counting only tensors above 2^21 elements
  // (smaller ones stay in the 126 MB L2 between producer and consumer); beta = complex
  // MACs per HBM element at the ridge (reading R18)
  int cost_model = 0;
  int beta = 24;
  int partition = 0;       // 1: odd restarts build recursive-bisection trees (NEXT-1)
};

// per-step cost under a cost model: nu = log2 MACs, na / nb / nc = log2 sizes of A, B, C
inline u128 step_cost(int model, int beta, int nu, int na, int nb, int nc) {
  const u128 macs = (u128)1 << nu;
  if (model == 0) return macs;
  auto mem = [](int n) -> u128 { return n > 21 ? ((u128)1 << n) : 0; };
  const u128 m = (u128)beta * (mem(na) + mem(nb) + mem(nc));
  return m > macs ? m : macs;
}

struct PathResult {
  std::vector<std::array<int, 2>> steps;  // SSA: leaves 0..L-1, step s creates id L+s
  std::vector<int> sliced;                // wire ids, first = most significant slice digit
  u128 macs_unsliced = 0;                 // sum_steps 2^|A u B|
  u128 macs_sliced = 0;                   // with slicing, over all slices (invariant steps once)
  int log2_max_unsliced = 0;              // largest intermediate (elements)
  int log2_max_sliced = 0;
  int restart = -1;                       // winning restart index
  u128 model_cost = 0;                    // objective value of the winner (= macs_sliced for model 0)
};

// Wire sets of the leaves + open wires; budget in elements (max entries of one intermediate).
PathResult plan_network(const Network& net, uint64_t budget_elems, const PlanOpts& opts);

// Sliced cost of a fixed path for a given sliced set (exact).
u128 sliced_macs(const std::vector<std::vector<int>>& leaves, int nwires,
                 const std::vector<std::array<int, 2>>& steps, const std::vector<int>& sliced,
                 int* log2_max);

std::string sha256_hex(const std::string& s);

}  // namespace tnqvm
