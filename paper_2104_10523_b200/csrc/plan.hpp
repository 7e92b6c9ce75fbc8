// Plan object: network structure + contraction path + slicing (+ compiled device program).
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "builder.hpp"
#include "planner.hpp"

namespace tnqvm {
struct Program;   // compiled device program (program.hpp)
void program_free(Program*);
struct ProgramDeleter {
  void operator()(Program* p) const { program_free(p); }
};
}  // namespace tnqvm

struct tnqvm_plan {
  tnqvm_circuit circuit;              // private copy (values are re-read for every bitstring)
  tnqvm::Closure closure;             // open pattern (bits: -1 open, 0 elsewhere) or Pauli
  tnqvm::NetMode mode;
  tnqvm_dtype dtype;
  uint64_t budget_bytes = 0;
  tnqvm_plan_opts opts;
  tnqvm::Network net;                 // structure (+ values of the planning bitstring)
  std::string structure;              // canonical structure string
  std::string network_hash;           // sha256(structure)
  tnqvm::PathResult path;
  std::vector<int32_t> out_qubits;
  uint64_t rev_snapshot = 0;           // *circuit.rev_token when the plan was made
  std::unique_ptr<tnqvm::Program, tnqvm::ProgramDeleter> program;  // compiled lazily per device
  int program_device = -1;
};

namespace tnqvm {
// plan construction shared by tnqvm_plan_create and tnqvm_expectation
tnqvm_plan* make_plan(const tnqvm_circuit& c, const Closure& cl, uint64_t budget_bytes,
                      const tnqvm_plan_opts& opts);
std::string plan_json(const tnqvm_plan& p);
}  // namespace tnqvm
