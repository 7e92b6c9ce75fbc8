// a2: circuit -> tensor network builder (host, complex128).
#pragma once

#include <string>
#include <vector>

#include "common.hpp"

namespace tnqvm {

enum NetMode : int {
  NET_KET = 0,          // <b|U|0> with open legs (Eq.(1), §4.4)
  NET_PURE_DOUBLED = 1, // ket copy U, bra copy U*, Pauli closure (Eq.(2), Fig. exp_val_double_depth)
  NET_SUPEROP = 2,      // merged ket/bra superoperator nodes sum_k K (x) K* (Eq.(3))
};

enum ClosureKind : int { CLOSE_PROJECT = 0, CLOSE_PAULI = 1 };

struct Closure {
  ClosureKind kind = CLOSE_PROJECT;
  std::vector<int8_t> bits;   // CLOSE_PROJECT: per qubit 0/1/-1 (open)
  std::vector<char> pauli;    // CLOSE_PAULI: per qubit 'I','X','Y','Z'
  bool cancel = true;         // CLOSE_PAULI: light-cone cancellation of U U^dagger pairs
};

struct WireRec {
  int side;     // 0 = ket, 1 = bra
  int qubit;
  int segment;  // number of 2-qubit ops on `qubit` (in the op list used) preceding the wire
  bool operator<(const WireRec& o) const {
    if (side != o.side) return side < o.side;
    if (qubit != o.qubit) return qubit < o.qubit;
    return segment < o.segment;
  }
  bool operator==(const WireRec& o) const {
    return side == o.side && qubit == o.qubit && segment == o.segment;
  }
};

struct Leaf {
  std::vector<int> wires;    // wire ids, first = slowest (row-major)
  std::vector<c128> data;    // 2^rank values
};

struct Network {
  int nq = 0;
  NetMode mode = NET_KET;
  std::vector<WireRec> wires;  // by wire id (canonical: sorted)
  std::vector<Leaf> leaves;
  std::vector<int> open;       // ordered open wire ids (the output axes)
  c128 scalar = 1.0;           // product of fully absorbed pieces
  std::string structure() const;  // canonical description (values excluded)
};

// Validation of a closure against the circuit (throws TNQVM_EINVAL).
NetMode mode_for(const tnqvm_circuit& c, const Closure& cl);
Network build_network(const tnqvm_circuit& c, const Closure& cl);

// Light-cone selection used by CLOSE_PAULI with cancel (reading R9): kept op indices.
std::vector<int> light_cone_ops(const tnqvm_circuit& c, const std::vector<int>& support,
                                std::vector<int>* qubits_out);

}  // namespace tnqvm
