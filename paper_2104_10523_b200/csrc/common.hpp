// Shared host-side definitions of libtnqvm (not an ABI header; see include/tnqvm.h).
#pragma once

#include <complex>
#include <memory>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tnqvm.h"

namespace tnqvm {

using c128 = std::complex<double>;
using u128 = unsigned __int128;

// Error carried inside the library; converted to a return code at the ABI.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
#define TNQVM_THROW(code, msg) throw ::tnqvm::Error((code), (msg))
#define TNQVM_CHECK(cond, code, msg) \
  do {                               \
    if (!(cond)) TNQVM_THROW(code, msg); \
  } while (0)

std::string u128_to_string(u128 v);
double u128_log2(u128 v);

// ---------------------------------------------------------------------------
// Circuit store (a1): ordered op list, copied from the caller, complex128.
// ---------------------------------------------------------------------------
struct OpRec {
  int kind = 0;               // 0 = gate, 1 = kraus
  int k = 1;                  // 1 or 2 qubits
  int q[2] = {0, 0};
  int m = 1;                  // number of matrices
  std::vector<c128> mats;     // m * (2^k)^2, row-major
  const c128* mat(int i) const { return mats.data() + (size_t)i * (1 << k) * (1 << k); }
};

}  // namespace tnqvm

struct tnqvm_circuit {
  int nq = 0;
  std::vector<tnqvm::OpRec> ops;
  uint64_t revision = 0;
  // shared with every plan made from this circuit (plans keep a private copy of the op list
  // and snapshot the revision; a later apply_* makes plan use return TNQVM_ESTATE, §8(b))
  std::shared_ptr<uint64_t> rev_token = std::make_shared<uint64_t>(0);
  bool noisy() const {
    for (auto& o : ops)
      if (o.kind == 1) return true;
    return false;
  }
};
