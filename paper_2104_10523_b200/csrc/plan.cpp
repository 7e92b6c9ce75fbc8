// Plan construction and the canonical plan JSON (a3/a4 outputs).
#include "plan.hpp"

#include <algorithm>
#include <sstream>

namespace tnqvm {

tnqvm_plan* make_plan(const tnqvm_circuit& c, const Closure& cl, uint64_t budget_bytes,
                      const tnqvm_plan_opts& opts) {
  auto p = std::make_unique<tnqvm_plan>();
  p->circuit = c;
  p->rev_snapshot = *c.rev_token;
  p->closure = cl;
  p->mode = mode_for(c, cl);
  p->dtype = opts.dtype;
  p->budget_bytes = budget_bytes;
  p->opts = opts;
  p->net = build_network(c, cl);
  p->structure = p->net.structure();
  p->network_hash = sha256_hex(p->structure);
  const uint64_t esize = opts.dtype == TNQVM_C64 ? 8 : 16;
  uint64_t budget = budget_bytes / esize;
  TNQVM_CHECK(budget >= 1, TNQVM_EINFEASIBLE, "max_slice_bytes below one element");
  PlanOpts po;
  po.seed = opts.seed;
  po.restarts = opts.restarts;
  po.threads = opts.threads;
  po.time_cap_s = opts.time_cap_s;
  po.min_slices = std::max<uint64_t>(1, opts.min_slices);
  po.cost_model = opts.cost_model;
  po.partition = opts.partition;
  po.beta = opts.dtype == TNQVM_C64 ? 24 : 20;  // measured complex-MAC rate / HBM element rate (R18)
  p->path = plan_network(p->net, budget, po);
  return p.release();
}

std::string plan_json(const tnqvm_plan& p) {
  // keys sorted, compact separators, integers and strings only
  const Network& n = p.net;
  const PathResult& r = p.path;
  std::ostringstream s;
  s << "{";
  s << "\"beta\":" << (p.dtype == TNQVM_C64 ? 24 : 20);  // cost-model balance (R18)
  s << ",\"budget_bytes\":" << p.budget_bytes;
  s << ",\"cost_model\":" << p.opts.cost_model;
  s << ",\"dtype\":\"" << (p.dtype == TNQVM_C64 ? "c64" : "c128") << "\"";
  s << ",\"leaves\":[";
  for (size_t i = 0; i < n.leaves.size(); ++i) {
    s << (i ? "," : "") << "[";
    for (size_t j = 0; j < n.leaves[i].wires.size(); ++j) s << (j ? "," : "") << n.leaves[i].wires[j];
    s << "]";
  }
  s << "]";
  int mx = r.log2_max_sliced;
  s << ",\"macs_sliced\":\"" << u128_to_string(r.macs_sliced) << "\"";
  s << ",\"macs_unsliced\":\"" << u128_to_string(r.macs_unsliced) << "\"";
  s << ",\"max_intermediate_elems\":\"" << u128_to_string((u128)1 << mx) << "\"";
  s << ",\"min_slices\":" << p.opts.min_slices;
  s << ",\"mode\":\"" << (p.mode == NET_KET ? "ket" : p.mode == NET_PURE_DOUBLED ? "braket" : "superop") << "\"";
  s << ",\"n_slices\":\"" << u128_to_string((u128)1 << r.sliced.size()) << "\"";
  s << ",\"network_hash\":\"" << p.network_hash << "\"";
  s << ",\"nq\":" << n.nq;
  s << ",\"open\":[";
  for (size_t i = 0; i < n.open.size(); ++i) s << (i ? "," : "") << n.open[i];
  s << "]";
  s << ",\"partition\":" << p.opts.partition;
  s << ",\"restarts\":" << p.opts.restarts;
  s << ",\"seed\":\"" << p.opts.seed << "\"";
  s << ",\"sliced\":[";
  for (size_t i = 0; i < r.sliced.size(); ++i) s << (i ? "," : "") << r.sliced[i];
  s << "]";
  s << ",\"steps\":[";
  for (size_t i = 0; i < r.steps.size(); ++i)
    s << (i ? "," : "") << "[" << r.steps[i][0] << "," << r.steps[i][1] << "]";
  s << "]";
  s << ",\"version\":1";
  s << ",\"wires\":[";
  for (size_t i = 0; i < n.wires.size(); ++i) {
    const WireRec& w = n.wires[i];
    s << (i ? "," : "") << "{\"id\":" << i << ",\"qubit\":" << w.qubit << ",\"segment\":" << w.segment
      << ",\"side\":\"" << (w.side == 0 ? "ket" : "bra") << "\"}";
  }
  s << "]";
  s << "}";
  return s.str();
}

}  // namespace tnqvm
