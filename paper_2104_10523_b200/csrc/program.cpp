// a5: program compilation -- layouts chosen for the consumer, per-step kernel class,
// fused small-step batches, liveness-planned arena offsets, launch list.
#include "program.hpp"

#include <algorithm>
#include <atomic>
#include <cstring>
#include <functional>
#include <map>
#include <numeric>
#include <set>

namespace tnqvm {
namespace {

constexpr int64_t kAlign = 64;  // elements (>= 512 B for c64)

int64_t align_up(int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

std::vector<int> set_xor(const std::vector<int>& a, const std::vector<int>& b) {
  std::vector<int> sa(a), sb(b), out;
  std::sort(sa.begin(), sa.end());
  std::sort(sb.begin(), sb.end());
  std::set_symmetric_difference(sa.begin(), sa.end(), sb.begin(), sb.end(), std::back_inserter(out));
  return out;
}
bool contains(const std::vector<int>& v, int w) { return std::find(v.begin(), v.end(), w) != v.end(); }
int pos_of(const std::vector<int>& v, int w) {
  auto it = std::find(v.begin(), v.end(), w);
  return it == v.end() ? -1 : (int)(it - v.begin());
}
int64_t stride_of(const Ten& t, int w) {
  int p = pos_of(t.layout, w);
  return p < 0 ? 0 : ((int64_t)1 << (t.rank - 1 - p));
}
// wires of `order` that are in `set`, keeping order
std::vector<int> filter(const std::vector<int>& order, const std::vector<int>& set, bool keep_in) {
  std::vector<int> out;
  for (int w : order)
    if (contains(set, w) == keep_in) out.push_back(w);
  return out;
}
std::vector<int> concat(std::vector<int> a, const std::vector<int>& b) {
  a.insert(a.end(), b.begin(), b.end());
  return a;
}
// do the |K| fastest wires of `layout` equal the set K?
bool k_fastest(const std::vector<int>& layout, const std::vector<int>& K) {
  if (K.size() > layout.size()) return false;
  for (size_t i = layout.size() - K.size(); i < layout.size(); ++i)
    if (!contains(K, layout[i])) return false;
  return true;
}
std::vector<int> fastest(const std::vector<int>& layout, size_t n) {
  return std::vector<int>(layout.end() - n, layout.end());
}

struct StepInfo {
  int a, b, c;
  std::vector<int> K, Afree, Bfree;  // sets (unordered)
  int cls;
  bool x_is_a;
};

}  // namespace

void program_free(Program* p) {
  if (!p) return;
  // free on the program's device, then restore the caller's current device (a plan may be
  // freed or recompiled while another device is current -- torch's, or another context's)
  int prev = -1;
  cudaGetDevice(&prev);
  if (p->device >= 0) cudaSetDevice(p->device);
  if (p->d_small_steps) cudaFree(p->d_small_steps);
  if (p->d_tasks) cudaFree(p->d_tasks);
  if (p->d_leaves) cudaFree(p->d_leaves);
  for (auto& g : p->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  delete p;
  if (prev >= 0) cudaSetDevice(prev);
}

Program* compile_program(const tnqvm_plan& p, int device) {
  auto prog = std::unique_ptr<Program, ProgramDeleter>(new Program);
  Program& P = *prog;
  P.dtype = p.dtype == TNQVM_C64 ? 0 : 1;
  P.esize = P.dtype == 0 ? 8 : 16;
  P.device = device;
  static std::atomic<uint64_t> next_uid{1};
  P.uid = next_uid.fetch_add(1);
  const Network& net = p.net;
  const PathResult& R = p.path;
  const int L = (int)net.leaves.size(), S = (int)R.steps.size();
  const int W = (int)net.wires.size();
  std::vector<int> sdig(W, -1);  // slice digit index (0 = MSB)
  for (size_t i = 0; i < R.sliced.size(); ++i) sdig[R.sliced[i]] = (int)i;
  const int nsl = (int)R.sliced.size();
  P.n_sliced = nsl;
  P.sliced = R.sliced;

  // ---- tensors and wire sets (sliced wires removed) ----
  std::vector<std::vector<int>> wset(L + S);
  P.tens.resize(L + S);
  for (int i = 0; i < L; ++i) {
    for (int w : net.leaves[i].wires)
      if (sdig[w] < 0) wset[i].push_back(w);
      else P.tens[i].dep = true;
    P.tens[i].leaf = true;
    P.tens[i].leaf_index = i;
    P.tens[i].rank = (int)wset[i].size();
  }
  std::vector<int> consumer(L + S, -1);
  std::vector<StepInfo> info(S);
  for (int s = 0; s < S; ++s) {
    int a = R.steps[s][0], b = R.steps[s][1], c = L + s;
    consumer[a] = s;
    consumer[b] = s;
    wset[c] = set_xor(wset[a], wset[b]);
    P.tens[c].rank = (int)wset[c].size();
    P.tens[c].dep = P.tens[a].dep || P.tens[b].dep;
    StepInfo& si = info[s];
    si.a = a; si.b = b; si.c = c;
    for (int w : wset[a]) (contains(wset[b], w) ? si.K : si.Afree).push_back(w);
    for (int w : wset[b])
      if (!contains(wset[a], w)) si.Bfree.push_back(w);
    int ra = (int)wset[a].size(), rb = (int)wset[b].size(), rc = (int)wset[c].size(), nk = (int)si.K.size();
    int fa = (int)si.Afree.size(), fb = (int)si.Bfree.size();
    // kernel class: one-CTA fused batch for tiny steps; split-K for tiny outputs over huge K;
    // whole-GPU strided kernel (any layout, no permutes) for skinny steps (K*M <= 64) and
    // mid-size steps; tensor-core / tiled GEMM for the rest
    // whole-GPU strided steps up to log2(K*|C|) = 22.  Fused small tasks only up to
    // log2(K*|C|) = 13: a task runs its steps serially in one CTA, and the C2 steps of 2^14-2^16
    // multiply-adds ran at 4-13 us each that way (small class 1.29 -> 0.73 ms per bench step
    // with them moved to the whole-GPU kernels; at 11 the expectation term batches of C4 stop
    // being single fused tasks and lose 8x)
    constexpr int strided_max = 22;
    if (nk <= dev::SMALL_MAXK && ra <= dev::SMALL_MAXC && rb <= dev::SMALL_MAXC && rc <= dev::SMALL_MAXC &&
        nk + rc <= 13)
      si.cls = CLS_SMALL;
    else if (nk >= 12 && (rc <= 4 || (fa <= 6 && fb <= 6 && (rc <= 10 || nk > 16))))
      si.cls = CLS_SPLITK;
    else if (nk <= 6 && std::max(fa, fb) <= 40 &&
             (P.dtype == 0 ? (std::min(fa, fb) <= 4 && nk + std::min(fa, fb) <= 7) : (std::min(fa, fb) <= 3 && nk + std::min(fa, fb) <= 6)))
      si.cls = CLS_SKINNY;
    else if (nk <= dev::SMALL_MAXK && rc <= 32 && (nk + std::min(fa, fb) <= 6 || nk + rc <= strided_max))
      si.cls = CLS_STRIDED;
    else
      si.cls = CLS_GEMM;
    si.x_is_a = fa > fb || (fa == fb && ra >= rb);
  }
  const int root = S > 0 ? L + S - 1 : (L == 1 ? 0 : -1);
  P.final_tensor = root;

  // ---- execution order: slice-invariant steps first (hoisted), then per-slice steps ----
  std::vector<int> order;
  for (int s = 0; s < S; ++s)
    if (!P.tens[L + s].dep) order.push_back(s);
  int n_inv = (int)order.size();
  for (int s = 0; s < S; ++s)
    if (P.tens[L + s].dep) order.push_back(s);

  auto decide_leaf = [&](int t, const std::vector<int>& layout) {
    Ten& T = P.tens[t];
    if (!T.leaf || T.decided) return;
    T.layout = layout;
    T.decided = true;
  };
  auto natural_leaf = [&](int t) {
    if (P.tens[t].leaf && !P.tens[t].decided) decide_leaf(t, wset[t]);
  };
  // split-K steps with a tiny output read both operands in any layout (k_splitk.cu)
  auto strided_splitk = [&](const StepInfo& si) {
    return dev::splitk_strided_supported((int)std::max(si.Afree.size(), si.Bfree.size()), (int)si.K.size(),
                                         (int)std::min(si.Afree.size(), si.Bfree.size()));
  };
  // tensor-core GEMM can gather X tiles itself (k_tc.cu) when X's fastest mode is contracted
  auto tc_gather_ok = [&](const Ten& X, const std::vector<int>& K, int nm) {
    const int nk = (int)K.size();
    return P.dtype == 0 && nk >= 1 && dev::tc_supported(nk, nm) && nk + nm >= 5 &&
           X.rank - nk <= 40 && !X.layout.empty() && contains(K, X.layout.back());
  };
  // requirement on the layout of tensor t from its consumer (for producers that can choose)
  auto desired = [&](int t, const std::vector<int>& natural) -> std::vector<int> {
    if (t == root) return net.open;
    int c = consumer[t];
    if (c < 0) return natural;
    const StepInfo& si = info[c];
    bool t_is_x = (si.a == t) == si.x_is_a;
    if (si.cls == CLS_GEMM && t_is_x) {
      return concat(filter(natural, si.K, false), filter(natural, si.K, true));
    }
    if (si.cls == CLS_SPLITK && strided_splitk(si)) return natural;
    if (si.cls == CLS_SPLITK) {
      int other = si.a == t ? si.b : si.a;
      const Ten& O = P.tens[other];
      std::vector<int> sigma;
      if (O.decided && k_fastest(O.layout, si.K)) sigma = fastest(O.layout, si.K.size());
      else sigma = filter(natural, si.K, true);
      return concat(filter(natural, si.K, false), sigma);
    }
    return natural;
  };

  // ---- emit ops ----
  struct SmallStep { int a, b, c; };
  std::vector<SmallStep> sm_steps;                 // all small steps, appended per batch
  std::vector<std::vector<int>> task_steps;        // per task: indices into sm_steps
  std::vector<int> op_of_task;
  std::vector<int> batch;                          // pending small steps (indices into sm_steps)
  bool batch_dep = false;
  auto flush = [&]() {
    if (batch.empty()) return;
    // connected components by data dependence inside the batch
    std::vector<int> comp(batch.size());
    std::iota(comp.begin(), comp.end(), 0);
    std::function<int(int)> find = [&](int x) { return comp[x] == x ? x : comp[x] = find(comp[x]); };
    std::map<int, int> producer;  // tensor -> batch index
    for (size_t i = 0; i < batch.size(); ++i) {
      const SmallStep& st = sm_steps[batch[i]];
      for (int in : {st.a, st.b}) {
        auto it = producer.find(in);
        if (it != producer.end()) comp[find((int)i)] = find(it->second);
      }
      producer[st.c] = (int)i;
    }
    std::map<int, std::vector<int>> groups;
    for (size_t i = 0; i < batch.size(); ++i) groups[find((int)i)].push_back(batch[i]);
    Op op;
    op.kind = OP_SMALL;
    op.dep = batch_dep;
    op.task_begin = (int)task_steps.size();
    for (auto& kv : groups) {
      task_steps.push_back(kv.second);
      op_of_task.push_back((int)P.ops.size());
    }
    op.task_end = (int)task_steps.size();
    for (int i : batch) {
      const SmallStep& st = sm_steps[i];
      int nk = (int)(P.tens[st.a].rank + P.tens[st.b].rank - P.tens[st.c].rank) / 2;
      double macs = std::ldexp(1.0, P.tens[st.c].rank + nk);
      op.flops += 8 * macs;
      op.bytes += P.esize * (double)(P.tens[st.a].size() + P.tens[st.b].size() + P.tens[st.c].size());
    }
    P.ops.push_back(op);
    batch.clear();
  };
  auto add_permute = [&](int src, const std::vector<int>& target, bool dep) {
    Ten t;
    t.rank = P.tens[src].rank;
    t.layout = target;
    t.decided = true;
    t.dep = dep;
    int id = (int)P.tens.size();
    P.tens.push_back(t);
    Op op;
    op.kind = OP_PERMUTE;
    op.dep = dep;
    op.x = src;
    op.c = id;
    for (int w : target) op.perm.push_back(pos_of(P.tens[src].layout, w));
    op.bytes = 2.0 * P.esize * (double)t.size();
    P.ops.push_back(op);
    return id;
  };

  std::vector<int> alias(L + S);  // current tensor id holding the value (after permutes)
  std::iota(alias.begin(), alias.end(), 0);
  // schedule a permute (N1) when the consumer cannot use the produced layout directly
  auto relayout_for_consumer = [&](int c) {
    std::vector<int> want = desired(c, P.tens[c].layout);
    if (want == P.tens[c].layout) return;
    bool need = true;
    int cc = consumer[c];
    if (cc >= 0 && c != root) {
      const StepInfo& ci = info[cc];
      bool c_is_x = (ci.a == c) == ci.x_is_a;
      if (ci.cls == CLS_SMALL || ci.cls == CLS_STRIDED || ci.cls == CLS_SKINNY || (ci.cls == CLS_GEMM && !c_is_x))
        need = false;
      if (ci.cls == CLS_GEMM && c_is_x && k_fastest(P.tens[c].layout, ci.K)) need = false;
      if (ci.cls == CLS_GEMM && c_is_x && tc_gather_ok(P.tens[c], ci.K, (int)(ci.x_is_a ? ci.Bfree : ci.Afree).size()))
        need = false;
    }
    if (need) {
      flush();
      alias[c] = add_permute(c, want, P.tens[c].dep);
    }
  };
  for (int oi = 0; oi < (int)order.size(); ++oi) {
    const int s = order[oi];
    const bool dep = oi >= n_inv;
    if (dep != batch_dep) {
      flush();
      batch_dep = dep;
    }
    StepInfo& si = info[s];
    const int c = si.c;
    int a = alias[si.a], b = alias[si.b];
    if (si.cls == CLS_SMALL) {
      natural_leaf(a);
      natural_leaf(b);
      std::vector<int> nat = concat(filter(P.tens[a].layout, si.Afree, true), filter(P.tens[b].layout, si.Bfree, true));
      P.tens[c].layout = desired(c, nat);
      P.tens[c].decided = true;
      sm_steps.push_back({a, b, c});
      batch.push_back((int)sm_steps.size() - 1);
      continue;
    }
    flush();
    if (si.cls == CLS_SKINNY) {
      natural_leaf(a);
      natural_leaf(b);
      const int x = si.x_is_a ? a : b, y = si.x_is_a ? b : a;
      const std::vector<int>& Xf = si.x_is_a ? si.Afree : si.Bfree;
      const std::vector<int>& Yf = si.x_is_a ? si.Bfree : si.Afree;
      // C's fastest modes = X's fastest free modes (coalesced writes) unless the consumer asks otherwise
      std::vector<int> nat = concat(filter(P.tens[y].layout, Yf, true), filter(P.tens[x].layout, Xf, true));
      std::vector<int> want = desired(c, nat);
      // keep coalesced writes: the consumer's layout only if its two fastest wires are the
      // streamed operand's two fastest free wires; otherwise write `nat` and let N1 re-lay it
      // coalesced if C's two fastest wires are X's two fastest free wires (consecutive lanes)
      // or free wires of Y (then they are m bits 0 and 1: contiguous within a thread)
      const size_t q = std::min<size_t>(2, nat.size());
      bool ok = want.size() >= q && std::equal(want.end() - q, want.end(), nat.end() - q);
      if (!ok && want.size() >= 2 && Yf.size() >= 2)
        ok = contains(Yf, want[want.size() - 1]) && contains(Yf, want[want.size() - 2]);
      P.tens[c].layout = ok ? want : nat;
      P.tens[c].decided = true;
      const Ten &X = P.tens[x], &Y = P.tens[y], &Cc = P.tens[c];
      Op op;
      op.kind = OP_SKINNY;
      op.dep = dep;
      op.x = x;
      op.y = y;
      op.c = c;
      for (int i = X.rank - 1; i >= 0; --i) {  // n bits: X's free wires, fastest first
        int w = X.layout[i];
        if (contains(si.K, w)) {
          op.sxk.push_back(stride_of(X, w));
          op.syk.push_back(stride_of(Y, w));
        } else {
          op.sxn.push_back(stride_of(X, w));
          op.scn.push_back(stride_of(Cc, w));
        }
      }
      for (int i = Cc.rank - 1; i >= 0; --i) {  // m bits: Y's free wires in C's order, fastest first
        int w = Cc.layout[i];
        if (contains(Yf, w)) {
          op.sym.push_back(stride_of(Y, w));
          op.scm.push_back(stride_of(Cc, w));
        }
      }
      op.nn = (int)op.sxn.size();
      op.nk = (int)op.sxk.size();
      op.nm = (int)op.sym.size();
      op.N = (int64_t)1 << op.nn;
      op.flops = 8 * std::ldexp(1.0, op.nn + op.nk + op.nm);
      op.bytes = P.esize * (double)(X.size() + Y.size() + Cc.size());
      P.ops.push_back(op);
      if (!ok) relayout_for_consumer(c);
      continue;
    }
    if (si.cls == CLS_STRIDED) {
      natural_leaf(a);
      natural_leaf(b);
      std::vector<int> nat = concat(filter(P.tens[a].layout, si.Afree, true), filter(P.tens[b].layout, si.Bfree, true));
      P.tens[c].layout = desired(c, nat);
      P.tens[c].decided = true;
      Op op;
      op.kind = OP_STRIDED;
      op.dep = dep;
      op.x = a;
      op.y = b;
      op.c = c;
      op.nk = (int)si.K.size();
      op.flops = 8 * std::ldexp(1.0, (int)(si.K.size() + wset[c].size()));
      op.bytes = P.esize * (double)(P.tens[a].size() + P.tens[b].size() + P.tens[c].size());
      P.ops.push_back(op);
      continue;
    }
    int x = si.x_is_a ? a : b, y = si.x_is_a ? b : a;
    const std::vector<int>& Xfree = si.x_is_a ? si.Afree : si.Bfree;
    const std::vector<int>& Yfree = si.x_is_a ? si.Bfree : si.Afree;
    Op op;
    op.dep = dep;
    if (si.cls == CLS_GEMM) {
      if (P.tens[x].leaf && !P.tens[x].decided)
        decide_leaf(x, concat(filter(wset[x], si.K, false), filter(wset[x], si.K, true)));
      // tensor-core gather: X need not be K-contiguous if its fastest mode is contracted
      // (16-byte pieces = two complex64 along that mode), so no permute is scheduled
      bool gather = false;
      if (!k_fastest(P.tens[x].layout, si.K)) {
        if (tc_gather_ok(P.tens[x], si.K, (int)Yfree.size()))
          gather = true;
        else
          x = add_permute(x, concat(filter(P.tens[x].layout, si.K, false), filter(P.tens[x].layout, si.K, true)),
                          P.tens[x].dep);
      }
      natural_leaf(y);
      const Ten& X = P.tens[x];
      const Ten& Y = P.tens[y];
      std::vector<int> korder = filter(X.layout, si.K, true);  // slowest..fastest (X's order)
      std::vector<int> norder = filter(X.layout, si.K, false);
      std::vector<int> morder = filter(Y.layout, Yfree, true);
      // look-ahead: put the consumer's contracted wires last among M
      std::vector<int> want = desired(c, concat(norder, morder));
      std::vector<int> mfast = filter(want, morder, true);
      // keep M wires in the order they appear in the desired layout (its suffix part last)
      morder = mfast;
      op.kind = OP_GEMM;
      op.x = x;
      op.y = y;
      op.c = c;
      op.nk = (int)korder.size();
      op.nm = (int)morder.size();
      op.N = (int64_t)1 << norder.size();
      for (int i = 0; i < op.nk; ++i) op.syk.push_back(stride_of(Y, korder[op.nk - 1 - i]));
      for (int i = 0; i < op.nm; ++i) op.sym.push_back(stride_of(Y, morder[op.nm - 1 - i]));
      P.tens[c].layout = concat(norder, morder);
      P.tens[c].decided = true;
      double macs = std::ldexp(1.0, (int)(norder.size() + morder.size() + korder.size()));
      op.flops = 8 * macs;
      op.bytes = P.esize * (double)(X.size() + Y.size() + P.tens[c].size());
      // method (the kernel-class choice; tensor cores when the step is dense enough)
      op.method = GM_SIMT;
      if (P.dtype == 0 && dev::tc_supported(op.nk, op.nm)) op.method = GM_TC;
      if (P.dtype == 1 && dev::dmma_supported(op.nk, op.nm)) op.method = GM_DMMA;
      if (op.method == GM_DMMA) P.wbuf_bytes = std::max(P.wbuf_bytes, dev::dmma_wbuf_bytes(op.N, op.nk, op.nm));
      if (op.nk + op.nm < 5) op.method = GM_SIMT;  // K*M < 32: far below the SIMT ridge
      if (op.method == GM_TC) P.wbuf_bytes = std::max(P.wbuf_bytes, dev::tc_wbuf_bytes(op.N, op.nk, op.nm));
      if (gather) {
        op.gather = 1;
        for (int i = 0; i < op.nk; ++i) op.sxk.push_back(stride_of(X, korder[op.nk - 1 - i]));
        for (int i = 0; i < (int)norder.size(); ++i) op.sxn.push_back(stride_of(X, norder[norder.size() - 1 - i]));
        op.nn = (int)norder.size();
      }
      P.ops.push_back(op);
    } else if (strided_splitk(si)) {
      // CLS_SPLITK, tiny output: both operands read in their stored layouts (no permute);
      // undecided leaves take Y's / X's contracted order so both streams coalesce
      std::vector<int> sigma;
      for (int t : {x, y})
        if (sigma.empty() && (!P.tens[t].leaf || P.tens[t].decided)) sigma = filter(P.tens[t].layout, si.K, true);
      if (sigma.empty()) sigma = filter(wset[x], si.K, true);
      for (int t : {x, y}) decide_leaf(t, concat(filter(wset[t], si.K, false), sigma));
      const Ten& X = P.tens[x];
      const Ten& Y = P.tens[y];
      std::vector<int> nat = concat(filter(X.layout, si.K, false), filter(Y.layout, si.K, false));
      P.tens[c].layout = desired(c, nat);
      P.tens[c].decided = true;
      const Ten& Cc = P.tens[c];
      op.kind = OP_SPLITK;
      op.gather = 1;
      op.x = x;
      op.y = y;
      op.c = c;
      for (int i = X.rank - 1; i >= 0; --i) {  // X's order, fastest first
        int w = X.layout[i];
        if (contains(si.K, w)) {
          op.sxk.push_back(stride_of(X, w));
          op.syk.push_back(stride_of(Y, w));
        } else {
          op.sxn.push_back(stride_of(X, w));
          op.scn.push_back(stride_of(Cc, w));
        }
      }
      for (int i = Y.rank - 1; i >= 0; --i) {
        int w = Y.layout[i];
        if (!contains(si.K, w)) {
          op.sym.push_back(stride_of(Y, w));
          op.scm.push_back(stride_of(Cc, w));
        }
      }
      op.nk = (int)op.sxk.size();
      op.nn = (int)op.sxn.size();
      op.nm = (int)op.sym.size();
      op.N = (int64_t)1 << op.nn;
      op.flops = 8 * std::ldexp(1.0, op.nk + op.nn + op.nm);
      op.bytes = P.esize * (double)(X.size() + Y.size() + Cc.size());
      P.scratch_bytes = std::max(P.scratch_bytes, dev::splitk_strided_scratch_bytes(op.nn, op.nm));
      P.ops.push_back(op);
    } else {  // CLS_SPLITK: both operands K-fastest with the same K order
      std::vector<int> sigma;
      for (int t : {x, y})
        if (!P.tens[t].leaf || P.tens[t].decided)
          if (sigma.empty() && k_fastest(P.tens[t].layout, si.K)) sigma = fastest(P.tens[t].layout, si.K.size());
      if (sigma.empty()) {
        const std::vector<int>& base = (!P.tens[x].leaf || P.tens[x].decided) ? P.tens[x].layout : wset[x];
        sigma = filter(base, si.K, true);
      }
      for (int* t : {&x, &y}) {
        const std::vector<int>& fr = (*t == x) ? Xfree : Yfree;
        (void)fr;
        if (P.tens[*t].leaf && !P.tens[*t].decided) {
          decide_leaf(*t, concat(filter(wset[*t], si.K, false), sigma));
        } else if (!(k_fastest(P.tens[*t].layout, si.K) && fastest(P.tens[*t].layout, si.K.size()) == sigma)) {
          *t = add_permute(*t, concat(filter(P.tens[*t].layout, si.K, false), sigma), P.tens[*t].dep);
        }
      }
      std::vector<int> nat = concat(filter(P.tens[x].layout, si.K, false), filter(P.tens[y].layout, si.K, false));
      op.kind = OP_SPLITK;
      op.x = x;
      op.y = y;
      op.c = c;
      op.nk = (int)si.K.size();
      op.N = (int64_t)1 << Xfree.size();
      op.nm = (int)Yfree.size();
      P.tens[c].layout = nat;
      P.tens[c].decided = true;
      op.flops = 8 * std::ldexp(1.0, (int)(si.K.size() + Xfree.size() + Yfree.size()));
      op.bytes = P.esize * (double)(P.tens[x].size() + P.tens[y].size() + P.tens[c].size());
      P.scratch_bytes = std::max(P.scratch_bytes, dev::splitk_scratch_bytes(P.dtype, op.N, (int64_t)1 << op.nm,
                                                                            (int64_t)1 << op.nk));
      P.ops.push_back(op);
    }
    // the consumer may need another layout than the natural one of a GEMM output
    relayout_for_consumer(c);
  }
  flush();
  // root: a bare leaf
  int final_t = root >= 0 ? alias[root] : -1;
  if (root >= 0 && S == 0) {
    decide_leaf(root, net.open);
    final_t = root;
  }
  for (int t = 0; t < L; ++t) natural_leaf(t);
  if (final_t >= 0 && P.tens[final_t].layout != net.open) {
    final_t = add_permute(final_t, net.open, P.tens[final_t].dep);
  }
  P.final_tensor = final_t;
  P.result_len = (int64_t)1 << net.open.size();
  P.final_dep = final_t >= 0 && P.tens[final_t].dep;
  if (final_t >= 0) {
    Op op;
    op.kind = OP_ACCUM;
    op.dep = P.final_dep;
    op.x = final_t;
    P.ops.push_back(op);
  }
  // invariant ops must precede dependent ones (permutes were appended in order already)
  std::stable_partition(P.ops.begin(), P.ops.end(), [](const Op& o) { return !o.dep; });
  // small tasks refer to ops by index only through task ranges (unchanged by the partition)

  // ---- arena allocation (liveness over the op sequence; invariant values feeding the
  //      slice loop stay live throughout) ----
  const int NT = (int)P.tens.size();
  std::vector<int> def(NT, -1), last(NT, -1);
  const int NOPS = (int)P.ops.size();
  auto use = [&](int t, int i) {
    if (t < 0) return;
    last[t] = std::max(last[t], i);
  };
  for (int i = 0; i < NOPS; ++i) {
    Op& op = P.ops[i];
    if (op.kind == OP_SMALL) {
      for (int tk = op.task_begin; tk < op.task_end; ++tk)
        for (int si : task_steps[tk]) {
          use(sm_steps[si].a, i);
          use(sm_steps[si].b, i);
          if (def[sm_steps[si].c] < 0) def[sm_steps[si].c] = i;
          use(sm_steps[si].c, i);
          op.rd.push_back(sm_steps[si].a);
          op.rd.push_back(sm_steps[si].b);
          op.wr.push_back(sm_steps[si].c);
        }
    } else {
      use(op.x, i);
      use(op.y, i);
      if (op.x >= 0) op.rd.push_back(op.x);
      if (op.y >= 0) op.rd.push_back(op.y);
      if (op.c >= 0) {
        if (def[op.c] < 0) def[op.c] = i;
        use(op.c, i);
        op.wr.push_back(op.c);
      }
    }
  }
  int first_dep = NOPS;
  for (int i = 0; i < NOPS; ++i)
    if (P.ops[i].dep) { first_dep = i; break; }
  for (int t = 0; t < NT; ++t)
    if (!P.tens[t].leaf && def[t] >= 0 && def[t] < first_dep && last[t] >= first_dep) last[t] = NOPS;
  std::vector<int> ids;
  for (int t = 0; t < NT; ++t)
    if (!P.tens[t].leaf && def[t] >= 0) ids.push_back(t);
  std::sort(ids.begin(), ids.end(), [&](int x, int y) {
    if (P.tens[x].rank != P.tens[y].rank) return P.tens[x].rank > P.tens[y].rank;
    return x < y;
  });
  // two pools: slice-invariant tensors [0, inv), per-slice tensors [inv, inv + dep); a
  // runtime lane l (concurrent slice stream) places its per-slice pool at + l * dep
  auto place = [&](bool dep_pool) {
    std::vector<int> placed;
    int64_t top = 0;
    for (int t : ids) {
      if (P.tens[t].dep != dep_pool) continue;
      std::vector<std::pair<int64_t, int64_t>> busy;
      for (int u : placed)
        if (!(last[u] < def[t] || last[t] < def[u])) busy.push_back({P.tens[u].off, P.tens[u].off + align_up(P.tens[u].size())});
      std::sort(busy.begin(), busy.end());
      int64_t off = 0, need = align_up(P.tens[t].size());
      for (auto& iv : busy) {
        if (off + need <= iv.first) break;
        off = std::max(off, iv.second);
      }
      P.tens[t].off = off;
      top = std::max(top, off + need);
      placed.push_back(t);
    }
    return top;
  };
  P.inv_elems = align_up(place(false));
  P.dep_elems = align_up(place(true));
  for (int t : ids)
    if (P.tens[t].dep) P.tens[t].off += P.inv_elems;
  P.arena_elems = std::max<int64_t>(P.inv_elems + P.dep_elems, kAlign);

  // ---- leaves: full host layout = sliced wires (slice-digit order) + per-slice layout ----
  P.leaf_full_layout.resize(L);
  P.leaves.resize(L);
  int64_t loff = 0;
  for (int i = 0; i < L; ++i) {
    std::vector<int> sw;
    for (int w : net.leaves[i].wires)
      if (sdig[w] >= 0) sw.push_back(w);
    std::sort(sw.begin(), sw.end(), [&](int x, int y) { return sdig[x] < sdig[y]; });
    uint64_t mask = 0;
    for (int w : sw) mask |= 1ULL << (nsl - 1 - sdig[w]);
    P.leaf_full_layout[i] = concat(sw, P.tens[i].layout);
    P.leaves[i].off = loff;
    P.leaves[i].subsize = P.tens[i].size();
    P.leaves[i].mask = mask;
    loff += align_up((int64_t)1 << P.leaf_full_layout[i].size());
  }
  P.leaf_elems = std::max<int64_t>(loff, kAlign);

  // ---- small / strided step descriptors and tasks ----
  auto make_desc = [&](int ta, int tb, int tc) {
    const Ten &A = P.tens[ta], &B = P.tens[tb], &C = P.tens[tc];
    dev::SmallStepDesc d{};
    d.a_leaf = A.leaf ? A.leaf_index : -1;
    d.b_leaf = B.leaf ? B.leaf_index : -1;
    d.a_off = A.leaf ? 0 : A.off;
    d.b_off = B.leaf ? 0 : B.off;
    d.c_off = C.off;
    d.a_dep = !A.leaf && A.dep;
    d.b_dep = !B.leaf && B.dep;
    d.c_dep = C.dep;
    d.nc = C.rank;
    std::vector<int> K;
    for (int w : A.layout)
      if (contains(B.layout, w)) K.push_back(w);
    d.nk = (int)K.size();
    for (int i = 0; i < C.rank; ++i) {
      int w = C.layout[C.rank - 1 - i];
      d.sa_c[i] = stride_of(A, w);
      d.sb_c[i] = stride_of(B, w);
    }
    for (int i = 0; i < d.nk; ++i) {
      d.sa_k[i] = (int32_t)stride_of(A, K[i]);
      d.sb_k[i] = (int32_t)stride_of(B, K[i]);
    }
    return d;
  };
  for (Op& op : P.ops)
    if (op.kind == OP_STRIDED) {
      op.task_begin = (int)P.small_steps.size();
      P.small_steps.push_back(make_desc(op.x, op.y, op.c));
    }
  std::vector<int> desc_index(sm_steps.size(), -1);
  // N4: a step output read only by later steps of its own task (its last use is
  // the task's op) stays in the CTA's shared-memory arena instead of global scratch; offsets
  // by first fit over the task's step order (an output is placed before its inputs are freed)
  std::vector<int> op_of_tk(task_steps.size(), -1);
  for (int i = 0; i < NOPS; ++i)
    if (P.ops[i].kind == OP_SMALL)
      for (int tk = P.ops[i].task_begin; tk < P.ops[i].task_end; ++tk) op_of_tk[tk] = i;
  const int64_t smem_cap = dev::SMALL_SMEM_BYTES / P.esize;
  std::vector<int64_t> soff(NT, -1);
  for (size_t tk = 0; tk < task_steps.size(); ++tk) {
    const std::vector<int>& ts = task_steps[tk];
    std::map<int, int> last_in_task;  // tensor -> last step (position in ts) reading it
    for (int j = 0; j < (int)ts.size(); ++j) {
      last_in_task[sm_steps[ts[j]].a] = j;
      last_in_task[sm_steps[ts[j]].b] = j;
    }
    std::vector<std::pair<int64_t, int64_t>> live;  // [off, end) of placed internal tensors
    std::vector<int> live_t;
    int64_t top = 0;
    for (int j = 0; j < (int)ts.size(); ++j) {
      const SmallStep& st = sm_steps[ts[j]];
      const int c = st.c;
      const int64_t need = (P.tens[c].size() + 3) / 4 * 4;  // 32-byte aligned (c64)
      const bool internal = op_of_tk[tk] >= 0 && last[c] == op_of_tk[tk] && c != P.final_tensor &&
                            last_in_task.count(c) && last_in_task[c] > j && need <= smem_cap;
      if (internal) {
        std::vector<std::pair<int64_t, int64_t>> busy = live;
        std::sort(busy.begin(), busy.end());
        int64_t off = 0;
        for (auto& iv : busy) {
          if (off + need <= iv.first) break;
          off = std::max(off, iv.second);
        }
        if (off + need <= smem_cap) {
          soff[c] = off;
          live.push_back({off, off + need});
          live_t.push_back(c);
          top = std::max(top, off + need);
        }
      }
      for (int in : {st.a, st.b})  // inputs whose last read is this step leave the arena
        if (soff[in] >= 0 && last_in_task[in] == j)
          for (size_t q = 0; q < live_t.size(); ++q)
            if (live_t[q] == in) {
              live.erase(live.begin() + q);
              live_t.erase(live_t.begin() + q);
              break;
            }
    }
    P.small_smem_elems = std::max(P.small_smem_elems, top);
  }
  for (size_t tk = 0; tk < task_steps.size(); ++tk) {
    dev::SmallTask task{};
    task.begin = (int)P.small_steps.size();
    for (int si : task_steps[tk]) {
      const SmallStep& st = sm_steps[si];
      const Ten &A = P.tens[st.a], &B = P.tens[st.b], &C = P.tens[st.c];
      dev::SmallStepDesc d{};
      d.a_leaf = A.leaf ? A.leaf_index : -1;
      d.b_leaf = B.leaf ? B.leaf_index : -1;
      d.a_off = A.leaf ? 0 : A.off;
      d.b_off = B.leaf ? 0 : B.off;
      d.c_off = C.off;
      d.a_dep = !A.leaf && A.dep;
      d.b_dep = !B.leaf && B.dep;
      d.c_dep = C.dep;
      d.nc = C.rank;
      std::vector<int> K;
      for (int w : A.layout)
        if (contains(B.layout, w)) K.push_back(w);
      d.nk = (int)K.size();
      for (int i = 0; i < C.rank; ++i) {
        int w = C.layout[C.rank - 1 - i];
        d.sa_c[i] = stride_of(A, w);
        d.sb_c[i] = stride_of(B, w);
      }
      for (int i = 0; i < d.nk; ++i) {
        d.sa_k[i] = (int32_t)stride_of(A, K[i]);
        d.sb_k[i] = (int32_t)stride_of(B, K[i]);
      }
      d.smem = 0;
      if (!A.leaf && soff[st.a] >= 0) { d.smem |= 1; d.a_off = soff[st.a]; }
      if (!B.leaf && soff[st.b] >= 0) { d.smem |= 2; d.b_off = soff[st.b]; }
      if (soff[st.c] >= 0) { d.smem |= 4; d.c_off = soff[st.c]; }
      desc_index[si] = (int)P.small_steps.size();
      P.small_steps.push_back(d);
    }
    task.end = (int)P.small_steps.size();
    task.result_slot = -1;
    task.rlen = 0;
    task.scale_re = 1;
    task.scale_im = 0;
    P.tasks.push_back(task);
  }
  for (const Op& op : P.ops) {
    if (op.dep) { P.flops_per_slice += op.flops; P.bytes_per_slice += op.bytes; }
    else { P.flops_invariant += op.flops; P.bytes_invariant += op.bytes; }
  }
  return prog.release();
}

void pack_leaves(const Program& P, const Network& net, void* out) {
  std::memset(out, 0, (size_t)P.leaf_elems * P.esize);
  for (size_t i = 0; i < net.leaves.size(); ++i) {
    const Leaf& lf = net.leaves[i];
    const std::vector<int>& full = P.leaf_full_layout[i];
    const int r = (int)full.size();
    std::vector<int> src_pos(r);
    for (int j = 0; j < r; ++j) src_pos[j] = pos_of(lf.wires, full[j]);
    const int64_t n = (int64_t)1 << r;
    for (int64_t t = 0; t < n; ++t) {
      int64_t sidx = 0;
      for (int j = 0; j < r; ++j)
        if ((t >> (r - 1 - j)) & 1) sidx |= (int64_t)1 << (r - 1 - src_pos[j]);
      c128 v = lf.data[sidx];
      int64_t o = P.leaves[i].off + t;
      if (P.dtype == 0) {
        float* f = (float*)out + 2 * o;
        f[0] = (float)v.real();
        f[1] = (float)v.imag();
      } else {
        double* d = (double*)out + 2 * o;
        d[0] = v.real();
        d[1] = v.imag();
      }
    }
  }
}

}  // namespace tnqvm
