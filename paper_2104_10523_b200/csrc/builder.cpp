// a2: circuit -> tensor network builder (host, complex128).
//
// Paper: qubits are rank-1, 1-qubit gates rank-2, 2-qubit gates rank-4 tensors wired
// in gate order (§3.1); "small gate tensors are contracted
// internally to form larger tensors": here every 1-qubit operator and every
// boundary vector (initial |0>, projection <b|, Pauli closure) is absorbed, in
// complex128, into an adjacent 2-qubit node, so the network handed to the planner has
// one node per 2-qubit operation.  Expectation values use the ket copy (U) and the
// bra copy (U*) joined through the Pauli tensors (Eq.(2), Fig. exp_val_double_depth,
// P:L181) after dropping U U^dagger pairs outside the observable's light cone
// (P:L188).  Noisy circuits use superoperator nodes sum_k K (x) K* acting on the ket
// and bra legs together (Eq.(3)), closed by projection or trace.
#include "builder.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <sstream>

namespace tnqvm {
namespace {

struct Leg {
  int side, q, dir;  // dir 0 = out, 1 = in
  int wire = -1;     // index into wire table, -1 = unassigned
};

struct Node {
  std::vector<Leg> legs;
  std::vector<c128> data;  // row-major, legs[0] slowest
  int q[2];
};

using Mat = std::vector<c128>;  // square row-major

Mat mat_id(int D) {
  Mat m((size_t)D * D, 0.0);
  for (int i = 0; i < D; ++i) m[(size_t)i * D + i] = 1.0;
  return m;
}
Mat mat_mul(const Mat& a, const Mat& b, int D) {
  Mat c((size_t)D * D, 0.0);
  for (int i = 0; i < D; ++i)
    for (int k = 0; k < D; ++k) {
      c128 x = a[(size_t)i * D + k];
      if (x == 0.0) continue;
      for (int j = 0; j < D; ++j) c[(size_t)i * D + j] += x * b[(size_t)k * D + j];
    }
  return c;
}
Mat mat_T(const Mat& a, int D) {
  Mat t((size_t)D * D);
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j) t[(size_t)j * D + i] = a[(size_t)i * D + j];
  return t;
}
Mat kron(const Mat& a, int Da, const Mat& b, int Db) {
  int D = Da * Db;
  Mat c((size_t)D * D);
  for (int i = 0; i < Da; ++i)
    for (int j = 0; j < Da; ++j)
      for (int k = 0; k < Db; ++k)
        for (int l = 0; l < Db; ++l)
          c[(size_t)(i * Db + k) * D + (j * Db + l)] = a[(size_t)i * Da + j] * b[(size_t)k * Db + l];
  return c;
}

// ----- small binary-leg tensor helpers -----
int leg_pos(const Node& n, int side, int q, int dir) {
  for (size_t i = 0; i < n.legs.size(); ++i)
    if (n.legs[i].side == side && n.legs[i].q == q && n.legs[i].dir == dir) return (int)i;
  TNQVM_THROW(TNQVM_EINVAL, "builder: leg not found");
}

// out = sum_x T[.., x@pos, ..] v[x]; removes legs `pos` (pos[0] = MSB of x).
void contract_vec(Node& n, const std::vector<int>& pos, const std::vector<c128>& v) {
  int R = (int)n.legs.size(), g = (int)pos.size();
  std::vector<char> sel(R, 0);
  for (int p : pos) sel[p] = 1;
  std::vector<c128> out((size_t)1 << (R - g), 0.0);
  for (uint64_t idx = 0; idx < ((uint64_t)1 << R); ++idx) {
    uint64_t x = 0, j = 0;
    for (int p : pos) x = (x << 1) | ((idx >> (R - 1 - p)) & 1);
    for (int p = 0; p < R; ++p)
      if (!sel[p]) j = (j << 1) | ((idx >> (R - 1 - p)) & 1);
    out[j] += n.data[idx] * v[x];
  }
  std::vector<Leg> legs;
  for (int p = 0; p < R; ++p)
    if (!sel[p]) legs.push_back(n.legs[p]);
  n.legs = legs;
  n.data = out;
}

// T'[.., y@pos, ..] = sum_x M[y, x] T[.., x@pos, ..]
void transform_legs(Node& n, const std::vector<int>& pos, const Mat& M) {
  int R = (int)n.legs.size(), g = (int)pos.size(), D = 1 << g;
  std::vector<c128> out(n.data.size(), 0.0);
  for (uint64_t idx = 0; idx < ((uint64_t)1 << R); ++idx) {
    c128 t = n.data[idx];
    if (t == 0.0) continue;
    uint64_t x = 0, rest = idx;
    for (int p : pos) {
      x = (x << 1) | ((idx >> (R - 1 - p)) & 1);
      rest &= ~((uint64_t)1 << (R - 1 - p));
    }
    for (int y = 0; y < D; ++y) {
      c128 m = M[(size_t)y * D + x];
      if (m == 0.0) continue;
      uint64_t o = rest;
      for (int i = 0; i < g; ++i)
        if ((y >> (g - 1 - i)) & 1) o |= (uint64_t)1 << (R - 1 - pos[i]);
      out[o] += m * t;
    }
  }
  n.data = out;
}

// ----- per-family chain records -----
struct Hop {
  int node;
  int unit;      // 0 or 1 within the node
  Mat pending;   // 1-qubit operators between the previous hop and this node
  int seg_after; // segment count after this node's op(s)
};

struct Family {
  std::vector<int> sides;  // lanes per unit: sides[i] for i < u (ket=0, bra=1)
  bool conj = false;       // bra copy of a pure circuit
};

bool is_diag(const OpRec& o) {
  int D = 1 << o.k;
  for (int i = 0; i < D; ++i)
    for (int j = 0; j < D; ++j)
      if (i != j && o.mats[(size_t)i * D + j] != 0.0) return false;
  return true;
}

}  // namespace

NetMode mode_for(const tnqvm_circuit& c, const Closure& cl) {
  if (c.noisy()) return NET_SUPEROP;
  return cl.kind == CLOSE_PAULI ? NET_PURE_DOUBLED : NET_KET;
}

std::vector<int> light_cone_ops(const tnqvm_circuit& c, const std::vector<int>& support,
                                std::vector<int>* qubits_out) {
  // Backward sweep.  A maximal run of consecutive diagonal gates is one layer
  // of commuting gates: its gates are kept iff they meet L as it stood after the run.
  std::vector<char> L(c.nq, 0);
  for (int q : support) L[q] = 1;
  std::vector<int> keep;
  int i = (int)c.ops.size() - 1;
  while (i >= 0) {
    const OpRec& o = c.ops[i];
    if (o.kind == 0 && is_diag(o)) {
      int j = i;
      while (j - 1 >= 0 && c.ops[j - 1].kind == 0 && is_diag(c.ops[j - 1])) --j;
      std::vector<char> L0 = L;
      for (int t = i; t >= j; --t) {
        const OpRec& ot = c.ops[t];
        bool hit = false;
        for (int a = 0; a < ot.k; ++a) hit |= L0[ot.q[a]] != 0;
        if (hit) {
          keep.push_back(t);
          for (int a = 0; a < ot.k; ++a) L[ot.q[a]] = 1;
        }
      }
      i = j - 1;
      continue;
    }
    bool hit = false;
    for (int a = 0; a < o.k; ++a) hit |= L[o.q[a]] != 0;
    if (hit) {
      keep.push_back(i);
      for (int a = 0; a < o.k; ++a) L[o.q[a]] = 1;
    }
    --i;
  }
  std::reverse(keep.begin(), keep.end());
  if (qubits_out) {
    qubits_out->clear();
    for (int q = 0; q < c.nq; ++q)
      if (L[q]) qubits_out->push_back(q);
  }
  return keep;
}

std::string Network::structure() const {
  std::ostringstream s;
  s << "nq=" << nq << ";mode=" << (int)mode << ";wires=";
  for (auto& w : wires) s << w.side << "," << w.qubit << "," << w.segment << ";";
  s << "leaves=";
  for (auto& l : leaves) {
    s << "[";
    for (int w : l.wires) s << w << ",";
    s << "]";
  }
  s << ";open=";
  for (int w : open) s << w << ",";
  return s.str();
}

Network build_network(const tnqvm_circuit& c, const Closure& cl) {
  const int nq = c.nq;
  NetMode mode = mode_for(c, cl);
  // ---- which ops / qubits take part ----
  std::vector<int> ops_idx;
  std::vector<char> active(nq, 1);
  std::vector<char> pauli(nq, 'I');
  if (cl.kind == CLOSE_PAULI) {
    TNQVM_CHECK((int)cl.pauli.size() == nq, TNQVM_EINVAL, "pauli closure size");
    std::vector<int> support;
    for (int q = 0; q < nq; ++q) {
      pauli[q] = cl.pauli[q];
      if (pauli[q] != 'I') support.push_back(q);
    }
    if (cl.cancel) {
      std::vector<int> qs;
      ops_idx = light_cone_ops(c, support, &qs);
      std::fill(active.begin(), active.end(), 0);
      for (int q : qs) active[q] = 1;
    }
  } else {
    TNQVM_CHECK((int)cl.bits.size() == nq, TNQVM_EINVAL, "bitstring size");
  }
  if (ops_idx.empty() && !(cl.kind == CLOSE_PAULI && cl.cancel))
    for (int i = 0; i < (int)c.ops.size(); ++i) ops_idx.push_back(i);

  // ---- families ----
  std::vector<Family> fams;
  if (mode == NET_KET) fams.push_back({{0}, false});
  else if (mode == NET_PURE_DOUBLED) { fams.push_back({{0}, false}); fams.push_back({{1}, true}); }
  else fams.push_back({{0, 1}, false});

  Network net;
  net.nq = nq;
  net.mode = mode;
  std::vector<Node> nodes;
  std::vector<WireRec> wtab;
  std::map<WireRec, int> wmap;
  auto wire_of = [&](int side, int q, int seg) {
    WireRec r{side, q, seg};
    auto it = wmap.find(r);
    if (it != wmap.end()) return it->second;
    int id = (int)wtab.size();
    wtab.push_back(r);
    wmap[r] = id;
    return id;
  };

  // final chain state per family and qubit
  struct Tail { int node = -1; int unit = 0; Mat pending; int seg = 0; };
  std::vector<std::vector<Tail>> tails(fams.size(), std::vector<Tail>(nq));

  for (size_t fi = 0; fi < fams.size(); ++fi) {
    const Family& F = fams[fi];
    const int u = (int)F.sides.size(), D = 1 << u;
    // operator matrix over u lanes per qubit for a k-qubit op (k units)
    auto op_matrix = [&](const OpRec& o) {
      int d = 1 << o.k;           // per-copy dimension
      int DD = 1 << (u * o.k);    // node dimension
      Mat M((size_t)DD * DD, 0.0);
      if (u == 1) {
        for (int i = 0; i < d * d; ++i) M[i] = F.conj ? std::conj(o.mats[i]) : o.mats[i];
        return M;
      }
      // superoperator: rows (k0,b0[,k1,b1]) cols likewise; value sum_K K[k,k'] conj(K[b,b'])
      for (int K = 0; K < o.m; ++K) {
        const c128* Km = o.mat(K);
        for (int r = 0; r < DD; ++r)
          for (int cc = 0; cc < DD; ++cc) {
            int kr = 0, br = 0, kc = 0, bc = 0;
            for (int a = 0; a < o.k; ++a) {
              int rb = (r >> (2 * (o.k - 1 - a))) & 3, cb = (cc >> (2 * (o.k - 1 - a))) & 3;
              kr = kr * 2 + (rb >> 1); br = br * 2 + (rb & 1);
              kc = kc * 2 + (cb >> 1); bc = bc * 2 + (cb & 1);
            }
            M[(size_t)r * DD + cc] += Km[kr * d + kc] * std::conj(Km[br * d + bc]);
          }
      }
      return M;
    };
    std::vector<Mat> pending(nq, mat_id(D));
    std::vector<int> last(nq, -1), seg(nq, 0);
    std::vector<std::vector<Hop>> chain(nq);
    std::vector<Mat> nmat;  // node matrices (D^2 x D^2) for this family
    std::vector<int> nid;   // global node index per family node
    for (int oi : ops_idx) {
      const OpRec& o = c.ops[oi];
      Mat M = op_matrix(o);
      if (o.k == 1) {
        pending[o.q[0]] = mat_mul(M, pending[o.q[0]], D);
        continue;
      }
      int q0 = o.q[0], q1 = o.q[1];
      int X = last[q0];
      if (X >= 0 && last[q1] == X) {
        // merge into the previous node on the same pair (the wire between them vanishes)
        Node& nd = nodes[nid[X]];
        int DD = D * D;
        Mat Mp = M;
        if (nd.q[0] != q0) {  // swap the two units
          for (int r = 0; r < DD; ++r)
            for (int cc = 0; cc < DD; ++cc) {
              int rs = (r % D) * D + r / D, cs = (cc % D) * D + cc / D;
              Mp[(size_t)rs * DD + cs] = M[(size_t)r * DD + cc];
            }
        }
        Mat pp = kron(pending[nd.q[0]], D, pending[nd.q[1]], D);
        nmat[X] = mat_mul(Mp, mat_mul(pp, nmat[X], DD), DD);
        for (int q : {q0, q1}) {
          pending[q] = mat_id(D);
          seg[q] += 1;
          chain[q].back().seg_after = seg[q];
        }
        continue;
      }
      int id = (int)nmat.size();
      nmat.push_back(M);
      nid.push_back((int)nodes.size());
      Node nd;
      nd.q[0] = q0; nd.q[1] = q1;
      nodes.push_back(nd);
      for (int a = 0; a < 2; ++a) {
        int q = o.q[a];
        seg[q] += 1;
        chain[q].push_back({id, a, pending[q], seg[q]});
        pending[q] = mat_id(D);
        last[q] = id;
      }
    }
    // materialise node tensors: legs = out(unit0 lanes, unit1 lanes), in(unit0, unit1)
    for (size_t X = 0; X < nmat.size(); ++X) {
      Node& nd = nodes[nid[X]];
      for (int dir = 0; dir < 2; ++dir)
        for (int a = 0; a < 2; ++a)
          for (int s : F.sides) nd.legs.push_back({s, nd.q[a], dir, -1});
      nd.data = nmat[X];
    }
    auto unit_pos = [&](Node& nd, int q, int dir) {
      std::vector<int> pos;
      for (int s : F.sides) pos.push_back(leg_pos(nd, s, q, dir));
      return pos;
    };
    // walk chains: absorb pending operators and the initial state, create wires
    for (int q = 0; q < nq; ++q) {
      int prev = -1, prev_seg = 0;
      for (Hop& h : chain[q]) {
        Node& nd = nodes[nid[h.node]];
        std::vector<int> pin = unit_pos(nd, q, 1);
        if (prev < 0) {
          std::vector<c128> v(D, 0.0);
          for (int i = 0; i < D; ++i) v[i] = h.pending[(size_t)i * D + 0];  // pending * e0
          contract_vec(nd, pin, v);
        } else {
          transform_legs(nd, pin, mat_T(h.pending, D));
          Node& pn = nodes[nid[prev]];
          for (int s : F.sides) {
            int w = wire_of(s, q, prev_seg);
            nd.legs[leg_pos(nd, s, q, 1)].wire = w;
            pn.legs[leg_pos(pn, s, q, 0)].wire = w;
          }
        }
        prev = h.node;
        prev_seg = h.seg_after;
      }
      Tail& t = tails[fi][q];
      t.node = prev < 0 ? -1 : nid[prev];
      t.pending = pending[q];
      t.seg = prev_seg;
    }
  }

  // ---- closures ----
  std::vector<int> open_ket, open_bra;
  if (mode == NET_KET || mode == NET_SUPEROP) {
    const int u = mode == NET_KET ? 1 : 2, D = 1 << u;
    const std::vector<int> sides = mode == NET_KET ? std::vector<int>{0} : std::vector<int>{0, 1};
    for (int q = 0; q < nq; ++q) {
      if (!active[q]) continue;
      Tail& t = tails[0][q];
      // closure row vector w over the unit (ket[,bra]) or open (empty)
      bool open = false;
      std::vector<c128> w(D, 0.0);
      if (cl.kind == CLOSE_PROJECT) {
        int b = cl.bits[q];
        if (b < 0) open = true;
        else if (u == 1) w[b] = 1.0;
        else w[b * 2 + b] = 1.0;
      } else {  // superop Pauli closure: w[i_ket*2 + j_bra] = P[j][i]
        c128 P[2][2];
        switch (pauli[q]) {
          case 'X': P[0][0] = 0; P[0][1] = 1; P[1][0] = 1; P[1][1] = 0; break;
          case 'Y': P[0][0] = 0; P[0][1] = c128(0, -1); P[1][0] = c128(0, 1); P[1][1] = 0; break;
          case 'Z': P[0][0] = 1; P[0][1] = 0; P[1][0] = 0; P[1][1] = -1; break;
          case '0': P[0][0] = 1; P[0][1] = 0; P[1][0] = 0; P[1][1] = 0; break;   // |0><0| (sampling)
          case '1': P[0][0] = 0; P[0][1] = 0; P[1][0] = 0; P[1][1] = 1; break;   // |1><1|
          default: P[0][0] = 1; P[0][1] = 0; P[1][0] = 0; P[1][1] = 1; break;
        }
        for (int i = 0; i < 2; ++i)
          for (int j = 0; j < 2; ++j) w[i * 2 + j] = P[j][i];
      }
      if (!open) {
        // r = w * pending
        std::vector<c128> r(D, 0.0);
        for (int i = 0; i < D; ++i)
          for (int j = 0; j < D; ++j) r[j] += w[i] * t.pending[(size_t)i * D + j];
        if (t.node < 0) {
          net.scalar *= r[0];  // r * e0
        } else {
          Node& nd = nodes[t.node];
          std::vector<int> pos;
          for (int s : sides) pos.push_back(leg_pos(nd, s, q, 0));
          contract_vec(nd, pos, r);
        }
      } else {
        if (t.node < 0) {
          Node nd;
          nd.q[0] = nd.q[1] = q;
          for (int s : sides) nd.legs.push_back({s, q, 0, -1});
          nd.data.assign(D, 0.0);
          for (int i = 0; i < D; ++i) nd.data[i] = t.pending[(size_t)i * D + 0];
          nodes.push_back(nd);
          t.node = (int)nodes.size() - 1;
        } else {
          Node& nd = nodes[t.node];
          std::vector<int> pos;
          for (int s : sides) pos.push_back(leg_pos(nd, s, q, 0));
          transform_legs(nd, pos, t.pending);
        }
        Node& nd = nodes[t.node];
        for (int s : sides) {
          int w2 = wire_of(s, q, t.seg);
          nd.legs[leg_pos(nd, s, q, 0)].wire = w2;
          (s == 0 ? open_ket : open_bra).push_back(w2);
        }
      }
    }
  } else {  // NET_PURE_DOUBLED with Pauli closure
    for (int q = 0; q < nq; ++q) {
      if (!active[q]) continue;
      Tail& tk = tails[0][q];
      Tail& tb = tails[1][q];
      c128 C[2][2];  // C[i_ket][j_bra] = P[j][i]
      c128 P[2][2];
      switch (pauli[q]) {
        case 'X': P[0][0] = 0; P[0][1] = 1; P[1][0] = 1; P[1][1] = 0; break;
        case 'Y': P[0][0] = 0; P[0][1] = c128(0, -1); P[1][0] = c128(0, 1); P[1][1] = 0; break;
        case 'Z': P[0][0] = 1; P[0][1] = 0; P[1][0] = 0; P[1][1] = -1; break;
        case '0': P[0][0] = 1; P[0][1] = 0; P[1][0] = 0; P[1][1] = 0; break;   // |0><0| (sampling)
        case '1': P[0][0] = 0; P[0][1] = 0; P[1][0] = 0; P[1][1] = 1; break;   // |1><1|
        default: P[0][0] = 1; P[0][1] = 0; P[1][0] = 0; P[1][1] = 1; break;
      }
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) C[i][j] = P[j][i];
      // M[a][b] = sum_{i,j} pk[i][a] C[i][j] pb[j][b]
      Mat M(4, 0.0);
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
          for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j)
              M[a * 2 + b] += tk.pending[i * 2 + a] * C[i][j] * tb.pending[j * 2 + b];
      if (tk.node < 0 && tb.node < 0) {
        net.scalar *= M[0];
      } else if (tk.node < 0) {
        contract_vec(nodes[tb.node], {leg_pos(nodes[tb.node], 1, q, 0)}, {M[0], M[1]});
      } else if (tb.node < 0) {
        contract_vec(nodes[tk.node], {leg_pos(nodes[tk.node], 0, q, 0)}, {M[0], M[2]});
      } else {
        Node& nk = nodes[tk.node];
        int p = leg_pos(nk, 0, q, 0);
        transform_legs(nk, {p}, mat_T(M, 2));  // new leg carries the bra index b
        int w = wire_of(1, q, tb.seg);
        nk.legs[p].wire = w;
        Node& nb = nodes[tb.node];
        nb.legs[leg_pos(nb, 1, q, 0)].wire = w;
      }
    }
  }

  // ---- canonical wire ids and leaves ----
  std::vector<int> order(wtab.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  std::sort(order.begin(), order.end(), [&](int a, int b) { return wtab[a] < wtab[b]; });
  std::vector<int> remap(wtab.size());
  for (size_t i = 0; i < order.size(); ++i) {
    remap[order[i]] = (int)i;
    net.wires.push_back(wtab[order[i]]);
  }
  std::vector<int> deg(wtab.size(), 0);
  for (Node& nd : nodes) {
    if (nd.legs.empty()) {
      if (!nd.data.empty()) net.scalar *= nd.data[0];
      continue;
    }
    Leaf lf;
    for (Leg& l : nd.legs) {
      TNQVM_CHECK(l.wire >= 0, TNQVM_EINVAL, "builder: dangling leg");
      lf.wires.push_back(remap[l.wire]);
      deg[l.wire]++;
    }
    lf.data = nd.data;
    net.leaves.push_back(std::move(lf));
  }
  for (int w : open_ket) net.open.push_back(remap[w]);
  for (int w : open_bra) net.open.push_back(remap[w]);
  for (size_t w = 0; w < wtab.size(); ++w) {
    bool is_open = false;
    for (int o : open_ket) is_open |= o == (int)w;
    for (int o : open_bra) is_open |= o == (int)w;
    TNQVM_CHECK(deg[w] == (is_open ? 1 : 2), TNQVM_EINVAL, "builder: wire degree");
  }
  return net;
}

}  // namespace tnqvm
