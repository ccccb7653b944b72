// Linear-frontier factorisation (see factorize.hpp).
#include "factorize.hpp"

#include <cstring>
#include <unordered_map>

#include "symel/tape.hpp"

namespace symel_cuda {

namespace {

using symel::ExprGraph;
using symel::kInvalidNode;
using symel::NodeId;
using symel::Op;

enum Cls : std::uint8_t { kConst = 0, kAffine = 1, kNonlinear = 2 };

// Rebuilds the sub-DAG under `root` with a node substitution; structurally identical parts
// come back as the same nodes (hash-consing).
struct Rebuilder {
  ExprGraph& g;
  std::unordered_map<NodeId, NodeId> memo;
  NodeId operator()(NodeId root) {
    const NodeId roots[1] = {root};
    g.for_each_postorder(roots, [&](NodeId id) {
      if (memo.count(id)) return;
      const symel::Node n = g.node(id);
      if (!symel::is_operation(n.op)) {
        memo.emplace(id, id);
        return;
      }
      const NodeId a = memo.at(n.child[0]);
      const NodeId b = n.arity > 1 ? memo.at(n.child[1]) : kInvalidNode;
      const NodeId c = n.arity > 2 ? memo.at(n.child[2]) : kInvalidNode;
      memo.emplace(id, g.make_op(n.op, a, b, c, n.iarg));
    });
    return memo.at(root);
  }
};

// Structural-zero elimination. The reference folds only the +0.0 bit pattern
// (expr.hpp:411-450), so d(-u)/dx of a dof-independent u yields neg(0) = -0.0 and every
// product with it survives as a live-but-zero subexpression. For finite operands these are
// exact zeros: x*(+-0) = +-0, (+-0)/y = +-0, z + x = x. Rebuilding with these rules removes
// them (and everything only they feed).
struct ZeroSimplifier {
  ExprGraph& g;
  NodeId zero;
  std::unordered_map<NodeId, NodeId> memo;
  bool is_zero(NodeId id) const { return g.node(id).op == Op::constant && g.node(id).value == 0.0; }
  NodeId operator()(NodeId root) {
    const NodeId roots[1] = {root};
    g.for_each_postorder(roots, [&](NodeId id) {
      if (memo.count(id)) return;
      const symel::Node n = g.node(id);
      if (!symel::is_operation(n.op)) {
        memo.emplace(id, is_zero(id) ? zero : id);
        return;
      }
      const NodeId a = memo.at(n.child[0]);
      const NodeId b = n.arity > 1 ? memo.at(n.child[1]) : kInvalidNode;
      const NodeId c = n.arity > 2 ? memo.at(n.child[2]) : kInvalidNode;
      NodeId r = kInvalidNode;
      switch (n.op) {
        case Op::mul: if (is_zero(a) || is_zero(b)) r = zero; break;
        case Op::div: if (is_zero(a)) r = zero; break;
        case Op::neg: if (is_zero(a)) r = zero; break;
        case Op::add: if (is_zero(a)) r = b; else if (is_zero(b)) r = a; break;
        case Op::sub: if (is_zero(b)) r = a; else if (is_zero(a)) r = g.make_op(Op::neg, b); break;
        case Op::branch: if (is_zero(b) && is_zero(c)) r = zero; break;
        default: break;
      }
      if (r == kInvalidNode) r = g.make_op(n.op, a, b, c, n.iarg);
      memo.emplace(id, r);
    });
    return memo.at(root);
  }
};

}  // namespace

std::optional<TapeIR> factorize_impl(const TapeIR& t, const std::vector<std::uint32_t>& dof_slots, FactorizeInfo* info,
                                     bool spd);

std::optional<TapeIR> factorize_linear_frontier(const TapeIR& t, const std::vector<std::uint32_t>& dof_slots,
                                                FactorizeInfo* info) {
  return factorize_impl(t, dof_slots, info, false);
}

std::optional<TapeIR> factorize_spd(const TapeIR& t, const std::vector<std::uint32_t>& dof_slots, FactorizeInfo* info) {
  return factorize_impl(t, dof_slots, info, true);
}

std::optional<TapeIR> factorize_impl(const TapeIR& t, const std::vector<std::uint32_t>& dof_slots, FactorizeInfo* info,
                                     bool spd) {
  const std::uint32_t n = static_cast<std::uint32_t>(dof_slots.size());
  if (n == 0 || t.n_outputs != 1 + n + n * n) return std::nullopt;
  try {
    ExprGraph G;
    std::vector<NodeId> node_of(t.n_regs, kInvalidNode);
    for (std::uint32_t k = 0; k < t.n_inputs; ++k) node_of[k] = G.symbol_id("in" + std::to_string(k), int(k));
    for (std::size_t c = 0; c < t.consts.size(); ++c) node_of[t.n_inputs + c] = G.constant_id(t.consts[c]);
    // import the energy's closure only (the gradient/Hessian part is re-derived)
    const std::uint32_t base = t.first_op_reg();
    std::vector<std::uint8_t> need(t.n_regs, 0);
    need[t.out_regs[0]] = 1;
    for (std::size_t k = t.instrs.size(); k-- > 0;) {
      const TInstr& in = t.instrs[k];
      if (!need[in.dst]) continue;
      const std::uint32_t ops[3] = {in.a, in.b, in.c};
      for (int q = 0; q < top_arity(in.op); ++q) need[ops[q]] = 1;
    }
    for (const TInstr& in : t.instrs) {
      if (!need[in.dst]) continue;
      const int ar = top_arity(in.op);
      node_of[in.dst] = G.make_op(static_cast<Op>(in.op), node_of[in.a], ar > 1 ? node_of[in.b] : kInvalidNode,
                                  ar > 2 ? node_of[in.c] : kInvalidNode, in.iarg);
    }
    (void)base;
    const NodeId E = node_of[t.out_regs[0]];
    std::vector<NodeId> xs(n);
    std::unordered_map<NodeId, std::uint32_t> dof_index;
    for (std::uint32_t k = 0; k < n; ++k) {
      xs[k] = node_of[dof_slots[k]];
      dof_index.emplace(xs[k], k);
    }

    // classify and find the affine frontier (post-order of E: deterministic)
    std::unordered_map<NodeId, Cls> cls;
    std::vector<NodeId> post;
    const NodeId eroot[1] = {E};
    G.for_each_postorder(eroot, [&](NodeId id) {
      post.push_back(id);
      const symel::Node& nd = G.node(id);
      Cls r = kConst;
      if (nd.op == Op::symbol) {
        r = dof_index.count(id) ? kAffine : kConst;
      } else if (nd.op == Op::constant) {
        r = kConst;
      } else {
        const Cls a = cls.at(nd.child[0]);
        const Cls b = nd.arity > 1 ? cls.at(nd.child[1]) : kConst;
        const Cls c = nd.arity > 2 ? cls.at(nd.child[2]) : kConst;
        switch (nd.op) {
          case Op::add: case Op::sub: r = std::max(a, b); break;
          case Op::neg: r = a; break;
          case Op::mul: r = (a == kConst || b == kConst) ? std::max(a, b) : kNonlinear; break;
          case Op::div: r = b == kConst ? a : kNonlinear; break;
          default: r = (a == kConst && b == kConst && c == kConst) ? kConst : kNonlinear; break;
        }
      }
      cls.emplace(id, r);
    });
    std::vector<NodeId> Y;
    std::unordered_map<NodeId, std::uint32_t> y_index;
    auto add_frontier = [&](NodeId id) {
      if (cls.at(id) == kAffine && !y_index.count(id)) {
        y_index.emplace(id, static_cast<std::uint32_t>(Y.size()));
        Y.push_back(id);
      }
    };
    for (NodeId id : post) {
      const symel::Node& nd = G.node(id);
      if (cls.at(id) != kNonlinear) continue;
      for (int q = 0; q < nd.arity; ++q) add_frontier(nd.child[q]);
    }
    add_frontier(E);
    const std::uint32_t m = static_cast<std::uint32_t>(Y.size());
    if (m == 0 || m >= n) return std::nullopt;

    // phi(s): E with every frontier node replaced by a fresh symbol
    std::vector<NodeId> s(m);
    for (std::uint32_t i = 0; i < m; ++i) s[i] = G.symbol_id("y" + std::to_string(i), int(t.n_inputs + i));
    Rebuilder to_phi{G, {}};
    for (std::uint32_t i = 0; i < m; ++i) to_phi.memo.emplace(Y[i], s[i]);
    const NodeId phi = to_phi(E);
    const symel::DerivativeBundle B = symel::gradient_hessian(G, phi, s);
    // back-substitute y for s
    Rebuilder to_y{G, {}};
    for (std::uint32_t i = 0; i < m; ++i) to_y.memo.emplace(s[i], Y[i]);
    const NodeId zero = G.constant_id(0.0);
    ZeroSimplifier simp{G, zero, {}};
    std::vector<NodeId> dphi(m), d2phi(std::size_t(m) * m);
    for (std::uint32_t i = 0; i < m; ++i) dphi[i] = simp(to_y(B.grad[i]));
    for (std::uint32_t i = 0; i < m; ++i)
      for (std::uint32_t j = i; j < m; ++j) d2phi[i * m + j] = d2phi[j * m + i] = simp(to_y(B.hess[i * m + j]));

    // L = dy/dx (dof-independent by construction)
    auto is_zero = [&](NodeId id) { return G.node(id).op == Op::constant && G.node(id).value == 0.0; };
    std::vector<NodeId> L(std::size_t(m) * n);
    std::uint32_t nnz = 0;
    for (std::uint32_t i = 0; i < m; ++i)
      for (std::uint32_t k = 0; k < n; ++k) {
        L[i * n + k] = simp(symel::derivative(G, Y[i], xs[k]));
        if (is_zero(L[i * n + k])) L[i * n + k] = zero;
        nnz += L[i * n + k] != zero;
      }
    auto dot = [&](auto&& term_a, auto&& term_b, std::uint32_t len) {
      NodeId acc = kInvalidNode;
      for (std::uint32_t q = 0; q < len; ++q) {
        const NodeId a = term_a(q), b = term_b(q);
        if (is_zero(a) || is_zero(b)) continue;
        const NodeId p = G.make_op(Op::mul, a, b);
        acc = acc == kInvalidNode ? p : G.make_op(Op::add, acc, p);
      }
      return acc == kInvalidNode ? zero : acc;
    };
    std::vector<NodeId> roots(1 + n + std::size_t(n) * n, zero);
    roots[0] = E;
    for (std::uint32_t k = 0; k < n; ++k)
      roots[1 + k] = dot([&](std::uint32_t i) { return L[i * n + k]; }, [&](std::uint32_t i) { return dphi[i]; }, m);
    if (spd) {
      // R = chol(L L^T) (lower), W = R^-1 L, M = R^T phi_yy R; H = W^T M W
      std::vector<NodeId> Gm(std::size_t(m) * m), R(std::size_t(m) * m, zero), W(std::size_t(m) * n, zero);
      for (std::uint32_t i = 0; i < m; ++i)
        for (std::uint32_t j = 0; j <= i; ++j)
          Gm[i * m + j] = Gm[j * m + i] =
              dot([&](std::uint32_t k) { return L[i * n + k]; }, [&](std::uint32_t k) { return L[j * n + k]; }, n);
      for (std::uint32_t j = 0; j < m; ++j) {
        NodeId s = Gm[j * m + j];
        for (std::uint32_t k = 0; k < j; ++k)
          if (!is_zero(R[j * m + k])) s = G.make_op(Op::sub, s, G.make_op(Op::mul, R[j * m + k], R[j * m + k]));
        R[j * m + j] = G.make_op(Op::sqrt, s);
        for (std::uint32_t i = j + 1; i < m; ++i) {
          NodeId v = Gm[i * m + j];
          for (std::uint32_t k = 0; k < j; ++k)
            if (!is_zero(R[i * m + k]) && !is_zero(R[j * m + k]))
              v = G.make_op(Op::sub, v, G.make_op(Op::mul, R[i * m + k], R[j * m + k]));
          R[i * m + j] = is_zero(v) ? zero : G.make_op(Op::div, v, R[j * m + j]);
        }
      }
      for (std::uint32_t i = 0; i < m; ++i)
        for (std::uint32_t c = 0; c < n; ++c) {
          NodeId v = L[i * n + c];
          for (std::uint32_t k = 0; k < i; ++k)
            if (!is_zero(R[i * m + k]) && !is_zero(W[k * n + c]))
              v = is_zero(v) ? G.make_op(Op::neg, G.make_op(Op::mul, R[i * m + k], W[k * n + c]))
                             : G.make_op(Op::sub, v, G.make_op(Op::mul, R[i * m + k], W[k * n + c]));
          W[i * n + c] = is_zero(v) ? zero : G.make_op(Op::div, v, R[i * m + i]);
        }
      std::vector<NodeId> T(std::size_t(m) * m);  // phi_yy R
      for (std::uint32_t i = 0; i < m; ++i)
        for (std::uint32_t b = 0; b < m; ++b)
          T[i * m + b] =
              dot([&](std::uint32_t j) { return d2phi[i * m + j]; }, [&](std::uint32_t j) { return R[j * m + b]; }, m);
      roots.resize(1 + n + std::size_t(m) * (m + 1) / 2 + std::size_t(m) * n, zero);
      std::size_t o = 1 + n;
      for (std::uint32_t a = 0; a < m; ++a)
        for (std::uint32_t b = a; b < m; ++b)
          roots[o++] = dot([&](std::uint32_t i) { return R[i * m + a]; }, [&](std::uint32_t i) { return T[i * m + b]; }, m);
      for (std::size_t q = 0; q < W.size(); ++q) roots[o++] = W[q];
      const symel::EvalPlan plan = symel::compress(G, roots);
      const symel::Tape Tp = symel::lower(G, plan, t.n_inputs, n);
      TapeIR out;
      out.digest = t.digest;
      out.n_inputs = Tp.n_inputs;
      out.n_outputs = Tp.n_outputs;
      out.n_dofs = Tp.n_dofs;
      out.n_regs = Tp.n_regs;
      out.consts = Tp.consts;
      for (const symel::TapeInstr& in : Tp.instrs)
        out.instrs.push_back({static_cast<TOp>(in.op), in.iarg, in.dst, in.a, in.b, in.c});
      out.out_regs = Tp.out_regs;
      if (info) *info = FactorizeInfo{m, n, t.instrs.size(), Tp.instrs.size(), nnz};
      return out;
    }
    for (std::uint32_t l = 0; l < n; ++l) {
      std::vector<NodeId> v(m);  // column l of phi_yy L
      for (std::uint32_t i = 0; i < m; ++i)
        v[i] = dot([&](std::uint32_t j) { return d2phi[i * m + j]; }, [&](std::uint32_t j) { return L[j * n + l]; }, m);
      for (std::uint32_t k = 0; k <= l; ++k) {
        const NodeId h = dot([&](std::uint32_t i) { return L[i * n + k]; }, [&](std::uint32_t i) { return v[i]; }, m);
        roots[1 + n + k * n + l] = roots[1 + n + l * n + k] = h;
      }
    }
    const symel::EvalPlan plan = symel::compress(G, roots);
    const symel::Tape T = symel::lower(G, plan, t.n_inputs, n);  // throws if a y-symbol survived
    if (T.instrs.size() >= t.instrs.size()) return std::nullopt;
    TapeIR out;
    out.digest = t.digest;
    out.n_inputs = T.n_inputs;
    out.n_outputs = T.n_outputs;
    out.n_dofs = T.n_dofs;
    out.n_regs = T.n_regs;
    out.consts = T.consts;
    for (const symel::TapeInstr& in : T.instrs)
      out.instrs.push_back({static_cast<TOp>(in.op), in.iarg, in.dst, in.a, in.b, in.c});
    out.out_regs = T.out_regs;
    if (info) *info = FactorizeInfo{m, n, t.instrs.size(), T.instrs.size(), nnz};
    return out;
  } catch (const std::exception&) {
    return std::nullopt;
  }
}

}  // namespace symel_cuda
