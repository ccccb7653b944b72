// A small expression DAG over the tape opcodes, used only by the factorisation pass
// (factorize.cpp) to re-derive an energy's gradient and Hessian in a narrower set of
// variables. It is not the reference's front end: it never sees user code, only the energy
// closure of a tape the reference produced, and everything it builds goes back out as a
// TapeIR (tape_io.hpp) for the code generator.
//
//   * nodes are interned (op, exponent, operands, constant bits) so equal subexpressions
//     are one node; add/mul operands are kept in id order so a+b and b+a intern together;
//   * `apply` folds constant operands (with the tape's arithmetic: pow_int as a multiply
//     loop, branch as c >= 0, expr.hpp:96-122) and the exact identities x+0, x-0, x*1, x/1,
//     -(-x); products with a zero factor and zero numerators fold to 0 -- exact for finite
//     operands, and a non-finite operand makes the energy itself non-finite, which the
//     assembler's finiteness check reports anyway;
//   * `gradient` is reverse mode (one adjoint sweep for all variables); `tangent` is forward
//     mode along one variable, used over the adjoint graph for Hessian columns;
//   * `lower` emits [inputs | constants | one register per op] in a post-order of the roots.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <unordered_map>
#include <vector>

#include "tape_io.hpp"

namespace symel_cuda::sym {

constexpr std::uint32_t kNone = 0xffffffffu;

struct Expr {
  TOp op;
  std::int32_t iarg;        // pow_int exponent
  std::uint32_t arg[3];     // operands, kNone when unused
  std::uint64_t bits;       // constant: bit pattern; symbol: input slot
};

class Dag {
 public:
  std::uint32_t input(std::uint32_t slot) { return intern(Expr{TOp::symbol, 0, {kNone, kNone, kNone}, slot}); }

  std::uint32_t constant(double v) {
    std::uint64_t b;
    std::memcpy(&b, &v, 8);
    return intern(Expr{TOp::constant, 0, {kNone, kNone, kNone}, b});
  }

  const Expr& at(std::uint32_t id) const { return nodes_[id]; }
  std::size_t size() const { return nodes_.size(); }

  bool is_const(std::uint32_t id) const { return nodes_[id].op == TOp::constant; }
  double value(std::uint32_t id) const {
    double v;
    std::memcpy(&v, &nodes_[id].bits, 8);
    return v;
  }
  bool is_value(std::uint32_t id, double v) const { return is_const(id) && value(id) == v; }
  bool is_zero(std::uint32_t id) const { return is_value(id, 0.0); }

  std::uint32_t apply(TOp op, std::uint32_t a, std::uint32_t b = kNone, std::uint32_t c = kNone, std::int32_t iarg = 0) {
    const int ar = top_arity(op);
    bool all_const = true;
    const std::uint32_t ops[3] = {a, b, c};
    for (int q = 0; q < ar; ++q) all_const = all_const && is_const(ops[q]);
    if (all_const) return constant(eval(op, iarg, ar > 0 ? value(a) : 0.0, ar > 1 ? value(b) : 0.0, ar > 2 ? value(c) : 0.0));
    switch (op) {
      case TOp::add:
        if (is_zero(a)) return b;
        if (is_zero(b)) return a;
        if (a > b) std::swap(a, b);
        break;
      case TOp::sub:
        if (is_zero(b)) return a;
        if (is_zero(a)) return apply(TOp::neg, b);
        if (a == b) return constant(0.0);
        break;
      case TOp::mul:
        if (is_zero(a) || is_zero(b)) return constant(0.0);
        if (is_value(a, 1.0)) return b;
        if (is_value(b, 1.0)) return a;
        if (is_value(a, -1.0)) return apply(TOp::neg, b);
        if (is_value(b, -1.0)) return apply(TOp::neg, a);
        if (a > b) std::swap(a, b);
        break;
      case TOp::div:
        if (is_zero(a)) return constant(0.0);
        if (is_value(b, 1.0)) return a;
        break;
      case TOp::neg:
        if (nodes_[a].op == TOp::neg) return nodes_[a].arg[0];
        break;
      case TOp::pow_int:
        if (iarg == 1) return a;
        if (iarg == 0) return constant(1.0);
        break;
      case TOp::branch:
        if (b == c) return b;
        if (is_const(a)) return value(a) >= 0.0 ? b : c;
        break;
      default:
        break;
    }
    return intern(Expr{op, op == TOp::pow_int ? iarg : 0, {a, ar > 1 ? b : kNone, ar > 2 ? c : kNone}, 0});
  }

  std::uint32_t add(std::uint32_t a, std::uint32_t b) { return apply(TOp::add, a, b); }
  std::uint32_t sub(std::uint32_t a, std::uint32_t b) { return apply(TOp::sub, a, b); }
  std::uint32_t mul(std::uint32_t a, std::uint32_t b) { return apply(TOp::mul, a, b); }
  std::uint32_t div(std::uint32_t a, std::uint32_t b) { return apply(TOp::div, a, b); }
  std::uint32_t neg(std::uint32_t a) { return apply(TOp::neg, a); }

  // Post-order (operands before users) of everything reachable from `roots`, iterative.
  std::vector<std::uint32_t> postorder(const std::vector<std::uint32_t>& roots) const {
    std::vector<std::uint32_t> out;
    std::vector<std::uint8_t> state(nodes_.size(), 0);  // 0 new, 1 open, 2 done
    std::vector<std::uint32_t> stack;
    for (std::uint32_t r : roots) {
      if (r == kNone || state[r] == 2) continue;
      stack.push_back(r);
      while (!stack.empty()) {
        const std::uint32_t id = stack.back();
        if (state[id] == 2) { stack.pop_back(); continue; }
        if (state[id] == 0) {
          state[id] = 1;
          const Expr& e = nodes_[id];
          for (int q = top_arity(e.op) - 1; q >= 0; --q)
            if (state[e.arg[q]] == 0) stack.push_back(e.arg[q]);
          continue;
        }
        state[id] = 2;
        out.push_back(id);
        stack.pop_back();
      }
    }
    return out;
  }

  // `root` rebuilt through apply (so it re-folds) with the nodes pre-seeded in `memo`
  // replaced by their mapped nodes; `memo` may be shared between roots.
  std::uint32_t substitute(std::uint32_t root, std::unordered_map<std::uint32_t, std::uint32_t>& memo) {
    for (std::uint32_t id : postorder({root})) {
      if (memo.count(id)) continue;
      const Expr e = nodes_[id];
      if (top_arity(e.op) == 0) {
        memo.emplace(id, id);
        continue;
      }
      const std::uint32_t a = memo.at(e.arg[0]);
      const std::uint32_t b = e.arg[1] == kNone ? kNone : memo.at(e.arg[1]);
      const std::uint32_t c = e.arg[2] == kNone ? kNone : memo.at(e.arg[2]);
      memo.emplace(id, apply(e.op, a, b, c, e.iarg));
    }
    return memo.at(root);
  }

  // Reverse mode: d f / d v for every leaf v in `wrt` (one adjoint sweep).
  std::vector<std::uint32_t> gradient(std::uint32_t f, const std::vector<std::uint32_t>& wrt) {
    const std::vector<std::uint32_t> order = postorder({f});
    std::unordered_map<std::uint32_t, std::uint32_t> adj;
    adj[f] = constant(1.0);
    auto bump = [&](std::uint32_t node, std::uint32_t v) {
      if (is_zero(v)) return;
      auto it = adj.find(node);
      if (it == adj.end()) adj.emplace(node, v);
      else it->second = add(it->second, v);
    };
    for (std::size_t k = order.size(); k-- > 0;) {
      const std::uint32_t id = order[k];
      auto it = adj.find(id);
      if (it == adj.end()) continue;
      const std::uint32_t w = it->second;
      const Expr e = nodes_[id];
      const std::uint32_t a = e.arg[0], b = e.arg[1], c = e.arg[2];
      switch (e.op) {
        case TOp::add: bump(a, w); bump(b, w); break;
        case TOp::sub: bump(a, w); bump(b, neg(w)); break;
        case TOp::neg: bump(a, neg(w)); break;
        case TOp::mul: bump(a, mul(w, b)); bump(b, mul(w, a)); break;
        case TOp::div: {  // id = a / b: d/da = 1/b, d/db = -id/b
          const std::uint32_t q = div(w, b);
          bump(a, q);
          bump(b, neg(mul(q, id)));
          break;
        }
        case TOp::pow_int:
          bump(a, mul(w, mul(constant(double(e.iarg)), apply(TOp::pow_int, a, kNone, kNone, e.iarg - 1))));
          break;
        case TOp::sqrt: bump(a, div(w, add(id, id))); break;
        case TOp::log: bump(a, div(w, a)); break;
        case TOp::sin: bump(a, mul(w, apply(TOp::cos, a))); break;
        case TOp::cos: bump(a, neg(mul(w, apply(TOp::sin, a)))); break;
        case TOp::branch: {
          const std::uint32_t z = constant(0.0);
          bump(b, apply(TOp::branch, a, w, z));
          bump(c, apply(TOp::branch, a, z, w));
          break;
        }
        default: break;
      }
    }
    std::vector<std::uint32_t> g(wrt.size());
    for (std::size_t k = 0; k < wrt.size(); ++k) {
      auto it = adj.find(wrt[k]);
      g[k] = it == adj.end() ? constant(0.0) : it->second;
    }
    return g;
  }

  // Forward mode: directional derivative of `root` along the leaf `v`; `memo` may be shared
  // between roots differentiated along the same leaf.
  std::uint32_t tangent(std::uint32_t root, std::uint32_t v, std::unordered_map<std::uint32_t, std::uint32_t>& memo) {
    for (std::uint32_t id : postorder({root})) {
      if (memo.count(id)) continue;
      const Expr e = nodes_[id];
      const std::uint32_t a = e.arg[0], b = e.arg[1], c = e.arg[2];
      auto T = [&](std::uint32_t x) { return memo.at(x); };
      std::uint32_t r;
      switch (e.op) {
        case TOp::symbol: r = constant(id == v ? 1.0 : 0.0); break;
        case TOp::constant: r = constant(0.0); break;
        case TOp::add: r = add(T(a), T(b)); break;
        case TOp::sub: r = sub(T(a), T(b)); break;
        case TOp::neg: r = neg(T(a)); break;
        case TOp::mul: r = add(mul(T(a), b), mul(a, T(b))); break;
        case TOp::div: r = div(sub(T(a), mul(id, T(b))), b); break;  // (a' - (a/b) b') / b
        case TOp::pow_int:
          r = mul(mul(constant(double(e.iarg)), apply(TOp::pow_int, a, kNone, kNone, e.iarg - 1)), T(a));
          break;
        case TOp::sqrt: r = div(T(a), add(id, id)); break;
        case TOp::log: r = div(T(a), a); break;
        case TOp::sin: r = mul(apply(TOp::cos, a), T(a)); break;
        case TOp::cos: r = neg(mul(apply(TOp::sin, a), T(a))); break;
        case TOp::branch: r = apply(TOp::branch, a, T(b), T(c)); break;
        default: throw std::runtime_error("sym: bad opcode");
      }
      memo.emplace(id, r);
    }
    return memo.at(root);
  }

  // Emits the roots as a tape: registers [inputs (slots 0..n_inputs-1) | constants in
  // first-use order | one per operation in post-order]. Throws when a symbol outside the
  // input range survived (an unresolved substitution).
  TapeIR lower(const std::vector<std::uint32_t>& roots, std::uint32_t n_inputs, std::uint32_t n_dofs) const {
    const std::vector<std::uint32_t> order = postorder(roots);
    TapeIR t;
    t.n_inputs = n_inputs;
    t.n_dofs = n_dofs;
    std::unordered_map<std::uint32_t, std::uint32_t> reg;
    std::unordered_map<std::uint64_t, std::uint32_t> const_reg;
    for (std::uint32_t id : order) {
      const Expr& e = nodes_[id];
      if (e.op == TOp::symbol) {
        if (e.bits >= n_inputs) throw std::runtime_error("sym: unresolved symbol in lowered tape");
        reg[id] = static_cast<std::uint32_t>(e.bits);
      } else if (e.op == TOp::constant && !const_reg.count(e.bits)) {
        const_reg[e.bits] = static_cast<std::uint32_t>(t.consts.size());
        double v;
        std::memcpy(&v, &e.bits, 8);
        t.consts.push_back(v);
      }
    }
    for (std::uint32_t id : order)
      if (nodes_[id].op == TOp::constant) reg[id] = n_inputs + const_reg.at(nodes_[id].bits);
    std::uint32_t next = n_inputs + static_cast<std::uint32_t>(t.consts.size());
    for (std::uint32_t id : order) {
      const Expr& e = nodes_[id];
      const int ar = top_arity(e.op);
      if (ar == 0) continue;
      TInstr in{e.op, e.iarg, next, reg.at(e.arg[0]), ar > 1 ? reg.at(e.arg[1]) : 0u, ar > 2 ? reg.at(e.arg[2]) : 0u};
      t.instrs.push_back(in);
      reg[id] = next++;
    }
    t.n_regs = next;
    t.out_regs.reserve(roots.size());
    for (std::uint32_t r : roots) t.out_regs.push_back(reg.at(r));
    t.n_outputs = static_cast<std::uint32_t>(t.out_regs.size());
    return t;
  }

  static double eval(TOp op, std::int32_t iarg, double a, double b, double c) {
    switch (op) {
      case TOp::add: return a + b;
      case TOp::sub: return a - b;
      case TOp::mul: return a * b;
      case TOp::div: return a / b;
      case TOp::neg: return -a;
      case TOp::pow_int: {
        long long n = iarg < 0 ? -static_cast<long long>(iarg) : iarg;
        double r = 1.0;
        while (n-- > 0) r *= a;
        return iarg < 0 ? 1.0 / r : r;
      }
      case TOp::sqrt: return std::sqrt(a);
      case TOp::log: return std::log(a);
      case TOp::sin: return std::sin(a);
      case TOp::cos: return std::cos(a);
      case TOp::branch: return a >= 0.0 ? b : c;
      default: throw std::runtime_error("sym: bad opcode");
    }
  }

 private:
  struct KeyHash {
    std::size_t operator()(const Expr& e) const {
      std::uint64_t h = 0x9e3779b97f4a7c15ull ^ static_cast<std::uint64_t>(e.op);
      auto mix = [&](std::uint64_t v) { h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2); };
      mix(static_cast<std::uint32_t>(e.iarg));
      mix(e.arg[0]);
      mix(e.arg[1]);
      mix(e.arg[2]);
      mix(e.bits);
      return static_cast<std::size_t>(h);
    }
  };
  struct KeyEq {
    bool operator()(const Expr& x, const Expr& y) const {
      return x.op == y.op && x.iarg == y.iarg && x.arg[0] == y.arg[0] && x.arg[1] == y.arg[1] && x.arg[2] == y.arg[2] &&
             x.bits == y.bits;
    }
  };

  std::uint32_t intern(const Expr& e) {
    auto it = index_.find(e);
    if (it != index_.end()) return it->second;
    const std::uint32_t id = static_cast<std::uint32_t>(nodes_.size());
    nodes_.push_back(e);
    index_.emplace(e, id);
    return id;
  }

  std::vector<Expr> nodes_;
  std::unordered_map<Expr, std::uint32_t, KeyHash, KeyEq> index_;
};

}  // namespace symel_cuda::sym
