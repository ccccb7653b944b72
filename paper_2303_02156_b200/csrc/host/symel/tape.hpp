// Symbolic front end, part 3: lowering an evaluation plan to the flat SSA tape and its binary
// wire format "SYTP" v1 -- the IR handed across the C ABI to libsymel_cuda.so.
// Register layout [inputs | constants (deduplicated by bit pattern) | one per operation] and the
// file layout follow the reference's tape.hpp (/root/reference/proj/include/symel/
// tape.hpp:18-39, 121-182, 211-291), so tapes are interchangeable with the reference's.
#pragma once

#include <cstdint>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "symel/autodiff.hpp"

namespace symel {

struct TapeInstr {
  Op op;
  std::int32_t iarg = 0;
  std::uint32_t dst = 0, a = 0, b = 0, c = 0;
};

struct Tape {
  std::uint32_t n_inputs = 0, n_outputs = 0, n_dofs = 0, n_regs = 0;
  ExprDigest digest{};
  std::vector<double> consts;
  std::vector<TapeInstr> instrs;
  std::vector<std::uint32_t> out_regs;

  // Host interpreter of one lane (test aid; the product evaluates tapes on the device).
  void eval(const double* in, double* out) const {
    std::vector<double> r(n_regs);
    std::memcpy(r.data(), in, sizeof(double) * n_inputs);
    std::memcpy(r.data() + n_inputs, consts.data(), sizeof(double) * consts.size());
    for (const TapeInstr& t : instrs) r[t.dst] = detail::apply(t.op, r[t.a], r[t.b], r[t.c], t.iarg);
    for (std::size_t k = 0; k < out_regs.size(); ++k) out[k] = r[out_regs[k]];
  }

  std::vector<std::uint8_t> serialize() const {
    std::vector<std::uint8_t> b;
    auto u32 = [&](std::uint32_t v) {
      for (int i = 0; i < 4; ++i) b.push_back(std::uint8_t(v >> (8 * i)));
    };
    auto u64 = [&](std::uint64_t v) {
      u32(std::uint32_t(v));
      u32(std::uint32_t(v >> 32));
    };
    b.insert(b.end(), {'S', 'Y', 'T', 'P'});
    u32(1);
    b.insert(b.end(), digest.bytes.begin(), digest.bytes.end());
    u32(n_inputs);
    u32(n_outputs);
    u32(n_dofs);
    u32(n_regs);
    u64(consts.size());
    for (double v : consts) u64(detail::bits_of(v));
    u64(instrs.size());
    for (const TapeInstr& t : instrs) {
      b.push_back(static_cast<std::uint8_t>(t.op));
      u32(static_cast<std::uint32_t>(t.iarg));
      u32(t.dst);
      u32(t.a);
      u32(t.b);
      u32(t.c);
    }
    u64(out_regs.size());
    for (auto r : out_regs) u32(r);
    return b;
  }
};

// Plan -> tape. Every symbol must carry an input slot in [0, n_inputs).
inline Tape lower(const ExprGraph& g, const EvalPlan& plan, std::uint32_t n_inputs, std::uint32_t n_dofs) {
  Tape t;
  t.n_inputs = n_inputs;
  t.n_dofs = n_dofs;
  t.n_outputs = static_cast<std::uint32_t>(plan.roots.size());
  t.digest = g.digest(plan.roots);
  std::string missing;
  for (NodeId id : plan.order) {
    const Node& n = g.node(id);
    if (n.op == Op::symbol && n.iarg < 0)
      missing += (missing.empty() ? "" : ", ") + (g.symbol_name(id).empty() ? std::string("<unnamed>") : g.symbol_name(id));
  }
  if (!missing.empty()) throw Error("lower: symbols without an input slot: " + missing);
  std::unordered_map<NodeId, std::uint32_t> reg;
  std::unordered_map<std::uint64_t, std::uint32_t> creg;
  for (NodeId id : plan.order) {  // inputs and constants first, so op registers are contiguous
    const Node& n = g.node(id);
    if (n.op == Op::symbol) {
      if (static_cast<std::uint32_t>(n.iarg) >= n_inputs)
        throw Error("lower: symbol '" + g.symbol_name(id) + "' slot " + std::to_string(n.iarg) +
                    " outside declared input count " + std::to_string(n_inputs));
      reg.emplace(id, static_cast<std::uint32_t>(n.iarg));
    } else if (n.op == Op::constant) {
      const auto bits = detail::bits_of(n.value);
      auto [it, fresh] = creg.emplace(bits, n_inputs + static_cast<std::uint32_t>(t.consts.size()));
      if (fresh) t.consts.push_back(n.value);
      reg.emplace(id, it->second);
    }
  }
  std::uint32_t next = n_inputs + static_cast<std::uint32_t>(t.consts.size());
  for (NodeId id : plan.order) {
    const Node& n = g.node(id);
    if (!is_operation(n.op)) continue;
    TapeInstr in;
    in.op = n.op;
    in.iarg = n.iarg;
    in.dst = next;
    in.a = reg.at(n.child[0]);
    if (n.arity >= 2) in.b = reg.at(n.child[1]);
    if (n.arity >= 3) in.c = reg.at(n.child[2]);
    t.instrs.push_back(in);
    reg.emplace(id, next++);
  }
  t.n_regs = next;
  for (NodeId r : plan.roots) t.out_regs.push_back(reg.at(r));
  return t;
}

}  // namespace symel
