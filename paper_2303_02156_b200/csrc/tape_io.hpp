// Reader/writer for the reference's binary tape format "SYTP" v1
// (/root/reference/proj/include/symel/tape.hpp:211-291): magic, u32 version, 32-byte digest,
// u32 n_inputs/n_outputs/n_dofs/n_regs, u64 n_consts + f64 bit patterns, u64 n_instrs +
// {u8 op, u32 iarg, u32 dst, u32 a, u32 b, u32 c}, u64 n_out + u32 out_regs. Little endian.
// The tape is the IR the CUDA code generator consumes; it is produced host-side by the
// symbolic front end (the reference: EnergySystem::compile_kernels + Tape::save).
#pragma once

#include <array>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace symel_cuda {

// Opcode numbering of symel::Op (expr.hpp:29-43).
enum class TOp : std::uint8_t {
  symbol = 0, constant, add, sub, mul, div, neg, pow_int, sqrt, log, sin, cos, branch
};

inline int top_arity(TOp op) {
  switch (op) {
    case TOp::add: case TOp::sub: case TOp::mul: case TOp::div: return 2;
    case TOp::branch: return 3;
    case TOp::symbol: case TOp::constant: return 0;
    default: return 1;
  }
}

struct TInstr {
  TOp op;
  std::int32_t iarg;
  std::uint32_t dst, a, b, c;
};

struct TapeIR {
  std::array<std::uint8_t, 32> digest{};
  std::uint32_t n_inputs = 0, n_outputs = 0, n_dofs = 0, n_regs = 0;
  std::vector<double> consts;
  std::vector<TInstr> instrs;
  std::vector<std::uint32_t> out_regs;

  std::uint32_t first_op_reg() const { return n_inputs + static_cast<std::uint32_t>(consts.size()); }
  std::string digest_hex() const {
    static const char* hx = "0123456789abcdef";
    std::string s;
    for (auto b : digest) { s += hx[b >> 4]; s += hx[b & 15]; }
    return s;
  }
};

class TapeError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {
struct Reader {
  const std::uint8_t* p;
  std::size_t n, off = 0;
  void need(std::size_t k) {
    if (off + k > n) throw TapeError("tape: truncated blob");
  }
  std::uint32_t u32() {
    need(4);
    std::uint32_t v = std::uint32_t(p[off]) | std::uint32_t(p[off + 1]) << 8 |
                      std::uint32_t(p[off + 2]) << 16 | std::uint32_t(p[off + 3]) << 24;
    off += 4;
    return v;
  }
  std::uint64_t u64() {
    std::uint64_t lo = u32();
    std::uint64_t hi = u32();
    return lo | hi << 32;
  }
  std::uint8_t u8() {
    need(1);
    return p[off++];
  }
};
}  // namespace detail

// Parses and validates a tape blob. Errors mirror Tape::load's checks (tape.hpp:247-291).
inline TapeIR parse_tape(const std::uint8_t* blob, std::size_t len) {
  if (!blob) throw TapeError("tape: null blob");
  detail::Reader r{blob, len};
  r.need(4);
  if (std::memcmp(blob, "SYTP", 4) != 0) throw TapeError("tape: bad magic");
  r.off = 4;
  if (r.u32() != 1) throw TapeError("tape: unsupported version");
  TapeIR t;
  r.need(32);
  std::memcpy(t.digest.data(), blob + r.off, 32);
  r.off += 32;
  t.n_inputs = r.u32();
  t.n_outputs = r.u32();
  t.n_dofs = r.u32();
  t.n_regs = r.u32();
  const std::uint64_t nc = r.u64();
  if (nc > (1ull << 32)) throw TapeError("tape: truncated header");
  t.consts.resize(nc);
  for (auto& v : t.consts) {
    const std::uint64_t bits = r.u64();
    std::memcpy(&v, &bits, 8);
  }
  const std::uint64_t ni = r.u64();
  if (ni > (1ull << 32)) throw TapeError("tape: truncated body");
  t.instrs.resize(ni);
  for (auto& in : t.instrs) {
    const std::uint8_t op = r.u8();
    if (op < 2 || op > 12) throw TapeError("tape: invalid opcode");
    in.op = static_cast<TOp>(op);
    in.iarg = static_cast<std::int32_t>(r.u32());
    in.dst = r.u32();
    in.a = r.u32();
    in.b = r.u32();
    in.c = r.u32();
  }
  const std::uint64_t no = r.u64();
  if (no > (1ull << 32)) throw TapeError("tape: truncated outputs");
  t.out_regs.resize(no);
  for (auto& o : t.out_regs) o = r.u32();
  if (t.n_outputs != t.out_regs.size()) throw TapeError("tape: inconsistent output count");
  // Structural checks: SSA, operands defined before use, registers in range.
  const std::uint32_t base = t.first_op_reg();
  for (std::size_t k = 0; k < t.instrs.size(); ++k) {
    const TInstr& in = t.instrs[k];
    if (in.dst != base + k) throw TapeError("tape: non-sequential destination register");
    const int ar = top_arity(in.op);
    const std::uint32_t ops[3] = {in.a, in.b, in.c};
    for (int q = 0; q < ar; ++q)
      if (ops[q] >= in.dst) throw TapeError("tape: operand register out of range");
  }
  if (t.n_regs != base + t.instrs.size()) throw TapeError("tape: register count mismatch");
  for (auto o : t.out_regs)
    if (o >= t.n_regs) throw TapeError("tape: output register out of range");
  return t;
}

}  // namespace symel_cuda
