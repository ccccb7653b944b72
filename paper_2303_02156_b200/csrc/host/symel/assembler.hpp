// Symbolic front end, part 6: the device Assembler. Same surface as the reference's
// `symel::Assembler` (/root/reference/proj/include/symel/assembly.hpp:90-187): assemble(),
// energy_only(), guard_min(), gradient(), hessian(), active_count(), timings() -- with the
// evaluation and assembly running in libsymel_cuda.so behind the C ABI (include/symel_cuda.h).
// There is no CPU fallback: constructing it without a CUDA device throws.
#pragma once

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "symel/system.hpp"
#include "symel_cuda.h"

namespace symel {

// BcrsMatrix (assembly.hpp:18-75): b x b blocks, row-major, columns sorted per block row.
struct BcrsMatrix {
  int b = 1;
  std::size_t n_block_rows = 0;
  std::vector<std::size_t> row_ptr, col_idx;
  std::vector<double> values;
  static constexpr std::size_t npos = static_cast<std::size_t>(-1);
  std::size_t n_blocks() const { return col_idx.size(); }
  std::size_t find_block(std::size_t r, std::size_t c) const {
    const auto first = col_idx.begin() + std::ptrdiff_t(row_ptr[r]), last = col_idx.begin() + std::ptrdiff_t(row_ptr[r + 1]);
    const auto it = std::lower_bound(first, last, c);
    return (it == last || *it != c) ? npos : std::size_t(it - col_idx.begin());
  }
  const double* block(std::size_t k) const { return values.data() + k * std::size_t(b) * std::size_t(b); }
};

enum class AssembleMode : std::uint32_t {
  deterministic = SYMEL_ASM_DETERMINISTIC,
  atomic = SYMEL_ASM_ATOMIC,
  ordered = SYMEL_ASM_ORDERED,
};

struct AssembleTimings {
  double eval_ms = 0.0, assemble_ms = 0.0;
};

class Assembler {
 public:
  explicit Assembler(EnergySystem& sys, int device = 0, AssembleMode mode = AssembleMode::deterministic)
      : sys_(&sys), device_(device), mode_(mode) {}
  ~Assembler() { release(); }
  Assembler(const Assembler&) = delete;
  Assembler& operator=(const Assembler&) = delete;

  // per-energy flags (SYMEL_ENERGY_SPD, SYMEL_ENERGY_EXACT), applied at registration
  void set_energy_flags(std::size_t energy, std::uint32_t flags) {
    if (flags_.size() <= energy) flags_.resize(energy + 1, 0);
    flags_[energy] = flags;
    if (ctx_) check(symel_cuda_set_energy_flags(ctx_, eid_.at(energy), flags));
  }

  double assemble() {
    prepare();
    double E = 0.0;
    symel_cuda_status st{};
    check(symel_cuda_assemble(ctx_, static_cast<std::uint32_t>(mode_), &E, &st));
    symel_cuda_timings t{};
    symel_cuda_get_timings(ctx_, &t);
    timings_.eval_ms += t.eval_ms;
    timings_.assemble_ms += t.assemble_ms;
    energy_ = E;
    return E;
  }
  double energy_only() {
    prepare();
    double E = 0.0;
    check(symel_cuda_energy_only(ctx_, &E));
    return E;
  }
  double guard_min() {
    prepare();
    double g = 0.0;
    check(symel_cuda_guard_min(ctx_, &g));
    return g;
  }

  const std::vector<double>& gradient() {
    std::uint64_t nd = 0;
    check(symel_cuda_pattern_info(ctx_, nullptr, nullptr, nullptr, &nd));
    grad_.resize(nd);
    check(symel_cuda_copy_gradient(ctx_, grad_.data()));
    return grad_;
  }
  const BcrsMatrix& hessian() {
    int b = 1;
    std::uint64_t nbr = 0, nb = 0;
    check(symel_cuda_pattern_info(ctx_, &b, &nbr, &nb, nullptr));
    std::vector<std::int64_t> rp(nbr + 1), ci(nb);
    check(symel_cuda_copy_pattern(ctx_, rp.data(), ci.data()));
    mat_.b = b;
    mat_.n_block_rows = nbr;
    mat_.row_ptr.assign(rp.begin(), rp.end());
    mat_.col_idx.assign(ci.begin(), ci.end());
    mat_.values.resize(nb * std::size_t(b) * std::size_t(b));
    check(symel_cuda_copy_hessian(ctx_, mat_.values.data()));
    return mat_;
  }
  double energy() const { return energy_; }
  std::size_t active_count(std::size_t energy) {
    std::uint64_t n = 0;
    check(symel_cuda_active_count(ctx_, eid_.at(energy), &n));
    return n;
  }
  const AssembleTimings& timings() const { return timings_; }
  void reset_timings() { timings_ = AssembleTimings{}; }
  symel_cuda_ctx* context() { return ctx_; }

 private:
  void check(int rc) const {
    if (rc != SYMEL_OK) throw Error(symel_cuda_last_error(ctx_));
  }
  void release() {
    if (ctx_) symel_cuda_destroy(ctx_);
    ctx_ = nullptr;
    eid_.clear();
    aid_.clear();
  }

  // (Re)registers the system when its topology changed; re-uploads dof arrays and params
  // every call (params are read at every assemble, registry.hpp:497-500).
  void prepare() {
    if (!ctx_ || sys_->topology_version() != version_) register_system();
    const auto& arrays = sys_->arrays();
    for (std::size_t i = 0; i < arrays.size(); ++i)
      if (arrays[i].is_dof) check(symel_cuda_set_array(ctx_, aid_[i], arrays[i].data.data(), arrays[i].data.size()));
    for (std::size_t d = 0; d < sys_->n_energies(); ++d) {
      const EnergyDef& def = sys_->energy_at(d);
      for (std::size_t k = 0; k < def.inputs.size(); ++k)
        if (def.inputs[k].kind == InputKind::param)
          check(symel_cuda_set_param(ctx_, eid_[d], static_cast<std::uint32_t>(k), *def.inputs[k].host));
    }
  }

  void register_system() {
    release();
    if (const int rc = symel_cuda_create(device_, &ctx_); rc != SYMEL_OK) {
      ctx_ = nullptr;
      throw Error(std::string("symel_cuda_create: ") + symel_cuda_last_error(nullptr));
    }
    if (const char* dir = std::getenv("SYMEL_CUDA_CACHE")) symel_cuda_set_cache_dir(ctx_, dir);
    sys_->compile_tapes();
    const auto& arrays = sys_->arrays();
    for (const auto& a : arrays) {
      int id = -1;
      check(symel_cuda_add_array(ctx_, a.name.c_str(), a.items, a.comps, a.is_dof ? 1 : 0, &id));
      check(symel_cuda_set_array(ctx_, id, a.data.data(), a.data.size()));
      aid_.push_back(id);
    }
    std::vector<int> cid;
    for (const auto& c : sys_->connectivities()) {
      int id = -1;
      check(symel_cuda_add_connectivity(ctx_, c.name.c_str(), c.arity, &id));
      check(symel_cuda_set_elements(ctx_, id, c.elems.data(), c.elems.size() / c.arity));
      cid.push_back(id);
    }
    for (std::size_t d = 0; d < sys_->n_energies(); ++d) {
      const EnergyDef& def = sys_->energy_at(d);
      std::vector<symel_input_src> ins;
      for (const InputSrc& s : def.inputs)
        ins.push_back({static_cast<std::uint32_t>(s.kind), static_cast<std::uint32_t>(aid_.at(s.array)), s.tuple_slot,
                       s.comp});
      std::vector<double> items;
      for (const auto& row : def.sum_items) items.insert(items.end(), row.begin(), row.end());
      const auto deriv = def.deriv->serialize();
      const std::vector<std::uint8_t> act = def.act ? def.act->serialize() : std::vector<std::uint8_t>{};
      const std::vector<std::uint8_t> grd = def.guard ? def.guard->serialize() : std::vector<std::uint8_t>{};
      int id = -1;
      check(symel_cuda_add_energy(ctx_, def.name.c_str(), cid.at(def.conn.idx), deriv.data(), deriv.size(), ins.data(),
                                  static_cast<std::uint32_t>(ins.size()), def.dof_slots.data(), def.n_dofs(),
                                  def.is_sum ? items.data() : nullptr,
                                  def.is_sum ? static_cast<std::uint32_t>(def.sum_items.size()) : 0u,
                                  def.is_sum ? def.sum_arity : 0u, def.act ? act.data() : nullptr, act.size(),
                                  def.act_kind == CmpKind::ge ? 0 : 1, def.guard ? grd.data() : nullptr, grd.size(), &id));
      eid_.push_back(id);
      if (d < flags_.size() && flags_[d]) check(symel_cuda_set_energy_flags(ctx_, id, flags_[d]));
    }
    if (sys_->has_pins()) {
      const auto mask = sys_->pinned_mask();
      check(symel_cuda_set_pins(ctx_, mask.data(), mask.size()));
    }
    version_ = sys_->topology_version();
  }

  EnergySystem* sys_;
  int device_;
  AssembleMode mode_;
  symel_cuda_ctx* ctx_ = nullptr;
  std::uint64_t version_ = ~0ull;
  std::vector<int> aid_, eid_;
  std::vector<std::uint32_t> flags_;
  std::vector<double> grad_;
  BcrsMatrix mat_;
  double energy_ = 0.0;
  AssembleTimings timings_;
};

}  // namespace symel
