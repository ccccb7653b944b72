// symel_cuda_assembler.hpp -- the reference-side half of the drop-in boundary.
//
// `symel::CudaAssembler` is a header-only adapter that a user of the reference includes next
// to the reference's own headers (/root/reference/proj/include/symel, unmodified). It takes
// the reference's `EnergySystem` + `KernelCache` exactly like `symel::Assembler`
// (assembly.hpp:90-187) and runs the hot path -- activation refresh, element evaluation,
// optional SPD projection, gradient + BCRS assembly, check_finite, pins -- in
// libsymel_cuda.so through the plain C ABI of include/symel_cuda.h. Nothing above the ABI
// changes: energies are still declared with EnergyBuilder and differentiated by the
// reference's own diff.hpp; their derivative / activation / guard kernels cross the ABI as the
// reference's Tape in its SYTP v1 wire format (tape.hpp:211-245), keyed by the reference's
// kernel_key digest (registry.hpp:415-428, stamped by KernelCache::get_or_build, cache.hpp:78).
//
// Same surface as symel::Assembler: assemble(), energy_only(), guard_min(), gradient(),
// hessian() (a reference BcrsMatrix, layout-identical: b, row_ptr, col_idx, values), energy(),
// active(i), active_count(i), timings(), reset_timings(). Errors are symel::Error with the
// reference's messages (check_finite: "energy 'NAME': non-finite derivative output at element
// N", assembly.hpp:426-438). There is no CPU fallback: without a device the constructor throws.
//
// Usage (the reference's flow; only the assembler type changes):
//   symel::EnergySystem sys;  ... add_dof_array / add_connectivity / add_solid_tet ...
//   symel::KernelCache cache(dir);
//   symel::CudaAssembler as(sys, cache);      // instead of symel::Assembler as(sys, cache, T, W)
//   double E = as.assemble();  const symel::BcrsMatrix& H = as.hessian();
// Link: -I<repo>/include -L<repo>/paper_2303_02156_b200 -lsymel_cuda
#pragma once

#include <algorithm>
#include <bit>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "symel/assembly.hpp"
#include "symel_cuda.h"

namespace symel {

// Tape::save's byte layout (tape.hpp:213-240), written to memory instead of a file.
inline std::vector<std::uint8_t> sytp_bytes(const Tape& t) {
  std::vector<std::uint8_t> b;
  auto u32 = [&](std::uint32_t v) {
    for (int i = 0; i < 4; ++i) b.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
  };
  auto u64 = [&](std::uint64_t v) {
    for (int i = 0; i < 8; ++i) b.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
  };
  b.insert(b.end(), {'S', 'Y', 'T', 'P'});
  u32(kTapeFormatVersion);
  b.insert(b.end(), t.digest.bytes.begin(), t.digest.bytes.end());
  u32(t.n_inputs);
  u32(t.n_outputs);
  u32(t.n_dofs);
  u32(t.n_regs);
  u64(t.consts.size());
  for (double v : t.consts) u64(std::bit_cast<std::uint64_t>(v));
  u64(t.instrs.size());
  for (const TapeInstr& i : t.instrs) {
    b.push_back(static_cast<std::uint8_t>(i.op));
    u32(static_cast<std::uint32_t>(i.iarg));
    u32(i.dst);
    u32(i.a);
    u32(i.b);
    u32(i.c);
  }
  u64(t.out_regs.size());
  for (std::uint32_t r : t.out_regs) u32(r);
  return b;
}

enum class CudaAssembleMode : std::uint32_t {
  deterministic = SYMEL_ASM_DETERMINISTIC,  // tile-ordered, atomic-free reduction (bitwise run to run)
  atomic = SYMEL_ASM_ATOMIC,                // red.global.add.f64 reduction
  ordered = SYMEL_ASM_ORDERED,              // tape-order IEEE eval + the reference's summation order
};

class CudaAssembler {
 public:
  CudaAssembler(EnergySystem& sys, KernelCache& cache, int device = 0,
                CudaAssembleMode mode = CudaAssembleMode::deterministic)
      : sys_(&sys), cache_(&cache), device_(device), mode_(mode) {
    create();
  }
  ~CudaAssembler() {
    if (ctx_) symel_cuda_destroy(ctx_);
  }
  CudaAssembler(const CudaAssembler&) = delete;
  CudaAssembler& operator=(const CudaAssembler&) = delete;

  EnergySystem& system() { return *sys_; }
  void set_mode(CudaAssembleMode m) { mode_ = m; }
  CudaAssembleMode mode() const { return mode_; }

  // Per-energy device options (SYMEL_ENERGY_SPD: per-element SPD projection of the element
  // Hessian; SYMEL_ENERGY_EXACT: the reference's rounding in every mode).
  void set_energy_flags(std::size_t energy, std::uint32_t flags) {
    if (flags_.size() <= energy) flags_.resize(energy + 1, 0);
    flags_[energy] = flags;
    if (energy < eid_.size()) check(symel_cuda_set_energy_flags(ctx_, eid_[energy], flags));
  }

  // Non-dof arrays are re-uploaded at every assemble by default (the reference reads every
  // array at gather time, registry.hpp:261-287, and assemble hooks may rewrite them); an array
  // marked constant is uploaded once per registration.
  void set_array_constant(ArrayHandle h, bool constant = true) { constant_[h.idx] = constant; }

  double assemble() {
    sys_->run_assemble_hooks();  // assembly.hpp:110
    prepare();
    double E = 0.0;
    symel_cuda_status st{};
    check(symel_cuda_assemble(ctx_, static_cast<std::uint32_t>(mode_), &E, &st));
    symel_cuda_timings t{};
    check(symel_cuda_get_timings(ctx_, &t));
    timings_.eval_ms += t.eval_ms;
    timings_.assemble_ms += t.assemble_ms;
    energy_ = E;
    have_grad_ = have_mat_ = false;
    return E;
  }

  // assembly.hpp:130-141: no hooks, no activation refresh; non-finite values are returned.
  double energy_only() {
    prepare();
    double E = 0.0;
    check(symel_cuda_energy_only(ctx_, &E));
    return E;
  }

  // assembly.hpp:143-173: minimum guard over all elements of guarded energies.
  double guard_min() {
    prepare();
    double g = 0.0;
    check(symel_cuda_guard_min(ctx_, &g));
    return g;
  }

  const std::vector<double>& gradient() {
    if (!have_grad_) {
      std::uint64_t nd = 0;
      check(symel_cuda_pattern_info(ctx_, nullptr, nullptr, nullptr, &nd));
      grad_.resize(nd);
      check(symel_cuda_copy_gradient(ctx_, grad_.data()));
      have_grad_ = true;
    }
    return grad_;
  }

  const BcrsMatrix& hessian() {
    if (!have_mat_) {
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
      have_mat_ = true;
    }
    return mat_;
  }

  double energy() const { return energy_; }

  const std::vector<std::uint8_t>& active(std::size_t energy_idx) {
    const std::size_t ne = sys_->n_elements(sys_->energy_at(energy_idx).conn);
    active_.assign(ne, 0);
    check(symel_cuda_copy_active(ctx_, eid_.at(energy_idx), active_.data()));
    return active_;
  }
  std::size_t active_count(std::size_t energy_idx) {
    std::uint64_t n = 0;
    check(symel_cuda_active_count(ctx_, eid_.at(energy_idx), &n));
    return n;
  }

  const AssembleTimings& timings() const { return timings_; }
  void reset_timings() { timings_ = AssembleTimings{}; }

  // The device context (for the device PCG, raw device results, cache statistics).
  symel_cuda_ctx* context() { return ctx_; }

 private:
  void check(int rc) const {
    if (rc != SYMEL_OK) throw Error(symel_cuda_last_error(ctx_));
  }

  void create() {
    if (const int rc = symel_cuda_create(device_, &ctx_); rc != SYMEL_OK) {
      ctx_ = nullptr;
      throw Error(std::string("CudaAssembler: ") + symel_cuda_last_error(nullptr));
    }
    // device kernels live beside the reference's own cache entries (cache.hpp:103-111)
    if (!cache_->dir().empty()) check(symel_cuda_set_cache_dir(ctx_, cache_->dir().string().c_str()));
  }

  // assembly.hpp:207-225 (prepare) + the registration the device needs: re-registers when the
  // topology stamp or the energy set changed; uploads state and params every call.
  void prepare() {
    if (sys_->topology_dirty()) sys_->refresh_topology();
    sys_->compile_kernels(*cache_);
    if (stamp_ != sys_->topology_stamp() || eid_.size() != sys_->n_energies()) register_system();
    for (const auto& [idx, id] : aid_) {
      const bool dof = dof_arrays_.count(idx) != 0;
      if (!dof && constant_[idx] && uploaded_once_.count(idx)) continue;
      const auto data = static_cast<const EnergySystem*>(sys_)->array_data(ArrayHandle{idx});
      check(symel_cuda_set_array(ctx_, id, data.data(), data.size()));
      uploaded_once_.insert(idx);
    }
    for (std::size_t d = 0; d < sys_->n_energies(); ++d) {
      const EnergyDef& def = sys_->energy_at(d);
      for (std::size_t k = 0; k < def.inputs.size(); ++k)
        if (def.inputs[k].kind == detail::InputKind::param)
          check(symel_cuda_set_param(ctx_, eid_[d], static_cast<std::uint32_t>(k), *def.inputs[k].host));
    }
    const std::vector<std::uint8_t>& mask = sys_->pinned();
    if (mask != pins_) {
      pins_ = mask;
      check(symel_cuda_set_pins(ctx_, pins_.data(), pins_.size()));
    }
  }

  // Connectivity of an energy, reconstructed through the reference's public API: the dof
  // binds of element e give its global dofs (element_dofs, registry.hpp:290-300), hence the
  // item of each tuple slot that binds a dof array. Slots read only by non-dof item inputs
  // cannot be recovered that way and are rejected.
  std::vector<std::int64_t> connectivity(const EnergyDef& def, std::uint32_t arity) const {
    const DofLayout& lay = sys_->layout();
    const std::size_t ne = sys_->n_elements(def.conn);
    std::vector<int> slot_bind(arity, -1);
    for (std::size_t k = 0; k < def.dof_binds.size(); ++k)
      if (slot_bind[def.dof_binds[k].tuple_slot] < 0) slot_bind[def.dof_binds[k].tuple_slot] = static_cast<int>(k);
    for (const detail::InputSrc& s : def.inputs)
      if (s.kind == detail::InputKind::item_comp && slot_bind[s.tuple_slot] < 0)
        throw Error("CudaAssembler: energy '" + def.name + "': tuple slot " + std::to_string(s.tuple_slot) +
                    " binds no dof array; its items cannot be recovered through the EnergySystem API");
    std::vector<std::int64_t> flat(ne * arity, 0);
    std::vector<std::size_t> dofs(def.n_dofs());
    for (std::size_t e = 0; e < ne; ++e) {
      sys_->element_dofs(def, e, dofs);
      for (std::uint32_t s = 0; s < arity; ++s) {
        const int k = slot_bind[s];
        if (k < 0) continue;
        const EnergyDef::DofBind& b = def.dof_binds[static_cast<std::size_t>(k)];
        const DofLayout::Set& set = lay.sets[sys_->dof_set_of_array(ArrayHandle{b.array})];
        flat[e * arity + s] = static_cast<std::int64_t>((dofs[static_cast<std::size_t>(k)] - set.offset - b.comp) / set.stride);
      }
    }
    return flat;
  }

  void register_system() {
    if (ctx_) symel_cuda_destroy(ctx_);
    ctx_ = nullptr;
    create();
    aid_.clear();
    eid_.clear();
    uploaded_once_.clear();
    pins_.clear();
    dof_arrays_.clear();
    // arrays: every dof array (they define the dof layout, in registration order,
    // registry.hpp:354-372) and every array an energy reads, in reference index order
    std::set<std::uint32_t> used;
    for (const DofLayout::Set& s : sys_->layout().sets) {
      used.insert(s.array);
      dof_arrays_.insert(s.array);
    }
    for (std::size_t d = 0; d < sys_->n_energies(); ++d)
      for (const detail::InputSrc& s : sys_->energy_at(d).inputs)
        if (s.kind == detail::InputKind::item_comp || s.kind == detail::InputKind::elem_comp) used.insert(s.array);
    for (std::uint32_t idx : used) {
      const ArrayHandle h{idx};
      int id = -1;
      check(symel_cuda_add_array(ctx_, sys_->array_name(h).c_str(), sys_->array_items(h), sys_->array_comps(h),
                                 dof_arrays_.count(idx) ? 1 : 0, &id));
      aid_[idx] = id;
    }
    // connectivities: one device connectivity per reference ConnHandle, arity = the largest
    // tuple slot any of its energies reads + 1
    std::map<std::uint32_t, std::uint32_t> arity;
    for (std::size_t d = 0; d < sys_->n_energies(); ++d) {
      const EnergyDef& def = sys_->energy_at(d);
      std::uint32_t a = 1;
      for (const detail::InputSrc& s : def.inputs)
        if (s.kind == detail::InputKind::item_comp) a = std::max(a, s.tuple_slot + 1);
      arity[def.conn.idx] = std::max(arity[def.conn.idx], a);
    }
    std::map<std::uint32_t, int> cid;
    for (std::size_t d = 0; d < sys_->n_energies(); ++d) {
      const EnergyDef& def = sys_->energy_at(d);
      if (cid.count(def.conn.idx)) continue;
      const std::uint32_t a = arity[def.conn.idx];
      const std::vector<std::int64_t> flat = connectivity(def, a);
      int id = -1;
      check(symel_cuda_add_connectivity(ctx_, ("conn" + std::to_string(def.conn.idx)).c_str(), a, &id));
      check(symel_cuda_set_elements(ctx_, id, flat.data(), flat.size() / a));
      cid[def.conn.idx] = id;
    }
    for (std::size_t d = 0; d < sys_->n_energies(); ++d) {
      const EnergyDef& def = sys_->energy_at(d);
      std::vector<symel_input_src> ins;
      for (const detail::InputSrc& s : def.inputs) {
        const bool arr = s.kind == detail::InputKind::item_comp || s.kind == detail::InputKind::elem_comp;
        ins.push_back({static_cast<std::uint32_t>(s.kind), arr ? static_cast<std::uint32_t>(aid_.at(s.array)) : 0u,
                       s.tuple_slot, s.comp});
      }
      std::vector<double> items;
      for (const auto& row : def.sum_items) items.insert(items.end(), row.begin(), row.end());
      const std::vector<std::uint8_t> deriv = sytp_bytes(def.deriv_kernel.tape());
      const std::vector<std::uint8_t> act =
          def.has_activation() ? sytp_bytes(def.act_kernel.tape()) : std::vector<std::uint8_t>{};
      const std::vector<std::uint8_t> grd =
          def.has_guard() ? sytp_bytes(def.guard_kernel.tape()) : std::vector<std::uint8_t>{};
      int id = -1;
      check(symel_cuda_add_energy(
          ctx_, def.name.c_str(), cid.at(def.conn.idx), deriv.data(), deriv.size(), ins.data(),
          static_cast<std::uint32_t>(ins.size()), def.dof_slots.data(), def.n_dofs(),
          def.is_sum ? items.data() : nullptr, def.is_sum ? static_cast<std::uint32_t>(def.sum_items.size()) : 0u,
          def.is_sum ? def.sum_arity : 0u, def.has_activation() ? act.data() : nullptr, act.size(),
          def.act_kind == CmpKind::ge ? 0 : 1, def.has_guard() ? grd.data() : nullptr, grd.size(), &id));
      eid_.push_back(id);
      if (d < flags_.size() && flags_[d]) check(symel_cuda_set_energy_flags(ctx_, id, flags_[d]));
    }
    stamp_ = sys_->topology_stamp();
  }

  EnergySystem* sys_;
  KernelCache* cache_;
  int device_;
  CudaAssembleMode mode_;
  symel_cuda_ctx* ctx_ = nullptr;
  std::uint64_t stamp_ = ~0ull;
  std::map<std::uint32_t, int> aid_;
  std::set<std::uint32_t> dof_arrays_, uploaded_once_;
  std::map<std::uint32_t, bool> constant_;
  std::vector<int> eid_;
  std::vector<std::uint32_t> flags_;
  std::vector<std::uint8_t> pins_, active_;
  std::vector<double> grad_;
  BcrsMatrix mat_;
  bool have_grad_ = false, have_mat_ = false;
  double energy_ = 0.0;
  AssembleTimings timings_;
};

}  // namespace symel
