// Symbolic front end, part 4: binding energies to state arrays and connectivity.
// Same user interface and input-slot rules as the reference's registry.hpp
// (/root/reference/proj/include/symel/registry.hpp): bind/bind_element/param/sum_items append
// kernel inputs in call order (registry.hpp:577-594); dof arrays are concatenated into the
// global dof layout in registration order (registry.hpp:354-372); the kernel cache key is the
// SHA-256 over (domain, n_inputs, n_dofs, dof slots, DAG) (registry.hpp:415-428) and is stored
// as the tape digest, so tapes match the reference's byte for byte.
#pragma once

#include <cstdint>
#include <cstdio>
#include <functional>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "symel/tape.hpp"

namespace symel {

struct ArrayHandle {
  std::uint32_t idx = ~0u;
  bool valid() const { return idx != ~0u; }
};
struct ConnHandle {
  std::uint32_t idx = ~0u;
  bool valid() const { return idx != ~0u; }
};
struct EnergyHandle {
  std::uint32_t idx = ~0u;
  bool valid() const { return idx != ~0u; }
};

enum class InputKind : std::uint8_t { item_comp, elem_comp, param, sum_comp };

struct InputSrc {
  InputKind kind = InputKind::item_comp;
  std::uint32_t array = 0, tuple_slot = 0, comp = 0;
  const double* host = nullptr;  // param: read at every assemble
};

struct EnergyDef {
  std::string name;
  ConnHandle conn;
  std::unique_ptr<ExprGraph> graph;
  std::vector<InputSrc> inputs;
  std::vector<std::uint32_t> dof_slots;
  std::vector<NodeId> dof_syms;
  NodeId energy_root = kInvalidNode, act_root = kInvalidNode, guard_root = kInvalidNode;
  CmpKind act_kind = CmpKind::ge;
  std::vector<std::vector<double>> sum_items;
  std::uint32_t sum_arity = 0;
  bool is_sum = false;
  std::optional<Tape> deriv, act, guard;  // built by EnergySystem::compile_tapes

  std::uint32_t n_inputs() const { return static_cast<std::uint32_t>(inputs.size()); }
  std::uint32_t n_dofs() const { return static_cast<std::uint32_t>(dof_slots.size()); }
  bool has_activation() const { return act_root != kInvalidNode; }
  bool has_guard() const { return guard_root != kInvalidNode; }
};

class EnergyBuilder;

class EnergySystem {
 public:
  struct ArrayDef {
    std::string name;
    std::size_t items = 0;
    std::uint32_t comps = 0;
    bool is_dof = false;
    std::vector<double> data;
  };
  struct ConnDef {
    std::string name;
    std::uint32_t arity = 0;
    std::vector<std::int64_t> elems;
  };

  EnergySystem() = default;
  EnergySystem(const EnergySystem&) = delete;
  EnergySystem& operator=(const EnergySystem&) = delete;

  ArrayHandle add_array(std::string name, std::size_t items, std::uint32_t comps) {
    return new_array(std::move(name), items, comps, false);
  }
  ArrayHandle add_dof_array(std::string name, std::size_t items, std::uint32_t comps) {
    return new_array(std::move(name), items, comps, true);
  }
  ConnHandle add_connectivity(std::string name, std::uint32_t arity) {
    if (arity == 0) throw Error("connectivity '" + name + "': arity must be positive");
    conns_.push_back({std::move(name), arity, {}});
    ++topology_version_;
    return {static_cast<std::uint32_t>(conns_.size() - 1)};
  }
  void set_elements(ConnHandle h, std::vector<std::int64_t> flat) {
    ConnDef& c = conn_at(h);
    if (flat.size() % c.arity != 0) throw Error("connectivity '" + c.name + "': element list not a multiple of arity");
    c.elems = std::move(flat);
    ++topology_version_;
  }
  std::size_t n_elements(ConnHandle h) const { return conn_at(h).elems.size() / conn_at(h).arity; }

  std::span<double> array_data(ArrayHandle h) { return array_at(h).data; }
  std::span<const double> array_data(ArrayHandle h) const { return array_at(h).data; }

  EnergyHandle add_energy(std::string name, ConnHandle conn, const std::function<void(EnergyBuilder&)>& define);

  std::size_t n_energies() const { return energies_.size(); }
  const EnergyDef& energy(EnergyHandle h) const { return *energies_.at(h.idx); }
  const EnergyDef& energy_at(std::size_t i) const { return *energies_.at(i); }
  EnergyDef& energy_at_mut(std::size_t i) { return *energies_.at(i); }
  const std::vector<ArrayDef>& arrays() const { return arrays_; }
  const std::vector<ConnDef>& connectivities() const { return conns_; }
  const ArrayDef& array_at(ArrayHandle h) const {
    if (h.idx >= arrays_.size()) throw Error("invalid array handle");
    return arrays_[h.idx];
  }
  const ConnDef& conn_at(ConnHandle h) const {
    if (h.idx >= conns_.size()) throw Error("invalid connectivity handle");
    return conns_[h.idx];
  }
  std::uint64_t topology_version() const { return topology_version_; }

  // pins (registry.hpp:175-191): mask over the global dof layout
  void pin(ArrayHandle h, std::size_t item) {
    for (std::uint32_t c = 0; c < array_at(h).comps; ++c) pin(h, item, c);
  }
  void pin(ArrayHandle h, std::size_t item, std::uint32_t comp) {
    const ArrayDef& a = array_at(h);
    if (!a.is_dof) throw Error("pin: array '" + a.name + "' is not a dof array");
    if (item >= a.items || comp >= a.comps) throw Error("pin: index out of range in array '" + a.name + "'");
    pins_.emplace_back(h.idx, item, comp);
  }
  void clear_pins() { pins_.clear(); }
  std::vector<std::uint8_t> pinned_mask() const {
    std::vector<std::size_t> off(arrays_.size(), 0);
    std::size_t n = 0;
    for (std::size_t i = 0; i < arrays_.size(); ++i)
      if (arrays_[i].is_dof) {
        off[i] = n;
        n += arrays_[i].items * arrays_[i].comps;
      }
    std::vector<std::uint8_t> m(n, 0);
    for (auto [a, item, comp] : pins_) m[off[a] + item * arrays_[a].comps + comp] = 1;
    return m;
  }
  bool has_pins() const { return !pins_.empty(); }

  // Differentiates and lowers every energy (E/g/H, activation and guard kernels).
  void compile_tapes();
  std::uint64_t differentiation_count() const { return diff_count_; }

  ExprDigest kernel_key(const EnergyDef& d, const char* domain, std::span<const NodeId> roots) const {
    detail::Sha256 h;
    static constexpr char tag[] = "symel-kernel-key-v1";
    h.update(tag, sizeof(tag) - 1);
    h.update(domain, std::char_traits<char>::length(domain));
    const std::uint32_t ni = d.n_inputs(), nd = d.n_dofs();
    h.update(&ni, 4);
    h.update(&nd, 4);
    for (std::uint32_t s : d.dof_slots) h.update(&s, 4);
    d.graph->digest_update(h, roots);
    return ExprDigest{h.finish()};
  }

  void warn(const std::string& m) const { std::fprintf(stderr, "[symel] warning: %s\n", m.c_str()); }

 private:
  friend class EnergyBuilder;
  ArrayHandle new_array(std::string name, std::size_t items, std::uint32_t comps, bool dof) {
    if (comps == 0) throw Error("array '" + name + "': component count must be positive");
    for (const ArrayDef& a : arrays_)
      if (a.name == name) throw Error("array '" + name + "' already registered");
    arrays_.push_back({std::move(name), items, comps, dof, std::vector<double>(items * comps, 0.0)});
    ++topology_version_;
    return {static_cast<std::uint32_t>(arrays_.size() - 1)};
  }
  ArrayDef& array_at(ArrayHandle h) {
    if (h.idx >= arrays_.size()) throw Error("invalid array handle");
    return arrays_[h.idx];
  }
  ConnDef& conn_at(ConnHandle h) {
    if (h.idx >= conns_.size()) throw Error("invalid connectivity handle");
    return conns_[h.idx];
  }

  std::vector<ArrayDef> arrays_;
  std::vector<ConnDef> conns_;
  std::vector<std::unique_ptr<EnergyDef>> energies_;
  std::vector<std::tuple<std::uint32_t, std::size_t, std::uint32_t>> pins_;
  std::uint64_t topology_version_ = 0, diff_count_ = 0;
};

class EnergyBuilder {
 public:
  ExprGraph& graph() { return *def_->graph; }

  // Components of the item at connectivity slot `tuple_slot` (dofs when the array is a dof array).
  Vector bind(ArrayHandle array, std::uint32_t tuple_slot) {
    const auto& a = sys_->array_at(array);
    const auto& c = sys_->conn_at(def_->conn);
    if (tuple_slot >= c.arity)
      throw Error("energy '" + def_->name + "': tuple slot " + std::to_string(tuple_slot) +
                  " outside connectivity arity " + std::to_string(c.arity));
    Vector v(*def_->graph);
    for (std::uint32_t k = 0; k < a.comps; ++k)
      v.push_back(input(InputKind::item_comp, array.idx, tuple_slot, k, nullptr, a.is_dof,
                        a.name + "[" + std::to_string(tuple_slot) + "]." + std::to_string(k)));
    return v;
  }
  Scalar bind_scalar(ArrayHandle array, std::uint32_t tuple_slot) {
    if (sys_->array_at(array).comps != 1) throw Error("bind_scalar: array has more than one component");
    return bind(array, tuple_slot)[0];
  }
  // Row `elem` of a per-element array.
  Vector bind_element(ArrayHandle array) {
    const auto& a = sys_->array_at(array);
    if (a.is_dof) throw Error("bind_element: dof array '" + a.name + "' not allowed");
    Vector v(*def_->graph);
    for (std::uint32_t k = 0; k < a.comps; ++k)
      v.push_back(input(InputKind::elem_comp, array.idx, 0, k, nullptr, false, a.name + "[elem]." + std::to_string(k)));
    return v;
  }
  Scalar bind_element_scalar(ArrayHandle array) {
    if (sys_->array_at(array).comps != 1) throw Error("bind_element_scalar: array has more than one component");
    return bind_element(array)[0];
  }
  // Runtime scalar read at every assemble; changing it never rebuilds a kernel.
  Scalar param(const double& host, std::string name = "param") {
    return input(InputKind::param, 0, 0, 0, &host, false, std::move(name));
  }
  Scalar param(const double&& host, std::string name = "param") = delete;
  Scalar constant(double v) { return def_->graph->constant(v); }

  // Fixed summation: fn is built once over symbolic item components; the kernel runs per row
  // of `items` and results accumulate left to right.
  Scalar sum_items(const std::vector<std::vector<double>>& items, const std::function<Scalar(const Vector&)>& fn) {
    if (def_->is_sum) throw Error("sum_items: already used for energy '" + def_->name + "'");
    std::uint32_t arity = 0;
    if (!items.empty()) {
      arity = static_cast<std::uint32_t>(items[0].size());
      if (arity == 0) throw Error("sum_items: empty item tuples");
      for (const auto& r : items)
        if (r.size() != arity) throw Error("sum_items: ragged item table");
    } else {
      sys_->warn("energy '" + def_->name + "': fixed summation over zero items, contributes 0");
    }
    def_->is_sum = true;
    def_->sum_items = items;
    def_->sum_arity = arity;
    if (items.empty()) {
      sum_root_ = def_->graph->constant_id(0.0);
      return {*def_->graph, sum_root_};
    }
    Vector item(*def_->graph);
    for (std::uint32_t k = 0; k < arity; ++k)
      item.push_back(input(InputKind::sum_comp, 0, k, 0, nullptr, false, "sum_item." + std::to_string(k)));
    const Scalar body = fn(item);
    if (&body.graph() != def_->graph.get()) throw Error("sum_items: body built on a foreign graph");
    sum_root_ = body.id();
    return body;
  }
  void set(const Scalar& e) {
    if (def_->energy_root != kInvalidNode) throw Error("energy '" + def_->name + "': set() called twice");
    if (&e.graph() != def_->graph.get()) throw Error("energy '" + def_->name + "': expression from a foreign graph");
    if (def_->is_sum && e.id() != sum_root_)
      throw Error("energy '" + def_->name + "': with sum_items the summed expression must be set unchanged");
    def_->energy_root = e.id();
  }
  void set(const Scalar& e, const Condition& activation) {
    set(e);
    def_->act_root = activation.value.id();
    def_->act_kind = activation.kind;
  }
  void set_guard(const Scalar& g) {
    if (def_->guard_root != kInvalidNode) throw Error("energy '" + def_->name + "': set_guard() called twice");
    def_->guard_root = g.id();
  }

 private:
  friend class EnergySystem;
  EnergyBuilder(EnergySystem& s, EnergyDef& d) : sys_(&s), def_(&d) {}
  Scalar input(InputKind kind, std::uint32_t array, std::uint32_t slot, std::uint32_t comp, const double* host,
               bool dof, std::string name) {
    const int k = static_cast<int>(def_->inputs.size());
    def_->inputs.push_back({kind, array, slot, comp, host});
    Scalar s = def_->graph->symbol(std::move(name), k);
    if (dof) {
      def_->dof_slots.push_back(static_cast<std::uint32_t>(k));
      def_->dof_syms.push_back(s.id());
    }
    return s;
  }
  EnergySystem* sys_;
  EnergyDef* def_;
  NodeId sum_root_ = kInvalidNode;
};

inline EnergyHandle EnergySystem::add_energy(std::string name, ConnHandle conn,
                                             const std::function<void(EnergyBuilder&)>& define) {
  conn_at(conn);
  for (const auto& d : energies_)
    if (d->name == name) throw Error("energy '" + name + "' already registered");
  auto d = std::make_unique<EnergyDef>();
  d->name = std::move(name);
  d->conn = conn;
  d->graph = std::make_unique<ExprGraph>();
  EnergyBuilder b(*this, *d);
  define(b);
  if (d->energy_root == kInvalidNode) throw Error("energy '" + d->name + "': definition did not call set()");
  energies_.push_back(std::move(d));
  ++topology_version_;
  return {static_cast<std::uint32_t>(energies_.size() - 1)};
}

inline void EnergySystem::compile_tapes() {
  for (auto& dp : energies_) {
    EnergyDef& d = *dp;
    ExprGraph& g = *d.graph;
    if (!d.deriv) {
      ++diff_count_;
      const NodeId root[1] = {d.energy_root};
      const DerivativeBundle b = gradient_hessian(g, d.energy_root, d.dof_syms);
      const auto outs = b.output_roots();
      Tape t = lower(g, compress(g, outs), d.n_inputs(), d.n_dofs());
      t.digest = kernel_key(d, "deriv", root);
      d.deriv = std::move(t);
    }
    if (d.has_activation() && !d.act) {
      const NodeId root[1] = {d.act_root};
      Tape t = lower(g, compress(g, root), d.n_inputs(), d.n_dofs());
      t.digest = kernel_key(d, "act", root);
      d.act = std::move(t);
    }
    if (d.has_guard() && !d.guard) {
      const NodeId root[1] = {d.guard_root};
      Tape t = lower(g, compress(g, root), d.n_inputs(), d.n_dofs());
      t.digest = kernel_key(d, "guard", root);
      d.guard = std::move(t);
    }
  }
}

}  // namespace symel
