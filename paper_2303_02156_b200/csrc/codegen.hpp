// CUDA backend of the code generator: emits one specialised sm_100a kernel per energy tape.
//
// Replaces the reference's C++ emitter (`emit_kernel_source`, kernel.hpp:47-97) for the
// device: the same Tape IR is lowered to a thread-per-element kernel whose gather
// (registry.hpp:261-287 `gather_element_inputs`) is specialised on the input binding, whose
// instruction order is rescheduled for register pressure, and whose outputs are either
// stored in the reference's per-element layout (`contrib_`, assembly.hpp:377-424) or fused
// straight into the assembly (gradient + 3x3 BSR).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "tape_io.hpp"

namespace symel_cuda {

inline constexpr int kMaxArrays = 24;
inline constexpr int kMaxParams = 32;

// detail::InputKind (registry.hpp:54-59)
enum class InKind : std::uint32_t { item_comp = 0, elem_comp = 1, param = 2, sum_comp = 3 };

struct InputBinding {
  InKind kind = InKind::item_comp;
  std::uint32_t array = 0;       // array id (item_comp / elem_comp)
  std::uint32_t tuple_slot = 0;  // connectivity slot (item_comp) / item column (sum_comp)
  std::uint32_t comp = 0;
};

enum class OutMode : std::uint32_t {
  contrib = 0,   // reference layout [E, g(n), H(n*n)] per active element (exact order path)
  fused_atomic,  // E per element; g and BSR via red.global.add.f64 (nondeterministic order)
  fused_tile,    // E per element; g / BSR entries to per-element staging for the tile reducer
  fused_tile_spd,  // tile kernel on a factorize_spd tape: in-register m x m eigen-clamp, then
                   // H = W^T clamp(M) W staged for the tile reducer (K2 fused with K1 + K3)
  value_only,    // activation / guard kernels: single output per element (+ item reduction)
};

struct KernelSpec {
  const TapeIR* tape = nullptr;
  std::vector<InputBinding> inputs;      // one per tape input slot
  std::vector<std::uint32_t> dof_slots;  // input slots that are dofs, bind order
  std::vector<std::uint32_t> array_comps;  // comps per array id
  std::uint32_t arity = 1;
  std::vector<double> sum_items;         // n_items x sum_arity, row-major (fixed summation)
  std::uint32_t n_items = 0, sum_arity = 0;
  std::uint32_t b = 3;                   // BSR block size (assembly.hpp:273-276)
  OutMode mode = OutMode::contrib;
  bool fast = true;        // division strength reduction + FMA contraction
  std::uint32_t spd_m = 0; // fused_tile_spd: size m of the reduced eigenproblem
  bool spd_lookahead = true;  // fused_tile_spd: QL with per-lane level lookahead (sy_ql_la)
  bool stage_global = false;  // tile modes: stage element outputs in global memory (large elements)
  int item_lanes = 1;         // tile mode with fixed summation: the n_items terms of an element
                              // run on adjacent lanes (one term each) and are summed in order
                              // with shuffles; elements per tile = threads_per_block / item_lanes
  bool soa_prefetch = true; // tile modes: bulk L2 prefetch of the tile's SoA component rows
  bool bulk_plan = true;   // tile modes: plan slice to shared memory by bulk (TMA) copies + mbarrier
  bool conn_soa = false;  // tile modes: item indices from the tile-ordered connectivity copy
  // tile modes: per SoA array, component -> row of the (deduplicated) SoA copy, -1 = the
  // component is +0.0 in every element (no load); empty = identity (row == component)
  std::vector<std::vector<int>> soa_rows;
  std::vector<std::uint8_t> soa_arrays;  // tile modes: per array, 1 = elem_comp inputs read
                                         // from a tile-ordered SoA copy a.arr[i][c * soa_n + t]
  int meta_depth_h = 1;       // tile reduction: segments' metadata loaded this many rounds ahead
  int meta_depth_g = 1;       // (Hessian / gradient segments; registers across the barrier)
  bool plan_global = false;   // tile modes: read the plan slice from global memory (L2) instead of
                              // prefetching it to shared memory (keeps two CTAs per SM)
  int value_reduce = 0;    // value_only over items: 1 = max (activation), 2 = min/NaN->-inf (guard)
  int schedule = 1;        // 0 = tape order, 1 = output-driven DFS, 2 = DFS with column-major
                           // Hessian, 3/4/5 = greedy min-live list schedule with ties broken
                           // by the 1/2/0 order, -1 = auto (min peak live)
  int threads_per_block = 128;
  int min_blocks = 2;
  std::string name = "sy_kernel";
};

// Derived facts about the element's dof -> block mapping (fused modes).
struct BlockMap {
  std::uint32_t n_lb = 0;                 // local blocks per element
  std::vector<std::uint32_t> lb_of_dof;   // per dof (bind order)
  std::vector<std::uint32_t> entry_of_dof;
  std::vector<std::uint32_t> lb_array, lb_slot, lb_comp0;  // per local block: source item
};

BlockMap make_block_map(const KernelSpec& spec);

// Shared declarations (argument struct) prepended to every generated kernel and used by
// the host launcher; layout must stay identical on both sides.
const char* kernel_prelude();

std::string emit_kernel(const KernelSpec& spec);

// Instruction order used for emission (indices into tape->instrs).
// Device-source fragment of the fused SPD projection (also compiled on the host by
// tests/test_spd_clamp.py).
const char* eig_source();

std::vector<std::uint32_t> schedule_instrs(const TapeIR& t, int schedule);
int pick_schedule(const TapeIR& t);  // schedule with the lowest peak of live values
// Peak number of simultaneously live values of an instruction order (inputs live from first use).
std::size_t max_live(const TapeIR& t, const std::vector<std::uint32_t>& order);

}  // namespace symel_cuda
