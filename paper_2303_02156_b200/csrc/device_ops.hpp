// Host-callable wrappers around the static sm_100a kernels in assembly_kernels.cu.
// All functions enqueue on `stream` and return cudaError_t as int (0 = success).
#pragma once

#include <cstddef>
#include <cstdint>

namespace symel_cuda::dev {

inline constexpr int kMaxLb = 32;  // local blocks per element (tet10: 10, pairs: 4)

// Local block descriptors of one energy (see codegen BlockMap): block of an element's local
// block q = (set_off[array[q]] + item * comps[array[q]] + comp0[q]) / b, item = conn[slot[q]].
struct LbDesc {
  int n_lb;
  int b;
  int arity;
  int slot[kMaxLb];
  long long off[kMaxLb];    // set offset + comp0 of the owning dof array
  int comps[kMaxLb];
};

// --- pattern (replaces build_pattern, assembly.hpp:271-375) ---------------------------
// Emits 64-bit keys (row << 32 | col) for every off-diagonal local block pair of every active
// element; returns the count written at keys + *n_out (device counter).
int pattern_keys(const LbDesc& d, const int* conn, const int* active, long long n_active,
                 unsigned long long* keys, unsigned long long* counter, void* stream);
int diag_keys(long long n_rows, unsigned long long* keys, void* stream);
// Sorts + uniques keys in place; builds row_ptr (n_rows+1) / col_idx; returns n_blocks.
int build_csr(unsigned long long* keys, long long n_keys, long long n_rows, int** row_ptr,
              int** col_idx, long long* n_blocks, void* stream);
// Slot map: per active element, n_lb*n_lb block ordinals (row-major over local blocks).
int slot_map(const LbDesc& d, const int* conn, const int* active, long long n_active,
             const int* row_ptr, const int* col_idx, int* slots, void* stream);

// --- ordered (reference-order) scatter, assembly.hpp:327-374 + 450-462 -----------------
// Builds per-block and per-row contribution lists in ascending (energy, element, a, c) order.
struct OrderedRefs {
  long long n_hess = 0, n_grad = 0;
  int* hess_ptr = nullptr;             // n_blocks + 1
  unsigned long long* hess_ref = nullptr;  // (contrib element ordinal << 10) | (li << 5) | lj
  int* grad_ptr = nullptr;             // n_rows + 1
  unsigned long long* grad_ref = nullptr;  // (contrib element ordinal << 5) | li
};
struct EnergyRefSrc {
  const int* slots;      // per active element n_lb^2
  const int* conn;
  const int* active;
  long long n_active;
  long long ord_base;    // first global contrib ordinal of this energy
  LbDesc d;
};
int ordered_refs(const EnergyRefSrc* src, int n_energies, long long n_blocks, long long n_rows,
                 OrderedRefs* out, void* stream);
void free_ordered_refs(OrderedRefs* r);

// Per energy: contrib row stride and the (lb, entry) -> dof index table (-1 = absent).
struct ContribLayout {
  long long ord_base;  // first element ordinal (global over energies) of the energy
  long long ord_end;
  const double* contrib;  // this energy's contrib block (stride doubles per element)
  int stride;
  int n_dofs;
  int n_lb;
  int b;
  signed char dof_of[kMaxLb * 3];
};
int ordered_scatter(const ContribLayout* lay, int n_energies, const OrderedRefs& r, long long n_blocks,
                    long long n_rows, double* vals, double* grad, void* stream);

// --- energy and finiteness (assembly.hpp:426-448) ---------------------------------------
// serial sum in (energy, element) order -- exact reference order, one thread
int energy_serial(const double* const* elemE, const long long* strides, const long long* counts,
                  int n_energies, double* out, void* stream);
// deterministic fixed-shape tree sum of n values (strided)
int energy_tree(const double* v, long long stride, long long n, double* partial, double* out, void* stream);
long long energy_tree_partials(long long n);
int energy_tree_launches(long long n);  // kernels energy_tree enqueues for n values
// combine per-energy totals in energy order (out = ((0 + e0) + e1) + ...)
int energy_combine(const double* per_energy, int n, double* out, void* stream);

// --- activation / guard (assembly.hpp:143-173, 227-261) ---------------------------------
int activation_mask(const double* v, long long n, int kind, unsigned char* mask, int* changed,
                    void* stream);
int compact_active(const unsigned char* mask, long long n, int* active, long long* n_active_host,
                   void* stream);
int min_reduce(const double* v, long long n, double* out, void* stream);

// --- SPD projection (K2): in place on contrib rows [E, g(n), H(n*n)], n in {3, 6, 9, 12}
int spd_project_contrib(double* contrib, long long stride, int n_dofs, long long n_elem, void* stream);
// per-element red.add scatter of contrib rows into g and the BSR (node-major dof binding)
int scatter_atomic_contrib(const double* contrib, long long stride, int n_dofs, const LbDesc& d, const int* slots,
                           const int* conn, const int* active, long long n, double* vals, double* grad, void* stream);

// --- measurement: FP64 DFMA throughput (TFLOP/s, FMA = 2 flops) over the whole device
int fp64_peak(int n_sm, double* tflops, void* stream);

// --- pins (assembly.hpp:464-489) -----------------------------------------------------------
int apply_pins(const unsigned char* mask, long long n_rows, int b, const int* row_ptr, const int* col_idx,
               double* vals, double* grad, void* stream);

// --- tile-ordered reduction (K3) ------------------------------------------------------------
// A tile = `tpb` consecutive active elements of one energy (one CTA of the tile kernel); tiles
// are numbered globally in (energy, element) order. For every (tile, BSR block) pair that
// receives contributions ("segment") the plan lists them in element order; a block touched by
// a single tile is written directly, otherwise each tile writes a partial and the fix-up adds
// the partials of the block in tile order. Same for gradient block rows.
struct TileSrc {
  const int* slots;  // per active element n_lb^2 block ordinals
  const int* conn;
  const int* active;
  const int* perm;   // tile position -> active ordinal (nullptr: identity)
  long long n_active;
  long long tile_base;
  int tpb;
  int h0;            // first Hessian staging slot (1 + n_dofs); staging slot k of element tl
                     // lives at shared double k * tpb + tl (codegen.cpp tile layout)
  int sort_segments; // order the tile's segments by contribution count (shared-memory staging)
  LbDesc d;
};
// A contribution is 16 bits (tpb = 128): Hessian (transpose << 15) | (sub(lo, hi) << 7) | tl,
// gradient (lb << 7) | tl, with tl the element's position in its tile and sub the index of the
// staged upper local-block pair (the kernel turns them into staging offsets).
// Spatially coherent tile order: active ordinals sorted by the Morton code of the element
// centroid (position arrays = the dof arrays of the local blocks, first 3 components, given
// per local block in `arrs`); also returns element ids in that order.
int tile_order(const LbDesc& d, const double* const* arrs_host, const int* conn, const int* active, long long n,
               int* perm, int* elems, void* stream);
struct SegPlan {  // one of {Hessian blocks, gradient rows}
  long long n_seg = 0, n_con = 0, n_partials = 0, n_pt = 0, n_untouched = 0;
  int* tile_seg_ptr = nullptr;  // n_tiles + 1
  int* tile_con_ptr = nullptr;  // n_tiles + 1: first contribution of each tile
  int* seg_target = nullptr;    // block (or row) ordinal per segment
  int* seg_mirror = nullptr;    // Hessian: transposed block (== target on the diagonal)
  int* seg_con_ptr = nullptr;   // n_seg + 1
  unsigned short* seg_rel = nullptr;  // n_seg: first contribution relative to its tile's
  unsigned short* con = nullptr;  // shared-memory offsets of the contributions (see TileSrc)
  int max_tile_seg = 0, max_tile_con = 0;  // per-tile maxima (shared-memory sizing)
  int* seg_dst = nullptr;       // >= 0 final target; < 0: -(partial index) - 1
  int* pt_ptr = nullptr;        // per partial target: range of its partials (tile order), n_pt + 1
  int* pt_target = nullptr;
  int* pt_mirror = nullptr;     // Hessian: transposed block of each partial target
  int* untouched = nullptr;     // targets without any contribution (zeroed every assemble)
};
struct TilePlan {
  long long n_tiles = 0;
  SegPlan h, g;
};
int build_tile_plan(const TileSrc* src, int n_energies, long long n_blocks, long long n_rows, const int* row_ptr,
                    const int* col_idx, TilePlan* out, void* stream);
void free_tile_plan(TilePlan* p);
// vals/grad for partial targets and untouched targets; deterministic (fixed order)
// which: 1 = Hessian targets, 2 = gradient rows, 3 = both
int tile_fixup(const TilePlan& p, const double* partials, const double* gpartials, int b, double* vals,
               double* grad, void* stream, int which = 3);
// Tile-ordered SoA copy of a per-element array: dst[c * stride + pos] = src[elem(pos) * comps + c],
// elem(pos) = map[pos] (map == nullptr: identity), pos < n.
// Tile-ordered, slot-major copy of an energy's connectivity (the tile kernels read their
// elements' item indices with one coalesced load per slot instead of active -> conn -> item).
int conn_soa(const int* conn, int arity, const int* map, long long n, int* dst, void* stream);
int soa_gather(const double* src, int comps, const int* map, long long n, long long stride, double* dst,
               void* stream);
// the same for a subset of component rows (device list `rows`, n_rows entries)
int soa_gather_rows(const double* src, int comps, const int* rows, int n_rows, const int* map, long long n,
                    long long stride, double* dst, void* stream);
// Component classes of a per-item array (items x comps): cls[c] = -1 when every item holds +0.0
// in component c, else the smallest component whose column is bit-for-bit identical (c itself
// when unique). Exact (hash grouping verified element by element). Host-synchronous.
int comp_classes(const double* src, int comps, long long items, int* cls, void* stream);
// fixed-order sum of per-tile energies [first, first + n) into *out
int tile_energy(const double* tileE, long long first, long long n, double* partial, double* out, void* stream);

}  // namespace symel_cuda::dev
