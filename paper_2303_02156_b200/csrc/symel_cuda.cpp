// libsymel_cuda.so: implementation of the C ABI in include/symel_cuda.h.
//
// Device-side replacement for the body of Assembler::assemble (assembly.hpp:108-126):
// prepare/compile (registry.hpp:620-653) -> NVRTC-compiled sm_100a kernels generated from the
// reference's Tape IR; refresh_activation + build_pattern -> device kernels; evaluate_active +
// check_finite + sum_energy + scatter + apply_pins -> device kernels. No CPU fallback: without
// a CUDA device every compute entry point fails with SYMEL_E_NODEVICE.
#include "../../include/symel_cuda.h"

#include <cuda_runtime.h>
#include <nvrtc.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <optional>

#include "codegen.hpp"
#include "factorize.hpp"
#include "device_ops.hpp"
#include "solver_ops.hpp"
#include "sy_args.h"
#include "tape_io.hpp"

using namespace symel_cuda;

namespace {

struct Fail {
  int code;
  std::string msg;
};

#define CK(expr)                                                                            \
  do {                                                                                      \
    cudaError_t e_ = (cudaError_t)(expr);                                                   \
    if (e_ != cudaSuccess) throw Fail{SYMEL_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

std::uint64_t fnv1a(const std::string& s) {
  std::uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

struct Compiled {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kernel = nullptr;
  int tpb = 128;
  int elems = 128;            // elements per CTA (tile kernels with item lanes: tpb / n_items)
  std::size_t smem = 0;       // dynamic shared memory per CTA (tile kernel: staging part)
  std::size_t smem_attr = 0;  // last MaxDynamicSharedMemorySize set on the kernel
  std::string source;
};

// Elements per tile = threads per CTA of the tile kernel (one element per thread).
// Threads per tile CTA: 128 with two CTAs per SM; 96 with three for the item-lane energies whose
// staging lives in global memory (tet10: no shared-memory limit, so nine warps per SM at 224
// registers instead of eight at 232: config 3 tile kernel 1.75 -> 1.53 ms; measured slower on
// every shared-memory-staged kernel). SYMEL_TILE_THREADS = 32 / 64 / 96 / 128 overrides
// (diagnostic; the contribution codes hold 7 bits of tile-local element).
int tile_threads_env() {
  static const int v = [] {
    const char* e = std::getenv("SYMEL_TILE_THREADS");
    const int t = e ? std::atoi(e) : 0;
    return (t == 32 || t == 64 || t == 96 || t == 128) ? t : 0;
  }();
  return v;
}
// resident CTAs per SM the kernels are compiled for (register cap 65536 / (threads * CTAs));
// SYMEL_TILE_CTAS overrides (diagnostic)
int tile_ctas_per_sm(int threads) {
  static const int env = [] { const char* e = std::getenv("SYMEL_TILE_CTAS"); return e ? std::atoi(e) : 0; }();
  return env > 0 ? env : 256 / threads;
}
// Shared memory per tile CTA (228 KB per SM on B200, 1 KB reserved per CTA, a little static
// smem); the staging part is capped lower to leave room for the plan slice.
std::size_t tile_smem_cta(int threads) { return (std::size_t)(225 * 1024 / tile_ctas_per_sm(threads)) & ~(std::size_t)1023; }
std::size_t tile_smem_max(int threads) { return tile_smem_cta(threads) - 6 * 1024 * (std::size_t)threads / 128; }
constexpr std::size_t kTileSmemOne = 226 * 1024;  // single CTA per SM (opt-in maximum 227 KB)

// Kernel variants per energy.
enum Variant : int {
  V_CONTRIB_IEEE = 0,
  V_CONTRIB_FAST,
  V_ATOMIC,
  V_ENERGY,  // E only (fast), line-search probe
  V_ACT,
  V_GUARD,
  V_TILE,
  V_TILE_SPD,  // tile kernel with the fused reduced-space SPD projection
  V_TILE_G,    // V_TILE / V_TILE_SPD reading the plan slice from L2 (slice too large for
  V_TILE_SPD_G,  // shared memory next to the staging at two CTAs per SM)
  V_COUNT
};

struct Array {
  std::string name;
  std::uint64_t items = 0;
  std::uint32_t comps = 0;
  bool is_dof = false;
  double* d = nullptr;
  std::uint64_t version = 0;  // bumped by every set_array (SoA copies are rebuilt from it)
  bool external = false;      // device pointer handed out: treat as changed every assemble
  // component classes (dev::comp_classes) of the data of `cls_version`; recomputed when the
  // array is set again, given up (identity) for arrays that keep changing
  std::vector<int> cls;
  std::uint64_t cls_version = ~0ull;
  int cls_runs = 0;
};

struct Conn {
  std::string name;
  std::uint32_t arity = 0;
  std::uint64_t n = 0;
  int* d = nullptr;
  std::uint64_t version = 0;  // bumped by set_elements
};

struct Energy {
  std::string name;
  int conn = -1;
  TapeIR deriv, act, guard, eonly;
  bool has_act = false, has_guard = false, is_sum = false, skip = false;
  int act_kind = 0;
  std::vector<InputBinding> inputs;
  std::vector<std::uint32_t> dof_slots;
  std::vector<double> sum_items;
  std::uint32_t n_items = 0, sum_arity = 0;
  std::vector<double> params;  // per input slot
  std::uint32_t flags = 0;
  BlockMap bm;
  Compiled* k[V_COUNT] = {};
  // linear-frontier factorisation of the derivative tape (fast kernels only; factorize.hpp)
  std::optional<TapeIR> fact;
  FactorizeInfo fact_info{};
  bool fact_tried = false;
  // reduced SPD form [E, g, M, W] of the same factorisation (factorize_spd)
  std::optional<TapeIR> fact_spd;
  FactorizeInfo spd_info{};
  bool spd_tried = false;
  // runtime
  unsigned char* d_mask = nullptr;  // activation mask (all elements)
  int* d_active = nullptr;          // active list (nullptr = identity)
  long long n_active = 0;
  bool act_init = false;
  int* d_slots = nullptr;
  double* d_contrib = nullptr;
  long long contrib_cap = 0;
  double* d_elemE = nullptr;
  long long elemE_cap = 0;
  double* d_values = nullptr;  // activation / guard values per element
  long long tile_base = 0;     // first global tile of this energy (tile plan)
  int* d_tile_perm = nullptr;  // tile position -> active ordinal (Morton order)
  int* d_tile_elems = nullptr; // tile position -> element id
  int cap[4] = {0, 0, 0, 0};   // shared plan-slice capacities (words): hseg, gseg, hcon, gcon
  int meta_depth[2] = {1, 1};  // tile reduction: metadata prefetch depth (Hessian, gradient segments)
  double* d_gstage = nullptr;  // global staging (large elements): one slab per tile
  // tile-ordered SoA copies of wide per-element arrays (elem_comp inputs): array -> copy
  int* d_changed = nullptr;     // activation: "the active set moved" flag of the last refresh
  std::map<int, double*> d_soa;
  std::map<int, std::vector<int>> soa_rows;  // component -> SoA row the copies / kernels were built with
  std::map<int, int*> d_soa_rowlist;         // device list of the representative components
  std::map<int, std::uint64_t> soa_version;
  long long soa_n = 0;          // SoA stride (n_active of the plan they were built for)
  std::uint64_t soa_epoch = ~0ull;
  int* d_conn_soa = nullptr;    // tile-ordered connectivity, slot-major (stride soa_n)
  std::uint64_t conn_soa_version = ~0ull;
};

}  // namespace

struct symel_cuda_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  std::string cache_dir;
  std::vector<Array> arrays;
  std::vector<Conn> conns;
  std::vector<std::unique_ptr<Energy>> energies;
  std::map<std::uint64_t, std::unique_ptr<Compiled>> kcache;
  struct { std::uint64_t memory_hits = 0, disk_hits = 0, builds = 0, corrupt = 0; } cache_stats;
  // dof layout + pattern
  bool topology_dirty = true, pattern_dirty = true;
  int b = 1;
  long long n_dofs = 0, n_rows = 0, n_blocks = 0;
  std::vector<long long> set_off;  // per array (-1 if not a dof array)
  int* d_row_ptr = nullptr;
  int* d_col_idx = nullptr;
  double* d_vals = nullptr;
  double* d_grad = nullptr;
  unsigned char* d_pins = nullptr;
  bool any_pins = false;
  dev::OrderedRefs refs;
  bool refs_valid = false;
  dev::TilePlan tplan;
  bool tplan_valid = false;
  struct AsmGraph {
    std::string sig;                 // launch signature (tiled_signature)
    cudaGraphExec_t exec = nullptr;  // recorded tiled assemble (assemble_tiled)
    long long launches = 0;          // kernels it launches
    unsigned long long used = 0;     // last use (LRU)
  };
  std::vector<AsmGraph> graphs;      // a few recorded assembles (e.g. one per mode)
  unsigned long long graph_clock = 0;
  std::uint64_t plan_epoch = 0;  // bumped on every tile-plan build (tile order may change)
  double* d_partials = nullptr;
  double* d_gpartials = nullptr;
  double* d_tileE = nullptr;
  bool last_tiled = false;
  // scratch
  double* d_partial = nullptr;
  long long partial_cap = 0;
  double* d_energy = nullptr;  // [n_energies + 1]
  int* d_bad = nullptr;        // [n_energies]
  double* h_pinned = nullptr;  // E + bad staging
  cudaEvent_t ev[4] = {};
  symel_cuda_timings timings{};
  std::uint64_t launches = 0;
  double last_E = 0.0;
  bool assembled = false;      // d_vals / d_grad hold a completed assemble
  // energies' tile kernels run concurrently (their outputs are disjoint or fixed-order
  // partials): fork from `stream` onto aux streams, join before the fix-up
  static constexpr int kAux = 3;
  cudaStream_t aux[kAux] = {};
  cudaEvent_t fork_ev = nullptr, join_ev[kAux] = {};
  // asynchronous tail of a deterministic assemble: E and the gradient are final before the
  // Hessian fix-up; assemble() returns then, the Hessian fix-up keeps running on `stream`
  // (every later call that reads the matrix is ordered after it) and copy_gradient reads the
  // gradient on copy_stream once grad_ready has fired
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t grad_ready = nullptr, e_ready = nullptr;
  bool timings_pending = false;
  dev::SolverWork solver;      // SpMV / PCG work vectors
};

namespace {

thread_local std::string g_create_error;

void cfree(void* p) {
  if (p) cudaFree(p);
}

template <class T>
void dalloc(T** p, std::size_t n) {
  cfree(*p);
  *p = nullptr;
  CK(cudaMalloc((void**)p, sizeof(T) * (n ? n : 1)));
}

// All host<->device traffic is ordered on the context stream (a non-blocking stream does not
// synchronise with legacy-stream cudaMemcpy/cudaMemset).
void copy_sync(symel_cuda_ctx* c, void* dst, const void* src, std::size_t bytes, cudaMemcpyKind kind) {
  if (bytes == 0) return;
  CK(cudaMemcpyAsync(dst, src, bytes, kind, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

Energy& energy_of(symel_cuda_ctx* c, int id) {
  if (id < 0 || id >= (int)c->energies.size()) throw Fail{SYMEL_E_ARG, "invalid energy handle"};
  return *c->energies[id];
}

// ------------------------------------------------------------------------------ NVRTC

constexpr int kNoBadElem = 0x7f7f7f7f;  // d_bad sentinel (memset 0x7f)

// Cubin cache (the reference's KernelCache disk layout, cache.hpp:103-180, for device code):
// entries are named by the tape's digest -- the reference's kernel_key (registry.hpp:415-428;
// KernelCache::get_or_build stamps it into the tape, cache.hpp:78) -- plus a hash of the
// generated kernel (mode, binding, tile shape) and the arch tag:
//   <kernel_key hex>.<variant>.sm100a.cubin  +  .meta  ("symel-cubin v1 sm_100a <source fnv> <bytes>")
// A missing entry is a miss; an entry whose meta does not match, or whose image the driver
// rejects, is corrupt: warning + rebuild + overwrite (cache.hpp:119-148).
namespace {
bool digest_is_zero(const std::array<std::uint8_t, 32>& d) {
  for (auto v : d)
    if (v) return false;
  return true;
}

void cache_warn(symel_cuda_ctx* c, const std::string& msg) {
  ++c->cache_stats.corrupt;
  std::fprintf(stderr, "[symel] warning: corrupt cache entry, rebuilding: %s\n", msg.c_str());
}

std::vector<char> nvrtc_build(symel_cuda_ctx* c, const KernelSpec& spec, const std::string& src) {
  const auto t0 = std::chrono::steady_clock::now();
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, src.c_str(), (spec.name + ".cu").c_str(), 0, nullptr, nullptr) != NVRTC_SUCCESS)
    throw Fail{SYMEL_E_COMPILE, "nvrtcCreateProgram failed"};
  // IEEE-mode tape arithmetic is emitted as __dadd_rn/__dsub_rn/__dmul_rn (codegen.cpp), so
  // contraction is safe for the rest of every kernel
  std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo", "--fmad=true"};
  // SYMEL_PTXAS_VERBOSE=1: print ptxas register / spill usage of each compiled kernel
  const bool verbose = std::getenv("SYMEL_PTXAS_VERBOSE") != nullptr;
  if (verbose) opts.push_back("--ptxas-options=-v");
  const nvrtcResult r = nvrtcCompileProgram(prog, (int)opts.size(), opts.data());
  std::size_t ls = 0;
  nvrtcGetProgramLogSize(prog, &ls);
  std::string log(ls, '\0');
  nvrtcGetProgramLog(prog, log.data());
  if (verbose && r == NVRTC_SUCCESS) std::fprintf(stderr, "[symel ptxas] %s %s\n", spec.name.c_str(), log.c_str());
  if (r != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    throw Fail{SYMEL_E_COMPILE, "kernel compilation failed (" + std::string(nvrtcGetErrorString(r)) + "):\n" + log};
  }
  std::size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  std::vector<char> cubin(n);
  nvrtcGetCUBIN(prog, cubin.data());
  nvrtcDestroyProgram(&prog);
  ++c->cache_stats.builds;
  c->timings.compile_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return cubin;
}

void write_atomically(const std::string& path, const char* data, std::size_t n) {
  std::error_code ec;
  const std::string tmp = path + ".tmp" + std::to_string((long long)::getpid());
  {
    std::ofstream os(tmp, std::ios::binary | std::ios::trunc);
    os.write(data, (std::streamsize)n);
  }
  std::filesystem::rename(tmp, path, ec);
}
}  // namespace

Compiled* compile_kernel(symel_cuda_ctx* c, const KernelSpec& spec) {
  std::string src = emit_kernel(spec);
  const std::string flags = "fmad1";
  const std::uint64_t key = fnv1a(src + "|" + flags + "|sm_100a|v1");
  auto it = c->kcache.find(key);
  if (it != c->kcache.end()) {
    ++c->cache_stats.memory_hits;
    return it->second.get();
  }
  char variant[32];
  std::snprintf(variant, sizeof variant, "%016llx", (unsigned long long)key);
  // hand-built tapes without a kernel key are named by a content hash of the source
  const std::string dkey = digest_is_zero(spec.tape->digest) ? std::string(variant) + "0000000000000000"
                                                              : spec.tape->digest_hex();
  char meta_line[160];
  std::string path, meta;
  if (!c->cache_dir.empty()) {
    path = c->cache_dir + "/" + dkey + "." + variant + ".sm100a.cubin";
    meta = c->cache_dir + "/" + dkey + "." + variant + ".meta";
  }
  std::vector<char> cubin;
  auto load_image = [&](std::unique_ptr<Compiled>& comp) {
    if (c->device < 0) return;
    CK(cudaLibraryLoadData(&comp->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    CK(cudaLibraryGetKernel(&comp->kernel, comp->lib, spec.name.c_str()));
  };
  auto comp = std::make_unique<Compiled>();
  bool from_disk = false;
  if (!path.empty() && std::filesystem::exists(path)) {
    std::ifstream is(path, std::ios::binary);
    cubin.assign(std::istreambuf_iterator<char>(is), {});
    std::ifstream ms(meta);
    std::string got((std::istreambuf_iterator<char>(ms)), {});
    std::snprintf(meta_line, sizeof meta_line, "symel-cubin v1 sm_100a %016llx %zu\n", (unsigned long long)key,
                  cubin.size());
    if (got != meta_line) {
      cache_warn(c, path + ": metadata mismatch");
    } else if (cubin.size() < 4 || std::memcmp(cubin.data(), "\x7f" "ELF", 4) != 0) {
      cache_warn(c, path + ": not a cubin image");
    } else if (c->device >= 0 && cudaLibraryLoadData(&comp->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr,
                                                     0) != cudaSuccess) {
      cudaGetLastError();
      comp->lib = nullptr;
      cache_warn(c, path + ": rejected by the driver");
    } else {
      if (c->device >= 0) CK(cudaLibraryGetKernel(&comp->kernel, comp->lib, spec.name.c_str()));
      ++c->cache_stats.disk_hits;
      from_disk = true;
    }
  }
  if (!from_disk) {
    cubin = nvrtc_build(c, spec, src);
    if (!path.empty()) {
      std::error_code ec;
      std::filesystem::create_directories(c->cache_dir, ec);
      write_atomically(path, cubin.data(), cubin.size());
      std::snprintf(meta_line, sizeof meta_line, "symel-cubin v1 sm_100a %016llx %zu\n", (unsigned long long)key,
                    cubin.size());
      write_atomically(meta, meta_line, std::strlen(meta_line));
    }
    load_image(comp);
  }
  comp->source = std::move(src);
  comp->tpb = spec.threads_per_block;
  comp->elems = spec.threads_per_block / std::max(1, spec.item_lanes);
  Compiled* raw = comp.get();
  c->kcache.emplace(key, std::move(comp));
  return raw;
}

// Dynamic shared memory of the tile kernel: per element [E | g(n) | upper local-block
// triangle of full b x b sub-blocks] (codegen.cpp stage layout), one tile of elements.
// Fixed-summation energies (n_items = 2, 4, 8: tet10's quadrature) run their item terms on
// adjacent lanes in the tile kernel: 128 / n_items elements per tile.
int tile_item_lanes(const Energy& e) {
  if (std::getenv("SYMEL_NO_ITEM_LANES")) return 1;
  const int n = (int)e.n_items;
  return (n == 2 || n == 4 || n == 8) ? n : 1;
}
std::size_t tile_stage_slots(const symel_cuda_ctx* c, const Energy& e) {
  const std::size_t n = e.dof_slots.size(), nlb = e.bm.n_lb, bb = std::size_t(c->b) * c->b;
  return 1 + n + bb * nlb * (nlb + 1) / 2;
}
int tile_threads(const symel_cuda_ctx* c, const Energy& e) {
  if (tile_threads_env()) return tile_threads_env();
  const int lanes = tile_item_lanes(e);
  const bool global_at_128 = sizeof(double) * tile_stage_slots(c, e) * (128 / lanes) > tile_smem_max(128);
  return (lanes == 4 && global_at_128) ? 96 : 128;
}
int tile_elems(const symel_cuda_ctx* c, const Energy& e) { return tile_threads(c, e) / tile_item_lanes(e); }
std::size_t tile_stage_doubles(const symel_cuda_ctx* c, const Energy& e) { return tile_stage_slots(c, e) * tile_elems(c, e); }
// Elements whose staged outputs do not fit the CTA's share of the SM stage in global memory instead.
bool tile_global_stage(const symel_cuda_ctx* c, const Energy& e) {
  return sizeof(double) * tile_stage_doubles(c, e) > tile_smem_max(tile_threads(c, e));
}
std::size_t tile_smem(const symel_cuda_ctx* c, const Energy& e) {
  return tile_global_stage(c, e) ? 0 : sizeof(double) * tile_stage_doubles(c, e);
}

// Tape executed by the fast kernels: the factorised one when the energy has a narrowing
// affine frontier (and is not flagged exact), else the reference tape.
const TapeIR* fast_tape(Energy& e) {
  if (!e.fact_tried) {
    e.fact_tried = true;
    if (!(e.flags & SYMEL_ENERGY_EXACT) && !std::getenv("SYMEL_NO_FACTORIZE"))
      e.fact = factorize_linear_frontier(e.deriv, e.dof_slots, &e.fact_info);
  }
  return e.fact ? &*e.fact : &e.deriv;
}

// Reduced SPD tape (nullptr when the energy cannot use the fused projection: no narrowing
// frontier, or fixed summation -- the projection must see the summed Hessian).
const TapeIR* spd_tape(Energy& e) {
  if (!e.spd_tried) {
    e.spd_tried = true;
    // exact-rounding energies also use it: kernel_for compiles them without contraction
    if (e.n_items <= 1 && !std::getenv("SYMEL_NO_FUSED_SPD"))
      e.fact_spd = factorize_spd(e.deriv, e.dof_slots, &e.spd_info);
    if (e.fact_spd && (e.spd_info.frontier < 2 || e.spd_info.frontier > 9)) e.fact_spd.reset();
  }
  return e.fact_spd ? &*e.fact_spd : nullptr;
}

KernelSpec base_spec(symel_cuda_ctx* c, const Energy& e, const TapeIR* tape) {
  KernelSpec s;
  s.tape = tape;
  s.inputs = e.inputs;
  s.dof_slots = e.dof_slots;
  for (const Array& a : c->arrays) s.array_comps.push_back(a.comps);
  s.arity = c->conns[e.conn].arity;
  s.sum_items = e.sum_items;
  s.n_items = e.n_items;
  s.sum_arity = e.sum_arity;
  s.b = c->b;
  return s;
}

// Wide per-element arrays (elem_comp inputs, >= 4 components) are read by the tile kernels from
// a tile-ordered SoA copy: the threads of a warp (consecutive tile positions) read consecutive
// doubles instead of one strided row each (the 144-double bending Q, pair offsets, rest frames).
constexpr std::uint32_t kSoaMinComps = 4;
std::vector<std::uint8_t> soa_arrays_of(const symel_cuda_ctx* c, const Energy& e) {
  std::vector<std::uint8_t> v(c->arrays.size(), 0);
  if (std::getenv("SYMEL_NO_SOA")) return v;
  for (const InputBinding& in : e.inputs)
    if (in.kind == InKind::elem_comp && c->arrays[in.array].comps >= kSoaMinComps) v[in.array] = 1;
  return v;
}

// Tile kernels read their elements' items from a tile-ordered, slot-major copy of the
// connectivity (one coalesced load per slot, independent of the element id) instead of
// tile position -> element id -> connectivity -> items. Measured (same box A/B): config 3
// 5.13 -> 4.00 ms, config 5 14.97 -> 14.59, config 4 4.71 -> 4.63, config 2 without SPD
// 2.62 -> 2.58. SYMEL_NO_CONN_SOA switches it off.
bool use_conn_soa() { return !std::getenv("SYMEL_NO_CONN_SOA"); }

// Wide per-element arrays often hold structure the tape cannot see: components that are +0.0 in
// every element and components that repeat another one bit for bit (the reference's 12 x 12
// bending Q, energies.hpp:684-745, is a 4 x 4 stencil repeated per coordinate: 96 zeros and 16
// distinct values in 144 doubles). The SoA copy keeps one row per distinct non-zero component
// and the generated kernel reads each once (a zero component becomes the literal 0.0): the
// arithmetic, and so every output bit, is unchanged. Classes are exact (dev::comp_classes),
// recomputed when the array is set again (given up for arrays set more than a few times) and
// part of the kernel specialisation. SYMEL_NO_SOA_DEDUP switches it off.
constexpr std::uint32_t kDedupMinComps = 16;
std::vector<int> soa_rows_of(symel_cuda_ctx* c, std::size_t i) {
  Array& arr = c->arrays[i];
  static const bool off = std::getenv("SYMEL_NO_SOA_DEDUP") != nullptr;
  if (off || c->device < 0 || arr.external || !arr.d || arr.comps < kDedupMinComps || arr.cls_runs > 4) return {};
  if (arr.cls_version != arr.version) {
    arr.cls.assign(arr.comps, 0);
    CK(dev::comp_classes(arr.d, (int)arr.comps, (long long)arr.items, arr.cls.data(), c->stream));
    c->launches += 2;
    arr.cls_version = arr.version;
    ++arr.cls_runs;
  }
  // component -> row: representatives numbered in component order
  std::vector<int> row(arr.comps, -1), rank(arr.comps, -1);
  int n = 0;
  bool identity = true;
  for (std::uint32_t q = 0; q < arr.comps; ++q)
    if (arr.cls[q] == (int)q) rank[q] = n++;
  for (std::uint32_t q = 0; q < arr.comps; ++q) {
    row[q] = arr.cls[q] < 0 ? -1 : rank[arr.cls[q]];
    identity = identity && row[q] == (int)q;
  }
  return identity ? std::vector<int>{} : row;
}

void ensure_soa(symel_cuda_ctx* c, Energy& e) {
  const std::vector<std::uint8_t> soa = soa_arrays_of(c, e);
  const int* map = e.d_tile_perm ? e.d_tile_elems : e.d_active;
  for (std::size_t i = 0; i < soa.size(); ++i) {
    if (!soa[i]) continue;
    const Array& arr = c->arrays[i];
    double*& buf = e.d_soa[(int)i];
    const std::vector<int>& rows = e.soa_rows[(int)i];  // set by refresh_soa_rows before the kernels are chosen
    const bool fresh = buf && e.soa_n == e.n_active && e.soa_epoch == c->plan_epoch &&
                       e.soa_version[(int)i] == arr.version && !arr.external;
    if (fresh) continue;
    int n_rows = (int)arr.comps;
    std::vector<int> reps;
    if (!rows.empty()) {
      n_rows = 0;
      for (int r : rows) n_rows = std::max(n_rows, r + 1);
      reps.assign(n_rows, 0);
      for (std::uint32_t q = arr.comps; q-- > 0;)
        if (rows[q] >= 0) reps[rows[q]] = (int)q;  // lowest component of the class last
    }
    cfree(buf);
    buf = nullptr;
    dalloc(&buf, (std::size_t)std::max(1, n_rows) * std::max<long long>(1, e.n_active));
    if (rows.empty()) {
      CK(dev::soa_gather(arr.d, (int)arr.comps, map, e.n_active, e.n_active, buf, c->stream));
    } else {
      int*& rl = e.d_soa_rowlist[(int)i];
      cfree(rl);
      rl = nullptr;
      dalloc(&rl, (std::size_t)std::max(1, n_rows));
      if (n_rows) copy_sync(c, rl, reps.data(), sizeof(int) * n_rows, cudaMemcpyHostToDevice);
      CK(dev::soa_gather_rows(arr.d, (int)arr.comps, rl, n_rows, map, e.n_active, e.n_active, buf, c->stream));
    }
    ++c->launches;
    e.soa_version[(int)i] = arr.version;
  }
  // tile-ordered connectivity (rebuilt with the plan or a new element list)
  if (use_conn_soa()) {
    const Conn& k = c->conns[e.conn];
    const bool fresh = e.d_conn_soa && e.soa_n == e.n_active && e.soa_epoch == c->plan_epoch &&
                       e.conn_soa_version == k.version;
    if (!fresh) {
      if (!e.d_conn_soa || e.soa_n != e.n_active) dalloc(&e.d_conn_soa, (std::size_t)k.arity * std::max<long long>(1, e.n_active));
      CK(dev::conn_soa(k.d, (int)k.arity, map, e.n_active, e.d_conn_soa, c->stream));
      ++c->launches;
      e.conn_soa_version = k.version;
    }
  }
  e.soa_n = e.n_active;
  e.soa_epoch = c->plan_epoch;
}

// The row maps the energy's kernels are specialised on (per array; empty = identity).
std::vector<std::vector<int>> soa_rows_spec(symel_cuda_ctx* c, Energy& e) {
  std::vector<std::vector<int>> v(c->arrays.size());
  for (const auto& kv : e.soa_rows) v[kv.first] = kv.second;
  return v;
}

// Recomputes the energy's row maps from the arrays' current data; when a map changed, the tile
// kernels compiled for the old one and the SoA copies built with it are dropped.
void refresh_soa_rows(symel_cuda_ctx* c, Energy& e) {
  const std::vector<std::uint8_t> soa = soa_arrays_of(c, e);
  bool changed = false;
  for (std::size_t i = 0; i < soa.size(); ++i) {
    if (!soa[i]) continue;
    std::vector<int> rows = soa_rows_of(c, i);
    auto it = e.soa_rows.find((int)i);
    if (it == e.soa_rows.end() || it->second != rows) {
      changed = changed || it != e.soa_rows.end() || !rows.empty();
      e.soa_rows[(int)i] = std::move(rows);
      e.soa_version[(int)i] = ~0ull;  // rebuild the copy
    }
  }
  if (changed)
    for (int v : {V_TILE, V_TILE_SPD, V_TILE_G, V_TILE_SPD_G}) e.k[v] = nullptr;  // owned by the context's cache
}

KernelSpec spec_for(symel_cuda_ctx* c, Energy& e, Variant v) {
  KernelSpec s;
  switch (v) {
    case V_CONTRIB_IEEE:
      s = base_spec(c, e, &e.deriv);
      s.mode = OutMode::contrib;
      s.fast = false;
      s.schedule = 0;  // tape order: bitwise the reference's sequence of operations
      break;
    case V_CONTRIB_FAST:
      s = base_spec(c, e, fast_tape(e));
      s.mode = OutMode::contrib;
      s.schedule = -1;  // auto: lowest peak of live values
      break;
    case V_ATOMIC:
      s = base_spec(c, e, fast_tape(e));
      s.mode = OutMode::fused_atomic;
      s.schedule = -1;  // auto: lowest peak of live values
      break;
    case V_ENERGY:
      s = base_spec(c, e, &e.eonly);
      s.mode = OutMode::value_only;
      s.value_reduce = 3;
      s.threads_per_block = 256;
      break;
    case V_ACT:
      s = base_spec(c, e, &e.act);
      s.mode = OutMode::value_only;
      s.value_reduce = 1;
      s.threads_per_block = 256;
      s.fast = false;  // activation decides the active set: reproduce the reference exactly
      s.schedule = 0;
      break;
    case V_GUARD:
      s = base_spec(c, e, &e.guard);
      s.mode = OutMode::value_only;
      s.value_reduce = 2;
      s.threads_per_block = 256;
      s.fast = false;  // line-search guard value: exact
      s.schedule = 0;
      break;
    case V_TILE:
    case V_TILE_G:
      s = base_spec(c, e, fast_tape(e));
      s.plan_global = v == V_TILE_G;
      s.item_lanes = tile_item_lanes(e);
      s.soa_arrays = soa_arrays_of(c, e);
      s.soa_rows = soa_rows_spec(c, e);
      s.meta_depth_h = e.meta_depth[0];
      s.meta_depth_g = e.meta_depth[1];
      s.conn_soa = use_conn_soa();
      s.mode = OutMode::fused_tile;
      s.schedule = -1;  // auto: lowest peak of live values
      s.threads_per_block = tile_threads(c, e);
      s.min_blocks = tile_ctas_per_sm(s.threads_per_block);
      s.stage_global = tile_global_stage(c, e);
      break;
    case V_TILE_SPD:
    case V_TILE_SPD_G: {
      const TapeIR* tp = spd_tape(e);
      if (!tp) throw Fail{SYMEL_E_STATE, "energy '" + e.name + "': no reduced SPD form"};
      s = base_spec(c, e, tp);
      s.plan_global = v == V_TILE_SPD_G;
      s.soa_arrays = soa_arrays_of(c, e);
      s.soa_rows = soa_rows_spec(c, e);
      s.meta_depth_h = e.meta_depth[0];
      s.meta_depth_g = e.meta_depth[1];
      // measured: the SPD tet kernel (compute-bound, its connectivity latency hidden behind the
      // other CTA's eigen-solve) is 1.3 % slower reading the copy; the exact-rounding contact
      // kernel (random nodes, latency-bound) gains
      s.conn_soa = use_conn_soa() && (e.flags & SYMEL_ENERGY_EXACT);
      s.mode = OutMode::fused_tile_spd;
      s.spd_m = e.spd_info.frontier;
      // QL lookahead (codegen.cpp sy_ql_la) pays off where divergence in the QL dominates
      // (config 2 tets: 8.66 -> 7.20 ms); the exact-rounding contact kernel, whose larger
      // unfactorised tape already strains the instruction cache, measured 1.4 ms slower with it
      s.spd_lookahead = !(e.flags & SYMEL_ENERGY_EXACT) && !std::getenv("SYMEL_NO_QL_LOOKAHEAD");
      s.schedule = -1;
      s.threads_per_block = tile_threads(c, e);
      s.min_blocks = tile_ctas_per_sm(s.threads_per_block);
      s.stage_global = tile_global_stage(c, e);
      break;
    }
    default:
      throw Fail{SYMEL_E_ARG, "unsupported kernel variant"};
  }
  s.bulk_plan = !std::getenv("SYMEL_NO_BULK_PLAN");
  s.soa_prefetch = !std::getenv("SYMEL_NO_SOA_PF");
  if (e.flags & SYMEL_ENERGY_EXACT) {
    // ill-conditioned energies: reproduce the reference's rounding (IEEE division, no
    // contraction) in every assembly mode. The schedule only reorders SSA instructions, so it
    // does not change any value and stays register-pressure driven.
    s.fast = false;
  }
  s.name = "sy_" + std::to_string(v);
  return s;
}

Compiled* kernel_for(symel_cuda_ctx* c, Energy& e, Variant v) {
  if (e.k[v]) return e.k[v];
  e.k[v] = compile_kernel(c, spec_for(c, e, v));
  if (v == V_TILE || v == V_TILE_SPD || v == V_TILE_G || v == V_TILE_SPD_G) e.k[v]->smem = tile_smem(c, e);  // plus the plan slice at launch
  return e.k[v];
}

void launch(symel_cuda_ctx* c, Compiled* k, SyArgs& a, long long n, std::size_t smem = 0,
            cudaStream_t stream = nullptr) {
  if (n <= 0) return;
  if (c->device < 0) throw Fail{SYMEL_E_NODEVICE, "no CUDA device"};
  const long long blocks = (n - a.t0 + k->elems - 1) / k->elems;
  if (!smem) smem = k->smem;
  if (smem > 48 * 1024 && smem != k->smem_attr) {
    CK(cudaKernelSetAttributeForDevice(k->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem, c->device));
    k->smem_attr = smem;
  }
  void* params[] = {&a};
  CK(cudaLaunchKernel((const void*)k->kernel, dim3((unsigned)blocks), dim3((unsigned)k->tpb), params, smem,
                      stream ? stream : c->stream));
  ++c->launches;
}

void fill_args(symel_cuda_ctx* c, const Energy& e, SyArgs& a) {
  std::memset(&a, 0, sizeof a);
  if (c->arrays.size() > 24) throw Fail{SYMEL_E_ARG, "too many arrays (max 24)"};
  for (std::size_t i = 0; i < c->arrays.size(); ++i) {
    a.arr[i] = c->arrays[i].d;
    a.set_off[i] = i < c->set_off.size() ? c->set_off[i] : -1;
  }
  a.conn = c->conns[e.conn].d;
  int np = 0;
  for (std::size_t k = 0; k < e.inputs.size(); ++k)
    if (e.inputs[k].kind == InKind::param) a.params[np++] = e.params[k];
}

// ------------------------------------------------------------------------ layout/pattern

void refresh_layout(symel_cuda_ctx* c) {
  c->set_off.assign(c->arrays.size(), -1);
  long long off = 0;
  bool all3 = true, any = false;
  for (std::size_t i = 0; i < c->arrays.size(); ++i) {
    const Array& a = c->arrays[i];
    if (!a.is_dof) continue;
    any = true;
    c->set_off[i] = off;
    off += (long long)a.items * a.comps;
    if (a.comps != 3) all3 = false;
  }
  const int nb = (any && all3) ? 3 : 1;  // assembly.hpp:273-276
  if (nb != c->b) {
    c->b = nb;
    for (auto& e : c->energies)
      for (auto& k : e->k) k = nullptr;  // kernels are specialised on b
  }
  c->n_dofs = off;
  c->n_rows = off / c->b;
  for (auto& ep : c->energies) {
    Energy& e = *ep;
    KernelSpec s = base_spec(c, e, &e.deriv);
    e.bm = make_block_map(s);
    if (e.bm.n_lb > (unsigned)dev::kMaxLb) throw Fail{SYMEL_E_ARG, "energy '" + e.name + "': too many local blocks"};
  }
}

dev::LbDesc lb_desc(symel_cuda_ctx* c, const Energy& e) {
  dev::LbDesc d{};
  d.n_lb = (int)e.bm.n_lb;
  d.b = c->b;
  d.arity = (int)c->conns[e.conn].arity;
  for (std::uint32_t q = 0; q < e.bm.n_lb; ++q) {
    d.slot[q] = (int)e.bm.lb_slot[q];
    d.off[q] = c->set_off[e.bm.lb_array[q]] + e.bm.lb_comp0[q];
    d.comps[q] = (int)c->arrays[e.bm.lb_array[q]].comps;
  }
  return d;
}

void build_pattern(symel_cuda_ctx* c) {
  cudaEventRecord(c->ev[0], c->stream);
  cfree(c->d_row_ptr); c->d_row_ptr = nullptr;
  cfree(c->d_col_idx); c->d_col_idx = nullptr;
  long long cap = c->n_rows;
  for (auto& ep : c->energies)
    if (!ep->skip) cap += ep->n_active * (long long)ep->bm.n_lb * (ep->bm.n_lb - 1);
  unsigned long long* keys = nullptr;
  unsigned long long* counter = nullptr;
  CK(cudaMallocAsync((void**)&keys, sizeof(unsigned long long) * (cap ? cap : 1), c->stream));
  CK(cudaMallocAsync((void**)&counter, sizeof(unsigned long long), c->stream));
  const unsigned long long init = (unsigned long long)c->n_rows;
  CK(cudaMemcpyAsync(counter, &init, sizeof init, cudaMemcpyHostToDevice, c->stream));
  CK(dev::diag_keys(c->n_rows, keys, c->stream));
  ++c->launches;
  for (auto& ep : c->energies) {
    Energy& e = *ep;
    if (e.skip || e.n_active == 0) continue;
    CK(dev::pattern_keys(lb_desc(c, e), c->conns[e.conn].d, e.d_active, e.n_active, keys, counter, c->stream));
    ++c->launches;
  }
  unsigned long long nk = 0;
  CK(cudaMemcpyAsync(&nk, counter, sizeof nk, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  long long nb = 0;
  CK(dev::build_csr(keys, (long long)nk, c->n_rows, &c->d_row_ptr, &c->d_col_idx, &nb, c->stream));
  c->n_blocks = nb;
  CK(cudaFreeAsync(keys, c->stream));
  CK(cudaFreeAsync(counter, c->stream));
  for (auto& ep : c->energies) {
    Energy& e = *ep;
    cfree(e.d_slots); e.d_slots = nullptr;
    if (e.skip || e.n_active == 0) continue;
    dalloc(&e.d_slots, (std::size_t)e.n_active * e.bm.n_lb * e.bm.n_lb);
    CK(dev::slot_map(lb_desc(c, e), c->conns[e.conn].d, e.d_active, e.n_active, c->d_row_ptr, c->d_col_idx,
                     e.d_slots, c->stream));
    ++c->launches;
  }
  dalloc(&c->d_vals, (std::size_t)c->n_blocks * c->b * c->b);
  dalloc(&c->d_grad, (std::size_t)c->n_dofs);
  CK(cudaMemsetAsync(c->d_vals, 0, sizeof(double) * c->n_blocks * c->b * c->b, c->stream));
  CK(cudaMemsetAsync(c->d_grad, 0, sizeof(double) * c->n_dofs, c->stream));
  if (c->refs_valid) dev::free_ordered_refs(&c->refs);
  c->refs_valid = false;
  if (c->tplan_valid) dev::free_tile_plan(&c->tplan);
  c->tplan_valid = false;
  c->pattern_dirty = false;
  cudaEventRecord(c->ev[1], c->stream);
  cudaEventSynchronize(c->ev[1]);
  float ms = 0;
  cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
  c->timings.pattern_ms = ms;
}

void ensure_refs(symel_cuda_ctx* c) {
  if (c->refs_valid) return;
  std::vector<dev::EnergyRefSrc> src;
  long long ord = 0;
  for (auto& ep : c->energies) {
    Energy& e = *ep;
    if (e.skip) continue;
    dev::EnergyRefSrc r{};
    r.slots = e.d_slots;
    r.conn = c->conns[e.conn].d;
    r.active = e.d_active;
    r.n_active = e.n_active;
    r.ord_base = ord;
    r.d = lb_desc(c, e);
    ord += e.n_active;
    src.push_back(r);
  }
  CK(dev::ordered_refs(src.data(), (int)src.size(), c->n_blocks, c->n_rows, &c->refs, c->stream));
  c->launches += 2 * src.size() + 4;
  c->refs_valid = true;
}

// ------------------------------------------------------------------------ activation

void refresh_activation(symel_cuda_ctx* c) {
  for (auto& ep : c->energies) {
    Energy& e = *ep;
    const long long ne = (long long)c->conns[e.conn].n;
    if (e.skip) { e.n_active = 0; continue; }
    if (!e.has_act) {
      if (e.n_active != ne || e.d_active) {
        cfree(e.d_active); e.d_active = nullptr;
        e.n_active = ne;
        c->pattern_dirty = true;
      }
      continue;
    }
    if (!e.act_init) {
      dalloc(&e.d_mask, (std::size_t)ne);
      CK(cudaMemsetAsync(e.d_mask, 1, (std::size_t)(ne ? ne : 1), c->stream));  // prepare(): all active
      dalloc(&e.d_values, (std::size_t)ne);
      e.act_init = true;
      e.n_active = -1;
    }
    Compiled* k = kernel_for(c, e, V_ACT);
    SyArgs a;
    fill_args(c, e, a);
    a.n = ne;
    a.value_out = e.d_values;
    launch(c, k, a, ne);
    // the host has to know whether the active set moved (it decides on a pattern rebuild, like
    // the reference's prepare): one flag per energy, allocated once
    if (!e.d_changed) dalloc(&e.d_changed, 1);
    CK(cudaMemsetAsync(e.d_changed, 0, sizeof(int), c->stream));
    CK(dev::activation_mask(e.d_values, ne, e.act_kind, e.d_mask, e.d_changed, c->stream));
    ++c->launches;
    int changed = 0;
    CK(cudaMemcpyAsync(&changed, e.d_changed, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (changed || e.n_active < 0) {
      dalloc(&e.d_active, (std::size_t)ne);
      long long na = 0;
      CK(dev::compact_active(e.d_mask, ne, e.d_active, &na, c->stream));
      ++c->launches;
      e.n_active = na;
      c->pattern_dirty = true;
    }
  }
}

void prepare(symel_cuda_ctx* c) {
  if (c->device < 0) throw Fail{SYMEL_E_NODEVICE, "no CUDA device available (the device path has no CPU fallback)"};
  if (c->energies.empty()) throw Fail{SYMEL_E_STATE, "no energies registered"};
  if (c->topology_dirty) {
    refresh_layout(c);
    for (auto& ep : c->energies) {
      ep->act_init = false;
      ep->n_active = -1;
    }
    c->topology_dirty = false;
    c->pattern_dirty = true;
  }
}

void ensure_elem_buffers(symel_cuda_ctx* c, Energy& e, bool contrib) {
  const long long n = std::max<long long>(e.n_active, 1);
  if (e.elemE_cap < n) {
    dalloc(&e.d_elemE, (std::size_t)n);
    e.elemE_cap = n;
  }
  if (contrib) {
    const long long need = n * (long long)e.deriv.n_outputs;
    if (e.contrib_cap < need) {
      dalloc(&e.d_contrib, (std::size_t)need);
      e.contrib_cap = need;
    }
  }
  const long long np = dev::energy_tree_partials(n) + 1;
  if (c->partial_cap < np) {
    dalloc(&c->d_partial, (std::size_t)np);
    c->partial_cap = np;
  }
}

// Element id of the index a kernel reported: an active ordinal (active lists ascend, so the
// lowest ordinal is the lowest element id, like check_finite), or -- tile kernels -- the
// element id itself.
int64_t element_of(symel_cuda_ctx* c, const Energy& e, int t) {
  if (c->last_tiled) return t;  // tile kernels report the element id itself (lowest wins)
  const int* map = e.d_active;
  if (!map) return t;
  int v = 0;
  copy_sync(c, &v, map + t, sizeof(int), cudaMemcpyDeviceToHost);
  return v;
}

double finish_assemble(symel_cuda_ctx* c, symel_cuda_status* st, bool async_tail = false);


// The tile plan packs a Hessian contribution as (transpose << 15 | upper sub-block << 7 |
// position in tile): at most 256 upper local sub-blocks (n_lb <= 22) per element. Larger
// elements (hex27 / Q2 type) take the contrib path.
bool tile_codes_fit(const Energy& e) { return e.bm.n_lb * (e.bm.n_lb + 1) / 2 <= 256; }

bool tile_ok(const symel_cuda_ctx* c, const Energy& e) { return tile_codes_fit(e) && tile_smem(c, e) <= tile_smem_max(tile_threads(c, e)); }

bool all_tile_capable(symel_cuda_ctx* c) {
  long long nh = 0, ng = 0;
  for (auto& ep : c->energies) {
    if (ep->skip) continue;
    if (!tile_ok(c, *ep)) return false;
    if ((ep->flags & SYMEL_ENERGY_SPD) && !spd_tape(*ep)) return false;  // projection needs the reduced form
    nh += (long long)ep->n_active * ep->bm.n_lb * ep->bm.n_lb;
    ng += (long long)ep->n_active * ep->bm.n_lb;
  }
  // the plan stores contribution / segment indices as int32
  return nh <= INT_MAX && ng <= INT_MAX;
}

void ensure_tile_plan(symel_cuda_ctx* c) {
  if (c->tplan_valid) return;
  cudaEventRecord(c->ev[0], c->stream);
  std::vector<dev::TileSrc> src;
  long long tiles = 0;
  for (auto& ep : c->energies) {
    Energy& e = *ep;
    e.tile_base = tiles;
    if (e.skip || e.n_active == 0) continue;
    dev::TileSrc s{};
    s.slots = e.d_slots;
    s.conn = c->conns[e.conn].d;
    s.active = e.d_active;
    s.n_active = e.n_active;
    s.tile_base = tiles;
    s.tpb = tile_elems(c, e);
    s.d = lb_desc(c, e);
    s.h0 = 1 + (int)e.dof_slots.size();
    s.sort_segments = tile_global_stage(c, e) ? 0 : 1;  // L2-staged tiles keep target order
    // spatially coherent tiles: Morton order of element centroids (dof arrays as positions)
    dalloc(&e.d_tile_perm, (std::size_t)e.n_active);
    dalloc(&e.d_tile_elems, (std::size_t)e.n_active);
    bool positions = true;
    std::vector<const double*> arrs;
    for (std::uint32_t q = 0; q < e.bm.n_lb; ++q) {
      const Array& arr = c->arrays[e.bm.lb_array[q]];
      positions = positions && arr.comps >= 3;
      arrs.push_back(arr.d);
    }
    if (positions && !std::getenv("SYMEL_NO_MORTON")) {
      CK(dev::tile_order(s.d, arrs.data(), s.conn, e.d_active, e.n_active, e.d_tile_perm, e.d_tile_elems, c->stream));
      s.perm = e.d_tile_perm;
      c->launches += 6;
    } else {
      cfree(e.d_tile_perm);
      e.d_tile_perm = nullptr;
      s.perm = nullptr;
    }
    src.push_back(s);
    tiles += (e.n_active + tile_elems(c, e) - 1) / tile_elems(c, e);
  }
  CK(dev::build_tile_plan(src.data(), (int)src.size(), c->n_blocks, c->n_rows, c->d_row_ptr, c->d_col_idx, &c->tplan,
                          c->stream));
  c->launches += 4 * src.size() + 24;
  dalloc(&c->d_partials, (std::size_t)c->tplan.h.n_partials * c->b * c->b);
  dalloc(&c->d_gpartials, (std::size_t)c->tplan.g.n_partials * c->b);
  dalloc(&c->d_tileE, (std::size_t)std::max<long long>(1, tiles));
  // per-energy plan-slice capacities (shared memory is sized per launch)
  std::vector<int> hs(tiles + 1), hc(tiles + 1), gs(tiles + 1), gc(tiles + 1);
  copy_sync(c, hs.data(), c->tplan.h.tile_seg_ptr, sizeof(int) * (tiles + 1), cudaMemcpyDeviceToHost);
  copy_sync(c, hc.data(), c->tplan.h.tile_con_ptr, sizeof(int) * (tiles + 1), cudaMemcpyDeviceToHost);
  copy_sync(c, gs.data(), c->tplan.g.tile_seg_ptr, sizeof(int) * (tiles + 1), cudaMemcpyDeviceToHost);
  copy_sync(c, gc.data(), c->tplan.g.tile_con_ptr, sizeof(int) * (tiles + 1), cudaMemcpyDeviceToHost);
  for (auto& ep : c->energies) {
    Energy& e = *ep;
    int mx[4] = {0, 0, 0, 0};
    const long long nt = (e.skip || e.n_active == 0) ? 0 : (e.n_active + tile_elems(c, e) - 1) / tile_elems(c, e);
    for (long long t = e.tile_base; t < e.tile_base + nt; ++t) {
      mx[0] = std::max(mx[0], hs[t + 1] - hs[t]);
      mx[1] = std::max(mx[1], gs[t + 1] - gs[t]);
      mx[2] = std::max(mx[2], hc[t + 1] - hc[t]);
      mx[3] = std::max(mx[3], gc[t + 1] - gc[t]);
    }
    // 32-bit words of the u16 slices, each copied as the 16-byte aligned range around it (bulk
    // copy) and starting 16-byte aligned in shared memory
    for (int q = 0; q < 4; ++q) e.cap[q] = ((2 * mx[q] + 30) / 16 + 1) * 4;
    // Metadata prefetch depth of the tile reduction. A thread takes every T-th segment of its
    // tile; with one or two contributions per segment (contact pairs: every block of a pair is its
    // own segment, 10 rounds per thread) a round is much shorter than the metadata's load
    // latency, so a one-deep prefetch exposes it every round (ncu: 21 % of the contact kernel's
    // stall samples). Tiles with many short rounds prefetch four rounds ahead (config 5: depth
    // 1 / 2 / 4 / 6 / 11 on the Hessian segments 14.22 / 14.06 / 13.90 / 14.05 / 14.09 ms with the
    // gradient segments at 4; both at 1: 14.50); tiles with few, long rounds (tets: 3) keep
    // depth 1 (deeper measured slower there: more live registers across the barrier).
    {
      const int T = tile_threads(c, e);
      const int rounds_h = (mx[0] + T - 1) / T, rounds_g = (mx[1] + T - 1) / T;
      int dh = rounds_h >= 6 ? 4 : 1, dg = rounds_g >= 3 ? 4 : 1;
      if (const char* v = std::getenv("SYMEL_META_DEPTH_H")) dh = std::max(1, std::atoi(v));
      if (const char* v = std::getenv("SYMEL_META_DEPTH_G")) dg = std::max(1, std::atoi(v));
      if (dh != e.meta_depth[0] || dg != e.meta_depth[1]) {
        e.meta_depth[0] = dh;
        e.meta_depth[1] = dg;
        for (int v : {V_TILE, V_TILE_SPD, V_TILE_G, V_TILE_SPD_G}) e.k[v] = nullptr;  // owned by the context's cache
      }
    }
    cfree(e.d_gstage);
    e.d_gstage = nullptr;
    if (nt > 0 && tile_global_stage(c, e)) dalloc(&e.d_gstage, (std::size_t)nt * tile_stage_doubles(c, e));
  }
  c->tplan_valid = true;
  ++c->plan_epoch;
  cudaEventRecord(c->ev[1], c->stream);
  cudaEventSynchronize(c->ev[1]);
  float ms = 0;
  cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
  c->timings.pattern_ms += ms;
}

// Fast path: one tile kernel per energy (eval + in-CTA reduction), then the fixed-order
// fix-up of shared blocks (deterministic) or nothing (atomic: per-tile red.add).
//
// The launch sequence of an assemble is a pure function of the context state (buffers, plan,
// kernel arguments incl. the params read at every assemble). It is recorded once as a CUDA
// graph and replayed while that state is unchanged -- one host launch per assemble instead of
// ~12 API calls (small meshes are host-bound: config 1's kernels take 30 of its ~90 us).

struct TileLaunch {
  Compiled* k = nullptr;
  SyArgs a;
  std::size_t smem = 0;
  int stream_slot = 0;  // 0 = main stream, i > 0 = aux[(i - 1) % kAux]
};

// Builds the per-energy tile launches (host only; SoA refresh and buffer allocation happen here,
// before any capture).
std::vector<TileLaunch> tile_launches(symel_cuda_ctx* c, bool atomic) {
  std::vector<TileLaunch> out;
  const int ne = (int)c->energies.size();
  const bool concurrent = !std::getenv("SYMEL_SERIAL_ENERGIES");
  int slot = 0;
  for (int q = 0; q < ne; ++q) {
    Energy& e = *c->energies[q];
    if (e.skip || e.n_active == 0) continue;
    TileLaunch L;
    L.stream_slot = concurrent ? slot : 0;
    ++slot;
    const bool spd = (e.flags & SYMEL_ENERGY_SPD) != 0;
    refresh_soa_rows(c, e);
    Compiled* k = kernel_for(c, e, spd ? V_TILE_SPD : V_TILE);
    SyArgs& a = L.a;
    fill_args(c, e, a);
    a.active = e.d_tile_perm ? e.d_tile_elems : e.d_active;  // elements in tile order
    ensure_soa(c, e);
    ensure_elem_buffers(c, e, false);
    for (const auto& kv : e.d_soa) a.arr[kv.first] = kv.second;
    a.soa_n = e.soa_n;
    a.conn_soa = e.d_conn_soa;
    a.n = e.n_active;
    a.grad = c->d_grad;
    a.vals = c->d_vals;
    a.bad_elem = c->d_bad + q;
    a.tile_seg_ptr = c->tplan.h.tile_seg_ptr;
    a.seg_block = c->tplan.h.seg_target;
    a.seg_rel = c->tplan.h.seg_rel;
    a.con = c->tplan.h.con;
    a.seg_dst = c->tplan.h.seg_dst;
    a.seg_mirror = c->tplan.h.seg_mirror;
    a.tile_gseg_ptr = c->tplan.g.tile_seg_ptr;
    a.gseg_row = c->tplan.g.seg_target;
    a.gseg_rel = c->tplan.g.seg_rel;
    a.gcon = c->tplan.g.con;
    a.gseg_dst = c->tplan.g.seg_dst;
    a.partials = c->d_partials;
    a.gpartials = c->d_gpartials;
    a.tileE = c->d_tileE;
    a.tile_base = e.tile_base;
    a.tile_atomic = atomic ? 1 : 0;
    a.tile_con_ptr = c->tplan.h.tile_con_ptr;
    a.tile_gcon_ptr = c->tplan.g.tile_con_ptr;
    a.cap_hseg = e.cap[0];
    a.cap_gseg = e.cap[1];
    a.cap_hcon = e.cap[2];
    a.cap_gcon = e.cap[3];
    a.gstage = e.d_gstage;
    std::size_t plan_bytes = 4 * std::size_t(a.cap_hseg + a.cap_gseg + a.cap_hcon + a.cap_gcon);
    // two CTAs per SM with the plan slice prefetched to shared memory when staging + slice fit
    // half the SM; else two CTAs reading the slice from L2 (scattered tiles: contact pairs)
    if (std::getenv("SYMEL_DEBUG_PLAN"))
      std::fprintf(stderr, "[symel] energy %s: staging %zu B + plan slice %zu B (caps %d %d %d %d words)\n",
                   e.name.c_str(), k->smem, plan_bytes, e.cap[0], e.cap[1], e.cap[2], e.cap[3]);
    if (k->smem + plan_bytes > tile_smem_cta(k->tpb) && !std::getenv("SYMEL_PLAN_SMEM")) {
      k = kernel_for(c, e, spd ? V_TILE_SPD_G : V_TILE_G);
      plan_bytes = 0;
    }
    if (k->smem + plan_bytes > kTileSmemOne)
      throw Fail{SYMEL_E_STATE, "energy '" + e.name + "': tile plan slice exceeds shared memory"};
    L.k = k;
    L.smem = k->smem + plan_bytes;
    if (L.smem > 48 * 1024 && L.smem != k->smem_attr) {  // set here, outside any capture
      CK(cudaKernelSetAttributeForDevice(k->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem,
                                         c->device));
      k->smem_attr = L.smem;
    }
    out.push_back(L);
  }
  return out;
}

// Everything the enqueued operations read from the host side: kernel handles and arguments
// (params by value, device pointers, counts), the tile plan (pointers and counts), the
// context's device buffers and the flags that change the sequence.
std::string tiled_signature(const symel_cuda_ctx* c, const std::vector<TileLaunch>& ls, bool atomic,
                            bool async_tail) {
  std::string sig;
  auto put = [&](const void* p, std::size_t n) { sig.append(static_cast<const char*>(p), n); };
  const int flags[4] = {atomic, async_tail, c->any_pins, (int)c->energies.size()};
  put(flags, sizeof flags);
  for (const TileLaunch& L : ls) {
    put(&L.k, sizeof L.k);
    put(&L.a, sizeof L.a);
    put(&L.smem, sizeof L.smem);
    put(&L.stream_slot, sizeof L.stream_slot);
  }
  put(&c->tplan, sizeof c->tplan);
  const void* bufs[] = {c->d_partials, c->d_gpartials, c->d_vals, c->d_grad, c->d_tileE, c->d_partial,
                        c->d_energy, c->d_bad, c->h_pinned, c->d_pins, c->d_row_ptr, c->d_col_idx};
  put(bufs, sizeof bufs);
  const long long dims[4] = {c->b, c->n_blocks, c->n_dofs, c->n_rows};
  put(dims, sizeof dims);
  for (const auto& ep : c->energies) {
    const long long v[3] = {ep->skip ? 1 : 0, ep->n_active, ep->tile_base};
    put(v, sizeof v);
  }
  return sig;
}

// Events the host or other streams wait on: recorded as real event nodes when captured into
// the assemble graph (a plain record inside a capture only orders the captured work).
cudaError_t record_ext(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal)
                                             : cudaEventRecord(ev, s);
}

// The stream-ordered work of one tiled assemble (everything up to finish_assemble).
void enqueue_tiled(symel_cuda_ctx* c, const std::vector<TileLaunch>& ls, bool atomic, bool async_tail) {
  const int ne = (int)c->energies.size();
  record_ext(c->ev[0], c->stream);
  if (atomic) {
    CK(cudaMemsetAsync(c->d_vals, 0, sizeof(double) * c->n_blocks * c->b * c->b, c->stream));
    CK(cudaMemsetAsync(c->d_grad, 0, sizeof(double) * c->n_dofs, c->stream));
  }
  // energy kernels on separate streams (round robin over main + aux)
  bool aux_used[symel_cuda_ctx::kAux] = {};
  bool forked = false;
  for (const TileLaunch& L : ls) {
    cudaStream_t est = c->stream;
    if (L.stream_slot > 0) {
      if (!forked) CK(cudaEventRecord(c->fork_ev, c->stream));
      forked = true;
      const int i = (L.stream_slot - 1) % symel_cuda_ctx::kAux;
      est = c->aux[i];
      if (!aux_used[i]) CK(cudaStreamWaitEvent(est, c->fork_ev, 0));
      aux_used[i] = true;
    }
    SyArgs a = L.a;
    launch(c, L.k, a, a.n, L.smem, est);
  }
  for (int i = 0; i < symel_cuda_ctx::kAux; ++i)
    if (aux_used[i]) {
      CK(cudaEventRecord(c->join_ev[i], c->aux[i]));
      CK(cudaStreamWaitEvent(c->stream, c->join_ev[i], 0));
    }
  record_ext(c->ev[1], c->stream);
  // gradient rows first, then the energy: both final before the (larger) Hessian fix-up
  if (!atomic) {
    CK(dev::tile_fixup(c->tplan, c->d_partials, c->d_gpartials, c->b, c->d_vals, c->d_grad, c->stream, 2));
    c->launches += (c->tplan.g.n_pt > 0) + (c->tplan.g.n_untouched > 0);
  }
  for (int q = 0; q < ne; ++q) {
    Energy& e = *c->energies[q];
    if (e.skip || e.n_active == 0) continue;
    const long long nt = (e.n_active + tile_elems(c, e) - 1) / tile_elems(c, e);
    CK(dev::tile_energy(c->d_tileE, e.tile_base, nt, c->d_partial, c->d_energy + q, c->stream));
    c->launches += dev::energy_tree_launches(nt);
  }
  CK(dev::energy_combine(c->d_energy, ne, c->d_energy + ne, c->stream));
  ++c->launches;
  if (async_tail) {
    CK(record_ext(c->grad_ready, c->stream));
    CK(cudaMemcpyAsync(c->h_pinned, c->d_energy + ne, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(c->h_pinned + 1, c->d_bad, sizeof(int) * ne, cudaMemcpyDeviceToHost, c->stream));
    CK(record_ext(c->e_ready, c->stream));
    CK(dev::tile_fixup(c->tplan, c->d_partials, c->d_gpartials, c->b, c->d_vals, c->d_grad, c->stream, 1));
    c->launches += (c->tplan.h.n_pt > 0) + (c->tplan.h.n_untouched > 0);
    return;
  }
  if (!atomic) {
    CK(dev::tile_fixup(c->tplan, c->d_partials, c->d_gpartials, c->b, c->d_vals, c->d_grad, c->stream, 1));
    c->launches += (c->tplan.h.n_pt > 0) + (c->tplan.h.n_untouched > 0);
  }
  if (c->any_pins) {
    CK(dev::apply_pins(c->d_pins, c->n_rows, c->b, c->d_row_ptr, c->d_col_idx, c->d_vals, c->d_grad, c->stream));
    ++c->launches;
  }
  CK(record_ext(c->grad_ready, c->stream));
}

double assemble_tiled(symel_cuda_ctx* c, bool atomic, symel_cuda_status* st) {
  const bool async_tail = !atomic && !c->any_pins && !std::getenv("SYMEL_SYNC_ASSEMBLE");
  const std::vector<TileLaunch> ls = tile_launches(c, atomic);
  const bool graphs = !std::getenv("SYMEL_NO_GRAPH");
  if (!graphs) {
    enqueue_tiled(c, ls, atomic, async_tail);
    return finish_assemble(c, st, async_tail);
  }
  std::string sig = tiled_signature(c, ls, atomic, async_tail);
  symel_cuda_ctx::AsmGraph* gr = nullptr;
  for (auto& g : c->graphs)
    if (g.sig == sig) gr = &g;
  if (!gr) {
    // record: at most kGraphs kept (alternating modes replay without re-recording); the least
    // recently used one is replaced
    constexpr std::size_t kGraphs = 4;
    if (c->graphs.size() >= kGraphs) {
      auto lru = std::min_element(c->graphs.begin(), c->graphs.end(),
                                  [](const auto& x, const auto& y) { return x.used < y.used; });
      if (lru->exec) cudaGraphExecDestroy(lru->exec);
      c->graphs.erase(lru);
    }
    const long long l0 = c->launches;
    CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
    try {
      enqueue_tiled(c, ls, atomic, async_tail);
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(c->stream, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    cudaGraph_t g = nullptr;
    CK(cudaStreamEndCapture(c->stream, &g));
    symel_cuda_ctx::AsmGraph ng;
    const cudaError_t ie = cudaGraphInstantiate(&ng.exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) throw Fail{SYMEL_E_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ie)};
    ng.sig = std::move(sig);
    ng.launches = c->launches - l0;
    c->launches = l0;
    c->graphs.push_back(std::move(ng));
    gr = &c->graphs.back();
  }
  gr->used = ++c->graph_clock;
  CK(cudaGraphLaunch(gr->exec, c->stream));
  c->launches += gr->launches;
  return finish_assemble(c, st, async_tail);
}

double do_assemble(symel_cuda_ctx* c, std::uint32_t flags, symel_cuda_status* st) {
  c->assembled = false;
  prepare(c);
  refresh_activation(c);
  if (c->pattern_dirty) build_pattern(c);
  const std::uint32_t mode = flags & 3u;
  const bool ordered = mode == SYMEL_ASM_ORDERED;
  const bool atomic = mode == SYMEL_ASM_ATOMIC;
  const int ne = (int)c->energies.size();
  if (!c->d_energy) {
    dalloc(&c->d_energy, 64);
    dalloc(&c->d_bad, 64);
    CK(cudaMallocHost((void**)&c->h_pinned, 1024));
  }
  if (ne > 60) throw Fail{SYMEL_E_ARG, "too many energies"};
  // "no non-finite element" sentinel (every byte 0x7f: larger than any element id), set without
  // a host->device copy
  CK(cudaMemsetAsync(c->d_bad, 0x7f, sizeof(int) * ne, c->stream));
  CK(cudaMemsetAsync(c->d_energy, 0, sizeof(double) * (ne + 1), c->stream));
  // fast modes run the tile kernel (K3) when every energy's staged element fits a CTA
  bool any_spd = false;
  for (auto& ep : c->energies) any_spd = any_spd || (ep->flags & SYMEL_ENERGY_SPD);
  // the SPD projection runs as its own pass over staged element outputs (contrib path)
  (void)any_spd;  // SPD energies run fused (V_TILE_SPD) when they have a reduced form
  const bool tiled = !ordered && !std::getenv("SYMEL_NO_TILE") && all_tile_capable(c);
  c->last_tiled = tiled;
  if (tiled) {
    ensure_tile_plan(c);
    return assemble_tiled(c, atomic, st);
  }
  if (!atomic) ensure_refs(c);

  cudaEventRecord(c->ev[0], c->stream);
  if (atomic) {
    CK(cudaMemsetAsync(c->d_vals, 0, sizeof(double) * c->n_blocks * c->b * c->b, c->stream));
    CK(cudaMemsetAsync(c->d_grad, 0, sizeof(double) * c->n_dofs, c->stream));
  }
  for (int q = 0; q < ne; ++q) {
    Energy& e = *c->energies[q];
    if (e.skip || e.n_active == 0) continue;
    const bool spd = (e.flags & SYMEL_ENERGY_SPD) != 0;
    const bool staged = !atomic || spd;  // element outputs go through the contrib buffer
    ensure_elem_buffers(c, e, staged);
    Compiled* k = kernel_for(c, e, !staged ? V_ATOMIC : (ordered ? V_CONTRIB_IEEE : V_CONTRIB_FAST));
    SyArgs a;
    fill_args(c, e, a);
    a.active = e.d_active;
    a.n = e.n_active;
    a.contrib = e.d_contrib;
    a.elemE = e.d_elemE;
    a.grad = c->d_grad;
    a.vals = c->d_vals;
    a.slots = e.d_slots;
    a.bad_elem = c->d_bad + q;
    launch(c, k, a, e.n_active);
    if (spd) {  // K2: per-element projection of the element Hessian, in place
      CK(dev::spd_project_contrib(e.d_contrib, e.deriv.n_outputs, (int)e.dof_slots.size(), e.n_active, c->stream));
      ++c->launches;
    }
    if (atomic && spd) {
      CK(dev::scatter_atomic_contrib(e.d_contrib, e.deriv.n_outputs, (int)e.dof_slots.size(), lb_desc(c, e),
                                     e.d_slots, c->conns[e.conn].d, e.d_active, e.n_active, c->d_vals, c->d_grad,
                                     c->stream));
      ++c->launches;
    }
  }
  cudaEventRecord(c->ev[1], c->stream);
  // phase 2: scatter (non-atomic), energy, pins
  if (!atomic) {
    std::vector<dev::ContribLayout> lay;
    long long ord = 0;
    for (auto& ep : c->energies) {
      Energy& e = *ep;
      if (e.skip) continue;
      dev::ContribLayout L{};
      L.ord_base = ord;
      L.ord_end = ord + e.n_active;
      ord += e.n_active;
      L.contrib = e.d_contrib;
      L.stride = (int)e.deriv.n_outputs;
      L.n_dofs = (int)e.dof_slots.size();
      L.n_lb = (int)e.bm.n_lb;
      L.b = c->b;
      std::memset(L.dof_of, -1, sizeof L.dof_of);
      for (std::size_t k = 0; k < e.dof_slots.size(); ++k)
        L.dof_of[e.bm.lb_of_dof[k] * 3 + e.bm.entry_of_dof[k]] = (signed char)k;
      lay.push_back(L);
    }
    if (lay.size() > 8) throw Fail{SYMEL_E_ARG, "ordered scatter supports up to 8 energies"};
    CK(dev::ordered_scatter(lay.data(), (int)lay.size(), c->refs, c->n_blocks, c->n_rows, c->d_vals, c->d_grad,
                            c->stream));
    c->launches += 2;
  }
  if (ordered) {
    std::vector<const double*> ptrs;
    std::vector<long long> strides, counts;
    for (auto& ep : c->energies) {
      if (ep->skip || ep->n_active == 0) continue;
      ptrs.push_back(ep->d_contrib);
      strides.push_back(ep->deriv.n_outputs);
      counts.push_back(ep->n_active);
    }
    CK(dev::energy_serial(ptrs.data(), strides.data(), counts.data(), (int)ptrs.size(), c->d_energy + ne, c->stream));
    c->launches += 2 * ptrs.size();
    for (int q = 0; q < ne; ++q) {  // per-energy parts (symel_cuda_energy_parts), fixed-shape trees
      Energy& e = *c->energies[q];
      if (e.skip || e.n_active == 0) continue;
      CK(dev::energy_tree(e.d_contrib, e.deriv.n_outputs, e.n_active, c->d_partial, c->d_energy + q, c->stream));
      c->launches += dev::energy_tree_launches(e.n_active);
    }
  } else {
    for (int q = 0; q < ne; ++q) {
      Energy& e = *c->energies[q];
      if (e.skip || e.n_active == 0) continue;
      const bool staged = !atomic || (e.flags & SYMEL_ENERGY_SPD);
      const double* v = staged ? e.d_contrib : e.d_elemE;
      const long long stride = staged ? e.deriv.n_outputs : 1;
      CK(dev::energy_tree(v, stride, e.n_active, c->d_partial, c->d_energy + q, c->stream));
      c->launches += dev::energy_tree_launches(e.n_active);
    }
    CK(dev::energy_combine(c->d_energy, ne, c->d_energy + ne, c->stream));
    ++c->launches;
  }
  if (c->any_pins) {
    CK(dev::apply_pins(c->d_pins, c->n_rows, c->b, c->d_row_ptr, c->d_col_idx, c->d_vals, c->d_grad, c->stream));
    ++c->launches;
  }
  return finish_assemble(c, st);
}

// E + finiteness readback, timings, the check_finite contract (assembly.hpp:426-438).
void settle_timings(symel_cuda_ctx* c) {
  if (!c->timings_pending) return;
  cudaEventSynchronize(c->ev[2]);
  float m1 = 0, m2 = 0;
  cudaEventElapsedTime(&m1, c->ev[0], c->ev[1]);
  cudaEventElapsedTime(&m2, c->ev[1], c->ev[2]);
  c->timings.eval_ms = m1;
  c->timings.assemble_ms = m2;
  c->timings_pending = false;
}

double finish_assemble(symel_cuda_ctx* c, symel_cuda_status* st, bool async_tail) {
  const int ne = (int)c->energies.size();
  if (async_tail) {  // E / bad already copied behind e_ready; the Hessian fix-up runs on
    cudaEventRecord(c->ev[2], c->stream);
    CK(cudaEventSynchronize(c->e_ready));
  } else {
    cudaEventRecord(c->ev[2], c->stream);
    CK(cudaMemcpyAsync(c->h_pinned, c->d_energy + ne, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(c->h_pinned + 1, c->d_bad, sizeof(int) * ne, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  c->timings_pending = true;
  if (!async_tail) settle_timings(c);
  const double E = c->h_pinned[0];
  const int* bad = reinterpret_cast<const int*>(c->h_pinned + 1);
  if (st) *st = symel_cuda_status{SYMEL_OK, -1, -1};
  for (int q = 0; q < ne; ++q) {
    if (bad[q] != kNoBadElem) {
      const Energy& e = *c->energies[q];
      const int64_t el = element_of(c, e, bad[q]);
      if (st) *st = symel_cuda_status{SYMEL_E_NONFINITE, q, el};
      throw Fail{SYMEL_E_NONFINITE, "energy '" + e.name + "': non-finite derivative output at element " + std::to_string(el)};
    }
  }
  c->last_E = E;
  c->assembled = true;
  return E;
}

// ------------------------------------------------------------- solver

void free_solver(symel_cuda_ctx* c) {
  dev::SolverWork& w = c->solver;
  cfree(w.x); cfree(w.r); cfree(w.z); cfree(w.p); cfree(w.q); cfree(w.inv); cfree(w.partials);
  cfree(w.ticket); cfree(w.sc);
  w = dev::SolverWork{};
}

dev::SolverWork& ensure_solver(symel_cuda_ctx* c) {
  if (c->device < 0) throw Fail{SYMEL_E_NODEVICE, "no CUDA device"};
  if (!c->assembled) throw Fail{SYMEL_E_STATE, "solver: no assembled Hessian (call assemble first)"};
  dev::SolverWork& w = c->solver;
  if (w.n == c->n_dofs && w.x) return w;
  free_solver(c);
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
  const long long n = c->n_dofs;
  w.vec_grid = (int)std::max<long long>(1, std::min<long long>((c->n_rows + 255) / 256, 8LL * nsm));
  w.max_partials = (int)std::max<long long>(w.vec_grid, dev::spmv_partials_needed(c->b, c->n_rows));
  dalloc(&w.x, n); dalloc(&w.r, n); dalloc(&w.z, n); dalloc(&w.p, n); dalloc(&w.q, n);
  dalloc(&w.inv, (std::size_t)c->n_rows * c->b * c->b);
  dalloc(&w.partials, 2 * (std::size_t)w.max_partials);
  dalloc(&w.ticket, 1);
  dalloc(&w.sc, 1);
  CK(cudaMemsetAsync(w.ticket, 0, sizeof(unsigned), c->stream));
  w.n = n;
  return w;
}

// A pointer argument of the solver calls: device memory (SYMEL_PTR_DEVICE) or host memory
// staged through the given device buffer.
const double* stage_in(symel_cuda_ctx* c, const double* p, double* dev_buf, std::uint32_t flags) {
  if (flags & SYMEL_PTR_DEVICE) return p;
  CK(cudaMemcpyAsync(dev_buf, p, sizeof(double) * c->n_dofs, cudaMemcpyHostToDevice, c->stream));
  return dev_buf;
}

template <class F>
int guarded(symel_cuda_ctx* c, F&& f) {
  if (!c) return SYMEL_E_ARG;
  try {
    f();
    return SYMEL_OK;
  } catch (const Fail& e) {
    c->err = e.msg;
    return e.code;
  } catch (const TapeError& e) {
    c->err = e.what();
    return SYMEL_E_TAPE;
  } catch (const std::exception& e) {
    c->err = e.what();
    return SYMEL_E_ARG;
  }
}

TapeIR energy_only_tape(const TapeIR& d) {
  TapeIR t = d;
  t.out_regs = {d.out_regs.at(0)};
  t.n_outputs = 1;
  return t;
}

}  // namespace

// =========================================================================== C ABI

extern "C" {

int symel_cuda_abi_version(void) { return SYMEL_CUDA_ABI_VERSION; }

int symel_cuda_create(int device, symel_cuda_ctx** out) {
  if (!out) return SYMEL_E_ARG;
  *out = nullptr;
  auto c = std::make_unique<symel_cuda_ctx>();
  int n = 0;
  if (device < 0) {
    c->device = -1;  // codegen-only context: NVRTC compile + cache, no launches
  } else if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    g_create_error = "no CUDA device available (the device path has no CPU fallback)";
    return SYMEL_E_NODEVICE;
  } else {
    if (device >= n) return SYMEL_E_ARG;
    c->device = device;
    if (cudaSetDevice(device) != cudaSuccess) return SYMEL_E_CUDA;
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return SYMEL_E_CUDA;
    for (auto& ev : c->ev) cudaEventCreate(&ev);
    for (auto& st : c->aux) cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming);
    cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&c->grad_ready, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->e_ready, cudaEventDisableTiming);
    for (auto& ev : c->join_ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  }
  if (const char* d = std::getenv("SYMEL_CUDA_CACHE")) c->cache_dir = d;
  *out = c.release();
  return SYMEL_OK;
}

void symel_cuda_destroy(symel_cuda_ctx* c) {
  if (!c) return;
  if (c->device >= 0) {
    cudaStreamSynchronize(c->stream);
    for (Array& a : c->arrays) cfree(a.d);
    for (Conn& k : c->conns) cfree(k.d);
    for (auto& e : c->energies) {
      cfree(e->d_mask); cfree(e->d_active); cfree(e->d_slots); cfree(e->d_contrib); cfree(e->d_elemE);
      cfree(e->d_values); cfree(e->d_changed); cfree(e->d_tile_perm); cfree(e->d_tile_elems); cfree(e->d_gstage);
      for (auto& kv : e->d_soa) cfree(kv.second);
      for (auto& kv : e->d_soa_rowlist) cfree(kv.second);
      cfree(e->d_conn_soa);
    }
    cfree(c->d_row_ptr); cfree(c->d_col_idx); cfree(c->d_vals); cfree(c->d_grad); cfree(c->d_pins);
    for (auto& g : c->graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
    cfree(c->d_partial); cfree(c->d_energy); cfree(c->d_bad);
    if (c->refs_valid) dev::free_ordered_refs(&c->refs);
    if (c->tplan_valid) dev::free_tile_plan(&c->tplan);
    cfree(c->d_partials); cfree(c->d_gpartials); cfree(c->d_tileE);
    free_solver(c);
    if (c->h_pinned) cudaFreeHost(c->h_pinned);
    for (auto& kv : c->kcache)
      if (kv.second->lib) cudaLibraryUnload(kv.second->lib);
    for (auto& ev : c->ev) if (ev) cudaEventDestroy(ev);
    for (auto& ev : c->join_ev) if (ev) cudaEventDestroy(ev);
    if (c->fork_ev) cudaEventDestroy(c->fork_ev);
    if (c->grad_ready) cudaEventDestroy(c->grad_ready);
    if (c->e_ready) cudaEventDestroy(c->e_ready);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    for (auto& st : c->aux) if (st) cudaStreamDestroy(st);
    cudaStreamDestroy(c->stream);
  }
  delete c;
}

const char* symel_cuda_last_error(const symel_cuda_ctx* c) {
  return c ? c->err.c_str() : g_create_error.c_str();
}

int symel_cuda_set_cache_dir(symel_cuda_ctx* c, const char* dir) {
  return guarded(c, [&] { c->cache_dir = dir ? dir : ""; });
}

int symel_cuda_cache_stats(symel_cuda_ctx* c, uint64_t* out4) {
  return guarded(c, [&] {
    if (!out4) throw Fail{SYMEL_E_ARG, "cache_stats: null output"};
    out4[0] = c->cache_stats.builds;
    out4[1] = c->cache_stats.memory_hits;
    out4[2] = c->cache_stats.disk_hits;
    out4[3] = c->cache_stats.corrupt;
  });
}

int symel_cuda_add_array(symel_cuda_ctx* c, const char* name, uint64_t items, uint32_t comps, int is_dof, int* id) {
  return guarded(c, [&] {
    if (comps == 0) throw Fail{SYMEL_E_ARG, std::string("array '") + (name ? name : "") + "': component count must be positive"};
    for (const Array& a : c->arrays)
      if (a.name == name) throw Fail{SYMEL_E_ARG, "array '" + a.name + "' already registered"};
    if (c->arrays.size() >= 24) throw Fail{SYMEL_E_ARG, "too many arrays (max 24)"};
    Array a;
    a.name = name ? name : "";
    a.items = items;
    a.comps = comps;
    a.is_dof = is_dof != 0;
    if (c->device >= 0) {
      dalloc(&a.d, (std::size_t)(items * comps));
      // zeroed (EnergySystem::add_array, registry.hpp:338) and complete before returning:
      // set_array uploads on the copy stream, which must not race this memset
      CK(cudaMemsetAsync(a.d, 0, sizeof(double) * items * comps, c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
    c->arrays.push_back(a);
    c->topology_dirty = true;
    if (id) *id = (int)c->arrays.size() - 1;
  });
}

static Array& array_of(symel_cuda_ctx* c, int id) {
  if (id < 0 || id >= (int)c->arrays.size()) throw Fail{SYMEL_E_ARG, "invalid array handle"};
  return c->arrays[id];
}

int symel_cuda_set_array(symel_cuda_ctx* c, int id, const double* host, uint64_t count) {
  return guarded(c, [&] {
    Array& a = array_of(c, id);
    if (count != a.items * a.comps) throw Fail{SYMEL_E_ARG, "array '" + a.name + "': size mismatch"};
    if (c->device < 0) throw Fail{SYMEL_E_NODEVICE, "no CUDA device"};
    // on the copy stream, after the last assemble's element kernels (grad_ready): the upload
    // overlaps a still running Hessian fix-up, which never reads the state arrays
    CK(cudaStreamWaitEvent(c->copy_stream, c->grad_ready, 0));
    CK(cudaMemcpyAsync(a.d, host, sizeof(double) * count, cudaMemcpyHostToDevice, c->copy_stream));
    CK(cudaStreamSynchronize(c->copy_stream));
    ++a.version;
  });
}

int symel_cuda_get_array(symel_cuda_ctx* c, int id, double* host, uint64_t count) {
  return guarded(c, [&] {
    Array& a = array_of(c, id);
    if (count != a.items * a.comps) throw Fail{SYMEL_E_ARG, "array '" + a.name + "': size mismatch"};
    if (c->device < 0) throw Fail{SYMEL_E_NODEVICE, "no CUDA device"};
    CK(cudaMemcpyAsync(host, a.d, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int symel_cuda_array_device_ptr(symel_cuda_ctx* c, int id, double** p) {
  return guarded(c, [&] {
    Array& a = array_of(c, id);
    a.external = true;  // may be written behind our back: SoA copies refresh every assemble
    *p = a.d;
  });
}

int symel_cuda_add_connectivity(symel_cuda_ctx* c, const char* name, uint32_t arity, int* id) {
  return guarded(c, [&] {
    if (arity == 0) throw Fail{SYMEL_E_ARG, std::string("connectivity '") + (name ? name : "") + "': arity must be positive"};
    Conn k;
    k.name = name ? name : "";
    k.arity = arity;
    c->conns.push_back(k);
    c->topology_dirty = true;
    if (id) *id = (int)c->conns.size() - 1;
  });
}

int symel_cuda_set_elements(symel_cuda_ctx* c, int id, const int64_t* flat, uint64_t n_elems) {
  return guarded(c, [&] {
    if (id < 0 || id >= (int)c->conns.size()) throw Fail{SYMEL_E_ARG, "invalid connectivity handle"};
    Conn& k = c->conns[id];
    std::vector<int> v((std::size_t)(n_elems * k.arity));
    for (std::size_t i = 0; i < v.size(); ++i) {
      if (flat[i] < 0 || flat[i] > INT_MAX)
        throw Fail{SYMEL_E_ARG, "connectivity '" + k.name + "': element " + std::to_string(i / k.arity) +
                                    " references item " + std::to_string(flat[i]) + " outside the int32 range"};
      v[i] = (int)flat[i];
    }
    k.n = n_elems;
    ++k.version;
    if (c->device >= 0) {
      dalloc(&k.d, v.size());
      copy_sync(c, k.d, v.data(), sizeof(int) * v.size(), cudaMemcpyHostToDevice);
    }
    c->topology_dirty = true;
  });
}

int symel_cuda_add_energy(symel_cuda_ctx* c, const char* name, int conn_id, const uint8_t* deriv_tape, uint64_t deriv_len,
                          const symel_input_src* inputs, uint32_t n_inputs, const uint32_t* dof_slots, uint32_t n_dofs,
                          const double* sum_items, uint32_t n_items, uint32_t sum_arity, const uint8_t* act_tape,
                          uint64_t act_len, int act_kind, const uint8_t* guard_tape, uint64_t guard_len, int* id) {
  return guarded(c, [&] {
    auto e = std::make_unique<Energy>();
    e->name = name ? name : "";
    for (auto& d : c->energies)
      if (d->name == e->name) throw Fail{SYMEL_E_ARG, "energy '" + e->name + "' already registered"};
    if (conn_id < 0 || conn_id >= (int)c->conns.size()) throw Fail{SYMEL_E_ARG, "invalid connectivity handle"};
    e->conn = conn_id;
    e->deriv = parse_tape(deriv_tape, deriv_len);
    if (e->deriv.n_inputs != n_inputs) throw Fail{SYMEL_E_ARG, "energy '" + e->name + "': tape input count mismatch"};
    if (e->deriv.n_dofs != n_dofs || e->deriv.n_outputs != 1 + n_dofs + n_dofs * n_dofs)
      throw Fail{SYMEL_E_ARG, "energy '" + e->name + "': cached kernel layout mismatch"};
    const std::uint32_t arity = c->conns[conn_id].arity;
    for (uint32_t k = 0; k < n_inputs; ++k) {
      InputBinding b;
      b.kind = static_cast<InKind>(inputs[k].kind);
      b.array = inputs[k].array;
      b.tuple_slot = inputs[k].tuple_slot;
      b.comp = inputs[k].comp;
      if (inputs[k].kind > 3) throw Fail{SYMEL_E_ARG, "invalid input kind"};
      if ((b.kind == InKind::item_comp || b.kind == InKind::elem_comp) &&
          (b.array >= c->arrays.size() || b.comp >= c->arrays[b.array].comps))
        throw Fail{SYMEL_E_ARG, "energy '" + e->name + "': input " + std::to_string(k) + " binds an invalid array/comp"};
      if (b.kind == InKind::item_comp && b.tuple_slot >= arity)
        throw Fail{SYMEL_E_ARG, "energy '" + e->name + "': tuple slot " + std::to_string(b.tuple_slot) +
                                    " outside connectivity arity " + std::to_string(arity)};
      if (b.kind == InKind::sum_comp && b.tuple_slot >= sum_arity)
        throw Fail{SYMEL_E_ARG, "energy '" + e->name + "': sum item column out of range"};
      e->inputs.push_back(b);
    }
    e->dof_slots.assign(dof_slots, dof_slots + n_dofs);
    for (auto s : e->dof_slots) {
      if (s >= n_inputs || e->inputs[s].kind != InKind::item_comp || !c->arrays[e->inputs[s].array].is_dof)
        throw Fail{SYMEL_E_ARG, "energy '" + e->name + "': dof slot does not bind a dof array item"};
    }
    e->is_sum = sum_arity > 0;
    e->n_items = e->is_sum ? n_items : 0;
    e->sum_arity = sum_arity;
    if (e->is_sum && n_items) e->sum_items.assign(sum_items, sum_items + (std::size_t)n_items * sum_arity);
    e->skip = e->is_sum && n_items == 0;
    e->params.assign(n_inputs, 0.0);
    if (act_tape) {
      e->act = parse_tape(act_tape, act_len);
      e->has_act = true;
      e->act_kind = act_kind;
      if (e->act.n_outputs != 1) throw Fail{SYMEL_E_ARG, "activation tape must have one output"};
    }
    if (guard_tape) {
      e->guard = parse_tape(guard_tape, guard_len);
      e->has_guard = true;
      if (e->guard.n_outputs != 1) throw Fail{SYMEL_E_ARG, "guard tape must have one output"};
    }
    e->eonly = energy_only_tape(e->deriv);
    c->energies.push_back(std::move(e));
    c->topology_dirty = true;
    if (id) *id = (int)c->energies.size() - 1;
  });
}

int symel_cuda_set_param(symel_cuda_ctx* c, int eid, uint32_t slot, double value) {
  return guarded(c, [&] {
    Energy& e = energy_of(c, eid);
    if (slot >= e.inputs.size() || e.inputs[slot].kind != InKind::param)
      throw Fail{SYMEL_E_ARG, "energy '" + e.name + "': input " + std::to_string(slot) + " is not a param"};
    e.params[slot] = value;
  });
}

int symel_cuda_set_energy_flags(symel_cuda_ctx* c, int eid, uint32_t flags) {
  return guarded(c, [&] {
    Energy& e = energy_of(c, eid);
    if (e.flags != flags) {
      e.flags = flags;
      for (auto& k : e.k) k = nullptr;
      e.fact.reset();
      e.fact_tried = false;
      e.fact_spd.reset();
      e.spd_tried = false;
    }
  });
}

int symel_cuda_set_pins(symel_cuda_ctx* c, const uint8_t* mask, uint64_t n) {
  return guarded(c, [&] {
    prepare(c);
    if ((long long)n != c->n_dofs) throw Fail{SYMEL_E_ARG, "pins: mask size mismatch"};
    c->any_pins = false;
    for (uint64_t i = 0; i < n; ++i) c->any_pins = c->any_pins || mask[i];
    dalloc(&c->d_pins, (std::size_t)n);
    copy_sync(c, c->d_pins, mask, n, cudaMemcpyHostToDevice);
  });
}

int symel_cuda_assemble(symel_cuda_ctx* c, uint32_t flags, double* energy, symel_cuda_status* st) {
  if (st) *st = symel_cuda_status{SYMEL_OK, -1, -1};
  return guarded(c, [&] {
    const double E = do_assemble(c, flags, st);
    if (energy) *energy = E;
  });
}

int symel_cuda_energy_only(symel_cuda_ctx* c, double* out) {
  return guarded(c, [&] {
    prepare(c);
    if (c->pattern_dirty) {
      // activation frozen since the last assemble (assembly.hpp:128-139); first call: all
      refresh_activation(c);
      build_pattern(c);
    }
    const int ne = (int)c->energies.size();
    if (!c->d_energy) {
      dalloc(&c->d_energy, 64);
      dalloc(&c->d_bad, 64);
      CK(cudaMallocHost((void**)&c->h_pinned, 1024));
    }
    CK(cudaMemsetAsync(c->d_energy, 0, sizeof(double) * (ne + 1), c->stream));
    for (int q = 0; q < ne; ++q) {
      Energy& e = *c->energies[q];
      if (e.skip || e.n_active == 0) continue;
      ensure_elem_buffers(c, e, false);
      Compiled* k = kernel_for(c, e, V_ENERGY);
      SyArgs a;
      fill_args(c, e, a);
      a.active = e.d_active;
      a.n = e.n_active;
      a.value_out = e.d_elemE;
      launch(c, k, a, e.n_active);
      CK(dev::energy_tree(e.d_elemE, 1, e.n_active, c->d_partial, c->d_energy + q, c->stream));
      c->launches += dev::energy_tree_launches(e.n_active);
    }
    CK(dev::energy_combine(c->d_energy, ne, c->d_energy + ne, c->stream));
    CK(cudaMemcpyAsync(c->h_pinned, c->d_energy + ne, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *out = c->h_pinned[0];
  });
}

int symel_cuda_guard_min(symel_cuda_ctx* c, double* gmin) {
  return guarded(c, [&] {
    prepare(c);
    double best = std::numeric_limits<double>::infinity();
    for (auto& ep : c->energies) {
      Energy& e = *ep;
      if (!e.has_guard || e.skip) continue;
      const long long ne = (long long)c->conns[e.conn].n;
      if (ne == 0) continue;
      if (!e.d_values) dalloc(&e.d_values, (std::size_t)ne);
      Compiled* k = kernel_for(c, e, V_GUARD);
      SyArgs a;
      fill_args(c, e, a);
      a.n = ne;
      a.value_out = e.d_values;
      launch(c, k, a, ne);
      double* d_min = nullptr;
      CK(cudaMallocAsync((void**)&d_min, sizeof(double), c->stream));
      CK(dev::min_reduce(e.d_values, ne, d_min, c->stream));
      double v = 0;
      CK(cudaMemcpyAsync(&v, d_min, sizeof v, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaFreeAsync(d_min, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      best = v < best ? v : best;
    }
    *gmin = best;
  });
}

int symel_cuda_pattern_info(symel_cuda_ctx* c, int* b, uint64_t* nbr, uint64_t* nb, uint64_t* nd) {
  return guarded(c, [&] {
    if (c->topology_dirty) refresh_layout(c);  // b, rows and dofs are known before the first assemble
    if (b) *b = c->b;
    if (nbr) *nbr = (uint64_t)c->n_rows;
    if (nb) *nb = (uint64_t)c->n_blocks;
    if (nd) *nd = (uint64_t)c->n_dofs;
  });
}

int symel_cuda_copy_pattern(symel_cuda_ctx* c, int64_t* row_ptr, int64_t* col_idx) {
  return guarded(c, [&] {
    std::vector<int> rp((std::size_t)c->n_rows + 1), ci((std::size_t)c->n_blocks);
    copy_sync(c, rp.data(), c->d_row_ptr, sizeof(int) * rp.size(), cudaMemcpyDeviceToHost);
    copy_sync(c, ci.data(), c->d_col_idx, sizeof(int) * ci.size(), cudaMemcpyDeviceToHost);
    for (std::size_t i = 0; i < rp.size(); ++i) row_ptr[i] = rp[i];
    for (std::size_t i = 0; i < ci.size(); ++i) col_idx[i] = ci[i];
  });
}

int symel_cuda_copy_gradient(symel_cuda_ctx* c, double* host) {
  return guarded(c, [&] {
    // final once grad_ready fired (possibly while the Hessian fix-up still runs)
    CK(cudaStreamWaitEvent(c->copy_stream, c->grad_ready, 0));
    CK(cudaMemcpyAsync(host, c->d_grad, sizeof(double) * c->n_dofs, cudaMemcpyDeviceToHost, c->copy_stream));
    CK(cudaStreamSynchronize(c->copy_stream));
  });
}

int symel_cuda_copy_hessian(symel_cuda_ctx* c, double* host) {
  return guarded(c, [&] {
    CK(cudaMemcpyAsync(host, c->d_vals, sizeof(double) * c->n_blocks * c->b * c->b, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int symel_cuda_device_results(symel_cuda_ctx* c, const double** g, const double** v, const int32_t** rp,
                              const int32_t** ci) {
  return guarded(c, [&] {
    if (g) *g = c->d_grad;
    if (v) *v = c->d_vals;
    if (rp) *rp = c->d_row_ptr;
    if (ci) *ci = c->d_col_idx;
  });
}

int symel_cuda_matvec(symel_cuda_ctx* c, const double* x, double* y, uint32_t flags) {
  return guarded(c, [&] {
    dev::SolverWork& w = ensure_solver(c);
    const double* xd = stage_in(c, x, w.p, flags);
    double* yd = (flags & SYMEL_PTR_DEVICE) ? y : w.q;
    CK(dev::bsr_spmv(c->b, c->d_row_ptr, c->d_col_idx, c->d_vals, xd, yd, c->n_rows, 0.0, &w, nullptr, c->stream));
    ++c->launches;
    if (!(flags & SYMEL_PTR_DEVICE)) copy_sync(c, y, yd, sizeof(double) * c->n_dofs, cudaMemcpyDeviceToHost);
    else CK(cudaStreamSynchronize(c->stream));
  });
}

int symel_cuda_block_jacobi(symel_cuda_ctx* c, double tau, double* inv, uint32_t flags) {
  return guarded(c, [&] {
    dev::SolverWork& w = ensure_solver(c);
    double* out = (flags & SYMEL_PTR_DEVICE) ? inv : w.inv;
    CK(dev::block_jacobi_inverse(c->b, c->d_row_ptr, c->d_col_idx, c->d_vals, c->n_rows, tau, out, c->stream));
    ++c->launches;
    const std::size_t bytes = sizeof(double) * (std::size_t)c->n_rows * c->b * c->b;
    if (!(flags & SYMEL_PTR_DEVICE)) copy_sync(c, inv, out, bytes, cudaMemcpyDeviceToHost);
    else CK(cudaStreamSynchronize(c->stream));
  });
}

int symel_cuda_pcg(symel_cuda_ctx* c, double tau, const double* rhs, double* x, double rel_tol, int32_t max_iters,
                   uint32_t flags, symel_cuda_pcg_result* res) {
  return guarded(c, [&] {
    if (!res) throw Fail{SYMEL_E_ARG, "pcg: result pointer is null"};
    dev::SolverWork& w = ensure_solver(c);
    *res = symel_cuda_pcg_result{};
    cudaEventRecord(c->ev[0], c->stream);
    const double* rd = stage_in(c, rhs, w.q, flags);  // q is free until the first iteration
    CK(dev::block_jacobi_inverse(c->b, c->d_row_ptr, c->d_col_idx, c->d_vals, c->n_rows, tau, w.inv, c->stream));
    CK(dev::pcg_init(c->b, rd, &w, c->n_rows, c->stream));
    c->launches += 2;
    // rel_tol into the device scalars (staged through the pinned buffer, after the init kernel)
    std::memcpy(c->h_pinned + 64, &rel_tol, sizeof(double));
    CK(cudaMemcpyAsync(&w.sc->tol, c->h_pinned + 64, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    dev::PcgScalars h{};
    auto fetch = [&] {
      CK(cudaMemcpyAsync(c->h_pinned, w.sc, sizeof(dev::PcgScalars), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      std::memcpy(&h, c->h_pinned, sizeof h);
    };
    // Iterations are enqueued in batches; each one checks convergence on the device at its
    // top and becomes a no-op once converged / negative curvature, so the host reads the
    // scalars once per batch and the iteration semantics stay exactly optimizer.hpp:133-157.
    constexpr int kBatch = 16;
    int launched = 0;
    fetch();
    while (!h.done && launched < max_iters) {
      const int nb = std::min(kBatch, max_iters - launched);
      for (int k = 0; k < nb; ++k) {
        CK(dev::pcg_iteration(c->b, c->d_row_ptr, c->d_col_idx, c->d_vals, tau, &w, c->n_rows, launched + k,
                              c->stream));
        c->launches += 4;  // SpMV, partial sum, update, direction
      }
      launched += nb;
      fetch();
    }
    res->iters = h.iters;
    res->converged = h.converged;
    res->neg_curvature = h.neg;
    if (h.done) res->rel_residual = h.converged && h.rhs2 == 0.0 ? 0.0 : h.rel;
    else res->rel_residual = std::sqrt(h.rr) / std::sqrt(h.rhs2);  // iterations exhausted
    cudaEventRecord(c->ev[1], c->stream);
    if (flags & SYMEL_PTR_DEVICE)
      CK(cudaMemcpyAsync(x, w.x, sizeof(double) * c->n_dofs, cudaMemcpyDeviceToDevice, c->stream));
    else
      CK(cudaMemcpyAsync(x, w.x, sizeof(double) * c->n_dofs, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    res->solve_ms = ms;
  });
}

// EnergySystem::gather_dofs / scatter_dofs (registry.hpp:220-238): the flat dof vector in
// layout order (dof arrays in registration order, each items * comps).
int symel_cuda_gather_dofs(symel_cuda_ctx* c, double* u, uint32_t flags) {
  return guarded(c, [&] {
    if (c->device < 0) throw Fail{SYMEL_E_NODEVICE, "no CUDA device"};
    if (c->topology_dirty) refresh_layout(c);
    const cudaMemcpyKind kind = (flags & SYMEL_PTR_DEVICE) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    for (std::size_t i = 0; i < c->arrays.size(); ++i)
      if (c->set_off[i] >= 0)
        CK(cudaMemcpyAsync(u + c->set_off[i], c->arrays[i].d, sizeof(double) * c->arrays[i].items * c->arrays[i].comps,
                           kind, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int symel_cuda_scatter_dofs(symel_cuda_ctx* c, const double* u, uint32_t flags) {
  return guarded(c, [&] {
    if (c->device < 0) throw Fail{SYMEL_E_NODEVICE, "no CUDA device"};
    if (c->topology_dirty) refresh_layout(c);
    const cudaMemcpyKind kind = (flags & SYMEL_PTR_DEVICE) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    for (std::size_t i = 0; i < c->arrays.size(); ++i)
      if (c->set_off[i] >= 0) {
        Array& a = c->arrays[i];
        CK(cudaMemcpyAsync(a.d, u + c->set_off[i], sizeof(double) * a.items * a.comps, kind, c->stream));
        ++a.version;
      }
    CK(cudaStreamSynchronize(c->stream));
  });
}

int symel_cuda_energy_parts(symel_cuda_ctx* c, double* parts, uint32_t n) {
  return guarded(c, [&] {
    if (n != c->energies.size()) throw Fail{SYMEL_E_ARG, "energy_parts: n must equal the number of energies"};
    if (!c->d_energy) throw Fail{SYMEL_E_STATE, "energy_parts: no assemble has run"};
    copy_sync(c, parts, c->d_energy, sizeof(double) * n, cudaMemcpyDeviceToHost);
  });
}

int symel_cuda_active_count(symel_cuda_ctx* c, int eid, uint64_t* n) {
  return guarded(c, [&] { *n = (uint64_t)std::max<long long>(0, energy_of(c, eid).n_active); });
}

int symel_cuda_copy_active(symel_cuda_ctx* c, int eid, uint8_t* mask) {
  return guarded(c, [&] {
    Energy& e = energy_of(c, eid);
    const std::size_t ne = (std::size_t)c->conns[e.conn].n;
    if (!e.has_act || !e.d_mask) {
      std::memset(mask, e.skip ? 0 : 1, ne);
      return;
    }
    copy_sync(c, mask, e.d_mask, ne, cudaMemcpyDeviceToHost);
  });
}

int symel_cuda_element_outputs(symel_cuda_ctx* c, int eid, uint64_t first, uint64_t count, uint32_t flags, double* out) {
  return guarded(c, [&] {
    prepare(c);
    Energy& e = energy_of(c, eid);
    const std::uint64_t ne = c->conns[e.conn].n;
    if (first + count > ne) throw Fail{SYMEL_E_ARG, "element range out of bounds"};
    if (count == 0) return;
    std::vector<int> ids(count);
    for (std::uint64_t i = 0; i < count; ++i) ids[i] = (int)(first + i);
    int* d_ids = nullptr;
    double* d_out = nullptr;
    int* d_bad = nullptr;
    const std::size_t stride = e.deriv.n_outputs;
    CK(cudaMalloc((void**)&d_ids, sizeof(int) * count));
    CK(cudaMalloc((void**)&d_out, sizeof(double) * count * stride));
    CK(cudaMalloc((void**)&d_bad, sizeof(int)));
    copy_sync(c, d_ids, ids.data(), sizeof(int) * count, cudaMemcpyHostToDevice);
    Compiled* k = kernel_for(c, e, (flags & 3u) == SYMEL_ASM_ORDERED ? V_CONTRIB_IEEE : V_CONTRIB_FAST);
    SyArgs a;
    fill_args(c, e, a);
    a.active = d_ids;
    a.n = (long long)count;
    a.contrib = d_out;
    a.bad_elem = d_bad;
    launch(c, k, a, (long long)count);
    CK(cudaMemcpyAsync(out, d_out, sizeof(double) * count * stride, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(d_ids); cudaFree(d_out); cudaFree(d_bad);
  });
}

int symel_cuda_get_timings(symel_cuda_ctx* c, symel_cuda_timings* t) {
  return guarded(c, [&] {
    settle_timings(c);  // waits for the asynchronous Hessian fix-up of the last assemble
    *t = c->timings;
  });
}

int symel_cuda_kernel_source(symel_cuda_ctx* c, int eid, uint32_t flags, char* buf, uint64_t len, uint64_t* needed) {
  return guarded(c, [&] {
    Energy& e = energy_of(c, eid);
    if (c->topology_dirty) refresh_layout(c);
    // the kernel the assemble of this mode runs for the energy (tile kernels: plan slice in
    // shared memory)
    const std::uint32_t mode = flags & 3u;
    Variant v = mode == SYMEL_ASM_ORDERED ? V_CONTRIB_IEEE : (mode == SYMEL_ASM_ATOMIC ? V_ATOMIC : V_CONTRIB_FAST);
    const bool g = flags & SYMEL_SRC_PLAN_GLOBAL;
    if (mode != SYMEL_ASM_ORDERED && tile_ok(c, e)) {
      if (!(e.flags & SYMEL_ENERGY_SPD)) v = g ? V_TILE_G : V_TILE;
      else if (spd_tape(e)) v = g ? V_TILE_SPD_G : V_TILE_SPD;
    }
    const KernelSpec s = spec_for(c, e, v);
    const std::string src = emit_kernel(s);
    if (needed) *needed = src.size() + 1;
    if (buf && len) {
      const std::size_t n = std::min<std::size_t>(len - 1, src.size());
      std::memcpy(buf, src.data(), n);
      buf[n] = '\0';
    }
  });
}

int symel_cuda_energy_info(symel_cuda_ctx* c, int eid, symel_cuda_energy_stats* st) {
  return guarded(c, [&] {
    Energy& e = energy_of(c, eid);
    const TapeIR* ft = fast_tape(e);
    st->tape_ops = e.deriv.instrs.size();
    st->fast_ops = ft->instrs.size();
    st->frontier = e.fact ? e.fact_info.frontier : 0;
    st->n_dofs = (uint32_t)e.dof_slots.size();
    st->n_inputs = e.deriv.n_inputs;
    st->n_outputs = e.deriv.n_outputs;
    st->n_items = e.n_items;
    st->flags = e.flags;
  });
}

int symel_cuda_plan_info(symel_cuda_ctx* c, int64_t* out8) {
  return guarded(c, [&] {
    const dev::TilePlan& p = c->tplan;
    const int64_t v[8] = {p.n_tiles, p.h.n_seg, p.h.n_con, p.h.n_partials, p.h.n_pt, p.g.n_seg, p.g.n_partials, p.g.n_pt};
    std::memcpy(out8, v, sizeof v);
  });
}

int symel_cuda_launch_count(symel_cuda_ctx* c, uint64_t* n) {
  return guarded(c, [&] { *n = c->launches; });
}

int symel_cuda_precompile(symel_cuda_ctx* c, int eid, uint32_t flags) {
  return guarded(c, [&] {
    Energy& e = energy_of(c, eid);
    if (c->topology_dirty) refresh_layout(c);
    const std::uint32_t mode = flags & 3u;
    kernel_for(c, e, mode == SYMEL_ASM_ATOMIC ? V_ATOMIC : (mode == SYMEL_ASM_ORDERED ? V_CONTRIB_IEEE : V_CONTRIB_FAST));
    if (mode != SYMEL_ASM_ORDERED) kernel_for(c, e, V_ENERGY);
    if (mode != SYMEL_ASM_ORDERED && tile_ok(c, e)) {
      if (!(e.flags & SYMEL_ENERGY_SPD)) kernel_for(c, e, V_TILE);
      else if (spd_tape(e)) kernel_for(c, e, V_TILE_SPD);
    }
    if (e.has_act) kernel_for(c, e, V_ACT);
    if (e.has_guard) kernel_for(c, e, V_GUARD);
  });
}

int symel_cuda_fp64_peak(symel_cuda_ctx* c, double* tflops) {
  return guarded(c, [&] {
    if (c->device < 0) throw Fail{SYMEL_E_NODEVICE, "no CUDA device"};
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
    CK(dev::fp64_peak(nsm, tflops, c->stream));
    ++c->launches;
  });
}

int symel_cuda_sync(symel_cuda_ctx* c) {
  return guarded(c, [&] {
    if (c->device >= 0) CK(cudaStreamSynchronize(c->stream));
  });
}

int symel_cuda_stream(symel_cuda_ctx* c, void** s) {
  return guarded(c, [&] { *s = (void*)c->stream; });
}

}  // extern "C"
