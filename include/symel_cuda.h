/*
 * symel_cuda.h — C ABI of libsymel_cuda.so, the B200 (sm_100a) device path for the
 * reference's hot path `Assembler::assemble()` (/root/reference/proj/include/symel/
 * assembly.hpp:108-126): per-element energy / gradient / Hessian evaluation from the
 * reference's Tape IR, optional per-element SPD projection, and assembly into the global
 * gradient and the 3x3 BCRS Hessian.
 *
 * Plain C types only (no torch, no C++ classes). Every entry point returns a status code
 * (SYMEL_OK = 0); symel_cuda_last_error() returns the message of the last failure on that
 * context. One host thread per context; calls are stream-ordered on the context's stream
 * and results are copied to the host only on request (copy_* / assemble's E and status).
 *
 * Reference interfaces each group replaces are cited per declaration.
 */
#ifndef SYMEL_CUDA_H
#define SYMEL_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SYMEL_CUDA_ABI_VERSION 1

typedef struct symel_cuda_ctx symel_cuda_ctx;

/* status codes */
enum {
  SYMEL_OK = 0,
  SYMEL_E_ARG = 1,       /* invalid argument / handle (symel::Error "invalid ... handle") */
  SYMEL_E_CUDA = 2,      /* CUDA runtime / launch failure */
  SYMEL_E_COMPILE = 3,   /* NVRTC failure; message carries the compiler log (kernel.hpp:128-130) */
  SYMEL_E_NONFINITE = 4, /* check_finite (assembly.hpp:426-438): status names energy + element */
  SYMEL_E_STATE = 5,     /* call order (e.g. assemble before any energy) */
  SYMEL_E_TAPE = 6,      /* malformed tape blob (Tape::load checks, tape.hpp:247-291) */
  SYMEL_E_NODEVICE = 7   /* no CUDA device: the product path never falls back to the CPU */
};

/* Input binding kinds = symel::detail::InputKind (registry.hpp:54-59). */
enum {
  SYMEL_IN_ITEM_COMP = 0, /* array[conn[e*arity + tuple_slot]*comps + comp] */
  SYMEL_IN_ELEM_COMP = 1, /* array[e*comps + comp] (bind_element) */
  SYMEL_IN_PARAM = 2,     /* runtime scalar (EnergyBuilder::param), set via set_param */
  SYMEL_IN_SUM_COMP = 3   /* column tuple_slot of the current fixed-summation item */
};

typedef struct {
  uint32_t kind, array, tuple_slot, comp;
} symel_input_src; /* = detail::InputSrc (registry.hpp:61-67) minus the host pointer */

/* Activation comparison = symel::CmpKind (expr.hpp:569): 0 = ge (v >= 0), 1 = gt (v > 0). */

/* Energy flags (symel_cuda_set_energy_flags). */
#define SYMEL_ENERGY_SPD 0x1u   /* project each element Hessian to SPD (clamp eigenvalues < 0) */
#define SYMEL_ENERGY_EXACT 0x2u /* evaluate in the reference's rounding (tape order, IEEE division,
                                   no FMA) in every mode; for ill-conditioned energies */

/* assemble() flags: exactly one assembly mode. */
#define SYMEL_ASM_DETERMINISTIC 0x0u /* fast eval + tile-ordered atomic-free reduction (default) */
#define SYMEL_ASM_ATOMIC 0x1u        /* fast eval + red.global.add.f64 into g and BSR */
#define SYMEL_ASM_ORDERED 0x2u       /* IEEE tape-order eval + the reference's exact per-entry
                                        summation order (assembly.hpp:327-374, 450-462) */

typedef struct {
  int32_t code;    /* SYMEL_OK or SYMEL_E_NONFINITE */
  int32_t energy;  /* first energy (registration order) with a non-finite output, else -1 */
  int64_t element; /* its first element (connectivity index) with a non-finite output */
} symel_cuda_status;

typedef struct {
  double eval_ms;     /* device time of the element kernels (AssembleTimings::eval_ms) */
  double assemble_ms; /* device time of reduction / scatter / energy / pins */
  double pattern_ms;  /* last pattern + slot-map build (amortised; build_pattern) */
  double compile_ms;  /* NVRTC time of the last add_energy (0 on a cache hit) */
} symel_cuda_timings;

/* ---- context (one per device stream) ------------------------------------------------- */
int symel_cuda_abi_version(void);
int symel_cuda_create(int device, symel_cuda_ctx** out);
void symel_cuda_destroy(symel_cuda_ctx* ctx);
const char* symel_cuda_last_error(const symel_cuda_ctx* ctx);
/* Kernel cache directory for <kernel_key>.<variant>.sm100a.cubin (cache.hpp:103-111 analogue);
   NULL or "" disables the disk cache. Default: $SYMEL_CUDA_CACHE or none. */
int symel_cuda_set_cache_dir(symel_cuda_ctx* ctx, const char* dir);
/* CacheStats (cache.hpp:17-24) of this context's kernel cache: {builds, memory_hits, disk_hits,
   corrupt}. Entries are <kernel_key hex>.<variant>.sm100a.cubin + .meta, kernel_key = the tape's
   digest (registry.hpp:415-428, stamped by KernelCache::get_or_build, cache.hpp:78); a corrupt
   entry (meta mismatch, not an image, rejected by the driver) is a warning + rebuild. */
int symel_cuda_cache_stats(symel_cuda_ctx* ctx, uint64_t* out4);

/* ---- state arrays: EnergySystem::add_array / add_dof_array (registry.hpp:124-133) ----- */
/* Dof arrays form the dof layout in registration order (registry.hpp:354-372). */
int symel_cuda_add_array(symel_cuda_ctx* ctx, const char* name, uint64_t items, uint32_t comps,
                         int is_dof, int* array_id);
int symel_cuda_set_array(symel_cuda_ctx* ctx, int array_id, const double* host, uint64_t count);
int symel_cuda_get_array(symel_cuda_ctx* ctx, int array_id, double* host, uint64_t count);
/* Device pointer of an array (zero-copy updates from other device code). */
int symel_cuda_array_device_ptr(symel_cuda_ctx* ctx, int array_id, double** dptr);

/* ---- connectivity: add_connectivity / set_elements (registry.hpp:135-147) ------------- */
int symel_cuda_add_connectivity(symel_cuda_ctx* ctx, const char* name, uint32_t arity, int* conn_id);
/* flat = n_elems * arity item indices (int64 like the reference; validated, stored int32). */
int symel_cuda_set_elements(symel_cuda_ctx* ctx, int conn_id, const int64_t* flat, uint64_t n_elems);

/* ---- energies: EnergySystem::add_energy + compile_kernels (registry.hpp:601-653) -------
 * deriv_tape: SYTP v1 blob of the derivative kernel, outputs [E, g(n), H(n*n)]
 * (diff.hpp:94-104). inputs: one binding per tape input slot. dof_slots: input slots that
 * are dofs, bind order (EnergyDef::dof_slots). sum_items: n_items x sum_arity row-major
 * (EnergyBuilder::sum_items, registry.hpp:507-535) or NULL. act_tape / guard_tape: optional
 * activation (act_kind = CmpKind) and line-search guard kernels (registry.hpp:537-564). */
int symel_cuda_add_energy(symel_cuda_ctx* ctx, const char* name, int conn_id,
                          const uint8_t* deriv_tape, uint64_t deriv_len,
                          const symel_input_src* inputs, uint32_t n_inputs,
                          const uint32_t* dof_slots, uint32_t n_dofs,
                          const double* sum_items, uint32_t n_items, uint32_t sum_arity,
                          const uint8_t* act_tape, uint64_t act_len, int act_kind,
                          const uint8_t* guard_tape, uint64_t guard_len, int* energy_id);
/* Runtime parameter value for a SYMEL_IN_PARAM input slot (read at every assemble). */
int symel_cuda_set_param(symel_cuda_ctx* ctx, int energy_id, uint32_t input_slot, double value);
int symel_cuda_set_energy_flags(symel_cuda_ctx* ctx, int energy_id, uint32_t flags);

/* ---- pins: EnergySystem::pin / clear_pins (registry.hpp:175-191) ----------------------- */
/* mask over global dofs (1 = pinned), applied like apply_pins (assembly.hpp:464-489). */
int symel_cuda_set_pins(symel_cuda_ctx* ctx, const uint8_t* mask, uint64_t n_dofs);

/* ---- assembly: Assembler::assemble / energy_only / guard_min (assembly.hpp:108-173) ---- */
/* Refreshes activation, (re)builds the pattern when topology or activation changed,
 * evaluates every active element, assembles g and the BCRS values on the device and
 * returns E. On a non-finite output returns SYMEL_E_NONFINITE with *status naming the first
 * (energy, element), like check_finite. Deterministic mode returns as soon as E and the
 * gradient are final; the Hessian fix-up may still run on the context stream, and every call
 * of this API that reads the matrix is ordered after it (raw device_results pointers: call
 * symel_cuda_sync first). */
int symel_cuda_assemble(symel_cuda_ctx* ctx, uint32_t flags, double* energy, symel_cuda_status* status);
/* Energy over the currently active elements; non-finite values are returned, not raised. */
int symel_cuda_energy_only(symel_cuda_ctx* ctx, double* energy);
/* Minimum guard over all elements of guarded energies; +inf if none; NaN -> -inf. */
int symel_cuda_guard_min(symel_cuda_ctx* ctx, double* gmin);

/* ---- results ----------------------------------------------------------------------------- */
/* BcrsMatrix shape (assembly.hpp:18-31). */
int symel_cuda_pattern_info(symel_cuda_ctx* ctx, int* b, uint64_t* n_block_rows, uint64_t* n_blocks,
                            uint64_t* n_dofs);
int symel_cuda_copy_pattern(symel_cuda_ctx* ctx, int64_t* row_ptr, int64_t* col_idx);
int symel_cuda_copy_gradient(symel_cuda_ctx* ctx, double* host);
int symel_cuda_copy_hessian(symel_cuda_ctx* ctx, double* host_values);
int symel_cuda_device_results(symel_cuda_ctx* ctx, const double** grad, const double** values,
                              const int32_t** row_ptr, const int32_t** col_idx);
/* ---- Consumer of the assembled Hessian (optimizer.hpp:52-158) -------------
 * All act on the BCRS Hessian of the last successful assemble. Vectors have n_dofs entries;
 * with SYMEL_PTR_DEVICE the pointers are device memory, otherwise host memory. */
#define SYMEL_PTR_DEVICE 0x1u
typedef struct {
  int32_t iters;          /* PcgResult::iters */
  int32_t converged;      /* PcgResult::converged */
  int32_t neg_curvature;  /* PcgResult::neg_curvature */
  int32_t reserved;
  double rel_residual;    /* PcgResult::rel_residual */
  double solve_ms;        /* device time of the solve (CUDA events) */
} symel_cuda_pcg_result;
/* y = H x (BcrsMatrix::matvec, assembly.hpp:43-57). */
int symel_cuda_matvec(symel_cuda_ctx* ctx, const double* x, double* y, uint32_t flags);
/* Inverses of the diagonal blocks + tau I, n_block_rows * b * b doubles, bit for bit as
 * detail::block_jacobi_inverse (optimizer.hpp:52-90). */
int symel_cuda_block_jacobi(symel_cuda_ctx* ctx, double tau, double* inv, uint32_t flags);
/* pcg (optimizer.hpp:119-158): block-Jacobi PCG on (H + tau I) x = rhs from x = 0. */
int symel_cuda_pcg(symel_cuda_ctx* ctx, double tau, const double* rhs, double* x, double rel_tol,
                   int32_t max_iters, uint32_t flags, symel_cuda_pcg_result* res);

/* The flat dof vector (n_dofs doubles, dof arrays in registration order): EnergySystem::
 * gather_dofs / scatter_dofs (registry.hpp:220-238), for a Newton loop on the device. */
int symel_cuda_gather_dofs(symel_cuda_ctx* ctx, double* u, uint32_t flags);
int symel_cuda_scatter_dofs(symel_cuda_ctx* ctx, const double* u, uint32_t flags);

/* Per-energy energy sums of the last assemble / energy_only (fixed-shape tree per energy; the
 * returned E is their sum in energy order). n must equal the number of energies. Used by the
 * sharded multi-GPU assembly, which all-reduces the part of the elements a rank owns. */
int symel_cuda_energy_parts(symel_cuda_ctx* ctx, double* parts, uint32_t n);
/* Active element count of an energy (Assembler::active_count) and the active mask. */
int symel_cuda_active_count(symel_cuda_ctx* ctx, int energy_id, uint64_t* count);
int symel_cuda_copy_active(symel_cuda_ctx* ctx, int energy_id, uint8_t* mask);
/* Raw per-element kernel outputs [E, g, H] (after fixed summation, before SPD) for
 * elements [first, first+count) of an energy's connectivity; for oracle diffing. */
int symel_cuda_element_outputs(symel_cuda_ctx* ctx, int energy_id, uint64_t first, uint64_t count,
                               uint32_t flags, double* out);
int symel_cuda_get_timings(symel_cuda_ctx* ctx, symel_cuda_timings* t);
/* Generated CUDA source of an energy's derivative kernel for a mode (debug / tests / profiling).
 * flags: the assembly mode, | SYMEL_SRC_PLAN_GLOBAL for the tile kernel variant that reads
 * its plan slice from L2 (the one assemble picks when the slice does not fit shared memory). */
#define SYMEL_SRC_PLAN_GLOBAL 0x100u
int symel_cuda_kernel_source(symel_cuda_ctx* ctx, int energy_id, uint32_t flags, char* buf,
                             uint64_t buf_len, uint64_t* needed);
typedef struct {
  uint64_t tape_ops;  /* operations of the reference tape (the algorithmic count) */
  uint64_t fast_ops;  /* operations the fast kernels execute (after factorisation) */
  uint32_t frontier;  /* affine frontier size m of the factorisation, 0 if not factorised */
  uint32_t n_dofs, n_inputs, n_outputs, n_items, flags;
} symel_cuda_energy_stats;
/* Kernel-level facts about one energy (roofline bookkeeping). */
int symel_cuda_energy_info(symel_cuda_ctx* ctx, int energy_id, symel_cuda_energy_stats* st);
/* Tile-plan sizes of the last fast-path assemble: {tiles, block segments, block contributions,
 * block partials, partial blocks, row segments, row partials, partial rows}. */
int symel_cuda_plan_info(symel_cuda_ctx* ctx, int64_t* out8);
/* Number of kernels launched on the device by this context since creation. */
int symel_cuda_launch_count(symel_cuda_ctx* ctx, uint64_t* count);
/* Compile (NVRTC, sm_100a) the kernels an assemble mode needs into the cubin cache without
 * launching anything; works on a device-less context (symel_cuda_create(-1, ...)). */
int symel_cuda_precompile(symel_cuda_ctx* ctx, int energy_id, uint32_t flags);
/* Measured FP64 FMA throughput of this device in TFLOP/s (roofline denominator). */
int symel_cuda_fp64_peak(symel_cuda_ctx* ctx, double* tflops);
/* Synchronise the context stream; raw cudaStream_t for event timing by callers. */
int symel_cuda_sync(symel_cuda_ctx* ctx);
int symel_cuda_stream(symel_cuda_ctx* ctx, void** stream);

#ifdef __cplusplus
}
#endif
#endif /* SYMEL_CUDA_H */
