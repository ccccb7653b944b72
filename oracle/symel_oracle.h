/* TEST INFRASTRUCTURE ONLY (the checker, never the product path).
 * Plain-C restatement of the reference's hot path, /root/reference/proj/include/symel/:
 *   oracle_tape_eval      <- Tape::eval_batch            (tape.hpp:54-113) + powi (expr.hpp:96-101)
 *   oracle_assemble       <- Assembler::assemble         (assembly.hpp:108-126), i.e.
 *                            refresh_activation (227-261), build_pattern (271-375),
 *                            evaluate_active (377-424), check_finite (426-438),
 *                            sum_energy (440-448), scatter (450-462), apply_pins (464-489),
 *                            with gather_element_inputs  (registry.hpp:261-287) and
 *                            element_dofs                (registry.hpp:290-300)
 *   oracle_energy_only / oracle_guard_min <- assembly.hpp:131-173
 *   oracle_bsr_matvec     <- BcrsMatrix::matvec          (assembly.hpp:43-57)
 *   oracle_block_jacobi_inverse / oracle_pcg <- detail::block_jacobi_inverse, pcg
 *                                               (optimizer.hpp:52-90, 119-158)
 * Pinned against the reference itself (oracle/_ref/ref_driver) by tests/test_oracle.py.
 */
#ifndef SYMEL_ORACLE_H
#define SYMEL_ORACLE_H
#include <stdint.h>

typedef struct {
  uint32_t kind, array, tuple_slot, comp; /* 0 item_comp, 1 elem_comp, 2 param, 3 sum_comp */
} oracle_input;

typedef struct {
  const double* data;
  uint64_t items;
  uint32_t comps;
  int32_t is_dof;
} oracle_array;

typedef struct {
  const uint8_t* tape; uint64_t tape_len;          /* derivative kernel [E, g, H] */
  const uint8_t* act_tape; uint64_t act_len; int32_t act_kind;
  const uint8_t* guard_tape; uint64_t guard_len;
  const oracle_input* inputs; uint32_t n_inputs;
  const uint32_t* dof_slots; uint32_t n_dofs;
  const int64_t* conn; uint32_t arity; uint64_t n_elems;
  const double* sum_items; uint32_t n_items, sum_arity; int32_t is_sum;
  const double* params;                            /* per input slot (param kinds) */
} oracle_energy;

typedef struct {
  int32_t status;       /* 0 ok, 4 non-finite, 6 bad tape, 1 bad argument */
  int32_t bad_energy;
  int64_t bad_element;
  double E;
  int32_t b;
  int64_t n_rows, n_blocks, n_dofs;
  int64_t* row_ptr;     /* malloc'ed; free with oracle_free_result */
  int64_t* col_idx;
  double* vals;
  double* grad;
  uint8_t* active;      /* concatenated activation masks, per energy n_elems */
} oracle_result;

/* W-lane batch evaluation, slot-major in[slot*W + lane], out[k*W + lane]. Returns 0 or 6. */
int oracle_tape_eval(const uint8_t* tape, uint64_t len, const double* in, double* out, int64_t W);
int oracle_assemble(const oracle_array* arrays, uint32_t n_arrays, const oracle_energy* energies,
                    uint32_t n_energies, const uint8_t* pins, int32_t threads, oracle_result* res);
/* Per-element raw outputs [E,g,H] (after fixed summation) for elements [first, first+count). */
/* E (serial, reference order), E (Kahan) and the gradient only -- full-size parity checks;
 * returns 0, 4 (non-finite: bad_energy / bad_element) or 6 (bad tape). grad has n_dofs entries. */
int oracle_energy_gradient(const oracle_array* arrays, uint32_t n_arrays, const oracle_energy* energies,
                           uint32_t n_energies, int32_t threads, double* energy, double* energy_kahan, double* grad,
                           int32_t* bad_energy, int64_t* bad_element);
int oracle_element_outputs(const oracle_array* arrays, uint32_t n_arrays, const oracle_energy* e,
                           uint64_t first, uint64_t count, double* out);
int oracle_energy_only(const oracle_array* arrays, uint32_t n_arrays, const oracle_energy* energies,
                       uint32_t n_energies, const uint8_t* active, double* E);
int oracle_guard_min(const oracle_array* arrays, uint32_t n_arrays, const oracle_energy* energies,
                     uint32_t n_energies, double* gmin);
void oracle_free_result(oracle_result* res);
int oracle_bsr_matvec(int32_t b, int64_t n_rows, const int64_t* rp, const int64_t* ci, const double* vals,
                      const double* x, double* y);
int oracle_block_jacobi_inverse(int32_t b, int64_t n_rows, const int64_t* rp, const int64_t* ci,
                                const double* vals, double tau, double* inv);
int oracle_pcg(int32_t b, int64_t n_rows, const int64_t* rp, const int64_t* ci, const double* vals, double tau,
               const double* rhs, double* x, double rel_tol, int32_t max_iters, int32_t* iters,
               int32_t* converged, int32_t* neg_curvature, double* rel_residual);
#endif
