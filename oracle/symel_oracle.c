/* TEST INFRASTRUCTURE ONLY — see symel_oracle.h. Plain C, built with the reference's
 * floating-point contract (-ffp-contract=off, /root/reference/proj/CMakeLists.txt:12-13). */
#include "symel_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ----------------------------------------------------------------- tape (tape.hpp:225-291) */
typedef struct {
  uint8_t op;
  int32_t iarg;
  uint32_t dst, a, b, c;
} instr_t;

typedef struct {
  uint32_t n_inputs, n_outputs, n_dofs, n_regs;
  uint64_t n_consts, n_instrs;
  double* consts;
  instr_t* ins;
  uint32_t* out;
} tape_t;

static uint32_t rd32(const uint8_t* p) { return p[0] | p[1] << 8 | p[2] << 16 | (uint32_t)p[3] << 24; }
static uint64_t rd64(const uint8_t* p) { return rd32(p) | (uint64_t)rd32(p + 4) << 32; }

static void tape_free(tape_t* t) {
  free(t->consts); free(t->ins); free(t->out);
  memset(t, 0, sizeof *t);
}

static int tape_parse(const uint8_t* b, uint64_t n, tape_t* t) {
  memset(t, 0, sizeof *t);
  uint64_t o = 0;
  if (!b || n < 8 + 32 + 16 + 8 || memcmp(b, "SYTP", 4) != 0 || rd32(b + 4) != 1) return 6;
  o = 8 + 32;
  t->n_inputs = rd32(b + o); t->n_outputs = rd32(b + o + 4); t->n_dofs = rd32(b + o + 8); t->n_regs = rd32(b + o + 12);
  o += 16;
  t->n_consts = rd64(b + o); o += 8;
  if (o + 8 * t->n_consts + 8 > n) return 6;
  t->consts = (double*)malloc(8 * (t->n_consts + 1));
  for (uint64_t k = 0; k < t->n_consts; ++k) { uint64_t u = rd64(b + o); memcpy(&t->consts[k], &u, 8); o += 8; }
  t->n_instrs = rd64(b + o); o += 8;
  if (o + 21 * t->n_instrs + 8 > n) { tape_free(t); return 6; }
  t->ins = (instr_t*)malloc(sizeof(instr_t) * (t->n_instrs + 1));
  for (uint64_t k = 0; k < t->n_instrs; ++k) {
    instr_t* i = &t->ins[k];
    i->op = b[o]; i->iarg = (int32_t)rd32(b + o + 1); i->dst = rd32(b + o + 5);
    i->a = rd32(b + o + 9); i->b = rd32(b + o + 13); i->c = rd32(b + o + 17);
    o += 21;
    if (i->op < 2 || i->op > 12 || i->dst >= t->n_regs || i->a >= t->n_regs || i->b >= t->n_regs || i->c >= t->n_regs) {
      tape_free(t); return 6;
    }
  }
  uint64_t no = rd64(b + o); o += 8;
  if (no != t->n_outputs || o + 4 * no > n) { tape_free(t); return 6; }
  t->out = (uint32_t*)malloc(4 * (no + 1));
  for (uint64_t k = 0; k < no; ++k) { t->out[k] = rd32(b + o); o += 4; if (t->out[k] >= t->n_regs) { tape_free(t); return 6; } }
  return 0;
}

/* expr.hpp:96-101: repeated multiply from 1.0, negative exponent -> 1 / powi(x, -n) */
static double powi(double x, long long n) {
  if (n < 0) return 1.0 / powi(x, -n);
  double r = 1.0;
  while (n-- > 0) r *= x;
  return r;
}

/* tape.hpp:54-113, one lane at a time (lanes are bit-identical to single-lane runs) */
static void tape_eval1(const tape_t* t, const double* in, double* out, double* regs) {
  memcpy(regs, in, sizeof(double) * t->n_inputs);
  memcpy(regs + t->n_inputs, t->consts, sizeof(double) * t->n_consts);
  for (uint64_t k = 0; k < t->n_instrs; ++k) {
    const instr_t* i = &t->ins[k];
    const double a = regs[i->a], b = regs[i->b], c = regs[i->c];
    double d;
    switch (i->op) {
      case 2: d = a + b; break;
      case 3: d = a - b; break;
      case 4: d = a * b; break;
      case 5: d = a / b; break;
      case 6: d = -a; break;
      case 7: d = powi(a, i->iarg); break;
      case 8: d = sqrt(a); break;
      case 9: d = log(a); break;
      case 10: d = sin(a); break;
      case 11: d = cos(a); break;
      default: d = a >= 0.0 ? b : c; break; /* branch: NaN selects the else side */
    }
    regs[i->dst] = d;
  }
  for (uint32_t k = 0; k < t->n_outputs; ++k) out[k] = regs[t->out[k]];
}

int oracle_tape_eval(const uint8_t* tape, uint64_t len, const double* in, double* out, int64_t W) {
  tape_t t;
  int rc = tape_parse(tape, len, &t);
  if (rc) return rc;
  double* regs = (double*)malloc(sizeof(double) * (t.n_regs + 1));
  double* one_in = (double*)malloc(sizeof(double) * (t.n_inputs + 1));
  double* one_out = (double*)malloc(sizeof(double) * (t.n_outputs + 1));
  for (int64_t l = 0; l < W; ++l) {
    for (uint32_t s = 0; s < t.n_inputs; ++s) one_in[s] = in[s * W + l];
    tape_eval1(&t, one_in, one_out, regs);
    for (uint32_t k = 0; k < t.n_outputs; ++k) out[k * W + l] = one_out[k];
  }
  free(regs); free(one_in); free(one_out);
  tape_free(&t);
  return 0;
}

/* --------------------------------------------------- gather (registry.hpp:261-287) */
static void gather(const oracle_array* A, const oracle_energy* e, uint64_t elem, const double* item, double* out) {
  const int64_t* tup = e->conn + elem * e->arity;
  for (uint32_t s = 0; s < e->n_inputs; ++s) {
    const oracle_input* src = &e->inputs[s];
    switch (src->kind) {
      case 0: out[s] = A[src->array].data[(uint64_t)tup[src->tuple_slot] * A[src->array].comps + src->comp]; break;
      case 1: out[s] = A[src->array].data[elem * A[src->array].comps + src->comp]; break;
      case 2: out[s] = e->params[s]; break;
      default: out[s] = item[src->tuple_slot]; break;
    }
  }
}

/* raw kernel outputs of one element with fixed summation (assembly.hpp:400-413) */
static void eval_element(const oracle_array* A, const oracle_energy* e, const tape_t* t, uint64_t elem,
                         double* in, double* tmp, double* acc, double* regs) {
  if (e->is_sum) {
    for (uint32_t it = 0; it < e->n_items; ++it) {
      gather(A, e, elem, e->sum_items + (uint64_t)it * e->sum_arity, in);
      tape_eval1(t, in, it == 0 ? acc : tmp, regs);
      if (it > 0)
        for (uint32_t k = 0; k < t->n_outputs; ++k) acc[k] += tmp[k];
    }
  } else {
    gather(A, e, elem, NULL, in);
    tape_eval1(t, in, acc, regs);
  }
}

/* ----------------------------------------------------------------- layout helpers */
typedef struct {
  int64_t* set_off; /* per array, -1 if not dof */
  int64_t n_dofs;
  int b;
} layout_t;

static void make_layout(const oracle_array* A, uint32_t na, layout_t* L) {
  L->set_off = (int64_t*)malloc(sizeof(int64_t) * (na + 1));
  int64_t off = 0;
  int all3 = 1, any = 0;
  for (uint32_t i = 0; i < na; ++i) {
    L->set_off[i] = -1;
    if (!A[i].is_dof) continue;
    any = 1;
    L->set_off[i] = off;
    off += (int64_t)(A[i].items * A[i].comps);
    if (A[i].comps != 3) all3 = 0;
  }
  L->n_dofs = off;
  L->b = (any && all3) ? 3 : 1; /* assembly.hpp:273-276 */
}

/* element_dofs (registry.hpp:290-300): global index of dof k of element elem */
static int64_t elem_dof(const oracle_array* A, const layout_t* L, const oracle_energy* e, uint64_t elem, uint32_t k) {
  const oracle_input* in = &e->inputs[e->dof_slots[k]];
  const int64_t item = e->conn[elem * e->arity + in->tuple_slot];
  return L->set_off[in->array] + item * (int64_t)A[in->array].comps + in->comp;
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

static int64_t find_block(const int64_t* rp, const int64_t* ci, int64_t r, int64_t c) {
  int64_t lo = rp[r], hi = rp[r + 1];
  while (lo < hi) {
    int64_t m = (lo + hi) / 2;
    if (ci[m] < c) lo = m + 1; else hi = m;
  }
  return (lo < rp[r + 1] && ci[lo] == c) ? lo : -1;
}

/* activation value of one element (assembly.hpp:233-246) */
static double act_value(const oracle_array* A, const oracle_energy* e, const tape_t* at, uint64_t elem,
                        double* in, double* regs) {
  double v, o;
  if (e->is_sum) {
    v = -INFINITY;
    for (uint32_t it = 0; it < e->n_items; ++it) {
      gather(A, e, elem, e->sum_items + (uint64_t)it * e->sum_arity, in);
      tape_eval1(at, in, &o, regs);
      v = o > v ? o : v;
    }
  } else {
    gather(A, e, elem, NULL, in);
    tape_eval1(at, in, &o, regs);
    v = o;
  }
  return v;
}

int oracle_assemble(const oracle_array* A, uint32_t na, const oracle_energy* E, uint32_t ne, const uint8_t* pins,
                    int32_t threads, oracle_result* res) {
  memset(res, 0, sizeof *res);
  res->bad_energy = -1;
  res->bad_element = -1;
  layout_t L;
  make_layout(A, na, &L);
  const int b = L.b;
  res->b = b;
  res->n_dofs = L.n_dofs;
  res->n_rows = L.n_dofs / b;
  tape_t* T = (tape_t*)calloc(ne + 1, sizeof(tape_t));
  uint64_t tot_elems = 0;
  for (uint32_t d = 0; d < ne; ++d) {
    if (tape_parse(E[d].tape, E[d].tape_len, &T[d])) { res->status = 6; goto done; }
    tot_elems += E[d].n_elems;
  }
  /* activation (prepare() starts all-active; refresh_activation evaluates the condition) */
  res->active = (uint8_t*)malloc(tot_elems + 1);
  {
    uint64_t off = 0;
    for (uint32_t d = 0; d < ne; ++d) {
      const oracle_energy* e = &E[d];
      const int skip = e->is_sum && e->n_items == 0;
      memset(res->active + off, skip ? 0 : 1, e->n_elems);
      if (e->act_tape && !skip) {
        tape_t at;
        if (tape_parse(e->act_tape, e->act_len, &at)) { res->status = 6; goto done; }
        double* in = (double*)malloc(sizeof(double) * (e->n_inputs + 1));
        double* regs = (double*)malloc(sizeof(double) * (at.n_regs + 1));
        for (uint64_t el = 0; el < e->n_elems; ++el) {
          const double v = act_value(A, e, &at, el, in, regs);
          res->active[off + el] = e->act_kind == 0 ? (v >= 0.0) : (v > 0.0); /* Condition::holds */
        }
        free(in); free(regs);
        tape_free(&at);
      }
      off += e->n_elems;
    }
  }
  /* pattern (assembly.hpp:295-325): diagonal per row + off-diagonal pairs of active elements */
  {
    uint64_t nk = (uint64_t)res->n_rows, cap = nk, off = 0;
    for (uint32_t d = 0; d < ne; ++d) cap += E[d].n_elems * (uint64_t)E[d].n_dofs * E[d].n_dofs;
    uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (cap + 1));
    for (int64_t r = 0; r < res->n_rows; ++r) keys[r] = ((uint64_t)r << 32) | (uint64_t)r;
    uint32_t max_nd = 1;
    for (uint32_t d = 0; d < ne; ++d) max_nd = E[d].n_dofs > max_nd ? E[d].n_dofs : max_nd;
    int64_t* dofs = (int64_t*)malloc(sizeof(int64_t) * max_nd);
    for (uint32_t d = 0; d < ne; ++d) {
      const oracle_energy* e = &E[d];
      for (uint64_t el = 0; el < e->n_elems; ++el) {
        if (!res->active[off + el]) continue;
        for (uint32_t k = 0; k < e->n_dofs; ++k) dofs[k] = elem_dof(A, &L, e, el, k);
        for (uint32_t a = 0; a < e->n_dofs; ++a)
          for (uint32_t c = 0; c < e->n_dofs; ++c) {
            const int64_t br = dofs[a] / b, bc = dofs[c] / b;
            if (br != bc) keys[nk++] = ((uint64_t)br << 32) | (uint64_t)bc;
          }
      }
      off += e->n_elems;
    }
    qsort(keys, nk, sizeof(uint64_t), cmp_u64);
    uint64_t nu = 0;
    for (uint64_t i = 0; i < nk; ++i)
      if (i == 0 || keys[i] != keys[i - 1]) keys[nu++] = keys[i];
    res->n_blocks = (int64_t)nu;
    res->row_ptr = (int64_t*)calloc((size_t)res->n_rows + 2, sizeof(int64_t));
    res->col_idx = (int64_t*)malloc(sizeof(int64_t) * (nu + 1));
    for (uint64_t i = 0; i < nu; ++i) {
      res->col_idx[i] = (int64_t)(keys[i] & 0xffffffffu);
      res->row_ptr[(keys[i] >> 32) + 1]++;
    }
    for (int64_t r = 0; r < res->n_rows; ++r) res->row_ptr[r + 1] += res->row_ptr[r];
    free(keys);
    free(dofs);
  }
  /* phase 1: evaluate active elements into contrib (assembly.hpp:377-424) */
  {
    uint64_t off = 0;
    double** contrib = (double**)calloc(ne + 1, sizeof(double*));
    for (uint32_t d = 0; d < ne; ++d) {
      const oracle_energy* e = &E[d];
      const tape_t* t = &T[d];
      const uint32_t S = t->n_outputs;
      contrib[d] = (double*)malloc(sizeof(double) * (e->n_elems * (uint64_t)S + 1));
      const uint8_t* act = res->active + off;
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
      {
        double* in = (double*)malloc(sizeof(double) * (e->n_inputs + 1));
        double* tmp = (double*)malloc(sizeof(double) * (S + 1));
        double* regs = (double*)malloc(sizeof(double) * (t->n_regs + 1));
#pragma omp for schedule(static)
        for (int64_t el = 0; el < (int64_t)e->n_elems; ++el)
          if (act[el]) eval_element(A, e, t, (uint64_t)el, in, tmp, contrib[d] + (uint64_t)el * S, regs);
        free(in); free(tmp); free(regs);
      }
      off += e->n_elems;
    }
    /* check_finite (assembly.hpp:426-438): first (energy, element) in order */
    off = 0;
    for (uint32_t d = 0; d < ne && res->status == 0; ++d) {
      const uint32_t S = T[d].n_outputs;
      for (uint64_t el = 0; el < E[d].n_elems && res->status == 0; ++el) {
        if (!res->active[off + el]) continue;
        for (uint32_t k = 0; k < S; ++k)
          if (!isfinite(contrib[d][el * S + k])) {
            res->status = 4; res->bad_energy = (int32_t)d; res->bad_element = (int64_t)el;
            break;
          }
      }
      off += E[d].n_elems;
    }
    /* sum_energy (assembly.hpp:440-448) + scatter (450-462) in (energy, element, a, c) order */
    res->vals = (double*)calloc((size_t)(res->n_blocks * b * b) + 1, sizeof(double));
    res->grad = (double*)calloc((size_t)res->n_dofs + 1, sizeof(double));
    double Esum = 0.0;
    uint32_t max_nd = 1;
    for (uint32_t d = 0; d < ne; ++d) max_nd = E[d].n_dofs > max_nd ? E[d].n_dofs : max_nd;
    int64_t* dofs = (int64_t*)malloc(sizeof(int64_t) * max_nd);
    off = 0;
    for (uint32_t d = 0; d < ne; ++d) {
      const oracle_energy* e = &E[d];
      const uint32_t S = T[d].n_outputs, nd = e->n_dofs;
      for (uint64_t el = 0; el < e->n_elems; ++el) {
        if (!res->active[off + el]) continue;
        const double* v = contrib[d] + el * S;
        Esum += v[0];
        for (uint32_t k = 0; k < nd; ++k) dofs[k] = elem_dof(A, &L, e, el, k);
        for (uint32_t a = 0; a < nd; ++a) {
          res->grad[dofs[a]] += v[1 + a];
          for (uint32_t c = 0; c < nd; ++c) {
            const int64_t blk = find_block(res->row_ptr, res->col_idx, dofs[a] / b, dofs[c] / b);
            res->vals[blk * b * b + (dofs[a] % b) * b + (dofs[c] % b)] += v[1 + nd + a * nd + c];
          }
        }
      }
      off += e->n_elems;
      free(contrib[d]);
    }
    free(contrib);
    free(dofs);
    res->E = Esum;
  }
  /* apply_pins (assembly.hpp:464-489) */
  if (pins) {
    int any = 0;
    for (int64_t i = 0; i < res->n_dofs; ++i) any |= pins[i] != 0;
    if (any) {
      for (int64_t i = 0; i < res->n_dofs; ++i)
        if (pins[i]) res->grad[i] = 0.0;
      for (int64_t r = 0; r < res->n_rows; ++r)
        for (int64_t k = res->row_ptr[r]; k < res->row_ptr[r + 1]; ++k) {
          double* v = res->vals + k * b * b;
          const int64_t c = res->col_idx[k];
          for (int i = 0; i < b; ++i)
            for (int j = 0; j < b; ++j)
              if (pins[r * b + i] || pins[c * b + j]) v[i * b + j] = 0.0;
        }
      for (int64_t i = 0; i < res->n_dofs; ++i)
        if (pins[i]) {
          const int64_t k = find_block(res->row_ptr, res->col_idx, i / b, i / b);
          res->vals[k * b * b + (i % b) * b + (i % b)] = 1.0;
        }
    }
  }
done:
  for (uint32_t d = 0; d < ne; ++d) tape_free(&T[d]);
  free(T);
  free(L.set_off);
  return res->status;
}

int oracle_element_outputs(const oracle_array* A, uint32_t na, const oracle_energy* e, uint64_t first, uint64_t count,
                           double* out) {
  (void)na;
  tape_t t;
  if (tape_parse(e->tape, e->tape_len, &t)) return 6;
  double* in = (double*)malloc(sizeof(double) * (e->n_inputs + 1));
  double* tmp = (double*)malloc(sizeof(double) * (t.n_outputs + 1));
  double* regs = (double*)malloc(sizeof(double) * (t.n_regs + 1));
  for (uint64_t q = 0; q < count; ++q) eval_element(A, e, &t, first + q, in, tmp, out + q * t.n_outputs, regs);
  free(in); free(tmp); free(regs);
  tape_free(&t);
  return 0;
}

int oracle_energy_only(const oracle_array* A, uint32_t na, const oracle_energy* E, uint32_t ne, const uint8_t* active,
                       double* Eout) {
  (void)na;
  double s = 0.0;
  uint64_t off = 0;
  for (uint32_t d = 0; d < ne; ++d) {
    tape_t t;
    if (tape_parse(E[d].tape, E[d].tape_len, &t)) return 6;
    double* in = (double*)malloc(sizeof(double) * (E[d].n_inputs + 1));
    double* tmp = (double*)malloc(sizeof(double) * (t.n_outputs + 1));
    double* acc = (double*)malloc(sizeof(double) * (t.n_outputs + 1));
    double* regs = (double*)malloc(sizeof(double) * (t.n_regs + 1));
    for (uint64_t el = 0; el < E[d].n_elems; ++el) {
      if (active && !active[off + el]) continue;
      if (E[d].is_sum && E[d].n_items == 0) continue;
      eval_element(A, &E[d], &t, el, in, tmp, acc, regs);
      s += acc[0];
    }
    off += E[d].n_elems;
    free(in); free(tmp); free(acc); free(regs);
    tape_free(&t);
  }
  *Eout = s;
  return 0;
}

int oracle_guard_min(const oracle_array* A, uint32_t na, const oracle_energy* E, uint32_t ne, double* gmin) {
  (void)na;
  double best = INFINITY;
  for (uint32_t d = 0; d < ne; ++d) {
    const oracle_energy* e = &E[d];
    if (!e->guard_tape) continue;
    tape_t t;
    if (tape_parse(e->guard_tape, e->guard_len, &t)) return 6;
    double* in = (double*)malloc(sizeof(double) * (e->n_inputs + 1));
    double* regs = (double*)malloc(sizeof(double) * (t.n_regs + 1));
    double o;
    for (uint64_t el = 0; el < e->n_elems; ++el) {
      double g = INFINITY;
      if (e->is_sum) {
        if (e->n_items == 0) continue;
        for (uint32_t it = 0; it < e->n_items; ++it) {
          gather(A, e, el, e->sum_items + (uint64_t)it * e->sum_arity, in);
          tape_eval1(&t, in, &o, regs);
          g = o < g ? o : g;
          if (isnan(o)) g = -INFINITY;
        }
      } else {
        gather(A, e, el, NULL, in);
        tape_eval1(&t, in, &o, regs);
        g = isnan(o) ? -INFINITY : o;
      }
      best = g < best ? g : best;
    }
    free(in); free(regs);
    tape_free(&t);
  }
  *gmin = best;
  return 0;
}

void oracle_free_result(oracle_result* r) {
  free(r->row_ptr); free(r->col_idx); free(r->vals); free(r->grad); free(r->active);
  memset(r, 0, sizeof *r);
}

/* ---- consumer of the assembled BCRS: SpMV, block-Jacobi, PCG ---- */

/* y = A x, BcrsMatrix::matvec (assembly.hpp:43-57): per block row, blocks in stored order,
 * acc[i] += v[i*b+j] * x[col*b+j] from 0.0. */
int oracle_bsr_matvec(int32_t b, int64_t n_rows, const int64_t* rp, const int64_t* ci, const double* vals,
                      const double* x, double* y) {
  if (b < 1 || b > 4) return 1;
  for (int64_t r = 0; r < n_rows; ++r) {
    double acc[16] = {0};
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
      const double* v = vals + k * b * b;
      const double* xc = x + ci[k] * b;
      for (int i = 0; i < b; ++i)
        for (int j = 0; j < b; ++j) acc[i] += v[i * b + j] * xc[j];
    }
    for (int i = 0; i < b; ++i) y[r * b + i] = acc[i];
  }
  return 0;
}

/* detail::block_jacobi_inverse (optimizer.hpp:52-90): inverse of each diagonal block + tau I by
 * the adjugate; missing block or unusable determinant -> identity; b = 1: 1/d or 1. */
int oracle_block_jacobi_inverse(int32_t b, int64_t n_rows, const int64_t* rp, const int64_t* ci,
                                const double* vals, double tau, double* inv) {
  if (b != 1 && b != 3) return 1;
  memset(inv, 0, sizeof(double) * (size_t)(n_rows * b * b));
  for (int64_t r = 0; r < n_rows; ++r) {
    const int64_t k = find_block(rp, ci, r, r);
    double* out = inv + r * b * b;
    if (k < 0) {
      for (int i = 0; i < b; ++i) out[i * b + i] = 1.0;
      continue;
    }
    const double* v = vals + k * b * b;
    if (b == 1) {
      const double d = v[0] + tau;
      out[0] = (isfinite(d) && d != 0.0) ? 1.0 / d : 1.0;
      continue;
    }
    double m[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) m[i * 3 + j] = v[i * 3 + j] + (i == j ? tau : 0.0);
    const double det = m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                       m[2] * (m[3] * m[7] - m[4] * m[6]);
    if (!isfinite(det) || fabs(det) < 1e-300) {
      for (int i = 0; i < 3; ++i) out[i * 3 + i] = 1.0;
      continue;
    }
    const double id = 1.0 / det;
    out[0] = (m[4] * m[8] - m[5] * m[7]) * id;
    out[1] = (m[2] * m[7] - m[1] * m[8]) * id;
    out[2] = (m[1] * m[5] - m[2] * m[4]) * id;
    out[3] = (m[5] * m[6] - m[3] * m[8]) * id;
    out[4] = (m[0] * m[8] - m[2] * m[6]) * id;
    out[5] = (m[2] * m[3] - m[0] * m[5]) * id;
    out[6] = (m[3] * m[7] - m[4] * m[6]) * id;
    out[7] = (m[1] * m[6] - m[0] * m[7]) * id;
    out[8] = (m[0] * m[4] - m[1] * m[3]) * id;
  }
  return 0;
}

static double sdot(const double* a, const double* b, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

static void block_apply(const double* blocks, int b, const double* x, double* y, int64_t n_rows) {
  for (int64_t r = 0; r < n_rows; ++r) {
    const double* m = blocks + r * b * b;
    for (int i = 0; i < b; ++i) {
      double acc = 0.0;
      for (int j = 0; j < b; ++j) acc += m[i * b + j] * x[r * b + j];
      y[r * b + i] = acc;
    }
  }
}

/* pcg (optimizer.hpp:119-158): block-Jacobi PCG on (H + tau I) x = rhs from x = 0; stops on
 * rel residual <= rel_tol (checked at the top of every iteration), non-positive curvature (at
 * iteration 0 the preconditioned rhs is returned) or max_iters. */
int oracle_pcg(int32_t b, int64_t n_rows, const int64_t* rp, const int64_t* ci, const double* vals, double tau,
               const double* rhs, double* x, double rel_tol, int32_t max_iters, int32_t* iters,
               int32_t* converged, int32_t* neg_curvature, double* rel_residual) {
  const int64_t n = n_rows * b;
  *iters = 0; *converged = 0; *neg_curvature = 0; *rel_residual = 0.0;
  for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
  const double rhs_norm = sqrt(sdot(rhs, rhs, n));
  if (rhs_norm == 0.0) { *converged = 1; return 0; }
  double* prec = malloc(sizeof(double) * (size_t)(n_rows * b * b));
  double* r = malloc(sizeof(double) * (size_t)n);
  double* z = malloc(sizeof(double) * (size_t)n);
  double* p = malloc(sizeof(double) * (size_t)n);
  double* q = malloc(sizeof(double) * (size_t)n);
  oracle_block_jacobi_inverse(b, n_rows, rp, ci, vals, tau, prec);
  memcpy(r, rhs, sizeof(double) * (size_t)n);
  block_apply(prec, b, r, z, n_rows);
  memcpy(p, z, sizeof(double) * (size_t)n);
  double rz = sdot(r, z, n);
  int done = 0;
  for (int it = 0; it < max_iters && !done; ++it) {
    const double rnorm = sqrt(sdot(r, r, n));
    *rel_residual = rnorm / rhs_norm;
    if (*rel_residual <= rel_tol) { *converged = 1; done = 1; break; }
    oracle_bsr_matvec(b, n_rows, rp, ci, vals, p, q);
    if (tau != 0.0)
      for (int64_t i = 0; i < n; ++i) q[i] += tau * p[i];
    const double pq = sdot(p, q, n);
    if (!(pq > 0.0)) {
      *neg_curvature = 1;
      if (it == 0) memcpy(x, z, sizeof(double) * (size_t)n);
      done = 1;
      break;
    }
    const double alpha = rz / pq;
    for (int64_t i = 0; i < n; ++i) x[i] += alpha * p[i];
    for (int64_t i = 0; i < n; ++i) r[i] -= alpha * q[i];
    block_apply(prec, b, r, z, n_rows);
    const double rz_next = sdot(r, z, n);
    const double beta = rz_next / rz;
    rz = rz_next;
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    ++*iters;
  }
  if (!done) *rel_residual = sqrt(sdot(r, r, n)) / rhs_norm;
  free(prec); free(r); free(z); free(p); free(q);
  return 0;
}

/* ---------------------------------------------------------------------------------------
 * E and gradient only, at full BASELINE sizes (tests/test_gpu_fullsize.py): the same
 * semantics as oracle_assemble -- activation (assembly.hpp:227-261), fixed summation
 * (400-413), check_finite on E and g (426-438), E summed serially in (energy, active element)
 * order from 0.0 (440-448), every gradient entry accumulated in (energy, element) order from
 * 0.0 (450-462) -- without the pattern and the Hessian. Each tape is pruned to the closure of
 * its E and g outputs (SSA: dropping dead instructions changes no value). Elements are
 * evaluated in parallel into a per-element buffer; the sums run serially. Also returns E with
 * compensated (Kahan) summation over the same terms. */
static uint64_t* needed_instrs(const tape_t* t, uint32_t n_out, uint64_t* count) {
  uint8_t* need = (uint8_t*)calloc(t->n_regs + 1, 1);
  for (uint32_t k = 0; k < n_out; ++k) need[t->out[k]] = 1;
  uint64_t n = 0;
  for (uint64_t k = t->n_instrs; k-- > 0;) {
    const instr_t* i = &t->ins[k];
    if (!need[i->dst]) continue;
    ++n;
    need[i->a] = 1;
    if (i->op >= 2 && i->op <= 5) need[i->b] = 1;
    if (i->op == 12) { need[i->b] = 1; need[i->c] = 1; }
  }
  uint64_t* list = (uint64_t*)malloc(sizeof(uint64_t) * (n + 1));
  uint64_t q = 0;
  for (uint64_t k = 0; k < t->n_instrs; ++k)
    if (need[t->ins[k].dst]) list[q++] = k;
  free(need);
  *count = n;
  return list;
}

static void tape_eval_subset(const tape_t* t, const uint64_t* list, uint64_t n, const double* in, double* regs) {
  memcpy(regs, in, sizeof(double) * t->n_inputs);
  memcpy(regs + t->n_inputs, t->consts, sizeof(double) * t->n_consts);
  for (uint64_t q = 0; q < n; ++q) {
    const instr_t* i = &t->ins[list[q]];
    const double a = regs[i->a], b = regs[i->b], c = regs[i->c];
    double d;
    switch (i->op) {
      case 2: d = a + b; break;
      case 3: d = a - b; break;
      case 4: d = a * b; break;
      case 5: d = a / b; break;
      case 6: d = -a; break;
      case 7: d = powi(a, i->iarg); break;
      case 8: d = sqrt(a); break;
      case 9: d = log(a); break;
      case 10: d = sin(a); break;
      case 11: d = cos(a); break;
      default: d = a >= 0.0 ? b : c; break;
    }
    regs[i->dst] = d;
  }
}

int oracle_energy_gradient(const oracle_array* A, uint32_t na, const oracle_energy* E, uint32_t ne, int32_t threads,
                           double* energy, double* energy_kahan, double* grad, int32_t* bad_energy,
                           int64_t* bad_element) {
  layout_t L;
  make_layout(A, na, &L);
  int status = 0;
  *bad_energy = -1;
  *bad_element = -1;
  for (int64_t k = 0; k < L.n_dofs; ++k) grad[k] = 0.0;
  double Es = 0.0, Ek = 0.0, comp = 0.0;
  for (uint32_t d = 0; d < ne && status == 0; ++d) {
    const oracle_energy* e = &E[d];
    if (e->is_sum && e->n_items == 0) continue;
    tape_t t;
    if (tape_parse(e->tape, e->tape_len, &t)) { status = 6; break; }
    const uint32_t nd = e->n_dofs, S = 1 + nd;
    uint64_t nlist = 0;
    uint64_t* list = needed_instrs(&t, S, &nlist);
    uint8_t* active = (uint8_t*)malloc(e->n_elems + 1);
    memset(active, 1, e->n_elems);
    tape_t at;
    const int has_act = e->act_tape != NULL;
    if (has_act && tape_parse(e->act_tape, e->act_len, &at)) { status = 6; free(list); free(active); tape_free(&t); break; }
    double* buf = (double*)malloc(sizeof(double) * (e->n_elems * S + 1));
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
    {
      double* in = (double*)malloc(sizeof(double) * (e->n_inputs + 1));
      double* regs = (double*)malloc(sizeof(double) * (t.n_regs + (has_act ? at.n_regs : 0) + 1));
#pragma omp for schedule(static)
      for (int64_t el = 0; el < (int64_t)e->n_elems; ++el) {
        if (has_act) {
          const double v = act_value(A, e, &at, (uint64_t)el, in, regs);
          active[el] = e->act_kind == 0 ? (v >= 0.0) : (v > 0.0);
          if (!active[el]) continue;
        }
        double* dst = buf + (uint64_t)el * S;
        if (e->is_sum) {
          for (uint32_t it = 0; it < e->n_items; ++it) {
            gather(A, e, (uint64_t)el, e->sum_items + (uint64_t)it * e->sum_arity, in);
            tape_eval_subset(&t, list, nlist, in, regs);
            for (uint32_t k = 0; k < S; ++k) dst[k] = it == 0 ? regs[t.out[k]] : dst[k] + regs[t.out[k]];
          }
        } else {
          gather(A, e, (uint64_t)el, NULL, in);
          tape_eval_subset(&t, list, nlist, in, regs);
          for (uint32_t k = 0; k < S; ++k) dst[k] = regs[t.out[k]];
        }
      }
      free(in);
      free(regs);
    }
    for (uint64_t el = 0; el < e->n_elems && status == 0; ++el) {
      if (!active[el]) continue;
      const double* v = buf + el * S;
      for (uint32_t k = 0; k < S; ++k)
        if (!isfinite(v[k])) { status = 4; *bad_energy = (int32_t)d; *bad_element = (int64_t)el; break; }
      if (status) break;
      Es += v[0];
      const double y = v[0] - comp, tt = Ek + y;  /* Kahan */
      comp = (tt - Ek) - y;
      Ek = tt;
      for (uint32_t k = 0; k < nd; ++k) grad[elem_dof(A, &L, e, el, k)] += v[1 + k];
    }
    free(buf);
    free(active);
    free(list);
    if (has_act) tape_free(&at);
    tape_free(&t);
  }
  free(L.set_off);
  *energy = Es;
  *energy_kahan = Ek;
  return status;
}
