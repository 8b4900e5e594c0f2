/*
 * sim_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * CPU restatement of `dartomp.simulator._Simulator` (pkg/src/dartomp/
 * simulator.py:180-708) over a lowered simulation program
 * (paper_2406_13881_b200/simlower.py).  Unlike the CUDA kernel, which runs
 * each variable on its own and settles loops per variable, this restates the
 * reference's GLOBAL schedule: one environment holding every variable
 * (insertion order kept, the untaken-arm rollback deleting variables it
 * created, simulator.py:466-475), one ordered event log and stale-read log,
 * `run_loop`'s signature test over the whole environment and the round's
 * events (simulator.py:500-550: rounds until two consecutive signatures
 * match, then `_scale_tail`; 10000-round cap with its warning), and
 * `warn_once` order.  It therefore reproduces the reference's log record for
 * record, which pins the lowering to the reference (tests/test_sim.py), and
 * the per-variable totals of the CUDA kernel are checked against it.
 *
 * Event identity: op_ev[pc] names the (variable name, bytes, line) of a
 * transfer op for the log; the signature compares (direction, op_ev, count)
 * and (var, space, site, count) exactly like the reference's tuples.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/dfx.h"

#define MAX_ROUNDS 10000

typedef struct { int64_t dir, ev, count; } xev;           /* transfer event */
typedef struct { int64_t var, space, site, count; } xst;  /* stale read */

typedef struct {
  const int32_t *ops;
  const int64_t *arg;
  const int32_t *op_ev;
  int n_vars;
  /* environment */
  int64_t *ref;
  uint8_t *hv, *dv, *present;
  int32_t *order;      /* insertion order of present variables */
  int n_order;
  /* per-variable shield stacks (per-thread copies of a kernel) */
  uint8_t *shield;     /* [n_vars * 64] */
  int32_t *ssp;
  /* logs */
  xev *ev; int64_t n_ev, cap_ev;
  xst *st; int64_t n_st, cap_st;
  int32_t *warn; int n_warn; uint8_t *warned; int n_warn_ids;
  int err;
} sim;

static void touch(sim *s, int v) {
  if (!s->present[v]) {
    s->present[v] = 1;
    s->ref[v] = 0; s->hv[v] = 1; s->dv[v] = 0;
    s->order[s->n_order++] = v;
  }
}
static void warn_once(sim *s, int id) {
  if (id < 0 || id >= s->n_warn_ids) { s->err = 1; return; }
  if (!s->warned[id]) { s->warned[id] = 1; s->warn[s->n_warn++] = id; }
}
static void log_ev(sim *s, int64_t dir, int64_t ev, int64_t count) {
  if (s->n_ev == s->cap_ev) {
    s->cap_ev = s->cap_ev ? 2 * s->cap_ev : 1024;
    s->ev = realloc(s->ev, sizeof(xev) * s->cap_ev);
  }
  s->ev[s->n_ev++] = (xev){dir, ev, count};
}
static void log_st(sim *s, int64_t var, int64_t space, int64_t site, int64_t count) {
  if (s->n_st == s->cap_st) {
    s->cap_st = s->cap_st ? 2 * s->cap_st : 1024;
    s->st = realloc(s->st, sizeof(xst) * s->cap_st);
  }
  s->st[s->n_st++] = (xst){var, space, site, count};
}

/* one op of the straight-line kinds; returns 0 */
static void step(sim *s, int pc) {
  const int32_t *o = s->ops + 4 * (int64_t)pc;
  const int code = o[0] & 0xFF, v = o[1];
  switch (code) {
    case DFX_SIM_READ:        /* simulator.py:265-270 */
      touch(s, v);
      if (!(o[2] ? s->dv[v] : s->hv[v])) log_st(s, v, o[2], o[3], 1);
      break;
    case DFX_SIM_WRITE:       /* simulator.py:272-280 */
      touch(s, v);
      if (o[2] == 0) { s->hv[v] = 1; if (s->ref[v] > 0) s->dv[v] = 0; }
      else { s->dv[v] = 1; s->hv[v] = 0; }
      break;
    case DFX_SIM_ENTER:       /* simulator.py:232-240 */
      touch(s, v);
      if (s->ref[v] == 0) {
        if (o[2] == 0 || o[2] == 1) { log_ev(s, 0, s->op_ev[pc], 1); s->dv[v] = s->hv[v]; }
        else s->dv[v] = 0;
      }
      s->ref[v]++;
      break;
    case DFX_SIM_EXIT:        /* simulator.py:242-252 */
      touch(s, v);
      if (s->ref[v] == 0) { warn_once(s, o[3]); break; }
      s->ref[v]--;
      if (s->ref[v] == 0) {
        if (o[2] == 1 || o[2] == 2) { log_ev(s, 1, s->op_ev[pc], 1); s->hv[v] = s->dv[v]; }
        s->dv[v] = 0;
      }
      break;
    case DFX_SIM_UPDATE:      /* simulator.py:254-260 */
      touch(s, v);
      if (s->ref[v] == 0) { warn_once(s, o[3]); break; }
      if (o[2] == 0) { log_ev(s, 0, s->op_ev[pc], 1); s->dv[v] = s->hv[v]; }
      else { log_ev(s, 1, s->op_ev[pc], 1); s->hv[v] = s->dv[v]; }
      break;
    case DFX_SIM_SHIELD_SAVE:
      touch(s, v);
      if (s->ssp[v] >= 64) { s->err = 1; break; }
      s->shield[(int64_t)v * 64 + s->ssp[v]++] = (uint8_t)(s->hv[v] | (s->dv[v] << 1));
      break;
    case DFX_SIM_SHIELD_SET:
      touch(s, v);
      s->dv[v] = 1;
      break;
    case DFX_SIM_UNSHIELD: {
      touch(s, v);
      if (s->ssp[v] <= 0) { s->err = 1; break; }
      const uint8_t b = s->shield[(int64_t)v * 64 + --s->ssp[v]];
      s->hv[v] = b & 1; s->dv[v] = b >> 1;
      break;
    }
    case DFX_SIM_WARN:
      warn_once(s, o[1]);
      break;
    default:
      s->err = 1;
  }
}

static int run_range(sim *s, int lo, int hi);

/* environment snapshot: presence and (ref, hv, dv) of every variable */
typedef struct { uint8_t *pr, *hv, *dv; int64_t *ref; } snap;
static void snap_alloc(snap *x, int n) {
  x->pr = malloc(n + 1); x->hv = malloc(n + 1); x->dv = malloc(n + 1);
  x->ref = malloc(sizeof(int64_t) * (n + 1));
}
static void snap_free(snap *x) { free(x->pr); free(x->hv); free(x->dv); free(x->ref); }
static void snap_take(sim *s, snap *x) {
  memcpy(x->pr, s->present, s->n_vars); memcpy(x->hv, s->hv, s->n_vars);
  memcpy(x->dv, s->dv, s->n_vars); memcpy(x->ref, s->ref, sizeof(int64_t) * s->n_vars);
}
static int snap_eq(sim *s, const snap *x) {
  for (int v = 0; v < s->n_vars; v++) {
    if (x->pr[v] != s->present[v]) return 0;
    if (!s->present[v]) continue;
    if (x->ref[v] != s->ref[v] || x->hv[v] != s->hv[v] || x->dv[v] != s->dv[v]) return 0;
  }
  return 1;
}

/* `run_loop` (simulator.py:528-550) over the loop at pc; returns pc after it */
static int run_loop(sim *s, int pc) {
  const int32_t *o = s->ops + 4 * (int64_t)pc;
  const int extent = o[1], nvar = o[3];
  const int64_t trip = s->arg[pc];
  int vpc[64];
  if (nvar < 1 || nvar > 64) { s->err = 1; return pc + extent; }
  int q = pc + 1;
  for (int k = 0; k < nvar; k++) { vpc[k] = q; q += s->ops[4 * (int64_t)q + 1] + 1; }
  snap prev; snap_alloc(&prev, s->n_vars);
  int have_prev = 0;
  int64_t prev_e0 = 0, prev_e1 = 0, prev_s0 = 0, prev_s1 = 0;
  int64_t done = 0;
  while (done < trip) {
    const int k = done + 1 < nvar ? (int)done : nvar - 1;
    const int b = vpc[k];
    const int32_t *bo = s->ops + 4 * (int64_t)b;
    const int ret = (bo[0] & DFX_SIM_F_RET) != 0;
    const int64_t mark_e = s->n_ev, mark_s = s->n_st;
    run_range(s, b + 1, b + bo[1]);
    if (s->err) break;
    done++;
    if (done >= trip) break;
    /* signature: environment + concrete values (equal iff the steady
     * variant ran twice) + this round's events and stale reads */
    const int conc_same = done >= nvar;
    int same = have_prev && conc_same && snap_eq(s, &prev);
    if (same) {
      const int64_t ne = s->n_ev - mark_e, ns = s->n_st - mark_s;
      same = ne == prev_e1 - prev_e0 && ns == prev_s1 - prev_s0;
      for (int64_t i = 0; same && i < ne; i++) {
        const xev a = s->ev[mark_e + i], c = s->ev[prev_e0 + i];
        same = a.dir == c.dir && a.ev == c.ev && a.count == c.count;
      }
      for (int64_t i = 0; same && i < ns; i++) {
        const xst a = s->st[mark_s + i], c = s->st[prev_s0 + i];
        same = a.var == c.var && a.space == c.space && a.site == c.site && a.count == c.count;
      }
    }
    if (same || done >= MAX_ROUNDS) {      /* _scale_tail(trip - done) */
      const int64_t rem = trip - done, e1 = s->n_ev, s1 = s->n_st;
      for (int64_t i = mark_e; i < e1; i++) log_ev(s, s->ev[i].dir, s->ev[i].ev, s->ev[i].count * rem);
      for (int64_t i = mark_s; i < s1; i++)
        log_st(s, s->st[i].var, s->st[i].space, s->st[i].site, s->st[i].count * rem);
      if (!same) warn_once(s, 0);   /* warn id 0: "loop did not settle; ..." */
      break;
    }
    if (ret) break;
    snap_take(s, &prev);
    have_prev = 1;
    prev_e0 = mark_e; prev_e1 = s->n_ev; prev_s0 = mark_s; prev_s1 = s->n_st;
  }
  snap_free(&prev);
  return pc + extent;
}

/* untaken arm (simulator.py:462-477): stale reads stay, events and state roll back */
static int run_check(sim *s, int pc) {
  const int extent = s->ops[4 * (int64_t)pc + 1];
  const int n = s->n_vars;
  snap x; snap_alloc(&x, n);
  snap_take(s, &x);
  int32_t *ord = malloc(sizeof(int32_t) * (n + 1));
  memcpy(ord, s->order, sizeof(int32_t) * s->n_order);
  const int n_order = s->n_order;
  const int64_t mark_e = s->n_ev;
  run_range(s, pc + 1, pc + extent);
  s->n_ev = mark_e;
  memcpy(s->present, x.pr, n); memcpy(s->hv, x.hv, n); memcpy(s->dv, x.dv, n);
  memcpy(s->ref, x.ref, sizeof(int64_t) * n);
  memcpy(s->order, ord, sizeof(int32_t) * n_order);
  s->n_order = n_order;
  free(ord);
  snap_free(&x);
  return pc + extent + 1;
}

static int run_range(sim *s, int lo, int hi) {
  int pc = lo;
  while (pc < hi && !s->err) {
    const int code = s->ops[4 * (int64_t)pc] & 0xFF;
    if (code == DFX_SIM_END) return pc;
    if (code == DFX_SIM_LOOP) { pc = run_loop(s, pc); continue; }
    if (code == DFX_SIM_CHECK_BEGIN) { pc = run_check(s, pc); continue; }
    step(s, pc);
    pc++;
  }
  return pc;
}

/* Run one program.  Outputs (caller-sized, counts returned):
 *   ev[n_ev*3]  (direction 0 htod / 1 dtoh, op_ev, count) in log order
 *   st[n_st*4]  (var, space, site, count) in log order
 *   warn[n_warn] warn ids in first-occurrence order (id 0 is the
 *               10000-round "did not settle" warning)
 *   order[n_order] variables in environment insertion order, with
 *   ref/hv/dv per variable.
 * Returns 0, -1 on a malformed program, -3 if a capacity is too small. */
int oracle_sim_run(const int32_t *ops, const int64_t *arg64, const int32_t *op_ev, int32_t n_ops,
                   int32_t n_vars, int32_t n_warn_ids, int64_t *ev, int64_t cap_ev, int64_t *n_ev,
                   int64_t *st, int64_t cap_st, int64_t *n_st, int32_t *warn, int32_t *n_warn,
                   int32_t *order, int32_t *n_order, int64_t *ref, uint8_t *hv, uint8_t *dv) {
  sim s;
  memset(&s, 0, sizeof s);
  s.ops = ops; s.arg = arg64; s.op_ev = op_ev; s.n_vars = n_vars;
  s.ref = calloc(n_vars + 1, sizeof(int64_t));
  s.hv = calloc(n_vars + 1, 1); s.dv = calloc(n_vars + 1, 1); s.present = calloc(n_vars + 1, 1);
  s.order = calloc(n_vars + 1, sizeof(int32_t));
  s.shield = calloc((size_t)(n_vars + 1) * 64, 1);
  s.ssp = calloc(n_vars + 1, sizeof(int32_t));
  s.warn = calloc(n_warn_ids + 1, sizeof(int32_t));
  s.warned = calloc(n_warn_ids + 1, 1);
  s.n_warn_ids = n_warn_ids;
  for (int v = 0; v < n_vars; v++) s.hv[v] = 1;
  run_range(&s, 0, n_ops);
  int rc = s.err ? -1 : 0;
  *n_ev = s.n_ev; *n_st = s.n_st; *n_warn = s.n_warn; *n_order = s.n_order;
  if (!rc && (s.n_ev > cap_ev || s.n_st > cap_st)) rc = -3;
  if (!rc) {
    for (int64_t i = 0; i < s.n_ev; i++) { ev[3 * i] = s.ev[i].dir; ev[3 * i + 1] = s.ev[i].ev; ev[3 * i + 2] = s.ev[i].count; }
    for (int64_t i = 0; i < s.n_st; i++) {
      st[4 * i] = s.st[i].var; st[4 * i + 1] = s.st[i].space; st[4 * i + 2] = s.st[i].site; st[4 * i + 3] = s.st[i].count;
    }
    memcpy(warn, s.warn, sizeof(int32_t) * s.n_warn);
    memcpy(order, s.order, sizeof(int32_t) * s.n_order);
    memcpy(ref, s.ref, sizeof(int64_t) * n_vars);
    memcpy(hv, s.hv, n_vars); memcpy(dv, s.dv, n_vars);
  }
  free(s.ref); free(s.hv); free(s.dv); free(s.present); free(s.order); free(s.shield); free(s.ssp);
  free(s.warn); free(s.warned); free(s.ev); free(s.st);
  return rc;
}
