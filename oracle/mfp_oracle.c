/*
 * mfp_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker and the CPU baseline,
 * never the product).
 *
 * CPU restatement of the north-star CSR fixpoint
 * and of the configuration-C3 synthetic graph generator.
 *
 * Semantics per node n and variable v (dartomp/dataflow.py:299-378 gen/kill
 * effects, AND meet of `_State.merge_conj` dataflow.py:130-134):
 *   IN[n]  = AND_{p in preds(n)} OUT[p]   IN = (H=1, D=0) for nodes without preds
 *   host node   (HR: H:=1 via update-from; HW: H:=1, D:=0):
 *       H' = H | A            D' = D & ~B        with A = R|W, B = W
 *   kernel node (DR: D:=1 via update-to, firstprivate for eligible scalars;
 *                DW: D:=1, H:=0):
 *       H' = H & ~B           D' = D | (A & ~(F & H))   F = A & ~B & S
 *   (S = scalar-variable mask; a scalar read but not written by a kernel is
 *    captured firstprivate while the host copy is valid: dataflow.py:343-347)
 * H does not depend on D, so the H planes are solved first and D second,
 * each to its greatest fixpoint (two monotone problems).  Solver here: plain
 * Gauss-Seidel sweeps in node order until a sweep changes nothing, OpenMP
 * over variable-word columns (variables are independent).
 *
 * Kernel (b) restated in oracle_mfp_requirements below.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- C3 generator (must match csrc/gen.cu bit for bit) ------------------ */
static inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static inline uint64_t node_key(uint64_t seed, int64_t n) {
  return mix64(mix64(seed ^ 0x243F6A8885A308D3ull) + (uint64_t)n);
}
int oracle_c3_is_kernel(uint64_t seed, int64_t n) {
  return (mix64(node_key(seed, n) ^ 0x13198A2E03707344ull) % 5u) == 0u;
}
/* number of extra predecessors: Poisson(1.5) by inverse CDF on 32 bits */
static const uint64_t POIS15_CDF[11] = {
    958336740u, 2395841851u, 3473970684u, 4013035101u, 4215184257u, 4275829004u, 4290990191u, 4294239016u, 4294848171u, 4294949697u, 4294964926u};
int oracle_c3_n_extra(uint64_t seed, int64_t n) {
  if (n == 0) return 0;
  uint32_t u = (uint32_t)(mix64(node_key(seed, n) ^ 0xA4093822299F31D0ull) >> 32);
  int k = 0;
  while (k < 11 && (uint64_t)u >= POIS15_CDF[k]) k++;
  return k;
}
int64_t oracle_c3_extra_pred(uint64_t seed, int64_t n, int j, int64_t n_nodes) {
  uint64_t h = mix64(node_key(seed, n) ^ (0x082EFA98EC4E6C89ull + (uint64_t)j));
  return (int64_t)(h % (uint64_t)n_nodes);
}
/* per (node, word): access mask with P(bit)=1/32, class split R 50%,
 * W-only 31.25%, RW 18.75% */
void oracle_c3_word(uint64_t seed, int64_t n, int w, uint32_t *R, uint32_t *W) {
  uint64_t base = mix64(node_key(seed, n) + 0x452821E638D01377ull * (uint64_t)(w + 1));
  uint64_t r0 = mix64(base + 1), r1 = mix64(base + 2), r2 = mix64(base + 3),
           r3 = mix64(base + 4), r4 = mix64(base + 5);
  uint32_t acc = (uint32_t)r0 & (uint32_t)(r0 >> 32) & (uint32_t)r1 & (uint32_t)(r1 >> 32) &
                 (uint32_t)r2;
  uint32_t u1 = (uint32_t)(r2 >> 32), u2 = (uint32_t)r3, u3 = (uint32_t)(r3 >> 32),
           u4 = (uint32_t)r4;
  uint32_t ronly = acc & u1, rest = acc & ~u1;
  uint32_t wsel = u2 | (u3 & u4);
  uint32_t wonly = rest & wsel, rw = rest & ~wsel;
  *R = ronly | rw;
  *W = wonly | rw;
}
uint32_t oracle_c3_scalar_word(int w, int n_scalar) {
  int lo = w * 32;
  if (n_scalar <= lo) return 0u;
  if (n_scalar >= lo + 32) return 0xFFFFFFFFu;
  return (1u << (n_scalar - lo)) - 1u;
}

/* Build CSR (row_ptr [n+1], col [nnz]); returns nnz.  col may be NULL to count. */
int64_t oracle_c3_csr(uint64_t seed, int64_t n_nodes, int32_t *row_ptr, int32_t *col) {
  int64_t e = 0;
  for (int64_t n = 0; n < n_nodes; n++) {
    if (row_ptr) row_ptr[n] = (int32_t)e;
    if (n == 0) continue;
    if (col) col[e] = (int32_t)(n - 1);
    e++;
    int k = oracle_c3_n_extra(seed, n);
    for (int j = 0; j < k; j++) {
      if (col) col[e] = (int32_t)oracle_c3_extra_pred(seed, n, j, n_nodes);
      e++;
    }
  }
  if (row_ptr) row_ptr[n_nodes] = (int32_t)e;
  return e;
}

/* planes for the global word columns [w0, w0 + words), stored compactly as
 * [n_nodes][words] (a column block is an exact sample: variables are
 * independent) */
void oracle_c3_planes(uint64_t seed, int64_t n_nodes, int words, int w0,
                      uint8_t *kind, uint32_t *A, uint32_t *B, uint32_t *USE) {
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < n_nodes; n++) {
    if (kind) kind[n] = (uint8_t)oracle_c3_is_kernel(seed, n);
    for (int w = 0; w < words; w++) {
      uint32_t r, wr;
      oracle_c3_word(seed, n, w0 + w, &r, &wr);
      size_t i = (size_t)n * words + w;
      A[i] = r | wr;
      B[i] = wr;
      if (USE) USE[i] = r;
    }
  }
}

/* ---- solver ------------------------------------------------------------- */
typedef struct {
  int64_t n_nodes;
  int words;
  const int32_t *row_ptr, *col;
  const uint8_t *kind;
  const uint32_t *A, *B, *S; /* S: [words] scalar mask */
} csr_prob;

/* Solve all `words` columns; OUT_H/OUT_D [n*words].  Returns the max over
 * columns of sweeps (H phase + D phase, each including the final no-change
 * sweep). */
int oracle_mfp_solve(const csr_prob *p, uint32_t *OH, uint32_t *OD) {
  const int w0 = 0, w1 = p->words;
  const int64_t N = p->n_nodes;
  const int W = p->words;
  int max_sweeps = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(max : max_sweeps)
  for (int w = w0; w < w1; w++) {
    for (int64_t n = 0; n < N; n++) { OH[(size_t)n * W + w] = ~0u; OD[(size_t)n * W + w] = ~0u; }
    int sweeps = 0, changed;
    /* H phase */
    do {
      changed = 0;
      sweeps++;
      for (int64_t n = 0; n < N; n++) {
        uint32_t in = ~0u; /* entry nodes: boundary H = 1 */
        for (int32_t e = p->row_ptr[n]; e < p->row_ptr[n + 1]; e++)
          in &= OH[(size_t)p->col[e] * W + w];
        size_t i = (size_t)n * W + w;
        uint32_t out = p->kind[n] ? (in & ~p->B[i]) : (in | p->A[i]);
        if (out != OH[i]) { OH[i] = out; changed = 1; }
      }
    } while (changed);
    /* D phase */
    do {
      changed = 0;
      sweeps++;
      for (int64_t n = 0; n < N; n++) {
        uint32_t in = p->row_ptr[n] == p->row_ptr[n + 1] ? 0u : ~0u, hin = ~0u;
        for (int32_t e = p->row_ptr[n]; e < p->row_ptr[n + 1]; e++) {
          in &= OD[(size_t)p->col[e] * W + w];
          hin &= OH[(size_t)p->col[e] * W + w];
        }
        size_t i = (size_t)n * W + w;
        uint32_t out;
        if (p->kind[n]) {
          uint32_t a = p->A[i], f = a & ~p->B[i] & p->S[w];
          out = in | (a & ~(f & hin));
        } else {
          out = in & ~p->B[i];
        }
        if (out != OD[i]) { OD[i] = out; changed = 1; }
      }
    } while (changed);
    if (sweeps > max_sweeps) max_sweeps = sweeps;
  }
  return max_sweeps;
}

/* Per-node requirement masks from the fixpoint (kernel (b) restated).  The
 * meet over in-edges gives IN = AND_p OUT[p]; then, as in host_read /
 * device_read (dataflow.py:299-368):
 *   host n:   REQ = USE & ~IN_H                          (update from needed)
 *   kernel n: REQ = (USE & ~F & ~IN_D) | (F & ~IN_D & ~IN_H)   (update to)
 *             FP  =  F & ~IN_D & IN_H                     (firstprivate)
 * Entry nodes (no preds) use the boundary IN = (H=1, D=0). */
void oracle_mfp_requirements(const csr_prob *p, const uint32_t *USE,
                             const uint32_t *OH, const uint32_t *OD, uint32_t *REQ,
                             uint32_t *FP) {
  const int W = p->words;
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < p->n_nodes; n++) {
    for (int w = 0; w < W; w++) {
      size_t i = (size_t)n * W + w;
      uint32_t ih = ~0u, id = ~0u;
      if (p->row_ptr[n] == p->row_ptr[n + 1]) id = 0u;
      for (int32_t e = p->row_ptr[n]; e < p->row_ptr[n + 1]; e++) {
        size_t j = (size_t)p->col[e] * W + w;
        ih &= OH[j];
        id &= OD[j];
      }
      if (!p->kind[n]) {
        REQ[i] = USE[i] & ~ih;
        FP[i] = 0u;
      } else {
        uint32_t f = p->A[i] & ~p->B[i] & p->S[w];
        REQ[i] = (USE[i] & ~f & ~id) | (f & ~id & ~ih);
        FP[i] = f & ~id & ih;
      }
    }
  }
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
