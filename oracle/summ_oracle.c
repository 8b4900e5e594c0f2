/*
 * summ_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * CPU restatement of `dartomp.interproc.summarize_all` (pkg/src/dartomp/
 * interproc.py:90-144) over the lowered call graph of
 * paper_2406_13881_b200/interproc.py: Gauss-Seidel passes over the defined
 * functions in the reference's dict order (:105), each function's `new`
 * summary rebuilt from its sources in order (:104-138) with insertion order
 * tracked like the reference's dicts, until a pass changes no set (:139-143)
 * or `max_passes` ran.  One byte per slot: bit0 R, bit1 W, bit2 HOST,
 * bit3 DEVICE.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/dfx.h"

static uint8_t force_dev(uint8_t b) { return (b & 3u) ? (uint8_t)((b & 3u) | 8u) : 0u; }

typedef struct { uint8_t *bits; int16_t *list; int32_t *len; } cg_state;

static void append(int16_t *list, int32_t *len, uint8_t *seen, int s) {
  if (!seen[s]) { seen[s] = 1; list[(*len)++] = (int16_t)s; }
}

int oracle_summaries(const dfx_cg_in *in, dfx_cg_out *out) {
  const int nf = in->n_funcs, ns = in->n_slots, P = in->n_params;
  const size_t tb = (size_t)nf * ns;
  /* S = the live `summaries` dict: entries are replaced in place as the pass
   * proceeds, so later functions see this pass's result (Gauss-Seidel) */
  cg_state S = {out->bits, out->list, out->len};
  memcpy(S.bits, in->init_bits, tb);
  memcpy(S.list, in->init_list, tb * sizeof(int16_t));
  memcpy(S.len, in->init_len, (size_t)nf * sizeof(int32_t));
  uint8_t *nb = malloc((size_t)ns), *seen = malloc((size_t)ns);
  int16_t *nl = malloc((size_t)ns * sizeof(int16_t));
  int pass = 0;
  while (pass < in->max_passes) {
    pass++;
    int changed = 0;
    for (int f = 0; f < nf; f++) {
      int32_t nlen = 0;
      memset(seen, 0, (size_t)ns);
      memcpy(nb, in->direct + (size_t)f * ns, (size_t)ns);
      for (int k = in->src_off[f]; k < in->src_off[f + 1]; k++) {
        const int32_t *r = in->src + 4 * (size_t)k;
        if ((r[0] & 0xFF) == 0) {           /* static slot list */
          for (int j = 0; j < r[2]; j++) append(nl, &nlen, seen, in->slist[r[1] + j]);
          continue;
        }
        const int dev = (r[0] >> 8) & 1, g = r[1];
        const uint8_t *gb = S.bits + (size_t)g * ns;
        const int16_t *gl = S.list + (size_t)g * ns;
        /* parameters, in the callee's param_effects order (:119-126) */
        for (int j = 0; j < S.len[g]; j++) {
          int x = gl[j];
          if (x >= P) continue;
          for (int b = r[2]; b < r[2] + r[3]; b++) {
            if (in->bind[2 * b] != x) continue;
            int s = in->bind[2 * b + 1];
            nb[s] |= dev ? force_dev(gb[x]) : gb[x];
            append(nl, &nlen, seen, s);
          }
        }
        /* globals, in the callee's global_effects order (:127-129) */
        for (int j = 0; j < S.len[g]; j++) {
          int x = gl[j];
          if (x < P) continue;
          nb[x] |= dev ? force_dev(gb[x]) : gb[x];
          append(nl, &nlen, seen, x);
        }
      }
      if (memcmp(nb, S.bits + (size_t)f * ns, (size_t)ns)) changed = 1;
      memcpy(S.bits + (size_t)f * ns, nb, (size_t)ns);
      memcpy(S.list + (size_t)f * ns, nl, (size_t)nlen * sizeof(int16_t));
      S.len[f] = nlen;
    }
    if (!changed) break;
  }
  free(nb); free(seen); free(nl);
  out->passes = pass;
  out->launches = 0;
  out->kernel_ms = 0.f;
  return 0;
}
