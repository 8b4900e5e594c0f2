// replay.cu -- E1: exact schedule replay of the reference analysis on sm_100a.
//
// Semantics: dartomp/dataflow.py:194-734 (`_Analyzer`), compiled to a
// structured bytecode by paper_2406_13881_b200/lower.py.  Work decomposition:
// one warp per (function, 32-variable chunk); lane = variable.  This is exact
// because the analysis separates per variable: each lane carries
// its own validity bits and provenance for every live state slot, while the
// control state (current slot, branch/loop frames, slot reference counts,
// record flag, visit counter) is uniform across the warp and kept in shared
// memory, updated by lane 0.  Lanes diverge only inside the per-access ops
// that touch their variable.
//
// Per lane state:  H, D  bitmask over slots (uint64 registers)
//                  provenance (device_producer | last_host_write << 16) per
//                  slot in shared memory, [slot][lane] (conflict-free)
// Outputs: order-keyed events (plans, suppressions, errors) appended with one
// global atomic per event, and per-variable result bits.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../../include/dfx.h"
#include "dfx_internal.h"

namespace dfx {

// Two instantiations of the same replay.  Narrow (every C4 function, the
// corpus, all generated programs): up to 64 live state slots as 32/64-bit
// register masks, 16-bit provenance statement ids, small control stacks, 4
// warps per block.  Wide (rare: e.g. an else-if chain of 13+ branches needs
// more than 64 slots, or a function of more than 65,534 statements): 256 slots
// as a 4 x 64-bit register mask, 32-bit provenance ids, deeper stacks, 2
// warps per block (provenance is 64 KB per warp at 256 slots).  The host
// routes each function to the narrow launch when it fits, else to the wide
// one (api.cu fn_class); the semantics are the same code.
struct Narrow {
  static constexpr int kWarps = 4, kMaxSlots = 64, kMaxBr = 48, kMaxArmStk = 192, kMaxLoop = 24;
  using Prov = uint32_t;        // device_producer | last_host_write << 16
  using Ref = uint8_t;
  using Skip = uint32_t;
  static constexpr uint32_t kNone = 0xFFFFu;
  __device__ static uint32_t dp(Prov p) { return p & 0xFFFFu; }
  __device__ static uint32_t lw(Prov p) { return p >> 16; }
  __device__ static Prov pack(uint32_t d, uint32_t l) { return d | (l << 16); }
};
struct Wide {
  static constexpr int kWarps = 2, kMaxSlots = 256, kMaxBr = 256, kMaxArmStk = 1024, kMaxLoop = 64;
  using Prov = uint64_t;        // device_producer | last_host_write << 32
  using Ref = uint16_t;
  using Skip = uint64_t;
  static constexpr uint32_t kNone = 0xFFFFFFFFu;
  __device__ static uint32_t dp(Prov p) { return (uint32_t)p; }
  __device__ static uint32_t lw(Prov p) { return (uint32_t)(p >> 32); }
  __device__ static Prov pack(uint32_t d, uint32_t l) { return (uint64_t)d | ((uint64_t)l << 32); }
};

// 256-bit slot mask for the wide replay; every index is resolved with
// compile-time word selects so the mask stays in registers
struct Mask256 { uint64_t w[4]; };

struct BrFrame { int16_t saved, arm_base, narms, pad; };
struct LoopFrame { int32_t stmt, body_pc, loop_start; int16_t slot; int8_t round, may_skip, rec_saved, pad[3]; };

template <class M, class P>
struct WarpCtl {
  M live;                    // bit i: ref[i] > 0 (slot masks as wide as the lane's H/D masks)
  typename P::Ref ref[P::kMaxSlots];
  BrFrame br[P::kMaxBr];
  uint8_t armstk[P::kMaxArmStk];
  LoopFrame lp[P::kMaxLoop];
  int cur, nbr, narm, nlp, record, fault;
  int bc0, bc1;          // broadcast scratch
};

__device__ __forceinline__ int st_start(const int32_t* span, int s) { return __ldg(span + 2 * s); }
__device__ __forceinline__ int st_end(const int32_t* span, int s) { return __ldg(span + 2 * s + 1); }

// ---- slot-mask primitives (integer masks and Mask256) ----------------------
template <class M> __device__ __forceinline__ M mzero() { return (M)0; }
template <class M> __device__ __forceinline__ M mones() { return ~(M)0; }
template <> __device__ __forceinline__ Mask256 mzero<Mask256>() { return Mask256{{0, 0, 0, 0}}; }
template <> __device__ __forceinline__ Mask256 mones<Mask256>() {
  return Mask256{{~0ull, ~0ull, ~0ull, ~0ull}};
}
template <class M>
__device__ __forceinline__ int getb(M m, int s) { return (int)((m >> s) & (M)1); }
template <class M>
__device__ __forceinline__ M setb(M m, int s, int v) {   // branch-free bit assignment
  const M bit = (M)1 << s;
  return m ^ ((((M)0 - (M)v) ^ m) & bit);
}
__device__ __forceinline__ int getb(const Mask256& m, int s) {
  const int k = s >> 6;
  const uint64_t x = k == 0 ? m.w[0] : k == 1 ? m.w[1] : k == 2 ? m.w[2] : m.w[3];
  return (int)((x >> (s & 63)) & 1ull);
}
__device__ __forceinline__ Mask256 setb(Mask256 m, int s, int v) {
  const int k = s >> 6;
  const uint64_t bit = 1ull << (s & 63), fill = 0ull - (uint64_t)v;
#pragma unroll
  for (int j = 0; j < 4; j++)
    if (j == k) m.w[j] ^= (fill ^ m.w[j]) & bit;
  return m;
}
// first slot index < nslots that is clear in `live`, or -1
template <class M>
__device__ __forceinline__ int first_free(M live, int nslots) {
  constexpr int kBits = 8 * sizeof(M);
  const M avail = ~live & (nslots >= kBits ? ~(M)0 : (((M)1 << nslots) - (M)1));
  if (!avail) return -1;
  if constexpr (sizeof(M) == 4) return __ffs((int)avail) - 1;
  else return __ffsll((long long)avail) - 1;
}
__device__ __forceinline__ int first_free(const Mask256& live, int nslots) {
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const int lo = 64 * j;
    const uint64_t lim = nslots >= lo + 64 ? ~0ull : nslots > lo ? (1ull << (nslots - lo)) - 1ull : 0ull;
    const uint64_t avail = ~live.w[j] & lim;
    if (avail) return lo + __ffsll((long long)avail) - 1;
  }
  return -1;
}

// first free slot from the live mask (lane 0 only)
template <class M, class P>
__device__ __forceinline__ int alloc_slot(WarpCtl<M, P>& c, int nslots) {
  const int i = first_free(c.live, nslots);
  if (i < 0) { c.fault = 1; return 0; }
  c.ref[i] = 1;
  c.live = setb(c.live, i, 1);
  return i;
}
template <class M, class P>
__device__ __forceinline__ void ref_inc(WarpCtl<M, P>& c, int i) { c.ref[i]++; }
template <class M, class P>
__device__ __forceinline__ void ref_dec(WarpCtl<M, P>& c, int i) {
  if (--c.ref[i] == 0) c.live = setb(c.live, i, 0);
}

__device__ __forceinline__ void emit(dfx_event* ev, unsigned long long* count, int64_t cap,
                                     uint64_t key, int fn, int var, int node, int kind, int pos) {
  unsigned long long i = atomicAdd(count, 1ull);
  if ((int64_t)i < cap) {
    dfx_event e;
    e.key = key; e.fn = fn; e.var = var; e.node = node;
    e.kind = (uint8_t)kind; e.pos = (uint8_t)pos; e.pad = 0;
    ev[i] = e;
  }
}

// `_State.merge_conj` provenance rule (dataflow.py:135-142)
template <class P>
__device__ __forceinline__ uint32_t pick(const int32_t* span, uint32_t mine, uint32_t other) {
  if (other == P::kNone || other == mine) return mine;
  if (mine == P::kNone || st_end(span, other) > st_end(span, mine)) return other;
  return mine;
}

// Algorithm 1 + finalize + normalize on the static site table
// (bounds.py:134-193, dataflow.py:270-295)
__device__ __forceinline__ int hoist(const int32_t* t, int loc_lim) {
  int n = __ldg(t), acc = __ldg(t + 1);
  int k = 0;
  while (k < n && __ldg(t + 2 + 2 * k) < loc_lim) k++;
  int c = k;
  while (c < n && !(__ldg(t + 3 + 2 * c) & DFX_AC_QUAL)) c++;
  if (c == n) return acc;
  for (int j = c; j < n; j++) {
    int code = __ldg(t + 3 + 2 * j);
    if (code & DFX_AC_CLEAN) return code & (DFX_AC_NODE_MASK | DFX_AC_ERR);
  }
  return acc;
}

template <class M, class P>
struct Lane {
  M H, D;
  typename P::Skip skipH, skipD;
  int presence, to_comp, from_comp;
  int halted;
};

// One work item (function item_fn[item], 32-variable chunk item_chunk[item]).
template <class M, class P>
__device__ __forceinline__ void
replay_one(int item, WarpCtl<M, P>& c, typename P::Prov* prov, int lane, const dfx_fn_desc* __restrict__ fns, const int32_t* __restrict__ ops,
              const int32_t* __restrict__ var_flags, const int32_t* __restrict__ stmt_span,
              const int32_t* __restrict__ sites, const int32_t* __restrict__ arms,
              const int32_t* __restrict__ item_fn, const int32_t* __restrict__ item_chunk,
              int n_items, int slots_per_warp, dfx_event* __restrict__ events,
              int64_t event_cap, unsigned long long* __restrict__ event_count,
              uint8_t* __restrict__ var_out) {
  const int fi = __ldg(item_fn + item);
  const dfx_fn_desc d = fns[fi];
  const int chunk = __ldg(item_chunk + item);
  const int var = chunk * 32 + lane;
  const bool active = var < d.n_vars;
  const int myvar = active ? var : -1;
  int vflags = 0, rank = 0;
  if (active) {
    int w = __ldg(var_flags + d.var_off + var);
    vflags = w & 0xFFFF;
    rank = (int)((uint32_t)w >> 16);
  }
  const int4* fops = reinterpret_cast<const int4*>(ops) + d.op_off;
  const int32_t* span = stmt_span + 2 * (int64_t)d.stmt_off;
  const int32_t* fsites = sites + d.site_off;
  const int32_t* farms = arms + 2 * (int64_t)d.arm_off;
  const int nslots = d.n_slots < slots_per_warp ? d.n_slots : slots_per_warp;
  const int rbs = d.region_begin_start;

  if (lane == 0) {
    for (int i = 0; i < P::kMaxSlots; i++) c.ref[i] = 0;
    c.live = mzero<M>();
    c.nbr = c.narm = c.nlp = 0;
    c.record = 1;
    c.fault = 0;
    c.cur = alloc_slot(c, nslots);
  }
  for (int s = 0; s < slots_per_warp; s++) prov[s * 32 + lane] = P::pack(P::kNone, P::kNone);
  __syncwarp();

  using Skip = typename P::Skip;
  Lane<M, P> L;
  L.H = mones<M>(); L.D = mzero<M>();
  L.skipH = L.skipD = 0u;
  L.presence = L.to_comp = L.from_comp = 0;
  L.halted = !active;
  int cur = c.cur;
  __syncwarp();         // as after every read of the warp's shared control block
  int record = 1;
  // visit counter (`_Analyzer` op order, the event key) of the op at pc is
  // sbase + pc + 1: it advances with pc, and sbase absorbs the jumps (loop
  // rounds, skipped regions), so the op loop does no 64-bit counting
  uint64_t sbase = 0;
  int pc = 0;
  auto key_now = [&]() { return (sbase + (uint64_t)pc + 1u) << 24; };

  // plan-log window bookkeeping for the zero-trip skip merge (dataflow.py:573-589)
  auto log_plan = [&](int kind, int pos, int node) {
    for (int l = 0; l < c.nlp; l++) {
      const LoopFrame& f = c.lp[l];
      if (f.round != 1) continue;
      int pre = (pos == DFX_POS_BEFORE && st_start(span, node) <= f.loop_start) ||
                (pos == DFX_POS_AFTER && st_end(span, node) <= f.loop_start);
      if (!pre) continue;
      if (kind == DFX_EV_UPDATE_FROM) L.skipH |= (Skip)1 << l; else L.skipD |= (Skip)1 << l;
    }
  };
  auto copy_slot = [&](int dst, int src) {
    L.H = setb(L.H, dst, getb(L.H, src));
    L.D = setb(L.D, dst, getb(L.D, src));
    prov[dst * 32 + lane] = prov[src * 32 + lane];
  };
  auto merge_conj = [&](int a, int b) {
    L.H = setb(L.H, a, getb(L.H, a) & getb(L.H, b));
    L.D = setb(L.D, a, getb(L.D, a) & getb(L.D, b));
    const typename P::Prov pa = prov[a * 32 + lane], pb = prov[b * 32 + lane];
    if (pa != pb) {   // equal provenance (the common case) merges to itself
      const uint32_t dp = pick<P>(span, P::dp(pa), P::dp(pb));
      const uint32_t lw = pick<P>(span, P::lw(pa), P::lw(pb));
      prov[a * 32 + lane] = P::pack(dp, lw);
    }
  };

  // op window: lane i holds op (wbase + i); an op is fetched by shuffles
  // instead of a dependent global load per op
  // `rel` marks the window's ops this warp must execute: an access op on a
  // variable outside this warp's 32-variable chunk only advances the visit
  // counter, so runs of them are skipped in one step (uniform across the warp)
  int wbase = -64;
  int4 wop = make_int4(0, 0, 0, 0);
  unsigned rel = 0u;
  for (;;) {
    if ((unsigned)(pc - wbase) >= 32u) {
      wbase = pc;
      bool r = true;
      if (wbase + lane < d.n_ops) {
        wop = __ldg(fops + wbase + lane);
        r = !((unsigned)((wop.x & 0xFF) - DFX_OP_HR) <= (unsigned)(DFX_OP_DW - DFX_OP_HR) &&
              (wop.y >> 5) != chunk);
      }
      rel = __ballot_sync(0xFFFFFFFFu, r);
    }
    const unsigned m = rel & (0xFFFFFFFFu << (pc - wbase));
    if (!m) {                       // the rest of the window is foreign accesses
      pc = wbase + 32;
      continue;
    }
    const int src = __ffs(m) - 1;
    pc = wbase + src;
    const int4 op = make_int4(__shfl_sync(0xFFFFFFFFu, wop.x, src), __shfl_sync(0xFFFFFFFFu, wop.y, src),
                              __shfl_sync(0xFFFFFFFFu, wop.z, src), __shfl_sync(0xFFFFFFFFu, wop.w, src));
    const int code = op.x & 0xFF, fl = op.x;
    switch (code) {
      case DFX_OP_END:
        goto replay_done;
      case DFX_OP_HR: {   // host_read, dataflow.py:299-324
        if (op.y != myvar || L.halted || getb(L.H, cur)) break;
        if (vflags & DFX_V_ALLOW_STALE) {
          if (record) emit(events, event_count, event_cap, key_now(), fi, var, op.z, DFX_EV_SUPPRESS, 0);
          L.H = setb(L.H, cur, 1); break;
        }
        if (fl & DFX_F_AFTER_REGION) {
          L.presence = 1; L.from_comp = 1; L.H = setb(L.H, cur, 1); break;
        }
        uint32_t dp = P::dp(prov[cur * 32 + lane]);
        int lim = dp == P::kNone ? 0 : st_end(span, dp);
        int pos, node;
        if (fl & DFX_F_OVR) { pos = DFX_POS_BODY_END; node = op.w; }
        else {
          int a = hoist(fsites + op.w, lim);
          if (a & DFX_AC_ERR) {
            emit(events, event_count, event_cap, key_now(), fi, var, a & DFX_AC_NODE_MASK, DFX_EV_ERR_BRACES_LOOP, 0);
            L.halted = 1; break;
          }
          pos = DFX_POS_BEFORE; node = a;
        }
        log_plan(DFX_EV_UPDATE_FROM, pos, node);
        if (record) emit(events, event_count, event_cap, key_now(), fi, var, node, DFX_EV_UPDATE_FROM, pos);
        L.H = setb(L.H, cur, 1);
        break;
      }
      case DFX_OP_HW: {   // host_write, dataflow.py:326-330
        if (op.y != myvar || L.halted) break;
        L.H = setb(L.H, cur, 1); L.D = setb(L.D, cur, 0);
        prov[cur * 32 + lane] = P::pack(P::dp(prov[cur * 32 + lane]), (uint32_t)op.z);
        break;
      }
      case DFX_OP_DR: {   // device_read, dataflow.py:332-368
        if (op.y != myvar || L.halted || getb(L.D, cur)) break;
        if (vflags & DFX_V_ALLOW_STALE) {
          if (record) emit(events, event_count, event_cap, key_now(), fi, var, op.z, DFX_EV_SUPPRESS, 0);
          L.D = setb(L.D, cur, 1); break;
        }
        if ((fl & DFX_F_FP) && getb(L.H, cur)) {
          if (record) emit(events, event_count, event_cap, key_now(), fi, var, op.z, DFX_EV_FIRSTPRIVATE, DFX_POS_KERNEL);
          break;
        }
        L.presence = 1;
        if (record && (vflags & DFX_V_DECL_LATE)) {
          emit(events, event_count, event_cap, key_now(), fi, var, op.z, DFX_EV_ERR_DECL, 0);
          L.halted = 1; break;
        }
        uint32_t lw = P::lw(prov[cur * 32 + lane]);
        bool in_region = lw != P::kNone && rbs >= 0 && st_start(span, lw) >= rbs;
        if (!in_region) { L.to_comp = 1; L.D = setb(L.D, cur, 1); break; }
        int lim = st_end(span, lw);
        int pos, node;
        if (fl & DFX_F_OVR) { pos = DFX_POS_BODY_END; node = op.w; }
        else {
          int a = hoist(fsites + op.w, lim);
          if (a & DFX_AC_ERR) {
            emit(events, event_count, event_cap, key_now(), fi, var, a & DFX_AC_NODE_MASK, DFX_EV_ERR_BRACES_LOOP, 0);
            L.halted = 1; break;
          }
          pos = DFX_POS_BEFORE; node = a;
        }
        log_plan(DFX_EV_UPDATE_TO, pos, node);
        if (record) emit(events, event_count, event_cap, key_now(), fi, var, node, DFX_EV_UPDATE_TO, pos);
        L.D = setb(L.D, cur, 1);
        break;
      }
      case DFX_OP_DW: {   // device_write, dataflow.py:370-378
        if (op.y != myvar || L.halted) break;
        L.presence = 1;
        if (record && (vflags & DFX_V_DECL_LATE)) {
          emit(events, event_count, event_cap, key_now(), fi, var, op.z, DFX_EV_ERR_DECL, 0);
          L.halted = 1; break;
        }
        L.D = setb(L.D, cur, 1); L.H = setb(L.H, cur, 0);
        prov[cur * 32 + lane] = P::pack((uint32_t)op.z, P::lw(prov[cur * 32 + lane]));
        break;
      }
      case DFX_OP_BR_BEGIN: {  // saved = self.state
        if (!(((uint32_t)op.z >> (chunk & 31)) & 1u)) goto skip_region;
        if (lane == 0) {
          if (c.nbr >= P::kMaxBr) c.fault = 1;
          else {
            BrFrame& b = c.br[c.nbr++];
            b.saved = (int16_t)cur; ref_inc(c, cur);
            b.arm_base = (int16_t)c.narm; b.narms = 0;
          }
        }
        __syncwarp();
        if (c.fault) goto fault;
        break;
      }
      case DFX_OP_ARM_FORK:      // state = saved.copy()  (F_CAPTURE: the arm is this slot)
      case DFX_OP_ARM_PASSIVE: { // arms += [(saved.copy(), None)]
        if (lane == 0) {
          BrFrame& b = c.br[c.nbr - 1];
          int s = alloc_slot(c, nslots);
          if (c.narm >= P::kMaxArmStk) c.fault = 1;
          c.bc0 = s; c.bc1 = b.saved;
          const bool room = c.narm < P::kMaxArmStk;
          if (code == DFX_OP_ARM_FORK) {
            ref_dec(c, cur); c.cur = s;
            if ((fl & DFX_F_CAPTURE) && room) { c.armstk[c.narm++] = (uint8_t)s; ref_inc(c, s); b.narms++; }
          } else if (room) {
            c.armstk[c.narm++] = (uint8_t)s; b.narms++;
          }
        }
        __syncwarp();
        int s = c.bc0, saved = c.bc1;
        copy_slot(s, saved);
        cur = c.cur;
        __syncwarp();
        if (c.fault) goto fault;
        break;
      }
      case DFX_OP_ARM_CLOSE: {   // switch arm = current slot
        if (lane == 0) {
          BrFrame& b = c.br[c.nbr - 1];
          if (c.narm >= P::kMaxArmStk) c.fault = 1;
          else { c.armstk[c.narm++] = (uint8_t)cur; ref_inc(c, cur); b.narms++; }
        }
        __syncwarp();
        if (c.fault) goto fault;
        break;
      }
      case DFX_OP_BR_END: {      // _merge_arms, dataflow.py:525-564
        const BrFrame b = c.br[c.nbr - 1];
        const uint8_t* arm = c.armstk + b.arm_base;
        const int n = b.narms;
        if (!L.halted) {
          int dev_newer = 0, host_newer = 0;
          for (int i = 0; i < n; i++) {
            int s = arm[i];
            int h = getb(L.H, s), dd = getb(L.D, s);
            dev_newer |= dd & !h;
            host_newer |= h & !dd;
          }
          if (dev_newer && host_newer) {
            for (int i = 0; i < n; i++) {
              int s = arm[i];
              if (!(getb(L.D, s) && !getb(L.H, s))) continue;
              uint64_t k2 = key_now() | ((uint64_t)rank << 8) | (uint64_t)i;
              int kind = __ldg(farms + 2 * (op.y + i)), node = __ldg(farms + 2 * (op.y + i) + 1);
              if (kind == DFX_ARM_ERR_ARM || kind == DFX_ARM_ERR_LOOP) {
                emit(events, event_count, event_cap, k2, fi, var, node,
                     kind == DFX_ARM_ERR_ARM ? DFX_EV_ERR_BRACES_ARM : DFX_EV_ERR_BRACES_LOOP, 0);
                L.halted = 1; break;
              }
              int pos = kind == DFX_ARM_BEFORE ? DFX_POS_BEFORE : DFX_POS_AFTER;
              log_plan(DFX_EV_UPDATE_FROM, pos, node);
              if (record) emit(events, event_count, event_cap, k2, fi, var, node, DFX_EV_UPDATE_FROM, pos);
              L.H = setb(L.H, s, 1);
            }
          }
        }
        for (int i = 1; i < n; i++) merge_conj(arm[0], arm[i]);
        __syncwarp();
        if (lane == 0) {
          // arm 0 becomes cur: its arm-stack reference turns into the cur
          // reference (net zero), the old cur's and the other arms' drop
          const int m = arm[0];
          ref_dec(c, cur); c.cur = m;
          for (int i = 1; i < n; i++) ref_dec(c, arm[i]);
          ref_dec(c, b.saved);
          c.narm = b.arm_base;
          c.nbr--;
        }
        __syncwarp();
        cur = c.cur;
        __syncwarp();   // every lane has read c.cur before lane 0 writes it again (racecheck)
        break;
      }
      case DFX_OP_LOOP_BEGIN: {  // _loop_rounds: entry = state.copy(); dry round
        if (!(((uint32_t)op.z >> (chunk & 31)) & 1u)) goto skip_region;
        // Dry round in closed form.  When the loop (body, condition, increment)
        // writes none of this warp's variables, their ops in it are reads, and
        // reads (and the reconciles they cause) only raise H/D bits and never
        // touch provenance: the dry round's exit state is >= its entry state,
        // so the weakened state merge_conj(entry, exit) (dataflow.py:572-574)
        // IS the entry state, and the planning round replays the dry round
        // from the same state with record on -- every dry-round side effect
        // (presence, to_comp, from_comp, the plan log an enclosing loop's skip
        // merge reads) recurs there, and a dry round records no events.  The
        // dry round is then jumped: the visit counter advances by its dynamic
        // length.  Exact under two conditions: no anchor of the function can
        // raise a braces error (DFX_FN_NO_ERR_SITES, from the lowering: no
        // error event of a skipped round is lost), and the loop does not hold
        // a branch while its entry slot is captured by an enclosing if-arm
        // (D4: that arm freezes at the dry round's first branch and is read
        // after the loop).  Region table: end.z = written-chunk mask.
        bool jump = false;
        uint32_t ew = 0u;
        if ((d.flags & DFX_FN_NO_ERR_SITES) && op.z != -1) {
          const int2 e2 = __ldg(reinterpret_cast<const int2*>(&fops[pc + op.w].z));
          ew = (uint32_t)e2.y;
          jump = !(((uint32_t)e2.x >> (chunk & 31)) & 1u) && !((ew >> 31) && c.ref[cur] >= 2);
        }
        if (lane == 0) {
          if (c.nlp >= P::kMaxLoop) c.fault = 1;
          else {
            LoopFrame& f = c.lp[c.nlp++];
            f.stmt = op.y; f.loop_start = st_start(span, op.y);
            f.may_skip = (fl & DFX_F_MAY_SKIP) != 0;
            f.body_pc = pc + 1; f.round = 0; f.rec_saved = (int8_t)record;
            f.slot = (int16_t)alloc_slot(c, nslots);
            c.bc0 = f.slot;
          }
        }
        __syncwarp();
        if (c.fault) goto fault;
        copy_slot(c.bc0, cur);
        record = 0;
        __syncwarp();
        if (jump) {   // to the LOOP_END of the dry round: one round = (dyn - 3) / 2 visits
          sbase += (uint64_t)(((ew & 0x7FFFFFFFu) - 3u) >> 1) + 1u - (uint64_t)op.w;
          pc += op.w;
          continue;
        }
        break;
      }
      case DFX_OP_LOOP_END: {
        const int lvl = c.nlp - 1;
        LoopFrame& f = c.lp[lvl];
        if (f.round == 0) {      // merge entry, weaken, planning round
          merge_conj(cur, f.slot);
          __syncwarp();
          if (lane == 0) {
            ref_dec(c, f.slot);
            f.slot = (int16_t)alloc_slot(c, nslots);
            f.round = 1;
          }
          __syncwarp();
          copy_slot(f.slot, cur);
          record = f.rec_saved;
          L.skipH &= ~((Skip)1 << lvl); L.skipD &= ~((Skip)1 << lvl);
          __syncwarp();
          if (c.fault) goto fault;
          sbase += (uint64_t)(pc + 1 - f.body_pc);   // the planning round
          pc = f.body_pc;
          continue;
        }
        if (f.may_skip) {        // zero-trip skip merge (dataflow.py:575-590)
          int w = f.slot;
          if (L.skipH & ((Skip)1 << lvl)) L.H = setb(L.H, w, 1);
          if (L.skipD & ((Skip)1 << lvl)) L.D = setb(L.D, w, 1);
          merge_conj(cur, w);
        }
        L.skipH &= ~((Skip)1 << lvl); L.skipD &= ~((Skip)1 << lvl);
        __syncwarp();
        if (lane == 0) { ref_dec(c, f.slot); c.nlp--; }
        __syncwarp();
        break;
      }
      case DFX_OP_ERR: {
        if (op.y == 1 && __ldg(item_chunk + item) == 0 && lane == 0)
          emit(events, event_count, event_cap, key_now(), fi, -1, op.z, DFX_EV_ERR_DATAMAP, 0);
        goto halt_all;
      }
      default:
        goto fault;
    }
    pc++;   // (control ops that can fault check c.fault in their case)
    continue;
  skip_region:
    // no access of this warp's variables (and no static error) anywhere in the
    // region: every arm / round leaves the state as it found it, so the region
    // only advances the visit counter, by its dynamic op count (region_kernel).
    // A region holding a branch still ends in a fresh slot (`_merge_arms`
    // returns a new state object): an enclosing arm captured by F_CAPTURE
    // keeps the old slot and must stay frozen at this point (D4)
    {
      const uint32_t ew = (uint32_t)__ldg(&fops[pc + op.w].w);
      sbase += (uint64_t)(ew & 0x7FFFFFFFu) - (uint64_t)(op.w + 1);
      pc += op.w + 1;
      if (!(ew >> 31)) continue;
    }
    {
      if (lane == 0) {
        const int s = alloc_slot(c, nslots);
        c.bc0 = s;
        ref_dec(c, cur);
        c.cur = s;
      }
      __syncwarp();
      copy_slot(c.bc0, cur);
      cur = c.cur;
      __syncwarp();
      if (c.fault) goto fault;
    }
  }
replay_done:
  if (active) {
    uint8_t o = 0;
    if (L.presence) o |= DFX_OUT_PRESENCE;
    if (L.to_comp) o |= DFX_OUT_TO;
    if (L.from_comp) o |= DFX_OUT_FROM;
    if (getb(L.H, cur)) o |= DFX_OUT_H;
    if (getb(L.D, cur)) o |= DFX_OUT_D;
    var_out[d.var_off + var] = L.halted ? 0 : o;
  }
  return;
fault:
  if (lane == 0)
    emit(events, event_count, event_cap, key_now(), fi, 0, 0, DFX_EV_ERR_ENGINE, 0);
halt_all:
  if (active) var_out[d.var_off + var] = 0;
}

// Range gating of the host-buffer pipeline (dfx_replay_batch): the programs
// arrive in K function ranges; range k's items wait until ready[k] is set
// (after its H2D and its region table), write their events into range k's
// region, and the last item of range k publishes the range's event count in
// mapped host memory, so its events go home while the launch runs on.

// Bounded wait (lane 0) for *p != 0; false after ~20 s (a range whose inputs
// never arrive must not hang the device)
__device__ __noinline__ bool wait_set(const volatile int* p, unsigned long long limit_ns) {
  if (*p) return true;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned ns = 64;
  while (!*p) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > limit_ns) return false;
    __nanosleep(ns);
    if (ns < 4096) ns <<= 1;
  }
  return true;
}

// Persistent: each warp takes work items from `next` (one atomic per item)
// until none are left, so no warp idles on the rest of its block and the
// long items (first in the order) never wait for a block slot.
template <class M, class P, bool GATED>
__global__ void __launch_bounds__(P::kWarps * 32, 8)
replay_kernel(const dfx_fn_desc* __restrict__ fns, const int32_t* __restrict__ ops,
              const int32_t* __restrict__ var_flags, const int32_t* __restrict__ stmt_span,
              const int32_t* __restrict__ sites, const int32_t* __restrict__ arms,
              const int32_t* __restrict__ item_fn, const int32_t* __restrict__ item_chunk,
              int n_items, int slots_per_warp, dfx_event* __restrict__ events,
              int64_t event_cap, unsigned long long* __restrict__ event_count,
              uint8_t* __restrict__ var_out, unsigned* __restrict__ next, GateDev gate) {
  __shared__ WarpCtl<M, P> ctl_all[P::kWarps];
  extern __shared__ __align__(16) unsigned char prov_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpCtl<M, P>& c = ctl_all[warp];
  typename P::Prov* prov = reinterpret_cast<typename P::Prov*>(prov_raw) + warp * slots_per_warp * 32;
  for (;;) {
    int item = 0;
    if (lane == 0) item = (int)atomicAdd(next, 1u);
    item = __shfl_sync(0xFFFFFFFFu, item, 0);
    if (item >= n_items) return;
    if constexpr (GATED) {
      const int f = __ldg(item_fn + item);
      int k = 0, hi = gate.K - 1;   // the range holding f: fn_cut[k] <= f < fn_cut[k+1]
      while (k < hi) {
        const int mid = (k + hi + 1) >> 1;
        if (f >= __ldg(gate.fn_cut + mid)) k = mid; else hi = mid - 1;
      }
      int ok = 1;
      if (lane == 0) {
        ok = wait_set(gate.ready + k, gate.timeout_ns);
        if (!ok) atomicExch(gate.timed_out, 1u);
      }
      if (!__shfl_sync(0xFFFFFFFFu, ok, 0)) return;
      replay_one<M, P>(item, c, prov, lane, fns, ops, var_flags, stmt_span, sites, arms, item_fn,
                    item_chunk, n_items, slots_per_warp, events + __ldg(gate.ev_off + k),
                    __ldg(gate.ev_cap + k), event_count + k, var_out);
      __threadfence();
      __syncwarp();
      if (lane == 0 &&
          atomicAdd(gate.items_done + k, 1u) + 1u == __ldg(gate.range_items + k)) {
        const unsigned long long cnt = atomicAdd(event_count + k, 0ull);
        __threadfence_system();
        *reinterpret_cast<volatile unsigned long long*>(gate.host_done + k) = cnt + 1ull;
      }
    } else {
      replay_one<M, P>(item, c, prov, lane, fns, ops, var_flags, stmt_span, sites, arms, item_fn,
                    item_chunk, n_items, slots_per_warp, events, event_cap, event_count, var_out);
      __syncwarp();
    }
  }
}

// Region table, one warp per function (runs before the replay of the same
// function range, on the same stream).  For every BR_BEGIN / LOOP_BEGIN it
// writes into the device copy of the program
//   begin.z = chunk mask: bit (v >> 5) & 31 for every variable v accessed
//             anywhere inside the region; all ones if the region holds a
//             static error op, nests deeper than the frame stack, or its
//             dynamic length does not fit 31 bits (never skipped)
//   begin.w = end pc - begin pc
//   end.z   = (LOOP_END) written-chunk mask: bit (v >> 5) & 31 for every
//             variable v with a HW/DW op inside the loop (the dry-round jump)
//   end.w   = dynamic op count of one visit of the region, begin and end
//             included: branch 2 + content, loop 3 + 2 x content (the dry
//             round and the planning round, `_loop_rounds`, dataflow.py:566-590)
//             | 1 << 31 if the region holds a branch (the current slot changes
//             identity across it)
// Idempotent; fields the replay reads from these ops are untouched.
constexpr int kRegionStack = Narrow::kMaxBr + Narrow::kMaxLoop;
constexpr int kRegionWarps = 8;

// One warp per function, 32 ops per step: a step without region ops (most
// of them) folds its accesses into the open region with two warp OR
// reductions and a population count; the region ops of a step are taken in
// order, the accesses between them folded segment by segment.  The walk's
// state is uniform across the warp (every lane computes the same values);
// the stack of enclosing regions lives in shared memory, written by lane 0.
// (A thread-per-function walk sat on the critical path of the pipelined
// host-buffer call: ranges opened ~50 ms after their programs had landed.)
__global__ void __launch_bounds__(kRegionWarps * 32)
region_kernel(const dfx_fn_desc* __restrict__ fns, int4* __restrict__ ops, int fn_lo, int fn_hi) {
  struct Frame { int64_t dyn; int pc; uint32_t mask, wmask; int br; };
  __shared__ Frame stk_all[kRegionWarps][kRegionStack + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f = fn_lo + blockIdx.x * kRegionWarps + warp;
  if (f >= fn_hi) return;
  Frame* stk = stk_all[warp];
  const dfx_fn_desc d = fns[f];
  int4* o = ops + d.op_off;
  int cpc = -1;          // begin pc of the open region (-1: the function body)
  uint32_t cmask = 0u, cwmask = 0u;
  int64_t cdyn = 0;
  int cbr = 0;
  int sp = 0, deep = 0;  // sp: enclosing regions stacked; deep: beyond the stack (never skipped)
  for (int base = 0; base < d.n_ops; base += 32) {
    const int pc = base + lane;
    const int2 op = pc < d.n_ops ? __ldcg(reinterpret_cast<const int2*>(o + pc))
                                 : make_int2(DFX_OP_END, 0);
    const int code = op.x & 0xFF;
    const bool acc = code >= DFX_OP_HR && code <= DFX_OP_DW;
    const bool wr = code == DFX_OP_HW || code == DFX_OP_DW;
    const bool ctl = code == DFX_OP_END || code == DFX_OP_BR_BEGIN || code == DFX_OP_LOOP_BEGIN ||
                     code == DFX_OP_BR_END || code == DFX_OP_LOOP_END;
    const uint32_t bit = acc ? 1u << ((op.y >> 5) & 31) : 0u;
    unsigned ctlm = __ballot_sync(0xFFFFFFFFu, ctl);
    int s = 0;             // first lane of the current segment
    bool done = false;
    for (;;) {
      // fold the segment [s, next region op) into the open region: accesses
      // set chunk bits, an ERR op marks it never skipped, every op counts 1
      const unsigned lo = s >= 32 ? 0u : 0xFFFFFFFFu << s;
      const unsigned hi = ctlm ? (1u << (__ffs(ctlm) - 1)) - 1u : 0xFFFFFFFFu;
      const unsigned seg = lo & hi;
      const bool in = (seg >> lane) & 1u;
      cmask |= __reduce_or_sync(0xFFFFFFFFu, in ? bit : 0u);
      cwmask |= __reduce_or_sync(0xFFFFFFFFu, in && wr ? bit : 0u);
      if (__any_sync(0xFFFFFFFFu, in && code == DFX_OP_ERR)) cmask = ~0u;
      cdyn += __popc(seg);
      if (!ctlm) break;
      const int j = __ffs(ctlm) - 1;
      ctlm &= ctlm - 1;
      s = j + 1;
      const int cj = __shfl_sync(0xFFFFFFFFu, code, j);
      const int pcj = base + j;
      if (cj == DFX_OP_END) { done = true; break; }
      if (cj == DFX_OP_BR_BEGIN || cj == DFX_OP_LOOP_BEGIN) {
        if (lane == 0) o[pcj].z = -1;          // until its end is seen
        if (deep || sp == kRegionStack) { deep++; cmask = ~0u; continue; }
        if (lane == 0) stk[sp] = Frame{cdyn, cpc, cmask, cwmask, cbr};
        sp++;
        cpc = pcj; cmask = 0u; cwmask = 0u; cdyn = 0; cbr = cj == DFX_OP_BR_BEGIN;
      } else {                                   // BR_END / LOOP_END
        if (deep) { deep--; continue; }
        if (sp == 0) continue;                   // unbalanced
        const int b = cpc;
        const bool loop = cj == DFX_OP_LOOP_END;
        const int64_t dyn = loop ? 3 + 2 * cdyn : 2 + cdyn;
        uint32_t mask = cmask;
        if (dyn > 0x7FFFFFFF || (int)loop == cbr) mask = ~0u;   // too long, or mismatched
        if (lane == 0) {
          o[b].z = (int)mask;
          o[b].w = pcj - b;
          o[pcj].w = (int)((uint32_t)(dyn > 0x7FFFFFFF ? 0x7FFFFFFF : dyn) | (cbr ? 0x80000000u : 0u));
          if (loop) o[pcj].z = (int)cwmask;
        }
        const int br = cbr;
        sp--;
        __syncwarp();
        const Frame fr = stk[sp];
        cpc = fr.pc; cmask = fr.mask | mask; cwmask = fr.wmask | cwmask;
        cdyn = fr.dyn + dyn; cbr = fr.br | br;
      }
    }
    if (done) break;
  }
}

int region_launch(const ReplayDev& r, int fn_lo, int fn_hi, cudaStream_t stream) {
  if (fn_hi > fn_lo)
    region_kernel<<<(fn_hi - fn_lo + kRegionWarps - 1) / kRegionWarps, kRegionWarps * 32, 0, stream>>>(
        r.fns, reinterpret_cast<int4*>(const_cast<int32_t*>(r.ops)), fn_lo, fn_hi);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

// Packed ops (dfx_replay_batch_packed, include/dfx.h) -> the 16-byte form, for
// the op range [lo, hi); region-table words are left 0 for region_kernel.
__host__ __device__ __forceinline__ int4 unpack_op(uint2 p) {
  const int code = (int)(p.x & 15u), fl = (int)((p.x >> 4) & 31u), c = (int)(p.x >> 9);
  const int a = (int)(p.y & 0xFFFFu), b = (int)(p.y >> 16);
  int4 o = make_int4(code | fl << 8, 0, 0, 0);
  switch (code) {
    case DFX_OP_HR: case DFX_OP_DR: o.y = a; o.z = b; o.w = c; break;
    case DFX_OP_HW: case DFX_OP_DW: case DFX_OP_ERR: o.y = a; o.z = b; break;
    case DFX_OP_BR_END: o.y = c; o.z = b; break;
    case DFX_OP_LOOP_BEGIN: o.y = a; break;
    case DFX_OP_LOOP_END: o.y = c; break;
    default: break;
  }
  return o;
}

__global__ void unpack_ops_kernel(const uint2* __restrict__ pk, int4* __restrict__ ops, int64_t lo,
                                  int64_t hi) {
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi;
       i += (int64_t)gridDim.x * blockDim.x)
    ops[i] = unpack_op(__ldg(pk + i));
}

int unpack_ops_launch(const uint32_t* packed, int32_t* ops, int64_t lo, int64_t hi, cudaStream_t st) {
  if (hi <= lo) return DFX_OK;
  int64_t g = (hi - lo + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  unpack_ops_kernel<<<(int)g, 256, 0, st>>>(reinterpret_cast<const uint2*>(packed),
                                            reinterpret_cast<int4*>(ops), lo, hi);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

void unpack_ops_host(const uint32_t* packed, int32_t* ops, int64_t n) {
  for (int64_t i = 0; i < n; i++) {
    const int4 o = unpack_op(make_uint2(packed[2 * i], packed[2 * i + 1]));
    ops[4 * i] = o.x; ops[4 * i + 1] = o.y; ops[4 * i + 2] = o.z; ops[4 * i + 3] = o.w;
  }
}


namespace {
// one persistent launch over an item list: narrow (slot bitmasks in 32-bit
// registers when every function of the list needs at most 32 live state
// slots -- all of C4 -- else 64-bit) or wide (Mask256, Wide traits)
int launch_items(const ReplayDev& r, const int32_t* item_fn, const int32_t* item_chunk,
                 int n_items, int slots, unsigned* next, bool wide, cudaStream_t stream,
                 const GateDev* gate, bool backfill = false) {
  if (slots < 2) slots = 2;
  if (slots > (wide ? Wide::kMaxSlots : Narrow::kMaxSlots)) return DFX_E_LIMIT;
  const int wpb = wide ? Wide::kWarps : Narrow::kWarps;
  const size_t smem = (size_t)wpb * slots * 32 * (wide ? sizeof(Wide::Prov) : sizeof(Narrow::Prov));
  const int need = (n_items + wpb - 1) / wpb;
  if (need == 0) return DFX_OK;
  // a gated launch's counter is zeroed with the gate block the caller uploads
  // before any range opens, so a backfill launch on another stream can never
  // see it reset
  if (!gate && cudaMemsetAsync(next, 0, sizeof(unsigned), stream) != cudaSuccess) return DFX_E_CUDA;
  // a persistent grid (resident blocks x SMs) over the item queue
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, wpb * 32, smem);
    int blocks = sms * (per_sm > 0 ? per_sm : 1);
    // gated: leave room for the region kernels that open the ranges
    if (gate) {
      // block slots left to the region kernels that open the ranges (they
      // run beside this launch); C4 sweep with 32 ranges, free 32 / 64 / 98 /
      // 148: 187.5 / 187.5 / 188.4 / 191.8 ms per host call (with 16 larger
      // ranges, 16 free slots starved the region kernels: 328 ms)
      int free_blocks = sms / 2;
      if (const char* e = getenv("DFX_GATE_FREE")) free_blocks = atoi(e);
      // the backfill launch takes exactly those slots once every range is
      // open, pulling from the same item queue
      blocks = backfill ? free_blocks : blocks - free_blocks;
    }
    if (blocks > need) blocks = need;
    if (blocks < 1) blocks = 1;
    kern<<<blocks, wpb * 32, smem, stream>>>(
        r.fns, r.ops, r.var_flags, r.stmt_span, r.sites, r.arms, item_fn, item_chunk,
        n_items, slots, r.events, r.event_cap, r.event_count, r.var_out, next,
        gate ? *gate : GateDev{});
  };
  if (wide) {
    if (gate) return DFX_E_ARG;             // the wide list runs after the gated launch
    launch(replay_kernel<Mask256, Wide, false>);
  } else if (slots <= 32) {
    if (gate) launch(replay_kernel<uint32_t, Narrow, true>);
    else launch(replay_kernel<uint32_t, Narrow, false>);
  } else {
    if (gate) launch(replay_kernel<uint64_t, Narrow, true>);
    else launch(replay_kernel<uint64_t, Narrow, false>);
  }
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}
}  // namespace

int replay_launch(const ReplayDev& r, cudaStream_t stream, const GateDev* gate) {
  if (!gate && r.fn_hi > r.fn_lo) {
    const int rc = region_launch(r, r.fn_lo, r.fn_hi, stream);
    if (rc != DFX_OK) return rc;
  }
  int rc = launch_items(r, r.item_fn, r.item_chunk, r.n_items, r.max_slots, r.next, false,
                        stream, gate);
  if (rc != DFX_OK || gate) return rc;
  return replay_launch_wide(r, stream);
}

int replay_launch_backfill(const ReplayDev& r, cudaStream_t stream, const GateDev* gate) {
  return launch_items(r, r.item_fn, r.item_chunk, r.n_items, r.max_slots, r.next, false, stream,
                      gate, true);
}

int replay_launch_wide(const ReplayDev& r, cudaStream_t stream) {
  if (r.n_wide_items <= 0) return DFX_OK;
  return launch_items(r, r.wide_item_fn, r.wide_item_chunk, r.n_wide_items, r.wide_max_slots,
                      r.wide_next, true, stream, nullptr);
}

}  // namespace dfx
