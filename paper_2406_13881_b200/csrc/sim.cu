// sim.cu -- the transfer simulator as a batched verifier.
//
// Semantics: dartomp/simulator.py:180-708 (`_Simulator`, `simulate`).  The
// host lowering (paper_2406_13881_b200/simlower.py) runs the simulator's walk
// with every control decision resolved -- concrete scalar values folded into
// `if` conditions and trip counts, returns, call inlining with alias
// bindings -- because none of them depends on any variable's state.  What is
// left is the per-variable state machine of `_VarSim` (ref count, host-valid,
// device-valid, simulator.py:170-177) driven by READ / WRITE / ENTER / EXIT /
// UPDATE ops, which this kernel runs with one lane per resolved variable and
// one warp per (program, 32-variable chunk), control uniform across the warp
// (the same layout as the E1 replay, replay.cu).
//
// Loops (`run_loop`, simulator.py:528-550).  The reference runs rounds until
// two consecutive rounds leave the whole environment, the concrete values and
// the round's events unchanged, then multiplies the last round's events by
// the remaining trip count (`_scale_tail`).  Per variable that is the same
// total: once a variable's state s_r equals s_{r-1} under the steady control
// variant (every round from then on runs the same ops), s_r is a fixed point
// of the round, so every later round -- concrete or scaled, whenever the
// reference's global test happens to fire -- produces the events of round
// r+1.  A lane therefore counts rounds until its own state repeats, runs one
// more round counted (trip - r) times, and is inert (counted 0 times) while
// other lanes of the warp go on.  Round 10000 (_MAX_CONCRETE_ROUNDS) counts
// (trip - 9999) times for lanes still unsettled, which is the reference's
// extrapolation from the last concrete round, and records the warning.
// Untaken if-arms (simulator.py:446-477) run between CHECK_BEGIN/END: their
// stale reads count, their state and transfer counts are rolled back.
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/dfx.h"
#include "dfx_internal.h"

namespace dfx {

constexpr int kSimNest = DFX_SIM_MAX_NEST;
enum : uint8_t { kActive = 0, kScale = 1, kInert = 2 };

struct SimLoopFrame {
  int pc, nvar, round, ret;
  long long trip;
};
struct SimWarpCtl {
  SimLoopFrame lp[kSimNest];
  int nlp, nck;
};

__device__ __forceinline__ bool mul_ovf(uint64_t a, uint64_t b, uint64_t& out) {
  out = a * b;
  return __umul64hi(a, b) != 0ull;
}

__device__ __forceinline__ void sim_emit(dfx_sim_rec* recs, unsigned long long* count, int64_t cap,
                                         int prog, int var, int id, int kind, uint64_t n) {
  const unsigned long long i = atomicAdd(count, 1ull);
  if ((int64_t)i < cap) {
    dfx_sim_rec r;
    r.prog = prog; r.var = var; r.id = id; r.kind = kind; r.count = n;
    recs[i] = r;
  }
}

__global__ void __launch_bounds__(128)
sim_kernel(const dfx_sim_prog* __restrict__ progs, const int4* __restrict__ ops,
           const long long* __restrict__ arg64, const int32_t* __restrict__ item_prog,
           const int32_t* __restrict__ item_chunk, int n_items, dfx_sim_var* __restrict__ vout,
           dfx_sim_rec* __restrict__ recs, int64_t rec_cap,
           unsigned long long* __restrict__ rec_count, unsigned* __restrict__ next) {
  __shared__ SimWarpCtl ctl_all[4];
  const int lane = threadIdx.x & 31;
  SimWarpCtl& c = ctl_all[threadIdx.x >> 5];
  for (;;) {
    int item = 0;
    if (lane == 0) item = (int)atomicAdd(next, 1u);
    item = __shfl_sync(0xFFFFFFFFu, item, 0);
    if (item >= n_items) return;
    const int pi = __ldg(item_prog + item), chunk = __ldg(item_chunk + item);
    const dfx_sim_prog pd = progs[pi];
    const int4* pops = ops + pd.op_off;
    const long long* parg = arg64 + pd.op_off;
    const int var = chunk * 32 + lane;
    const bool lane_on = var < pd.n_vars;
    const int myvar = lane_on ? var : -1;
    if (lane == 0) { c.nlp = 0; c.nck = 0; }
    __syncwarp();

    // lane state (`_VarSim`) and counters
    long long ref = 0;
    int hv = 1, dv = 0;
    uint64_t htc = 0, htb = 0, dtc = 0, dtb = 0, stale = 0;
    uint64_t m = 1;                 // how many times the current round counts
    uint64_t shield = 0;            // (hv, dv) pairs pushed by SHIELD_SAVE
    int ssp = 0;
    int vflags = 0;
    // per loop level: status, multiplier of the enclosing code, state at round start
    uint8_t lst[kSimNest];
    uint64_t lmpar[kSimNest];
    long long lref[kSimNest];
    uint8_t lhd[kSimNest];
    // per untaken-arm level: state and transfer counts to roll back to
    long long cref[kSimNest];
    uint8_t chd[kSimNest];
    uint64_t cc[kSimNest][4];

    auto add = [&](uint64_t& acc, uint64_t mult, uint64_t v) {
      uint64_t p;
      if (mul_ovf(mult, v, p)) vflags |= DFX_SIM_VF_OVERFLOW;
      const uint64_t s = acc + p;
      if (s < acc) vflags |= DFX_SIM_VF_OVERFLOW;
      acc = s;
    };
    // jump to the VAR_BEGIN of variant k (1-based) of the loop at lpc
    auto variant_pc = [&](int lpc, int k) {
      int q = lpc + 1;
      for (int i = 1; i < k; i++) q += __ldg(&pops[q].y) + 1;
      return q;
    };

    int pc = 0;
    int wbase = -64;
    int4 wop = make_int4(0, 0, 0, 0);
    unsigned rel = 0u;
    for (;;) {
      if ((unsigned)(pc - wbase) >= 32u) {
        wbase = pc;
        bool r = true;
        if (wbase + lane < pd.n_ops) {
          wop = __ldg(pops + wbase + lane);
          const int cd = wop.x & 0xFF;
          r = !(cd >= DFX_SIM_READ && cd <= DFX_SIM_UNSHIELD && (wop.y >> 5) != chunk);
        } else {
          wop = make_int4(DFX_SIM_END, 0, 0, 0);   // past the end: stop
        }
        rel = __ballot_sync(0xFFFFFFFFu, r);
      }
      const unsigned msk = rel & (0xFFFFFFFFu << (pc - wbase));
      if (!msk) { pc = wbase + 32; continue; }
      const int src = __ffs(msk) - 1;
      pc = wbase + src;
      const int4 op = make_int4(__shfl_sync(0xFFFFFFFFu, wop.x, src), __shfl_sync(0xFFFFFFFFu, wop.y, src),
                                __shfl_sync(0xFFFFFFFFu, wop.z, src), __shfl_sync(0xFFFFFFFFu, wop.w, src));
      const int code = op.x & 0xFF;
      switch (code) {
        case DFX_SIM_END:
          goto done;
        case DFX_SIM_READ: {            // simulator.py:265-270
          if (op.y != myvar) break;
          const int ok = op.z ? dv : hv;
          if (!ok) {
            add(stale, m, 1ull);
            if (m) sim_emit(recs, rec_count, rec_cap, pi, var, op.w | (op.z << 30), DFX_SIM_REC_STALE, m);
          }
          break;
        }
        case DFX_SIM_WRITE: {           // simulator.py:272-280
          if (op.y != myvar) break;
          if (op.z == 0) { hv = 1; if (ref > 0) dv = 0; }
          else { dv = 1; hv = 0; }
          break;
        }
        case DFX_SIM_ENTER: {           // map_enter, simulator.py:232-240
          if (op.y != myvar) break;
          if (ref == 0) {
            if (op.z == 0 || op.z == 1) {
              add(htc, m, 1ull);
              add(htb, m, (uint64_t)__ldg(parg + pc));
              dv = hv;
            } else {
              dv = 0;
            }
          }
          ref++;
          break;
        }
        case DFX_SIM_EXIT: {            // map_exit, simulator.py:242-252
          if (op.y != myvar) break;
          if (ref == 0) {
            if (m) sim_emit(recs, rec_count, rec_cap, pi, var, op.w, DFX_SIM_REC_WARN, 1ull);
            break;
          }
          ref--;
          if (ref == 0) {
            if (op.z == 1 || op.z == 2) {
              add(dtc, m, 1ull);
              add(dtb, m, (uint64_t)__ldg(parg + pc));
              hv = dv;
            }
            dv = 0;
          }
          break;
        }
        case DFX_SIM_UPDATE: {          // update, simulator.py:254-260 (_copy :222-230)
          if (op.y != myvar) break;
          if (ref == 0) {
            if (m) sim_emit(recs, rec_count, rec_cap, pi, var, op.w, DFX_SIM_REC_WARN, 1ull);
            break;
          }
          if (op.z == 0) { add(htc, m, 1ull); add(htb, m, (uint64_t)__ldg(parg + pc)); dv = hv; }
          else { add(dtc, m, 1ull); add(dtb, m, (uint64_t)__ldg(parg + pc)); hv = dv; }
          break;
        }
        case DFX_SIM_SHIELD_SAVE: {     // per-thread copies, simulator.py:679-687
          if (op.y != myvar) break;
          if (ssp >= 32) { vflags |= DFX_SIM_VF_FAULT; break; }
          shield |= (uint64_t)(hv | (dv << 1)) << (2 * ssp);
          ssp++;
          break;
        }
        case DFX_SIM_SHIELD_SET:
          if (op.y == myvar) dv = 1;
          break;
        case DFX_SIM_UNSHIELD: {
          if (op.y != myvar) break;
          if (ssp <= 0) { vflags |= DFX_SIM_VF_FAULT; break; }
          ssp--;
          const int b = (int)((shield >> (2 * ssp)) & 3ull);
          shield &= ~(3ull << (2 * ssp));
          hv = b & 1; dv = b >> 1;
          break;
        }
        case DFX_SIM_CHECK_BEGIN: {     // untaken arm: roll back afterwards
          if (!(((uint32_t)op.z >> (chunk & 31)) & 1u)) { pc += op.y + 1; continue; }
          const int k = c.nck;
          if (k >= kSimNest) { vflags |= DFX_SIM_VF_FAULT; goto done; }
          cref[k] = ref; chd[k] = (uint8_t)(hv | (dv << 1));
          cc[k][0] = htc; cc[k][1] = htb; cc[k][2] = dtc; cc[k][3] = dtb;
          __syncwarp();
          if (lane == 0) c.nck = k + 1;
          __syncwarp();
          break;
        }
        case DFX_SIM_CHECK_END: {       // stale reads stay, the rest rolls back
          const int k = c.nck - 1;
          ref = cref[k]; hv = chd[k] & 1; dv = chd[k] >> 1;
          htc = cc[k][0]; htb = cc[k][1]; dtc = cc[k][2]; dtb = cc[k][3];
          __syncwarp();
          if (lane == 0) c.nck = k;
          __syncwarp();
          break;
        }
        case DFX_SIM_LOOP: {
          if (!(((uint32_t)op.z >> (chunk & 31)) & 1u)) { pc += op.y; continue; }
          const int k = c.nlp;
          if (k >= kSimNest) { vflags |= DFX_SIM_VF_FAULT; goto done; }
          const long long trip = __ldg(parg + pc);
          lst[k] = kActive;
          lmpar[k] = m;
          lref[k] = ref; lhd[k] = (uint8_t)(hv | (dv << 1));
          __syncwarp();
          if (lane == 0) {
            SimLoopFrame& f = c.lp[k];
            f.pc = pc; f.nvar = op.w; f.round = 1; f.ret = 0; f.trip = trip;
            c.nlp = k + 1;
          }
          __syncwarp();
          pc = pc + 1;            // variant 1
          continue;
        }
        case DFX_SIM_VAR_BEGIN: {
          if (lane == 0) c.lp[c.nlp - 1].ret = (op.x & DFX_SIM_F_RET) ? 1 : 0;
          __syncwarp();
          break;
        }
        case DFX_SIM_VAR_END: {         // end of round r of the innermost loop
          const int k = c.nlp - 1;
          const SimLoopFrame f = c.lp[k];
          const int r = f.round;
          const bool steady = r >= f.nvar;
          if (!f.ret && (long long)r < f.trip) {
            if (lst[k] == kScale) {
              lst[k] = kInert;
            } else if (lst[k] == kActive) {
              const bool same = ref == lref[k] && (uint8_t)(hv | (dv << 1)) == lhd[k];
              if (r >= DFX_SIM_MAX_ROUNDS) {
                // the cap round was already counted trip - r + 1 times
                if (!(same && steady) && lane_on)
                  sim_emit(recs, rec_count, rec_cap, pi, var, 0, DFX_SIM_REC_NOSETTLE, 1ull);
                lst[k] = kInert;
              } else if (steady && same) {
                lst[k] = kScale;
              }
            }
          }
          const bool more = !f.ret && (long long)r < f.trip && r < DFX_SIM_MAX_ROUNDS &&
                            __any_sync(0xFFFFFFFFu, lst[k] != kInert);
          if (!more) {
            m = lmpar[k];
            __syncwarp();
            if (lane == 0) c.nlp = k;
            __syncwarp();
            pc = f.pc + __ldg(&pops[f.pc].y);   // after the last variant
            continue;
          }
          const int rn = r + 1;
          // multiplier of round rn
          if (lst[k] == kActive) {
            lref[k] = ref; lhd[k] = (uint8_t)(hv | (dv << 1));
            if (rn >= DFX_SIM_MAX_ROUNDS && (long long)rn < f.trip) {
              // last concrete round: it also stands for the trip - rn
              // extrapolated ones (`_scale_tail` at _MAX_CONCRETE_ROUNDS)
              if (mul_ovf(lmpar[k], (uint64_t)(f.trip - rn + 1), m)) vflags |= DFX_SIM_VF_OVERFLOW;
            } else {
              m = lmpar[k];
            }
          } else if (lst[k] == kScale) {
            if (mul_ovf(lmpar[k], (uint64_t)(f.trip - r), m)) vflags |= DFX_SIM_VF_OVERFLOW;
          } else {
            m = 0;
          }
          __syncwarp();
          if (lane == 0) c.lp[k].round = rn;
          __syncwarp();
          pc = variant_pc(f.pc, rn < f.nvar ? rn : f.nvar);
          continue;
        }
        case DFX_SIM_WARN:               // reported by the host from the lowering
          break;
        default:
          vflags |= DFX_SIM_VF_FAULT;
          goto done;
      }
      pc++;
    }
  done:
    __syncwarp();
    if (lane_on) {
      dfx_sim_var o;
      o.htod_calls = htc; o.htod_bytes = htb; o.dtoh_calls = dtc; o.dtoh_bytes = dtb;
      o.stale = stale; o.ref = ref;
      o.host_valid = (uint8_t)hv; o.device_valid = (uint8_t)dv; o.flags = (uint8_t)vflags;
      for (int i = 0; i < 5; i++) o.pad[i] = 0;
      vout[pd.var_off + var] = o;
    }
  }
}

int sim_launch(const SimDev& s, cudaStream_t stream) {
  if (s.n_items <= 0) return DFX_OK;
  if (cudaMemsetAsync(s.next, 0, sizeof(unsigned), stream) != cudaSuccess) return DFX_E_CUDA;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sim_kernel, 128, 0);
  int blocks = sms * (per_sm > 0 ? per_sm : 1);
  const int need = (s.n_items + 3) / 4;
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  sim_kernel<<<blocks, 128, 0, stream>>>(s.progs, reinterpret_cast<const int4*>(s.ops),
                                         reinterpret_cast<const long long*>(s.arg64), s.item_prog,
                                         s.item_chunk, s.n_items, s.vars, s.recs, s.rec_cap,
                                         s.rec_count, s.next);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

}  // namespace dfx
