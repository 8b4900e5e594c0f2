// summ.cu -- kernel (c): interprocedural summaries, replaying the reference's
// Gauss-Seidel pass schedule exactly (dartomp/interproc.py:105-143).
//
// Each pass rebuilds every defined function's summary from its sources in
// order; a function reads its callee's summary from the current pass when
// the callee comes earlier in dict order, else from the previous pass
// (double-buffered tables).  Functions are grouped into waves so that a
// wave reads only earlier waves' same-pass results: one launch per wave,
// one warp per function.
//   bits : one byte per slot (R, W, HOST, DEVICE), lanes over 16-byte quads
//   order: the summary dicts' insertion order, rebuilt by warp-cooperative
//          first-occurrence appends (ballot + prefix popcount, a per-warp
//          seen-bitmap in shared memory)
// Passes repeat until no function's bit set changes (the reference's
// termination test compares snapshots, i.e. sets).
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/dfx.h"
#include "dfx_internal.h"

namespace dfx {

constexpr unsigned FULLM = 0xFFFFFFFFu;
constexpr int kCgWarps = 8;

__device__ __forceinline__ uint32_t force_dev4(uint32_t x) {
  uint32_t rw = x & 0x03030303u;
  uint32_t has = (rw | (rw >> 1)) & 0x01010101u;
  return rw | (has << 3);
}

struct CgBuf {
  uint8_t* bits;     // [nf][nsp]
  int16_t* list;     // [nf][nsp]
  int32_t* len;      // [nf]
};

__global__ void __launch_bounds__(kCgWarps * 32)
cg_wave_kernel(CgDev g, CgBuf prev, CgBuf cur, int lo, int hi, int shard, int nshards,
               int* __restrict__ changed) {
  extern __shared__ uint32_t seen_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sw = g.nsp >> 5;                       // seen words per warp
  uint32_t* seen = seen_all + warp * sw;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int nq = g.nsp >> 4;
  const int P = g.n_params;
  int any = 0;
  for (int pos = lo + shard + nshards * ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); pos < hi;
       pos += nshards * warps) {
    const int f = __ldg(g.wave_fns + pos);
    const int s0 = __ldg(g.src_off + f), s1 = __ldg(g.src_off + f + 1);
    // ---- bits: direct | OR of transformed callee rows ----------------------
    bool ch = false;
    for (int q = lane; q < nq; q += 32) {
      uint4 acc = __ldg(reinterpret_cast<const uint4*>(g.direct + (size_t)f * g.nsp) + q);
      uint8_t* ab = reinterpret_cast<uint8_t*>(&acc);
      for (int k = s0; k < s1; k++) {
        const int4 r = __ldg(reinterpret_cast<const int4*>(g.src) + k);
        if ((r.x & 0xFF) == 0) continue;
        const bool dev = (r.x >> 8) & 1;
        const int callee = r.y;
        const CgBuf& b = callee < f ? cur : prev;
        uint4 v = __ldcg(reinterpret_cast<const uint4*>(b.bits + (size_t)callee * g.nsp) + q);
        uint8_t* vb = reinterpret_cast<uint8_t*>(&v);
#pragma unroll
        for (int t = 0; t < 16; t++)
          if (q * 16 + t < P) vb[t] = 0;                  // callee params bind below
        if (dev) { v.x = force_dev4(v.x); v.y = force_dev4(v.y); v.z = force_dev4(v.z); v.w = force_dev4(v.w); }
        acc.x |= v.x; acc.y |= v.y; acc.z |= v.z; acc.w |= v.w;
        for (int j = r.z; j < r.z + r.w; j++) {
          const int i = __ldg(g.bind + 2 * j), s = __ldg(g.bind + 2 * j + 1);
          if ((s >> 4) != q) continue;
          uint32_t e = __ldcg(b.bits + (size_t)callee * g.nsp + i);
          if (!(e & 3u)) continue;
          if (dev) e = (e & 3u) | 8u;
          ab[s & 15] |= (uint8_t)e;
        }
      }
      const uint4 old = __ldcg(reinterpret_cast<const uint4*>(prev.bits + (size_t)f * g.nsp) + q);
      ch |= (old.x != acc.x) | (old.y != acc.y) | (old.z != acc.z) | (old.w != acc.w);
      __stcg(reinterpret_cast<uint4*>(cur.bits + (size_t)f * g.nsp) + q, acc);
    }
    any |= __any_sync(FULLM, ch);
    // ---- insertion order ------------------------------------------------------
    for (int w = lane; w < sw; w += 32) seen[w] = 0u;
    __syncwarp();
    int16_t* out = cur.list + (size_t)f * g.nsp;
    int len = 0;
    auto append = [&](int cand) {       // one candidate slot (or -1) per lane
      bool fresh = cand >= 0 && !((seen[cand >> 5] >> (cand & 31)) & 1u);
      // keep the first lane of each duplicate group (lane order = list order)
      const unsigned grp = __match_any_sync(FULLM, fresh ? cand : -1 - lane);
      fresh = fresh && (__ffs(grp) - 1) == lane;
      const unsigned m = __ballot_sync(FULLM, fresh);
      __syncwarp();
      if (fresh) {
        out[len + __popc(m & ((1u << lane) - 1u))] = (int16_t)cand;
        atomicOr(&seen[cand >> 5], 1u << (cand & 31));
      }
      len += __popc(m);
      __syncwarp();
    };
    for (int k = s0; k < s1; k++) {
      const int4 r = __ldg(reinterpret_cast<const int4*>(g.src) + k);
      if ((r.x & 0xFF) == 0) {            // static list
        for (int j = 0; j < r.z; j += 32)
          append(j + lane < r.z ? (int)__ldg(g.slist + r.y + j + lane) : -1);
        continue;
      }
      const int callee = r.y;
      const CgBuf& b = callee < f ? cur : prev;
      const int glen = __ldcg(b.len + callee);
      const int16_t* gl = b.list + (size_t)callee * g.nsp;
      for (int j = 0; j < glen; j += 32) {      // bound parameters, callee order
        int cand = -1;
        if (j + lane < glen) {
          const int x = __ldcg(gl + j + lane);
          if (x < P)
            for (int t = r.z; t < r.z + r.w; t++)
              if (__ldg(g.bind + 2 * t) == x) { cand = __ldg(g.bind + 2 * t + 1); break; }
        }
        append(cand);
      }
      for (int j = 0; j < glen; j += 32) {      // globals, callee order
        int cand = -1;
        if (j + lane < glen) {
          const int x = __ldcg(gl + j + lane);
          if (x >= P) cand = x;
        }
        append(cand);
      }
    }
    if (lane == 0) __stcg(cur.len + f, len);
  }
  if (any && lane == 0) atomicOr(changed, 1);
}

int cg_wave(const CgDev& g, uint8_t* pbits, int16_t* plist, int32_t* plen, uint8_t* cbits,
            int16_t* clist, int32_t* clen, int wave, int shard, int nshards, int* d_changed,
            cudaStream_t st) {
  const int lo = g.h_wave_off[wave], hi = g.h_wave_off[wave + 1];
  const int n = (hi - lo + nshards - 1) / nshards;
  if (n <= 0) return DFX_OK;
  int blocks = (n + kCgWarps - 1) / kCgWarps;
  if (blocks > 148 * 8) blocks = 148 * 8;
  const size_t smem = (size_t)kCgWarps * (g.nsp / 32) * sizeof(uint32_t);
  CgBuf prev{pbits, plist, plen}, cur{cbits, clist, clen};
  cg_wave_kernel<<<blocks, kCgWarps * 32, smem, st>>>(g, prev, cur, lo, hi, shard, nshards,
                                                      d_changed);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

}  // namespace dfx
