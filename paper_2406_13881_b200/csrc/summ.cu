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
#include <cooperative_groups.h>

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

// Rebuild function f's summary (bits + insertion order) into `cur`; returns
// (warp-uniform) whether its bit set differs from `prev`.
// Per-warp shared memory of cg_function: the seen bitmap (nsp / 32 words)
// and, for functions with many sources, the summary row being built (nsp / 4).
// (both parts kept at multiples of 4 words: the row is read as 16-byte quads)
// and first-occurrence positions (nsp words) for those functions' order
__host__ __device__ __forceinline__ int cg_seen_words(int nsp) { return (((nsp + 31) >> 5) + 3) & ~3; }
__host__ __device__ __forceinline__ int cg_row_words(int nsp) { return (((nsp + 3) >> 2) + 3) & ~3; }
constexpr int kCgManySources = 24;
__host__ __device__ __forceinline__ int cg_warp_words(int nsp, bool many) {
  return cg_seen_words(nsp) + (many ? cg_row_words(nsp) + ((nsp + 3) & ~3) : 0);
}

bool cg_many_sources(const int32_t* src_off, int n_funcs) {
  for (int f = 0; f < n_funcs; f++)
    if (src_off[f + 1] - src_off[f] > kCgManySources) return true;
  return false;
}

__device__ __forceinline__ bool cg_function(const CgDev& g, const CgBuf& prev, const CgBuf& cur,
                                            int f, uint32_t* seen, int lane) {
  const int sw = g.nsp >> 5;                       // seen words per warp
  const int nq = g.nsp >> 4;
  const int P = g.n_params;
  {
    const int s0 = __ldg(g.src_off + f), s1 = __ldg(g.src_off + f + 1);
    // ---- bits: direct | OR of transformed callee rows ----------------------
    bool ch = false;
    if (g.many && s1 - s0 > kCgManySources) {
      // many sources (a driver calling hundreds of functions): lanes over
      // sources, 32 callee rows per step OR-reduced quad by quad into the
      // row in shared memory, each lane's bound parameters ORed in with
      // shared atomics -- instead of every lane walking all sources serially
      uint32_t* row = seen + cg_seen_words(g.nsp);
      for (int w = lane; w < (g.nsp >> 2); w += 32)
        row[w] = __ldg(reinterpret_cast<const uint32_t*>(g.direct + (size_t)f * g.nsp) + w);
      __syncwarp();
      for (int k0 = s0; k0 < s1; k0 += 32) {
        const int k = k0 + lane;
        const int4 r = k < s1 ? __ldg(reinterpret_cast<const int4*>(g.src) + k) : make_int4(0, 0, 0, 0);
        const bool call = (r.x & 0xFF) != 0;
        const bool dev = (r.x >> 8) & 1;
        const uint8_t* cb = call ? (r.y < f ? cur.bits : prev.bits) + (size_t)r.y * g.nsp : nullptr;
        for (int q = 0; q < nq; q++) {
          uint4 v = call ? __ldcg(reinterpret_cast<const uint4*>(cb) + q) : make_uint4(0u, 0u, 0u, 0u);
          if (q * 16 < P) {
            uint8_t* vb = reinterpret_cast<uint8_t*>(&v);
#pragma unroll
            for (int t = 0; t < 16; t++)
              if (q * 16 + t < P) vb[t] = 0;            // callee params bind below
          }
          if (dev) { v.x = force_dev4(v.x); v.y = force_dev4(v.y); v.z = force_dev4(v.z); v.w = force_dev4(v.w); }
          v.x = __reduce_or_sync(FULLM, v.x);
          v.y = __reduce_or_sync(FULLM, v.y);
          v.z = __reduce_or_sync(FULLM, v.z);
          v.w = __reduce_or_sync(FULLM, v.w);
          if (lane == 0) {
            row[4 * q] |= v.x; row[4 * q + 1] |= v.y; row[4 * q + 2] |= v.z; row[4 * q + 3] |= v.w;
          }
        }
        __syncwarp();
        if (call)
          for (int j = r.z; j < r.z + r.w; j++) {
            const int i = __ldg(g.bind + 2 * j), sl = __ldg(g.bind + 2 * j + 1);
            uint32_t e = __ldcg(cb + i);
            if (!(e & 3u)) continue;
            if (dev) e = (e & 3u) | 8u;
            atomicOr(&row[sl >> 2], e << (8 * (sl & 3)));
          }
        __syncwarp();
      }
      for (int q = lane; q < nq; q += 32) {
        const uint4 acc = *reinterpret_cast<const uint4*>(row + 4 * q);
        const uint4 old = __ldcg(reinterpret_cast<const uint4*>(prev.bits + (size_t)f * g.nsp) + q);
        ch |= (old.x != acc.x) | (old.y != acc.y) | (old.z != acc.z) | (old.w != acc.w);
        __stcg(reinterpret_cast<uint4*>(cur.bits + (size_t)f * g.nsp) + q, acc);
      }
    } else
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
    const bool any = __any_sync(FULLM, ch);
    // ---- insertion order ------------------------------------------------------
    int16_t* out = cur.list + (size_t)f * g.nsp;
    if (g.many && s1 - s0 > kCgManySources && s1 - s0 < (1 << 12)) {
      // many sources: the order is the distinct candidates sorted by first
      // occurrence, so each candidate's position in the candidate sequence --
      // (source, part: bound parameters before globals, index in the list)
      // -- is min-reduced per slot with shared atomics, lanes over sources;
      // a slot's place in the list is then the number of slots seen earlier
      uint32_t* fpos = seen + cg_seen_words(g.nsp) + cg_row_words(g.nsp);
      for (int w = lane; w < g.nsp; w += 32) fpos[w] = 0xFFFFFFFFu;
      __syncwarp();
      for (int k0 = s0; k0 < s1; k0 += 32) {
        const int k = k0 + lane;
        if (k >= s1) continue;
        const int4 r = __ldg(reinterpret_cast<const int4*>(g.src) + k);
        const uint32_t kb = (uint32_t)(k - s0) << 20;
        if ((r.x & 0xFF) == 0) {                 // static list
          for (int j = 0; j < r.z; j++)
            atomicMin(&fpos[__ldg(g.slist + r.y + j)], kb | (uint32_t)j);
          continue;
        }
        const int callee = r.y;
        const CgBuf& b = callee < f ? cur : prev;
        const int glen = __ldcg(b.len + callee);
        const int16_t* gl = b.list + (size_t)callee * g.nsp;
        for (int j = 0; j < glen; j++) {
          const int x = __ldcg(gl + j);
          if (x >= P) {                          // globals, after the bound parameters
            atomicMin(&fpos[x], kb | (1u << 19) | (uint32_t)j);
          } else {
            for (int t = r.z; t < r.z + r.w; t++)
              if (__ldg(g.bind + 2 * t) == x) {
                atomicMin(&fpos[__ldg(g.bind + 2 * t + 1)], kb | (uint32_t)j);
                break;
              }
          }
        }
      }
      __syncwarp();
      int len = 0;
      for (int s0l = 0; s0l < g.nsp; s0l += 32) {
        const int sl = s0l + lane;
        const uint32_t mine = sl < g.nsp ? fpos[sl] : 0xFFFFFFFFu;
        if (mine != 0xFFFFFFFFu) {
          int rank = 0;
          for (int t = 0; t < g.nsp; t++) rank += fpos[t] < mine;
          out[rank] = (int16_t)sl;
        }
        len += __popc(__ballot_sync(FULLM, mine != 0xFFFFFFFFu));
      }
      if (lane == 0) __stcg(cur.len + f, len);
      return any;
    }
    for (int w = lane; w < sw; w += 32) seen[w] = 0u;
    __syncwarp();
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
    return any;
  }
}

__global__ void __launch_bounds__(kCgWarps * 32)
cg_wave_kernel(CgDev g, CgBuf prev, CgBuf cur, int lo, int hi, int shard, int nshards,
               int* __restrict__ changed) {
  extern __shared__ uint32_t seen_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* seen = seen_all + warp * cg_warp_words(g.nsp, g.many);
  const int warps = (gridDim.x * blockDim.x) >> 5;
  bool any = false;
  for (int pos = lo + shard + nshards * ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); pos < hi;
       pos += nshards * warps)
    any |= cg_function(g, prev, cur, __ldg(g.wave_fns + pos), seen, lane);
  if (any && lane == 0) atomicOr(changed, 1);
}

// All passes in one persistent cooperative launch: waves are separated by
// grid-wide barriers, passes alternate the two tables, and the kernel exits
// uniformly after the first pass that changed no bit set.  changed[p] is the
// flag of pass p (zeroed by the host); *passes_out = passes run.
__global__ void __launch_bounds__(kCgWarps * 32)
cg_solve_kernel(CgDev g, CgBuf t0, CgBuf t1, const int* __restrict__ wave_off, int first_pass,
                int max_passes, int* __restrict__ changed, int* __restrict__ passes_out) {
  namespace cgr = cooperative_groups;
  cgr::grid_group grid = cgr::this_grid();
  extern __shared__ uint32_t seen_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* seen = seen_all + warp * cg_warp_words(g.nsp, g.many);
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int pass = first_pass; pass <= max_passes; pass++) {
    const CgBuf& prev = (pass & 1) ? t0 : t1;
    const CgBuf& cur = (pass & 1) ? t1 : t0;
    bool any = false;
    for (int w = 0; w < g.n_waves; w++) {
      const int lo = __ldg(wave_off + w), hi = __ldg(wave_off + w + 1);
      for (int pos = lo + gw; pos < hi; pos += warps)
        any |= cg_function(g, prev, cur, __ldg(g.wave_fns + pos), seen, lane);
      grid.sync();
    }
    if (any && lane == 0) atomicOr(changed + pass, 1);
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) *passes_out = pass;
    if (!__ldcg(changed + pass)) break;
  }
}

int cg_wave(const CgDev& g, uint8_t* pbits, int16_t* plist, int32_t* plen, uint8_t* cbits,
            int16_t* clist, int32_t* clen, int wave, int shard, int nshards, int* d_changed,
            cudaStream_t st) {
  const int lo = g.h_wave_off[wave], hi = g.h_wave_off[wave + 1];
  const int n = (hi - lo + nshards - 1) / nshards;
  if (n <= 0) return DFX_OK;
  int blocks = (n + kCgWarps - 1) / kCgWarps;
  if (blocks > 148 * 8) blocks = 148 * 8;
  const size_t smem = (size_t)kCgWarps * cg_warp_words(g.nsp, g.many) * sizeof(uint32_t);
  CgBuf prev{pbits, plist, plen}, cur{cbits, clist, clen};
  cg_wave_kernel<<<blocks, kCgWarps * 32, smem, st>>>(g, prev, cur, lo, hi, shard, nshards,
                                                      d_changed);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

// Final exchange of the component-sharded solve (api.cu
// dfx_summaries_sharded): each rank packs the rows it owns -- bits, insertion
// order, length -- into one contiguous send block; after the all-gather every
// rank scatters the other ranks' blocks into its table.  One warp per row.
__global__ void cg_pack_kernel(CgBuf t, int nsp, const int32_t* __restrict__ fns, int n,
                               uint8_t* __restrict__ out, int rowb) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += (gridDim.x * blockDim.x) >> 5) {
    const int f = __ldg(fns + i);
    uint8_t* o = out + (size_t)i * rowb;
    for (int c = lane; c < nsp; c += 32) o[c] = t.bits[(size_t)f * nsp + c];
    int16_t* ol = reinterpret_cast<int16_t*>(o + nsp);
    for (int c = lane; c < nsp; c += 32) ol[c] = t.list[(size_t)f * nsp + c];
    if (lane == 0) *reinterpret_cast<int32_t*>(o + 3 * nsp) = t.len[f];
  }
}
__global__ void cg_unpack_kernel(CgBuf t, int nsp, const int32_t* __restrict__ fns, int n,
                                 const uint8_t* __restrict__ in, int rowb) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += (gridDim.x * blockDim.x) >> 5) {
    const int f = __ldg(fns + i);
    const uint8_t* o = in + (size_t)i * rowb;
    for (int c = lane; c < nsp; c += 32) t.bits[(size_t)f * nsp + c] = o[c];
    const int16_t* ol = reinterpret_cast<const int16_t*>(o + nsp);
    for (int c = lane; c < nsp; c += 32) t.list[(size_t)f * nsp + c] = ol[c];
    if (lane == 0) t.len[f] = *reinterpret_cast<const int32_t*>(o + 3 * nsp);
  }
}

int cg_pack(uint8_t* b, int16_t* l, int32_t* n, int nsp, const int32_t* fns, int count,
            uint8_t* out, int rowb, bool unpack, cudaStream_t st) {
  if (count <= 0) return DFX_OK;
  int blocks = (count + 7) / 8;
  if (blocks > 148 * 8) blocks = 148 * 8;
  CgBuf t{b, l, n};
  if (unpack) cg_unpack_kernel<<<blocks, 256, 0, st>>>(t, nsp, fns, count, out, rowb);
  else cg_pack_kernel<<<blocks, 256, 0, st>>>(t, nsp, fns, count, out, rowb);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

// row re-pitching between the ABI's dense [rows][n] layout and the kernels'
// padded [rows][np] layout (elements of `es` bytes; padding zero-filled)
__global__ void repitch_kernel(const uint8_t* __restrict__ src, size_t sp, uint8_t* __restrict__ dst,
                               size_t dp, size_t width, size_t rows) {
  const size_t total = rows * dp;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / dp, c = i - r * dp;
    dst[i] = c < width ? src[r * sp + c] : (uint8_t)0;
  }
}

int repitch(const void* src, size_t sp, void* dst, size_t dp, size_t width, size_t rows,
            cudaStream_t st) {
  if (!rows || !dp) return DFX_OK;
  size_t g = (rows * dp + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  repitch_kernel<<<(int)g, 256, 0, st>>>((const uint8_t*)src, sp, (uint8_t*)dst, dp, width, rows);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

// whole solve on the device; returns the passes run through *passes (device)
int cg_solve(const CgDev& g, uint8_t* b0, int16_t* l0, int32_t* n0, uint8_t* b1, int16_t* l1,
             int32_t* n1, const int32_t* d_wave_off, int max_passes, int* d_changed,
             int* d_passes, cudaStream_t st, int first_pass) {
  const size_t smem = (size_t)kCgWarps * cg_warp_words(g.nsp, g.many) * sizeof(uint32_t);
  // occupancy per (device, smem size)
  constexpr int kDevs = 64;
  static int sms_d[kDevs] = {}, per_sm_d[kDevs] = {};
  static size_t smem_d[kDevs];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kDevs) return DFX_E_CUDA;
  if (!sms_d[dev]) {
    cudaDeviceGetAttribute(&sms_d[dev], cudaDevAttrMultiProcessorCount, dev);
    smem_d[dev] = (size_t)-1;
  }
  if (smem != smem_d[dev]) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_d[dev], cg_solve_kernel, kCgWarps * 32, smem);
    smem_d[dev] = smem;
  }
  const int sms = sms_d[dev], per_sm = per_sm_d[dev];
  if (per_sm < 1) return DFX_E_LIMIT;
  int max_wave = 0;
  for (int w = 0; w < g.n_waves; w++) {
    const int n = g.h_wave_off[w + 1] - g.h_wave_off[w];
    if (n > max_wave) max_wave = n;
  }
  int blocks = (max_wave + kCgWarps - 1) / kCgWarps;
  if (blocks > sms * per_sm) blocks = sms * per_sm;
  if (blocks < 1) blocks = 1;
  CgDev gg = g;
  CgBuf t0{b0, l0, n0}, t1{b1, l1, n1};
  void* args[] = {&gg, &t0, &t1, &d_wave_off, &first_pass, &max_passes, &d_changed, &d_passes};
  if (cudaLaunchCooperativeKernel((const void*)cg_solve_kernel, dim3(blocks), dim3(kCgWarps * 32),
                                  args, smem, st) != cudaSuccess)
    return DFX_E_CUDA;
  return DFX_OK;
}

// ---------------------------------------------------------------------------
// cgpeer.cu -- kernel (c) across GPUs with the exchange fused into the
// producing kernel, over peer memory (NVLink P2P through CUDA IPC).
//
// The reference's pass schedule (interproc.py:105-143) runs wave by wave;
// a wave's functions are split round-robin over the ranks.  In the NCCL
// path (distributed.py) every rank rebuilds its share, then the ranks
// all-gather the rebuilt rows and scatter them into their tables.  Here the
// kernel that rebuilds a function's summary row also stores it straight into
// every peer's table (one warp-wide coalesced copy per peer), so the rows
// cross NVLink while other warps are still computing.  A wave ends when
// every rank's wave kernel has released its arrival on every peer:
//   writer: row stores -> fence.sc.sys -> (last block) atomicAdd_system on
//           each rank's arrival counter
//   reader: a one-warp wait kernel acquires (ld.acquire.sys) its own
//           counter until it reaches waves_done * nranks; the next wave's
//           kernel is stream-ordered after it.
// The changed flag of a pass is raised on every rank's flag the same way
// (atomicMax of the solve's generation number, so flags need no clearing
// between solves), so every rank takes the same termination decision.
constexpr unsigned FULLP = 0xFFFFFFFFu;
constexpr int kPeerWarps = 8;


__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(kPeerWarps * 32)
cg_wave_peer_kernel(CgDev g, PeerTables tab, int cur, int lo, int hi, int rank, int nranks,
                    int pass, int gen, unsigned int* blocks_done) {
  extern __shared__ uint32_t seen_all[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t* seen = seen_all + warp * cg_warp_words(g.nsp, g.many);
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int prev = cur ^ 1;
  const size_t nsp = (size_t)g.nsp;
  uint8_t* const lbits = tab.bits[rank][cur];
  int16_t* const llist = tab.list[rank][cur];
  int32_t* const llen = tab.len[rank][cur];
  bool any = false;
  for (int pos = lo + rank + nranks * ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); pos < hi;
       pos += nranks * warps) {
    const int f = __ldg(g.wave_fns + pos);
    const CgBuf pb{tab.bits[rank][prev], tab.list[rank][prev], tab.len[rank][prev]};
    const CgBuf cb{lbits, llist, llen};
    any |= cg_function(g, pb, cb, f, seen, lane);
    __syncwarp();
    // the rebuilt row goes to every peer's table (16-B lanes, coalesced)
    const uint4* sb = reinterpret_cast<const uint4*>(lbits + (size_t)f * nsp);
    const uint4* sl = reinterpret_cast<const uint4*>(llist + (size_t)f * nsp);
    const int len = __ldcg(llen + f);
    for (int r = 0; r < nranks; r++) {
      if (r == rank) continue;
      uint4* db = reinterpret_cast<uint4*>(tab.bits[r][cur] + (size_t)f * nsp);
      uint4* dl = reinterpret_cast<uint4*>(tab.list[r][cur] + (size_t)f * nsp);
      for (int q = lane; q < (int)(nsp / 16); q += 32) __stcg(db + q, __ldcg(sb + q));
      for (int q = lane; q < (int)(nsp / 8); q += 32) __stcg(dl + q, __ldcg(sl + q));
      if (lane == 0) tab.len[r][cur][f] = len;
    }
  }
  if (__any_sync(FULLP, any) && lane == 0)
    for (int r = 0; r < nranks; r++) atomicMax_system(tab.changed[r] + pass, gen);
  // release: this block's peer stores, then (last block) the arrivals
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev_done = atomicAdd(blocks_done, 1u);
    if (prev_done == gridDim.x - 1) {
      __threadfence_system();
      for (int r = 0; r < nranks; r++) atomicAdd_system(tab.arrive[r], 1ull);
    }
  }
}

// one warp: wait until every rank has finished `waves` waves (acquire), or
// give up after `spins` polls (a peer that never arrives) with *err = 1
__global__ void cg_wait_kernel(const unsigned long long* arrive, unsigned long long expect,
                               long long spins, int* err) {
  if (threadIdx.x != 0) return;
  for (long long i = 0; i < spins; i++) {
    if (ld_acquire_sys(arrive) >= expect) return;
    __nanosleep(200);
  }
  atomicExch(err, 1);
}

int cg_peer_wave(const CgDev& g, const PeerTables& tab, int cur, int wave, int rank, int nranks,
                 int pass, int gen, unsigned int* blocks_done, cudaStream_t st) {
  const int lo = g.h_wave_off[wave], hi = g.h_wave_off[wave + 1];
  const int n = (hi - lo + nranks - 1) / nranks;
  int blocks = (n + kPeerWarps - 1) / kPeerWarps;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;            // an empty share still signals its arrival
  const size_t smem = (size_t)kPeerWarps * cg_warp_words(g.nsp, g.many) * sizeof(uint32_t);
  if (cudaMemsetAsync(blocks_done, 0, sizeof(unsigned int), st) != cudaSuccess) return DFX_E_CUDA;
  cg_wave_peer_kernel<<<blocks, kPeerWarps * 32, smem, st>>>(g, tab, cur, lo, hi, rank, nranks,
                                                             pass, gen, blocks_done);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

int cg_peer_wait(const unsigned long long* arrive, unsigned long long expect, long long spins,
                 int* err, cudaStream_t st) {
  cg_wait_kernel<<<1, 32, 0, st>>>(arrive, expect, spins, err);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

}  // namespace dfx
