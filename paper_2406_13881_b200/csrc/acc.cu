// acc.cu -- access-list input and requirement-list output of kernels (a)+(b).
//
// The reference's front end describes every statement by a list of memory
// accesses (dartomp/access.py:58-86 `MemoryAccess`: variable, kind
// READ/WRITE/READWRITE; `classify_accesses` access.py:387-402), and its
// analysis answers with per-statement directive plans naming variables
// (dataflow.py:37-95 `DirectivePlan`).  The list forms below carry exactly
// that across the boundary, so the host<->device traffic is proportional to
// the accesses and the planned transfers, not to nodes x variables:
//
//   access entry    uint16  var | kind << 14   (kind 1 read, 2 write, 3 both)
//   requirement     uint16  var | 0x8000 if firstprivate
//
// expand_acc_kernel  : access lists -> the A/B/USE bitplanes of kernel (a)
// export_acc_kernel  : bitplanes -> access lists (benchmark/test export)
// compact_list_kernel: requirement planes of kernel (b) -> per-node variable
//                      lists, transfer requirements ascending, then
//                      firstprivate captures ascending
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/dfx.h"
#include "dfx_internal.h"

namespace dfx {

namespace {
constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int kWarps = 8;   // warps per block

__device__ __forceinline__ int warp_exclusive_scan(int v, int lane, int* total) {
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += t;
  }
  *total = __shfl_sync(FULL, incl, 31);
  return incl - v;
}
}  // namespace

// One warp per node: OR the node's access entries into two shared-memory
// rows (reads, writes), then store USE = R, B = W, A = R | W coalesced.
__global__ void __launch_bounds__(kWarps * 32)
expand_acc_kernel(int64_t n_lo, int64_t n_nodes, int words, const int64_t* __restrict__ off,
                  const uint16_t* __restrict__ acc, uint32_t* __restrict__ A,
                  uint32_t* __restrict__ B, uint32_t* __restrict__ USE, int* bad) {
  extern __shared__ uint32_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* r = sm + (size_t)warp * 2 * words;
  uint32_t* w = r + words;
  const int nvars = words * 32;
  const int64_t wstride = (int64_t)gridDim.x * kWarps;
  for (int64_t n = n_lo + (int64_t)blockIdx.x * kWarps + warp; n < n_nodes; n += wstride) {
    for (int i = lane; i < words; i += 32) r[i] = w[i] = 0u;
    __syncwarp();
    const int64_t e1 = off[n + 1];
    for (int64_t e = off[n] + lane; e < e1; e += 32) {
      const uint32_t a = acc[e];
      const uint32_t v = a & 0x3FFFu, k = a >> 14;
      if (v >= (uint32_t)nvars || k == 0u) { atomicExch(bad, 1); continue; }
      const uint32_t bit = 1u << (v & 31);
      if (k & 1u) atomicOr(&r[v >> 5], bit);
      if (k & 2u) atomicOr(&w[v >> 5], bit);
    }
    __syncwarp();
    const size_t row = (size_t)n * words;
    for (int i = 4 * lane; i < words; i += 128) {
      const uint4 rr = *reinterpret_cast<const uint4*>(r + i);
      const uint4 ww = *reinterpret_cast<const uint4*>(w + i);
      __stcs(reinterpret_cast<uint4*>(USE + row + i), rr);
      __stcs(reinterpret_cast<uint4*>(B + row + i), ww);
      __stcs(reinterpret_cast<uint4*>(A + row + i),
             make_uint4(rr.x | ww.x, rr.y | ww.y, rr.z | ww.z, rr.w | ww.w));
    }
    __syncwarp();
  }
}

// Per node: number of accessed variables (popcount of R | W).
__global__ void __launch_bounds__(kWarps * 32)
count_acc_kernel(int64_t n_nodes, int words, const uint32_t* __restrict__ A, int32_t* counts) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * kWarps;
  for (int64_t n = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); n < n_nodes; n += wstride) {
    int c = 0;
    for (int i = lane; i < words; i += 32) c += __popc(__ldg(A + (size_t)n * words + i));
    c = (int)__reduce_add_sync(FULL, (unsigned)c);
    if (lane == 0) counts[n] = c;
  }
}

// Per node: the access entries in ascending variable order.  Lane l covers
// words l, l+32, ...; a warp scan of per-lane counts gives each lane's slot.
__global__ void __launch_bounds__(kWarps * 32)
export_acc_kernel(int64_t n_nodes, int words, const uint32_t* __restrict__ R,
                  const uint32_t* __restrict__ W, const int64_t* __restrict__ off,
                  uint16_t* __restrict__ acc) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * kWarps;
  for (int64_t n = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); n < n_nodes; n += wstride) {
    int64_t base = off[n];
    for (int i0 = 0; i0 < words; i0 += 32) {
      const int i = i0 + lane;
      uint32_t r = 0u, w = 0u;
      if (i < words) {
        r = __ldg(R + (size_t)n * words + i);
        w = __ldg(W + (size_t)n * words + i);
      }
      uint32_t m = r | w;
      int tot;
      int64_t pos = base + warp_exclusive_scan(__popc(m), lane, &tot);
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t k = ((r >> b) & 1u) | (((w >> b) & 1u) << 1);
        acc[pos++] = (uint16_t)((uint32_t)(32 * i + b) | (k << 14));
      }
      base += tot;
    }
  }
}

// Requirement planes (REQ, FPQ from requirements_kernel with bit counts) ->
// per-node variable lists at offsets[n]: requirement vars ascending, then
// firstprivate vars ascending with DFX_REQ_FIRSTPRIVATE set.
__global__ void __launch_bounds__(kWarps * 32)
compact_list_kernel(int64_t n_lo, int64_t n_hi, int words, const uint32_t* __restrict__ REQ,
                    const uint32_t* __restrict__ FPQ, const int32_t* __restrict__ fp_slot,
                    int n_fp_slots, const int64_t* __restrict__ offsets,
                    uint16_t* __restrict__ vars, int64_t cap) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * kWarps;
  for (int64_t n = n_lo + (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); n < n_hi; n += wstride) {
    int64_t base = offsets[n];
    for (int pass = 0; pass < 2; pass++) {
      for (int i0 = 0; i0 < words; i0 += 32) {
        const int i = i0 + lane;
        uint32_t m = 0u;
        if (i < words) {
          if (pass == 0) {
            m = __ldg(REQ + (size_t)n * words + i);
          } else {
            const int slot = fp_slot[i >> 2];
            if (slot >= 0) m = __ldg(FPQ + ((size_t)n * n_fp_slots + slot) * 4 + (i & 3));
          }
        }
        int tot;
        int64_t pos = base + warp_exclusive_scan(__popc(m), lane, &tot);
        const uint32_t flag = pass ? (uint32_t)DFX_REQ_FIRSTPRIVATE : 0u;
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          if (pos < cap) vars[pos] = (uint16_t)((uint32_t)(32 * i + b) | flag);
          pos++;
        }
        base += tot;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Byte-coded lists (include/dfx.h "B8"): b = kind << 6 | d, d == 63 continues
// the entry (+63), d < 63 ends it (+d); var = prev + 1 + sum of its d fields.
// A byte contributes d (+1 if it ends an entry) to a running sum that starts
// at 0 for the node (and for its firstprivate list): the variable of an
// entry is the inclusive sum through its last byte, minus 1.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int warp_inclusive_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// One warp per node: decode 32 bytes per step (a warp scan gives every
// entry's variable), OR the entries into shared-memory rows, store the planes.
__global__ void __launch_bounds__(kWarps * 32)
expand_b8_kernel(int64_t n_lo, int64_t n_nodes, int words, const int32_t* __restrict__ off,
                 const uint8_t* __restrict__ bytes, uint32_t* __restrict__ A,
                 uint32_t* __restrict__ B, uint32_t* __restrict__ USE, int* bad) {
  extern __shared__ uint32_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* r = sm + (size_t)warp * 2 * words;
  uint32_t* w = r + words;
  const int nvars = words * 32;
  const int64_t wstride = (int64_t)gridDim.x * kWarps;
  for (int64_t n = n_lo + (int64_t)blockIdx.x * kWarps + warp; n < n_nodes; n += wstride) {
    for (int i = lane; i < words; i += 32) r[i] = w[i] = 0u;
    __syncwarp();
    const int e0 = off[n], e1 = off[n + 1];
    int carry = 0;
    for (int e = e0; e < e1; e += 32) {
      const bool in = e + lane < e1;
      const uint32_t b = in ? bytes[e + lane] : 63u;     // padding: a continuation adding 0
      const int d = (int)(b & 63u), end = in && d < 63;
      const int sum = carry + warp_inclusive_scan(in ? d + end : 0, lane);
      if (end) {
        const int v = sum - 1;
        const uint32_t k = b >> 6;
        if ((unsigned)v >= (unsigned)nvars || k == 0u) {   // (a huge run of continuations wraps)
          atomicExch(bad, 1);
        } else {
          const uint32_t bit = 1u << (v & 31);
          if (k & 1u) atomicOr(&r[v >> 5], bit);
          if (k & 2u) atomicOr(&w[v >> 5], bit);
        }
      }
      carry = __shfl_sync(FULL, sum, 31);
    }
    // a node's stream must end with a completed entry
    if (e1 > e0 && lane == 0 && (bytes[e1 - 1] & 63u) == 63u) atomicExch(bad, 1);
    __syncwarp();
    const size_t row = (size_t)n * words;
    for (int i = 4 * lane; i < words; i += 128) {
      const uint4 rr = *reinterpret_cast<const uint4*>(r + i);
      const uint4 ww = *reinterpret_cast<const uint4*>(w + i);
      __stcs(reinterpret_cast<uint4*>(USE + row + i), rr);
      __stcs(reinterpret_cast<uint4*>(B + row + i), ww);
      __stcs(reinterpret_cast<uint4*>(A + row + i),
             make_uint4(rr.x | ww.x, rr.y | ww.y, rr.z | ww.z, rr.w | ww.w));
    }
    __syncwarp();
  }
}

// The requirement planes of node n as B8 bytes (write == false: only count
// them).  Lane l covers the 128-variable quad l (+32, ...), loaded as one
// 16-byte vector: the previous set variable of a lane's first entry is the
// last set variable of the lanes below it (warp max scan), or of the quads
// before.
__device__ __forceinline__ int b8_node(int64_t n, int words, const uint32_t* __restrict__ REQ,
                                       const uint32_t* __restrict__ FPQ,
                                       const int32_t* __restrict__ fp_slot, int n_fp_slots,
                                       uint8_t* __restrict__ out, int64_t pos, int64_t cap,
                                       bool write, int lane) {
  const int nq = words >> 2;
  int total = 0;
  for (int pass = 0; pass < 2; pass++) {
    int prev = -1;
    const uint32_t kb = (pass ? DFX_B8_FP : DFX_B8_REQ) << 6;
    for (int q0 = 0; q0 < nq; q0 += 32) {
      const int q = q0 + lane;
      uint4 m = make_uint4(0u, 0u, 0u, 0u);
      if (q < nq) {
        if (pass == 0) {
          m = __ldg(reinterpret_cast<const uint4*>(REQ + (size_t)n * words) + q);
        } else {
          const int slot = fp_slot[q];
          if (slot >= 0) m = __ldg(reinterpret_cast<const uint4*>(FPQ) + (size_t)n * n_fp_slots + slot);
        }
      }
      if (!__any_sync(FULL, (m.x | m.y | m.z | m.w) != 0u)) continue;   // no entries here (most FP rows)
      const uint32_t mw[4] = {m.x, m.y, m.z, m.w};
      int last = -1;
#pragma unroll
      for (int k = 0; k < 4; k++)
        if (mw[k]) last = 128 * q + 32 * k + 31 - __clz(mw[k]);
      int before = last;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, before, o);
        if (lane >= o) before = max(before, t);
      }
      int p = __shfl_up_sync(FULL, before, 1);
      if (lane == 0) p = -1;
      p = max(p, prev);
      // bytes of this lane's entries
      int cnt = 0, v0 = p;
#pragma unroll
      for (int k = 0; k < 4; k++)
        for (uint32_t mm = mw[k]; mm; mm &= mm - 1) {
          const int v = 128 * q + 32 * k + __ffs(mm) - 1;
          cnt += 1 + (v - v0 - 1) / 63;
          v0 = v;
        }
      int tot;
      const int at = warp_exclusive_scan(cnt, lane, &tot);
      if (write) {
        int64_t o = pos + total + at;
        v0 = p;
#pragma unroll
        for (int k = 0; k < 4; k++)
          for (uint32_t mm = mw[k]; mm; mm &= mm - 1) {
            const int v = 128 * q + 32 * k + __ffs(mm) - 1;
            int dlt = v - v0 - 1;
            for (; dlt >= 63; dlt -= 63, o++)
              if (o < cap) out[o] = (uint8_t)(kb | 63u);
            if (o < cap) out[o] = (uint8_t)(kb | (uint32_t)dlt);
            o++;
            v0 = v;
          }
      }
      total += tot;
      prev = max(prev, __shfl_sync(FULL, before, 31));
    }
  }
  return total;
}

__global__ void __launch_bounds__(kWarps * 32)
count_b8_kernel(int64_t n_lo, int64_t n_hi, int words, const uint32_t* __restrict__ REQ,
                const uint32_t* __restrict__ FPQ, const int32_t* __restrict__ fp_slot,
                int n_fp_slots, int32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * kWarps;
  for (int64_t n = n_lo + (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); n < n_hi; n += wstride) {
    const int c = b8_node(n, words, REQ, FPQ, fp_slot, n_fp_slots, nullptr, 0, 0, false, lane);
    if (lane == 0) counts[n] = c;
  }
}

__global__ void __launch_bounds__(kWarps * 32)
compact_b8_kernel(int64_t n_lo, int64_t n_hi, int words, const uint32_t* __restrict__ REQ,
                  const uint32_t* __restrict__ FPQ, const int32_t* __restrict__ fp_slot,
                  int n_fp_slots, const int64_t* __restrict__ offsets, uint8_t* __restrict__ out,
                  int64_t cap) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * kWarps;
  for (int64_t n = n_lo + (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5); n < n_hi; n += wstride)
    b8_node(n, words, REQ, FPQ, fp_slot, n_fp_slots, out, offsets[n], cap, true, lane);
}

// Graph validation on the device, before any kernel indexes through the CSR
// (ADVICE r1): row_ptr[0] == 0, non-decreasing, row_ptr[n] == nnz, every
// predecessor id in [0, n).  Sets bit 2 of *bad.
__global__ void __launch_bounds__(256)
check_csr_kernel(const int32_t* __restrict__ row_ptr, int64_t n, const int32_t* __restrict__ col,
                 int64_t nnz, int* bad) {
  int ok = 1;
  const int64_t total = n + 1 + nnz;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i <= n) {
      const int32_t r = __ldg(row_ptr + i);
      if (r < 0 || (int64_t)r > nnz) ok = 0;
      if (i == 0 && r != 0) ok = 0;
      if (i > 0 && r < __ldg(row_ptr + i - 1)) ok = 0;
      if (i == n && (int64_t)r != nnz) ok = 0;
    } else if ((uint64_t)(uint32_t)__ldg(col + (i - n - 1)) >= (uint64_t)n) {
      ok = 0;
    }
  }
  if (!__all_sync(0xFFFFFFFFu, ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 2);
}

int check_csr(const CsrDev& p, int* bad, cudaStream_t st) {
  int64_t blocks = (p.n_nodes + 1 + p.nnz + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  check_csr_kernel<<<(int)(blocks < 1 ? 1 : blocks), 256, 0, st>>>(p.row_ptr, p.n_nodes, p.col,
                                                                   p.nnz, bad);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

static int grid_nodes(int64_t n) {
  int64_t g = (n + kWarps - 1) / kWarps;
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

int expand_acc(const CsrDev& p, const int64_t* off, const uint16_t* acc, int* bad, int64_t n_lo,
               int64_t n_hi, cudaStream_t st) {
  if (n_hi <= n_lo) return DFX_OK;
  const size_t smem = (size_t)kWarps * 2 * p.words * sizeof(uint32_t);
  // the attribute is per device: set it on every call (cheap)
  cudaFuncSetAttribute(expand_acc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  expand_acc_kernel<<<grid_nodes(n_hi - n_lo), kWarps * 32, smem, st>>>(n_lo, n_hi, p.words, off,
                                                                         acc, p.A, p.B, p.USE, bad);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

int expand_b8(const CsrDev& p, const int32_t* off, const uint8_t* bytes, int* bad, int64_t n_lo,
              int64_t n_hi, cudaStream_t st) {
  if (n_hi <= n_lo) return DFX_OK;
  const size_t smem = (size_t)kWarps * 2 * p.words * sizeof(uint32_t);
  cudaFuncSetAttribute(expand_b8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  expand_b8_kernel<<<grid_nodes(n_hi - n_lo), kWarps * 32, smem, st>>>(n_lo, n_hi, p.words, off,
                                                                        bytes, p.A, p.B, p.USE, bad);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

int count_b8(const CsrDev& p, int32_t* counts, int64_t n_lo, int64_t n_hi, cudaStream_t st) {
  if (n_hi <= n_lo) return DFX_OK;
  count_b8_kernel<<<grid_nodes(n_hi - n_lo), kWarps * 32, 0, st>>>(
      n_lo, n_hi, p.words, p.REQ, p.FPQ, p.fp_slot, p.n_fp_slots, counts);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

int compact_b8(const CsrDev& p, const int64_t* offsets, uint8_t* out, int64_t cap, int64_t n_lo,
               int64_t n_hi, cudaStream_t st) {
  if (n_hi <= n_lo) return DFX_OK;
  compact_b8_kernel<<<grid_nodes(n_hi - n_lo), kWarps * 32, 0, st>>>(
      n_lo, n_hi, p.words, p.REQ, p.FPQ, p.fp_slot, p.n_fp_slots, offsets, out, cap);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

int count_acc(const CsrDev& p, int32_t* counts, cudaStream_t st) {
  count_acc_kernel<<<grid_nodes(p.n_nodes), kWarps * 32, 0, st>>>(p.n_nodes, p.words, p.A, counts);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

int export_acc(const CsrDev& p, const int64_t* off, uint16_t* acc, cudaStream_t st) {
  export_acc_kernel<<<grid_nodes(p.n_nodes), kWarps * 32, 0, st>>>(p.n_nodes, p.words, p.USE, p.B,
                                                                   off, acc);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

int compact_list(const CsrDev& p, const int64_t* offsets, uint16_t* vars, int64_t cap,
                 int64_t n_lo, int64_t n_hi, cudaStream_t st) {
  if (n_hi <= n_lo) return DFX_OK;
  compact_list_kernel<<<grid_nodes(n_hi - n_lo), kWarps * 32, 0, st>>>(
      n_lo, n_hi, p.words, p.REQ, p.FPQ, p.fp_slot, p.n_fp_slots, offsets, vars, cap);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

}  // namespace dfx
