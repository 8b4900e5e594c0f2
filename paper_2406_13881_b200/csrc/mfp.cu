// mfp.cu -- kernels (a) and (b): the CSR data-flow fixpoint and the
// transfer-requirement pass, plus the configuration-C3 generator.
//
// Semantics (oracle/mfp_oracle.c restates them on the CPU):
//   IN[n] = AND_{p in preds(n)} OUT[p]     IN[entry] = (H=1, D=0)
//   host   node: H' = H | A          D' = D & ~B
//   kernel node: H' = H & ~B         D' = D | (A & ~(F & H_in)),  F = A & ~B & S
// (A = R|W, B = W, S = scalar-variable mask; gen/kill effects of
// dartomp/dataflow.py:299-378, AND meet of dataflow.py:130-134.)
// H does not depend on D: the H planes are solved to their greatest fixpoint
// first, then D.
//
// Schedule: frontier-driven chaotic relaxation.  A warp owns one node row at
// a time (V = 4096 variables = 512 B per plane row = one 16-B load per lane,
// fully coalesced); warps pull chunks of consecutive nodes from an atomic
// counter and sweep them in node order, carrying OUT[n-1] in registers (the
// CFG's fall-through edge), so a round propagates information along the whole
// chunk (Gauss-Seidel) instead of one edge (Jacobi).  Other predecessors are
// read from HBM with whatever value they hold; every value read is >= the
// fixpoint, so for this monotone framework the iteration converges to the
// unique greatest fixpoint regardless of order.  A node is re-evaluated in
// round r only if one of its predecessors changed in round r-1 or r
// (per-node change stamps = the frontier); unchanged rows are not rewritten.
// The host stops when a round changes nothing.
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdlib>
#include <cstdio>

#include "../../include/dfx.h"
#include "c3gen.cuh"
#include "dfx_internal.h"

namespace dfx {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int KP = 4;   // predecessor ids preloaded per node (Poisson(1.5)+1: 93% of nodes)

__device__ __forceinline__ uint4 and4(uint4 a, uint4 b) { return make_uint4(a.x & b.x, a.y & b.y, a.z & b.z, a.w & b.w); }
__device__ __forceinline__ uint4 or4(uint4 a, uint4 b) { return make_uint4(a.x | b.x, a.y | b.y, a.z | b.z, a.w | b.w); }
__device__ __forceinline__ uint4 andn4(uint4 a, uint4 b) { return make_uint4(a.x & ~b.x, a.y & ~b.y, a.z & ~b.z, a.w & ~b.w); }
__device__ __forceinline__ bool nz4(uint4 a) { return (a.x | a.y | a.z | a.w) != 0u; }
__device__ __forceinline__ bool ne4(uint4 a, uint4 b) { return ((a.x ^ b.x) | (a.y ^ b.y) | (a.z ^ b.z) | (a.w ^ b.w)) != 0u; }
__device__ __forceinline__ uint4 all4() { return make_uint4(FULL, FULL, FULL, FULL); }
__device__ __forceinline__ uint4 zero4() { return make_uint4(0u, 0u, 0u, 0u); }

__device__ __forceinline__ uint4 ldg4(const uint4* p) { return __ldg(p); }
// rows written by other warps during the same launch: bypass L1 (ld.global.cg)
__device__ __forceinline__ uint4 ldcg4(const uint4* p) { return __ldcg(p); }

// ---------------------------------------------------------------------------
// C3 generator
// ---------------------------------------------------------------------------
__global__ void c3_degree_kernel(uint64_t seed, int64_t n_nodes, int32_t* deg) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes;
       n += (int64_t)gridDim.x * blockDim.x)
    deg[n] = n == 0 ? 0 : 1 + c3_n_extra(seed, n);
}

__global__ void c3_cols_kernel(uint64_t seed, int64_t n_nodes, const int32_t* row_ptr,
                               int32_t* col, uint8_t* kind) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    kind[n] = (uint8_t)c3_is_kernel(seed, n);
    if (n == 0) continue;
    int32_t e = row_ptr[n];
    col[e++] = (int32_t)(n - 1);
    int k = c3_n_extra(seed, n);
    for (int j = 0; j < k; j++) col[e++] = (int32_t)c3_extra_pred(seed, n, j, n_nodes);
  }
}

// one thread per (node, word)
__global__ void c3_planes_kernel(uint64_t seed, int64_t n_nodes, int words, int w0,
                                 uint32_t* A, uint32_t* B, uint32_t* USE) {
  const int64_t total = n_nodes * words;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t n = i / words;
    int w = (int)(i - n * words);
    uint32_t r, wr;
    c3_word(c3_node_key(seed, n), w0 + w, r, wr);
    A[i] = r | wr;
    B[i] = wr;
    USE[i] = r;
  }
}

// A = R | W from uploaded R (= USE) and W (= B) planes
__global__ void or_planes_kernel(const uint4* R, const uint4* W, uint4* A, int64_t nq) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq;
       i += (int64_t)gridDim.x * blockDim.x)
    A[i] = or4(ldg4(R + i), ldg4(W + i));
}

// ---------------------------------------------------------------------------
// kernel (a): one relaxation round of one phase
// ---------------------------------------------------------------------------
struct RoundCounters {
  unsigned long long chunk;      // work queue
  unsigned long long changed;    // rows changed this round
  unsigned long long evaluated;  // rows evaluated this round
  unsigned long long rows_read;  // 16-B*32 row loads (state + planes)
  unsigned long long rows_written;
};

constexpr int kTraceRounds = 64;   // per-round counters kept for traces
constexpr int kMaxSlices = 4;      // V <= 16384: up to four 4096-variable slices

// Device-side control of one phase (one persistent launch).  Rounds use a
// ring of four counter slots (slot round & 3; the slot of round r+1 is
// cleared during round r), so the number of rounds is unbounded.
struct RoundCtl {
  RoundCounters ring[4];
  RoundCounters cnt[kTraceRounds + 1];          // copies of the first rounds (traces)
  unsigned long long t_end[kTraceRounds + 1];   // %globaltimer after each round
  unsigned long long tot_eval, tot_read, tot_written;
  int rounds;                                   // rounds run (incl. the last, unchanged one)
};

// stamp[p] and seen[e] are full round numbers (a node can go unevaluated
// for any number of rounds before a predecessor changes, so no wrapped
// encoding is safe)
__device__ __forceinline__ bool newer(int stamp, int seen) { return stamp > seen; }

// ---------------------------------------------------------------------------
// per-node descriptor (32 B, built once per problem): CSR start, degree,
// kind and the first four predecessor ids -- one 2x16-B load replaces the
// dependent row_ptr -> col chain in the round kernels
// ---------------------------------------------------------------------------
__global__ void build_desc_kernel(int64_t n_nodes, const int32_t* row_ptr, const int32_t* col,
                                  const uint8_t* kind, int4* desc) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    const int rs = row_ptr[n], deg = row_ptr[n + 1] - rs;
    int pr[4];
    for (int k = 0; k < 4; k++) pr[k] = k < deg ? col[rs + k] : 0;
    desc[2 * n] = make_int4(rs, deg | ((int)kind[n] << 30), pr[0], pr[1]);
    desc[2 * n + 1] = make_int4(pr[2], pr[3], 0, 0);
  }
}

// Inclusive prefix sums for the CSR builders and kernel (b)'s compaction
// (out[i] = in[0] + ... + in[i]; in and out may alias).  Reduce-then-scan over
// tiles of 4096 elements (1024 threads x 4): per-tile sums, one block scans
// those (exclusive), each tile rescans itself from its prefix.  Two reads of
// the counts (8 MB at C3) instead of a single decoupled look-back pass: a few
// microseconds beside the kernels it serves.
constexpr int kScanThreads = 1024, kScanItems = 4, kScanTile = kScanThreads * kScanItems;

// block-wide inclusive scan of one value per thread; returns the block total
__device__ __forceinline__ int64_t block_scan(int64_t& v, int64_t* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t t = __shfl_up_sync(FULL, v, d);
    if (lane >= d) v += t;
  }
  if (lane == 31) warp_tot[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t t = __shfl_up_sync(FULL, w, d);
      if (lane >= d) w += t;
    }
    warp_tot[lane] = w;                    // inclusive over warps
  }
  __syncthreads();
  if (warp > 0) v += warp_tot[warp - 1];
  const int64_t total = warp_tot[(blockDim.x >> 5) - 1];
  __syncthreads();                         // warp_tot is reused by the caller's next scan
  return total;
}

template <class TI>
__global__ void __launch_bounds__(kScanThreads) scan_tile_sums_kernel(const TI* in, int64_t n,
                                                                      int64_t* tile_sums) {
  __shared__ int64_t warp_tot[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t v = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; k++)
    if (base + k < n) v += (int64_t)in[base + k];
  const int64_t total = block_scan(v, warp_tot);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// one block: tile_sums[0..n) -> exclusive prefixes, in place
__global__ void __launch_bounds__(kScanThreads) scan_tile_prefix_kernel(int64_t* tile_sums, int64_t n) {
  __shared__ int64_t warp_tot[32];
  int64_t carry = 0;
  for (int64_t b = 0; b < n; b += kScanThreads) {
    const int64_t i = b + threadIdx.x;
    const int64_t x = i < n ? tile_sums[i] : 0;
    int64_t v = x;
    const int64_t total = block_scan(v, warp_tot);
    if (i < n) tile_sums[i] = carry + v - x;
    carry += total;
  }
}

template <class TI, class TO>
__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const TI* in, TO* out, int64_t n,
                                                                  const int64_t* tile_prefix) {
  __shared__ int64_t warp_tot[32];
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int64_t x[kScanItems];
  int64_t v = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    x[k] = base + k < n ? (int64_t)in[base + k] : 0;
    v += x[k];
  }
  block_scan(v, warp_tot);                 // every read of this tile precedes every write
  int64_t run = tile_prefix[blockIdx.x] + v - (x[0] + x[1] + x[2] + x[3]);
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    run += x[k];
    if (base + k < n) out[base + k] = (TO)run;
  }
}

template <class TI, class TO>
static int inclusive_scan(const TI* in, TO* out, int64_t n, void* scratch, size_t scratch_bytes,
                          cudaStream_t st) {
  if (n <= 0) return DFX_OK;
  const int64_t tiles = (n + kScanTile - 1) / kScanTile;
  if ((size_t)tiles * sizeof(int64_t) > scratch_bytes) return DFX_E_NOSPC;
  int64_t* sums = static_cast<int64_t*>(scratch);
  scan_tile_sums_kernel<TI><<<(unsigned)tiles, kScanThreads, 0, st>>>(in, n, sums);
  scan_tile_prefix_kernel<<<1, kScanThreads, 0, st>>>(sums, tiles);
  scan_apply_kernel<TI, TO><<<(unsigned)tiles, kScanThreads, 0, st>>>(in, out, n, sums);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

__global__ void succ_count_kernel(int64_t nnz, const int32_t* col, int32_t* cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + col[e], 1);
}
__global__ void succ_fill_kernel(int64_t n_nodes, const int32_t* row_ptr, const int32_t* col,
                                 int32_t* cursor, int32_t* succ) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n_nodes;
       n += (int64_t)gridDim.x * blockDim.x)
    for (int e = row_ptr[n]; e < row_ptr[n + 1]; e++) succ[atomicAdd(cursor + col[e], 1)] = (int32_t)n;
}

// reverse (successor) CSR: succ_ptr [n+1], succ [nnz]; order inside a row
// is irrelevant (it only feeds the per-chunk candidate flags of kernel (a))
int build_succ(const CsrDev& p, void* scratch, size_t scratch_bytes, int32_t* tmp, cudaStream_t st) {
  int g = (int)((p.nnz + 255) / 256);
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  if (cudaMemsetAsync(p.succ_ptr, 0, sizeof(int32_t) * (p.n_nodes + 1), st) != cudaSuccess) return DFX_E_CUDA;
  if (p.nnz) succ_count_kernel<<<g, 256, 0, st>>>(p.nnz, p.col, p.succ_ptr + 1);
  if (int rc = inclusive_scan(p.succ_ptr + 1, p.succ_ptr + 1, p.n_nodes, scratch, scratch_bytes, st))
    return rc;
  if (cudaMemcpyAsync(tmp, p.succ_ptr, sizeof(int32_t) * p.n_nodes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return DFX_E_CUDA;
  int gn = (int)((p.n_nodes + 255) / 256);
  if (gn > 148 * 64) gn = 148 * 64;
  succ_fill_kernel<<<gn, 256, 0, st>>>(p.n_nodes, p.row_ptr, p.col, tmp, p.succ);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

int build_desc(const CsrDev& p, cudaStream_t st) {
  int g = (int)((p.n_nodes + 255) / 256);
  if (g > 148 * 64) g = 148 * 64;
  build_desc_kernel<<<g, 256, 0, st>>>(p.n_nodes, p.row_ptr, p.col, p.kind,
                                       reinterpret_cast<int4*>(p.desc));
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

// ---------------------------------------------------------------------------
// kernel (a), V <= 4096 fast path.  Node descriptors are prefetched one
// 32-node batch ahead.  The frontier is per edge ("seen" rounds):
//   stamp[p]      last round in which p's row changed
//   chunk_done[c] last round in which chunk c was completely swept; a chunk's
//                 rows are final for that round once its flag is set
//   seen[e]       for edge e = (p -> n): n has incorporated every change of
//                 p up to the end of round seen[e] -- r if p's chunk was done
//                 in round r when n's batch checked it (or p is n's
//                 fall-through predecessor taken from registers), else r-1
// n is re-evaluated in round r+1 iff some edge has stamp[p] > seen[e] (plus
// the Gauss-Seidel rule: a node whose fall-through predecessor changed
// earlier in the same sweep is re-evaluated at once).  Round 1 reads every
// predecessor whose chunk is already done and treats the others as top.
// Values only decrease from top, so any value read is >= the fixpoint; a
// round without changes leaves no edge with stamp > seen, so the phase ends
// at the greatest fixpoint.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
// cumulative release: the warp's row stores (ordered before this by the
// preceding __syncwarp) become visible before the flag
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// LDGSTS (cp.async, 16 B per lane) helpers
__device__ __forceinline__ void cp16(uint4* sdst, const uint4* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

template <int PHASE, int MINB>
__global__ void __launch_bounds__(256, MINB)
mfp_phase_kernel(CsrDev p, int q0, int chunk_nodes, int n_chunks, RoundCtl* ctl, uint8_t* flags,
                 int max_rounds) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  // per-warp metadata of the current 32-node batch in shared memory (read
  // by the node loop as broadcasts, so it holds no registers), and the next
  // batch's descriptors landing by cp.async
  struct BatchMeta { int4 d[2][32][2]; int opc[32]; unsigned dn[32]; };
  __shared__ BatchMeta bm_all[256 / 32];
  const int lane = threadIdx.x & 31;
  BatchMeta& bm = bm_all[threadIdx.x >> 5];
  // this launch solves the 4096-variable slice of quads [q0, q0 + 32)
  const int nq = p.words >> 2;          // row stride in quads
  const int ql = q0 + lane;
  const bool act = ql < nq;
  const uint4* A = reinterpret_cast<const uint4*>(p.A);
  const uint4* B = reinterpret_cast<const uint4*>(p.B);
  const uint4* OH = reinterpret_cast<const uint4*>(p.OH);
  uint4* OUT = reinterpret_cast<uint4*>(PHASE == 0 ? p.OH : p.OD);
  const int4* desc = reinterpret_cast<const int4*>(p.desc);
  const uint4 smask = act ? ldg4(reinterpret_cast<const uint4*>(p.S) + ql) : zero4();
  const bool has_s = nz4(smask);
  const uint4 boundary = PHASE == 0 ? all4() : zero4();
  for (int round = 1; round <= max_rounds; round++) {
  const int first = round == 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) {   // slot of round + 1 (last used in round - 3)
    RoundCounters& z = ctl->ring[(round + 1) & 3];
    z.chunk = z.changed = z.evaluated = z.rows_read = z.rows_written = 0ull;
  }
  RoundCounters* cnt = &ctl->ring[round & 3];
  uint8_t* fcur = flags + (size_t)(round & 1) * n_chunks;
  uint8_t* fnext = flags + (size_t)((round + 1) & 1) * n_chunks;
  unsigned n_changed = 0, n_eval = 0, n_read = 0, n_written = 0;   // per warp
  // sparse rounds (late, few changes): static chunk striding, and only chunks
  // a predecessor change flagged during the previous round are swept
  // mark(r): round r flags successor chunks for round r+1, decided on round
  // r-1's change count (final: the previous launch has completed)
  auto marks = [&](int r) {
    return r >= 2 && 8 * __ldcg(&ctl->ring[(r - 1) & 3].changed) <= 3ull * (unsigned long long)p.n_nodes;
  };
  const bool mark = marks(round);
  const bool sparse = round >= 3 && marks(round - 1);
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  int chunk = sparse ? gwarp - nwarps : 0;

  for (;;) {
    if (sparse) {
      chunk += nwarps;
    } else {
      if (lane == 0) chunk = (int)atomicAdd(&cnt->chunk, 1ull);
      chunk = __shfl_sync(FULL, chunk, 0);
    }
    if (chunk >= n_chunks) break;
    // an unflagged chunk's rows are final for this round
    if (sparse) {
      int f = 0;
      if (lane == 0) {
        f = __ldcg(fcur + chunk);
        if (f) fcur[chunk] = 0;               // reused as fnext next round
        else st_relaxed(p.chunk_done + chunk, round);
      }
      if (!__shfl_sync(FULL, f, 0)) continue;
    }
    const int n0 = chunk * chunk_nodes;
    const int n1 = min(n0 + chunk_nodes, (int)p.n_nodes);
    uint4 prev = zero4();
    int prev_n = -2;
    bool carry = false;
    // descriptors of the first batch
    int buf = 0;
    if (n0 + lane < n1) {
      cp16(reinterpret_cast<uint4*>(&bm.d[0][lane][0]), reinterpret_cast<const uint4*>(desc + 2 * (n0 + lane)));
      cp16(reinterpret_cast<uint4*>(&bm.d[0][lane][1]), reinterpret_cast<const uint4*>(desc + 2 * (n0 + lane) + 1));
    }
    cp_commit();
    for (int nb = n0; nb < n1; nb += 32, buf ^= 1) {
      const int n = nb + lane;
      const bool valid = n < n1;
      // next batch's descriptors in flight while this batch is processed
      const int nn1 = nb + 32 + lane;
      if (nn1 < n1) {
        cp16(reinterpret_cast<uint4*>(&bm.d[buf ^ 1][lane][0]), reinterpret_cast<const uint4*>(desc + 2 * nn1));
        cp16(reinterpret_cast<uint4*>(&bm.d[buf ^ 1][lane][1]), reinterpret_cast<const uint4*>(desc + 2 * nn1 + 1));
      }
      cp_commit();
      cp_wait<1>();
      __syncwarp();              // every lane's descriptor copies are visible warp-wide
      const int4 d0 = bm.d[buf][lane][0], d1 = bm.d[buf][lane][1];
      const int rs = d0.x, deg = d0.y & 0x3FFFFFFF, kd = (d0.y >> 30) & 1;
      const int pr0 = d0.z, pr1 = d0.w, pr2 = d1.x, pr3 = d1.y;
      const int cur_opc = first ? 32 * p.words : (valid ? __ldcg(p.popc + n) : 0);
      // dn bit k: pred k's chunk is done for this round (its row is final);
      // the acquire orders the warp's later row loads after the release
      unsigned dn = 0;
      bool dirty = first != 0;
      if (valid) {
        if (!first) {
          const int4 s4 = __ldcg(reinterpret_cast<const int4*>(p.seen4) + n);
          const int sk[KP] = {s4.x, s4.y, s4.z, s4.w};
#define DFX_DIRTY(K, Q) \
  if (deg > K) dirty |= newer(__ldcg(p.stamp + (Q)), sk[K]);
          DFX_DIRTY(0, pr0) DFX_DIRTY(1, pr1) DFX_DIRTY(2, pr2) DFX_DIRTY(3, pr3)
#undef DFX_DIRTY
          for (int e = rs + KP; e < rs + deg && !dirty; e++)
            dirty = newer(__ldcg(p.stamp + __ldg(p.col + e)), __ldcg(p.seen + e));
        }
        if (dirty) {
#define DFX_DONE(K, Q)                                                                   \
  if (deg > K) {                                                                         \
    const int c_ = (Q) / chunk_nodes;                                                    \
    if (c_ != chunk && ld_acquire(p.chunk_done + c_) == round) dn |= 1u << K;           \
  }
          DFX_DONE(0, pr0) DFX_DONE(1, pr1) DFX_DONE(2, pr2) DFX_DONE(3, pr3)
#undef DFX_DONE
        }
      }
      bm.opc[lane] = cur_opc;
      bm.dn[lane] = dn;
      __syncwarp();
      unsigned dm = __ballot_sync(FULL, valid && dirty);
      if (carry && nb < n1) dm |= 1u;
      carry = false;
      const unsigned vmask = __ballot_sync(FULL, valid);
      while (dm) {
        const int j = __ffs(dm) - 1;
        dm &= dm - 1;
        const int nn = nb + j;
        const int4 e0 = bm.d[buf][j][0], e1 = bm.d[buf][j][1];     // broadcasts
        const int nrs = e0.x;
        const int ndeg = e0.y & 0x3FFFFFFF;
        const bool kern = (e0.y >> 30) & 1;
        const int old_pc = bm.opc[j];
        const unsigned ndn = bm.dn[j];
        const int q0 = e0.z, q1 = e0.w, q2 = e1.x, q3 = e1.y;
        const size_t row = (size_t)nn * nq;
        const bool have_prev = prev_n == nn - 1;
        const uint4* plane = (PHASE == 0) == kern ? B : A;
        uint4 pl = zero4(), b0 = zero4(), oh = zero4();
        uint4 in = ndeg == 0 ? boundary : all4();
        if (act) {
          pl = ldg4(plane + row + ql);
          // D phase, kernel node: F & H_in = F & OUT_H[n] (F = A & ~B & S is
          // disjoint from B and OUT_H = H_in & ~B), only scalar lanes
          if (PHASE == 1 && kern && has_s) { b0 = ldg4(B + row + ql); oh = ldcg4(OH + row + ql); }
        }
        // gathers, all issued before use; per edge the round whose final
        // value this evaluation incorporates
        int sv[KP] = {0, 0, 0, 0};
        uint4 g0 = all4(), g1 = all4(), g2 = all4(), g3 = all4();
#define DFX_GATHER(K, Q, G)                                                              \
  if (ndeg > K) {                                                                        \
    if ((Q) == nn - 1 && have_prev) {                                                    \
      G = prev;                                                                          \
      sv[K] = round;                                                                     \
    } else {                                                                             \
      const bool fin_ = (ndn >> K) & 1u;                                                 \
      sv[K] = fin_ ? round : round - 1;                                                  \
      if (!first || fin_) {                                                              \
        if (act) G = ldcg4(OUT + (size_t)(Q) * nq + ql);                               \
        n_read++;                                                                        \
      }                                                                                  \
    }                                                                                    \
  }
        DFX_GATHER(0, q0, g0) DFX_GATHER(1, q1, g1) DFX_GATHER(2, q2, g2) DFX_GATHER(3, q3, g3)
#undef DFX_GATHER
        in = and4(and4(in, and4(g0, g1)), and4(g2, g3));
        if (ndeg > KP) {                                   // rare: more than KP preds
          for (int e = nrs + KP; e < nrs + ndeg; e++) {
            const int qk = __ldg(p.col + e);
            int sr = round;
            if (qk == nn - 1 && have_prev) {
              in = and4(in, prev);
            } else {
              const int c = qk / chunk_nodes;
              const bool fin = c != chunk && ld_acquire(p.chunk_done + c) == round;
              sr = fin ? round : round - 1;
              if (!first || fin) {
                if (act) in = and4(in, ldcg4(OUT + (size_t)qk * nq + ql));
                n_read++;
              }
            }
            if (lane == 0) p.seen[e] = sr;
          }
        }
        uint4 out;
        if (PHASE == 0) {
          out = kern ? andn4(in, pl) : or4(in, pl);
        } else if (kern) {
          out = or4(in, andn4(pl, and4(and4(andn4(pl, b0), smask), oh)));
        } else {
          out = andn4(in, pl);
        }
        const int pc = (int)__reduce_add_sync(
            FULL, act ? (unsigned)(__popc(out.x) + __popc(out.y) + __popc(out.z) + __popc(out.w)) : 0u);
        const bool ch = pc != old_pc;
        n_eval++;
        n_read++;
        if (ch || first) {
          if (act) __stcg(OUT + row + ql, out);
          n_written++;
        }
        if (lane == 0) {
          reinterpret_cast<int4*>(p.seen4)[nn] = make_int4(sv[0], sv[1], sv[2], sv[3]);
          if (ch || first) p.popc[nn] = pc;
          if (ch) p.stamp[nn] = round;
          else if (first) p.stamp[nn] = 0;
        }
        n_changed += ch;
        prev = out;
        prev_n = nn;
        if (ch && !first) {
          if (j < 31) dm |= (1u << (j + 1)) & vmask;
          else carry = true;
          if (mark) {   // flag the successors' chunks for the next round
            const int s0 = __ldg(p.succ_ptr + nn), s1 = __ldg(p.succ_ptr + nn + 1);
            for (int e = s0 + lane; e < s1; e += 32) fnext[__ldg(p.succ + e) / chunk_nodes] = 1;
          }
        }
      }
    }
    // release the chunk: its rows are final for this round
    __syncwarp();
    if (lane == 0) st_release(p.chunk_done + chunk, round);
  }
  if (lane == 0) {
    if (n_changed) atomicAdd(&cnt->changed, (unsigned long long)n_changed);
    if (n_eval) atomicAdd(&cnt->evaluated, (unsigned long long)n_eval);
    if (n_read) atomicAdd(&cnt->rows_read, (unsigned long long)n_read);
    if (n_written) atomicAdd(&cnt->rows_written, (unsigned long long)n_written);
  }
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    ctl->tot_eval += cnt->evaluated;
    ctl->tot_read += cnt->rows_read;
    ctl->tot_written += cnt->rows_written;
    if (round <= kTraceRounds) { ctl->cnt[round] = *cnt; ctl->t_end[round] = t; }
    ctl->rounds = round;
  }
  // every thread reads the same final count: a uniform exit
  if (round > 1 && __ldcg(&cnt->changed) == 0) break;
  }   // rounds
}

// ---------------------------------------------------------------------------
// kernel (b): requirement planes + per-node nonzero-word counts
// ---------------------------------------------------------------------------
// Bytes of one ascending list in the B8 coding (include/dfx.h) whose bits are
// spread as quads: lane l holds quads l, l + 32, ... (uniform across the warp)
template <int VPL>
__device__ __forceinline__ int b8_bytes(const uint4 (&m)[VPL], int lane) {
  int total = 0, prev = -1;
#pragma unroll
  for (int v = 0; v < VPL; v++) {
    const int q = lane + 32 * v;
    if (!__any_sync(FULL, (m[v].x | m[v].y | m[v].z | m[v].w) != 0u)) continue;   // no entries here
    const uint32_t mw[4] = {m[v].x, m[v].y, m[v].z, m[v].w};
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
    int v0 = max(p, prev), cnt = 0;
#pragma unroll
    for (int k = 0; k < 4; k++)
      for (uint32_t mm = mw[k]; mm; mm &= mm - 1) {
        const int var = 128 * q + 32 * k + __ffs(mm) - 1;
        cnt += 1 + (var - v0 - 1) / 63;
        v0 = var;
      }
    total += (int)__reduce_add_sync(FULL, (unsigned)cnt);
    prev = max(prev, __shfl_sync(FULL, before, 31));
  }
  return total;
}
template <int VPL>
__global__ void __launch_bounds__(256)
requirements_kernel(CsrDev p, int32_t* counts, int count_bits, int n_lo, int n_hi) {
  const int lane = threadIdx.x & 31;
  const int nq = p.words >> 2;
  const uint4* A = reinterpret_cast<const uint4*>(p.A);
  const uint4* B = reinterpret_cast<const uint4*>(p.B);
  const uint4* U = reinterpret_cast<const uint4*>(p.USE);
  const uint4* OH = reinterpret_cast<const uint4*>(p.OH);
  const uint4* OD = reinterpret_cast<const uint4*>(p.OD);
  uint4* REQ = reinterpret_cast<uint4*>(p.REQ);
  uint4* FPQ = reinterpret_cast<uint4*>(p.FPQ);
  const uint4* S4 = reinterpret_cast<const uint4*>(p.S);
  uint4 smask[VPL];
  bool active[VPL];
#pragma unroll
  for (int v = 0; v < VPL; v++) {
    int q = lane + 32 * v;
    active[v] = q < nq;
    smask[v] = active[v] ? ldg4(S4 + q) : zero4();
  }
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int n = n_lo + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); n < n_hi; n += warps) {
    const int rs = __ldg(p.row_ptr + n), re = __ldg(p.row_ptr + n + 1);
    const bool kern = __ldg(p.kind + n) != 0;
    const size_t row = (size_t)n * nq;
    uint4 ih[VPL], id[VPL];
#pragma unroll
    for (int v = 0; v < VPL; v++) { ih[v] = all4(); id[v] = re == rs ? zero4() : all4(); }
    // host nodes read only IN_H; kernel nodes read IN_D, and IN_H only on
    // the scalar quads (the firstprivate term F is zero elsewhere)
    for (int e = rs; e < re; e++) {
      const int q = __ldg(p.col + e);
#pragma unroll
      for (int v = 0; v < VPL; v++)
        if (active[v]) {
          if (!kern || nz4(smask[v])) ih[v] = and4(ih[v], ldg4(OH + (size_t)q * nq + lane + 32 * v));
          if (kern) id[v] = and4(id[v], ldg4(OD + (size_t)q * nq + lane + 32 * v));
        }
    }
    int cnt = 0;
    uint4 rq[VPL], fq[VPL];
#pragma unroll
    for (int v = 0; v < VPL; v++) {
      rq[v] = fq[v] = zero4();
      if (!active[v]) continue;
      const int q = lane + 32 * v;
      const uint4 use = ldg4(U + row + q);
      uint4 req, fp = zero4();
      if (!kern) {
        req = andn4(use, ih[v]);
      } else {
        uint4 f = zero4();
        if (nz4(smask[v])) f = and4(andn4(ldg4(A + row + q), ldg4(B + row + q)), smask[v]);
        req = or4(andn4(andn4(use, f), id[v]), andn4(andn4(f, id[v]), ih[v]));
        fp = and4(andn4(f, id[v]), ih[v]);
      }
      rq[v] = req;
      __stcs(REQ + row + q, req);
      cnt += count_bits ? __popc(req.x) + __popc(req.y) + __popc(req.z) + __popc(req.w)
                        : (req.x != 0) + (req.y != 0) + (req.z != 0) + (req.w != 0);
      if (p.fp_slot[q] >= 0) {
        fq[v] = fp;
        FPQ[(size_t)n * p.n_fp_slots + p.fp_slot[q]] = fp;
        cnt += count_bits ? __popc(fp.x) + __popc(fp.y) + __popc(fp.z) + __popc(fp.w)
                          : (fp.x != 0) + (fp.y != 0) + (fp.z != 0) + (fp.w != 0);
      }
    }
    if (count_bits == 2) {      // byte-coded lists: the node's bytes (requirements, then captures)
      cnt = b8_bytes<VPL>(rq, lane) + b8_bytes<VPL>(fq, lane);
    } else {
#pragma unroll
      for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
    }
    if (lane == 0) counts[n] = cnt;
  }
}

// order-preserving compaction into sparse word-rows: per node two occupancy
// bitmaps (requirement words, firstprivate words) and the nonzero masks in
// order (requirement words ascending, then firstprivate words ascending)
template <int VPL>
__global__ void __launch_bounds__(256)
compact_kernel(CsrDev p, const int64_t* offsets, uint32_t* occ, uint32_t* masks, int64_t cap) {
  const int lane = threadIdx.x & 31;
  const int nq = p.words >> 2;
  const int ow = (p.words + 31) >> 5;          // occupancy words per kind
  const uint4* REQ = reinterpret_cast<const uint4*>(p.REQ);
  const uint4* FPQ = reinterpret_cast<const uint4*>(p.FPQ);
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int n = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; n < p.n_nodes; n += warps) {
    int64_t base = offsets[n];
    const size_t row = (size_t)n * nq;
    for (int pass = 0; pass < 2; pass++) {
#pragma unroll
      for (int v = 0; v < VPL; v++) {
        const int q = lane + 32 * v;
        uint4 m = zero4();
        if (q < nq) {
          if (pass == 0) m = ldg4(REQ + row + q);
          else if (p.fp_slot[q] >= 0) m = ldg4(FPQ + (size_t)n * p.n_fp_slots + p.fp_slot[q]);
        }
        const uint32_t w4[4] = {m.x, m.y, m.z, m.w};
        const uint32_t nib = (w4[0] != 0) | ((w4[1] != 0) << 1) | ((w4[2] != 0) << 2) | ((w4[3] != 0) << 3);
        // occupancy word (q / 8) gathers the nibbles of 8 consecutive lanes
        uint32_t ov = nib << (4 * (q & 7));
        ov |= __shfl_xor_sync(FULL, ov, 1);
        ov |= __shfl_xor_sync(FULL, ov, 2);
        ov |= __shfl_xor_sync(FULL, ov, 4);
        if ((q & 7) == 0 && (q >> 3) < ow) occ[(size_t)n * 2 * ow + pass * ow + (q >> 3)] = ov;
        const int c = __popc(nib);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int t = __shfl_up_sync(FULL, incl, o);
          if (lane >= o) incl += t;
        }
        int64_t pos = base + incl - c;
#pragma unroll
        for (int k = 0; k < 4; k++)
          if (w4[k]) {
            if (pos < cap) masks[pos] = w4[k];
            pos++;
          }
        base += __shfl_sync(FULL, incl, 31);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host-side drivers
// ---------------------------------------------------------------------------
static int grid_for(int64_t work, int block) {
  int64_t g = (work + block - 1) / block;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return (int)g;
}

int c3_generate(CsrDev& p, uint64_t seed, int w0, cudaStream_t st, void* scratch,
                size_t scratch_bytes) {
  int32_t* deg = p.row_ptr + 1;  // degrees land in row_ptr[1..n], scanned in place
  c3_degree_kernel<<<grid_for(p.n_nodes, 256), 256, 0, st>>>(seed, p.n_nodes, deg);
  if (cudaMemsetAsync(p.row_ptr, 0, sizeof(int32_t), st) != cudaSuccess) return DFX_E_CUDA;
  if (int rc = inclusive_scan(deg, deg, p.n_nodes, scratch, scratch_bytes, st)) return rc;
  c3_cols_kernel<<<grid_for(p.n_nodes, 256), 256, 0, st>>>(seed, p.n_nodes, p.row_ptr, p.col,
                                                           p.kind);
  c3_planes_kernel<<<grid_for(p.n_nodes * p.words, 256), 256, 0, st>>>(
      seed, p.n_nodes, p.words, w0, p.A, p.B, p.USE);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

int or_planes(const CsrDev& p, cudaStream_t st) {
  int64_t nq = p.n_nodes * (p.words / 4);
  or_planes_kernel<<<grid_for(nq, 256), 256, 0, st>>>(
      reinterpret_cast<const uint4*>(p.USE), reinterpret_cast<const uint4*>(p.B),
      reinterpret_cast<uint4*>(p.A), nq);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

// kernel (a): one persistent cooperative launch per (slice, phase) runs
// every round (grid-wide barrier between rounds, uniform exit on a round
// without changes) -- no host round trips and no launch gaps.  V > 4096 is
// solved as independent 4096-variable slices (variables are independent).
template <int PHASE>
static int launch_phase(const CsrDev& p, int q0, int chunk_nodes, int n_chunks, RoundCtl* ctl,
                        uint8_t* flags, cudaStream_t st) {
  // occupancy per device (a thread may drive handles on several devices)
  constexpr int kDevs = 64;
  static int sms[kDevs] = {}, per_sm[kDevs] = {};
  auto* fn = mfp_phase_kernel<PHASE, 4>;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kDevs) return DFX_E_CUDA;
  if (!sms[dev]) {
    cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], fn, 256, 0);
    if (per_sm[dev] < 1) per_sm[dev] = 1;
  }
  CsrDev pp = p;
  int max_rounds = 1 << 30;
  void* args[] = {&pp, &q0, &chunk_nodes, &n_chunks, &ctl, &flags, &max_rounds};
  if (cudaLaunchCooperativeKernel((const void*)fn, dim3(sms[dev] * per_sm[dev]), dim3(256), args, 0,
                                  st) != cudaSuccess)
    return DFX_E_CUDA;
  return DFX_OK;
}

int vpl_for(int words) {
  int nq = words / 4;
  if (words % 4) return -1;
  if (nq <= 32) return 1;
  if (nq <= 64) return 2;
  if (nq <= 128) return 4;
  return -1;
}

size_t round_ctl_bytes() { return 2 * kMaxSlices * sizeof(RoundCtl); }

int mfp_solve(const CsrDev& p, void* ctl_mem, uint8_t* flags, cudaStream_t st, int chunk_nodes,
              SolveStats* stats, bool collect) {
  const int vpl = vpl_for(p.words);
  if (vpl < 0) return DFX_E_LIMIT;
  const int n_slices = vpl;                 // 32 quads (4096 variables) per slice
  const int n_chunks = (int)((p.n_nodes + chunk_nodes - 1) / chunk_nodes);
  RoundCtl* ctls = reinterpret_cast<RoundCtl*>(ctl_mem);   // [slice][phase]
  // timing events per (thread, device): an event may only be recorded on a
  // stream of the device it was created on
  constexpr int kDevs = 64;
  static thread_local cudaEvent_t ev_dev[kDevs][2 * 2 * kMaxSlices] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kDevs) return DFX_E_CUDA;
  cudaEvent_t* ev = ev_dev[dev];
  if (!ev[0])
    for (int i = 0; i < 2 * 2 * kMaxSlices; i++)
      if (cudaEventCreate(&ev[i]) != cudaSuccess) return DFX_E_CUDA;
  static int trace = -1;
  if (trace < 0) trace = getenv("DFX_TRACE") ? 1 : 0;
  if (cudaMemsetAsync(ctls, 0, sizeof(RoundCtl) * 2 * n_slices, st) != cudaSuccess) return DFX_E_CUDA;
  for (int sl = 0; sl < n_slices; sl++)
    for (int phase = 0; phase < 2; phase++) {
      if (cudaMemsetAsync(flags, 0, 2 * (size_t)n_chunks, st) != cudaSuccess) return DFX_E_CUDA;
      if (cudaMemsetAsync(p.chunk_done, 0, sizeof(int) * (size_t)n_chunks, st) != cudaSuccess) return DFX_E_CUDA;
      const int k = 2 * sl + phase;
      if (cudaEventRecord(ev[2 * k], st) != cudaSuccess) return DFX_E_CUDA;
      int rc = phase == 0 ? launch_phase<0>(p, 32 * sl, chunk_nodes, n_chunks, ctls + k, flags, st)
                          : launch_phase<1>(p, 32 * sl, chunk_nodes, n_chunks, ctls + k, flags, st);
      if (rc != DFX_OK) return rc;
      if (cudaEventRecord(ev[2 * k + 1], st) != cudaSuccess) return DFX_E_CUDA;
    }
  if (!collect) return DFX_OK;        // enqueued only: no host synchronisation
  static thread_local RoundCtl h[2 * kMaxSlices];
  if (cudaMemcpyAsync(h, ctls, sizeof(RoundCtl) * 2 * n_slices, cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return DFX_E_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return DFX_E_CUDA;
  stats->rounds[0] = stats->rounds[1] = 0;
  stats->evaluated = stats->rows_read = stats->rows_written = 0;
  stats->kernel_ms = 0.f;
  for (int k = 0; k < 2 * n_slices; k++) {
    float kms = 0.f;
    cudaEventElapsedTime(&kms, ev[2 * k], ev[2 * k + 1]);
    stats->kernel_ms += kms;
    const RoundCtl& c = h[k];
    const int phase = k & 1;
    if (c.rounds > stats->rounds[phase]) stats->rounds[phase] = c.rounds;
    stats->evaluated += (int64_t)c.tot_eval;
    stats->rows_read += (int64_t)c.tot_read;
    stats->rows_written += (int64_t)c.tot_written;
    if (trace)
      for (int r = 1; r <= c.rounds && r <= kTraceRounds; r++)
        fprintf(stderr, "dfx-trace slice %d phase %d round %d evaluated %llu changed %llu rows_read %llu "
                "rows_written %llu round_us %.1f\n", k >> 1, phase, r, c.cnt[r].evaluated,
                c.cnt[r].changed, c.cnt[r].rows_read, c.cnt[r].rows_written,
                r > 1 ? (c.t_end[r] - c.t_end[r - 1]) / 1e3 : 0.0);
  }
  return DFX_OK;
}

int requirements_scan(const CsrDev& p, int32_t* counts, int64_t* offsets, void* scratch,
                      size_t scratch_bytes, int count_bits, int64_t* n_out, cudaStream_t st) {
  const int vpl = vpl_for(p.words);
  int blocks = grid_for(p.n_nodes * 32, 256);
  switch (vpl) {
    case 1: requirements_kernel<1><<<blocks, 256, 0, st>>>(p, counts, count_bits, 0, (int)p.n_nodes); break;
    case 2: requirements_kernel<2><<<blocks, 256, 0, st>>>(p, counts, count_bits, 0, (int)p.n_nodes); break;
    case 4: requirements_kernel<4><<<blocks, 256, 0, st>>>(p, counts, count_bits, 0, (int)p.n_nodes); break;
    default: return DFX_E_LIMIT;
  }
  return scan_counts(p.n_nodes, counts, offsets, scratch, scratch_bytes, n_out, st);
}

// kernel (b) bit counts + scan over the node range [n_lo, n_hi): on return
// (stream order) offsets[n_lo+1 .. n_hi] are global offsets, continuing from
// offsets[n_lo] (set by the previous range; offsets[0] = 0 by the caller)
__global__ void add_base_kernel(int64_t* out, int64_t len, const int64_t* base) {
  const int64_t b = *base;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] += b;
}

int requirements_range(const CsrDev& p, int32_t* counts, int64_t* offsets, void* scratch,
                       size_t scratch_bytes, int n_lo, int n_hi, cudaStream_t st, bool b8) {
  const int vpl = vpl_for(p.words);
  const int n = n_hi - n_lo;
  if (n <= 0) return DFX_OK;
  int blocks = grid_for((int64_t)n * 32, 256);
  switch (vpl) {
    // byte-coded lists (b8): the counts are bytes, not entries
    case 1: requirements_kernel<1><<<blocks, 256, 0, st>>>(p, counts, b8 ? 2 : 1, n_lo, n_hi); break;
    case 2: requirements_kernel<2><<<blocks, 256, 0, st>>>(p, counts, b8 ? 2 : 1, n_lo, n_hi); break;
    case 4: requirements_kernel<4><<<blocks, 256, 0, st>>>(p, counts, b8 ? 2 : 1, n_lo, n_hi); break;
    default: return DFX_E_LIMIT;
  }
  if (int rc = inclusive_scan(counts + n_lo, offsets + n_lo + 1, (int64_t)n, scratch, scratch_bytes, st))
    return rc;
  add_base_kernel<<<grid_for(n, 256), 256, 0, st>>>(offsets + n_lo + 1, n, offsets + n_lo);
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

int scan_counts(int64_t n, const int32_t* counts, int64_t* offsets, void* scratch,
                size_t scratch_bytes, int64_t* n_out, cudaStream_t st) {
  if (cudaMemsetAsync(offsets, 0, sizeof(int64_t), st) != cudaSuccess) return DFX_E_CUDA;
  if (int rc = inclusive_scan(counts, offsets + 1, n, scratch, scratch_bytes, st)) return rc;
  if (n_out && cudaMemcpyAsync(n_out, offsets + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st) !=
                   cudaSuccess)
    return DFX_E_CUDA;
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

int requirements(const CsrDev& p, int32_t* counts, int64_t* offsets, void* scratch,
                 size_t scratch_bytes, uint32_t* occ, uint32_t* masks, int64_t cap,
                 int64_t* n_out, cudaStream_t st) {
  const int vpl = vpl_for(p.words);
  int blocks = grid_for(p.n_nodes * 32, 256);
  switch (vpl) {
    case 1: requirements_kernel<1><<<blocks, 256, 0, st>>>(p, counts, 0, 0, (int)p.n_nodes); break;
    case 2: requirements_kernel<2><<<blocks, 256, 0, st>>>(p, counts, 0, 0, (int)p.n_nodes); break;
    case 4: requirements_kernel<4><<<blocks, 256, 0, st>>>(p, counts, 0, 0, (int)p.n_nodes); break;
    default: return DFX_E_LIMIT;
  }
  // offsets[0] = 0; offsets[1..n] = inclusive prefix of counts
  if (cudaMemsetAsync(offsets, 0, sizeof(int64_t), st) != cudaSuccess) return DFX_E_CUDA;
  if (int rc = inclusive_scan(counts, offsets + 1, p.n_nodes, scratch, scratch_bytes, st)) return rc;
  if (cudaMemcpyAsync(n_out, offsets + p.n_nodes, sizeof(int64_t), cudaMemcpyDeviceToHost, st) !=
      cudaSuccess)
    return DFX_E_CUDA;
  if (masks) {
    switch (vpl) {
      case 1: compact_kernel<1><<<blocks, 256, 0, st>>>(p, offsets, occ, masks, cap); break;
      case 2: compact_kernel<2><<<blocks, 256, 0, st>>>(p, offsets, occ, masks, cap); break;
      case 4: compact_kernel<4><<<blocks, 256, 0, st>>>(p, offsets, occ, masks, cap); break;
    }
  }
  return cudaGetLastError() == cudaSuccess ? DFX_OK : DFX_E_CUDA;
}

size_t scan_scratch_bytes(int64_t n) {
  return (size_t)((n + kScanTile - 1) / kScanTile) * sizeof(int64_t) + 256;
}

}  // namespace dfx


