// gather_bw.cu -- practical bandwidth of kernel (a)'s access pattern on one
// B200: per node row (512 B = 32 lanes x 16 B) read the node's own
// transfer row (sequential), AND G random predecessor rows (gathered), and
// write the result row.  Reports GB/s of row traffic for G = 0..4 and a
// plain streaming copy for reference.  Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a gather_bw.cu -o gather_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull; x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull; return x ^ (x >> 31);
}

template <int G>
__global__ void __launch_bounds__(256) rows(const uint4* T, const uint4* S, uint4* O, int n, int chunk) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c * chunk < n; c += warps)
    for (int node = c * chunk; node < min(n, (c + 1) * chunk); node++) {
      uint4 a = __ldg(T + (size_t)node * 32 + lane);
#pragma unroll
      for (int g = 0; g < G; g++) {
        const int q = (int)(mix(node * 8 + g) % (uint64_t)n);
        const uint4 b = __ldcg(S + (size_t)q * 32 + lane);
        a.x &= b.x; a.y &= b.y; a.z &= b.z; a.w &= b.w;
      }
      __stcg(O + (size_t)node * 32 + lane, a);
    }
}

// two nodes per iteration: both nodes' loads in flight together (ILP 2)
template <int G>
__global__ void __launch_bounds__(256) rows2(const uint4* T, const uint4* S, uint4* O, int n, int chunk) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c * chunk < n; c += warps)
    for (int node = c * chunk; node < min(n, (c + 1) * chunk); node += 2) {
      uint4 a = __ldg(T + (size_t)node * 32 + lane), a2 = __ldg(T + (size_t)(node + 1) * 32 + lane);
      uint4 b[G > 0 ? G : 1], b2[G > 0 ? G : 1];
#pragma unroll
      for (int g = 0; g < G; g++) {
        b[g] = __ldcg(S + (mix(node * 8 + g) % (uint64_t)n) * 32 + lane);
        b2[g] = __ldcg(S + (mix((node + 1) * 8 + g) % (uint64_t)n) * 32 + lane);
      }
#pragma unroll
      for (int g = 0; g < G; g++) {
        a.x &= b[g].x; a.y &= b[g].y; a.z &= b[g].z; a.w &= b[g].w;
        a2.x &= b2[g].x; a2.y &= b2[g].y; a2.z &= b2[g].z; a2.w &= b2[g].w;
      }
      __stcg(O + (size_t)node * 32 + lane, a);
      __stcg(O + (size_t)(node + 1) * 32 + lane, a2);
    }
}

// TMA variant (Blackwell bulk copies): per warp a ring of S stages in shared
// memory; lane 0 issues the node's transfer row and G gathered rows as 512-B
// cp.async.bulk copies completing on the stage's mbarrier, S - 1 nodes ahead;
// the lanes wait on the barrier, AND their 16 B of each row, store the row.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile("{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
               "@!p bra WAIT_%=;\n\t}" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}

template <int G, int S, int WPB>
__global__ void __launch_bounds__(WPB * 32) rows_tma(const uint4* T, const uint4* Sg, uint4* O, int n, int chunk) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int R = 1 + G;                          // rows per node
  uint4* ring = reinterpret_cast<uint4*>(smem) + (size_t)w * S * R * 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)WPB * S * R * 512) + w * S;
  if (lane == 0) for (int i = 0; i < S; i++) mbar_init(bars + i, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int warps = (gridDim.x * blockDim.x) >> 5;
  unsigned phase = 0;       // bit i: parity of stage i
  auto issue = [&](int node, int st) {
    if (lane == 0) {
      mbar_expect(bars + st, R * 512);
      uint4* dst = ring + (size_t)st * R * 32;
      bulk_g2s(dst, T + (size_t)node * 32, 512, bars + st);
#pragma unroll
      for (int g = 0; g < G; g++) {
        const int q = (int)(mix(node * 8 + g) % (uint64_t)n);
        bulk_g2s(dst + (g + 1) * 32, Sg + (size_t)q * 32, 512, bars + st);
      }
    }
  };
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c * chunk < n; c += warps) {
    const int n0 = c * chunk, n1 = min(n, (c + 1) * chunk);
    for (int k = 0; k < S - 1 && n0 + k < n1; k++) issue(n0 + k, k);
    for (int node = n0, i = 0; node < n1; node++, i++) {
      const int st = i % S;
      if (node + S - 1 < n1) issue(node + S - 1, (i + S - 1) % S);
      mbar_wait(bars + st, (phase >> st) & 1u);
      phase ^= 1u << st;
      const uint4* src = ring + (size_t)st * R * 32;
      uint4 a = src[lane];
#pragma unroll
      for (int g = 0; g < G; g++) {
        const uint4 b = src[(g + 1) * 32 + lane];
        a.x &= b.x; a.y &= b.y; a.z &= b.z; a.w &= b.w;
      }
      __stcg(O + (size_t)node * 32 + lane, a);
      __syncwarp();            // the stage is reused S nodes later
    }
  }
}

template <int G, int S, int WPB>
void run_tma(const uint4* T, const uint4* Sg, uint4* O, int n, int sms) {
  const size_t smem = (size_t)WPB * S * (1 + G) * 512 + (size_t)WPB * S * 8;
  auto k = rows_tma<G, S, WPB>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, WPB * 32, smem);
  if (occ < 1) { printf("{\"pattern\": \"TMA G=%d S=%d\", \"error\": \"no occupancy\"}\n", G, S); return; }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < 2; it++) k<<<sms * occ, WPB * 32, smem>>>(T, Sg, O, n, 32);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int it = 0; it < reps; it++) k<<<sms * occ, WPB * 32, smem>>>(T, Sg, O, n, 32);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  const cudaError_t err = cudaGetLastError();
  const double bytes = (double)n * 512.0 * (2 + G) * reps;
  printf("{\"pattern\": \"T + %d gathers + write, TMA bulk rows, %d stages per warp\", \"GB_s\": %.1f, "
         "\"rows_per_node\": %d, \"warps_per_sm\": %d, \"err\": \"%s\"}\n",
         G, S, bytes / (ms / 1e3) / 1e9, 2 + G, occ * WPB, cudaGetErrorString(err));
}

__global__ void copyk(const uint4* a, uint4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

template <int G, bool ILP2 = false>
void run(const uint4* T, const uint4* S, uint4* O, int n, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int occ = 0;
  auto k = ILP2 ? rows2<G> : rows<G>;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0);
  for (int it = 0; it < 2; it++) k<<<sms * occ, 256>>>(T, S, O, n, 32);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int it = 0; it < reps; it++) k<<<sms * occ, 256>>>(T, S, O, n, 32);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)n * 512.0 * (2 + G) * reps;
  printf("{\"pattern\": \"T + %d gathers + write%s\", \"GB_s\": %.1f, \"rows_per_node\": %d, \"warps_per_sm\": %d}\n", G,
         ILP2 ? ", 2 nodes in flight per warp" : "", bytes / (ms / 1e3) / 1e9, 2 + G, occ * 8);
}

int main() {
  const int n = 1 << 20;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint4 *T, *S, *O;
  cudaMalloc(&T, (size_t)n * 512); cudaMalloc(&S, (size_t)n * 512); cudaMalloc(&O, (size_t)n * 512);
  cudaMemset(T, 0xFF, (size_t)n * 512); cudaMemset(S, 0xFF, (size_t)n * 512);
  run<0>(T, S, O, n, sms); run<1>(T, S, O, n, sms); run<2>(T, S, O, n, sms);
  run<3>(T, S, O, n, sms); run<4>(T, S, O, n, sms);
  run<1, true>(T, S, O, n, sms); run<2, true>(T, S, O, n, sms); run<3, true>(T, S, O, n, sms);
  run_tma<1, 2, 8>(T, S, O, n, sms); run_tma<1, 4, 8>(T, S, O, n, sms);
  run_tma<2, 2, 8>(T, S, O, n, sms); run_tma<2, 4, 8>(T, S, O, n, sms);
  run_tma<2, 3, 4>(T, S, O, n, sms); run_tma<3, 3, 4>(T, S, O, n, sms);
  run_tma<0, 4, 8>(T, S, O, n, sms);
  // streaming copy of the same 512 MB
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const size_t q = (size_t)n * 32;
  copyk<<<sms * 8, 256>>>(T, O, q);
  cudaEventRecord(e0);
  for (int it = 0; it < 10; it++) copyk<<<sms * 8, 256>>>(T, O, q);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"pattern\": \"stream copy\", \"GB_s\": %.1f}\n", (double)q * 16 * 2 * 10 / (ms / 1e3) / 1e9);
  return 0;
}
