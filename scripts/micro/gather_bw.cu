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
