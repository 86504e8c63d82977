// Microbenchmark (profiling aid): the read bandwidth a single kernel reaches on
// this B200 when it streams N MB (argv[1], default 200) from HBM with a cold L2
// (512 MB memset before each run), via LDG.128 grid-stride loops and via
// cp.async.bulk rings through shared memory (per-warp rings of D stages of S
// bytes), no compute. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -std=c++17 -o stream_read_bench tools/stream_read_bench.cu
// argv[2] = 1 (default): after the memset, a 512 MB read of another buffer
// evicts the memset's dirty lines, so the timed kernel reads from a cold AND
// clean L2. r02: 50 MB 3.7 TB/s, 200 MB 6.0 (LDG.128). The r01f figures
// (50 MB 3.2, 200 MB 4.65; argv[2] = 0) had up to 126 MB of dirty L2 lines
// written back inside the timed kernel.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su(b))); }
__device__ __forceinline__ void mexp(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory"); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) { uint32_t d; do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(d) : "r"(su(b)), "r"(ph) : "memory"); } while (!d); }
template <int D>
__global__ void k_tma(const char* src, long total, int S, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nwc = blockDim.x >> 5;
  unsigned char* ring = sm + (size_t)w * D * S;
  uint64_t* bar = (uint64_t*)(sm + (size_t)nwc * D * S) + w * D;
  long gw = (long)blockIdx.x * nwc + w, nw = (long)gridDim.x * nwc;
  long nchunk = total / S, c0 = gw * nchunk / nw, c1 = (gw + 1) * nchunk / nw;
  if (lane == 0) { for (int i = 0; i < D; ++i) minit(&bar[i]); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncwarp();
  if (lane == 0) for (int i = 0; i < D && c0 + i < c1; ++i) { mexp(&bar[i], S); bulk(ring + i * S, src + (c0 + i) * S, S, &bar[i]); }
  double acc = 0;
  for (long c = c0, i = 0; c < c1; ++c, ++i) {
    int st = i % D; mwait(&bar[st], (i / D) & 1);
    acc += ((double*)(ring + st * S))[lane];
    __syncwarp();
    if (lane == 0 && c + D < c1) { asm volatile("fence.proxy.async.shared::cta;"); mexp(&bar[st], S); bulk(ring + st * S, src + (c + D) * S, S, &bar[st]); }
  }
  if (acc == 12345.0) out[0] = acc;
}
__global__ void k_ldg(const double2* src, long n2, double* out) {
  double acc = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n2; i += (long)gridDim.x * blockDim.x) { double2 v = __ldg(src + i); acc += v.x + v.y; }
  if (acc == 12345.0) out[0] = acc;
}
int main(int argc, char** argv) {
  long total = (argc > 1 ? atol(argv[1]) : 200l) << 20; char* src; double* out; cudaMalloc(&src, total); cudaMalloc(&out, 8); cudaMemset(src, 0, total);
  char* flush; cudaMalloc(&flush, 512l << 20);
  char* flush2; cudaMalloc(&flush2, 512l << 20); cudaMemset(flush2, 1, 512l << 20);
  const int clean = argc > 2 ? atoi(argv[2]) : 1;  // 1: evict the memset's dirty lines with a 512 MB read before timing
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto launch, const char* name) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) { cudaMemset(flush, it, 512l << 20); if (clean) k_ldg<<<148 * 8, 256>>>((const double2*)flush2, (512l << 20) / 16, out); cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
    printf("%-40s %7.1f us  %6.2f TB/s  (%s)\n", name, best * 1000, total / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  };
  run([&] { k_ldg<<<148 * 8, 256>>>((const double2*)src, total / 16, out); }, "LDG.128 grid-stride");
  int Ss[] = {4096, 9408, 16384};
  for (int S : Ss) for (int warps : {4, 8, 10}) {
    for (int D : {2, 3, 4}) {
      size_t smem = (size_t)warps * D * S + warps * D * 8;
      if (smem > 227 * 1024) continue;
      int occ = 0;
      auto kern = D == 2 ? k_tma<2> : (D == 3 ? k_tma<3> : k_tma<4>);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, warps * 32, smem);
      char name[128]; snprintf(name, sizeof name, "TMA S=%5d D=%d warps=%d occ=%d inflight/SM=%zuKB", S, D, warps, occ, (size_t)occ * warps * D * S / 1024);
      run([&] { kern<<<148 * occ, warps * 32, smem>>>(src, total, S, out); }, name);
    }
  }
  return 0;
}
