// Shared device helpers for the adipc B200 path (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace adipc_gpu {

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define ADIPC_CUDA(expr)                                                                  \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess)                                                            \
            throw ::adipc_gpu::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e) + \
                                         " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
    } while (0)

// Every kernel launch of the library is followed by ADIPC_LAUNCH_CHECK, which
// also counts it (adipc_gpu_kernel_launches(), the bench's gpu_launches).
// Launches recorded into a CUDA graph are counted on the capturing thread
// (capture_count) and added to the global counter each time the graph is
// replayed, so the counter reports kernels actually executed.
std::atomic<long long>& launch_counter();
struct CaptureCount {
    bool active = false;
    long long n = 0;
};
CaptureCount& capture_count();
inline void count_launch() {
    CaptureCount& cc = capture_count();
    if (cc.active)
        ++cc.n;
    else
        launch_counter().fetch_add(1, std::memory_order_relaxed);
}
#define ADIPC_LAUNCH_CHECK()                \
    do {                                    \
        ::adipc_gpu::count_launch();        \
        ADIPC_CUDA(cudaGetLastError());     \
    } while (0)

__host__ __device__ inline std::int64_t ceil_div(std::int64_t a, std::int64_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch (sm_90+): a kernel launched with
// launch_pdl(..., pdl = true) may start while its predecessor in the stream
// drains; it runs its independent prologue (constant data, shared-memory and
// barrier setup, prefetches of operands that do not change during the solve)
// and calls pdl_wait() before touching anything the predecessor writes.
// pdl_launch() lets the successor's CTAs be scheduled. Both are no-ops for
// ordinary launches.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t st,
                              bool pdl, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Grid size for grid-stride kernels: enough CTAs for every SM several times
// over, never more than the work needs.
inline int grid_for(std::int64_t work_items, int items_per_cta, int per_sm = 8) {
    std::int64_t g = ceil_div(work_items, items_per_cta);
    const std::int64_t cap = static_cast<std::int64_t>(kSMs) * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return static_cast<int>(g);
}

// Growable device buffer (capacity only grows; contents not preserved).
template <class T>
struct DBuf {
    T* p = nullptr;
    std::size_t cap = 0;
    std::size_t n = 0;
    void reserve(std::size_t count) {
        if (count <= cap) {
            n = count;
            return;
        }
        // growing an existing buffer leaves 25 % headroom, so sizes that
        // fluctuate (contact patterns between Newton iterations) do not
        // reallocate every time
        const std::size_t want = cap ? count + count / 4 : count;
        if (p) cudaFree(p);
        p = nullptr;
        std::size_t c = want < 1 ? 1 : want;
        ADIPC_CUDA(cudaMalloc(&p, c * sizeof(T)));
        cap = c;
        n = count;
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = n = 0;
    }
    std::size_t bytes() const { return n * sizeof(T); }
};

// pinned host staging for device -> host copies of hierarchy data (pageable
// copies stage through the driver at a few GB/s)
struct HostStage {
    unsigned char* p = nullptr;
    std::size_t cap = 0;
    void* reserve(std::size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            const std::size_t want = bytes + bytes / 4;
            ADIPC_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p), want));
            cap = want;
        }
        return p;
    }
    void free() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Block value storage of the assembled matrix: 32-block tiles, SoA inside a
// tile ("AoSoA"): element k (column-major within the 3x3 block) of block e
// lives at blk(e, k). A warp working on 32 consecutive blocks reads one
// contiguous 2,304-byte tile with nine fully coalesced 256-byte loads.
__host__ __device__ __forceinline__ std::int64_t blk(std::int64_t e, int k) { return (e >> 5) * 288 + 32 * k + (e & 31); }
inline std::size_t blk_doubles(std::int64_t U) { return static_cast<std::size_t>((U + 31) >> 5) * 288; }

// Symmetric-packed storage of a d x d subdomain inverse: upper triangle by
// columns, entry (j, k), j <= k, at k(k+1)/2 + j; padded to an even count so
// every inverse starts 16-byte aligned (one TMA bulk copy each).
__host__ __device__ __forceinline__ std::int64_t packed_doubles(int d) {
    const std::int64_t n = static_cast<std::int64_t>(d) * (d + 1) / 2;
    return (n + 1) & ~std::int64_t(1);
}
__host__ __device__ __forceinline__ int packed_idx(int j, int k) {  // any order
    return j <= k ? k * (k + 1) / 2 + j : j * (j + 1) / 2 + k;
}

// Block-wide sum of a double; result valid in thread 0. blockDim <= 1024.
__device__ __forceinline__ double block_sum(double v, double* smem32) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) smem32[w] = v;
    __syncthreads();
    double s = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < nw; ++i) s += smem32[i];  // fixed order: deterministic
    return s;
}

}  // namespace adipc_gpu

namespace adipc_gpu {

// Grid-wide deterministic reduction of one double per CTA: every CTA stores
// its partial, the last CTA to arrive (ticket) sums all partials in a fixed
// order and writes *out, then re-arms the ticket. Must be called by all
// threads of every CTA; `v` is this thread's contribution.
// `advance` (optional): incremented once by the last CTA, after *out is
// written (the PCG iteration index, advanced by the iteration's first kernel).
__device__ __forceinline__ void grid_sum_last_block(double v, double* partials, unsigned* ticket, double* out,
                                                    int* advance = nullptr) {
    __shared__ double red[32];
    __shared__ bool last;
    const double bs = block_sum(v, red);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = bs;
        __threadfence();
        const unsigned t = atomicAdd(ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double s = 0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) s += __ldcg(partials + i);
    const double tot = block_sum(s, red);
    if (threadIdx.x == 0) {
        *out = tot;
        *ticket = 0;
        if (advance) *advance += 1;
    }
}

}  // namespace adipc_gpu
