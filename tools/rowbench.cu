// Random-row bandwidth microbenchmark (B200): how fast can 400-byte rows at random positions of a
// large table be read / read-modify-written? Sets the ceiling for the gather, chain-rule and
// Adagrad kernels (random node rows of 69 GB tables). Build: nvcc -O3 -arch=sm_100a rowbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// mode 0: read rows (sum into a sink), mode 1: read-modify-write rows. Row ids come from an index
// array (like the edge lists of the real kernels); a warp issues the loads of all its rows first.
template <int MODE, int ROWS_PER_WARP>
__global__ void k_rows(float* table, const uint32_t* __restrict__ idx, uint32_t d, uint32_t n, float* sink) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w * ROWS_PER_WARP >= n) return;
    const uint32_t my = lane < ROWS_PER_WARP ? idx[w * ROWS_PER_WARP + lane] : 0u;
    float acc = 0.f;
    float4 v[ROWS_PER_WARP];
    float4* p[ROWS_PER_WARP];
#pragma unroll
    for (int k = 0; k < ROWS_PER_WARP; ++k) {
        const uint32_t row = __shfl_sync(0xffffffffu, my, k);
        p[k] = reinterpret_cast<float4*>(table + (uint64_t)row * d);
        if (lane < d / 4) v[k] = p[k][lane];
    }
#pragma unroll
    for (int k = 0; k < ROWS_PER_WARP; ++k) {
        if (lane < d / 4) {
            if (MODE == 1) {
                v[k].x += 1.f;
                p[k][lane] = v[k];
            } else {
                acc += v[k].x + v[k].y + v[k].z + v[k].w;
            }
        }
    }
    if (MODE != 1 && acc == 12345.f) sink[0] = acc;
}

__global__ void k_idx(uint32_t* idx, uint32_t n, uint64_t nrows, uint64_t seed) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) idx[i] = (uint32_t)(mix(seed + i) % nrows);
}

template <int MODE, int R>
void run(const char* name, float* table, uint64_t nrows, uint32_t d, uint32_t n, float* sink) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 20;
    uint32_t* idx = nullptr;
    cudaMalloc(&idx, (size_t)n * (iters + 3) * 4);
    k_idx<<<(n * (iters + 3) + 255) / 256, 256>>>(idx, n * (iters + 3), nrows, 77);
    const uint32_t warps = (n + R - 1) / R;
    for (int it = 0; it < 3; ++it) k_rows<MODE, R><<<(warps * 32 + 255) / 256, 256>>>(table, idx + (size_t)it * n, d, n, sink);
    cudaEventRecord(a);
    for (int it = 0; it < iters; ++it)
        k_rows<MODE, R><<<(warps * 32 + 255) / 256, 256>>>(table, idx + (size_t)(3 + it) * n, d, n, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)n * d * 4 * (MODE == 1 ? 2 : 1) * iters;
    printf("%-28s rows=%u  %.2f us/launch  %.0f GB/s\n", name, n, 1e3 * ms / iters, bytes / (ms * 1e-3) / 1e9);
    cudaFree(idx);
}

int main() {
    const uint32_t d = 100;
    float* table = nullptr;
    float* sink = nullptr;
    const uint64_t full = 86054151ull;  // FB86m: one table of theta (34 GB)
    if (cudaMalloc(&table, full * d * 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMalloc(&sink, 4);
    cudaMemset(table, 0, full * d * 4);
    // table spans: L2-resident, TLB-reach-ish, beyond both, the full FB86m table
    const uint64_t spans[4] = {250000ull, 2500000ull, 20000000ull, full};
    for (uint64_t nrows : spans) {
        printf("table %.2f GB\n", nrows * d * 4 / 1e9);
        run<0, 1>("read, 1 row/warp", table, nrows, d, 200000, sink);
        run<0, 4>("read, 4 rows/warp", table, nrows, d, 200000, sink);
        run<0, 8>("read, 8 rows/warp", table, nrows, d, 200000, sink);
        run<1, 1>("rmw, 1 row/warp", table, nrows, d, 200000, sink);
        run<1, 4>("rmw, 4 rows/warp", table, nrows, d, 200000, sink);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
