// SPDX-License-Identifier: Apache-2.0
//
// On-device self-test of the tcgen05 building blocks the tensor-core engine relies on: one CTA,
// one 128 x N x K product checked against a double-precision host product. Modes:
//   0  SS: A K-major [128 x K], B K-major [N x K]            D = A B^T
//   1  SS: B stored as a K-major tile of its transpose, read MN-major (lbo = 128 B, sbo = K*16)
//   2  as 1 with lbo/sbo swapped
//   3  TS: A in TMEM (lane = row, column c = bf16 pair (2c, 2c+1)), B as in mode 1
//   4  TS: A in TMEM, B K-major as in mode 0
//   5  as 4, A copied smem -> TMEM by tcgen05.cp.128x256b (one k-step of 16 per copy) in the MMA pipe
#include <cuda_bf16.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "engine.h"
#include "tc_common.cuh"

namespace ember {
namespace {

__global__ void __launch_bounds__(256, 1)
    k_tc_selftest(int mode, const uint16_t* __restrict__ A, const uint16_t* __restrict__ B, int K, int N, float* D) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sB = smem + 128 * K * 2;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const bool b_mn = (mode == 1 || mode == 2 || mode == 3);
    for (int i = tid; i < 128 * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        *reinterpret_cast<uint16_t*>(sA + tc::kmajor_off(r, k, 128)) = A[i];
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        if (b_mn) {  // B row-major [K x N]: stored as a K-major tile with K rows, N "columns"
            const int kk = i / N, n = i % N;
            *reinterpret_cast<uint16_t*>(sB + tc::kmajor_off(kk, n, K)) = B[i];
        } else {  // B row-major [N x K]
            const int n = i / K, k = i % K;
            *reinterpret_cast<uint16_t*>(sB + tc::kmajor_off(n, k, N)) = B[i];
        }
    }
    if (tid == 0) {
        tc::mbar_init(&bar, 1);
        tc::fence_mbar_init();
    }
    tc::fence_async_smem();
    __syncthreads();
    if (warp == 1) tc::tmem_alloc(&tslot, 256);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t taddr = tslot;
    const bool a_tmem = (mode == 3 || mode == 4 || mode == 5);
    if ((mode == 3 || mode == 4) && warp >= 4) {
        const int r = 32 * (warp % 4) + lane;
        for (int c0 = 0; c0 < K / 2; c0 += 32) {
            uint32_t v[32];
            for (int c = 0; c < 32; ++c) {
                const int k = 2 * (c0 + c);
                v[c] = (k < K) ? tc::pack2(A[r * K + k], A[r * K + k + 1]) : 0u;
            }
            tc::tmem_st32(taddr + ((uint32_t)(32 * (warp % 4)) << 16) + 128 + c0, v);
        }
        tc::tmem_st_wait();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (tid == 32) {
        const uint32_t id = tc::idesc_bf16(128, N, false, b_mn);
        const uint32_t a0 = tc::smem_addr(sA), b0 = tc::smem_addr(sB);
        for (int s = 0; s < K / 16; ++s) {
            uint64_t bd;
            if (mode == 1 || mode == 3) bd = tc::sdesc(b0 + s * 256, 128, K * 16);
            else if (mode == 2) bd = tc::sdesc(b0 + s * 256, K * 16, 128);
            else bd = tc::sdesc(b0 + s * 2 * N * 16, N * 16, 128);
            if (mode == 5)
                asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr + 128 + s * 8),
                             "l"(tc::sdesc(a0 + s * 2 * 128 * 16, 128 * 16, 128))
                             : "memory");
            if (a_tmem)
                tc::mma_ts(taddr, taddr + 128 + s * 8, bd, id, s > 0);
            else
                tc::mma_ss(taddr, tc::sdesc(a0 + s * 2 * 128 * 16, 128 * 16, 128), bd, id, s > 0);
        }
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::fence_after();
    if (warp >= 4) {
        const int r = 32 * (warp % 4) + lane;
        for (int c0 = 0; c0 < N; c0 += 16) {
            uint32_t v[16];
            tc::tmem_ld16(taddr + ((uint32_t)(32 * (warp % 4)) << 16) + c0, v);
            tc::tmem_ld_wait();
            for (int c = 0; c < 16; ++c) D[r * N + c0 + c] = __uint_as_float(v[c]);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(taddr, 256);
}

uint16_t to_bf16_bits(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}
float bf16_to_float(uint16_t h) {
    const uint32_t u = static_cast<uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

}  // namespace

double tc_selftest(int device, int mode, int K, int N, uint64_t seed) {
    if (K % 16 || K > 128 || N % 16 || N > 128 || N < 16) throw ConfigError("selftest: K, N multiples of 16 <= 128");
    EMBER_CUDA(cudaSetDevice(device));
    std::vector<uint16_t> a(128 * K), b(N * K);
    Rng g(seed);
    for (auto& x : a) x = to_bf16_bits(g.uniform(-1.f, 1.f));
    for (auto& x : b) x = to_bf16_bits(g.uniform(-1.f, 1.f));
    uint16_t *dA, *dB;
    float* dD;
    EMBER_CUDA(cudaMalloc(&dA, a.size() * 2));
    EMBER_CUDA(cudaMalloc(&dB, b.size() * 2));
    EMBER_CUDA(cudaMalloc(&dD, 128 * N * 4));
    EMBER_CUDA(cudaMemcpy(dA, a.data(), a.size() * 2, cudaMemcpyHostToDevice));
    EMBER_CUDA(cudaMemcpy(dB, b.data(), b.size() * 2, cudaMemcpyHostToDevice));
    EMBER_CUDA(cudaMemset(dD, 0xFF, 128 * N * 4));
    const int smem = 128 * K * 2 + 128 * 128 * 2;
    EMBER_CUDA(cudaFuncSetAttribute(k_tc_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_tc_selftest<<<1, 256, smem>>>(mode, dA, dB, K, N, dD);
    EMBER_CUDA(cudaGetLastError());
    EMBER_CUDA(cudaDeviceSynchronize());
    std::vector<float> d(128 * N);
    EMBER_CUDA(cudaMemcpy(d.data(), dD, d.size() * 4, cudaMemcpyDeviceToHost));
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    const bool b_mn = (mode == 1 || mode == 2 || mode == 3);
    double maxref = 0, maxerr = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            double ref = 0;
            for (int k = 0; k < K; ++k)
                ref += (double)bf16_to_float(a[m * K + k]) *
                       (double)bf16_to_float(b_mn ? b[k * N + n] : b[n * K + k]);
            maxref = std::max(maxref, std::fabs(ref));
            const double e = std::isfinite(d[m * N + n]) ? std::fabs(ref - d[m * N + n]) : 1e30;
            maxerr = std::max(maxerr, e);
        }
    return maxerr / std::max(maxref, 1e-30);
}

}  // namespace ember

// ---- MMA issue-throughput microbenchmark ------------------------------------------------------
// One CTA, one elected thread issues `iters` back-to-back tcgen05.mma (M=128, K=16, bf16) into one
// accumulator and waits for completion; returns cycles per MMA. mode: 0 SS (A, B K-major smem),
// 1 TS (A in TMEM, B K-major), 2 TS with B MN-major, 3 SS with B MN-major. Operand contents are
// irrelevant (zeros); only the timing is reported.
namespace ember {
namespace {
__global__ void __launch_bounds__(128, 1) k_tc_mmabench(int mode, int N, int iters, int nacc, long long* out) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar, 1);
        tc::fence_mbar_init();
    }
    tc::fence_async_smem();
    __syncthreads();
    if (warp == 0) tc::tmem_alloc(&tslot, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t t = tslot;
    if (warp == 0) {
        const bool b_mn = (mode == 2 || mode == 3);
        const uint32_t id = tc::idesc_bf16(128, N, false, b_mn);
        const uint32_t a0 = tc::smem_addr(smem), b0 = tc::smem_addr(smem + 32768);
        const uint64_t ad = tc::sdesc(a0, 128 * 16, 128);
        const uint64_t bd = b_mn ? tc::sdesc(b0, 128, 16 * 16) : tc::sdesc(b0, N * 16, 128);
        __syncwarp();
        const uint32_t d1 = t + (nacc > 1 ? (uint32_t)N : 0u), d2 = t + (nacc > 2 ? 2u * N : 0u),
                       d3 = t + (nacc > 3 ? 3u * N : 0u);
        const long long c0 = clock64();
        // 8 MMAs per trip, accumulators cycled t, d1, d2, d3 (nacc distinct values), no per-MMA math
        if (mode == 1 || mode == 2) {
            tc::mma_ts_elect(t, t + 256, bd, id, 0u);
            tc::mma_ts_elect(d1, t + 256, bd, id, 0u);
            tc::mma_ts_elect(d2, t + 256, bd, id, 0u);
            tc::mma_ts_elect(d3, t + 256, bd, id, 0u);
            for (int i = 0; i < iters; i += 8) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    tc::mma_ts_elect(t, t + 256, bd, id, 1u);
                    tc::mma_ts_elect(d1, t + 256, bd, id, 1u);
                    tc::mma_ts_elect(d2, t + 256, bd, id, 1u);
                    tc::mma_ts_elect(d3, t + 256, bd, id, 1u);
                }
            }
        } else {
            tc::mma_ss_elect(t, ad, bd, id, 0u);
            tc::mma_ss_elect(d1, ad, bd, id, 0u);
            tc::mma_ss_elect(d2, ad, bd, id, 0u);
            tc::mma_ss_elect(d3, ad, bd, id, 0u);
            for (int i = 0; i < iters; i += 8) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    tc::mma_ss_elect(t, ad, bd, id, 1u);
                    tc::mma_ss_elect(d1, ad, bd, id, 1u);
                    tc::mma_ss_elect(d2, ad, bd, id, 1u);
                    tc::mma_ss_elect(d3, ad, bd, id, 1u);
                }
            }
        }
        tc::mma_commit_elect(&bar);
        tc::mbar_wait(&bar, 0);
        const long long c1 = clock64();
        if (threadIdx.x == 0) *out = c1 - c0;
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(t, 512);
}
}  // namespace

double tc_mmabench(int device, int mode, int N, int iters, int nacc) {
    EMBER_CUDA(cudaSetDevice(device));
    long long* d;
    EMBER_CUDA(cudaMalloc(&d, 8));
    EMBER_CUDA(cudaFuncSetAttribute(k_tc_mmabench, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    long long best = -1;
    for (int rep = 0; rep < 3; ++rep) {
        k_tc_mmabench<<<1, 128, 65536>>>(mode, N, iters, nacc < 1 ? 1 : nacc, d);
        EMBER_CUDA(cudaGetLastError());
        EMBER_CUDA(cudaDeviceSynchronize());
        long long h;
        EMBER_CUDA(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
        if (best < 0 || h < best) best = h;
    }
    cudaFree(d);
    return (double)best / iters;
}
}  // namespace ember
