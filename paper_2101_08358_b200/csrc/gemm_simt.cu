// SPDX-License-Identifier: Apache-2.0
//
// SIMT fp32 engine for the shared-negative contraction (EMBER_ENGINE_SIMT_FP32): the fp32
// correctness baseline the tensor-core engine is measured against, available to tests only
// (the context rejects it unless EMBER_TEST_ENGINES=1 is set). Three batched GEMMs per
// (chunk, side) with the score matrix materialised in HBM:
//   S  = A N^T          (scores, SPEC.md:139-147 as a dense contraction)
//   P  = softmax rows   (log-sum-exp with the positive as an extra column)
//   dA = P N            (gradient wrt the adjusted vectors, before the positive term)
//   dN = P^T A          (gradient of the shared negatives; split over rows, reduced in order)
#include <cuda_runtime.h>

#include "engine.h"

namespace ember {
namespace {

// Element (r, c) of batch (q, s) lives at p[q*sq + s*ss + r*rs + c*cs].
struct Operand {
    const float* p;
    int64_t rs, cs, sq, ss;
};

struct GemmArgs {
    Operand a, b;
    float* c;
    int64_t ldc, csq, css;  // C offsets per (q, s); element (r, n) at c[q*csq + s*css + r*ldc + n]
    int M, N, K;            // full (un-ragged) extents
    int ragged;             // 0 none, 1: M is the chunk row count, 2: K is the chunk row count
    int chunk_rows, total_rows;
    int ksplit;             // split of K; partial results at c + ks*part_stride (accumulated later)
    int64_t part_stride;
    float alpha;
};

constexpr int BM = 64, BN = 64, BK = 16;

__global__ void __launch_bounds__(256) k_gemm(GemmArgs g) {
    const int z = blockIdx.z;
    const int q = z >> 1, sd = z & 1;
    int M = g.M, K = g.K;
    const int rows_q = min(g.chunk_rows, g.total_rows - q * g.chunk_rows);
    if (g.ragged == 1) M = rows_q;
    if (g.ragged == 2) K = rows_q;
    const int tiles_n = (g.N + BN - 1) / BN;
    const int m0 = (blockIdx.x / tiles_n) * BM;
    const int n0 = (blockIdx.x % tiles_n) * BN;
    if (m0 >= M) return;
    const int kper = (K + g.ksplit - 1) / g.ksplit;
    const int kbeg = blockIdx.y * kper;
    const int kend = min(K, kbeg + kper);

    const float* A = g.a.p + q * g.a.sq + sd * g.a.ss;
    const float* B = g.b.p + q * g.b.sq + sd * g.b.ss;
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    float acc[4][4] = {};
    for (int k0 = kbeg; k0 < kend; k0 += BK) {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            const int idx = tid + l * 256;  // 0..1023 over a 64x16 tile
            // A tile: (m, k) with m fastest when the operand is M-contiguous, else k fastest
            int mm, kk;
            if (g.a.rs == 1) { mm = idx % BM; kk = idx / BM; } else { kk = idx % BK; mm = idx / BK; }
            const int gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < M && gk < kend) ? A[gm * g.a.rs + gk * g.a.cs] : 0.f;
            int nn, kb;
            if (g.b.cs == 1) { nn = idx % BN; kb = idx / BN; } else { kb = idx % BK; nn = idx / BK; }
            const int gn = n0 + nn, gkb = k0 + kb;
            Bs[kb][nn] = (gn < g.N && gkb < kend) ? B[gkb * g.b.rs + gn * g.b.cs] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
    float* C = g.c + q * g.csq + sd * g.css + blockIdx.y * g.part_stride;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gm = m0 + ty * 4 + i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tx * 4 + j;
            if (gn < g.N) C[gm * g.ldc + gn] = g.alpha * acc[i][j];
        }
    }
}

void run_gemm(const Engine& E, const GemmArgs& g, int batches, cudaStream_t st) {
    const int tiles = ((g.M + BM - 1) / BM) * ((g.N + BN - 1) / BN);
    dim3 grid(tiles, g.ksplit, batches);
    k_gemm<<<grid, 256, 0, st>>>(g);
    EMBER_LAUNCHED(E);
}

// Row-wise log-sum-exp over [fpos, S row] (chunk-local negatives), P = exp(S - lse) / nb in place.
__global__ void k_softmax_rows(float* S, const float* fpos, float* lse, float* g0, uint32_t nb, uint32_t nt,
                               float inv_b) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (warp >= 2 * nb) return;
    const uint32_t side = warp / nb, e = warp % nb;
    float* row = S + (uint64_t)side * nb * nt + (uint64_t)e * nt;
    const float f = fpos[e];
    float mx = f;
    for (uint32_t k = lane; k < nt; k += 32) mx = fmaxf(mx, row[k]);
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float z = 0.f;
    for (uint32_t k = lane; k < nt; k += 32) z += expf(row[k] - mx);
    for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    z += expf(f - mx);
    const float l = mx + logf(z);
    for (uint32_t k = lane; k < nt; k += 32) row[k] = expf(row[k] - l) * inv_b;
    if (lane == 0) {
        lse[(uint64_t)side * nb + e] = l;
        g0[(uint64_t)side * nb + e] = (expf(f - l) - 1.0f) * inv_b;
    }
}

// dN row k (negative slot 2nb + k) -> its sorted gradient position grows[rank[2nb + k]].
__global__ void k_sum_parts(const float* parts, uint32_t nparts, uint64_t stride, uint64_t n, uint32_t d,
                            const uint32_t* __restrict__ rank, uint32_t slot0, float* out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float acc = 0.f;
    for (uint32_t k = 0; k < nparts; ++k) acc += parts[k * stride + i];
    out[(uint64_t)rank[slot0 + i / d] * d + i % d] = acc;
}

}  // namespace

void launch_contract_simt(Engine& E, uint32_t nb) {
    const int d = (int)E.dim, nt = (int)E.nt, C = (int)E.chunks;
    const int cr = (int)((nb + E.chunks - 1) / E.chunks);
    const int batches = 2 * C;
    cudaStream_t st = E.stream;
    Scratch& s = E.s;

    // 1) S = A N^T : M = chunk rows, N = nt, K = d
    GemmArgs g{};
    g.a = {s.A, d, 1, (int64_t)cr * d, (int64_t)nb * d};
    g.b = {s.N, 1, d, (int64_t)2 * nt * d, (int64_t)nt * d};  // B(k, n) = N[n][k]
    g.c = s.S;
    g.ldc = nt;
    g.csq = (int64_t)cr * nt;
    g.css = (int64_t)nb * nt;
    g.M = cr; g.N = nt; g.K = d;
    g.ragged = 1; g.chunk_rows = cr; g.total_rows = (int)nb;
    g.ksplit = 1; g.part_stride = 0; g.alpha = 1.f;
    run_gemm(E, g, batches, st);

    // 2) softmax with the positive column
    const uint32_t warps = 2 * nb;
    k_softmax_rows<<<(warps * 32 + 255) / 256, 256, 0, st>>>(s.S, s.fpos, s.lse, s.g0, nb, E.nt, 1.0f / (float)nb);
    EMBER_LAUNCHED(E);

    // 3) dA = P N : M = chunk rows, N = d, K = nt
    GemmArgs h{};
    h.a = {s.S, nt, 1, (int64_t)cr * nt, (int64_t)nb * nt};
    h.b = {s.N, d, 1, (int64_t)2 * nt * d, (int64_t)nt * d};
    h.c = s.dA;
    h.ldc = d;
    h.csq = (int64_t)cr * d;
    h.css = (int64_t)nb * d;
    h.M = cr; h.N = d; h.K = nt;
    h.ragged = 1; h.chunk_rows = cr; h.total_rows = (int)nb;
    h.ksplit = 1; h.part_stride = 0; h.alpha = 1.f;
    run_gemm(E, h, batches, st);

    // 4) dN = P^T A : M = nt, N = d, K = chunk rows; split-K partials then ordered sum into grows
    const int ks = (int)E.dsplit;
    GemmArgs n{};
    n.a = {s.S, 1, nt, (int64_t)cr * nt, (int64_t)nb * nt};  // A(m=k_neg, k=row) = P[row][k_neg]
    n.b = {s.A, d, 1, (int64_t)cr * d, (int64_t)nb * d};
    n.c = s.dN_part;
    n.ldc = d;
    n.csq = (int64_t)2 * nt * d;
    n.css = (int64_t)nt * d;
    n.M = nt; n.N = d; n.K = cr;
    n.ragged = 2; n.chunk_rows = cr; n.total_rows = (int)nb;
    n.ksplit = ks; n.part_stride = (int64_t)E.n_neg * d; n.alpha = 1.f;
    run_gemm(E, n, batches, st);
    const uint64_t total = (uint64_t)E.n_neg * d;
    E.join_sorted();
    k_sum_parts<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(s.dN_part, ks, total, total, (uint32_t)d, s.rank,
                                                                  2 * nb, s.grows);
    EMBER_LAUNCHED(E);
}

}  // namespace ember
