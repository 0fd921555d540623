// SPDX-License-Identifier: Apache-2.0
//
// SIMT fp32 engine for the shared-negative contraction (EMBER_ENGINE_SIMT_FP32): the
// correctness baseline the tensor-core engine is measured against. Three batched GEMMs per
// (chunk, side) with the score matrix materialised in HBM:
//   S  = A N^T          (scores, SPEC.md:139-147 as a dense contraction)
//   P  = softmax rows   (log-sum-exp with the positive as an extra column)
//   dA = P N            (gradient wrt the adjusted vectors, before the positive term)
//   dN = P^T A          (gradient of the shared negatives; split over rows, reduced in order)
#include <cublas_v2.h>  // types and enums only: the library is bound at run time (dlopen)
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

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

// ---- EMBER_ENGINE_TC_BLAS: the same materialised-score contraction on tensor cores through
// cuBLAS bf16 GEMMs with the bf16x3 split (hi.lo + lo.hi + hi.hi, fp32 accumulation: the
// tensor-core engine's arithmetic), for d > 128 where the hand-written kernels' TMEM layout ends
// (config C5, d = 800). cuBLAS is bound at run time from the process (torch's copy when loaded)
// or the CUDA toolkit, so the library has no link-time dependency on it.
namespace {

struct BlasApi {
    void* h = nullptr;
    decltype(&cublasCreate_v2) create = nullptr;
    decltype(&cublasDestroy_v2) destroy = nullptr;
    decltype(&cublasSetStream_v2) set_stream = nullptr;
    using GemmFn = cublasStatus_t (*)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const void*,
                                      const void*, cudaDataType, int, long long, const void*, cudaDataType, int,
                                      long long, const void*, void*, cudaDataType, int, long long, int,
                                      cublasComputeType_t, cublasGemmAlgo_t);
    GemmFn gemm = nullptr;
};

const BlasApi& blas_api() {
    static BlasApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        for (const char* n : {"libcublas.so.12", "/usr/local/cuda/lib64/libcublas.so.12"})
            if ((api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
        if (api.h) {
            api.create = reinterpret_cast<decltype(api.create)>(dlsym(api.h, "cublasCreate_v2"));
            api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(api.h, "cublasDestroy_v2"));
            api.set_stream = reinterpret_cast<decltype(api.set_stream)>(dlsym(api.h, "cublasSetStream_v2"));
            api.gemm = reinterpret_cast<decltype(api.gemm)>(dlsym(api.h, "cublasGemmStridedBatchedEx"));
        }
    }
    if (!api.create || !api.destroy || !api.set_stream || !api.gemm)
        throw EmberError("cuBLAS (libcublas.so.12) not loadable: the blas engine needs it");
    return api;
}

void blas_check(cublasStatus_t st, const char* what) {
    if (st != CUBLAS_STATUS_SUCCESS) throw EmberError(std::string("cuBLAS ") + what + " failed: status " + std::to_string((int)st));
}

// hi = bf16(x), lo = bf16(x - hi), elementwise (n multiple of 4 not required)
__global__ void k_split_bf16(const float* __restrict__ x, uint64_t n, __nv_bfloat16* __restrict__ hi,
                             __nv_bfloat16* __restrict__ lo) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float v = x[i];
        const __nv_bfloat16 h = __float2bfloat16_rn(v);
        hi[i] = h;
        lo[i] = __float2bfloat16_rn(v - __bfloat162float(h));
    }
}

void split(const Engine& E, const float* x, uint64_t n, __nv_bfloat16* hi, __nv_bfloat16* lo) {
    const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)E.sm_count * 16);
    k_split_bf16<<<blocks, 256, 0, E.stream>>>(x, n, hi, lo);
    EMBER_LAUNCHED(E);
}

// Column-major C[m x n] (+)= op(A) op(B) over 2 batches (the corruption sides), bf16x3.
struct Split {
    const __nv_bfloat16 *hi, *lo;
    int ld;
    long long stride;
};
void gemm3(const Engine& E, cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k, const Split& a,
           const Split& b, float* c, int ldc, long long sc) {
    const BlasApi& api = blas_api();
    cublasHandle_t h = static_cast<cublasHandle_t>(E.blas);
    const float one = 1.f, zero = 0.f;
    const __nv_bfloat16* as[3] = {a.hi, a.lo, a.hi};
    const __nv_bfloat16* bs[3] = {b.lo, b.hi, b.hi};  // small terms first, then hi.hi
    for (int t = 0; t < 3; ++t)
        blas_check(api.gemm(h, ta, tb, m, n, k, &one, as[t], CUDA_R_16BF, a.ld, a.stride, bs[t], CUDA_R_16BF, b.ld,
                            b.stride, t ? &one : &zero, c, CUDA_R_32F, ldc, sc, 2, CUBLAS_COMPUTE_32F,
                            CUBLAS_GEMM_DEFAULT),
                   "gemm");
    EMBER_LAUNCHED(E);
}

}  // namespace

void blas_setup(Engine& E) {
    const BlasApi& api = blas_api();
    cublasHandle_t h = nullptr;
    blas_check(api.create(&h), "create");
    blas_check(api.set_stream(h, E.stream), "set stream");
    E.blas = h;
}

void blas_release(Engine& E) {
    if (E.blas) blas_api().destroy(static_cast<cublasHandle_t>(E.blas));
    E.blas = nullptr;
}

void launch_contract_blas(Engine& E, uint32_t nb) {
    const int d = (int)E.dim, nt = (int)E.nt, b = (int)nb;
    Scratch& s = E.s;
    using bf = __nv_bfloat16;
    bf* Ahi = reinterpret_cast<bf*>(s.Ahl);
    bf* Alo = Ahi + (size_t)2 * E.cap_b * d;
    bf* Nhi = reinterpret_cast<bf*>(s.Nhl);
    bf* Nlo = Nhi + (size_t)2 * nt * d;
    bf* Phi = reinterpret_cast<bf*>(s.Phl);
    bf* Plo = Phi + (size_t)2 * E.cap_b * nt;
    // s.A: [2][nb][d] (side stride nb*d), s.N: [2][nt][d], s.S: [2][nb][nt] -- all row-major
    split(E, s.A, (uint64_t)2 * b * d, Ahi, Alo);
    split(E, s.N, (uint64_t)2 * nt * d, Nhi, Nlo);
    const Split A{Ahi, Alo, d, (long long)b * d}, N{Nhi, Nlo, d, (long long)nt * d};
    // 1) S = A N^T  (row-major [nb x nt]) == column-major S^T = N A^T
    gemm3(E, CUBLAS_OP_T, CUBLAS_OP_N, nt, b, d, N, A, s.S, nt, (long long)b * nt);
    // 2) softmax with the positive column: P = exp(S - lse) / nb in place
    const uint32_t warps = 2 * nb;
    k_softmax_rows<<<(warps * 32 + 255) / 256, 256, 0, E.stream>>>(s.S, s.fpos, s.lse, s.g0, nb, E.nt,
                                                                   1.0f / (float)nb);
    EMBER_LAUNCHED(E);
    split(E, s.S, (uint64_t)2 * b * nt, Phi, Plo);
    const Split P{Phi, Plo, nt, (long long)b * nt};
    // 3) dA = P N  (row-major [nb x d]) == column-major dA^T = N^T P^T
    gemm3(E, CUBLAS_OP_N, CUBLAS_OP_N, d, b, nt, N, P, s.dA, d, (long long)b * d);
    // 4) dN = P^T A  (row-major [nt x d]) == column-major dN^T = A^T P
    gemm3(E, CUBLAS_OP_N, CUBLAS_OP_T, d, nt, b, A, P, s.dN_part, d, (long long)nt * d);
    const uint64_t total = (uint64_t)E.n_neg * d;
    E.join_sorted();
    k_sum_parts<<<(unsigned)((total + 255) / 256), 256, 0, E.stream>>>(s.dN_part, 1, total, total, (uint32_t)d, s.rank,
                                                                        2 * nb, s.grows);
    EMBER_LAUNCHED(E);
}

}  // namespace ember
