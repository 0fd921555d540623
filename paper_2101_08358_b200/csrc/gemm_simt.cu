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
#include <mutex>
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
    static std::mutex mu;  // contexts may be created from several host threads
    std::lock_guard<std::mutex> lock(mu);
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

// The bf16x3 product hi.lo + hi.hi + lo.hi as ONE GEMM over a 3x longer K: the K-concatenated
// operands carry [hi | hi | lo] and [lo | hi | hi] blocks (so the output is written once, no beta
// accumulation). Each operand is needed with K along its columns ("kd": [side][rows][3 cols]) or
// along its rows ("stack": [side][3 rows][cols]); lo_first selects [lo, hi, hi] over [hi, hi, lo].
__device__ __forceinline__ void put3(__nv_bfloat16* base, uint64_t blk, __nv_bfloat16 h, __nv_bfloat16 l, bool lo_first) {
    base[0] = lo_first ? l : h;
    base[blk] = h;
    base[2 * blk] = lo_first ? h : l;
}

__global__ void k_split3(const float* __restrict__ x, uint32_t rows, uint32_t cols, __nv_bfloat16* __restrict__ kd,
                         bool kd_lo_first, __nv_bfloat16* __restrict__ st, bool st_lo_first) {
    const uint32_t per = rows * cols, n = 2 * per;  // < 2^32 (checked by the caller)
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t side = i >= per, rc = i - side * per, r = rc / cols, c = rc - r * cols;
        const float v = x[i];
        const __nv_bfloat16 h = __float2bfloat16_rn(v), l = __float2bfloat16_rn(v - __bfloat162float(h));
        put3(kd + (uint64_t)side * 3 * per + (uint64_t)r * 3 * cols + c, cols, h, l, kd_lo_first);
        put3(st + (uint64_t)side * 3 * per + rc, per, h, l, st_lo_first);
    }
}

// Softmax rows with the positive column (as k_softmax_rows) writing P = exp(S - lse) / nb straight
// into its two split layouts: kd [hi | hi | lo] (dA = P N) and stack [lo; hi; hi] (dN = P^T A).
__global__ void k_softmax_split(const float* __restrict__ S, const float* __restrict__ fpos, float* lse, float* g0,
                                uint32_t nb, uint32_t nt, float inv_b, __nv_bfloat16* __restrict__ pkd,
                                __nv_bfloat16* __restrict__ pst) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (warp >= 2 * nb) return;
    const uint32_t side = warp / nb, e = warp % nb;
    const float* row = S + (uint64_t)side * nb * nt + (uint64_t)e * nt;
    const float f = fpos[e];
    float mx = f;
    for (uint32_t k = lane; k < nt; k += 32) mx = fmaxf(mx, row[k]);
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float z = 0.f;
    for (uint32_t k = lane; k < nt; k += 32) z += expf(row[k] - mx);
    for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
    z += expf(f - mx);
    const float l = mx + logf(z);
    const uint64_t per = (uint64_t)nb * nt;
    __nv_bfloat16* kd = pkd + side * 3 * per + (uint64_t)e * 3 * nt;
    __nv_bfloat16* st = pst + side * 3 * per + (uint64_t)e * nt;
    if ((nt & 1) == 0) {  // pairs of columns per lane: 4-byte stores
        for (uint32_t k = 2 * lane; k < nt; k += 64) {
            const float2 x = *reinterpret_cast<const float2*>(row + k);
            const float v0 = expf(x.x - l) * inv_b, v1 = expf(x.y - l) * inv_b;
            const __nv_bfloat162 h = __floats2bfloat162_rn(v0, v1);
            const float2 hf = __bfloat1622float2(h);
            const __nv_bfloat162 lo = __floats2bfloat162_rn(v0 - hf.x, v1 - hf.y);
            __nv_bfloat162* k2 = reinterpret_cast<__nv_bfloat162*>(kd + k);
            __nv_bfloat162* s2 = reinterpret_cast<__nv_bfloat162*>(st + k);
            k2[0] = h;
            k2[nt / 2] = h;
            k2[nt] = lo;
            s2[0] = lo;
            s2[per / 2] = h;
            s2[per] = h;
        }
    } else {
        for (uint32_t k = lane; k < nt; k += 32) {
            const float v = expf(row[k] - l) * inv_b;
            const __nv_bfloat16 h = __float2bfloat16_rn(v), lo = __float2bfloat16_rn(v - __bfloat162float(h));
            put3(kd + k, nt, h, lo, false);
            put3(st + k, per, h, lo, true);
        }
    }
    if (lane == 0) {
        lse[(uint64_t)side * nb + e] = l;
        g0[(uint64_t)side * nb + e] = (expf(f - l) - 1.0f) * inv_b;
    }
}

// dN partials [side][kc][nt][d] -> sum over the kc chunks in order -> sorted gradient rows.
__global__ void k_sum_chunks(const float* __restrict__ parts, uint32_t kc, uint64_t per, uint64_t n, uint32_t d,
                             const uint32_t* __restrict__ rank, uint32_t slot0, float* out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t side = i / per, rest = i % per;
    const float* p = parts + side * kc * per + rest;
    float acc = 0.f;
    for (uint32_t k = 0; k < kc; ++k) acc += p[k * per];
    out[(uint64_t)rank[slot0 + i / d] * d + i % d] = acc;
}

// Column-major C[m x n] = op(A) op(B) over the 2 corruption sides, bf16 in, fp32 out.
void gemm(const Engine& E, cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k, const __nv_bfloat16* a,
          int lda, long long sa, const __nv_bfloat16* b, int ldb, long long sb, float* c, int ldc, long long sc,
          int batches = 2) {
    const BlasApi& api = blas_api();
    const float one = 1.f, zero = 0.f;
    blas_check(api.gemm(static_cast<cublasHandle_t>(E.blas), ta, tb, m, n, k, &one, a, CUDA_R_16BF, lda, sa, b,
                        CUDA_R_16BF, ldb, sb, &zero, c, CUDA_R_32F, ldc, sc, batches, CUBLAS_COMPUTE_32F,
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
    const size_t ab = (size_t)2 * 3 * E.cap_b * d, nbf = (size_t)2 * 3 * nt * d;
    bf* Akd = reinterpret_cast<bf*>(s.Ahl);
    bf* Ast = Akd + ab;
    bf* Nkd = reinterpret_cast<bf*>(s.Nhl);
    bf* Nst = Nkd + nbf;
    bf* Pkd = reinterpret_cast<bf*>(s.Phl);
    bf* Pst = Pkd + (size_t)2 * 3 * E.cap_b * nt;
    const unsigned sb = (unsigned)E.sm_count * 16;
    if ((uint64_t)2 * b * d >= (1ull << 32) || (uint64_t)2 * nt * d >= (1ull << 32))
        throw ConfigError("blas engine: 2 * batch_size * dim must be < 2^32");
    // s.A: [2][nb][d], s.N: [2][nt][d], s.S: [2][nb][nt] -- row-major fp32
    // (A's splits, [hi hi lo] both ways, were written by the gather: k_gather_adjust<true>)
    k_split3<<<sb, 256, 0, E.stream>>>(s.N, (uint32_t)nt, (uint32_t)d, Nkd, true, Nst, true);  // [lo hi hi]
    EMBER_LAUNCHED(E);
    const int d3 = 3 * d, nt3 = 3 * nt, b3 = 3 * b;
    // 1) S = A N^T (row-major [nb x nt]) == column-major S^T = N A^T, K = 3d
    gemm(E, CUBLAS_OP_T, CUBLAS_OP_N, nt, b, d3, Nkd, d3, (long long)nt * d3, Akd, d3, (long long)b * d3, s.S, nt,
         (long long)b * nt);
    // 2) softmax with the positive column, P split into both layouts
    const uint32_t warps = 2 * nb;
    k_softmax_split<<<(warps * 32 + 255) / 256, 256, 0, E.stream>>>(s.S, s.fpos, s.lse, s.g0, nb, E.nt,
                                                                    1.0f / (float)nb, Pkd, Pst);
    EMBER_LAUNCHED(E);
    // 3) dA = P N (row-major [nb x d]) == column-major dA^T = N^T P^T, K = 3 nt (stacked N, kd P)
    gemm(E, CUBLAS_OP_N, CUBLAS_OP_N, d, b, nt3, Nst, d, (long long)nt3 * d, Pkd, nt3, (long long)b * nt3, s.dA, d,
         (long long)b * d);
    // 4) dN = P^T A (row-major [nt x d]) == column-major dN^T = A^T P, K = 3 nb (stacked A, stacked P).
    // The output is small (d x nt) and K long, so K is cut into kc chunks that run as extra GEMM
    // batches (batch = side * kc + chunk: uniform strides because a side's K is kc chunks long);
    // the partials are added in chunk order (deterministic) while scattering the rows.
    int kc = 1;
    for (int c : {16, 12, 8, 6, 4, 3, 2})
        if (b3 % c == 0) {
            kc = c;
            break;
        }
    const int kch = b3 / kc;
    gemm(E, CUBLAS_OP_N, CUBLAS_OP_T, d, nt, kch, Ast, d, (long long)kch * d, Pst, nt, (long long)kch * nt, s.dN_part, d,
         (long long)nt * d, 2 * kc);
    const uint64_t total = (uint64_t)E.n_neg * d;
    E.join_sorted();
    k_sum_chunks<<<(unsigned)((total + 255) / 256), 256, 0, E.stream>>>(s.dN_part, (uint32_t)kc, (uint64_t)nt * d,
                                                                         total, (uint32_t)d, s.rank, 2 * nb, s.grows);
    EMBER_LAUNCHED(E);
}

}  // namespace ember
