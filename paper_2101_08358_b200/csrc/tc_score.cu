// SPDX-License-Identifier: Apache-2.0
//
// Tensor-core engine (EMBER_ENGINE_TC_BF16X3): the shared-negative contraction of the step
// (SPEC.md:139-165 — scores of every positive's adjusted vector against the batch's shared
// negatives, log-softmax with the positive as an extra column, and its gradients) on the
// sm_100a 5th-generation tensor cores.
//
// Precision. Every fp32 operand x is split x = hi + lo with hi = bf16(x), lo = bf16(x - hi);
// a product uses the three terms hi*hi + hi*lo + lo*hi (fp32 accumulate in TMEM), ~2^-16
// relative per product — inside the 1e-4 per-step tolerance of the north_star.
//
// Operand layout in HBM (written by k_pack_*): per side, [2*CB column blocks][rows][8 bf16],
// CB = KP/8 (KP = dim rounded up to 16), hi blocks then lo blocks. Any row range of it is one
// TMA box {8, R, 2CB} that lands in shared memory as the canonical no-swizzle K-major UMMA
// tile [cb][R][16 B] (tc_common.cuh), and the same bytes serve as the MN-major operand of the
// transposed products.
//
// Per side, with A = adjusted vectors [nb x d], N = shared negatives [nt x d], b = nb:
//   k_tc_rows  (row-parallel, FlashAttention-forward shape): for each 128-row tile,
//              S = A N^T streamed over 64-negative tiles (TMEM, double-buffered), online
//              row max/sum with lazy rescaling, P = exp(S - m) in bf16 hi/lo to smem, and
//              dA += P N accumulated in TMEM. Epilogue: lse, g0 = (p_pos - 1)/b, dA /= Z*b.
//   k_tc_negs  (negative-parallel, FA-backward dK shape): for each 128-negative tile and a
//              chunk of 64-row sub-tiles, S^T = N A^T, P^T = exp(S^T - lse)/b, and
//              dN += P^T A in TMEM; partial dN per chunk, summed in fixed order by k_dn_reduce.
// Warp roles (both kernels): warp 0 = TMA producer, warp 1 = TMEM owner + MMA issuer
// (one thread), warps 2..5 = epilogue (TMEM lane quadrant = warp % 4).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "engine.h"
#include "tc_common.cuh"

namespace ember {
namespace {

constexpr int RT = 128;      // k_tc_rows: rows per tile (MMA M)
constexpr int NT1 = 64;      // k_tc_rows: negatives per tile (S: MMA N; P.N: K)
constexpr int NS1 = 3;       // k_tc_rows: negative-tile ring depth
constexpr int MT2 = 128;     // k_tc_negs: negatives per item (MMA M)
constexpr int RS2 = 64;      // k_tc_negs: rows per sub-tile
constexpr int NS2 = 3;       // k_tc_negs: row-sub-tile ring depth
constexpr int KPMAX = 128;   // largest padded dim
constexpr uint32_t TCOLS = 256;  // TMEM columns: S double buffer (2 x 64) + accumulator (<= 128)
constexpr int NTHREADS = 192;

struct TcArgs {
    int KP, CB, d, nb, nt, n_pad;
    float inv_b, tau;
    const float* fpos;
    float* lse;
    float* g0;
    float* dA;       // [2][nb][d]
    float* dN_part;  // [chunks][2][n_pad][d]
    int chunks2;
};

// Shared-memory carve-up (bytes), identical for both kernels:
//   big   : resident tile, 128 rows x KP x (hi, lo) bf16   = 512*KP
//   ring  : 3 stages of 64 rows x KP x (hi, lo)             = 3*256*KP
//   P     : 2 buffers of 128 x 64 x (hi, lo) bf16           = 2*32 KB
//   bars  : mbarriers + TMEM slot
struct Smem {
    uint8_t* big;
    uint8_t* ring[3];
    uint8_t* P[2];
    uint64_t* bars;
};
__host__ __device__ constexpr size_t big_bytes(int KP) { return (size_t)512 * KP; }
__host__ __device__ constexpr size_t stage_bytes(int KP) { return (size_t)256 * KP; }
constexpr size_t P_BYTES = 128 * 64 * 4;
__host__ __device__ constexpr size_t smem_total(int KP) {
    return 1024 + big_bytes(KP) + 3 * stage_bytes(KP) + 2 * P_BYTES + 256;
}

__device__ __forceinline__ Smem carve(uint8_t* raw, int KP) {
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    Smem s;
    s.big = base;
    uint8_t* p = base + big_bytes(KP);
    for (int i = 0; i < 3; ++i, p += stage_bytes(KP)) s.ring[i] = p;
    s.P[0] = p;
    s.P[1] = p + P_BYTES;
    s.bars = reinterpret_cast<uint64_t*>(p + 2 * P_BYTES);
    return s;
}

// barrier slots
enum {
    B_BIG_FULL = 0, B_BIG_EMPTY = 1,
    B_RING_FULL = 2,   // +3
    B_RING_EMPTY = 5,  // +3
    B_S_FULL = 8,      // +2
    B_S_EMPTY = 10,    // +2
    B_P_FULL = 12,     // +2
    B_P_EMPTY = 14,    // +2
    B_ACC_FULL = 16, B_ACC_EMPTY = 17,
    B_TMEM_SLOT = 18,  // uint32 slot lives here
    NBARS = 19
};

__device__ __forceinline__ uint32_t u32_of(float f) { return __float_as_uint(f); }

// Descriptor of a canonical K-major tile [cb][R][16 B] at k-step s (16 elements = 2 blocks).
__device__ __forceinline__ uint64_t kdesc(const uint8_t* tile, int R, int s, int cb0) {
    return tc::sdesc(tc::smem_addr(tile) + (uint32_t)((cb0 + 2 * s) * R * 16), (uint32_t)(R * 16), 128u);
}
// Same bytes read as the MN-major operand of the transposed product: K = R rows, k-step s.
__device__ __forceinline__ uint64_t mndesc(const uint8_t* tile, int R, int s, int cb0) {
    return tc::sdesc(tc::smem_addr(tile) + (uint32_t)(cb0 * R * 16 + s * 256), 128u, (uint32_t)(R * 16));
}

__device__ __forceinline__ void init_bars(uint64_t* bars) {
    tc::mbar_init(&bars[B_BIG_FULL], 1);
    tc::mbar_init(&bars[B_BIG_EMPTY], 1);
    for (int i = 0; i < 3; ++i) {
        tc::mbar_init(&bars[B_RING_FULL + i], 1);
        tc::mbar_init(&bars[B_RING_EMPTY + i], 1);
    }
    for (int i = 0; i < 2; ++i) {
        tc::mbar_init(&bars[B_S_FULL + i], 1);
        tc::mbar_init(&bars[B_S_EMPTY + i], 128);
        tc::mbar_init(&bars[B_P_FULL + i], 128);
        tc::mbar_init(&bars[B_P_EMPTY + i], 1);
    }
    tc::mbar_init(&bars[B_ACC_FULL], 1);
    tc::mbar_init(&bars[B_ACC_EMPTY], 128);
    tc::fence_mbar_init();
}

// Every epilogue thread arrives (count 128): its own TMEM reads / smem writes are ordered
// before its own release-arrive.
__device__ __forceinline__ void epi_arrive(uint64_t* bar) { tc::mbar_arrive(bar); }

// Loads 64 fp32 TMEM columns of this warp's lane quadrant.
__device__ __forceinline__ void ld64(uint32_t taddr, float (&v)[64]) {
    uint32_t a[32], b[32];
    tc::tmem_ld32(taddr, a);
    tc::tmem_ld32(taddr + 32, b);
    tc::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        v[i] = __uint_as_float(a[i]);
        v[32 + i] = __uint_as_float(b[i]);
    }
}

// Writes row `r` of a 128-row K-major bf16 hi/lo operand tile (64 K-elements) from 64 values.
__device__ __forceinline__ void store_p_row(uint8_t* P, int r, const float (&p)[64]) {
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        float x[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = p[8 * g + i];
        uint4 hi, lo;
        tc::split8(x, hi, lo);
        *reinterpret_cast<uint4*>(P + g * (128 * 16) + r * 16) = hi;
        *reinterpret_cast<uint4*>(P + 16384 + g * (128 * 16) + r * 16) = lo;
    }
}

// =========================================================================================
// k_tc_rows: scores, online LSE and dA for 128-row tiles (items = 2 sides x row tiles).
// =========================================================================================
__global__ void __launch_bounds__(NTHREADS, 1)
    k_tc_rows(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapN, TcArgs g) {
    extern __shared__ uint8_t smem_raw[];
    const Smem sm = carve(smem_raw, g.KP);
    uint64_t* bars = sm.bars;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(&bars[B_TMEM_SLOT]);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int KP = g.KP, CB = g.CB;
    const int row_tiles = (g.nb + RT - 1) / RT;
    const int n_items = 2 * row_tiles;
    const int J = (g.nt + NT1 - 1) / NT1;  // negative tiles
    const int KS = KP / 16;                // k-steps of the score product

    if (threadIdx.x == 0) {
        init_bars(bars);
        tc::tmap_prefetch(&mapA);
        tc::tmap_prefetch(&mapN);
    }
    if (warp == 1) tc::tmem_alloc(tslot, TCOLS);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = *tslot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------------------------------------------- TMA producer
            uint32_t it = 0, gn = 0;
            const uint32_t bytesA = (uint32_t)(RT * KP * 4), bytesN = (uint32_t)(NT1 * KP * 4);
            for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
                const int side = item / row_tiles, tile = item % row_tiles;
                tc::mbar_wait(&bars[B_BIG_EMPTY], (it & 1) ^ 1);
                tc::mbar_expect_tx(&bars[B_BIG_FULL], bytesA);
                tc::tma_load_4d(sm.big, &mapA, 0, tile * RT, 0, side, &bars[B_BIG_FULL]);
                for (int j = 0; j < J; ++j, ++gn) {
                    const int st = gn % NS1;
                    tc::mbar_wait(&bars[B_RING_EMPTY + st], ((gn / NS1) & 1) ^ 1);
                    tc::mbar_expect_tx(&bars[B_RING_FULL + st], bytesN);
                    tc::tma_load_4d(sm.ring[st], &mapN, 0, j * NT1, 0, side, &bars[B_RING_FULL + st]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ----------------------------------------------------- MMA issuer
            const uint32_t id_s = tc::idesc_bf16(128, NT1, false, false);
            const uint32_t id_pn = tc::idesc_bf16(128, KP, false, true);
            const uint32_t t_acc = tbase + 2 * NT1;
            uint32_t it = 0, gn = 0, gs = 0, gp = 0;
            for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
                tc::mbar_wait(&bars[B_BIG_FULL], it & 1);
                tc::fence_after();
                int prev_st = 0;
                for (int j = 0; j <= J; ++j) {
                    int st = 0;
                    if (j < J) {  // S_j = A . N_j^T
                        st = gn % NS1;
                        tc::mbar_wait(&bars[B_RING_FULL + st], (gn / NS1) & 1);
                        const int sb = gs & 1;
                        tc::mbar_wait(&bars[B_S_EMPTY + sb], ((gs >> 1) & 1) ^ 1);
                        tc::fence_after();
                        const uint32_t t_s = tbase + sb * NT1;
                        const uint8_t* Nt = sm.ring[st];
                        for (int s = 0; s < KS; ++s) {
                            const uint64_t ah = kdesc(sm.big, RT, s, 0), al = kdesc(sm.big, RT, s, CB);
                            const uint64_t nh = kdesc(Nt, NT1, s, 0), nl = kdesc(Nt, NT1, s, CB);
                            tc::mma_ss(t_s, al, nh, id_s, s > 0 ? 1u : 0u);
                            tc::mma_ss(t_s, ah, nl, id_s, 1u);
                            tc::mma_ss(t_s, ah, nh, id_s, 1u);
                        }
                        tc::mma_commit(&bars[B_S_FULL + sb]);
                        ++gs;
                        ++gn;
                    }
                    if (j > 0) {  // dA += P_{j-1} . N_{j-1}
                        const int pb = gp & 1;
                        tc::mbar_wait(&bars[B_P_FULL + pb], (gp >> 1) & 1);
                        if (j == 1) tc::mbar_wait(&bars[B_ACC_EMPTY], (it & 1) ^ 1);
                        tc::fence_after();
                        const uint8_t* Nt = sm.ring[prev_st];
                        const uint8_t* Pt = sm.P[pb];
                        for (int s = 0; s < NT1 / 16; ++s) {
                            const uint64_t ph = kdesc(Pt, 128, s, 0), pl = kdesc(Pt, 128, s, 8);
                            const uint64_t nh = mndesc(Nt, NT1, s, 0), nl = mndesc(Nt, NT1, s, CB);
                            tc::mma_ss(t_acc, pl, nh, id_pn, (j > 1 || s > 0) ? 1u : 0u);
                            tc::mma_ss(t_acc, ph, nl, id_pn, 1u);
                            tc::mma_ss(t_acc, ph, nh, id_pn, 1u);
                        }
                        tc::mma_commit(&bars[B_P_EMPTY + pb]);
                        tc::mma_commit(&bars[B_RING_EMPTY + prev_st]);
                        ++gp;
                    }
                    prev_st = st;
                }
                tc::mma_commit(&bars[B_ACC_FULL]);
                tc::mma_commit(&bars[B_BIG_EMPTY]);
            }
        }
    } else {  // ------------------------------------------------------------------ epilogue
        const int q = warp & 3;
        const int r = 32 * q + lane;
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        const uint32_t t_acc = tbase + 2 * NT1 + lane_off;
        const float L2E = 1.4426950408889634f;
        uint32_t it = 0, gs = 0, gp = 0;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
            const int side = item / row_tiles, tile = item % row_tiles;
            const int row = tile * RT + r;
            const bool valid = row < g.nb;
            const float fp = valid ? g.fpos[row] : 0.f;
            float m = fp, z = 0.f;
            for (int j = 0; j < J; ++j) {
                const int sb = gs & 1;
                tc::mbar_wait(&bars[B_S_FULL + sb], (gs >> 1) & 1);
                tc::fence_after();
                float v[64];
                ld64(tbase + sb * NT1 + lane_off, v);
                tc::fence_before();
                epi_arrive(&bars[B_S_EMPTY + sb]);
                ++gs;
                const int k0 = j * NT1;
                float tm = -INFINITY;
#pragma unroll
                for (int c = 0; c < 64; ++c) {
                    if (k0 + c >= g.nt) v[c] = -INFINITY;
                    tm = fmaxf(tm, v[c]);
                }
                if (j == 0) {
                    m = fmaxf(m, tm);
                } else {
                    const bool need = tm > m + g.tau;
                    if (__any_sync(0xffffffffu, need)) {
                        // lazy rescale: wait until P.N of tile j-1 has landed in the accumulator
                        const uint32_t u = gp - 1;
                        tc::mbar_wait(&bars[B_P_EMPTY + (u & 1)], (u >> 1) & 1);
                        tc::fence_after();
                        const float mn = need ? tm : m;
                        const float f = __expf(m - mn);
                        for (int c0 = 0; c0 < KP; c0 += 16) {
                            uint32_t a[16];
                            tc::tmem_ld16(t_acc + c0, a);
                            tc::tmem_ld_wait();
#pragma unroll
                            for (int i = 0; i < 16; ++i) a[i] = u32_of(__uint_as_float(a[i]) * f);
                            tc::tmem_st16(t_acc + c0, a);
                        }
                        tc::tmem_st_wait();
                        z *= f;
                        m = mn;
                    }
                }
                const float mL = m * L2E;
#pragma unroll
                for (int c = 0; c < 64; ++c) {
                    const float p = exp2f(fmaf(v[c], L2E, -mL));  // 0 for masked columns
                    v[c] = p;
                    z += p;
                }
                const int pb = gp & 1;
                tc::mbar_wait(&bars[B_P_EMPTY + pb], ((gp >> 1) & 1) ^ 1);
                store_p_row(sm.P[pb], r, v);
                tc::fence_async_smem();
                tc::fence_before();
                epi_arrive(&bars[B_P_FULL + pb]);
                ++gp;
            }
            // accumulator epilogue
            tc::mbar_wait(&bars[B_ACC_FULL], it & 1);
            tc::fence_after();
            const float Z = z + __expf(fp - m);
            const float l = m + __logf(Z);
            const float scale = g.inv_b / Z;
            float* out = g.dA + ((size_t)side * g.nb + (valid ? row : 0)) * g.d;
            for (int c0 = 0; c0 < KP; c0 += 16) {
                uint32_t a[16];
                tc::tmem_ld16(t_acc + c0, a);
                tc::tmem_ld_wait();
                if (valid) {
#pragma unroll
                    for (int i = 0; i < 16; i += 4)
                        if (c0 + i < g.d)
                            *reinterpret_cast<float4*>(out + c0 + i) =
                                make_float4(__uint_as_float(a[i]) * scale, __uint_as_float(a[i + 1]) * scale,
                                            __uint_as_float(a[i + 2]) * scale, __uint_as_float(a[i + 3]) * scale);
                }
            }
            tc::fence_before();
            epi_arrive(&bars[B_ACC_EMPTY]);
            if (valid) {
                g.lse[(size_t)side * g.nb + row] = l;
                g.g0[(size_t)side * g.nb + row] = (expf(fp - l) - 1.0f) * g.inv_b;
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tbase, TCOLS);
}

// =========================================================================================
// k_tc_negs: dN partials for (side, 128-negative tile, row chunk) items.
// =========================================================================================
__device__ __forceinline__ void negs_item(int item, int ntl, int chunks, int nsub, int& side, int& ntile, int& chunk,
                                          int& u0, int& U) {
    side = item / (ntl * chunks);
    const int rem = item % (ntl * chunks);
    ntile = rem / chunks;
    chunk = rem % chunks;
    u0 = (int)((long long)chunk * nsub / chunks);
    U = (int)((long long)(chunk + 1) * nsub / chunks) - u0;
}

__global__ void __launch_bounds__(NTHREADS, 1)
    k_tc_negs(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapN, TcArgs g) {
    extern __shared__ uint8_t smem_raw[];
    const Smem sm = carve(smem_raw, g.KP);
    uint64_t* bars = sm.bars;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(&bars[B_TMEM_SLOT]);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int KP = g.KP, CB = g.CB;
    const int ntl = g.n_pad / MT2;
    const int nsub = (g.nb + RS2 - 1) / RS2;
    const int n_items = 2 * ntl * g.chunks2;
    const int KS = KP / 16;

    if (threadIdx.x == 0) {
        init_bars(bars);
        tc::tmap_prefetch(&mapA);
        tc::tmap_prefetch(&mapN);
    }
    if (warp == 1) tc::tmem_alloc(tslot, TCOLS);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = *tslot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------------------------------------------- TMA producer
            uint32_t it = 0, ga = 0;
            const uint32_t bytesN = (uint32_t)(MT2 * KP * 4), bytesA = (uint32_t)(RS2 * KP * 4);
            for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
                int side, ntile, chunk, u0, U;
                negs_item(item, ntl, g.chunks2, nsub, side, ntile, chunk, u0, U);
                if (U == 0) continue;
                tc::mbar_wait(&bars[B_BIG_EMPTY], (it & 1) ^ 1);
                tc::mbar_expect_tx(&bars[B_BIG_FULL], bytesN);
                tc::tma_load_4d(sm.big, &mapN, 0, ntile * MT2, 0, side, &bars[B_BIG_FULL]);
                for (int u = 0; u < U; ++u, ++ga) {
                    const int st = ga % NS2;
                    tc::mbar_wait(&bars[B_RING_EMPTY + st], ((ga / NS2) & 1) ^ 1);
                    tc::mbar_expect_tx(&bars[B_RING_FULL + st], bytesA);
                    tc::tma_load_4d(sm.ring[st], &mapA, 0, (u0 + u) * RS2, 0, side, &bars[B_RING_FULL + st]);
                }
                ++it;
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ----------------------------------------------------- MMA issuer
            const uint32_t id_s = tc::idesc_bf16(128, RS2, false, false);
            const uint32_t id_dn = tc::idesc_bf16(128, KP, false, true);
            const uint32_t t_acc = tbase + 2 * RS2;
            uint32_t it = 0, ga = 0, gs = 0, gp = 0;
            for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
                int side, ntile, chunk, u0, U;
                negs_item(item, ntl, g.chunks2, nsub, side, ntile, chunk, u0, U);
                if (U == 0) continue;
                tc::mbar_wait(&bars[B_BIG_FULL], it & 1);
                tc::fence_after();
                int prev_st = 0;
                for (int u = 0; u <= U; ++u) {
                    int st = 0;
                    if (u < U) {
                        st = ga % NS2;
                        tc::mbar_wait(&bars[B_RING_FULL + st], (ga / NS2) & 1);
                        const int sb = gs & 1;
                        tc::mbar_wait(&bars[B_S_EMPTY + sb], ((gs >> 1) & 1) ^ 1);
                        tc::fence_after();
                        const uint32_t t_s = tbase + sb * RS2;
                        const uint8_t* At = sm.ring[st];
                        for (int s = 0; s < KS; ++s) {
                            const uint64_t nh = kdesc(sm.big, MT2, s, 0), nl = kdesc(sm.big, MT2, s, CB);
                            const uint64_t ah = kdesc(At, RS2, s, 0), al = kdesc(At, RS2, s, CB);
                            tc::mma_ss(t_s, nl, ah, id_s, s > 0 ? 1u : 0u);
                            tc::mma_ss(t_s, nh, al, id_s, 1u);
                            tc::mma_ss(t_s, nh, ah, id_s, 1u);
                        }
                        tc::mma_commit(&bars[B_S_FULL + sb]);
                        ++gs;
                        ++ga;
                    }
                    if (u > 0) {  // dN += P^T_{u-1} . A_{u-1}
                        const int pb = gp & 1;
                        tc::mbar_wait(&bars[B_P_FULL + pb], (gp >> 1) & 1);
                        if (u == 1) tc::mbar_wait(&bars[B_ACC_EMPTY], (it & 1) ^ 1);
                        tc::fence_after();
                        const uint8_t* At = sm.ring[prev_st];
                        const uint8_t* Pt = sm.P[pb];
                        for (int s = 0; s < RS2 / 16; ++s) {
                            const uint64_t ph = kdesc(Pt, 128, s, 0), pl = kdesc(Pt, 128, s, 8);
                            const uint64_t ah = mndesc(At, RS2, s, 0), al = mndesc(At, RS2, s, CB);
                            tc::mma_ss(t_acc, pl, ah, id_dn, (u > 1 || s > 0) ? 1u : 0u);
                            tc::mma_ss(t_acc, ph, al, id_dn, 1u);
                            tc::mma_ss(t_acc, ph, ah, id_dn, 1u);
                        }
                        tc::mma_commit(&bars[B_P_EMPTY + pb]);
                        tc::mma_commit(&bars[B_RING_EMPTY + prev_st]);
                        ++gp;
                    }
                    prev_st = st;
                }
                tc::mma_commit(&bars[B_ACC_FULL]);
                tc::mma_commit(&bars[B_BIG_EMPTY]);
                ++it;
            }
        }
    } else {  // ------------------------------------------------------------------ epilogue
        const int q = warp & 3;
        const int n = 32 * q + lane;  // negative within the tile
        const uint32_t lane_off = (uint32_t)(32 * q) << 16;
        const uint32_t t_acc = tbase + 2 * RS2 + lane_off;
        const float L2E = 1.4426950408889634f;
        const float log2_inv_b = log2f(g.inv_b);
        uint32_t it = 0, gs = 0, gp = 0;
        for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
            int side, ntile, chunk, u0, U;
            negs_item(item, ntl, g.chunks2, nsub, side, ntile, chunk, u0, U);
            float* out = g.dN_part + (((size_t)chunk * 2 + side) * g.n_pad + (size_t)ntile * MT2 + n) * g.d;
            if (U == 0) {
                for (int c = 0; c < g.d; c += 4) *reinterpret_cast<float4*>(out + c) = make_float4(0.f, 0.f, 0.f, 0.f);
                continue;
            }
            const float* lse = g.lse + (size_t)side * g.nb;
            for (int u = 0; u < U; ++u) {
                const int sb = gs & 1;
                tc::mbar_wait(&bars[B_S_FULL + sb], (gs >> 1) & 1);
                tc::fence_after();
                float v[64];
                ld64(tbase + sb * RS2 + lane_off, v);
                tc::fence_before();
                epi_arrive(&bars[B_S_EMPTY + sb]);
                ++gs;
                const int row0 = (u0 + u) * RS2;
#pragma unroll
                for (int c = 0; c < 64; ++c) {
                    const int row = row0 + c;
                    // P^T = exp(S - lse) / b, folded into one exp2; rows past the batch -> 0
                    const float l = row < g.nb ? __ldg(lse + row) : INFINITY;
                    v[c] = exp2f(fmaf(v[c], L2E, fmaf(-l, L2E, log2_inv_b)));
                }
                const int pb = gp & 1;
                tc::mbar_wait(&bars[B_P_EMPTY + pb], ((gp >> 1) & 1) ^ 1);
                store_p_row(sm.P[pb], n, v);
                tc::fence_async_smem();
                tc::fence_before();
                epi_arrive(&bars[B_P_FULL + pb]);
                ++gp;
            }
            tc::mbar_wait(&bars[B_ACC_FULL], it & 1);
            tc::fence_after();
            for (int c0 = 0; c0 < KP; c0 += 16) {
                uint32_t a[16];
                tc::tmem_ld16(t_acc + c0, a);
                tc::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                    if (c0 + i < g.d)
                        *reinterpret_cast<float4*>(out + c0 + i) = make_float4(
                            __uint_as_float(a[i]), __uint_as_float(a[i + 1]), __uint_as_float(a[i + 2]),
                            __uint_as_float(a[i + 3]));
            }
            tc::fence_before();
            epi_arrive(&bars[B_ACC_EMPTY]);
            ++it;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tbase, TCOLS);
}

// =========================================================================================
// Operand packing and the dN reduction (memory-bound helpers).
// =========================================================================================

// src [2 sides][rows][d] fp32 (side stride side_stride rows) -> dst [2][2CB][cap][8] bf16 hi|lo.
// One thread per (side, cb, row); rows in [0, rows_pad) (zero past `rows`).
__global__ void k_pack(const float* __restrict__ src, uint64_t side_stride, int rows, int rows_pad, int cap, int d,
                       int CB, uint16_t* __restrict__ dst) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per_side = (int64_t)CB * rows_pad;
    if (t >= 2 * per_side) return;
    const int side = (int)(t / per_side);
    const int rem = (int)(t % per_side);
    const int cb = rem / rows_pad, row = rem % rows_pad;
    float x[8];
    const float* p = src + side * side_stride + (size_t)row * d + cb * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (row < rows && cb * 8 + i < d) ? p[i] : 0.f;
    uint4 hi, lo;
    tc::split8(x, hi, lo);
    uint4* out = reinterpret_cast<uint4*>(dst);
    const size_t base = (size_t)side * 2 * CB * cap;
    out[base + (size_t)cb * cap + row] = hi;
    out[base + (size_t)(CB + cb) * cap + row] = lo;
}

__global__ void k_dn_reduce(const float* __restrict__ part, int chunks, int nt, int n_pad, int d,
                            float* __restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per_side = (int64_t)nt * d;
    if (t >= 2 * per_side) return;
    const int side = (int)(t / per_side);
    const int rem = (int)(t % per_side);
    const int n = rem / d, k = rem % d;
    float acc = 0.f;
    for (int c = 0; c < chunks; ++c) acc += part[(((size_t)c * 2 + side) * n_pad + n) * d + k];
    out[t] = acc;
}

// ---- tensor maps (driver entry point fetched through the runtime: no libcuda link) ---------
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
    static EncodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        EMBER_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw EmberError("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiled>(p);
    }
    return fn;
}

// 4-D view {8 bf16, rows (cap), 2CB blocks, 2 sides} of a packed operand; box {8, box_rows, 2CB, 1}.
CUtensorMap make_map(uint16_t* base, int cap, int CB, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[4] = {8, (cuuint64_t)cap, (cuuint64_t)(2 * CB), 2};
    const cuuint64_t strides[3] = {16, (cuuint64_t)cap * 16, (cuuint64_t)cap * 16 * 2 * CB};
    const cuuint32_t box[4] = {8, (cuuint32_t)box_rows, (cuuint32_t)(2 * CB), 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw EmberError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

}  // namespace

// Engine-side state of the tensor-core engine (allocated once per context).
struct TcState {
    int KP = 0, CB = 0, b_cap = 0, n_pad = 0, chunks2 = 1;
    uint16_t* A = nullptr;   // [2][2CB][b_cap][8]
    uint16_t* N = nullptr;   // [2][2CB][n_pad][8]
    float* dN_part = nullptr;
    CUtensorMap mA128, mA64, mN64, mN128;
    float tau = 30.f;
};

bool tc_engine_supported(const Engine& E) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, E.device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, E.device);
    return major == 10 && minor == 0 && E.dim <= (uint32_t)KPMAX && E.chunks == 1 && E.nt >= 1;
}

void tc_setup(Engine& E) {
    auto* t = new TcState();
    t->KP = (int)((E.dim + 15) / 16 * 16);
    t->CB = t->KP / 8;
    t->b_cap = (int)((E.cap_b + RT - 1) / RT * RT);
    t->n_pad = (int)((E.nt + MT2 - 1) / MT2 * MT2);
    const int ntl = t->n_pad / MT2;
    t->chunks2 = std::max(1, E.sm_count / (2 * ntl));
    if (const char* s = getenv("EMBER_TC_TAU")) t->tau = (float)atof(s);
    EMBER_CUDA(cudaMalloc(&t->A, (size_t)2 * 2 * t->CB * t->b_cap * 16));
    EMBER_CUDA(cudaMalloc(&t->N, (size_t)2 * 2 * t->CB * t->n_pad * 16));
    EMBER_CUDA(cudaMalloc(&t->dN_part, (size_t)t->chunks2 * 2 * t->n_pad * E.dim * sizeof(float)));
    t->mA128 = make_map(t->A, t->b_cap, t->CB, RT);
    t->mA64 = make_map(t->A, t->b_cap, t->CB, RS2);
    t->mN64 = make_map(t->N, t->n_pad, t->CB, NT1);
    t->mN128 = make_map(t->N, t->n_pad, t->CB, MT2);
    const size_t smem = smem_total(t->KP);
    EMBER_CUDA(cudaFuncSetAttribute(k_tc_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    EMBER_CUDA(cudaFuncSetAttribute(k_tc_negs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    E.tc = t;
}

void tc_release(Engine& E) {
    if (!E.tc) return;
    cudaFree(E.tc->A);
    cudaFree(E.tc->N);
    cudaFree(E.tc->dN_part);
    delete E.tc;
    E.tc = nullptr;
}

void launch_contract_tc(Engine& E, uint32_t nb) {
    TcState& t = *E.tc;
    const int d = (int)E.dim, nt = (int)E.nt;
    Scratch& s = E.s;
    const int rows_pad = (int)((nb + RT - 1) / RT * RT);
    {
        const int64_t n = (int64_t)2 * t.CB * rows_pad;
        k_pack<<<(unsigned)((n + 255) / 256), 256, 0, E.stream>>>(s.A, (uint64_t)nb * d, (int)nb, rows_pad, t.b_cap, d,
                                                                  t.CB, t.A);
        EMBER_LAUNCHED(E);
        const int64_t m = (int64_t)2 * t.CB * t.n_pad;
        k_pack<<<(unsigned)((m + 255) / 256), 256, 0, E.stream>>>(s.N, (uint64_t)nt * d, nt, t.n_pad, t.n_pad, d, t.CB,
                                                                  t.N);
        EMBER_LAUNCHED(E);
    }
    TcArgs a{};
    a.KP = t.KP;
    a.CB = t.CB;
    a.d = d;
    a.nb = (int)nb;
    a.nt = nt;
    a.n_pad = t.n_pad;
    a.inv_b = 1.0f / (float)nb;
    a.tau = t.tau;
    a.fpos = s.fpos;
    a.lse = s.lse;
    a.g0 = s.g0;
    a.dA = s.dA;
    a.dN_part = t.dN_part;
    const int nsub = (int)((nb + RS2 - 1) / RS2);
    a.chunks2 = std::min(t.chunks2, nsub);
    const size_t smem = smem_total(t.KP);
    const int items1 = 2 * (rows_pad / RT);
    k_tc_rows<<<std::min(items1, E.sm_count), NTHREADS, smem, E.stream>>>(t.mA128, t.mN64, a);
    EMBER_LAUNCHED(E);
    const int items2 = 2 * (t.n_pad / MT2) * a.chunks2;
    k_tc_negs<<<std::min(items2, E.sm_count), NTHREADS, smem, E.stream>>>(t.mA64, t.mN128, a);
    EMBER_LAUNCHED(E);
    const int64_t r = (int64_t)2 * nt * d;
    k_dn_reduce<<<(unsigned)((r + 255) / 256), 256, 0, E.stream>>>(t.dN_part, a.chunks2, nt, t.n_pad, d,
                                                                    s.grows + (size_t)2 * nb * d);
    EMBER_LAUNCHED(E);
}

}  // namespace ember
