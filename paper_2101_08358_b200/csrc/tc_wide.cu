// SPDX-License-Identifier: Apache-2.0
//
// Tensor-core contraction for wide embeddings (d > 128, e.g. config C5's ComplEx d = 800), the
// same arithmetic as tc_score.cu (every fp32 operand split into bf16 hi + lo,
// products hi.hi + hi.lo + lo.hi accumulated in fp32 in TMEM) for dimensions whose operands and
// accumulators no longer fit one SM (tc_score.cu keeps a 128-row resident operand and the dA
// accumulator in TMEM, KP <= 128 columns each).
//
// Three passes of one persistent tcgen05 GEMM kernel (k_wide<PASS>), per corruption side:
//   SCORES  S = A N^T          M = 128 batch rows, N = 256 negatives, K = d        epilogue: P~ =
//           exp(S - f_pos) as bf16 hi|lo into HBM + partial row sums Z_j (the positive's score is the
//           row shift, as in tc_score.cu: no running max)
//   (stats) Z = 1 + sum_j Z_j, lse = f_pos + log Z, g0, row scale 1/(Z b); overflowed rows recomputed
//           exactly (k_wide_fixup); A' = A / (Z b) packed for the third pass
//   DA      dA = P~ N * 1/(Z b) M = 128 rows, N = a d-slab (<= 256), K = negatives  -> column-blocked dA
//   DN      dN = P~^T A'       M = 128 negatives, N = a d-slab, K = a chunk of batch rows -> partials,
//           summed in a fixed order by k_dn_reduce (tc_score.cu)
// Only P~ (bf16 hi|lo, 2 x b x n_t x 4 B) is materialised: at d = 800 it is ~8% of the operand
// bytes the three products stream through L2, and it replaces the score recompute of the fused
// kernels. Every operand is a packed bf16 hi|lo buffer [side][2 x blocks][rows][8] (blocks of 8
// columns; tc_score.cu's layout) read by TMA as canonical no-swizzle tiles, K-major or MN-major.
// Warps: 0 = TMA producer, 1 = MMA issuer (elected lane), 2..5 = epilogue (TMEM lanes 32 (w % 4)).
// TMEM: two 256-column fp32 accumulators (tile i+1's MMAs overlap tile i's epilogue).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>

#include "engine.h"
#include "tc_common.cuh"

namespace ember {

CUtensorMap make_packed_map(uint16_t* base, int cap, int nblocks2, int box_rows, int box_blocks);  // tc_score.cu

namespace {

enum { PASS_SCORES = 0, PASS_DA = 1, PASS_DN = 2 };
constexpr int WM = 128;       // output tile rows (MMA M)
constexpr int WKC = 64;       // K per pipeline stage (8 column blocks, or 64 rows of an MN-major operand)
constexpr int WNEG = 256;     // negatives per SCORES tile (MMA N)
constexpr int WSTAGES = 2;
constexpr int WTHREADS = 192;
constexpr float WL2E = 1.4426950408889634f;

struct WideArgs {
    int nb, nt, d;
    int chunks;     // num_chunks: chunk q = batch rows [q cr, min((q+1) cr, nb)) with its own negatives
    int cr, CP;     // batch rows per chunk; packed rows per chunk (multiple of 128)
    int CBA;        // column blocks (of 8) of the packed A / N / A' operands: KPW / 8
    int NBP;        // column blocks of P~: n_padw / 8
    int b_cap, n_pad;
    int slab;       // output columns per DA / DN tile (multiple of 16, <= 256)
    int n_slabs;
    int row_tiles;  // 128-row tiles per chunk: CP / 128
    int neg_tiles;  // n_pad / 256 (SCORES) ; n_pad / 128 (DN)
    int kchunks;    // SCORES: KPW / 64; DA: n_pad / 64; DN: rows per split chunk / 64 (last may be shorter)
    int dn_split, dn_rows64;  // DN: split-K chunks, 64-row groups per chunk
    int items;
    float inv_b;
    const float* fpos;
    const float* scale;  // [2][b_cap] 1 / (Z b), by packed row
    float* zpart;        // [n_pad/256][2][b_cap]
    uint16_t* Ppk;       // P~ packed [2][2 NBP][b_cap][8]
    float* dA;           // column-blocked [2][d/4][b_cap] float4
    float* dN_part;      // column-blocked [dn_split][2][d/4][n_pad] float4
};

struct WItem {
    int side, m0, n0, k0, nk;  // M offset (rows or negatives), N offset (negatives or columns), K range (chunks)
    int chunk;                 // DN: split-K chunk
    int q;                     // negative set (model chunk)
};

// Packed row pr of the A / P~ operands -> batch row (or -1 for padding).
__device__ __forceinline__ int batch_row(const WideArgs& g, int pr) {
    const int q = pr / g.CP, r = pr - q * g.CP;
    const int e = q * g.cr + r;
    return (r < g.cr && e < g.nb) ? e : -1;
}

template <int PASS>
__device__ __forceinline__ WItem witem(const WideArgs& g, int item) {
    WItem w{};
    if (PASS == PASS_SCORES) {  // (side, chunk, row tile, negative tile)
        const int per = g.row_tiles * g.neg_tiles;
        w.side = item / (per * g.chunks);
        w.q = (item / per) % g.chunks;
        const int r = item % per;
        w.m0 = w.q * g.CP + (r / g.neg_tiles) * WM;
        w.n0 = (r % g.neg_tiles) * WNEG;
        w.k0 = 0;
        w.nk = g.kchunks;
    } else if (PASS == PASS_DA) {  // (side, chunk, row tile, d-slab)
        const int per = g.row_tiles * g.n_slabs;
        w.side = item / (per * g.chunks);
        w.q = (item / per) % g.chunks;
        const int r = item % per;
        w.m0 = w.q * g.CP + (r / g.n_slabs) * WM;
        w.n0 = (r % g.n_slabs) * g.slab;
        w.k0 = 0;
        w.nk = g.kchunks;
    } else {  // (side, chunk, negative tile, d-slab, row chunk)
        const int per = g.neg_tiles * g.n_slabs * g.dn_split;
        w.side = item / (per * g.chunks);
        w.q = (item / per) % g.chunks;
        int r = item % per;
        w.chunk = r % g.dn_split;
        r /= g.dn_split;
        w.m0 = (r / g.n_slabs) * WM;
        w.n0 = (r % g.n_slabs) * g.slab;
        const int total64 = 2 * g.row_tiles;  // the chunk's 64-row groups (SCORES wrote zeros past its rows)
        w.k0 = w.q * (g.CP / 64) + w.chunk * g.dn_rows64;
        w.nk = min(g.dn_rows64, total64 - w.chunk * g.dn_rows64);  // >= 1: dn_split leaves no chunk empty
    }
    return w;
}

__host__ __device__ constexpr uint32_t stage_bytes_w() { return 2u * (WM * WKC * 2) + 2u * (WNEG * WKC * 2); }

template <int PASS>
__global__ void __launch_bounds__(WTHREADS, 1)
    k_wide(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, WideArgs g) {
    extern __shared__ __align__(128) uint8_t wsm_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(wsm_raw) + 127) & ~uintptr_t(127));
    const uint32_t SB = stage_bytes_w();
    uint64_t* bars = reinterpret_cast<uint64_t*>(base + WSTAGES * SB);
    uint64_t* full = bars;                 // [WSTAGES]
    uint64_t* empty = bars + WSTAGES;      // [WSTAGES]
    uint64_t* acc_full = bars + 2 * WSTAGES;   // [2]
    uint64_t* acc_empty = bars + 2 * WSTAGES + 2;  // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * WSTAGES + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NT = PASS == PASS_SCORES ? WNEG : g.slab;  // MMA N of this pass
    // operand tile bytes per stage (hi and lo halves back to back)
    const uint32_t a_half = WM * WKC * 2;                   // 128 x 64 bf16
    const uint32_t b_half = (uint32_t)NT * WKC * 2;         // NT x 64 bf16
    if (threadIdx.x == 0) {
        for (int i = 0; i < WSTAGES; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&acc_full[i], 1);
            tc::mbar_init(&acc_empty[i], 128);
        }
        tc::fence_mbar_init();
        tc::tmap_prefetch(&mapA);
        tc::tmap_prefetch(&mapB);
    }
    if (warp == 1) tc::tmem_alloc(tslot, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = *tslot;
    griddep_wait();

    if (warp == 0) {
        if (lane == 0) {  // ------------------------------------------------------------ TMA producer
            uint32_t gk = 0;
            for (int item = blockIdx.x; item < g.items; item += gridDim.x) {
                const WItem w = witem<PASS>(g, item);
                for (int kc = 0; kc < w.nk; ++kc, ++gk) {
                    const int st = gk % WSTAGES;
                    tc::mbar_wait(&empty[st], ((gk / WSTAGES) & 1) ^ 1);
                    tc::mbar_expect_tx(&full[st], 2 * a_half + 2 * b_half);
                    uint8_t* sa = base + st * SB;
                    uint8_t* sb = sa + 2 * a_half;
                    const int k = w.k0 + kc;
                    if (PASS == PASS_SCORES) {
                        // A: K-major rows m0.., column blocks 8k..8k+7 (hi) and CBA + .. (lo)
                        tc::tma_load_4d(sa, &mapA, 0, w.m0 / 32, 8 * k, w.side, &full[st]);
                        tc::tma_load_4d(sa + a_half, &mapA, 0, w.m0 / 32, g.CBA + 8 * k, w.side, &full[st]);
                        // N: K-major negatives n0..n0+255 of set q
                        const int nr = (w.q * g.n_pad + w.n0) / 32;
                        tc::tma_load_4d(sb, &mapB, 0, nr, 8 * k, w.side, &full[st]);
                        tc::tma_load_4d(sb + b_half, &mapB, 0, nr, g.CBA + 8 * k, w.side, &full[st]);
                    } else if (PASS == PASS_DA) {
                        // P~: K-major (K = negatives 64k..), rows m0..
                        tc::tma_load_4d(sa, &mapA, 0, w.m0 / 32, 8 * k, w.side, &full[st]);
                        tc::tma_load_4d(sa + a_half, &mapA, 0, w.m0 / 32, g.NBP + 8 * k, w.side, &full[st]);
                        // N: MN-major, K = negatives 64k.. of set q (rows of N), N = columns n0.. (blocks n0/8..)
                        const int nr = (w.q * g.n_pad) / 32 + 2 * k;
                        tc::tma_load_4d(sb, &mapB, 0, nr, w.n0 / 8, w.side, &full[st]);
                        tc::tma_load_4d(sb + b_half, &mapB, 0, nr, g.CBA + w.n0 / 8, w.side, &full[st]);
                    } else {
                        // P~: MN-major, M = negatives m0.. (blocks m0/8..), K = batch rows 64k..
                        tc::tma_load_4d(sa, &mapA, 0, 2 * k, w.m0 / 8, w.side, &full[st]);
                        tc::tma_load_4d(sa + a_half, &mapA, 0, 2 * k, g.NBP + w.m0 / 8, w.side, &full[st]);
                        // A': MN-major, K = batch rows 64k.., N = columns n0..
                        tc::tma_load_4d(sb, &mapB, 0, 2 * k, w.n0 / 8, w.side, &full[st]);
                        tc::tma_load_4d(sb + b_half, &mapB, 0, 2 * k, g.CBA + w.n0 / 8, w.side, &full[st]);
                    }
                }
            }
        }
    } else if (warp == 1) {  // ---------------------------------------------------------- MMA issuer
        // K-major tiles: [8 blocks][R rows][16 B] (k-step s = blocks 2s, 2s+1); MN-major tiles:
        // [blocks][64 rows][16 B] (k-step s = rows 16s..16s+15).
        const uint32_t idesc = tc::idesc_bf16(WM, (uint32_t)NT, PASS == PASS_DN, PASS != PASS_SCORES);
        uint32_t gk = 0, it = 0;
        for (int item = blockIdx.x; item < g.items; item += gridDim.x, ++it) {
            const WItem w = witem<PASS>(g, item);
            const uint32_t buf = it & 1;
            tc::mbar_wait_warp(&acc_empty[buf], ((it >> 1) & 1) ^ 1);
            tc::fence_after();
            const uint32_t acc = tbase + buf * 256;
            for (int kc = 0; kc < w.nk; ++kc, ++gk) {
                const int st = gk % WSTAGES;
                tc::mbar_wait_warp(&full[st], (gk / WSTAGES) & 1);
                tc::fence_after();
                const uint32_t sa = tc::smem_addr(base + st * SB), sb = sa + 2 * a_half;
#pragma unroll
                for (int s = 0; s < WKC / 16; ++s) {
                    uint64_t ah, al, bh, bl;
                    if (PASS == PASS_DN) {  // A MN-major: [16 blocks][64 rows][16 B]
                        ah = tc::sdesc(sa + s * 256, 128, WKC * 16);
                    } else {  // A K-major: [8 blocks][128 rows][16 B]
                        ah = tc::sdesc(sa + 2 * s * WM * 16, WM * 16, 128);
                    }
                    al = ah + (a_half >> 4);
                    if (PASS == PASS_SCORES) {  // B K-major: [8 blocks][256 rows][16 B]
                        bh = tc::sdesc(sb + 2 * s * WNEG * 16, WNEG * 16, 128);
                    } else {  // B MN-major: [NT/8 blocks][64 rows][16 B]
                        bh = tc::sdesc(sb + s * 256, 128, WKC * 16);
                    }
                    bl = bh + (b_half >> 4);
                    const uint32_t first = (kc == 0 && s == 0) ? 0u : 1u;
                    tc::mma_ss_elect(acc, al, bh, idesc, first);
                    tc::mma_ss_elect(acc, ah, bl, idesc, 1u);
                    tc::mma_ss_elect(acc, ah, bh, idesc, 1u);
                }
                tc::mma_commit_elect(&empty[st]);
            }
            tc::mma_commit_elect(&acc_full[buf]);
        }
    } else {  // ------------------------------------------------------------------------- epilogue
        const int qd = warp & 3;
        const int lr = 32 * qd + lane;  // TMEM lane = output tile row
        uint32_t it = 0;
        for (int item = blockIdx.x; item < g.items; item += gridDim.x, ++it) {
            const WItem w = witem<PASS>(g, item);
            const uint32_t buf = it & 1;
            tc::mbar_wait(&acc_full[buf], (it >> 1) & 1);
            tc::fence_after();
            const uint32_t t_row = tbase + ((uint32_t)(32 * qd) << 16) + buf * 256;
            const int row = w.m0 + lr;  // packed row (SCORES, DA) or negative (DN)
            if (PASS == PASS_SCORES) {
                const int e = batch_row(g, row);
                const bool live = e >= 0;
                const float shift = live ? -g.fpos[e] * WL2E : 0.f;
                float z = 0.f;
                uint4* ph = reinterpret_cast<uint4*>(g.Ppk) + ((size_t)w.side * 2 * g.NBP) * g.b_cap + row;
                uint4* pl = ph + (size_t)g.NBP * g.b_cap;
                for (int c0 = 0; c0 < WNEG; c0 += 32) {
                    uint32_t v[32];
                    tc::tmem_ld32(t_row + c0, v);
                    tc::tmem_ld_wait();
                    float p[32];
#pragma unroll
                    for (int c = 0; c < 32; ++c) {
                        const int k = w.n0 + c0 + c;
                        p[c] = (live && k < g.nt) ? tc::ex2(fmaf(__uint_as_float(v[c]), WL2E, shift)) : 0.f;
                        z += p[c];
                    }
#pragma unroll
                    for (int b8 = 0; b8 < 4; ++b8) {
                        float x[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) x[i] = p[8 * b8 + i];
                        uint4 hi, lo;
                        tc::split8(x, hi, lo);
                        const size_t blk = (size_t)(w.n0 + c0) / 8 + b8;
                        ph[blk * g.b_cap] = hi;
                        pl[blk * g.b_cap] = lo;
                    }
                }
                g.zpart[((size_t)(w.n0 / WNEG) * 2 + w.side) * g.b_cap + row] = z;
            } else {
                float sc = 1.f;
                float4* out;
                size_t cstride;
                bool ok = true;
                if (PASS == PASS_DA) {  // dA by batch row, column-blocked [side][d/4][b_cap]
                    const int e = batch_row(g, row);
                    ok = e >= 0;
                    sc = ok ? g.scale[(size_t)w.side * g.b_cap + row] : 0.f;
                    out = reinterpret_cast<float4*>(g.dA) + (size_t)w.side * (g.d / 4) * g.b_cap + (ok ? e : 0);
                    cstride = (size_t)g.b_cap;
                } else {  // dN partial of negative set (q, side): [split][2 chunks][d/4][n_pad]
                    out = reinterpret_cast<float4*>(g.dN_part) +
                          (((size_t)w.chunk * g.chunks + w.q) * 2 + w.side) * (g.d / 4) * g.n_pad + row;
                    cstride = (size_t)g.n_pad;
                }
                for (int c0 = 0; c0 < NT; c0 += 16) {
                    uint32_t v[16];
                    tc::tmem_ld16(t_row + c0, v);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; j += 4) {
                        const int c = w.n0 + c0 + j;
                        if (ok && c < g.d)
                            out[(size_t)(c / 4) * cstride] =
                                make_float4(__uint_as_float(v[j]) * sc, __uint_as_float(v[j + 1]) * sc,
                                            __uint_as_float(v[j + 2]) * sc, __uint_as_float(v[j + 3]) * sc);
                    }
                }
            }
            tc::fence_before();
            tc::mbar_arrive(&acc_empty[buf]);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tbase, 512);
}

// fp32 rows -> packed bf16 hi|lo [2][2 CBA][cap][8], zero padding for unused rows and columns >= d.
// Packed row pr of side s holds, for the batch operand (nt == 0), batch row e of chunk q = pr / CP
// (x: [2][nb][d], scale (nullable): per (side, packed row) factor applied first); for the negatives
// (nt > 0), negative k = pr % CP of set q = pr / CP (x: [chunks][2][nt][d], CP = the padded set size).
// Thread per (side, block, row): 8 columns, one 16-byte store each for hi and lo, coalesced along rows.
__global__ void k_pack_rows(const float* __restrict__ x, int nb, int nt, int cr, int CP, int d, int CBA, int cap,
                            int chunks, const float* __restrict__ scale, uint16_t* __restrict__ out) {
    griddep_wait();
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t total = (size_t)2 * CBA * cap;
    if (t >= total) return;
    const int pr = (int)(t % cap);
    const int blk = (int)((t / cap) % CBA);
    const int side = (int)(t / ((size_t)cap * CBA));
    const int q = pr / CP, r = pr - q * CP;
    const float* src = nullptr;
    if (q < chunks) {
        if (nt == 0) {
            const int e = q * cr + r;
            if (r < cr && e < nb) src = x + ((size_t)side * nb + e) * d;
        } else if (r < nt) {
            src = x + (((size_t)q * 2 + side) * nt + r) * d;
        }
    }
    const float s = src ? (scale ? scale[(size_t)side * cap + pr] : 1.f) : 0.f;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int c = 8 * blk + i;
        v[i] = (src && c < d) ? src[c] * s : 0.f;
    }
    uint4 hi, lo;
    tc::split8(v, hi, lo);
    uint4* o = reinterpret_cast<uint4*>(out) + ((size_t)side * 2 * CBA + blk) * cap + pr;
    o[0] = hi;
    o[(size_t)CBA * cap] = lo;
}

// A' = A / (Z b) in the packed layout, from the packed A itself (x = hi + lo, scaled, split again):
// thread per (side, block, packed row), reads and writes coalesced along rows. Rows without an
// edge have scale 0.
__global__ void k_repack_scaled(const uint16_t* __restrict__ in, int CBA, int cap, const float* __restrict__ scale,
                                uint16_t* __restrict__ out) {
    griddep_wait();
    const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t total = (size_t)2 * CBA * cap;
    if (t >= total) return;
    const int pr = (int)(t % cap);
    const int blk = (int)((t / cap) % CBA);
    const int side = (int)(t / ((size_t)cap * CBA));
    const uint4* I = reinterpret_cast<const uint4*>(in) + ((size_t)side * 2 * CBA + blk) * cap + pr;
    const uint4 h = I[0], l = I[(size_t)CBA * cap];
    const float s = scale[(size_t)side * cap + pr];
    const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[4] = {l.x, l.y, l.z, l.w};
    float v[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hw[i]));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&lw[i]));
        v[2 * i] = (a.x + b.x) * s;
        v[2 * i + 1] = (a.y + b.y) * s;
    }
    uint4 hi, lo;
    tc::split8(v, hi, lo);
    uint4* o = reinterpret_cast<uint4*>(out) + ((size_t)side * 2 * CBA + blk) * cap + pr;
    o[0] = hi;
    o[(size_t)CBA * cap] = lo;
}

// Row statistics after SCORES: Z = 1 + sum of the tiles' partial sums (fixed order), lse, g0, the
// dA / A' row scale 1/(Z b); rows whose Z left the safe range are listed for k_wide_fixup.
__global__ void k_wide_stats(const float* __restrict__ zpart, int ntiles, int nb, int cr, int CP, int b_cap, float inv_b,
                             float zmax, const float* __restrict__ fpos, float* lse, float* g0, float* scale,
                             uint32_t* flags) {
    griddep_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * b_cap) return;
    const int side = i / b_cap, pr = i % b_cap;
    const int q = pr / CP, r = pr - q * CP, e = q * cr + r;
    if (r >= cr || e >= nb) {
        scale[i] = 0.f;
        return;
    }
    float z = 1.0f;  // exp(f_pos - f_pos): the positive
    for (int j = 0; j < ntiles; ++j) z += zpart[((size_t)j * 2 + side) * b_cap + pr];
    const float f = fpos[e];
    const float l = f + __logf(z);
    lse[(size_t)side * nb + e] = l;
    g0[(size_t)side * nb + e] = (__expf(f - l) - 1.0f) * inv_b;
    scale[i] = inv_b / z;
    if (!(z < zmax)) flags[1 + atomicAdd(flags, 1u)] = (uint32_t)i;
}

// Exact recompute (fp32, CUDA cores, two passes with the row maximum) of the rows k_wide_stats
// flagged: normalised P written over the row's P~ with row scale 1/b, lse and g0 rewritten. One warp
// per flagged row; the operands as the tensor cores saw them (hi + lo).
__device__ __forceinline__ float wpacked(const uint16_t* pk, int cap, int CBA, int side, int row, int c) {
    const size_t hi = (((size_t)side * 2 * CBA + c / 8) * cap + row) * 8 + c % 8;
    const size_t lo = hi + (size_t)CBA * cap * 8;
    return __bfloat162float(__ushort_as_bfloat16(pk[hi])) + __bfloat162float(__ushort_as_bfloat16(pk[lo]));
}

__global__ void k_wide_fixup(const uint32_t* flags, const uint16_t* __restrict__ Apk, const uint16_t* __restrict__ Npk,
                             int CBA, int b_cap, int n_pad, int n_cap, int NBP, int nb, int nt, int d, int cr, int CP,
                             float inv_b,
                             const float* __restrict__ fpos, float* lse, float* g0, float* scale, uint16_t* Ppk) {
    griddep_wait();
    const uint32_t n = *(volatile const uint32_t*)flags;
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t f = gw; f < n; f += nw) {
        const uint32_t code = flags[1 + f];
        const int side = (int)(code / b_cap), pr = (int)(code % b_cap);
        const int q = pr / CP, e = q * cr + (pr - q * CP);
        const int nrow0 = q * n_pad;  // the chunk's negatives in the packed N
        auto score = [&](int k) {
            float s = 0.f;
            for (int c = lane; c < d; c += 32)
                s += wpacked(Apk, b_cap, CBA, side, pr, c) * wpacked(Npk, n_cap, CBA, side, nrow0 + k, c);
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            return s;
        };
        const float fp = fpos[e];
        float mx = fp;
        for (int k = 0; k < nt; ++k) mx = fmaxf(mx, score(k));
        float z = expf(fp - mx);
        for (int k = 0; k < nt; ++k) z += expf(score(k) - mx);
        const float l = mx + logf(z);
        uint16_t* ph = Ppk + ((size_t)side * 2 * NBP) * b_cap * 8;
        for (int k = 0; k < nt; ++k) {
            const float p = expf(score(k) - l);
            if (lane == 0) {
                const __nv_bfloat16 h = __float2bfloat16_rn(p);
                const __nv_bfloat16 lo = __float2bfloat16_rn(p - __bfloat162float(h));
                const size_t at = ((size_t)(k / 8) * b_cap + pr) * 8 + k % 8;
                ph[at] = __bfloat16_as_ushort(h);
                ph[at + (size_t)NBP * b_cap * 8] = __bfloat16_as_ushort(lo);
            }
        }
        if (lane == 0) {
            lse[(size_t)side * nb + e] = l;
            g0[(size_t)side * nb + e] = (expf(fp - l) - 1.0f) * inv_b;
            scale[(size_t)side * b_cap + pr] = inv_b;
        }
    }
}

}  // namespace

// Wide-engine state (allocated once per context; d > 128 or num_chunks > 1).
struct WideState {
    int KPW = 0, CBA = 0, chunks = 1, CP = 0, b_cap = 0, n_pad = 0, n_cap = 0, NBP = 0, slab = 0, n_slabs = 0;
    int dn_split = 1;
    uint16_t *Apk = nullptr, *Npk = nullptr, *Ascaled = nullptr, *Ppk = nullptr;
    float *zpart = nullptr, *scale = nullptr, *dN_part = nullptr;
    uint32_t* flags = nullptr;
    unsigned long long* flags_total = nullptr;
    float zmax = 1e30f;
    int max_grid = 0;  // test hook (EMBER_TC_MAXGRID): several items per CTA
    CUtensorMap mA_k, mN_k, mP_k, mN_mn, mP_mn, mAs_mn;
};

bool wide_supported(const Engine& E) { return (E.dim > 128 || E.chunks > 1) && E.dim % 4 == 0 && E.nt >= 1; }

void wide_setup(Engine& E) {
    auto* w = new WideState();
    w->KPW = (int)((E.dim + WKC - 1) / WKC * WKC);
    w->CBA = w->KPW / 8;
    w->chunks = (int)E.chunks;
    const int cr_max = (int)((E.cap_b + E.chunks - 1) / E.chunks);
    w->CP = (cr_max + WM - 1) / WM * WM;  // each chunk's rows padded to whole 128-row tiles
    w->b_cap = w->chunks * w->CP;
    w->n_pad = (int)((E.nt + WNEG - 1) / WNEG * WNEG);
    w->n_cap = w->chunks * w->n_pad;
    w->NBP = w->n_pad / 8;
    // d-slabs of <= 256 columns (multiples of 16) covering the padded width
    w->n_slabs = (w->KPW + 255) / 256;
    w->slab = (w->KPW / w->n_slabs + 15) / 16 * 16;
    while (w->slab * w->n_slabs < (int)E.dim) w->slab += 16;
    const int neg128 = w->n_pad / WM;
    w->dn_split = std::max(1, (E.sm_count * 4) / (2 * w->chunks * neg128 * w->n_slabs));
    if (const char* s = getenv("EMBER_TC_ZMAX")) w->zmax = (float)atof(s);  // test hook: 0 flags every row
    if (const char* s = getenv("EMBER_TC_MAXGRID")) w->max_grid = atoi(s);
    const size_t d = E.dim;
    auto alloc = [&](size_t bytes) {
        void* p = nullptr;
        EMBER_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
        return p;
    };
    w->Apk = static_cast<uint16_t*>(alloc((size_t)2 * 2 * w->CBA * w->b_cap * 16));
    w->Ascaled = static_cast<uint16_t*>(alloc((size_t)2 * 2 * w->CBA * w->b_cap * 16));
    w->Npk = static_cast<uint16_t*>(alloc((size_t)2 * 2 * w->CBA * w->n_cap * 16));
    w->Ppk = static_cast<uint16_t*>(alloc((size_t)2 * 2 * w->NBP * w->b_cap * 16));
    w->zpart = static_cast<float*>(alloc((size_t)(w->n_pad / WNEG) * 2 * w->b_cap * 4));
    w->scale = static_cast<float*>(alloc((size_t)2 * w->b_cap * 4));
    w->dN_part = static_cast<float*>(alloc((size_t)w->dn_split * w->chunks * 2 * w->n_pad * d * 4));
    w->flags = static_cast<uint32_t*>(alloc((size_t)(1 + 2 * w->b_cap) * 4));
    EMBER_CUDA(cudaMemset(w->flags, 0, 4));
    w->flags_total = static_cast<unsigned long long*>(alloc(8));
    EMBER_CUDA(cudaMemset(w->flags_total, 0, 8));
    // K-major boxes (128 or 256 rows x 8 blocks) and MN-major boxes (64 rows x slab/8 or 16 blocks)
    w->mA_k = make_packed_map(w->Apk, w->b_cap, 2 * w->CBA, WM, 8);
    w->mN_k = make_packed_map(w->Npk, w->n_cap, 2 * w->CBA, WNEG, 8);
    w->mP_k = make_packed_map(w->Ppk, w->b_cap, 2 * w->NBP, WM, 8);
    w->mN_mn = make_packed_map(w->Npk, w->n_cap, 2 * w->CBA, WKC, w->slab / 8);
    w->mP_mn = make_packed_map(w->Ppk, w->b_cap, 2 * w->NBP, WKC, WM / 8);
    w->mAs_mn = make_packed_map(w->Ascaled, w->b_cap, 2 * w->CBA, WKC, w->slab / 8);
    const int smem = (int)(WSTAGES * stage_bytes_w() + 256 + 128);
    EMBER_CUDA(cudaFuncSetAttribute(k_wide<PASS_SCORES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    EMBER_CUDA(cudaFuncSetAttribute(k_wide<PASS_DA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    EMBER_CUDA(cudaFuncSetAttribute(k_wide<PASS_DN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    // dA (by batch row, column-blocked with stride b_cap: the chain rule's dcap)
    EMBER_CUDA(cudaFree(E.s.dA));
    E.s.dA = static_cast<float*>(alloc((size_t)2 * w->b_cap * d * 4));
    E.b_cap = w->b_cap;
    E.wide = w;
}

void wide_release(Engine& E) {
    WideState* w = E.wide;
    if (!w) return;
    for (void* p : {(void*)w->Apk, (void*)w->Ascaled, (void*)w->Npk, (void*)w->Ppk, (void*)w->zpart, (void*)w->scale,
                    (void*)w->dN_part, (void*)w->flags, (void*)w->flags_total})
        if (p) cudaFree(p);
    delete w;
    E.wide = nullptr;
}

uint64_t wide_overflow_rows(Engine& E) {
    if (!E.wide) return 0;
    unsigned long long v = 0;
    EMBER_CUDA(cudaStreamSynchronize(E.stream));
    EMBER_CUDA(cudaMemcpy(&v, E.wide->flags_total, sizeof(v), cudaMemcpyDeviceToHost));
    return v;
}

void dn_reduce_launch(Engine& E, const float* part, int chunks, int nt, int n_pad, int d, uint32_t slot0,
                      uint32_t* flags, unsigned long long* flags_total, int nsides);  // tc_score.cu

// The batch's rows gathered straight into the packed A (k_gather_pack_wide) and s.N [chunks][2][nt][d]
// (fp32, written by the negatives' gather) -> lse, g0, dA, sorted dN rows.
void launch_contract_wide(Engine& E, uint32_t nb, const uint32_t* edges, const PartView& pi, const PartView& pj) {
    WideState& w = *E.wide;
    Scratch& s = E.s;
    const int d = (int)E.dim, nt = (int)E.nt;
    WideArgs a{};
    a.nb = (int)nb;
    a.nt = nt;
    a.d = d;
    a.chunks = w.chunks;
    a.cr = (int)((nb + w.chunks - 1) / w.chunks);
    a.CP = w.CP;
    a.CBA = w.CBA;
    a.NBP = w.NBP;
    a.b_cap = w.b_cap;
    a.n_pad = w.n_pad;
    a.slab = w.slab;
    a.n_slabs = w.n_slabs;
    a.row_tiles = (a.cr + WM - 1) / WM;
    a.inv_b = 1.0f / (float)nb;
    a.fpos = s.fpos;
    a.scale = w.scale;
    a.zpart = w.zpart;
    a.Ppk = w.Ppk;
    a.dA = s.dA;
    a.dN_part = w.dN_part;
    const int smem = (int)(WSTAGES * stage_bytes_w() + 256 + 128);
    const int sms = w.max_grid > 0 ? std::min(w.max_grid, E.sm_count) : E.sm_count;
    const size_t tA = (size_t)2 * w.CBA * w.b_cap, tN = (size_t)2 * w.CBA * w.n_cap;
    // operands packed into the tensor-core layout (chunk q's rows / negatives at packed row q CP / q n_pad)
    launch_gather_pack_wide(E, edges, nb, pi, pj, w.Apk, (uint32_t)w.CBA, (uint32_t)w.b_cap, (uint32_t)w.CP,
                            (uint32_t)a.cr);
    launch_pdl(k_pack_rows, dim3((unsigned)((tN + 255) / 256)), dim3(256), 0, E.stream, (const float*)s.N, (int)nb, nt,
               a.cr, w.n_pad, d, w.CBA, w.n_cap, w.chunks, (const float*)nullptr, w.Npk);
    EMBER_LAUNCHED(E);
    // 1) scores -> P~, partial row sums
    a.neg_tiles = w.n_pad / WNEG;
    a.kchunks = w.KPW / WKC;
    a.items = 2 * w.chunks * a.row_tiles * a.neg_tiles;
    launch_pdl(k_wide<PASS_SCORES>, dim3(std::min(a.items, sms)), dim3(WTHREADS), smem, E.stream, w.mA_k, w.mN_k, a);
    EMBER_LAUNCHED(E);
    // row statistics, exact recompute of overflowed rows, A' = A / (Z b)
    launch_pdl(k_wide_stats, dim3((unsigned)((2 * w.b_cap + 255) / 256)), dim3(256), 0, E.stream, (const float*)w.zpart,
               a.neg_tiles, (int)nb, a.cr, w.CP, w.b_cap, a.inv_b, w.zmax, (const float*)s.fpos, s.lse, s.g0, w.scale,
               w.flags);
    EMBER_LAUNCHED(E);
    launch_pdl(k_wide_fixup, dim3(E.sm_count), dim3(256), 0, E.stream, (const uint32_t*)w.flags, (const uint16_t*)w.Apk,
               (const uint16_t*)w.Npk, w.CBA, w.b_cap, w.n_pad, w.n_cap, w.NBP, (int)nb, nt, d, a.cr, w.CP, a.inv_b,
               (const float*)s.fpos, s.lse, s.g0, w.scale, w.Ppk);
    EMBER_LAUNCHED(E);
    launch_pdl(k_repack_scaled, dim3((unsigned)((tA + 255) / 256)), dim3(256), 0, E.stream, (const uint16_t*)w.Apk,
               w.CBA, w.b_cap, (const float*)w.scale, w.Ascaled);
    EMBER_LAUNCHED(E);
    // 2) dA = P~ N / (Z b)
    a.kchunks = w.n_pad / WKC;
    a.items = 2 * w.chunks * a.row_tiles * w.n_slabs;
    launch_pdl(k_wide<PASS_DA>, dim3(std::min(a.items, sms)), dim3(WTHREADS), smem, E.stream, w.mP_k, w.mN_mn, a);
    EMBER_LAUNCHED(E);
    // 3) dN partials = P~^T A' over row chunks of each negative set's rows
    a.neg_tiles = w.n_pad / WM;
    const int rows64 = 2 * a.row_tiles;
    const int split = std::min(w.dn_split, rows64);
    a.dn_rows64 = (rows64 + split - 1) / split;
    a.dn_split = (rows64 + a.dn_rows64 - 1) / a.dn_rows64;  // every chunk holds >= 1 row group
    a.items = 2 * w.chunks * a.neg_tiles * w.n_slabs * a.dn_split;
    launch_pdl(k_wide<PASS_DN>, dim3(std::min(a.items, sms)), dim3(WTHREADS), smem, E.stream, w.mP_mn, w.mAs_mn, a);
    EMBER_LAUNCHED(E);
    E.join_sorted();
    dn_reduce_launch(E, w.dN_part, a.dn_split, nt, w.n_pad, d, 2 * nb, w.flags, w.flags_total, 2 * w.chunks);
}

}  // namespace ember
