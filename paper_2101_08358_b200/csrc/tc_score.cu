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
// Operand layout in HBM (written by k_pack): per side, [2*CB column blocks][rows][8 bf16],
// CB = KP/8 (KP = dim rounded up to 16), hi blocks then lo blocks. A 128-row range is one TMA box
// that lands in shared memory as the canonical no-swizzle K-major UMMA tile [cb][128][16 B]
// (tc_common.cuh); the same bytes are the MN-major operand of the transposed product.
//
// One kernel template, two modes, per side (A = adjusted vectors [nb x d], N = shared
// negatives [nt x d], b = nb):
//   MODE_ROWS  item = 128-row tile of A (resident), streamed over 128-negative tiles of N:
//              S = A N^T, P = exp(S - f_pos) (the positive's score is the fixed row shift: it
//              is part of every row's log-sum-exp, so no online rescaling is needed), dA += P N.
//              Item end: lse = f_pos + log(1 + sum P), g0 = (exp(f_pos - lse) - 1)/b, dA/(Z b).
//              Rows whose sum overflows the safe range are listed and recomputed exactly by
//              by the dN kernel's CTAs (tc_fixup_rows) before anything reads lse.
//   MODE_NEGS  item = 128-negative tile of N (resident) x a chunk of 128-row tiles of A:
//              S^T = N A^T, P^T = exp(S^T - lse)/b, dN += P^T A; per-chunk partials are summed
//              in a fixed order by the dN reduction (k_dn_reduce / the chain rule's prologue).
// TMEM (512 columns): [0,128) and [128,256) two S buffers of 128 fp32 columns, each overwritten
// in place by P as bf16 pairs (per 32-column chunk: 16 hi columns then 16 lo columns) — the A
// operand of the second product (TS mode); [256,256+KP) the accumulator; [384,384+KP) the
// resident operand (hi|lo pairs), copied smem -> TMEM by tcgen05.cp in the MMA pipe, so every
// MMA reads only its B operand from shared memory.
// Warps: 0 = TMA producer, 1 = S issuer (+ TMEM owner, R staging), 2 = P.T issuer (whole warps
// converged, one elected lane issues), 3..10 = two epilogue warpgroups that take alternate
// streamed tiles (ping-pong).
//
// MMA ordering: tcgen05.mma / tcgen05.cp from one thread execute in issue order, which the
// kernel relies on for the two write-after-read reuses of TMEM: S_{k+2} overwrites the buffer
// that P_k.T_k read, and the next item's tcgen05.cp overwrites the resident operand that this
// item's last S read (the same convention as CUTLASS's sm100 FMHA S/P aliasing).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "engine.h"
#include "tc_common.cuh"

namespace ember {
namespace {

enum { MODE_ROWS = 0, MODE_NEGS = 1 };
constexpr int RES = 128;       // resident rows per item (MMA M)
constexpr int TILE = 96;       // streamed rows per tile (first product's N, second product's K)
constexpr int NSTAGE_MAX = 5;  // streamed-tile ring depth (as many as fit in shared memory, + the resident buffer)
constexpr int KPMAX = 128;     // largest padded dim
constexpr int NTHREADS = 352;  // producer, S issuer, P.T issuer, 2 x 4 epilogue warps
constexpr uint32_t TCOLS = 512;
constexpr int NSP_MAX = 4;     // S/P buffers: (512 - 2 KP) / TILE of them fit next to acc and R
constexpr float L2E = 1.4426950408889634f;

struct TcArgs {
    int KP, CB, d, nb, nt, n_pad, b_cap, chunks2, nstage, nsp;
    // res_stage: every CTA runs one item, so once its resident tile is in TMEM the resident buffer
    // serves as one more ring stage (the dN kernel: its ring depth is what limits its tile period)
    int res_stage;
    int rows128, rows_pad;  // batch rows covered by the 128-row items / by the packed padding
    float inv_b, log2_inv_b, zmax;
    const float* fpos;
    float* lse;       // [2][nb]
    float* lse_pad;   // [2][b_cap]: log2(1/b) - lse*log2(e), -inf past nb
    float* g0;        // [2][nb]
    float* dA;        // column-blocked [2][d/4][b_cap] float4
    float* dN_part;   // column-blocked [chunks][2][d/4][n_pad] float4
    uint32_t* flags;  // [0] = count, [1..] = side * b_cap + row
    int early;        // tiles 0 .. early-1 of an item go to epilogue group 0 (tile_group)
    int l2_keep;      // dA stored with an L2 evict_last policy: the chain rule reads it back after the
                      // dN kernel has streamed the packed operands through L2 (EMBER_DA_L2=0: plain stores)
    int diag;         // EMBER_TC_DIAG=1 (measurement only, wrong results): the epilogue skips its TMEM work
    unsigned long long* trace;  // debug timeline of CTA 0 (EMBER_TC_TRACE), nullptr normally
    unsigned long long* cta_times;  // EMBER_TC_CTATIMES: per CTA (start, end) %globaltimer ns, nullptr normally
    // Items go to CTAs in arrival order, not blockIdx order: a CTA that becomes resident late (its SM
    // was still running a helper-stream kernel) takes the last of the grid-stride item sequences,
    // which are the shorter ones when the items do not divide evenly. rank = atomicAdd - base.
    uint32_t* arrive;
    uint32_t arrive_base;
    // dyn: after its first item a CTA claims the next from a counter (claim - claim_base + grid), so
    // SMs that run faster take more items; the producer publishes each work's item to the other roles.
    int dyn;
    uint32_t* claim;
    uint32_t claim_base;
    // MODE_NEGS: rows flagged by the rows kernel are recomputed exactly by the dN kernel's CTAs
    // before any reads their lse (all CTAs arrive on fix_bar; they wait only when a row is flagged)
    const uint16_t* Apk;
    const uint16_t* Npk;
    uint32_t* fix_bar;
    uint32_t fix_base;
};

// Debug timeline: (clock64, event << 32 | arg) records from CTA 0's producer, MMA issuer and one
// warp of each epilogue group, each role writing its own region with a register counter
// (fire-and-forget stores: no atomics on the issuing threads' critical path).
constexpr int TRACE_ROLE = 4096;  // records per role
#define TC_TRACE(ev, arg)                                                                              \
    do {                                                                                               \
        if (g.trace && blockIdx.x == 0 && lane == 0 && tr_n < TRACE_ROLE) {                            \
            unsigned long long* p_ = g.trace + 2 * ((size_t)tr_role * TRACE_ROLE + tr_n++);            \
            p_[0] = clock64();                                                                         \
            p_[1] = ((unsigned long long)(ev) << 32) | (uint32_t)(arg);                                \
        }                                                                                              \
    } while (0)

// ---- shared memory ------------------------------------------------------------------------
// [res: 128-row resident tile][ring: nstage x (TILE-row tile + lse trailer in MODE_NEGS)][zbuf][bars]
__host__ __device__ constexpr size_t res_bytes(int KP) { return (size_t)RES * KP * 4; }
__host__ __device__ constexpr size_t trailer_bytes(int mode) { return mode == MODE_NEGS ? TILE * 4 : 0; }
__host__ __device__ constexpr size_t stage_bytes(int KP, int mode) {
    return ((size_t)TILE * KP * 4 + trailer_bytes(mode) + 127) & ~size_t(127);
}
__host__ __device__ constexpr size_t zbuf_bytes(int mode) { return mode == MODE_ROWS ? 4 * RES * 4 : 0; }
__host__ __device__ constexpr size_t smem_total(int KP, int nstage, int mode) {
    return 128 + res_bytes(KP) + nstage * stage_bytes(KP, mode) + zbuf_bytes(mode) + 512;  // bars: 53 x 8 B
}
constexpr size_t SMEM_LIMIT = 232448;
inline int stages_for(int KP) {
    int n = NSTAGE_MAX;
    while (n > 2 && std::max(smem_total(KP, n, MODE_ROWS), smem_total(KP, n, MODE_NEGS)) > SMEM_LIMIT) --n;
    return n;
}

enum {
    B_RES_FULL = 0, B_RES_EMPTY = 1,
    B_RING_FULL = 2,                     // + NSTAGE_MAX
    B_RING_EMPTY = 2 + NSTAGE_MAX,       // + NSTAGE_MAX
    // Every barrier below has exactly one consumer that waits each of its phases in order, so a
    // waiter can never see a phase two completions ahead (mbarrier parity aliasing).
    B_S_FULL = 2 + 2 * NSTAGE_MAX,                   // + 2 * NSP_MAX: [epilogue group][S buffer]
    B_P_FULL = 2 + 2 * NSTAGE_MAX + 2 * NSP_MAX,     // + NSP_MAX (consumer: P.T issuer)
    B_PN_DONE = 2 + 2 * NSTAGE_MAX + 3 * NSP_MAX,    // + NSP_MAX: P.T of a buffer completed (S issuer)
    B_ACC_FULL = 2 + 2 * NSTAGE_MAX + 4 * NSP_MAX,   // consumer: epilogue group 1 (item tails)
    B_ACC_EMPTY = 3 + 2 * NSTAGE_MAX + 4 * NSP_MAX,  // consumer: P.T issuer
    B_Z_READY = 4 + 2 * NSTAGE_MAX + 4 * NSP_MAX,    // + 4: group 0's row sums of item i in zbuf[i % 4]
    B_ZB_FREE = 8 + 2 * NSTAGE_MAX + 4 * NSP_MAX,    // + 4: group 1 has read zbuf[i % 4]
    B_TMEM_SLOT = 12 + 2 * NSTAGE_MAX + 4 * NSP_MAX,  // [0] TMEM base, [1] arrival rank
    B_WORK = 13 + 2 * NSTAGE_MAX + 4 * NSP_MAX,       // + WORK_SLOTS: (work << 32 | item), by the producer
};
constexpr uint32_t WORK_SLOTS = 16;  // the producer runs at most ~3 works ahead of the slowest role

struct Smem {
    uint8_t* res;   // the item's resident tile (TMA landing zone, copied to TMEM by tcgen05.cp)
    uint8_t* ring;  // nstage x stage; a stage = tile [2CB][TILE][16 B] (+ TILE floats in MODE_NEGS)
    float* zbuf;    // [4 items][128]: group 0's partial row sums (MODE_ROWS)
    uint64_t* bars;
    uint32_t sbytes;
    int nring;  // stages in `ring`; stage nring (if used) is the resident buffer
    __device__ uint8_t* stage(int st) const { return st < nring ? ring + (size_t)st * sbytes : res; }
};

template <int MODE>
__device__ __forceinline__ Smem carve(uint8_t* raw, int KP, int nstage) {
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
    Smem s;
    s.sbytes = (uint32_t)stage_bytes(KP, MODE);
    s.res = base;
    s.ring = base + res_bytes(KP);
    s.nring = nstage;
    s.zbuf = reinterpret_cast<float*>(s.ring + (size_t)nstage * s.sbytes);
    s.bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(s.zbuf) + zbuf_bytes(MODE));
    return s;
}

// Descriptor of a canonical K-major tile [cb][R][16 B] at k-step s (16 elements = 2 blocks).
__device__ __forceinline__ uint64_t kdesc(const uint8_t* tile, int R, int s, int cb0) {
    return tc::sdesc(tc::smem_addr(tile) + (uint32_t)((cb0 + 2 * s) * R * 16), (uint32_t)(R * 16), 128u);
}
// The same bytes read as the MN-major operand of the transposed product: K = R rows.
__device__ __forceinline__ uint64_t mndesc(const uint8_t* tile, int R, int s, int cb0) {
    return tc::sdesc(tc::smem_addr(tile) + (uint32_t)(cb0 * R * 16 + s * 256), 128u, (uint32_t)(R * 16));
}


__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
    asm volatile(
        "{ .reg .pred e; elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.cp.cta_group::1.128x256b [%0], %1; }" ::"r"(taddr),
        "l"(sdesc)
        : "memory");
}

// ---- item geometry -------------------------------------------------------------------------
struct Item {
    int side, r0, t0, T, chunk, ntile;
};

template <int MODE>
__device__ __forceinline__ int n_items(const TcArgs& g) {
    if (MODE == MODE_ROWS) return 2 * ((g.nb + RES - 1) / RES);
    return 2 * ((g.nt + RES - 1) / RES) * g.chunks2;
}

template <int MODE>
__device__ __forceinline__ Item item_geo(const TcArgs& g, int item) {
    Item it;
    if (MODE == MODE_ROWS) {
        const int row_tiles = (g.nb + RES - 1) / RES;
        it.side = item / row_tiles;
        it.r0 = (item % row_tiles) * RES;
        it.t0 = 0;
        it.T = (g.nt + TILE - 1) / TILE;
        it.chunk = it.ntile = 0;
    } else {
        const int ntl = (g.nt + RES - 1) / RES, nsub = (g.nb + TILE - 1) / TILE;
        it.side = item / (ntl * g.chunks2);
        const int rem = item % (ntl * g.chunks2);
        it.ntile = rem / g.chunks2;
        it.chunk = rem % g.chunks2;
        const int u0 = (int)((long long)it.chunk * nsub / g.chunks2);
        it.T = (int)((long long)(it.chunk + 1) * nsub / g.chunks2) - u0;
        it.r0 = it.ntile * RES;
        it.t0 = u0 * TILE;
    }
    return it;
}

// Epilogue body for NC 32-column chunks of an S buffer starting at column c0: P = exp(...) in bf16
// hi|lo pairs written back in place (per 32-column chunk: 16 hi columns, then 16 lo columns).
template <int MODE, int NC>
__device__ __forceinline__ void epi_chunk(uint32_t tS, int c0, int k, const TcArgs& g, const Smem& sm, int st, int KP,
                                          float cshift, float& z) {
    float v[32 * NC];
    {
        uint32_t a[NC][32];
#pragma unroll
        for (int j = 0; j < NC; ++j) tc::tmem_ld32(tS + c0 + 32 * j, a[j]);
        tc::tmem_ld_wait();  // the registers are valid only after the wait
#pragma unroll
        for (int j = 0; j < NC; ++j)
#pragma unroll
            for (int i = 0; i < 32; ++i) v[32 * j + i] = __uint_as_float(a[j][i]);
    }
    if (MODE == MODE_ROWS) {
        const int k0 = k * TILE + c0;
        float zz[4] = {0.f, 0.f, 0.f, 0.f};  // 4 independent sums (latency)
        if (k0 + 32 * NC <= g.nt) {
#pragma unroll
            for (int c = 0; c < 32 * NC; ++c) {
                v[c] = tc::ex2(fmaf(v[c], L2E, cshift));
                zz[c & 3] += v[c];
            }
        } else {  // last tile: negatives past n_t contribute nothing
#pragma unroll
            for (int c = 0; c < 32 * NC; ++c) {
                v[c] = (k0 + c < g.nt) ? tc::ex2(fmaf(v[c], L2E, cshift)) : 0.f;
                zz[c & 3] += v[c];
            }
        }
        z += (zz[0] + zz[1]) + (zz[2] + zz[3]);
    } else {
        // per batch row: log2(1/b) - lse*log2(e) (k_tc<ROWS> stores it; -inf past the batch), from
        // the stage's trailer (TMA'd with the tile)
        const float4* L = reinterpret_cast<const float4*>(sm.stage(st) + TILE * KP * 4) + c0 / 4;
#pragma unroll
        for (int c4 = 0; c4 < 8 * NC; ++c4) {
            const float4 l = L[c4];  // broadcast read
            v[4 * c4 + 0] = tc::ex2(fmaf(v[4 * c4 + 0], L2E, l.x));
            v[4 * c4 + 1] = tc::ex2(fmaf(v[4 * c4 + 1], L2E, l.y));
            v[4 * c4 + 2] = tc::ex2(fmaf(v[4 * c4 + 2], L2E, l.z));
            v[4 * c4 + 3] = tc::ex2(fmaf(v[4 * c4 + 3], L2E, l.w));
        }
    }
#pragma unroll
    for (int cc = 0; cc < NC; ++cc) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float x0 = v[32 * cc + 2 * i], x1 = v[32 * cc + 2 * i + 1];
            const __nv_bfloat162 hh = __floats2bfloat162_rn(x0, x1);
            const float2 hf = __bfloat1622float2(hh);
            hi[i] = *reinterpret_cast<const uint32_t*>(&hh);
            lo[i] = tc::pack_bf16x2(x0 - hf.x, x1 - hf.y);
        }
        tc::tmem_st16(tS + c0 + 32 * cc, hi);  // P overwrites S in place
        tc::tmem_st16(tS + c0 + 32 * cc + 16, lo);
    }
}

// The item of work `it` (published by the producer; items = no more work).
// (shared-memory atomics: the slot is written by the producer while the other roles poll it)
__device__ __forceinline__ void work_publish(uint64_t* bars, uint32_t it, int item) {
    auto* w = reinterpret_cast<unsigned long long*>(bars + B_WORK + (it % WORK_SLOTS));
    atomicExch(w, ((unsigned long long)it << 32) | (uint32_t)item);
}
__device__ __forceinline__ int work_fetch(uint64_t* bars, uint32_t it) {
    volatile uint64_t* w = bars + B_WORK + (it % WORK_SLOTS);
    uint64_t v;
    do {
        v = *w;
    } while ((uint32_t)(v >> 32) != it);
    return (int)(uint32_t)v;
}

// Epilogue group of an item's streamed tile k. Group 1 also drains every item's accumulator
// (the tail), which delays its next tile; so the first tiles of each item (0, 1, 2) go to group 0
// and the rest alternate (odd -> group 1): group 1's first tile of the next item comes ~3 tiles
// after the boundary, by when its tail is done. (EMBER_TC_EARLY=1: plain alternation, A/B.)
__device__ __forceinline__ int tile_group(int k, int early) { return k < early ? 0 : (k & 1); }

__device__ __noinline__ void tc_fixup_rows(const TcArgs& g, uint32_t n);

template <int MODE>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_tc(const __grid_constant__ CUtensorMap mapR, const __grid_constant__ CUtensorMap mapT, const __grid_constant__ TcArgs g) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const Smem sm = carve<MODE>(smem_raw, g.KP, g.nstage);
    const int NSTAGE = g.nstage + (g.res_stage ? 1 : 0);  // ring depth (the last stage may be the resident buffer)
    uint64_t* bars = sm.bars;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(&bars[B_TMEM_SLOT]);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int KP = g.KP, CB = g.CB;
    const int items = n_items<MODE>(g);
    const int KS = KP / 16;
    const int NSP = g.nsp;
    const uint64_t lo_off = (uint64_t)((CB * TILE * 16) >> 4);  // lo blocks follow hi blocks (descriptor units)
    // TMEM columns: S/P buffer b at b*TILE, accumulator, then the resident operand (KP each)
    const uint32_t T_ACC = (uint32_t)(NSP * TILE), T_RES = T_ACC + (uint32_t)KP;
    const int tr_role = warp == 0 ? 0 : warp == 1 ? 1 : warp == 2 ? 4 : (warp - 3) < 4 ? 2 : 3;  // TC_TRACE region
    int tr_n = 0;

    if (threadIdx.x == 0) {
        tc::mbar_init(&bars[B_RES_FULL], 1);
        tc::mbar_init(&bars[B_RES_EMPTY], 1);
        for (int i = 0; i < NSTAGE; ++i) {
            tc::mbar_init(&bars[B_RING_FULL + i], 1);
            tc::mbar_init(&bars[B_RING_EMPTY + i], 1);
        }
        for (int i = 0; i < 2 * NSP_MAX; ++i) tc::mbar_init(&bars[B_S_FULL + i], 1);
        for (int i = 0; i < g.nsp; ++i) {
            tc::mbar_init(&bars[B_P_FULL + i], 128);
            tc::mbar_init(&bars[B_PN_DONE + i], 1);
        }
        tc::mbar_init(&bars[B_ACC_FULL], 1);
        tc::mbar_init(&bars[B_ACC_EMPTY], 128);
        for (int i = 0; i < 4; ++i) {
            tc::mbar_init(&bars[B_Z_READY + i], 128);
            tc::mbar_init(&bars[B_ZB_FREE + i], 128);
        }
        tc::fence_mbar_init();
        tc::tmap_prefetch(&mapR);
        tc::tmap_prefetch(&mapT);
        tslot[1] = atomicAdd(g.arrive, 1u) - g.arrive_base;  // this CTA's rank in arrival order
        for (uint32_t w = 0; w < WORK_SLOTS; ++w)  // no work published yet
            atomicExch(reinterpret_cast<unsigned long long*>(bars + B_WORK + w), ~0ull);
    }
    if (warp == 1) tc::tmem_alloc(tslot, TCOLS);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    // All 512 columns belong to this CTA (one CTA per SM), so the allocation starts at lane 0,
    // column 0: the MMA issuer uses compile-time TMEM addresses.
    const uint32_t tbase = *tslot;
    if (tbase != 0) __trap();
    const int cta = (int)tslot[1];
    griddep_wait();  // set-up above overlaps the previous kernel's tail (PDL)
    if (g.cta_times && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g.cta_times[2 * blockIdx.x] = t;
    }
    if (MODE == MODE_ROWS && blockIdx.x == 0) {
        // streamed 96-row tiles may reach past the last 128-row item: those rows never score
        for (int i = threadIdx.x; i < 2 * (g.rows_pad - g.rows128); i += blockDim.x) {
            const int side = i / (g.rows_pad - g.rows128), row = g.rows128 + i % (g.rows_pad - g.rows128);
            g.lse_pad[(size_t)side * g.b_cap + row] = -INFINITY;
        }
    }
    if (MODE == MODE_NEGS) {  // rows the rows kernel flagged: exact recompute before any lse is read
        const uint32_t nflag = *(volatile uint32_t*)g.flags;
        if (nflag) {
            tc_fixup_rows(g, nflag);
            __threadfence();
            asm volatile("fence.proxy.async.global;" ::: "memory");  // the producers read lse_pad by TMA
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            atomicAdd(g.fix_bar, 1u);
            if (nflag) {  // every CTA's repairs visible before any producer loads an lse
                while ((int)(*(volatile uint32_t*)g.fix_bar - (g.fix_base + gridDim.x)) < 0) __nanosleep(64);
                __threadfence();
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
        }
        __syncthreads();
    }

    if (warp == 0) {
        if (lane == 0) {  // ------------------------------------------------------ TMA producer
            const uint32_t bytesR = (uint32_t)res_bytes(KP);
            const uint32_t bytesT = (uint32_t)(TILE * KP * 4 + trailer_bytes(MODE));  // TMA'd bytes per tile
            uint32_t it = 0, gr = 0;  // gr: streamed-tile ring slots used
            for (int item = cta;; ++it) {
                if (it > 0)
                    item = g.dyn ? (int)(atomicAdd(g.claim, 1u) - g.claim_base) + (int)gridDim.x
                                 : item + (int)gridDim.x;
                work_publish(bars, it, min(item, items));
                if (item >= items) break;
                const Item I = item_geo<MODE>(g, item);
                // resident tile: its previous occupant has been copied into TMEM (RES_EMPTY)
                if (g.res_stage && it > 0) __trap();  // (res_stage: one item per CTA, set by the host)
                tc::mbar_wait(&bars[B_RES_EMPTY], (it & 1) ^ 1);
                tc::mbar_expect_tx(&bars[B_RES_FULL], bytesR);
                tc::tma_load_4d(sm.res, &mapR, 0, I.r0 / 32, 0, I.side, &bars[B_RES_FULL]);
                TC_TRACE(1, it);
                for (int k = 0; k < I.T; ++k, ++gr) {
                    const int st = gr % NSTAGE;
                    tc::mbar_wait(&bars[B_RING_EMPTY + st], ((gr / NSTAGE) & 1) ^ 1);
                    // first use of the resident buffer as a ring stage: its tile is in TMEM by now
                    if (st == g.nstage && gr < (uint32_t)NSTAGE) tc::mbar_wait(&bars[B_RES_EMPTY], 0);
                    TC_TRACE(2, gr);
                    tc::mbar_expect_tx(&bars[B_RING_FULL + st], bytesT);
                    uint8_t* dst = sm.stage(st);
                    const int row = I.t0 + k * TILE;
                    tc::tma_load_4d(dst, &mapT, 0, row / 32, 0, I.side, &bars[B_RING_FULL + st]);
                    if (MODE == MODE_NEGS)
                        tc::bulk_g2s(dst + TILE * KP * 4, g.lse_pad + (size_t)I.side * g.b_cap + row, TILE * 4,
                                     &bars[B_RING_FULL + st]);
                }
            }
        }
    } else if (warp == 1) {  // ---------------------------------------------- S issuer (+ R staging)
        // Warps 1 and 2 run their loops converged (warp-uniform waits and values in uniform
        // registers); one elected lane issues each tcgen05 instruction. Splitting the two products
        // over two issuing warps lets each warp's barrier waits hide behind the other's issue.
        const uint32_t id_s = tc::idesc_bf16(128, TILE, false, false);
        uint32_t it = 0, gt = 0;  // gt: streamed tiles (S/P buffers and ring slots)
        for (;; ++it) {
            const int item = work_fetch(bars, it);
            if (item >= items) break;
            const Item I = item_geo<MODE>(g, item);
            {  // resident operand smem -> TMEM, in this warp's MMA stream after the previous item's last S
                tc::mbar_wait_warp(&bars[B_RES_FULL], it & 1);
                TC_TRACE(10, it);
                tc::fence_after();
#pragma unroll
                for (int s = 0; s < KPMAX / 16; ++s) {
                    if (s < KS) {
                        tmem_cp_128x256b(T_RES + s * 8, kdesc(sm.res, RES, s, 0));
                        tmem_cp_128x256b(T_RES + KP / 2 + s * 8, kdesc(sm.res, RES, s, CB));
                    }
                }
                tc::mma_commit_elect(&bars[B_RES_EMPTY]);
            }
            for (int k = 0; k < I.T; ++k) {  // S_k = R . T_k^T   (R from TMEM, T_k K-major from smem)
                const uint32_t q = gt + k;
                const int st = q % NSTAGE;
                const uint32_t b = q % NSP;
                if (q >= (uint32_t)NSP)  // buffer b free: P.T of tile q - NSP has completed
                    tc::mbar_wait_warp(&bars[B_PN_DONE + b], (q / NSP - 1) & 1);
                TC_TRACE(16, q);
                tc::mbar_wait_warp(&bars[B_RING_FULL + st], (q / NSTAGE) & 1);
                TC_TRACE(11, q);
                tc::fence_after();
                const uint32_t tS = b * TILE;
                const uint64_t t0 = kdesc(sm.stage(st), TILE, 0, 0);
#pragma unroll
                for (int s = 0; s < KPMAX / 16; ++s) {
                    if (s < KS) {
                        const uint32_t rh = T_RES + s * 8, rl = T_RES + KP / 2 + s * 8;
                        const uint64_t th = t0 + (uint64_t)(s * ((2 * TILE * 16) >> 4)), tl = th + lo_off;
                        tc::mma_ts_elect(tS, rl, th, id_s, s > 0 ? 1u : 0u);
                        tc::mma_ts_elect(tS, rh, tl, id_s, 1u);
                        tc::mma_ts_elect(tS, rh, th, id_s, 1u);
                    }
                }
                tc::mma_commit_elect(&bars[B_S_FULL + tile_group(k, g.early) * NSP_MAX + b]);  // tile k -> its group
                TC_TRACE(12, q);
            }
            gt += I.T;
        }
    } else if (warp == 2) {  // ----------------------------------------------------- P.T issuer
        const uint32_t id_a = tc::idesc_bf16(128, KP, false, true);
        uint32_t it = 0, gt = 0;
        for (;; ++it) {
            const int item = work_fetch(bars, it);
            if (item >= items) break;
            const Item I = item_geo<MODE>(g, item);
            for (int k = 0; k < I.T; ++k) {  // acc += P_k . T_k   (P from TMEM, T MN-major from smem)
                const uint32_t q = gt + k;
                const int st = q % NSTAGE;
                const uint32_t b = q % NSP;
                TC_TRACE(17, q);
                tc::mbar_wait_warp(&bars[B_P_FULL + b], (q / NSP) & 1);
                TC_TRACE(13, q);
                if (k == 0) tc::mbar_wait_warp(&bars[B_ACC_EMPTY], (it & 1) ^ 1);
                if (k == 0) TC_TRACE(15, it);
                tc::fence_after();
                const uint32_t tP = b * TILE;
                const uint64_t t0 = mndesc(sm.stage(st), TILE, 0, 0);
                const uint32_t acc0 = k > 0 ? 1u : 0u;
#pragma unroll
                for (int s = 0; s < TILE / 16; ++s) {
                    // k-step s covers streamed rows 16s..16s+15: 32-column chunk s/2 of the P buffer
                    // holds 16 hi pair columns then 16 lo pair columns
                    const uint32_t ph = tP + (s >> 1) * 32 + (s & 1) * 8, pl = ph + 16;
                    const uint64_t th = t0 + (uint64_t)(s * (256 >> 4)), tl = th + lo_off;
                    tc::mma_ts_elect(T_ACC, pl, th, id_a, s > 0 ? 1u : acc0);
                    tc::mma_ts_elect(T_ACC, ph, tl, id_a, 1u);
                    tc::mma_ts_elect(T_ACC, ph, th, id_a, 1u);
                }
                tc::mma_commit_elect(&bars[B_RING_EMPTY + st]);
                tc::mma_commit_elect(&bars[B_PN_DONE + b]);
                TC_TRACE(14, q);
            }
            tc::mma_commit_elect(&bars[B_ACC_FULL]);
            gt += I.T;
        }
    } else {  // -------------------------------------------------------------------- epilogue
        const int G = (warp - 3) >> 2;          // ping-pong group: takes the tiles k with tile_group(k) == G
        const int qd = warp & 3;                // TMEM lane quadrant
        const int r = 32 * qd + lane;           // resident row (MODE_ROWS: batch row; NEGS: negative)
        const uint32_t t_row = tbase + ((uint32_t)(32 * qd) << 16);
        // Tile k of every item goes to group tile_group(k) (group 0 always starts an item); group 1
        // also does every item tail, so group 0 moves straight on to the next item's first tiles.
        uint32_t it = 0, gt = 0;
        uint32_t sphase = 0;  // bit b: parity of this group's next wait on S_FULL[G][b]
        for (;; ++it) {
            const int item = work_fetch(bars, it);
            if (item >= items) break;
            const Item I = item_geo<MODE>(g, item);
            const int row = I.r0 + r;
            float fp = 0.f, z = 0.f;
            if (MODE == MODE_ROWS) fp = row < g.nb ? g.fpos[row] : 0.f;
            const float cshift = -fp * L2E;
            for (int k = 0; k < I.T; ++k) {
                if (tile_group(k, g.early) != G) continue;
                const uint32_t q = gt + k;
                const uint32_t b = q % NSP;
                const uint32_t tS = t_row + b * TILE;
                const int st = q % NSTAGE;
                if (MODE == MODE_NEGS) tc::mbar_wait(&bars[B_RING_FULL + st], (q / NSTAGE) & 1);
                tc::mbar_wait(&bars[B_S_FULL + G * NSP_MAX + b], (sphase >> b) & 1);
                sphase ^= 1u << b;
                if (qd == 2) TC_TRACE(20 + G, q);
                tc::fence_after();
                // 64 columns per TMEM round trip, then the 32-column remainder (TILE = 96)
                if (!g.diag) {
                    if (MODE == MODE_ROWS) {  // 32 columns per TMEM round trip: no epilogue spills
                        epi_chunk<MODE, 1>(tS, 0, k, g, sm, st, KP, cshift, z);
                        epi_chunk<MODE, 1>(tS, 32, k, g, sm, st, KP, cshift, z);
                        epi_chunk<MODE, 1>(tS, 64, k, g, sm, st, KP, cshift, z);
                    } else {  // 64 columns, then the 32-column remainder (TILE = 96)
                        epi_chunk<MODE, 2>(tS, 0, k, g, sm, st, KP, cshift, z);
                        epi_chunk<MODE, 1>(tS, 64, k, g, sm, st, KP, cshift, z);
                    }
                }
                tc::tmem_st_wait();
                tc::fence_before();
                tc::mbar_arrive(&bars[B_P_FULL + b]);
                if (qd == 2) TC_TRACE(22 + G, q);
            }
            if (G == 0) {  // hand the row sums to group 1 (4 slots, each reused in order)
                if (MODE == MODE_ROWS) {
                    const uint32_t zs = it & 3;
                    tc::mbar_wait(&bars[B_ZB_FREE + zs], ((it >> 2) & 1) ^ 1);
                    sm.zbuf[zs * 128 + r] = z;
                    tc::mbar_arrive(&bars[B_Z_READY + zs]);
                }
                gt += I.T;
                continue;
            }
            tc::mbar_wait(&bars[B_ACC_FULL], it & 1);
            if (qd == 2) TC_TRACE(26 + G, it);
            tc::fence_after();
            // Accumulator row in two batches of <= 4 chunks of 16 columns; the accumulator is released
            // right after the last TMEM read, before the last batch's stores.
            const int nchunks = KP / 16;
            float scale = 1.0f, lse = 0.f, Z = 1.f;
            const bool valid = MODE == MODE_NEGS || row < g.nb;
            if (MODE == MODE_ROWS) {
                const uint32_t zs = it & 3;
                tc::mbar_wait(&bars[B_Z_READY + zs], (it >> 2) & 1);
                if (qd == 2) TC_TRACE(32, it);
                Z = 1.0f + z + sm.zbuf[zs * 128 + r];  // + exp(f_pos - f_pos) = 1: the positive
                tc::mbar_arrive(&bars[B_ZB_FREE + zs]);
                lse = fp + __logf(Z);
                scale = g.inv_b / Z;
            }
            // column-blocked outputs: float4 block c4 of row e at [..][c4][e]
            float4* out = MODE == MODE_ROWS
                              ? reinterpret_cast<float4*>(g.dA) + (size_t)I.side * (g.d / 4) * g.b_cap + row
                              : reinterpret_cast<float4*>(g.dN_part) +
                                    ((size_t)I.chunk * 2 + I.side) * (g.d / 4) * g.n_pad + row;
            const size_t cstride = MODE == MODE_ROWS ? (size_t)g.b_cap : (size_t)g.n_pad;
            uint64_t l2pol = 0;
            if (MODE == MODE_ROWS && g.l2_keep)
                asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(l2pol));
            // batches: chunks [0, nchunks - 4), then the last 4 (one batch when nchunks <= 4)
            const int b0 = nchunks > 4 ? nchunks - 4 : nchunks;
            for (int half = 0; half < 2; ++half) {
                const int c0 = half ? b0 : 0, cn = half ? nchunks : b0;
                uint32_t accv[4][16];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (c0 + i < cn) tc::tmem_ld16(t_row + T_ACC + 16 * (c0 + i), accv[i]);
                tc::tmem_ld_wait();
                if (qd == 2) TC_TRACE(30 + half, it);
                if (cn == nchunks) {
                    tc::fence_before();
                    tc::mbar_arrive(&bars[B_ACC_EMPTY]);
                }
                if (valid) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int c = c0 + i;
                        if (c >= cn) continue;
#pragma unroll
                        for (int j = 0; j < 16; j += 4)
                            if (16 * c + j < g.d) {
                                float4* o = out + (size_t)((16 * c + j) / 4) * cstride;
                                const float x0 = __uint_as_float(accv[i][j]) * scale,
                                            x1 = __uint_as_float(accv[i][j + 1]) * scale,
                                            x2 = __uint_as_float(accv[i][j + 2]) * scale,
                                            x3 = __uint_as_float(accv[i][j + 3]) * scale;
                                if (MODE == MODE_ROWS && g.l2_keep)  // dA: read back by the chain rule
                                    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(o),
                                                 "f"(x0), "f"(x1), "f"(x2), "f"(x3), "l"(l2pol)
                                                 : "memory");
                                else
                                    *o = make_float4(x0, x1, x2, x3);
                            }
                    }
                }
                if (cn == nchunks) break;
            }
            if (MODE == MODE_ROWS) {
                if (valid) {
                    g.lse[(size_t)I.side * g.nb + row] = lse;
                    g.g0[(size_t)I.side * g.nb + row] = (__expf(fp - lse) - 1.0f) * g.inv_b;
                    if (!(Z < g.zmax)) g.flags[1 + atomicAdd(g.flags, 1u)] = (uint32_t)(I.side * g.b_cap + row);
                }
                g.lse_pad[(size_t)I.side * g.b_cap + row] = valid ? fmaf(-lse, L2E, g.log2_inv_b) : -INFINITY;
            }
            if (qd == 2) TC_TRACE(28 + G, it);
            gt += I.T;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tbase, TCOLS);
    if (g.cta_times && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g.cta_times[2 * blockIdx.x + 1] = t;
    }
}

// Exact two-pass recomputation (fp32, CUDA cores) of the rows k_tc<MODE_ROWS> flagged because
// sum exp(S - f_pos) left the safe range (a negative scoring > f_pos + ~55). One block; normally
// the list is empty and the kernel exits at once. Resets the list for the next step.
__device__ __forceinline__ float packed_at(const uint16_t* pk, int cap, int CB, int side, int row, int c) {
    const size_t hi = (((size_t)side * 2 * CB + c / 8) * cap + row) * 8 + c % 8;
    const size_t lo = hi + (size_t)CB * cap * 8;
    return __bfloat162float(__ushort_as_bfloat16(pk[hi])) + __bfloat162float(__ushort_as_bfloat16(pk[lo]));
}

__device__ __noinline__ void tc_fixup_rows(const TcArgs& g, uint32_t n) {
    const uint16_t* __restrict__ Apk = g.Apk;
    const uint16_t* __restrict__ Npk = g.Npk;
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t f = gw; f < n; f += nw) {  // a warp per flagged row, all blocks
        const uint32_t code = g.flags[1 + f];
        const int side = (int)(code / g.b_cap), row = (int)(code % g.b_cap);
        // operands as the tensor cores saw them (hi + lo), rows of at most 128 floats: 4 per lane
        float a[4], nv[4];
        for (int c = lane, i = 0; i < 4; c += 32, ++i) a[i] = c < g.d ? packed_at(Apk, g.b_cap, g.CB, side, row, c) : 0.f;
        const float fp = g.fpos[row];
        auto score = [&](int k) {
            float s = 0.f;
            for (int c = lane, i = 0; i < 4; c += 32, ++i) {
                nv[i] = c < g.d ? packed_at(Npk, g.n_pad, g.CB, side, k, c) : 0.f;
                s += a[i] * nv[i];
            }
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            return s;
        };
        float mx = fp;
        for (int k = 0; k < g.nt; ++k) mx = fmaxf(mx, score(k));
        float z = expf(fp - mx), acc[4] = {0.f, 0.f, 0.f, 0.f};
        for (int k = 0; k < g.nt; ++k) {
            const float p = expf(score(k) - mx);
            z += p;
            for (int i = 0; i < 4; ++i) acc[i] += p * nv[i];
        }
        const float lse = mx + logf(z);
        const float scale = g.inv_b / z;
        float* out = g.dA + (size_t)side * g.d * g.b_cap;  // column-blocked [side][c/4][row][c%4]
        for (int c = lane, i = 0; i < 4; c += 32, ++i)
            if (c < g.d) out[((size_t)(c / 4) * g.b_cap + row) * 4 + c % 4] = acc[i] * scale;
        if (lane == 0) {
            g.lse[(size_t)side * g.nb + row] = lse;
            g.lse_pad[(size_t)side * g.b_cap + row] = fmaf(-lse, L2E, g.log2_inv_b);
            g.g0[(size_t)side * g.nb + row] = (expf(fp - lse) - 1.0f) * g.inv_b;
        }
    }
    // (the flag count is reset by the dN reduction, after every reader)
}

// =========================================================================================
// The dN reduction (memory-bound helper; the operands are packed by the gathers, kernels_step.cu).
// =========================================================================================

// dN rows summed over chunks in fixed order; row (side, n) is gradient slot 2nb + side*nt + n and
// goes to its sorted position grows[rank[slot]]. Thread per (side, column block, negative): the
// column-blocked partials [chunk][side][d/4][n_pad] float4 are read coalesced along n.
// nsides: 2 (one shared negative set per side), or 2 x num_chunks ([chunk][side] sets, tc_wide.cu).
__global__ void k_dn_reduce(DnReduce r, const uint32_t* __restrict__ rank, float* __restrict__ out) {
    griddep_wait();
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // overflow list consumed (tc_fixup_rows): count, reset
        r.flags_total[0] += r.flags[0];
        *r.flags = 0u;
    }
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)r.nsides * (r.d / 4) * r.nt) return;
    dn_reduce_item(r, t, rank, out);
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

// 4-D view of a packed operand [2 sides][2CB blocks][cap rows][8 bf16]: within one column block,
// 32 consecutive rows are one contiguous 512-byte run, so the view is {256 elements, cap/32 row
// groups, 2CB blocks, 2 sides} and a box {256, box_rows/32, 2CB, 1} moves 512-byte rows (a 16-byte
// inner box would cost one TMA request per 16 B). It lands in smem as [cb][box_rows][16 B], the
// canonical K-major tile. Coordinates: (0, row/32, 0, side).
CUtensorMap make_map(uint16_t* base, int cap, int CB, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[4] = {256, (cuuint64_t)(cap / 32), (cuuint64_t)(2 * CB), 2};
    const cuuint64_t strides[3] = {512, (cuuint64_t)cap * 16, (cuuint64_t)cap * 16 * 2 * CB};
    const cuuint32_t box[4] = {256, (cuuint32_t)(box_rows / 32), (cuuint32_t)(2 * CB), 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw EmberError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

}  // namespace

// 4-D view of any packed operand [2 sides][nblocks2][cap rows][8 bf16] with a box of box_rows rows
// (a multiple of 32) x box_blocks column blocks: lands in smem as [box_blocks][box_rows][16 B], the
// canonical K-major tile (columns along K) or MN-major tile (rows along K). Used by tc_wide.cu.
CUtensorMap make_packed_map(uint16_t* base, int cap, int nblocks2, int box_rows, int box_blocks) {
    CUtensorMap m;
    const cuuint64_t dims[4] = {256, (cuuint64_t)(cap / 32), (cuuint64_t)nblocks2, 2};
    const cuuint64_t strides[3] = {512, (cuuint64_t)cap * 16, (cuuint64_t)cap * 16 * nblocks2};
    const cuuint32_t box[4] = {256, (cuuint32_t)(box_rows / 32), (cuuint32_t)box_blocks, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw EmberError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return m;
}

// The fixed-order dN reduction of k_dn_reduce for the wide engine's partials (tc_wide.cu).
void dn_reduce_launch(Engine& E, const float* part, int chunks, int nt, int n_pad, int d, uint32_t slot0,
                      uint32_t* flags, unsigned long long* flags_total, int nsides) {
    DnReduce r;
    r.part = reinterpret_cast<const float4*>(part);
    r.chunks = chunks;
    r.nt = nt;
    r.n_pad = n_pad;
    r.d = d;
    r.nsides = nsides;
    r.slot0 = slot0;
    r.flags = flags;
    r.flags_total = flags_total;
    dn_reduce_run(E, r);
}

void dn_reduce_run(const Engine& E, const DnReduce& r) {
    const int64_t n = (int64_t)r.nsides * r.nt * (r.d / 4);
    launch_pdl(k_dn_reduce, dim3((unsigned)((n + 255) / 256)), dim3(256), 0, E.stream, r, (const uint32_t*)E.s.rank,
               E.s.grows);
    EMBER_LAUNCHED(E);
}

// Engine-side state of the tensor-core engine (allocated once per context).
struct TcState {
    int KP = 0, CB = 0, b_cap = 0, n_pad = 0, chunks2 = 1, nstage = 4, nsp = 2;
    bool res_stage = true;  // the dN kernel's resident buffer as an extra ring stage (EMBER_TC_RES_STAGE=0: off)
    float* dN_part = nullptr;
    float* lse_pad = nullptr;
    uint32_t* flags = nullptr;
    unsigned long long* flags_total = nullptr;  // overflowed rows recomputed exactly, since creation
    CUtensorMap mA128, mA96, mN128, mN96;  // resident (RES rows) and streamed (TILE rows) boxes
    float zmax = 1e30f;  // sum exp(S - f_pos) above this: exact recompute (fp32 and the P.N sums stay finite)
    int max_grid = 0;  // test hook (EMBER_TC_MAXGRID): several items per CTA at small sizes
    unsigned long long* trace = nullptr;  // EMBER_TC_TRACE=<file prefix>: CTA-0 timeline dump
    unsigned long long* cta_times = nullptr;  // EMBER_TC_CTATIMES=<file>: per-CTA spans of one rows + one dN launch
    uint32_t* arrive = nullptr;     // [3]: CTA arrival counters of the rows / dN kernels, rows-item claims (never reset)
    uint32_t arrive_base[2] = {0, 0};
    uint32_t claim_base = 0;
    uint32_t* fix_bar = nullptr;    // dN-kernel CTA arrivals (never reset) and their expected count
    uint32_t fix_base = 0;
    bool dyn = true;                // dynamic rows-item claims (EMBER_TC_DYNAMIC=0: static grid stride)
    std::string trace_path;
    int trace_calls = 0;
};

bool tc_engine_supported(const Engine& E) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, E.device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, E.device);
    return major == 10 && minor == 0 && E.nt >= 1 && ((E.dim <= (uint32_t)KPMAX && E.chunks == 1) || wide_supported(E));
}

void tc_setup(Engine& E) {
    auto* t = new TcState();
    t->KP = E.KP;  // packed operands (E.s.Apk / E.s.Npk) are allocated by the engine
    t->CB = E.CB;
    t->b_cap = E.b_cap;
    t->n_pad = E.n_pad;
    const int ntl = (int)((E.nt + RES - 1) / RES);
    t->nsp = std::min(NSP_MAX, (512 - 2 * t->KP) / TILE);
    if (t->nsp < 2) throw ConfigError("tensor-core engine: dim too large for the TMEM layout");
    t->chunks2 = std::max(1, E.sm_count / (2 * ntl));
    t->nstage = stages_for(t->KP);
    if (const char* s = getenv("EMBER_TC_NSTAGE")) t->nstage = std::max(2, std::min(t->nstage, atoi(s)));  // A/B
    if (const char* s = getenv("EMBER_TC_RES_STAGE")) t->res_stage = atoi(s) != 0;
    if (const char* s = getenv("EMBER_TC_ZMAX")) t->zmax = (float)atof(s);  // test hook: 0 flags every row
    if (const char* s = getenv("EMBER_TC_MAXGRID")) t->max_grid = atoi(s);
    if (getenv("EMBER_TC_CTATIMES")) EMBER_CUDA(cudaMalloc(&t->cta_times, (size_t)2 * 2 * E.sm_count * 8));
    EMBER_CUDA(cudaMalloc(&t->arrive, 3 * sizeof(uint32_t)));
    EMBER_CUDA(cudaMemset(t->arrive, 0, 3 * sizeof(uint32_t)));
    EMBER_CUDA(cudaMalloc(&t->fix_bar, sizeof(uint32_t)));
    EMBER_CUDA(cudaMemset(t->fix_bar, 0, sizeof(uint32_t)));
    if (const char* s = getenv("EMBER_TC_DYNAMIC")) t->dyn = atoi(s) != 0;
    if (const char* s = getenv("EMBER_TC_TRACE")) {
        t->trace_path = s;
        EMBER_CUDA(cudaMalloc(&t->trace, (size_t)2 * 5 * TRACE_ROLE * 8));
    }
    EMBER_CUDA(cudaMalloc(&t->dN_part, (size_t)t->chunks2 * 2 * t->n_pad * E.dim * sizeof(float)));
    EMBER_CUDA(cudaMalloc(&t->lse_pad, (size_t)2 * t->b_cap * sizeof(float)));
    EMBER_CUDA(cudaMalloc(&t->flags, (size_t)(1 + 2 * t->b_cap) * sizeof(uint32_t)));
    EMBER_CUDA(cudaMemset(t->flags, 0, sizeof(uint32_t)));
    EMBER_CUDA(cudaMalloc(&t->flags_total, sizeof(unsigned long long)));
    EMBER_CUDA(cudaMemset(t->flags_total, 0, sizeof(unsigned long long)));
    t->mA128 = make_map(E.s.Apk, t->b_cap, t->CB, RES);
    t->mA96 = make_map(E.s.Apk, t->b_cap, t->CB, TILE);
    t->mN128 = make_map(E.s.Npk, t->n_pad, t->CB, RES);
    t->mN96 = make_map(E.s.Npk, t->n_pad, t->CB, TILE);
    EMBER_CUDA(cudaFuncSetAttribute(k_tc<MODE_ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem_total(t->KP, t->nstage, MODE_ROWS)));
    EMBER_CUDA(cudaFuncSetAttribute(k_tc<MODE_NEGS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem_total(t->KP, t->nstage, MODE_NEGS)));
    E.tc = t;
}

uint64_t tc_overflow_rows(Engine& E) {
    if (E.wide) return wide_overflow_rows(E);
    if (!E.tc) return 0;
    unsigned long long v = 0;
    EMBER_CUDA(cudaStreamSynchronize(E.stream));
    EMBER_CUDA(cudaMemcpy(&v, E.tc->flags_total, sizeof(v), cudaMemcpyDeviceToHost));
    return v;
}

void tc_release(Engine& E) {
    if (!E.tc) return;
    cudaFree(E.tc->dN_part);
    cudaFree(E.tc->lse_pad);
    cudaFree(E.tc->flags);
    cudaFree(E.tc->flags_total);
    if (E.tc->trace) cudaFree(E.tc->trace);
    if (E.tc->cta_times) cudaFree(E.tc->cta_times);
    cudaFree(E.tc->arrive);
    cudaFree(E.tc->fix_bar);
    delete E.tc;
    E.tc = nullptr;
}

void launch_contract_tc(Engine& E, uint32_t nb) {
    TcState& t = *E.tc;
    const int d = (int)E.dim, nt = (int)E.nt;
    Scratch& s = E.s;
    const int rows_pad = (int)((nb + RES - 1) / RES * RES);  // 128-row items of k_tc<ROWS>
    TcArgs a{};
    a.KP = t.KP;
    a.CB = t.CB;
    a.d = d;
    a.nb = (int)nb;
    a.nt = nt;
    a.n_pad = t.n_pad;
    a.b_cap = t.b_cap;
    a.inv_b = 1.0f / (float)nb;
    a.log2_inv_b = log2f(a.inv_b);
    a.zmax = t.zmax;
    a.fpos = s.fpos;
    a.lse = s.lse;
    a.lse_pad = t.lse_pad;
    a.g0 = s.g0;
    a.dA = s.dA;
    a.dN_part = t.dN_part;
    a.flags = t.flags;
    a.early = 3;
    if (const char* e = getenv("EMBER_TC_EARLY")) a.early = std::max(1, atoi(e));  // A/B (1: plain alternation)
    a.diag = getenv("EMBER_TC_DIAG") ? 1 : 0;
    a.l2_keep = getenv("EMBER_DA_L2") && atoi(getenv("EMBER_DA_L2")) == 0 ? 0 : 1;
    a.trace = nullptr;
    const int nsub = (int)((nb + TILE - 1) / TILE);
    a.chunks2 = std::min(t.chunks2, nsub);
    a.nstage = t.nstage;
    a.nsp = t.nsp;
    a.rows128 = rows_pad;
    a.rows_pad = E.pad_rows(nb);
    const int items1 = 2 * (rows_pad / RES);
    const int items2 = 2 * ((nt + RES - 1) / RES) * a.chunks2;
    const int gmax = t.max_grid > 0 ? std::min(t.max_grid, E.sm_count) : E.sm_count;
    const bool tr = t.trace && t.trace_calls++ == 4;  // one warmed-up call per process
    auto dump = [&](const char* tag) {
        EMBER_CUDA(cudaStreamSynchronize(E.stream));
        std::vector<unsigned long long> buf((size_t)2 * 5 * TRACE_ROLE);
        EMBER_CUDA(cudaMemcpy(buf.data(), t.trace, buf.size() * 8, cudaMemcpyDeviceToHost));
        FILE* f = fopen((t.trace_path + tag).c_str(), "wb");
        if (f) {
            fwrite(buf.data(), 8, buf.size(), f);
            fclose(f);
        }
    };
    if (tr) {
        EMBER_CUDA(cudaMemsetAsync(t.trace, 0, (size_t)2 * 5 * TRACE_ROLE * 8, E.stream));
        a.trace = t.trace;
    }
    const bool ct = t.cta_times && t.trace_calls++ == 6;  // one warmed-up call: rows CTAs then dN CTAs
    a.cta_times = ct ? t.cta_times : nullptr;
    // programmatic launch: the CTAs set up barriers and TMEM while the gathers drain
    // Performance only: when the dN kernel's grid (items2, e.g. 144 of 148 SMs) leaves at most
    // kSpareSms SMs idle, the rows kernel takes the same grid (the same number of waves), and the
    // free SMs run the helper stream's key sort. Test caps (EMBER_TC_MAXGRID) are used as given.
    constexpr int kSpareSms = 8;
    const int g2 = std::min(items2, gmax);
    static const int rows_grid = getenv("EMBER_TC_ROWS_GRID") ? atoi(getenv("EMBER_TC_ROWS_GRID")) : 0;  // A/B
    const int grid1 = rows_grid > 0 ? std::min(items1, std::min(rows_grid, gmax))
                                    : std::min(items1, t.max_grid == 0 && E.sm_count - g2 <= kSpareSms ? g2 : gmax);
    a.arrive = t.arrive;
    a.arrive_base = t.arrive_base[0];
    t.arrive_base[0] += (uint32_t)grid1;
    // every CTA claims until a claim fails: items1 - grid1 successful + grid1 failed claims
    a.dyn = t.dyn ? 1 : 0;
    a.claim = t.arrive + 2;
    a.claim_base = t.claim_base;
    if (t.dyn) t.claim_base += (uint32_t)items1;
    launch_pdl(k_tc<MODE_ROWS>, dim3(grid1), dim3(NTHREADS), smem_total(t.KP, t.nstage, MODE_ROWS),
               E.stream, t.mA128, t.mN96, a);
    EMBER_LAUNCHED(E);
    if (tr) {
        dump(".rows.bin");
        EMBER_CUDA(cudaMemsetAsync(t.trace, 0, (size_t)2 * 5 * TRACE_ROLE * 8, E.stream));
    }
    // rows flagged by the rows kernel (normally none) are recomputed by the dN kernel's CTAs, a warp
    // each, before its producers load any lse (tc_fixup_rows)
    a.Apk = s.Apk;
    a.Npk = s.Npk;
    a.fix_bar = t.fix_bar;
    a.fix_base = t.fix_base;
    t.fix_base += (uint32_t)std::min(items2, gmax);
    if (ct) a.cta_times = t.cta_times + 2 * E.sm_count;
    a.arrive = t.arrive + 1;
    a.arrive_base = t.arrive_base[1];
    // one item per CTA, and a barrier pair left for the extra stage
    a.res_stage = (t.res_stage && std::min(items2, gmax) >= items2 && t.nstage < NSTAGE_MAX) ? 1 : 0;
    a.dyn = 0;  // one item per CTA
    t.arrive_base[1] += (uint32_t)std::min(items2, gmax);
    launch_pdl(k_tc<MODE_NEGS>, dim3(std::min(items2, gmax)), dim3(NTHREADS), smem_total(t.KP, t.nstage, MODE_NEGS),
               E.stream, t.mN128, t.mA96, a);
    EMBER_LAUNCHED(E);
    if (ct) {  // host copy of both launches' spans (measurement only: synchronises the stream)
        EMBER_CUDA(cudaStreamSynchronize(E.stream));
        std::vector<unsigned long long> buf((size_t)4 * E.sm_count);
        EMBER_CUDA(cudaMemcpy(buf.data(), t.cta_times, buf.size() * 8, cudaMemcpyDeviceToHost));
        if (FILE* f = fopen(getenv("EMBER_TC_CTATIMES"), "wb")) {
            fwrite(buf.data(), 8, buf.size(), f);
            fclose(f);
        }
    }
    if (tr) dump(".negs.bin");
    // the fixed-order dN reduction: the chain rule's prologue (launch_chain_rule) does it
    DnReduce& r = E.dn;
    r.part = reinterpret_cast<const float4*>(t.dN_part);
    r.chunks = a.chunks2;
    r.nt = nt;
    r.n_pad = t.n_pad;
    r.d = d;
    r.nsides = 2;
    r.slot0 = 2 * nb;
    r.flags = t.flags;
    r.flags_total = t.flags_total;
    E.dn_pending = true;
    (void)s;
}

}  // namespace ember
