// SPDX-License-Identifier: Apache-2.0
//
// Memory-bound kernels of the training step (everything but the dense contraction):
//   k_sample          sample_negatives, SPEC.md:148-156 (counter-based, bit-exact with the oracle)
//   k_gather_adjust   formBatch gather + "adjust" to per-side dot-product operands,
//                     written as fp32 (SIMT engine) or straight into the tensor-core engine's
//                     bf16 hi|lo operand layout
//   k_gather_negs     negative rows, fp32 or packed
//   k_keys            gradient-slot keys for the (key, slot) sort (sort.cu)
//   k_chain_rule      chain rule back through adjust, rows written in sorted order
//   k_loss            deterministic loss reduction (fixed-order partials, last block finishes)
//   k_long_plan       (helper stream, after the sort) chunk plan of the keys with many rows
//   k_segments(_pipe), k_long_final
//                     segmented sum of the sorted gradient rows + sparse Adagrad;
//                     long keys as chunk partials (the segment kernels' prologue) + k_long_final
// Rows are dim floats (dim % 4 == 0) and are moved warp-per-row with 128-bit accesses.
#include <cuda_runtime.h>

#include <map>
#include <mutex>

#include "engine.h"
#include "tc_common.cuh"

namespace ember {
namespace {

__device__ __forceinline__ const float* node_row(const PartView& v, uint32_t id, uint32_t d) {
    return v.theta + (uint64_t)(id - v.first) * d;
}

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// Negative `slot` ([chunk][side][k] layout) of the batch whose stream seed is `base`.
__device__ __forceinline__ uint32_t sample_one(uint32_t slot, uint32_t nt, uint32_t n_deg, uint64_t base,
                                               const uint32_t* __restrict__ bucket, uint64_t bucket_n,
                                               uint64_t src_first, uint64_t src_rows, uint64_t dst_first,
                                               uint64_t dst_rows) {
    const uint32_t k = slot % nt;
    const uint32_t side = (slot / nt) & 1u;
    Rng g(mix_seed(base, (uint64_t)slot));
    if (k < n_deg && bucket_n > 0) {
        const uint64_t e = g.uniform_below(bucket_n);
        return bucket[3 * e + (side == 0 ? 2 : 0)];  // endpoint of a uniform bucket edge
    }
    if (side == 0) return (uint32_t)(dst_first + g.uniform_below(dst_rows));
    return (uint32_t)(src_first + g.uniform_below(src_rows));
}

__global__ void k_sample(uint32_t* out, uint32_t nt, uint32_t n_deg, uint32_t total, uint64_t base,
                         const uint32_t* __restrict__ bucket, uint64_t bucket_n, uint64_t src_first, uint64_t src_rows,
                         uint64_t dst_first, uint64_t dst_rows) {
    griddep_wait();
    const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
    if (slot >= total) return;
    out[slot] = sample_one(slot, nt, n_deg, base, bucket, bucket_n, src_first, src_rows, dst_first, dst_rows);
}

// Coordinates are handled in quads: quad q of a row is its 16 bytes at float offset 4q. For
// Dot/DistMult that is coordinates {4q .. 4q+3}; a ComplEx row ([re | im] halves of h = d/2 in the
// on-disk layout) is held in HBM with its halves interleaved by pairs (hbm_pos,
// engine.h), so quad q is the two complex coordinates {re 2q, re 2q+1, im 2q, im 2q+1} and every
// lane moves its rows' quads with one aligned 128-bit access and computes ComplEx products locally.
struct Quad {
    float v[4];
};

__device__ __forceinline__ Quad load_quad(const float* row, uint32_t q) {
    const float4 a = ldg4(row + 4 * q);
    Quad x;
    x.v[0] = a.x, x.v[1] = a.y, x.v[2] = a.z, x.v[3] = a.w;
    return x;
}

__device__ __forceinline__ void store_quad(float* row, uint32_t q, const Quad& x) {
    *reinterpret_cast<float4*>(row + 4 * q) = make_float4(x.v[0], x.v[1], x.v[2], x.v[3]);
}

// Adjusted quads: ad = the row the destination is scored against (s o r; ComplEx s * r), as = the
// row the source is scored against (r o t; ComplEx r * conj(t)), so that f(s, r, t) = ad . t = s . as
// (ComplEx quads {re, re, im, im}, see above). Products are rounded individually (no
// FMA contraction), like the oracle.
__device__ __forceinline__ void adjust_quad(int kind, const Quad& S, const Quad& R, const Quad& T, Quad& ad,
                                            Quad& as) {
    if (kind == EMBER_DOT) {
        ad = S;
        as = T;
    } else if (kind == EMBER_DISTMULT) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            ad.v[i] = __fmul_rn(S.v[i], R.v[i]);
            as.v[i] = __fmul_rn(R.v[i], T.v[i]);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 2; ++i) {  // i: re index i, im index 2 + i
            const float a = S.v[i], b = S.v[2 + i], c = R.v[i], e = R.v[2 + i], x = T.v[i], y = T.v[2 + i];
            ad.v[i] = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, e));
            as.v[i] = __fadd_rn(__fmul_rn(c, x), __fmul_rn(e, y));
            ad.v[2 + i] = __fadd_rn(__fmul_rn(a, e), __fmul_rn(b, c));
            as.v[2 + i] = __fsub_rn(__fmul_rn(c, y), __fmul_rn(e, x));
        }
    }
}

// Packed negative row w of [2 sides][n_pad] (side 0 rows from partition j, side 1 from i; zero past
// n_t): lane < CB splits 8 coordinates into bf16 hi|lo core-matrix rows of Npk.
// Without negs (ns.bucket set instead) the warp draws the negative id itself with the same
// counter-based stream as k_sample_keys (sample_one: slot side * nt + k), so the gather does not wait
// for the sampling kernel, which then runs on the helper stream beside it.
struct NegSampling {
    uint64_t base = 0, bucket_n = 0;
    const uint32_t* bucket = nullptr;
    uint32_t n_deg = 0;
    int on = 0;
};
__device__ __forceinline__ void negs_pack_warp(uint32_t w, uint32_t lane, const uint32_t* __restrict__ negs,
                                               const NegSampling& ns, uint32_t nt, uint32_t n_pad, const PartView& pi,
                                               const PartView& pj, uint32_t d, uint32_t CB,
                                               uint16_t* __restrict__ Npk) {
    if (w >= 2 * n_pad || lane >= CB) return;
    const uint32_t side = w / n_pad, slot = w % n_pad;
    float x[8];
    if (slot < nt) {
        const uint32_t id = ns.on ? sample_one(side * nt + slot, nt, ns.n_deg, ns.base, ns.bucket, ns.bucket_n, pi.first,
                                               pi.rows, pj.first, pj.rows)
                                  : negs[side * nt + slot];
        const float* src = node_row(side == 0 ? pj : pi, id, d);
        // d % 4 == 0: each quad is all in or all out (lanes past d read nothing: the K padding is 0)
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 a = 8 * lane < d ? ldg4(src + 8 * lane) : z;
        const float4 b = 8 * lane + 4 < d ? ldg4(src + 8 * lane + 4) : z;
        x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = 0.f;
    }
    uint4 h, l;
    tc::split8(x, h, l);
    uint4* P = reinterpret_cast<uint4*>(Npk);
    P[((uint64_t)side * 2 * CB + lane) * n_pad + slot] = h;
    P[((uint64_t)side * 2 * CB + CB + lane) * n_pad + slot] = l;
}

// Edges per CTA of the packed gather: one 512-byte run per column block (the TMA box row group).
constexpr uint32_t GP_ROWS = 32, GP_WARPS = 8;

// Packed gather (tensor-core engine): a CTA builds the operand rows of GP_ROWS consecutive edges
// (rows up to rows_pad: the packed layout is zero-padded to whole tiles). Each warp takes
// GP_ROWS / GP_WARPS edges: lanes load their quads of the source, relation and destination rows
// into registers and form the adjusted quads; lane pairs swap quads (shuffle) so that each lane
// < 2CB holds the 8 consecutive coordinates of one column block of one side, split into bf16 hi|lo
// 16-byte core-matrix rows of a shared tile
// [2 sides][2CB blocks][GP_ROWS][16 B] (row slot XOR-swizzled by the block, so the lanes' 16-byte
// stores are bank-conflict free), which leaves in 512-byte coalesced runs, one per column block
// (per-lane 16-byte stores would scatter over 56 blocks). fpos[e] = ad . t.
// (Staging the rows with one TMA bulk copy per 400-byte row measured slower than register loads.)
__global__ void __launch_bounds__(32 * GP_WARPS) k_gather_pack(const uint32_t* __restrict__ edges, uint32_t nb,
                                                               PartView pi, PartView pj, const float* __restrict__ rel,
                                                               int kind, uint32_t d, uint32_t CB, uint32_t cap,
                                                               uint16_t* __restrict__ Apk, float* __restrict__ fpos,
                                                               uint32_t row_ctas, const uint32_t* __restrict__ negs,
                                                               NegSampling ns, uint32_t nt, uint32_t n_pad,
                                                               uint16_t* __restrict__ Npk) {
    griddep_wait();
    if (blockIdx.x >= row_ctas) {  // the trailing CTAs pack the shared negatives (one warp per row)
        const uint32_t w = (blockIdx.x - row_ctas) * GP_WARPS + (threadIdx.x >> 5);
        negs_pack_warp(w, threadIdx.x & 31, negs, ns, nt, n_pad, pi, pj, d, CB, Npk);
        return;
    }
    extern __shared__ uint4 gsm[];
    uint4* tile = gsm;  // [2][2CB][GP_ROWS]
    const uint32_t nblk = 4 * CB;
    const uint32_t wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t e0 = blockIdx.x * GP_ROWS;
    const uint32_t nq = d / 4;
    // this warp's edges' (s, r, t) in one round of loads (lane 3k + i: word i of the k-th edge), so
    // each edge's row loads wait for one memory latency, not two
    constexpr uint32_t GP_PER_WARP = GP_ROWS / GP_WARPS;
    uint32_t idx = 0;
    {
        const uint32_t k = lane / 3, e = e0 + wib + k * GP_WARPS;
        if (lane < 3 * GP_PER_WARP && e < nb) idx = edges[3 * e + lane % 3];
    }
    for (uint32_t rr = wib, kk = 0; rr < GP_ROWS; rr += GP_WARPS, ++kk) {
        const uint32_t e = e0 + rr;
        const uint32_t s = __shfl_sync(0xffffffffu, idx, 3 * kk), r = __shfl_sync(0xffffffffu, idx, 3 * kk + 1),
                       t = __shfl_sync(0xffffffffu, idx, 3 * kk + 2);
        if (e >= nb) {  // padding rows of the last tiles
            for (uint32_t c = lane; c < nblk; c += 32) tile[c * GP_ROWS + (rr ^ (c % GP_ROWS))] = make_uint4(0, 0, 0, 0);
            continue;
        }
        // d <= 128: lane q holds quad q of each row (zeros past d: the K padding)
        Quad ad{}, as{};
        float part = 0.f;
        if (lane < nq) {
            const Quad S = load_quad(node_row(pi, s, d), lane), T = load_quad(node_row(pj, t, d), lane);
            const Quad R = kind != EMBER_DOT ? load_quad(rel + (uint64_t)r * d, lane) : S;
            adjust_quad(kind, S, R, T, ad, as);
#pragma unroll
            for (int i = 0; i < 4; ++i) part += ad.v[i] * T.v[i];
        }
        // Column block cb (8 coordinates) = quads 2cb and 2cb + 1. Lane 2cb packs side 0's block and
        // lane 2cb + 1 side 1's, each taking the other quad from its neighbour (registers only).
        const bool odd = lane & 1;
        float v[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float got = __shfl_xor_sync(0xffffffffu, odd ? ad.v[i] : as.v[i], 1);
            v[i] = odd ? got : ad.v[i];
            v[4 + i] = odd ? as.v[i] : got;
        }
        if (lane < 2 * CB) {
            uint4 hq, lq;
            tc::split8(v, hq, lq);
            // row slot rr ^ block: the lanes (one block each) hit distinct 16-byte bank groups
            const uint32_t bh = (lane & 1) * 2 * CB + (lane >> 1), bl = bh + CB;
            tile[bh * GP_ROWS + (rr ^ (bh % GP_ROWS))] = hq;
            tile[bl * GP_ROWS + (rr ^ (bl % GP_ROWS))] = lq;
        }
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        if (lane == 0) fpos[e] = part;
    }
    __syncthreads();
    uint4* P = reinterpret_cast<uint4*>(Apk);
    for (uint32_t i = threadIdx.x; i < nblk * GP_ROWS; i += blockDim.x) {
        const uint32_t blk = i / GP_ROWS, rr = i % GP_ROWS;  // blk = side * 2CB + column block
        P[(uint64_t)blk * cap + e0 + rr] = tile[blk * GP_ROWS + (rr ^ (blk % GP_ROWS))];
    }
}

// Packed gather of the wide tensor-core path (tc_wide.cu; d > 128 or chunked negatives): the same
// job as k_gather_pack for rows of any width, into the wide layout [side][2 CBA blocks][cap][8 bf16]
// with chunk q's rows at packed rows [q CP, q CP + cr). A CTA builds GW_ROWS consecutive packed rows
// (a warp each; rows without an edge are zero) in a shared tile [2 sides x 2 CBA blocks][GW_ROWS]
// of 16-byte core-matrix rows (slot XOR-swizzled by the block) that leaves in 128-byte runs. Lane
// pairs swap quads (shuffle) so each lane packs one 8-column block of one side per 64 columns.
constexpr uint32_t GW_ROWS = 8;
__global__ void __launch_bounds__(32 * GW_ROWS) k_gather_pack_wide(const uint32_t* __restrict__ edges, uint32_t nb,
                                                                  PartView pi, PartView pj,
                                                                  const float* __restrict__ rel, int kind, uint32_t d,
                                                                  uint32_t CBA, uint32_t cap, uint32_t CP, uint32_t cr,
                                                                  uint16_t* __restrict__ Apk, float* __restrict__ fpos) {
    griddep_wait();
    extern __shared__ uint4 gws[];  // [4 CBA][GW_ROWS]
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t pr = blockIdx.x * GW_ROWS + w, q = pr / CP, r = pr - q * CP, e = q * cr + r;
    const bool valid = r < cr && e < nb;
    const uint32_t nq = d / 4, nqp = CBA * 2;  // quads with data / quads of the padded width
    uint32_t s = 0, rr = 0, t = 0;
    if (valid) {
        s = edges[3 * e];
        rr = edges[3 * e + 1];
        t = edges[3 * e + 2];
    }
    const float* ss = valid ? node_row(pi, s, d) : nullptr;
    const float* st = valid ? node_row(pj, t, d) : nullptr;
    const float* sr = valid && kind != EMBER_DOT ? rel + (uint64_t)rr * d : nullptr;
    float part = 0.f;
    const bool odd = lane & 1;
    for (uint32_t q0 = 0; q0 < nqp; q0 += 32) {  // warp-uniform (shuffles)
        const uint32_t q4 = q0 + lane;
        Quad ad{}, as{};
        if (valid && q4 < nq) {
            const Quad S = load_quad(ss, q4), T = load_quad(st, q4);
            const Quad R = sr ? load_quad(sr, q4) : S;
            adjust_quad(kind, S, R, T, ad, as);
#pragma unroll
            for (int i = 0; i < 4; ++i) part += ad.v[i] * T.v[i];
        }
        float v[8];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float got = __shfl_xor_sync(0xffffffffu, odd ? ad.v[i] : as.v[i], 1);
            v[i] = odd ? got : ad.v[i];
            v[4 + i] = odd ? as.v[i] : got;
        }
        const uint32_t blk = q4 >> 1;  // column block of this lane pair
        if (blk < CBA) {
            uint4 hq, lq;
            tc::split8(v, hq, lq);
            const uint32_t bh = (lane & 1) * 2 * CBA + blk, bl = bh + CBA;
            gws[bh * GW_ROWS + (w ^ (bh % GW_ROWS))] = hq;
            gws[bl * GW_ROWS + (w ^ (bl % GW_ROWS))] = lq;
        }
    }
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (valid && lane == 0) fpos[e] = part;
    __syncthreads();
    uint4* P = reinterpret_cast<uint4*>(Apk);
    const uint32_t row0 = blockIdx.x * GW_ROWS;
    for (uint32_t i = threadIdx.x; i < 4 * CBA * GW_ROWS; i += blockDim.x) {
        const uint32_t blk = i / GW_ROWS, row = i % GW_ROWS;  // blk = side * 2CBA + column block
        P[(uint64_t)blk * cap + row0 + row] = gws[blk * GW_ROWS + (row ^ (blk % GW_ROWS))];
    }
}

// fp32 gather (SIMT engine, and the wide tensor-core path that packs it afterwards, tc_wide.cu):
// one warp per edge, A[0][e] = ad, A[1][e] = as, fpos[e] = ad . t.
__global__ void k_gather_adjust(const uint32_t* __restrict__ edges, uint32_t nb, PartView pi, PartView pj,
                                const float* __restrict__ rel, int kind, uint32_t d, float* __restrict__ A,
                                float* __restrict__ fpos) {
    const uint32_t wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t e = blockIdx.x * (blockDim.x >> 5) + wib;
    if (e >= nb) return;
    const uint32_t s = edges[3 * e], r = edges[3 * e + 1], t = edges[3 * e + 2];
    const float* ss = node_row(pi, s, d);
    const float* st = node_row(pj, t, d);
    const float* sr = kind != EMBER_DOT ? rel + (uint64_t)r * d : nullptr;
    const uint32_t nq = d / 4;
    float part = 0.f;
    for (uint32_t q = lane; q < nq; q += 32) {
        const Quad S = load_quad(ss, q), T = load_quad(st, q);
        const Quad R = sr ? load_quad(sr, q) : S;
        Quad ad, as;
        adjust_quad(kind, S, R, T, ad, as);
#pragma unroll
        for (int i = 0; i < 4; ++i) part += ad.v[i] * T.v[i];
        store_quad(A + (uint64_t)e * d, q, ad);
        store_quad(A + ((uint64_t)nb + e) * d, q, as);
    }
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) fpos[e] = part;
}

// Negative rows: slot -> row (side 0 rows come from partition j, side 1 from i).
// PACKED: slots [0, 2 n_pad), zero past n_t per side; else fp32 N[slot] for slots < n.
template <bool PACKED>
__global__ void k_gather_negs(const uint32_t* __restrict__ negs, uint32_t n, uint32_t nt, uint32_t n_pad, PartView pi,
                              PartView pj, uint32_t d, uint32_t CB, float* __restrict__ N, uint16_t* __restrict__ Npk) {
    griddep_wait();
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (!PACKED) {
        if (w >= n) return;
        const uint32_t side = (w / nt) & 1u;
        const float* src = node_row(side == 0 ? pj : pi, negs[w], d);
        float4* dst = reinterpret_cast<float4*>(N + (uint64_t)w * d);
        for (uint32_t v = lane; v < d / 4; v += 32) dst[v] = ldg4(src + 4 * v);
        return;
    }
    negs_pack_warp(w, lane, negs, NegSampling{}, nt, n_pad, pi, pj, d, CB, Npk);
}

__device__ __forceinline__ uint32_t node_key(const KeySpace& ks, uint32_t id) {
    const uint64_t o = (uint64_t)id - ks.lo.first;
    return o < ks.lo.rows ? (uint32_t)o : (uint32_t)(ks.lo.rows + ((uint64_t)id - ks.hi.first));
}

// keys[slot] (slot layout: engine.h); the sort numbers the slots itself.
__global__ void k_keys(const uint32_t* __restrict__ edges, uint32_t nb, const uint32_t* __restrict__ negs,
                       uint32_t n_neg, uint32_t n_slots, KeySpace ks, uint32_t* keys, uint32_t* longs) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {  // long-segment list of this step's reduction
        longs[0] = 0u;
        longs[1] = 0u;
        longs[2] = 0u;
    }
    if (i >= n_slots) return;
    uint32_t k;
    if (i < nb) k = node_key(ks, edges[3 * i]);
    else if (i < 2 * nb) k = node_key(ks, edges[3 * (i - nb) + 2]);
    else if (i < 2 * nb + n_neg) k = node_key(ks, negs[i - 2 * nb]);
    else k = (uint32_t)ks.node_range + edges[3 * (i - 2 * nb - n_neg) + 1];
    keys[i] = k;
}

// The training step's first kernel: sample_negatives fused with the gradient-slot keys (the
// negative slots sample their id and key it at once). It runs on the step stream, so every read
// of the caller's batch / bucket is ordered after the caller's earlier work on that stream; only
// the key sort forks onto the helper stream.
__global__ void k_sample_keys(const uint32_t* __restrict__ edges, uint32_t nb, uint32_t* __restrict__ negs,
                              uint32_t n_neg, uint32_t nt, uint32_t n_deg, uint64_t base,
                              const uint32_t* __restrict__ bucket, uint64_t bucket_n, PartView src, PartView dst,
                              uint32_t n_slots, KeySpace ks, uint32_t* keys, uint32_t* longs) {
    griddep_wait();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {  // long-segment list of this step's reduction
        longs[0] = 0u;
        longs[1] = 0u;
        longs[2] = 0u;
    }
    if (i >= n_slots) return;
    uint32_t k;
    if (i < nb) {
        k = node_key(ks, edges[3 * i]);
    } else if (i < 2 * nb) {
        k = node_key(ks, edges[3 * (i - nb) + 2]);
    } else if (i < 2 * nb + n_neg) {
        const uint32_t id =
            sample_one(i - 2 * nb, nt, n_deg, base, bucket, bucket_n, src.first, src.rows, dst.first, dst.rows);
        negs[i - 2 * nb] = id;
        k = node_key(ks, id);
    } else {
        k = (uint32_t)ks.node_range + edges[3 * (i - 2 * nb - n_neg) + 1];
    }
    keys[i] = k;
}

// The sorted position p holds a key that occurs exactly once among the batch's gradient slots.
__device__ __forceinline__ bool slot_unique(const uint32_t* __restrict__ ks, uint32_t n, uint32_t p) {
    const uint32_t k = ks[p];
    return (p == 0 || ks[p - 1] != k) && (p + 1 == n || ks[p + 1] != k);
}

__device__ __forceinline__ void adagrad_one(float& th, float& ac, float g, float lr, float eps) {
    const float a = __fadd_rn(ac, __fmul_rn(g, g));
    ac = a;
    th = __fsub_rn(th, __fdiv_rn(__fmul_rn(lr, g), __fadd_rn(__fsqrt_rn(a), eps)));
}

// Adagrad of one quad of a row whose parameters Th were already loaded.
__device__ __forceinline__ void adagrad_quad(float* th_row, float* ac_row, uint32_t q, Quad Th, Quad Ac, const Quad& G,
                                             float lr, float eps) {
#pragma unroll
    for (int i = 0; i < 4; ++i) adagrad_one(Th.v[i], Ac.v[i], G.v[i], lr, eps);
    store_quad(th_row, q, Th);
    store_quad(ac_row, q, Ac);
}

// dA quad q of (side, edge e): column-blocked [2][d/4][dcap][4] (tensor-core engine) or
// row-major [2][nb][d] (SIMT engine, dcap == 0); its columns are the rows' HBM coordinates.
__device__ __forceinline__ Quad load_dA_quad(const float* __restrict__ dA, uint32_t dcap, uint32_t nb, uint32_t side,
                                             uint32_t e, uint32_t d, uint32_t q) {
    if (!dcap) return load_quad(dA + ((uint64_t)side * nb + e) * d, q);
    return load_quad(dA + ((uint64_t)side * (d / 4) + q) * dcap * 4 + (uint64_t)e * 4, 0);
}

// Chain rule (one warp per edge, lanes on quads in registers), adjusted vectors recomputed from
// the rows. dA excludes the positive term, added here:
//   grad adj_dst = g0_dst * t + dA_dst,  grad adj_src = g0_src * s + dA_src,
//   grad t += g0_dst * adj_dst (positive score = adj_dst . t), grad s += g0_src * adj_src.
// Rows go to their sorted positions: source -> grows[rank[e]], destination -> grows[rank[nb + e]],
// relation -> grows[rank[2nb + n_neg + e]].
__global__ void __launch_bounds__(256, 4) k_chain_rule(const uint32_t* __restrict__ edges, uint32_t nb, uint32_t n_neg, PartView pi,
                             PartView pj, const float* __restrict__ rel, int kind, uint32_t d,
                             const float* __restrict__ dA, uint32_t dcap, const float* __restrict__ g0,
                             const uint32_t* __restrict__ rank, float* __restrict__ grows,
                             const uint32_t* __restrict__ keys_sorted, uint32_t n_slots, int direct, float lr,
                             float eps) {
    const uint32_t wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t e = blockIdx.x * (blockDim.x >> 5) + wib;
    if (e >= nb) return;
    const uint32_t s = edges[3 * e], r = edges[3 * e + 1], t = edges[3 * e + 2];
    const float* ss = node_row(pi, s, d);
    const float* st = node_row(pj, t, d);
    const float* sr = kind != EMBER_DOT ? rel + (uint64_t)r * d : nullptr;
    const float gd = g0[e], gs = g0[(uint64_t)nb + e];
    const uint32_t ps = rank[e], pt = rank[nb + e];
    // A node row whose key occurs once in the batch (the common case) is final here: Adagrad is
    // applied in place (the row was just read), skipping the sorted-row round trip.
    const bool us = direct && slot_unique(keys_sorted, n_slots, ps);
    const bool ut = direct && slot_unique(keys_sorted, n_slots, pt);
    float* gS = grows + (uint64_t)ps * d;
    float* gT = grows + (uint64_t)pt * d;
    float* gR = kind != EMBER_DOT ? grows + (uint64_t)rank[2 * nb + n_neg + e] * d : nullptr;
    float* aS = pi.acc + (uint64_t)(s - pi.first) * d;
    float* aT = pj.acc + (uint64_t)(t - pj.first) * d;
    const uint32_t nq = d / 4;
    for (uint32_t q = lane; q < nq; q += 32) {
        const Quad S = load_quad(ss, q), T = load_quad(st, q);
        const Quad R = sr ? load_quad(sr, q) : S;
        const Quad U = load_dA_quad(dA, dcap, nb, 0, e, d, q);  // destination side
        const Quad W = load_dA_quad(dA, dcap, nb, 1, e, d, q);  // source side
        Quad AS, AT;  // accumulators, loaded with the rows (speculatively: used when the key is unique)
        if (direct) {
            AS = load_quad(aS, q);
            AT = load_quad(aT, q);
        }
        Quad ad, as, oS, oR, oT;
        adjust_quad(kind, S, R, T, ad, as);
        if (kind == EMBER_COMPLEX) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const float a = S.v[i], b = S.v[2 + i], c = R.v[i], ee = R.v[2 + i], x = T.v[i], y = T.v[2 + i];
                const float u0 = U.v[i] + gd * x, u1 = U.v[2 + i] + gd * y;
                const float w0 = W.v[i] + gs * a, w1 = W.v[2 + i] + gs * b;
                oS.v[i] = gs * as.v[i] + (u0 * c + u1 * ee);
                oS.v[2 + i] = gs * as.v[2 + i] + (u1 * c - u0 * ee);
                oR.v[i] = (u0 * a + u1 * b) + (w0 * x + w1 * y);
                oR.v[2 + i] = (u1 * a - u0 * b) + (w0 * y - w1 * x);
                oT.v[i] = gd * ad.v[i] + (w0 * c - w1 * ee);
                oT.v[2 + i] = gd * ad.v[2 + i] + (w0 * ee + w1 * c);
            }
        } else if (kind == EMBER_DISTMULT) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float uk = U.v[i] + gd * T.v[i], wk = W.v[i] + gs * S.v[i];
                oS.v[i] = gs * as.v[i] + uk * R.v[i];
                oR.v[i] = uk * S.v[i] + wk * T.v[i];
                oT.v[i] = gd * ad.v[i] + wk * R.v[i];
            }
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                oS.v[i] = gs * T.v[i] + (U.v[i] + gd * T.v[i]);
                oT.v[i] = gd * S.v[i] + (W.v[i] + gs * S.v[i]);
            }
        }
        if (us) adagrad_quad(const_cast<float*>(ss), aS, q, S, AS, oS, lr, eps);
        else store_quad(gS, q, oS);
        if (ut) adagrad_quad(const_cast<float*>(st), aT, q, T, AT, oT, lr, eps);
        else store_quad(gT, q, oT);
        if (gR) store_quad(gR, q, oR);
    }
}

// ---- software-pipelined chain rule (tensor-core engine, d <= 128: one quad per lane) ---------
// Persistent warps walk the edges e = gw, gw + nw, ...; while a warp computes edge e, the seven
// row quads of its next edge (theta_s, theta_t, theta_r, acc_s, acc_t, dA_dst, dA_src) are already
// in flight as cp.async copies into the lane's own shared-memory stage (double-buffered), so
// every warp keeps two edges' random rows outstanding without holding them in registers. The
// edge's indices, ranks, uniqueness flags and g0 are loaded with its copies (one latency).
constexpr int CP_ROLES = 7;  // S, T, R, acc_S, acc_T, U (dA dst), W (dA src)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tc::smem_addr(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// quad q of a row -> one float4 slot in shared memory
__device__ __forceinline__ void cp_quad(float4* dst, const float* row, uint32_t q) { cp_async16(dst, row + 4 * q); }

// dA quad q of (side, row e), column-blocked [2][d/4][dcap][4]
__device__ __forceinline__ void cp_dA_quad(float4* dst, const float* dA, uint32_t dcap, uint32_t side, uint32_t e,
                                           uint32_t d, uint32_t q) {
    cp_async16(dst, dA + ((uint64_t)side * (d / 4) + q) * dcap * 4 + (uint64_t)e * 4);
}

__device__ __forceinline__ Quad quad_of(const float4& v) {
    Quad x;
    x.v[0] = v.x, x.v[1] = v.y, x.v[2] = v.z, x.v[3] = v.w;
    return x;
}

struct EdgeMeta {
    uint32_t s, r, t, ps, pt, pr;
    uint32_t uq;  // bit 0: source row unique, bit 1: destination row unique
    float gd, gs;
    float lterm;  // the edge's loss term (lse_dst - f) + (lse_src - f)
};

template <int NS, int MINB>
__global__ void __launch_bounds__(256, MINB) k_chain_pipe(const uint32_t* __restrict__ edges, uint32_t nb, uint32_t n_neg,
                                                      PartView pi, PartView pj, const float* __restrict__ rel,
                                                      int kind, uint32_t d, const float* __restrict__ dA,
                                                      uint32_t dcap, const float* __restrict__ g0,
                                                      const uint32_t* __restrict__ rank,
                                                      const uint8_t* __restrict__ uniq, float* __restrict__ grows,
                                                      int direct, float lr, float eps,
                                                      const float* __restrict__ lse, const float* __restrict__ fpos,
                                                      double* __restrict__ loss_part, uint32_t* __restrict__ loss_done,
                                                      float* __restrict__ loss_out, unsigned long long* bad,
                                                      unsigned long long tag, DnReduce dn, int dn_on) {
    griddep_wait();
    if (dn_on) {  // the contraction's dN reduction first (independent of the edges below: other slots)
        if (blockIdx.x == 0 && threadIdx.x == 0) {  // overflow list consumed (tc_fixup_rows): count, reset
            dn.flags_total[0] += dn.flags[0];
            *dn.flags = 0u;
        }
        const int64_t total = (int64_t)dn.nsides * (dn.d / 4) * dn.nt, step = (int64_t)gridDim.x * blockDim.x;
        for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += step)
            dn_reduce_item(dn, t, rank, grows);
    }
    extern __shared__ float4 cpbuf[];  // [warps][NS stages][CP_ROLES][32 lanes]
    const uint32_t wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + wib, nw = gridDim.x * (blockDim.x >> 5);
    float4* my = cpbuf + (size_t)wib * NS * CP_ROLES * 32 + lane;
    const uint32_t nq = d / 4;
    const bool ql = lane < nq;
    // An edge's indices, ranks, flags and scalars are loaded one edge ahead of its row copies, so
    // the copies of edge e + nw are issued without waiting on those dependent loads.
    auto load_meta = [&](uint32_t e, EdgeMeta& m) {
        m.s = edges[3 * e];
        m.r = edges[3 * e + 1];
        m.t = edges[3 * e + 2];
        m.ps = rank[e];
        m.pt = rank[nb + e];
        m.pr = kind != EMBER_DOT ? rank[2 * nb + n_neg + e] : 0u;
        m.uq = direct ? (uint32_t)uniq[e] | ((uint32_t)uniq[nb + e] << 1) : 0u;
        m.gd = g0[e];
        m.gs = g0[(uint64_t)nb + e];
        {
            const float f = fpos[e];
            m.lterm = 0.f;
            if (lane == 0) m.lterm = (lse[e] - f) + (lse[(uint64_t)nb + e] - f);  // same terms as k_loss
        }
    };
    auto issue = [&](uint32_t e, int st, const EdgeMeta& m) {
        if (ql) {
            float4* b = my + (size_t)st * CP_ROLES * 32;
            cp_quad(b + 0 * 32, node_row(pi, m.s, d), lane);
            cp_quad(b + 1 * 32, node_row(pj, m.t, d), lane);
            if (kind != EMBER_DOT) cp_quad(b + 2 * 32, rel + (uint64_t)m.r * d, lane);
            if (m.uq & 1u) cp_quad(b + 3 * 32, pi.acc + (uint64_t)(m.s - pi.first) * d, lane);
            if (m.uq & 2u) cp_quad(b + 4 * 32, pj.acc + (uint64_t)(m.t - pj.first) * d, lane);
            cp_dA_quad(b + 5 * 32, dA, dcap, 0, e, d, lane);
            cp_dA_quad(b + 6 * 32, dA, dcap, 1, e, d, lane);
        }
        cp_commit();
    };
    // q[k]: the metadata of edge gw + (it + k) nw, whose copies sit in stage (it + k) % NS; each
    // iteration issues edge e + (NS - 1) nw into the stage the previous edge freed before waiting on
    // edge e, so NS edges are in flight through the wait and NS - 1 through the compute.
    // pre: the metadata one edge beyond the newest issued.
    EdgeMeta q[NS]{}, pre{};
#pragma unroll
    for (int k = 0; k + 1 < NS; ++k) {
        const uint32_t e = gw + k * nw;
        if (e < nb) {
            load_meta(e, q[k]);
            issue(e, k, q[k]);
        } else {
            cp_commit();
        }
    }
    if (gw + (NS - 1) * nw < nb) load_meta(gw + (NS - 1) * nw, q[NS - 1]);
    int st = 0;
    double lacc = 0.0;  // lane 0: this warp's loss terms, in its (fixed) edge order
    for (uint32_t e = gw; e < nb; e += nw) {
        const EdgeMeta& cur = q[0];
        lacc += (double)cur.lterm;
        const uint32_t en = e + (NS - 1) * nw;
        if (en < nb) issue(en, st == 0 ? NS - 1 : st - 1, q[NS - 1]);
        else cp_commit();
        if (en + nw < nb) load_meta(en + nw, pre);  // consumed next iteration
        cp_wait<NS - 1>();  // this edge's copies (this lane's own) have landed
        if (ql) {
            const float4* b = my + (size_t)st * CP_ROLES * 32;
            const Quad S = quad_of(b[0]), T = quad_of(b[32]);
            const Quad R = kind != EMBER_DOT ? quad_of(b[2 * 32]) : S;
            const Quad U = quad_of(b[5 * 32]), W = quad_of(b[6 * 32]);
            const float gd = cur.gd, gs = cur.gs;
            Quad ad, as, oS, oR, oT;
            adjust_quad(kind, S, R, T, ad, as);
            if (kind == EMBER_COMPLEX) {
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const float a = S.v[i], bb = S.v[2 + i], c = R.v[i], ee = R.v[2 + i], x = T.v[i], y = T.v[2 + i];
                    const float u0 = U.v[i] + gd * x, u1 = U.v[2 + i] + gd * y;
                    const float w0 = W.v[i] + gs * a, w1 = W.v[2 + i] + gs * bb;
                    oS.v[i] = gs * as.v[i] + (u0 * c + u1 * ee);
                    oS.v[2 + i] = gs * as.v[2 + i] + (u1 * c - u0 * ee);
                    oR.v[i] = (u0 * a + u1 * bb) + (w0 * x + w1 * y);
                    oR.v[2 + i] = (u1 * a - u0 * bb) + (w0 * y - w1 * x);
                    oT.v[i] = gd * ad.v[i] + (w0 * c - w1 * ee);
                    oT.v[2 + i] = gd * ad.v[2 + i] + (w0 * ee + w1 * c);
                }
            } else if (kind == EMBER_DISTMULT) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float uk = U.v[i] + gd * T.v[i], wk = W.v[i] + gs * S.v[i];
                    oS.v[i] = gs * as.v[i] + uk * R.v[i];
                    oR.v[i] = uk * S.v[i] + wk * T.v[i];
                    oT.v[i] = gd * ad.v[i] + wk * R.v[i];
                }
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    oS.v[i] = gs * T.v[i] + (U.v[i] + gd * T.v[i]);
                    oT.v[i] = gd * S.v[i] + (W.v[i] + gs * S.v[i]);
                }
            }
            float* thS = pi.theta + (uint64_t)(cur.s - pi.first) * d;
            float* thT = pj.theta + (uint64_t)(cur.t - pj.first) * d;
            if (cur.uq & 1u)
                adagrad_quad(thS, pi.acc + (uint64_t)(cur.s - pi.first) * d, lane, S, quad_of(b[3 * 32]), oS,
                             lr, eps);
            else
                store_quad(grows + (uint64_t)cur.ps * d, lane, oS);
            if (cur.uq & 2u)
                adagrad_quad(thT, pj.acc + (uint64_t)(cur.t - pj.first) * d, lane, T, quad_of(b[4 * 32]), oT,
                             lr, eps);
            else
                store_quad(grows + (uint64_t)cur.pt * d, lane, oT);
            if (kind != EMBER_DOT) store_quad(grows + (uint64_t)cur.pr * d, lane, oR);
        }
#pragma unroll
        for (int k = 0; k + 1 < NS; ++k) q[k] = q[k + 1];
        q[NS - 1] = pre;
        st = st + 1 == NS ? 0 : st + 1;
    }
    cp_wait<0>();
    // the loss (replaces k_loss): per-warp partials in warp order, summed by the last warp to finish
    // in a fixed lane / tree order (deterministic)
    __shared__ bool last_warp[8];
    if (lane == 0) {
        loss_part[gw] = lacc;
        __threadfence();
        last_warp[wib] = atomicAdd(loss_done, 1u) == nw - 1;
    }
    __syncwarp();
    if (!last_warp[wib]) return;
    __threadfence();
    double v = 0.0;
    for (uint32_t k = lane; k < nw; k += 32) v += ((volatile double*)loss_part)[k];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) {
        loss_out[0] = (float)(v / (double)nb);
        *loss_done = 0u;
        if (!isfinite(v)) atomicCAS(bad, 0ull, tag);  // SPEC.md:161, reported at the next sync
    }
}

// loss = (1/nb) sum_e (lse_dst - f) + (lse_src - f): each block sums a contiguous range in a fixed
// order, the last block to finish adds the block partials in index order (deterministic).
constexpr uint32_t LOSS_THREADS = 512;
__global__ void k_loss(const float* __restrict__ lse, const float* __restrict__ fpos, uint32_t nb, uint32_t per_block,
                       double* __restrict__ part, uint32_t* __restrict__ done, float* __restrict__ out,
                       unsigned long long* bad, unsigned long long tag) {
    griddep_wait();
    __shared__ double red[LOSS_THREADS];
    __shared__ bool last;
    const uint32_t b0 = blockIdx.x * per_block, b1 = min(nb, b0 + per_block);
    double acc = 0.0;
    for (uint32_t e = b0 + threadIdx.x; e < b1; e += blockDim.x)
        acc += (double)(lse[e] - fpos[e]) + (double)(lse[(uint64_t)nb + e] - fpos[e]);
    red[threadIdx.x] = acc;
    __syncthreads();
    for (uint32_t s = blockDim.x / 2; s; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[blockIdx.x] = red[0];
        __threadfence();
        last = atomicAdd(done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // the last block adds the block partials: loaded in parallel, reduced in a fixed tree order
    double v = 0.0;
    for (uint32_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) v += ((volatile double*)part)[b];
    red[threadIdx.x] = v;
    __syncthreads();
    for (uint32_t s = blockDim.x / 2; s; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = (float)(red[0] / (double)nb);
        *done = 0u;
        if (!isfinite(red[0])) atomicCAS(bad, 0ull, tag);  // SPEC.md:161, reported at the next sync
    }
}

__device__ __forceinline__ float adagrad_elem(float& th, float& ac, float g, float lr, float eps) {
    adagrad_one(th, ac, g, lr, eps);
    return th;
}

struct SegArgs {
    const uint32_t* ukeys;
    const uint32_t* offsets;
    const uint32_t* nruns;
    uint32_t* nunique;   // [2] written: node uniques, relation uniques
    uint32_t* longs;     // [0] long segments, [1] chunk slots, [2] active runs; then u, base, nch per long
    const uint32_t* act; // runs the segment kernel visits (k_long_plan), longs[2] of them; null: every run
    uint32_t* owner;     // chunk slot -> long index
    float* partial;      // chunk slot -> partial sum row
    uint32_t long_cap;
    int early_final;     // k_long_final scheduled once the segment kernel's CTAs have written the partials
    const float* rows;   // sorted gradient rows
    KeySpace ks;
    float* rel_theta;
    float* rel_acc;
    float* rel_dense;    // non-null: relation sums go here (summed over ranks later), no Adagrad
    const uint32_t* vals_sorted;  // sorted position -> gradient slot
    uint32_t direct_hi;  // node keys occurring once with slot < direct_hi were applied by their producer
    uint32_t d;
    float lr, eps;
    int apply;
    uint32_t* node_ids_out;
    float* node_rows_out;
    uint32_t* rel_ids_out;
    float* rel_rows_out;
    int part;                 // 0 every key; 1 relation keys [nsplit, nr); 2 node keys [0, nsplit)
    const uint32_t* nsplit;   // first relation run (~0u: none)
};

// The unique keys this launch reduces: [lo, hi) of the nr runs.
__device__ __forceinline__ void seg_range(const SegArgs& a, uint32_t nr, uint32_t& lo, uint32_t& hi) {
    const uint32_t split = min(*a.nsplit, nr);
    lo = a.part == 1 ? split : 0u;
    hi = a.part == 2 ? split : nr;
}

// A long segment's key belongs to this launch's part.
__device__ __forceinline__ bool seg_in_part(const SegArgs& a, uint32_t u) {
    if (a.part == 0) return true;
    const bool rel = a.ukeys[u] >= a.ks.node_range;
    return a.part == 1 ? rel : !rel;
}

// Segments longer than LONG_SEG rows (hot relations, hub nodes) are cut into LONG_CHUNK-row chunks
// summed by separate warps; a block per long segment then adds the chunk partials in a fixed
// order (stream s of 2 LONG_WARPS takes chunks s, s + 2 LONG_WARPS, ...; the stream sums are then added
// in stream order): deterministic.
constexpr uint32_t LONG_SEG = EMBER_LONG_SEG;
constexpr uint32_t LONG_CHUNK = EMBER_LONG_CHUNK;
constexpr uint32_t LONG_WARPS = 16;
constexpr uint32_t LONG_HDR = 3;  // longs[]: header words before the long-segment records

// Where unique key u's summed row goes: Adagrad target (th, ac) or export/dense destination.
struct SegTarget {
    float* th;
    float* ac;
    float* out;  // export / dense row (may be null)
    bool node;
};

__device__ __forceinline__ uint32_t n_node_unique(const SegArgs& a, uint32_t nr) {
    uint32_t lo = 0, hi = nr;  // first u with key >= node_range
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a.ukeys[mid] < a.ks.node_range) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ SegTarget seg_target(const SegArgs& a, uint32_t u, uint32_t nr, bool write_id) {
    SegTarget t{nullptr, nullptr, nullptr, true};
    const uint32_t key = a.ukeys[u];
    const uint32_t d = a.d;
    if (key < a.ks.node_range) {
        const bool lo = key < a.ks.lo.rows;
        const PartView& v = lo ? a.ks.lo : a.ks.hi;
        const uint64_t row = lo ? key : key - a.ks.lo.rows;
        t.th = v.theta + row * d;
        t.ac = v.acc + row * d;
        if (!a.apply) {
            if (a.node_rows_out) t.out = a.node_rows_out + (uint64_t)u * d;
            if (write_id && a.node_ids_out) a.node_ids_out[u] = (uint32_t)(v.first + row);
        }
    } else {
        t.node = false;
        const uint32_t r = key - (uint32_t)a.ks.node_range;
        t.th = a.rel_theta + (uint64_t)r * d;
        t.ac = a.rel_acc + (uint64_t)r * d;
        if (a.rel_dense) {
            t.out = a.rel_dense + (uint64_t)r * d;
        } else if (!a.apply) {
            const uint32_t k = u - n_node_unique(a, nr);
            if (a.rel_rows_out) t.out = a.rel_rows_out + (uint64_t)k * d;
            if (write_id && a.rel_ids_out) a.rel_ids_out[k] = r;
        }
    }
    return t;
}

__device__ __forceinline__ bool seg_applies(const SegArgs& a, const SegTarget& t) {
    return a.apply && !(!t.node && a.rel_dense);
}

// g: the summed gradient of columns 4*c4..4*c4+3; th/ac: the preloaded parameter/accumulator.
__device__ __forceinline__ void seg_finish(const SegArgs& a, const SegTarget& t, uint32_t c4, float4 g, float4 th,
                                           float4 ac) {
    if (t.out) reinterpret_cast<float4*>(t.out)[c4] = g;
    if (!seg_applies(a, t)) return;
    adagrad_elem(th.x, ac.x, g.x, a.lr, a.eps);
    adagrad_elem(th.y, ac.y, g.y, a.lr, a.eps);
    adagrad_elem(th.z, ac.z, g.z, a.lr, a.eps);
    adagrad_elem(th.w, ac.w, g.w, a.lr, a.eps);
    reinterpret_cast<float4*>(t.th)[c4] = th;
    reinterpret_cast<float4*>(t.ac)[c4] = ac;
}

__device__ __forceinline__ void add4(float4& s, const float4& x) {
    s.x += x.x;
    s.y += x.y;
    s.z += x.z;
    s.w += x.w;
}


// Sum of rows [0, cnt) at column blocks c4a and c4b (c4b valid iff hasb), in row order, 4 loads
// in flight.
__device__ __forceinline__ void sum_rows2(const float* base, uint32_t cnt, uint32_t d, uint32_t c4a, uint32_t c4b,
                                          bool hasb, float4& sa, float4& sb) {
    sa = make_float4(0.f, 0.f, 0.f, 0.f);
    sb = sa;
    uint32_t r = 0;
    for (; r + 2 <= cnt; r += 2) {
        const float4 x0 = ldg4(base + (uint64_t)r * d + 4 * c4a);
        const float4 x1 = ldg4(base + (uint64_t)(r + 1) * d + 4 * c4a);
        float4 y0 = sb, y1 = sb;
        if (hasb) {
            y0 = ldg4(base + (uint64_t)r * d + 4 * c4b);
            y1 = ldg4(base + (uint64_t)(r + 1) * d + 4 * c4b);
        }
        add4(sa, x0);
        add4(sa, x1);
        if (hasb) {
            add4(sb, y0);
            add4(sb, y1);
        }
    }
    if (r < cnt) {
        add4(sa, ldg4(base + (uint64_t)r * d + 4 * c4a));
        if (hasb) add4(sb, ldg4(base + (uint64_t)r * d + 4 * c4b));
    }
}

// Two unique keys per warp, one per 16-lane half (more independent rows in flight per warp): the
// half sums its key's contiguous rows (slot order) and applies Adagrad / export. A lane owns
// column blocks c4 and c4 + 16 (d <= 128; larger d loops).
constexpr uint32_t SEG_LANES = 16;
__device__ __forceinline__ void long_partials(const SegArgs& a, uint32_t gw, uint32_t nw, uint32_t lane);

__global__ void __launch_bounds__(256, 4) k_segments(const __grid_constant__ SegArgs a) {
    griddep_wait();
    const uint32_t lane = threadIdx.x & 31, hl = lane & (SEG_LANES - 1);
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t u = gw * 2 + (lane >> 4);
    long_partials(a, gw, (gridDim.x * blockDim.x) >> 5, lane);  // the long segments' chunk partials first
    const uint32_t nr = *a.nruns;
    uint32_t lo, hi;
    seg_range(a, nr, lo, hi);
    if (u < lo || u >= hi) return;
    const uint32_t key = a.ukeys[u];
    const uint32_t off = a.offsets[u], cnt = a.offsets[u + 1] - off;
    if (cnt == 1 && key < a.ks.node_range && a.vals_sorted[off] < a.direct_hi) return;  // applied already
    if (cnt > LONG_SEG) return;  // chunked (long_partials, k_long_final)
    const SegTarget t = seg_target(a, u, nr, hl == 0);
    const bool app = seg_applies(a, t);
    const float* base = a.rows + (uint64_t)off * a.d;
    const uint32_t d4 = a.d / 4;
    for (uint32_t c4 = hl; c4 < d4; c4 += 2 * SEG_LANES) {
        const uint32_t c4b = c4 + SEG_LANES;
        const bool hasb = c4b < d4;
        float4 tha = make_float4(0.f, 0.f, 0.f, 0.f), aca = tha, thb = tha, acb = tha;
        if (app) {  // issue the parameter loads before the row sums
            tha = reinterpret_cast<const float4*>(t.th)[c4];
            aca = reinterpret_cast<const float4*>(t.ac)[c4];
            if (hasb) {
                thb = reinterpret_cast<const float4*>(t.th)[c4b];
                acb = reinterpret_cast<const float4*>(t.ac)[c4b];
            }
        }
        float4 ga, gb;
        sum_rows2(base, cnt, a.d, c4, c4b, hasb, ga, gb);
        seg_finish(a, t, c4, ga, tha, aca);
        if (hasb) seg_finish(a, t, c4b, gb, thb, acb);
    }
}

// Persistent version for d <= 128: each 16-lane half-warp walks the unique keys u = gh, gh + nh, ...
// and, while it sums the current key's rows, the next key's theta / acc quads are already in
// flight (cp.async into the lane's own stage), so the random parameter reads of two keys overlap.
// Same arithmetic and order as k_segments (bit-identical results).
struct SegKey {
    uint32_t u, off, cnt;
    bool active;
    SegTarget t;
};

struct SegMeta {
    uint32_t u, key, off, cnt;
};

__global__ void __launch_bounds__(256, 4) k_segments_pipe(const __grid_constant__ SegArgs a) {
    griddep_wait();
    long_partials(a, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, (gridDim.x * blockDim.x) >> 5,
                  threadIdx.x & 31);  // the long segments' chunk partials first
    // k_long_final only needs the partials: once every CTA is past this point it may be scheduled
    // on the SMs this grid's tail leaves idle (it reads them through L2 and waits for this grid
    // before it completes)
    if (a.early_final) {  // every warp of the CTA past its partials (fenced) before the CTA triggers
        __threadfence();
        __syncthreads();
        griddep_launch();
    }
    extern __shared__ float4 sst[];  // [warps][2 halves][2 stages][2 roles][2 column blocks][16 lanes]
    const uint32_t lane = threadIdx.x & 31, hl = lane & (SEG_LANES - 1), half = lane >> 4, wib = threadIdx.x >> 5;
    const uint32_t gh = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 2 + half;
    const uint32_t nh = ((gridDim.x * blockDim.x) >> 5) * 2;
    const uint32_t nr = *a.nruns, d4 = a.d / 4;
    uint32_t u_lo, u_hi;
    seg_range(a, nr, u_lo, u_hi);
    float4* my = sst + (size_t)(wib * 2 + half) * 2 * 2 * 2 * SEG_LANES + hl;
    auto slot = [&](int st, int role, int cb) { return my + (size_t)((st * 2 + role) * 2 + cb) * SEG_LANES; };
    // The runs this half-warp visits: the plan's list of runs with work (k_long_plan), else every
    // run of the part. A run's (key, offset, count) are loaded one run ahead of its parameter copies,
    // so the copies of run i + nh are issued without waiting on those loads.
    const bool list = a.act != nullptr;
    const uint32_t n_items = list ? *(volatile uint32_t*)&a.longs[2] : u_hi - u_lo;
    auto load_meta = [&](uint32_t i, SegMeta& m) {
        m.u = list ? a.act[i] : u_lo + i;
        m.key = a.ukeys[m.u];
        m.off = a.offsets[m.u];
        m.cnt = a.offsets[m.u + 1] - m.off;
    };
    auto issue = [&](uint32_t i, int st, const SegMeta& m, SegKey& k) {
        k.u = m.u;
        k.active = false;
        if (i < n_items && m.u >= u_lo && m.u < u_hi) {
            const uint32_t key = m.key;
            k.off = m.off;
            k.cnt = m.cnt;
            const bool done = k.cnt > LONG_SEG ||  // chunked (long_partials)
                              (!list && k.cnt == 1 && key < a.ks.node_range &&
                               a.vals_sorted[k.off] < a.direct_hi);  // applied by the chain rule
            if (!done) {
                k.active = true;
                k.t = seg_target(a, m.u, nr, hl == 0);
                if (seg_applies(a, k.t))
                    for (int cb = 0; cb < 2; ++cb) {
                        const uint32_t c4 = hl + cb * SEG_LANES;
                        if (c4 < d4) {
                            cp_async16(slot(st, 0, cb), k.t.th + 4 * c4);
                            cp_async16(slot(st, 1, cb), k.t.ac + 4 * c4);
                        }
                    }
            }
        }
        cp_commit();
    };
    SegKey cur, nxt;
    SegMeta mn{}, mnn{};
    if (gh < n_items) load_meta(gh, mn);
    issue(gh, 0, mn, cur);
    if (gh + nh < n_items) load_meta(gh + nh, mn);
    for (uint32_t i = gh, it = 0; i < n_items; i += nh, ++it) {
        const int st = it & 1;
        issue(i + nh, st ^ 1, mn, nxt);
        if (i + 2 * nh < n_items) load_meta(i + 2 * nh, mnn);  // consumed next iteration
        cp_wait<1>();
        if (cur.active) {
            const bool app = seg_applies(a, cur.t);
            const float* base = a.rows + (uint64_t)cur.off * a.d;
            const uint32_t c4 = hl, c4b = hl + SEG_LANES;
            const bool hasa = c4 < d4, hasb = c4b < d4;
            if (hasa) {
                float4 ga, gb;
                sum_rows2(base, cur.cnt, a.d, c4, c4b, hasb, ga, gb);
                const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
                seg_finish(a, cur.t, c4, ga, app ? *slot(st, 0, 0) : z, app ? *slot(st, 1, 0) : z);
                if (hasb) seg_finish(a, cur.t, c4b, gb, app ? *slot(st, 0, 1) : z, app ? *slot(st, 1, 1) : z);
            }
        }
        cur = nxt;
        mn = mnn;
    }
    cp_wait<0>();
}


// The same for two column blocks at once (c4a, and c4b when hasb): 8 loads in flight, and per
// column the same row order (bit-identical to two sum_rows_strided passes).
// CG: loads through L2 only (rows written by a grid that may still be running: k_long_final)
template <bool CG = false>
__device__ __forceinline__ float4 ld4(const float* p) {
    return CG ? __ldcg(reinterpret_cast<const float4*>(p)) : __ldg(reinterpret_cast<const float4*>(p));
}
template <bool CG = false>
__device__ __forceinline__ void sum_rows_strided2(const float* base, uint32_t r0, uint32_t step, uint32_t cnt,
                                                  uint32_t d, uint32_t c4a, uint32_t c4b, bool hasb, float4& sa,
                                                  float4& sb) {
    sa = make_float4(0.f, 0.f, 0.f, 0.f);
    sb = sa;
    uint32_t r = r0;
    for (; r + 3 * step < cnt; r += 4 * step) {
        float4 x[4], y[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = ld4<CG>(base + (uint64_t)(r + i * step) * d + 4 * c4a);
        if (hasb) {
#pragma unroll
            for (int i = 0; i < 4; ++i) y[i] = ld4<CG>(base + (uint64_t)(r + i * step) * d + 4 * c4b);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) add4(sa, x[i]);
        if (hasb) {
#pragma unroll
            for (int i = 0; i < 4; ++i) add4(sb, y[i]);
        }
    }
    for (; r < cnt; r += step) {
        add4(sa, ld4<CG>(base + (uint64_t)r * d + 4 * c4a));
        if (hasb) add4(sb, ld4<CG>(base + (uint64_t)r * d + 4 * c4b));
    }
}

__device__ __forceinline__ float4 shfl_xor4(float4 v, int m) {
    v.x = __shfl_xor_sync(0xffffffffu, v.x, m);
    v.y = __shfl_xor_sync(0xffffffffu, v.y, m);
    v.z = __shfl_xor_sync(0xffffffffu, v.z, m);
    v.w = __shfl_xor_sync(0xffffffffu, v.w, m);
    return v;
}

// One warp per chunk slot of the long segments: partial[slot] = sum of its <= LONG_CHUNK rows;
// the two half-warps take the even and the odd rows, then even + odd (fixed order).
// Warp gw's share of the long segments' chunk partials (the segment kernels' prologue):
// partial[slot] = sum of its <= LONG_CHUNK rows; the two half-warps take the even and the odd rows,
// then even + odd (fixed order). The chunk plan comes from k_long_plan (helper stream, after the sort).
__device__ __forceinline__ void long_partials(const SegArgs& a, uint32_t gw, uint32_t nw, uint32_t lane) {
    const uint32_t hl = lane & 15, half = lane >> 4, d4 = a.d / 4;
    const uint32_t n_slots = a.longs[1];
    for (uint32_t sl = gw; sl < n_slots; sl += nw) {
        const uint32_t* rec = a.longs + LONG_HDR + 3 * a.owner[sl];
        const uint32_t u = rec[0], c = sl - rec[1];
        if (!seg_in_part(a, u)) continue;  // warp-uniform: reduced by the other launch
        const uint32_t r0 = c * LONG_CHUNK, cnt = min(LONG_CHUNK, a.offsets[u + 1] - a.offsets[u] - r0);
        const float* base = a.rows + ((uint64_t)a.offsets[u] + r0) * a.d;
        for (uint32_t c0 = 0; c0 < d4; c0 += 32) {  // warp-uniform trip count (shuffles below)
            const uint32_t c4 = c0 + hl, c4b = c4 + 16;
            const bool hasa = c4 < d4, hasb = c4b < d4;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f), vb = v;
            if (hasa) sum_rows_strided2(base, half, 2, cnt, a.d, c4, c4b, hasb, v, vb);
            const float4 o = shfl_xor4(v, 16), ob = shfl_xor4(vb, 16);
            if (half == 0) {  // even rows + odd rows
                float4* out = reinterpret_cast<float4*>(a.partial + (uint64_t)sl * a.d);
                if (hasa) {
                    add4(v, o);
                    out[c4] = v;
                }
                if (hasb) {
                    add4(vb, ob);
                    out[c4b] = vb;
                }
            }
        }
    }
}

// The reduction's plan, on the helper stream after the sort (thread per run): keys with more than
// LONG_SEG rows get LONG_CHUNK-row chunk slots (record (u, base, nch), owner per slot); the other
// runs the segment kernel has work for (repeated keys, relations, node keys whose single row was not
// applied by the chain rule: slot >= direct) are listed in act (any order: each run is reduced
// alone, in its fixed row order), so its warps skip the runs the chain rule already applied.
__global__ void k_long_plan(const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ nruns, uint32_t n_max,
                            const uint32_t* __restrict__ ukeys, const uint32_t* __restrict__ vals_sorted,
                            uint64_t node_range, uint32_t direct, const uint32_t* __restrict__ nsplit,
                            uint32_t* __restrict__ nunique, uint32_t* __restrict__ longs,
                            uint32_t* __restrict__ owner, uint32_t* __restrict__ act) {
    griddep_wait();
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t nr = *nruns;
    if (u == 0) {  // runs of node keys / of relation keys (the sort's first run with key >= node_range)
        const uint32_t split = min(*nsplit, nr);
        nunique[0] = split;
        nunique[1] = nr - split;
    }
    if (u >= nr || u >= n_max) return;
    const uint32_t off = offsets[u], cnt = offsets[u + 1] - off;
    if (cnt <= LONG_SEG) {
        if (cnt == 1 && ukeys[u] < node_range && vals_sorted[off] < direct) return;  // applied by the chain rule
        act[atomicAdd(&longs[2], 1u)] = u;
        return;
    }
    const uint32_t nch = (cnt + LONG_CHUNK - 1) / LONG_CHUNK;
    const uint32_t li = atomicAdd(&longs[0], 1u);
    const uint32_t base = atomicAdd(&longs[1], nch);
    uint32_t* rec = longs + LONG_HDR + 3 * li;
    rec[0] = u;
    rec[1] = base;
    rec[2] = nch;
    for (uint32_t c = 0; c < nch; ++c) owner[base + c] = li;
}

// One block per long segment: 2 * LONG_WARPS half-warp streams each add the chunk partials
// c = stream, stream + 2 LONG_WARPS, ... (in order); warp 0 then adds the stream sums in stream
// order (a fixed two-level order: deterministic) and applies Adagrad / export.
constexpr uint32_t LONG_BIG = 8;  // long segments with more chunk partials than this get a whole block

__device__ __forceinline__ void long_final_body(const SegArgs& a) {
    extern __shared__ float4 wsum[];  // [2 * LONG_WARPS][d/4]
    const uint32_t lane = threadIdx.x & 31, hl = lane & 15, stream = threadIdx.x >> 4, d4 = a.d / 4;
    const uint32_t NS = 2 * LONG_WARPS;
    const uint32_t n_long = *(volatile uint32_t*)&a.longs[0], nr = *a.nruns;
    // big segments (hot relations): a block each, 2 LONG_WARPS half-warp streams
    for (uint32_t li = blockIdx.x; li < n_long; li += gridDim.x) {
        const uint32_t* rec = a.longs + LONG_HDR + 3 * li;
        const uint32_t u = rec[0], base = rec[1], nch = rec[2];
        if (nch <= LONG_BIG || !seg_in_part(a, u)) continue;  // block-uniform
        for (uint32_t c4 = hl; c4 < d4; c4 += 32) {
            float4 va, vb;
            sum_rows_strided2<true>(a.partial + (uint64_t)base * a.d, stream, NS, nch, a.d, c4, c4 + 16, c4 + 16 < d4, va, vb);
            wsum[stream * d4 + c4] = va;
            if (c4 + 16 < d4) wsum[stream * d4 + c4 + 16] = vb;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            const SegTarget t = seg_target(a, u, nr, lane == 0);
            const bool app = seg_applies(a, t);
            for (uint32_t c4 = lane; c4 < d4; c4 += 32) {
                float4 th = make_float4(0.f, 0.f, 0.f, 0.f), ac = th;
                if (app) {
                    th = reinterpret_cast<const float4*>(t.th)[c4];
                    ac = reinterpret_cast<const float4*>(t.ac)[c4];
                }
                float4 g = wsum[c4];
                for (uint32_t k = 1; k < NS; ++k) add4(g, wsum[k * d4 + c4]);
                seg_finish(a, t, c4, g, th, ac);
            }
        }
        __syncthreads();
    }
    // the many small ones: a warp each (even / odd chunk streams, then their sum)
    const uint32_t half = lane >> 4, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t li = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; li < n_long; li += nw) {
        const uint32_t* rec = a.longs + LONG_HDR + 3 * li;
        const uint32_t u = rec[0], base = rec[1], nch = rec[2];
        if (nch > LONG_BIG || !seg_in_part(a, u)) continue;  // warp-uniform
        const SegTarget t = seg_target(a, u, nr, lane == 0);
        const bool app = seg_applies(a, t);
        for (uint32_t c0 = 0; c0 < d4; c0 += 32) {  // warp-uniform trip count (shuffles below)
            const uint32_t c4 = c0 + hl, c4b = c4 + 16;
            const bool hasa = c4 < d4, hasb = c4b < d4;
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            float4 th = z, ac = z, thb = z, acb = z;
            if (app && half == 0) {
                if (hasa) {
                    th = reinterpret_cast<const float4*>(t.th)[c4];
                    ac = reinterpret_cast<const float4*>(t.ac)[c4];
                }
                if (hasb) {
                    thb = reinterpret_cast<const float4*>(t.th)[c4b];
                    acb = reinterpret_cast<const float4*>(t.ac)[c4b];
                }
            }
            float4 g = z, gb = z;
            if (hasa) sum_rows_strided2<true>(a.partial + (uint64_t)base * a.d, half, 2, nch, a.d, c4, c4b, hasb, g, gb);
            const float4 o = shfl_xor4(g, 16), ob = shfl_xor4(gb, 16);
            if (half == 0) {
                if (hasa) {
                    add4(g, o);
                    seg_finish(a, t, c4, g, th, ac);
                }
                if (hasb) {
                    add4(gb, ob);
                    seg_finish(a, t, c4b, gb, thb, acb);
                }
            }
        }
    }
}

__global__ void __launch_bounds__(32 * LONG_WARPS) k_long_final(SegArgs a) {
    if (!a.early_final) griddep_wait();
    long_final_body(a);
    if (a.early_final) griddep_wait();  // not complete before the segment kernel: stream order for what follows
}

__global__ void k_adagrad_rows(const uint32_t* __restrict__ ids, const float* __restrict__ rows, uint32_t n,
                               uint32_t d, int kind, PartView pi, PartView pj, int relations, float* rel_theta, float* rel_acc,
                               uint32_t n_rel, float lr, float eps, uint32_t* bad) {
    const uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (u >= n) return;
    const uint32_t key = ids[u];
    float* th;
    float* ac;
    if (relations) {
        if (key >= n_rel) {  // out of range: counted, never written
            if (lane == 0) atomicAdd(bad, 1u);
            return;
        }
        th = rel_theta + (uint64_t)key * d;
        ac = rel_acc + (uint64_t)key * d;
    } else {
        if (key - pi.first >= pi.rows && key - pj.first >= pj.rows) {
            if (lane == 0) atomicAdd(bad, 1u);
            return;
        }
        const PartView& v = (key - pi.first < pi.rows) ? pi : pj;
        th = v.theta + (uint64_t)(key - v.first) * d;
        ac = v.acc + (uint64_t)(key - v.first) * d;
    }
    for (uint32_t c = lane; c < d; c += 32) {  // c: on-disk coordinate of the caller's row
        const uint32_t k = hbm_pos(kind, d, c);
        adagrad_elem(th[k], ac[k], rows[(uint64_t)u * d + c], lr, eps);
    }
}

// Warp per (row, negative): debug scores for parity tests.
__global__ void k_debug_scores(const float* A, const float* N, uint32_t rows, uint32_t nt, uint32_t d, float* out) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows * nt) return;
    const uint32_t r = w / nt, k = w % nt;
    float acc = 0.f;
    for (uint32_t c = lane; c < d; c += 32) acc += A[(uint64_t)r * d + c] * N[(uint64_t)k * d + c];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[w] = acc;
}

// Row r's draws are its coordinates in on-disk order; each lands at its HBM
// position (hbm_pos: ComplEx pair interleave).
__global__ void k_init_rows(float* theta, float* acc, uint64_t first, uint64_t rows, uint32_t d, int kind,
                            uint64_t seed, float a) {
    const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    Rng g(mix_seed(seed, first + r));
    float* out = theta + r * d;
    if (kind == EMBER_COMPLEX) {
        for (uint32_t c = 0; c < d; ++c) out[hbm_pos(kind, d, c)] = g.uniform(-a, a);
    } else {
        for (uint32_t k = 0; k < d; k += 4) {
            float4 v;
            v.x = g.uniform(-a, a);
            v.y = g.uniform(-a, a);
            v.z = g.uniform(-a, a);
            v.w = g.uniform(-a, a);
            reinterpret_cast<float4*>(out)[k / 4] = v;
        }
    }
    if (acc)
        for (uint32_t k = 0; k < d; k += 4) reinterpret_cast<float4*>(acc + r * d)[k / 4] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// Rows between the on-disk coordinate order and the HBM layout (in place, a warp per row; no-op
// unless ComplEx). n_dev (nullable): the row count is read on the device (export buffers whose
// length the step produced).
__global__ void k_rows_layout(float* rows, uint64_t n, const uint32_t* n_dev, uint32_t d, int to_hbm) {
    extern __shared__ float rl_tmp[];  // [warps][d]
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wib;
    const uint64_t cnt = n_dev ? (uint64_t)*n_dev : n;
    if (r >= cnt) return;
    float* row = rows + r * d;
    float* t = rl_tmp + (size_t)wib * d;
    for (uint32_t c = lane; c < d; c += 32) t[c] = row[c];
    __syncwarp();
    for (uint32_t c = lane; c < d; c += 32) {
        const uint32_t p = hbm_pos(EMBER_COMPLEX, d, c);
        if (to_hbm) row[p] = t[c];
        else row[c] = t[p];
    }
}


}  // namespace

// Dynamic shared memory above 48 KB needs a per-kernel opt-in, and the attribute is per device:
// remember the largest size set per (kernel, device) (several contexts / GPUs in one process).
void opt_in_smem(const void* fn, size_t bytes, int device) {
    if (bytes <= 48 * 1024) return;
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = done[{fn, device}];
    if (bytes <= have) return;
    EMBER_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    have = bytes;
}

void launch_sample(const Engine& E, uint32_t* out, uint64_t base, const uint32_t* bucket, uint64_t bucket_n,
                   const PartView& src, const PartView& dst) {
    const uint32_t n_deg = (uint32_t)ceil((double)E.m.alpha * (double)E.nt);
    const uint32_t total = E.n_neg;
    if (!total) return;
    launch_pdl(k_sample, dim3((total + 255) / 256), dim3(256), 0, E.stream, out, E.nt, n_deg, total, base, bucket,
               bucket_n, src.first, src.rows, dst.first, dst.rows);
    EMBER_LAUNCHED(E);
}

void launch_sample_on(const Engine& E, cudaStream_t st, uint32_t* out, uint64_t base, const uint32_t* bucket,
                      uint64_t bucket_n, const PartView& src, const PartView& dst) {
    const uint32_t n_deg = (uint32_t)ceil((double)E.m.alpha * (double)E.nt);
    const uint32_t total = E.n_neg;
    if (!total) return;
    k_sample<<<(total + 255) / 256, 256, 0, st>>>(out, E.nt, n_deg, total, base, bucket, bucket_n, src.first, src.rows,
                                                   dst.first, dst.rows);
    EMBER_LAUNCHED(E);
}

void launch_gather_adjust(const Engine& E, const uint32_t* edges, uint32_t nb, const PartView& pi, const PartView& pj,
                          bool packed, const uint32_t* negs) {
    if (packed) {
        const uint32_t rows_pad = (uint32_t)Engine::pad_rows(nb);  // a multiple of GP_ROWS
        const uint32_t row_ctas = rows_pad / GP_ROWS, neg_ctas = (2 * E.n_pad + GP_WARPS - 1) / GP_WARPS;
        const size_t sm = (size_t)4 * E.CB * GP_ROWS * 16;
        opt_in_smem((const void*)k_gather_pack, sm, E.device);
        NegSampling ns;
        if (E.neg_inline.on) {  // the step's negatives drawn here (k_sample_keys runs on the helper stream)
            ns.on = 1;
            ns.base = E.neg_inline.base;
            ns.bucket = E.neg_inline.bucket;
            ns.bucket_n = E.neg_inline.bucket_n;
            ns.n_deg = (uint32_t)ceil((double)E.m.alpha * (double)E.nt);
        }
        launch_pdl(k_gather_pack, dim3(row_ctas + neg_ctas), dim3(32 * GP_WARPS), sm, E.stream, edges, nb, pi, pj,
                   E.rel_theta, E.m.kind, E.dim, E.CB, (uint32_t)E.b_cap, E.s.Apk, E.s.fpos, row_ctas,
                   negs, ns, E.nt, (uint32_t)E.n_pad, E.s.Npk);
    } else {
        const uint32_t warps = 8;
        k_gather_adjust<<<(nb + warps - 1) / warps, warps * 32, 0, E.stream>>>(edges, nb, pi, pj, E.rel_theta,
                                                                                E.m.kind, E.dim, E.s.A, E.s.fpos);
    }
    EMBER_LAUNCHED(E);
}

void launch_gather_pack_wide(const Engine& E, const uint32_t* edges, uint32_t nb, const PartView& pi, const PartView& pj,
                             uint16_t* Apk, uint32_t CBA, uint32_t cap, uint32_t CP, uint32_t cr) {
    const size_t sm = (size_t)4 * CBA * GW_ROWS * 16;
    opt_in_smem((const void*)k_gather_pack_wide, sm, E.device);
    launch_pdl(k_gather_pack_wide, dim3(cap / GW_ROWS), dim3(32 * GW_ROWS), sm, E.stream, edges, nb, pi, pj,
               (const float*)E.rel_theta, E.m.kind, E.dim, CBA, cap, CP, cr, Apk, E.s.fpos);
    EMBER_LAUNCHED(E);
}

void launch_gather_negatives(const Engine& E, const uint32_t* negs, const PartView& pi, const PartView& pj,
                             bool packed) {
    if (!E.n_neg) return;
    if (packed) return;  // packed by k_gather_pack's trailing CTAs
    const uint32_t warps = packed ? 2 * E.n_pad : E.n_neg;
    if (packed)
        launch_pdl(k_gather_negs<true>, dim3((warps * 32 + 255) / 256), dim3(256), 0, E.stream, negs, E.n_neg, E.nt,
                   (uint32_t)E.n_pad, pi, pj, E.dim, E.CB, (float*)nullptr, E.s.Npk);
    else
        k_gather_negs<false><<<(warps * 32 + 255) / 256, 256, 0, E.stream>>>(negs, E.n_neg, E.nt, 0, pi, pj, E.dim, 0,
                                                                             E.s.N, nullptr);
    EMBER_LAUNCHED(E);
}

void launch_keys(const Engine& E, const uint32_t* edges, uint32_t nb, const uint32_t* negs, const KeySpace& ks) {
    const uint32_t n = E.slots(nb);
    k_keys<<<(n + 255) / 256, 256, 0, E.side>>>(edges, nb, negs, E.n_neg, n, ks, E.s.keys, E.s.longs);
    EMBER_LAUNCHED(E);
}

void launch_sample_keys(const Engine& E, const uint32_t* edges, uint32_t nb, uint64_t base, const uint32_t* bucket,
                        uint64_t bucket_n, const PartView& src, const PartView& dst, const KeySpace& ks,
                        cudaStream_t st) {
    const uint32_t n = E.slots(nb);
    const uint32_t n_deg = (uint32_t)ceil((double)E.m.alpha * (double)E.nt);
    launch_pdl(k_sample_keys, dim3((n + 255) / 256), dim3(256), 0, st ? st : E.stream, edges, nb, E.s.negs, E.n_neg,
               E.nt, n_deg,
               base, bucket, bucket_n, src, dst, n, ks, E.s.keys, E.s.longs);
    EMBER_LAUNCHED(E);
}


void launch_chain_rule(const Engine& E, const uint32_t* edges, uint32_t nb, const PartView& pi, const PartView& pj) {
    const uint32_t warps = 8;
    if (E.tc_engine() && E.dim <= 128 && !getenv("EMBER_CHAIN_PLAIN")) {
        // persistent pipelined warps: 8 warps per CTA, each with NS shared stages of 7 x 512 B;
        // 2 stages -> 3 CTAs per SM (57 KB each), 3 stages -> 2 CTAs per SM (86 KB each)
        static const int ns = [] {
            const char* v = getenv("EMBER_CHAIN_STAGES");
            return v && atoi(v) == 3 ? 3 : 2;
        }();
        const size_t sm = (size_t)warps * ns * CP_ROLES * 32 * sizeof(float4);
        const uint32_t per_sm = ns == 3 ? 2 : 3;
        const uint32_t blocks = std::min<uint32_t>((nb + warps - 1) / warps, (uint32_t)E.sm_count * per_sm);
        auto kern = ns == 3 ? k_chain_pipe<3, 2> : k_chain_pipe<2, 3>;
        opt_in_smem((const void*)kern, sm, E.device);
        launch_pdl(kern, dim3(blocks), dim3(warps * 32), sm, E.stream, edges, nb, E.n_neg, pi, pj,
                   (const float*)E.rel_theta, E.m.kind, E.dim, (const float*)E.s.dA, (uint32_t)E.b_cap,
                   (const float*)E.s.g0, (const uint32_t*)E.s.rank, (const uint8_t*)E.s.uniq, E.s.grows,
                   E.direct_hi ? 1 : 0, E.m.lr, E.m.eps, (const float*)E.s.lse, (const float*)E.s.fpos,
                   reinterpret_cast<double*>(E.s.loss_part), E.s.loss_done, E.loss_target, E.s.bad_batch,
                   E.batch_tag, E.dn, E.dn_pending ? 1 : 0);
        E.dn_pending = false;
        E.loss_fused = true;
    } else {
        if (E.dn_pending) {
            dn_reduce_run(E, E.dn);
            E.dn_pending = false;
        }
        k_chain_rule<<<(nb + warps - 1) / warps, warps * 32, 0, E.stream>>>(
            edges, nb, E.n_neg, pi, pj, E.rel_theta, E.m.kind, E.dim, E.s.dA, E.tc_engine() ? (uint32_t)E.b_cap : 0u,
            E.s.g0, E.s.rank, E.s.grows, E.s.keys_sorted, E.slots(nb), E.direct_hi ? 1 : 0, E.m.lr, E.m.eps);
    }
    EMBER_LAUNCHED(E);
}

void launch_loss(const Engine& E, uint32_t nb, float* loss_out) {
    if (E.loss_fused) {  // the chain rule already reduced the loss into E.loss_target
        if (loss_out != E.loss_target)
            EMBER_CUDA(cudaMemcpyAsync(loss_out, E.loss_target, sizeof(float), cudaMemcpyDeviceToDevice, E.stream));
        E.loss_fused = false;
        return;
    }
    const uint32_t per = LOSS_THREADS;  // ~100 blocks at b = 5e4: latency, not bandwidth
    const uint32_t blocks = (nb + per - 1) / per;
    launch_pdl(k_loss, dim3(blocks), dim3(LOSS_THREADS), 0, E.stream, (const float*)E.s.lse, (const float*)E.s.fpos, nb,
               per, reinterpret_cast<double*>(E.s.loss_part), E.s.loss_done, loss_out, E.s.bad_batch, E.batch_tag);
    EMBER_LAUNCHED(E);
}

void launch_segments(const Engine& E, uint32_t n_slots, const KeySpace& ks, bool apply, bool rel_dense,
                     uint32_t* node_ids_out, float* node_rows_out, uint32_t* rel_ids_out, float* rel_rows_out,
                     int part, cudaStream_t st) {
    if (!n_slots) return;
    if (!st) st = E.stream;
    SegArgs a{};
    a.part = part;
    a.nsplit = E.s.nsplit;
    a.ukeys = E.s.ukeys;
    a.offsets = E.s.offsets;
    a.nruns = E.s.nruns;
    a.nunique = E.s.nunique;
    a.longs = E.s.longs;
    a.owner = E.s.long_owner;
    a.partial = E.s.long_partial;
    a.rows = E.s.grows;
    a.ks = ks;
    a.rel_theta = E.rel_theta;
    a.rel_acc = E.rel_acc;
    a.rel_dense = rel_dense ? (E.rel_ext ? E.rel_ext : E.s.rel_dense) : nullptr;
    a.vals_sorted = E.s.vals_sorted;
    a.direct_hi = apply ? E.direct_hi : 0u;
    // the plan's run list is valid when it was built for the same direct-apply threshold
    a.act = (!E.seg_walk && a.direct_hi == E.plan_direct) ? E.s.seg_act : nullptr;  // (E.seg_walk: A/B)
    a.d = E.dim;
    a.lr = E.m.lr;
    a.eps = E.m.eps;
    a.apply = apply ? 1 : 0;
    a.node_ids_out = node_ids_out;
    a.node_rows_out = node_rows_out;
    a.rel_ids_out = rel_ids_out;
    a.rel_rows_out = rel_rows_out;
    if (E.dim <= 128 && !getenv("EMBER_SEG_PLAIN")) {  // persistent, pipelined (A/B: EMBER_SEG_PLAIN=1)
        const size_t sm = (size_t)8 * 2 * 2 * 2 * 2 * SEG_LANES * sizeof(float4);
        opt_in_smem((const void*)k_segments_pipe, sm, E.device);
        const uint32_t blocks = std::min<uint32_t>((n_slots + 15) / 16, (uint32_t)E.sm_count * 4);
        a.early_final = pdl_enabled() && !getenv("EMBER_LONG_FINAL_LATE") ? 1 : 0;
        launch_pdl(k_segments_pipe, dim3(blocks), dim3(256), sm, st, a);
    } else {
        k_segments<<<(n_slots * 16 + 255) / 256, 256, 0, st>>>(a);  // 2 keys per warp
    }
    EMBER_LAUNCHED(E);
    const size_t lf_smem = 2 * LONG_WARPS * E.dim * sizeof(float);  // > 48 KB from d = 376 on (C5: d = 800)
    opt_in_smem((const void*)k_long_final, lf_smem, E.device);
    launch_pdl(k_long_final, dim3(E.sm_count), dim3(32 * LONG_WARPS), lf_smem, st,
               a);
    EMBER_LAUNCHED(E);
}

void launch_long_plan(const Engine& E, uint32_t n_slots, uint64_t node_range, uint32_t direct) {
    if (!n_slots) return;
    launch_pdl(k_long_plan, dim3((n_slots + 255) / 256), dim3(256), 0, E.side, (const uint32_t*)E.s.offsets,
               (const uint32_t*)E.s.nruns, n_slots, (const uint32_t*)E.s.ukeys, (const uint32_t*)E.s.vals_sorted,
               node_range, direct, (const uint32_t*)E.s.nsplit, E.s.nunique, E.s.longs, E.s.long_owner,
               E.s.seg_act);
    E.plan_direct = direct;
    EMBER_LAUNCHED(E);
}

void launch_adagrad_rows(const Engine& E, const uint32_t* ids, const float* rows, uint32_t n, const PartView& pi,
                         const PartView& pj, bool relations, uint32_t* bad) {
    if (!n) return;
    k_adagrad_rows<<<(n * 32 + 255) / 256, 256, 0, E.stream>>>(ids, rows, n, E.dim, E.m.kind, pi, pj, relations ? 1 : 0,
                                                                E.rel_theta, E.rel_acc, E.g.num_relations, E.m.lr,
                                                                E.m.eps, bad);
    EMBER_LAUNCHED(E);
}

// ParameterSlice gather (getGpuParameters): warp per id, the theta
// (and acc) row of a node of partition i or j, or of a relation, copied out in id order. Ids
// outside both partitions (outside [0, R) for relations) are counted in *bad, their rows untouched.
__global__ void k_gather_rows(const uint32_t* __restrict__ ids, uint32_t n, uint32_t d, int kind, PartView pi, PartView pj,
                              int relations, const float* rel_theta, const float* rel_acc, uint32_t n_rel,
                              float* th_out, float* ac_out, uint32_t* bad) {
    const uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (u >= n) return;
    const uint32_t key = ids[u];
    const float* th;
    const float* ac;
    if (relations) {
        if (key >= n_rel) {
            if (lane == 0) atomicAdd(bad, 1u);
            return;
        }
        th = rel_theta + (uint64_t)key * d;
        ac = rel_acc + (uint64_t)key * d;
    } else {
        const bool in_i = key - pi.first < pi.rows, in_j = key - pj.first < pj.rows;
        if (!in_i && !in_j) {
            if (lane == 0) atomicAdd(bad, 1u);
            return;
        }
        const PartView& v = in_i ? pi : pj;
        th = v.theta + (uint64_t)(key - v.first) * d;
        ac = v.acc + (uint64_t)(key - v.first) * d;
    }
    for (uint32_t c = lane; c < d; c += 32) {  // out in on-disk coordinate order
        const uint32_t k = hbm_pos(kind, d, c);
        th_out[(uint64_t)u * d + c] = th[k];
        if (ac_out) ac_out[(uint64_t)u * d + c] = ac[k];
    }
}

void launch_gather_rows(const Engine& E, const uint32_t* ids, uint32_t n, const PartView& pi, const PartView& pj,
                        bool relations, float* th_out, float* ac_out, uint32_t* bad) {
    if (!n) return;
    k_gather_rows<<<(n * 32 + 255) / 256, 256, 0, E.stream>>>(ids, n, E.dim, E.m.kind, pi, pj, relations ? 1 : 0, E.rel_theta,
                                                               E.rel_acc, E.g.num_relations, th_out, ac_out, bad);
    EMBER_LAUNCHED(E);
}

void launch_init_rows(cudaStream_t st, float* theta, float* acc, uint64_t first, uint64_t rows, uint32_t dim,
                      int kind, uint64_t seed) {
    if (!rows) return;
    const float a = (float)(1.0 / sqrt((double)dim));
    k_init_rows<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(theta, acc, first, rows, dim, kind, seed, a);
    EMBER_CUDA(cudaGetLastError());
}

void launch_rows_layout(cudaStream_t st, float* rows, uint64_t n, const uint32_t* n_dev, uint32_t dim, int kind,
                        bool to_hbm) {
    if (kind != EMBER_COMPLEX || !rows || (!n && !n_dev)) return;
    const uint32_t warps = 8;
    k_rows_layout<<<(unsigned)((n + warps - 1) / warps), warps * 32, warps * dim * sizeof(float), st>>>(
        rows, n, n_dev, dim, to_hbm ? 1 : 0);
    EMBER_CUDA(cudaGetLastError());
}

void launch_debug_scores(const Engine& E, const uint32_t* edges, uint32_t nb, const uint32_t* negs, int side,
                         uint32_t rows, float* out, const PartView& pi, const PartView& pj) {
    launch_gather_adjust(E, edges, nb, pi, pj, false, negs);
    launch_gather_negatives(E, negs, pi, pj, false);
    const float* A = E.s.A + (uint64_t)side * nb * E.dim;
    const float* N = E.s.N + (uint64_t)side * E.nt * E.dim;
    const uint32_t w = rows * E.nt;
    k_debug_scores<<<(w * 32 + 255) / 256, 256, 0, E.stream>>>(A, N, rows, E.nt, E.dim, out);
    EMBER_LAUNCHED(E);
}

}  // namespace ember
