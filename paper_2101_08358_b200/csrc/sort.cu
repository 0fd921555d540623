// SPDX-License-Identifier: Apache-2.0
//
// The step's gradient-slot sort, hand-written for its shape: n ~ 3b + n_neg (152 k at the FB86m
// bench) 32-bit keys of `bits` significant bits (24 at p = 16), stably sorted with their slot
// numbers, then cut into runs (one GradientDelta row per id). Outputs (engine.h):
//   keys_sorted / vals_sorted   (key, slot) ascending; rank[slot] = sorted position
//   ukeys[u], offsets[u]        run u's key and first position; offsets[nruns] = n; nruns
//   uniq[slot]                  the slot's key occurs once
// Kernels (helper stream, PDL-chained), 4096-slot tiles of 1024 threads (32 warps x 4 chunks of 32):
//   k_sort_hist       per-tile digit-0 histograms; zeroes the later passes' histograms
//   k_sort_pass       LSD pass over an 8-bit digit: each tile finds its bins' bases from the per-tile
//                     histograms (no separate scan kernel), ranks its slots stably warp by warp
//                     (match.any peers, per-warp counters) and scatters them; it counts the NEXT
//                     digit per destination tile as it writes (one atomic per distinct (tile, digit)
//                     of a 32-slot chunk: hot keys would serialise per-slot atomics on one address),
//                     and the last pass writes rank[] instead
//   k_sort_runs       run heads, run numbers by a decoupled look-back scan over tiles, ukeys /
//                     offsets / uniq / nruns, and the first run whose key >= split_key (nsplit:
//                     the node / relation boundary of the step's keys; ~0u when there is none)
// Everything here moves ~1.2 MB per pass (L2-resident): the kernels are bound by dependent global
// round trips, so each issues its independent loads together (keys, values and the histogram
// column at once) and keeps the serial per-warp work to 4 chunks.
#include <cuda_runtime.h>

#include "engine.h"

namespace ember {
namespace {

constexpr uint32_t SORT_THREADS = 1024;
constexpr uint32_t SORT_WARPS = SORT_THREADS / 32;
constexpr uint32_t SORT_C = 4;                              // 32-slot chunks per warp
constexpr uint32_t SORT_TILE = SORT_THREADS * SORT_C;       // 4096 slots per tile
constexpr uint32_t SORT_BINS = 256;                         // 8-bit digits
constexpr uint32_t SORT_QUARTERS = SORT_THREADS / SORT_BINS;
constexpr uint32_t SORT_MAX_TILES_PER_Q = 16;               // histogram loads in flight per thread
constexpr uint32_t NO_DIGIT = 0xffffffffu;

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// slot index of (tile, warp, chunk, lane): each warp owns 128 consecutive slots of its tile
__device__ __forceinline__ uint32_t tile_index(uint32_t tile, uint32_t w, uint32_t c, uint32_t lane) {
    return tile * SORT_TILE + w * (SORT_C * 32) + c * 32 + lane;
}

// Exclusive scan of v over the first 256 threads (warps 0-7; every thread of the block calls it).
__device__ __forceinline__ uint32_t scan256(uint32_t v, uint32_t* warp_sums) {
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
    }
    if (lane == 31 && w < 8) warp_sums[w] = x;
    __syncthreads();
    uint32_t before = 0;
#pragma unroll
    for (uint32_t k = 0; k < 8; ++k) before += k < w ? warp_sums[k] : 0u;
    return before + x - v;
}

// Digit-0 histogram of each tile (hist0[tile][bin]); zeroes hist[1..passes) for the scatter passes'
// counts and the run scan's tile counter / status words.
__global__ void __launch_bounds__(SORT_THREADS) k_sort_hist(const uint32_t* __restrict__ keys, uint32_t n,
                                                            uint32_t* __restrict__ hist, uint32_t n_tiles,
                                                            uint32_t passes, unsigned long long* __restrict__ status,
                                                            uint32_t* __restrict__ tile_ctr, uint32_t* __restrict__ nsplit) {
    __shared__ uint32_t h[SORT_BINS];
    griddep_wait();
    const uint32_t t = blockIdx.x, tid = threadIdx.x;
    uint32_t k[SORT_C];
#pragma unroll
    for (uint32_t c = 0; c < SORT_C; ++c) {
        const uint32_t i = t * SORT_TILE + c * SORT_THREADS + tid;
        k[c] = i < n ? keys[i] & (SORT_BINS - 1) : NO_DIGIT;  // (a key may be 0xffffffff: count digits)
    }
    if (tid < SORT_BINS) {
        h[tid] = 0;
        for (uint32_t p = 1; p < passes; ++p) hist[((uint64_t)p * n_tiles + t) * SORT_BINS + tid] = 0;
    }
    if (tid == 0) status[t] = 0ull;
    if (t == 0 && tid == 0) {
        *tile_ctr = 0u;
        *nsplit = ~0u;
    }
    __syncthreads();
#pragma unroll
    for (uint32_t c = 0; c < SORT_C; ++c)
        if (k[c] != NO_DIGIT) atomicAdd(&h[k[c]], 1u);
    __syncthreads();
    if (tid < SORT_BINS) hist[(uint64_t)t * SORT_BINS + tid] = h[tid];
}

// One stable LSD pass on digit (key >> shift) & 255. FIRST: values are the slot numbers (identity);
// LAST: rank[slot] = position, else count digit (key >> shift + 8) of each slot's destination tile.
template <bool FIRST, bool LAST>
__global__ void __launch_bounds__(SORT_THREADS) k_sort_pass(const uint32_t* __restrict__ keys_in,
                                                            const uint32_t* __restrict__ vals_in,
                                                            uint32_t* __restrict__ keys_out,
                                                            uint32_t* __restrict__ vals_out, uint32_t n,
                                                            uint32_t shift, const uint32_t* __restrict__ hist,
                                                            uint32_t n_tiles, uint32_t* __restrict__ hist_next,
                                                            uint32_t* __restrict__ rank) {
    __shared__ uint32_t wbase[SORT_WARPS][SORT_BINS];  // per-warp counts, then per-warp running bases
    __shared__ uint32_t part[2][SORT_QUARTERS][SORT_BINS];
    __shared__ uint32_t warp_sums[8];
    const uint32_t t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    griddep_wait();
    // every independent load first: this tile's keys (and values), then the histogram column
    uint32_t key[SORT_C], val[SORT_C], peers[SORT_C], dig[SORT_C];
#pragma unroll
    for (uint32_t c = 0; c < SORT_C; ++c) {
        const uint32_t i = tile_index(t, w, c, lane);
        key[c] = i < n ? keys_in[i] : 0u;
        val[c] = FIRST ? i : (i < n ? vals_in[i] : 0u);
        dig[c] = i < n ? (key[c] >> shift) & (SORT_BINS - 1) : NO_DIGIT;
    }
    // bin base of this tile: every earlier bin's total + this bin's count in earlier tiles; thread
    // (quarter q, bin b) sums tiles q, q + 4, ... (one round of loads up to 64 tiles)
    {
        const uint32_t b = tid & (SORT_BINS - 1), q = tid / SORT_BINS;
        uint32_t earlier = 0, total = 0;
        for (uint32_t u0 = q; u0 < n_tiles; u0 += SORT_QUARTERS * SORT_MAX_TILES_PER_Q) {
            uint32_t cnt[SORT_MAX_TILES_PER_Q];
#pragma unroll
            for (uint32_t k = 0; k < SORT_MAX_TILES_PER_Q; ++k) {
                const uint32_t u = u0 + k * SORT_QUARTERS;
                cnt[k] = u < n_tiles ? hist[(uint64_t)u * SORT_BINS + b] : 0u;
            }
#pragma unroll
            for (uint32_t k = 0; k < SORT_MAX_TILES_PER_Q; ++k) {
                earlier += u0 + k * SORT_QUARTERS < t ? cnt[k] : 0u;
                total += cnt[k];
            }
        }
        part[0][q][b] = earlier;
        part[1][q][b] = total;
    }
#pragma unroll
    for (uint32_t k = 0; k < SORT_BINS / 32; ++k) wbase[w][k * 32 + lane] = 0;
    __syncthreads();
    uint32_t earlier = 0, total = 0;
    if (tid < SORT_BINS) {
#pragma unroll
        for (uint32_t q = 0; q < SORT_QUARTERS; ++q) {
            earlier += part[0][q][tid];
            total += part[1][q][tid];
        }
    }
    const uint32_t bin_start = scan256(total, warp_sums) + earlier;  // (threads < 256)
#pragma unroll
    for (uint32_t c = 0; c < SORT_C; ++c) {
        peers[c] = __match_any_sync(0xffffffffu, dig[c]);
        if (dig[c] != NO_DIGIT && (peers[c] & lanemask_lt()) == 0) wbase[w][dig[c]] += __popc(peers[c]);
        __syncwarp();
    }
    __syncthreads();
    if (tid < SORT_BINS) {  // warp bases: the tile's bin start + the bin's counts in earlier warps
        uint32_t run = bin_start;
#pragma unroll 8
        for (uint32_t k = 0; k < SORT_WARPS; ++k) {
            const uint32_t x = wbase[k][tid];
            wbase[k][tid] = run;
            run += x;
        }
    }
    __syncthreads();
#pragma unroll
    for (uint32_t c = 0; c < SORT_C; ++c) {
        const uint32_t d = dig[c];
        uint32_t pos = 0;
        if (d != NO_DIGIT) pos = wbase[w][d] + __popc(peers[c] & lanemask_lt());
        __syncwarp();
        if (d != NO_DIGIT) {
            if ((peers[c] & lanemask_lt()) == 0) wbase[w][d] += __popc(peers[c]);
            keys_out[pos] = key[c];
            vals_out[pos] = val[c];
            if (LAST) rank[val[c]] = pos;
        }
        if (!LAST) {  // next digit's count per destination tile, one atomic per distinct (tile, digit) of the chunk
            const uint32_t slot = d != NO_DIGIT ? (pos / SORT_TILE) * SORT_BINS + ((key[c] >> (shift + 8)) & (SORT_BINS - 1))
                                                : NO_DIGIT;
            const uint32_t same = __match_any_sync(0xffffffffu, slot);
            if (slot != NO_DIGIT && (same & lanemask_lt()) == 0) atomicAdd(&hist_next[slot], __popc(same));
        }
        __syncwarp();
    }
}

// Run heads of the sorted keys -> ukeys / offsets / nruns / uniq. Tiles take their ids in launch
// order from tile_ctr and chain their head counts by a decoupled look-back (status word per tile:
// bit 32 = aggregate published, bit 33 = inclusive prefix published, low 32 bits = the count).
__global__ void __launch_bounds__(SORT_THREADS) k_sort_runs(const uint32_t* __restrict__ ks,
                                                            const uint32_t* __restrict__ vs, uint32_t n,
                                                            uint32_t* __restrict__ ukeys, uint32_t* __restrict__ offsets,
                                                            uint32_t* __restrict__ nruns, uint8_t* __restrict__ uniq,
                                                            unsigned long long* status, uint32_t* tile_ctr,
                                                            uint32_t n_tiles, uint32_t split_key,
                                                            uint32_t* __restrict__ nsplit) {
    constexpr unsigned long long AGG = 1ull << 32, INC = 1ull << 33;
    __shared__ uint32_t s_tile, s_prefix;
    __shared__ uint32_t warp_heads[SORT_WARPS];
    const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    griddep_wait();
    if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t t = s_tile;
    uint32_t key[SORT_C], val[SORT_C], edge[SORT_C];
#pragma unroll
    for (uint32_t c = 0; c < SORT_C; ++c) {  // keys, values and each chunk's outer neighbour at once
        const uint32_t i = tile_index(t, w, c, lane);
        key[c] = i < n ? ks[i] : 0u;
        val[c] = i < n ? vs[i] : 0u;
        const uint32_t j = lane == 0 ? i - 1 : i + 1;  // lane 0: the slot before, lane 31: the slot after
        edge[c] = (lane == 0 || lane == 31) && i < n && j < n ? ks[j] : 0u;
    }
    uint32_t head_bits[SORT_C], split_bits[SORT_C];
    uint32_t mine = 0;  // heads of this warp
#pragma unroll
    for (uint32_t c = 0; c < SORT_C; ++c) {
        const uint32_t i = tile_index(t, w, c, lane);
        const uint32_t prev = __shfl_up_sync(0xffffffffu, key[c], 1);
        const uint32_t next = __shfl_down_sync(0xffffffffu, key[c], 1);
        bool head = false, split = false;
        if (i < n) {
            const bool prev_differs = i == 0 || (lane ? prev : edge[c]) != key[c];
            split = key[c] >= split_key && (i == 0 || (lane ? prev : edge[c]) < split_key);
            const bool next_differs = i + 1 >= n || (lane != 31 ? next : edge[c]) != key[c];
            head = prev_differs;
            uniq[val[c]] = prev_differs && next_differs ? 1 : 0;
        }
        head_bits[c] = __ballot_sync(0xffffffffu, head);
        split_bits[c] = __ballot_sync(0xffffffffu, split);
        mine += __popc(head_bits[c]);
    }
    if (lane == 0) warp_heads[w] = mine;
    __syncthreads();
    if (w == 0) {  // warp 0: tile total, publish, then look back over 32 predecessors at a time
        const uint32_t x = warp_heads[lane];
        uint32_t incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += y;
        }
        warp_heads[lane] = incl - x;  // exclusive prefix of warp `lane` within the tile
        const uint32_t tile_total = __shfl_sync(0xffffffffu, incl, 31);
        volatile unsigned long long* st = status;
        if (lane == 0) st[t] = (t == 0 ? INC : AGG) | tile_total;
        uint32_t acc = 0;
        int32_t j = (int32_t)t - 1;
        while (j >= 0) {
            const int32_t q = j - (int32_t)lane;  // lane l reads tile j - l
            const unsigned long long s = q >= 0 ? st[q] : INC;
            if (__ballot_sync(0xffffffffu, (s & (AGG | INC)) != 0) != 0xffffffffu) continue;  // not all published
            const uint32_t inc = __ballot_sync(0xffffffffu, (s & INC) != 0);
            const uint32_t stop = inc ? __ffs(inc) - 1 : 31;  // nearest tile holding an inclusive prefix
            uint32_t v = lane <= stop && q >= 0 ? (uint32_t)s : 0u;
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc += v;
            if (inc) break;
            j -= 32;
        }
        if (lane == 0) {
            if (t) st[t] = INC | (acc + tile_total);
            s_prefix = acc;
            if (t == n_tiles - 1) {
                *nruns = acc + tile_total;
                offsets[acc + tile_total] = n;
            }
        }
    }
    __syncthreads();
    uint32_t u = s_prefix + warp_heads[w];
#pragma unroll
    for (uint32_t c = 0; c < SORT_C; ++c) {
        const uint32_t hb = head_bits[c];
        if (hb >> lane & 1u) {
            const uint32_t r = u + __popc(hb & lanemask_lt());
            ukeys[r] = key[c];
            if (split_bits[c] >> lane & 1u) *nsplit = r;
            offsets[r] = tile_index(t, w, c, lane);
        }
        u += __popc(hb);
    }
}

}  // namespace

uint32_t slot_sort_tiles(uint32_t cap) { return (cap + SORT_TILE - 1) / SORT_TILE; }

size_t slot_sort_scratch_words(uint32_t cap) {
    return (size_t)4 * slot_sort_tiles(cap) * SORT_BINS;  // up to 4 passes of per-tile histograms
}

void launch_slot_sort(const Engine& E, uint32_t n, uint32_t bits, uint32_t split_key) {
    const Scratch& s = E.s;
    cudaStream_t st = E.side;
    if (n == 0) {
        EMBER_CUDA(cudaMemsetAsync(s.nsplit, 0xff, sizeof(uint32_t), st));
        EMBER_CUDA(cudaMemsetAsync(s.nruns, 0, sizeof(uint32_t), st));
        EMBER_CUDA(cudaMemsetAsync(s.offsets, 0, sizeof(uint32_t), st));
        return;
    }
    const uint32_t passes = std::max(1u, std::min(4u, (bits + 7) / 8));
    const uint32_t tiles = slot_sort_tiles(n);
    launch_pdl(k_sort_hist, dim3(tiles), dim3(SORT_THREADS), 0, st, (const uint32_t*)s.keys, n, s.sort_hist, tiles,
               passes, s.sort_status, s.sort_ctr, s.nsplit);
    EMBER_LAUNCHED(E);
    // ping-pong: pass p reads src(p) and writes dst(p); the last pass writes keys_sorted / vals_sorted
    const uint32_t* kin = s.keys;
    const uint32_t* vin = nullptr;
    for (uint32_t p = 0; p < passes; ++p) {
        const bool first = p == 0, last = p + 1 == passes;
        uint32_t* kout = last ? s.keys_sorted : s.sort_keys[p & 1];
        uint32_t* vout = last ? s.vals_sorted : s.sort_vals[p & 1];
        const uint32_t* h = s.sort_hist + (size_t)p * tiles * SORT_BINS;
        uint32_t* hn = s.sort_hist + (size_t)(p + 1) * tiles * SORT_BINS;
        auto k = first ? (last ? k_sort_pass<true, true> : k_sort_pass<true, false>)
                       : (last ? k_sort_pass<false, true> : k_sort_pass<false, false>);
        launch_pdl(k, dim3(tiles), dim3(SORT_THREADS), 0, st, kin, vin, kout, vout, n, 8 * p, h, tiles, hn, s.rank);
        EMBER_LAUNCHED(E);
        kin = kout;
        vin = vout;
    }
    launch_pdl(k_sort_runs, dim3(tiles), dim3(SORT_THREADS), 0, st, (const uint32_t*)s.keys_sorted,
               (const uint32_t*)s.vals_sorted, n, s.ukeys, s.offsets, s.nruns, s.uniq, s.sort_status, s.sort_ctr,
               tiles, split_key, s.nsplit);
    EMBER_LAUNCHED(E);
}

}  // namespace ember
