// C entry points over the REFERENCE's own ordering code, for ctypes.
//
// TEST INFRASTRUCTURE ONLY (checker, never shipped or measured). Compiled by
// oracle/Makefile together with /root/reference/proj/src/ordering.cpp and the
// reference headers /root/reference/proj/include/ember/{common,ordering}.h, in
// place (no reference source is copied into this repo). Output goes to
// oracle/_ref/libember_ref.so. Each wrapper names the reference symbol it calls.
#include <cstdint>
#include <cstring>
#include <exception>

#include "ember/common.h"    // reference: proj/include/ember/common.h
#include "ember/ordering.h"  // reference: proj/include/ember/ordering.h

using namespace ember;

extern "C" {

// 0 ok, 1 ConfigError, 2 other EmberError / exception.
static int status_of(const std::exception_ptr& ep) {
    try {
        std::rethrow_exception(ep);
    } catch (const ConfigError&) {
        return 1;
    } catch (...) {
        return 2;
    }
}

// make_plan (ordering.cpp:384). seq_out: 2*p*p u32 (i,j pairs); adm_out: up to
// c + 2*p*p u32; swaps_out: 3 u32 per swap (step, evicted, admitted), up to 2*p*p.
int ref_make_plan(int kind, uint32_t p, uint32_t c, uint64_t seed, uint32_t* seq_out, uint64_t* swap_count,
                  uint32_t* adm_out, uint32_t* n_adm, uint32_t* swaps_out, uint32_t* bucket_state_out) {
    try {
        OrderingPlan plan = make_plan(static_cast<OrderingKind>(kind), p, c, seed);
        plan.validate();
        for (size_t t = 0; t < plan.bucket_sequence.size(); ++t) {
            seq_out[2 * t] = plan.bucket_sequence[t].i;
            seq_out[2 * t + 1] = plan.bucket_sequence[t].j;
            if (bucket_state_out) bucket_state_out[t] = plan.bucket_state[t];
        }
        *swap_count = plan.swap_count;
        *n_adm = static_cast<uint32_t>(plan.admission_schedule.size());
        for (size_t k = 0; k < plan.admission_schedule.size(); ++k) adm_out[k] = plan.admission_schedule[k];
        for (size_t k = 0; k < plan.swap_events.size(); ++k) {
            swaps_out[3 * k] = plan.swap_events[k].step;
            swaps_out[3 * k + 1] = plan.swap_events[k].evicted;
            swaps_out[3 * k + 2] = plan.swap_events[k].admitted;
        }
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

// lower_bound_swaps (ordering.cpp:163); returns ~0 on ConfigError.
uint64_t ref_lower_bound_swaps(uint32_t p, uint32_t c) {
    try {
        return lower_bound_swaps(p, c);
    } catch (...) {
        return ~0ULL;
    }
}

// elimination_swap_formula (ordering.cpp:173).
uint64_t ref_elimination_swap_formula(uint32_t p, uint32_t c) {
    try {
        return elimination_swap_formula(p, c);
    } catch (...) {
        return ~0ULL;
    }
}

// simulate_io (ordering.cpp:394).
int ref_simulate_io(int kind, uint32_t p, uint32_t c, uint64_t seed, uint64_t part_bytes, uint64_t* out3) {
    try {
        IOReport r = simulate_io(make_plan(static_cast<OrderingKind>(kind), p, c, seed), part_bytes);
        out3[0] = r.reads;
        out3[1] = r.writes;
        out3[2] = r.total_bytes;
        return 0;
    } catch (...) {
        return status_of(std::current_exception());
    }
}

// hilbert_d2xy (ordering.cpp:300).
void ref_hilbert_d2xy(uint32_t n, uint64_t d, uint32_t* xy) {
    auto r = hilbert_d2xy(n, d);
    xy[0] = r.first;
    xy[1] = r.second;
}

// RNG primitives, common.h:51-117.
uint64_t ref_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t ref_mix_seed(uint64_t base, uint64_t salt) { return mix_seed(base, salt); }
uint64_t ref_mix_seed3(uint64_t base, uint64_t a, uint64_t b) { return mix_seed(base, a, b); }
void ref_rng_next(uint64_t seed, uint32_t k, uint64_t* out) {
    Rng r(seed);
    for (uint32_t i = 0; i < k; ++i) out[i] = r.next();
}
void ref_rng_uniform_below(uint64_t seed, uint64_t n, uint32_t k, uint64_t* out) {
    Rng r(seed);
    for (uint32_t i = 0; i < k; ++i) out[i] = r.uniform_below(n);
}
void ref_rng_uniform(uint64_t seed, float lo, float hi, uint32_t k, float* out) {
    Rng r(seed);
    for (uint32_t i = 0; i < k; ++i) out[i] = r.uniform(lo, hi);
}
void ref_rng_shuffle_iota(uint64_t seed, uint32_t n, uint32_t* out) {
    std::vector<uint32_t> v(n);
    for (uint32_t i = 0; i < n; ++i) v[i] = i;
    Rng r(seed);
    r.shuffle(v);
    std::memcpy(out, v.data(), n * sizeof(uint32_t));
}

}  // extern "C"
