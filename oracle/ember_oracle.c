/* CPU oracle for the minibatch training step — see ember_oracle.h for scope and parity status.
 * TEST INFRASTRUCTURE ONLY (the checker; never the measured or shipped path).
 *
 * Every function cites the reference line it restates. Arithmetic is fp32 storage with fp32
 * accumulation in a fixed order (built with -ffp-contract=off), OpenMP over independent rows only,
 * so results are bit-reproducible for any thread count.
 */
#include "ember_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ---------------------------------------------------------------- RNG (common.h:51-117) */

/* common.h:51-56 */
uint64_t orc_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* common.h:59 */
uint64_t orc_mix_seed(uint64_t base, uint64_t salt) { return orc_splitmix64(base ^ orc_splitmix64(salt)); }
/* common.h:60 */
uint64_t orc_mix_seed3(uint64_t base, uint64_t a, uint64_t b) { return orc_mix_seed(orc_mix_seed(base, a), b); }

typedef struct {
    uint64_t s;
} orc_rng;

/* Rng::Rng, common.h:67 */
static inline orc_rng rng_make(uint64_t seed) {
    orc_rng r = {orc_splitmix64(seed ^ 0x2545f4914f6cdd1dULL)};
    return r;
}
/* Rng::next, common.h:69-72 */
static inline uint64_t rng_next(orc_rng* r) {
    r->s = orc_splitmix64(r->s);
    return r->s;
}
/* Rng::uniform_below, common.h:75-87 (Lemire multiply-shift with rejection) */
static inline uint64_t rng_below(orc_rng* r, uint64_t n) {
    for (;;) {
        uint64_t x = rng_next(r);
        unsigned __int128 m = (unsigned __int128)x * n;
        uint64_t lo = (uint64_t)m;
        if (lo < n) {
            uint64_t threshold = (0ULL - n) % n;
            if (lo < threshold) continue;
        }
        return (uint64_t)(m >> 64);
    }
}
/* Rng::uniform01 / uniform, common.h:90-92 */
static inline float rng_uniform(orc_rng* r, float lo, float hi) {
    double u = (double)(rng_next(r) >> 11) * (1.0 / 9007199254740992.0);
    return lo + (float)u * (hi - lo);
}

void orc_rng_next(uint64_t seed, uint32_t k, uint64_t* out) {
    orc_rng r = rng_make(seed);
    for (uint32_t i = 0; i < k; ++i) out[i] = rng_next(&r);
}
void orc_rng_uniform_below(uint64_t seed, uint64_t n, uint32_t k, uint64_t* out) {
    orc_rng r = rng_make(seed);
    for (uint32_t i = 0; i < k; ++i) out[i] = rng_below(&r, n);
}
void orc_rng_uniform(uint64_t seed, float lo, float hi, uint32_t k, float* out) {
    orc_rng r = rng_make(seed);
    for (uint32_t i = 0; i < k; ++i) out[i] = rng_uniform(&r, lo, hi);
}

/* ---------------------------------------------------------------- partitions */

uint64_t orc_part_offset(uint64_t V, uint32_t p, uint32_t k) {
    uint64_t q = V / p, rem = V % p;
    return (uint64_t)k * q + (k < rem ? k : rem);
}
uint64_t orc_part_size(uint64_t V, uint32_t p, uint32_t k) {
    uint64_t q = V / p, rem = V % p;
    return q + (k < rem ? 1 : 0);
}

/* ---------------------------------------------------------------- model */

/* Per-edge "adjusted" vectors so that every score is a plain dot product:
 *   destination corruption: f(s, r, x) = adj_dst(s, r) . x
 *   source corruption:      f(x, r, t) = adj_src(r, t) . x
 * Dot:      adj_dst = s,        adj_src = t
 * DistMult: adj_dst = s*r,      adj_src = r*t
 * ComplEx (halves [re | im]): f = Re(<s, r, conj(t)>)
 *           adj_dst = s*r (complex product) as [re | im]
 *           adj_src = [Re(r conj t) | -Im(r conj t)]                                        */
static void adjust_dst(int32_t kind, uint32_t d, const float* s, const float* r, float* out) {
    if (kind == ORC_DOT) {
        memcpy(out, s, d * sizeof(float));
    } else if (kind == ORC_DISTMULT) {
        for (uint32_t k = 0; k < d; ++k) out[k] = s[k] * r[k];
    } else {
        uint32_t h = d / 2;
        for (uint32_t k = 0; k < h; ++k) {
            float a = s[k], b = s[h + k], c = r[k], e = r[h + k];
            out[k] = a * c - b * e;
            out[h + k] = a * e + b * c;
        }
    }
}

static void adjust_src(int32_t kind, uint32_t d, const float* r, const float* t, float* out) {
    if (kind == ORC_DOT) {
        memcpy(out, t, d * sizeof(float));
    } else if (kind == ORC_DISTMULT) {
        for (uint32_t k = 0; k < d; ++k) out[k] = r[k] * t[k];
    } else {
        uint32_t h = d / 2;
        for (uint32_t k = 0; k < h; ++k) {
            float c = r[k], e = r[h + k], x = t[k], y = t[h + k];
            out[k] = c * x + e * y;
            out[h + k] = c * y - e * x;
        }
    }
}

static inline float dotf(const float* a, const float* b, uint32_t d) {
    float acc = 0.f;
    for (uint32_t k = 0; k < d; ++k) acc += a[k] * b[k];
    return acc;
}

/* SPEC.md:139-147 */
float orc_score(int32_t kind, uint32_t dim, const float* s, const float* r, const float* d) {
    float* tmp = (float*)malloc(dim * sizeof(float));
    adjust_dst(kind, dim, s, r, tmp);
    float f = dotf(tmp, d, dim);
    free(tmp);
    return f;
}

/* SPEC.md:175-183. One Rng stream per global row keeps init order-independent and
 * identical between the GPU initializer and this oracle. */
void orc_init_rows(uint64_t seed, uint32_t dim, uint64_t row_begin, uint64_t rows, float* theta) {
    const float a = (float)(1.0 / sqrt((double)dim));
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < (int64_t)rows; ++r) {
        orc_rng g = rng_make(orc_mix_seed(seed, row_begin + (uint64_t)r));
        float* out = theta + (uint64_t)r * dim;
        for (uint32_t k = 0; k < dim; ++k) out[k] = rng_uniform(&g, -a, a);
    }
}

/* SPEC.md:148-156 + design decisions SPEC.md:194-195, 425 (negatives from the resident
 * partitions: destination side from the dst partition, source side from the src partition).
 * Counter-based stream: every slot owns Rng(mix_seed(mix_seed(seed, epoch, bucket_step),
 * batch_in_bucket, (chunk*2 + side)*n_t + slot)), so slots are independent of each other
 * and of evaluation order. */
void orc_sample_negatives(const orc_model* m, uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket,
                          const uint32_t* bucket_edges, uint64_t bucket_n, uint64_t src_off, uint64_t src_size,
                          uint64_t dst_off, uint64_t dst_size, uint32_t* out) {
    const uint32_t nt = m->num_negatives;
    const uint32_t n_deg = (uint32_t)ceil((double)m->alpha * (double)nt);
    const uint64_t base = orc_mix_seed(orc_mix_seed3(m->neg_seed, epoch, bucket_step), batch_in_bucket);
    const uint32_t chunks = m->num_chunks ? m->num_chunks : 1;
    for (uint32_t q = 0; q < chunks; ++q) {
        for (uint32_t side = 0; side < 2; ++side) {
            for (uint32_t k = 0; k < nt; ++k) {
                uint64_t slot = ((uint64_t)q * 2 + side) * nt + k;
                orc_rng g = rng_make(orc_mix_seed(base, slot));
                uint32_t id;
                if (k < n_deg && bucket_n > 0) {
                    uint64_t e = rng_below(&g, bucket_n);
                    id = side == 0 ? bucket_edges[3 * e + 2] : bucket_edges[3 * e + 0];
                } else if (side == 0) {
                    id = (uint32_t)(dst_off + rng_below(&g, dst_size));
                } else {
                    id = (uint32_t)(src_off + rng_below(&g, src_size));
                }
                out[slot] = id;
            }
        }
    }
}

typedef struct {
    uint32_t key;
    uint32_t idx;
} kv;

static int kv_cmp(const void* a, const void* b) {
    const kv* x = (const kv*)a;
    const kv* y = (const kv*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* Sums gradient rows per id in ascending (id, occurrence) order; returns #unique. */
static uint32_t reduce_rows(const uint32_t* keys, uint32_t n, const float* rows, uint32_t d, uint32_t* ids_out,
                            float* rows_out) {
    kv* v = (kv*)malloc((size_t)n * sizeof(kv));
    for (uint32_t i = 0; i < n; ++i) {
        v[i].key = keys[i];
        v[i].idx = i;
    }
    qsort(v, n, sizeof(kv), kv_cmp);
    uint32_t* seg = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
    uint32_t nu = 0;
    for (uint32_t i = 0; i < n; ++i)
        if (i == 0 || v[i].key != v[i - 1].key) seg[nu++] = i;
    seg[nu] = n;
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < (int64_t)nu; ++u) {
        float* out = rows_out ? rows_out + (uint64_t)u * d : NULL;
        if (ids_out) ids_out[u] = v[seg[u]].key;
        if (!out) continue;
        memset(out, 0, d * sizeof(float));
        for (uint32_t i = seg[u]; i < seg[u + 1]; ++i) {
            const float* g = rows + (uint64_t)v[i].idx * d;
            for (uint32_t k = 0; k < d; ++k) out[k] += g[k];
        }
    }
    free(seg);
    free(v);
    return nu;
}

/* SPEC.md:157-165 with the sign fix of SPEC.md:192: per edge and corruption side
 *   loss = -f + log(e^f + sum_k e^{f'_k})  (max-subtracted), total = mean over positives;
 * dL/df = (p0 - 1)/nb, dL/df'_k = p_k/nb; chain rule through the adjusted vectors. */
double orc_loss_and_grad(const orc_model* m, const uint32_t* edges, uint32_t nb, const uint32_t* negs,
                         const float* node_theta, const float* rel_theta, float* fpos_out, float* lse_out,
                         uint32_t* node_ids, float* node_rows, uint32_t* n_node, uint32_t* rel_ids, float* rel_rows,
                         uint32_t* n_rel) {
    const uint32_t d = m->dim, nt = m->num_negatives;
    const uint32_t chunks = m->num_chunks ? m->num_chunks : 1;
    const int32_t kind = m->kind;
    const float inv_b = 1.0f / (float)nb;
    const uint32_t chunk_rows = (nb + chunks - 1) / chunks;
    const uint64_t nneg = (uint64_t)chunks * 2 * nt;

    float* A = (float*)malloc((size_t)2 * nb * d * sizeof(float));   /* [side][edge][d] adjusted */
    float* dA = (float*)calloc((size_t)2 * nb * d, sizeof(float));   /* [side][edge][d] */
    float* P = (float*)malloc((size_t)2 * nb * (nt ? nt : 1) * sizeof(float)); /* [side][edge][k] */
    float* N = (float*)malloc((nneg ? nneg : 1) * d * sizeof(float));  /* negative rows */
    float* dN = (float*)calloc((nneg ? nneg : 1) * d, sizeof(float));
    float* fpos = (float*)malloc((size_t)nb * sizeof(float));
    float* g0 = (float*)malloc((size_t)2 * nb * sizeof(float));
    double* loss_e = (double*)malloc((size_t)nb * sizeof(double));
    int bad = 0;

    for (uint64_t i = 0; i < nneg; ++i) memcpy(N + i * d, node_theta + (uint64_t)negs[i] * d, d * sizeof(float));
    /* N^T per (chunk, side): [j][k], so the scores of one edge against all n_t negatives run as
     * independent sums across k, each accumulated over j in the order dotf uses (same result bits) */
    float* NT = (float*)malloc((nneg ? nneg : 1) * d * sizeof(float));
    for (uint64_t cs = 0; cs < (uint64_t)chunks * 2; ++cs)
        for (uint32_t k = 0; k < nt; ++k)
            for (uint32_t j = 0; j < d; ++j) NT[(cs * d + j) * nt + k] = N[(cs * nt + k) * d + j];

    /* gather + adjust + positive score (Alg.1 formBatch) */
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)nb; ++e) {
        const uint32_t s = edges[3 * e], r = edges[3 * e + 1], t = edges[3 * e + 2];
        const float* ts = node_theta + (uint64_t)s * d;
        const float* tt = node_theta + (uint64_t)t * d;
        const float* tr = kind == ORC_DOT ? NULL : rel_theta + (uint64_t)r * d;
        adjust_dst(kind, d, ts, tr, A + (uint64_t)e * d);
        adjust_src(kind, d, tr, tt, A + ((uint64_t)nb + e) * d);
        fpos[e] = dotf(A + (uint64_t)e * d, tt, d);
    }

    /* scores vs shared negatives, log-sum-exp, dA */
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t e = 0; e < (int64_t)nb; ++e) {
        const uint32_t q = (uint32_t)(e / chunk_rows);
        double le = 0.0;
        for (uint32_t side = 0; side < 2; ++side) {
            const float* a = A + ((uint64_t)side * nb + e) * d;
            const float* Ns = N + ((uint64_t)q * 2 + side) * nt * d;
            const float* NTs = NT + ((uint64_t)q * 2 + side) * nt * d;
            float* p = P + ((uint64_t)side * nb + e) * nt;
            const float f = fpos[e];
            float mx = f;
            for (uint32_t k = 0; k < nt; ++k) p[k] = 0.f;
            for (uint32_t j = 0; j < d; ++j) {  /* p[k] = dotf(a, N_k) for every k */
                const float aj = a[j];
                const float* col = NTs + (uint64_t)j * nt;
                for (uint32_t k = 0; k < nt; ++k) p[k] += aj * col[k];
            }
            for (uint32_t k = 0; k < nt; ++k) {
                if (!(p[k] == p[k]) || isinf(p[k])) bad = 1;
                if (p[k] > mx) mx = p[k];
            }
            float z = expf(f - mx);
            for (uint32_t k = 0; k < nt; ++k) z += expf(p[k] - mx);
            const float lse = mx + logf(z);
            if (lse_out) lse_out[(uint64_t)side * nb + e] = lse;
            le += (double)(lse - f);
            const float p0 = expf(f - lse);
            const float gpos = (p0 - 1.0f) * inv_b;
            g0[(uint64_t)side * nb + e] = gpos;
            float* da = dA + ((uint64_t)side * nb + e) * d;
            /* d f / d adj = the "other" endpoint: t for dst corruption, s for src corruption */
            const float* other = node_theta + (uint64_t)edges[3 * e + (side == 0 ? 2 : 0)] * d;
            for (uint32_t j = 0; j < d; ++j) da[j] = gpos * other[j];
            for (uint32_t k = 0; k < nt; ++k) {
                const float pk = expf(p[k] - lse) * inv_b;
                p[k] = pk;
                const float* nk = Ns + (uint64_t)k * d;
                for (uint32_t j = 0; j < d; ++j) da[j] += pk * nk[j];
            }
        }
        loss_e[e] = le;
    }

    /* dN = P^T A per chunk and side, fixed edge order; blocks of 16 negatives walk the
     * edges once (row-contiguous reads of P and A), every element still summed in edge order */
    const uint64_t nblk = (nt + 15) / 16;
#pragma omp parallel for schedule(dynamic)
    for (int64_t bi = 0; bi < (int64_t)((uint64_t)chunks * 2 * nblk); ++bi) {
        const uint32_t cs = (uint32_t)(bi / nblk);
        const uint32_t q = cs / 2, side = cs % 2;
        const uint32_t k0 = (uint32_t)(bi % nblk) * 16;
        const uint32_t k1 = k0 + 16 < nt ? k0 + 16 : nt;
        const uint32_t e0 = q * chunk_rows;
        const uint32_t e1 = e0 + chunk_rows < nb ? e0 + chunk_rows : nb;
        for (uint32_t e = e0; e < e1; ++e) {
            const float* prow = P + ((uint64_t)side * nb + e) * nt;
            const float* a = A + ((uint64_t)side * nb + e) * d;
            for (uint32_t k = k0; k < k1; ++k) {
                const float pk = prow[k];
                float* out = dN + ((uint64_t)cs * nt + k) * d;
                for (uint32_t j = 0; j < d; ++j) out[j] += pk * a[j];
            }
        }
    }

    /* chain rule back through adjust (per edge: src row, dst row, rel row) */
    float* Gs = (float*)calloc((size_t)nb * d, sizeof(float));
    float* Gt = (float*)calloc((size_t)nb * d, sizeof(float));
    float* Gr = (float*)calloc((size_t)nb * d, sizeof(float));
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)nb; ++e) {
        const uint32_t s = edges[3 * e], r = edges[3 * e + 1], t = edges[3 * e + 2];
        const float* ts = node_theta + (uint64_t)s * d;
        const float* tt = node_theta + (uint64_t)t * d;
        const float* tr = kind == ORC_DOT ? NULL : rel_theta + (uint64_t)r * d;
        const float* ad = A + (uint64_t)e * d;
        const float* as = A + ((uint64_t)nb + e) * d;
        const float* u = dA + (uint64_t)e * d;          /* grad wrt adj_dst */
        const float* w = dA + ((uint64_t)nb + e) * d;   /* grad wrt adj_src */
        const float gd = g0[e], gs = g0[(uint64_t)nb + e];
        float* gS = Gs + (uint64_t)e * d;
        float* gT = Gt + (uint64_t)e * d;
        float* gR = Gr + (uint64_t)e * d;
        /* positive-score terms: f = adj_dst . t  and  f = adj_src . s */
        for (uint32_t j = 0; j < d; ++j) {
            gT[j] = gd * ad[j];
            gS[j] = gs * as[j];
        }
        if (kind == ORC_DOT) {
            for (uint32_t j = 0; j < d; ++j) {
                gS[j] += u[j];
                gT[j] += w[j];
            }
        } else if (kind == ORC_DISTMULT) {
            for (uint32_t j = 0; j < d; ++j) {
                gS[j] += u[j] * tr[j];
                gR[j] = u[j] * ts[j] + w[j] * tt[j];
                gT[j] += w[j] * tr[j];
            }
        } else {
            const uint32_t h = d / 2;
            for (uint32_t j = 0; j < h; ++j) {
                const float a = ts[j], b = ts[h + j], c = tr[j], ee = tr[h + j], x = tt[j], y = tt[h + j];
                const float u0 = u[j], u1 = u[h + j], w0 = w[j], w1 = w[h + j];
                gS[j] += u0 * c + u1 * ee;
                gS[h + j] += u1 * c - u0 * ee;
                gR[j] = (u0 * a + u1 * b) + (w0 * x + w1 * y);
                gR[h + j] = (u1 * a - u0 * b) + (w0 * y - w1 * x);
                gT[j] += w0 * c - w1 * ee;
                gT[h + j] += w0 * ee + w1 * c;
            }
        }
    }

    /* GradientDelta: one summed row per unique id */
    const uint32_t nkeys = 2 * nb + (uint32_t)nneg;
    uint32_t* keys = (uint32_t*)malloc((size_t)nkeys * sizeof(uint32_t));
    float* rows = (float*)malloc((size_t)nkeys * d * sizeof(float));
    for (uint32_t e = 0; e < nb; ++e) {
        keys[e] = edges[3 * e];
        keys[nb + e] = edges[3 * e + 2];
    }
    memcpy(rows, Gs, (size_t)nb * d * sizeof(float));
    memcpy(rows + (size_t)nb * d, Gt, (size_t)nb * d * sizeof(float));
    for (uint64_t i = 0; i < nneg; ++i) keys[2 * nb + i] = negs[i];
    memcpy(rows + (size_t)2 * nb * d, dN, nneg * d * sizeof(float));
    uint32_t nu = reduce_rows(keys, nkeys, rows, d, node_ids, node_rows);
    if (n_node) *n_node = nu;
    if (kind != ORC_DOT) {
        uint32_t* rk = (uint32_t*)malloc((size_t)nb * sizeof(uint32_t));
        for (uint32_t e = 0; e < nb; ++e) rk[e] = edges[3 * e + 1];
        uint32_t nr = reduce_rows(rk, nb, Gr, d, rel_ids, rel_rows);
        if (n_rel) *n_rel = nr;
        free(rk);
    } else if (n_rel) {
        *n_rel = 0;
    }

    double loss = 0.0;
    for (uint32_t e = 0; e < nb; ++e) loss += loss_e[e];
    loss /= (double)nb;
    if (fpos_out) memcpy(fpos_out, fpos, (size_t)nb * sizeof(float));

    free(keys);
    free(rows);
    free(Gs);
    free(Gt);
    free(Gr);
    free(A);
    free(dA);
    free(P);
    free(N);
    free(NT);
    free(dN);
    free(fpos);
    free(g0);
    free(loss_e);
    return bad ? NAN : loss;
}

/* SPEC.md:166-174 */
void orc_adagrad_apply(uint32_t d, float lr, float eps, const uint32_t* ids, const float* rows, uint32_t n,
                       float* theta, float* acc) {
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < (int64_t)n; ++u) {
        float* th = theta + (uint64_t)ids[u] * d;
        float* ac = acc + (uint64_t)ids[u] * d;
        const float* g = rows + (uint64_t)u * d;
        for (uint32_t k = 0; k < d; ++k) {
            const float a = ac[k] + g[k] * g[k];
            ac[k] = a;
            th[k] -= lr * g[k] / (sqrtf(a) + eps);
        }
    }
}

/* Algorithm 1, one batch: getBatchEdges -> sample -> formBatch ->
 * computeGradients -> updateGpuParameters (relations) -> updateCpuParameters (nodes). */
double orc_train_batch(const orc_model* m, uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket,
                       const uint32_t* bucket_edges, uint64_t bucket_n, uint64_t batch_begin, uint32_t nb,
                       uint64_t src_off, uint64_t src_size, uint64_t dst_off, uint64_t dst_size, float* node_theta,
                       float* node_acc, float* rel_theta, float* rel_acc) {
    const uint32_t chunks = m->num_chunks ? m->num_chunks : 1;
    const uint64_t nneg = (uint64_t)chunks * 2 * m->num_negatives;
    uint32_t* negs = (uint32_t*)malloc((nneg ? nneg : 1) * sizeof(uint32_t));
    orc_sample_negatives(m, epoch, bucket_step, batch_in_bucket, bucket_edges, bucket_n, src_off, src_size, dst_off,
                         dst_size, negs);
    const uint32_t cap = 2 * nb + (uint32_t)nneg;
    uint32_t* ids = (uint32_t*)malloc((size_t)cap * sizeof(uint32_t));
    float* rows = (float*)malloc((size_t)cap * m->dim * sizeof(float));
    uint32_t* rids = (uint32_t*)malloc((size_t)nb * sizeof(uint32_t));
    float* rrows = (float*)malloc((size_t)nb * m->dim * sizeof(float));
    uint32_t nu = 0, nr = 0;
    double loss = orc_loss_and_grad(m, bucket_edges + 3 * batch_begin, nb, negs, node_theta, rel_theta, NULL, NULL,
                                    ids, rows, &nu, rids, rrows, &nr);
    if (nr) orc_adagrad_apply(m->dim, m->lr, m->eps, rids, rrows, nr, rel_theta, rel_acc);
    orc_adagrad_apply(m->dim, m->lr, m->eps, ids, rows, nu, node_theta, node_acc);
    free(negs);
    free(ids);
    free(rows);
    free(rids);
    free(rrows);
    return loss;
}

/* ---------------------------------------------------------------- eval */

static int key_in(const uint64_t* keys, uint64_t n, uint64_t k) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (keys[mid] < k)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo < n && keys[lo] == k;
}

static inline uint64_t pack_key(uint64_t s, uint64_t r, uint64_t t) { return (s << 40) | (r << 24) | t; }

void orc_eval_ranks(int32_t kind, uint32_t d, const float* node_theta, const float* rel_theta, uint64_t V,
                    const uint32_t* test, uint32_t n_test, int filtered, const uint64_t* fkeys, uint64_t n_filter,
                    const uint32_t* train, uint64_t n_train, uint32_t n_eval_neg, float alpha_eval, uint32_t block,
                    uint64_t eval_seed, uint32_t* ranks_out) {
    if (block == 0) block = 1;
    uint32_t nblocks = (n_test + block - 1) / block;
    uint32_t* negs = NULL;
    if (!filtered) {
        orc_model em;
        memset(&em, 0, sizeof em);
        em.num_negatives = n_eval_neg;
        em.alpha = alpha_eval;
        em.num_chunks = 1;
        em.neg_seed = eval_seed;
        negs = (uint32_t*)malloc((size_t)nblocks * 2 * (n_eval_neg ? n_eval_neg : 1) * sizeof(uint32_t));
        for (uint32_t q = 0; q < nblocks; ++q)
            orc_sample_negatives(&em, 0, 0, q, train, n_train, 0, V, 0, V, negs + (size_t)q * 2 * n_eval_neg);
    }
#pragma omp parallel
    {
        float* a = (float*)malloc(d * sizeof(float));
#pragma omp for schedule(dynamic, 16)
        for (int64_t e = 0; e < (int64_t)n_test; ++e) {
            const uint32_t s = test[3 * e], r = test[3 * e + 1], t = test[3 * e + 2];
            const float* ts = node_theta + (uint64_t)s * d;
            const float* tt = node_theta + (uint64_t)t * d;
            const float* tr = kind == ORC_DOT ? NULL : rel_theta + (uint64_t)r * d;
            for (uint32_t side = 0; side < 2; ++side) {
                if (side == 0)
                    adjust_dst(kind, d, ts, tr, a);
                else
                    adjust_src(kind, d, tr, tt, a);
                const float pos = dotf(a, side == 0 ? tt : ts, d);
                uint32_t rank = 1;
                if (filtered) {
                    for (uint64_t c = 0; c < V; ++c) {
                        if (c == (side == 0 ? t : s)) continue;
                        uint64_t key = side == 0 ? pack_key(s, r, c) : pack_key(c, r, t);
                        float sc = dotf(a, node_theta + c * d, d);
                        if (sc >= pos && !key_in(fkeys, n_filter, key)) ++rank;
                    }
                } else {
                    const uint32_t* ng = negs + ((size_t)(e / block) * 2 + side) * n_eval_neg;
                    for (uint32_t k = 0; k < n_eval_neg; ++k)
                        if (dotf(a, node_theta + (uint64_t)ng[k] * d, d) >= pos) ++rank;
                }
                ranks_out[(uint64_t)side * n_test + e] = rank;
            }
        }
        free(a);
    }
    free(negs);
}

/* SPEC.md:461-467 */
void orc_aggregate(const uint32_t* ranks, uint64_t n, const uint32_t* ks, uint32_t nk, double* out) {
    double mrr = 0.0;
    for (uint32_t j = 0; j < nk; ++j) out[1 + j] = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        mrr += 1.0 / (double)ranks[i];
        for (uint32_t j = 0; j < nk; ++j) out[1 + j] += ranks[i] <= ks[j] ? 1.0 : 0.0;
    }
    out[0] = n ? mrr / (double)n : 0.0;
    for (uint32_t j = 0; j < nk; ++j) out[1 + j] = n ? out[1 + j] / (double)n : 0.0;
}

/* ---------------------------------------------------------------- preprocessing */

static int u32_cmp(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}

typedef struct {
    uint64_t key;
    uint32_t idx;
} orc_ki;

static int ki_cmp(const void* a, const void* b) {
    const orc_ki* x = (const orc_ki*)a;
    const orc_ki* y = (const orc_ki*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : x->idx > y->idx;
}

static uint32_t sorted_unique(uint32_t* a, uint64_t n) {
    qsort(a, n, sizeof(uint32_t), u32_cmp);
    uint64_t m = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (i == 0 || a[i] != a[i - 1]) a[m++] = a[i];
    return (uint32_t)m;
}

static uint32_t lower_bound32(const uint32_t* a, uint32_t n, uint32_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        uint32_t mid = (lo + hi) / 2;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

/* order[i] = index of the i-th smallest (mix_seed(seed, index), index) */
static void seeded_order(uint64_t seed, uint64_t n, uint32_t* order) {
    orc_ki* v = (orc_ki*)malloc(n * sizeof(orc_ki));
    for (uint64_t i = 0; i < n; ++i) {
        v[i].key = orc_mix_seed(seed, i);
        v[i].idx = (uint32_t)i;
    }
    qsort(v, n, sizeof(orc_ki), ki_cmp);
    for (uint64_t i = 0; i < n; ++i) order[i] = v[i].idx;
    free(v);
}

static uint32_t part_of(uint64_t id, uint64_t V, uint32_t p) {
    const uint64_t q = V / p, r = V % p, big = r * (q + 1);
    return id < big ? (uint32_t)(id / (q + 1)) : (uint32_t)(r + (id - big) / q);
}

void orc_preprocess(const uint32_t* raw, uint64_t n, uint32_t p, uint64_t seed, float train_frac, float valid_frac,
                    uint32_t* train_out, uint64_t* offsets, uint32_t* valid_out, uint32_t* test_out, uint64_t* counts,
                    uint32_t* node_tokens, uint32_t* rel_tokens, uint64_t* num_nodes, uint32_t* num_rel) {
    uint32_t* U = (uint32_t*)malloc(2 * n * sizeof(uint32_t));
    uint32_t* RU = (uint32_t*)malloc(n * sizeof(uint32_t));
    for (uint64_t e = 0; e < n; ++e) {
        U[e] = raw[3 * e];
        U[n + e] = raw[3 * e + 2];
        RU[e] = raw[3 * e + 1];
    }
    const uint32_t V = sorted_unique(U, 2 * n), R = sorted_unique(RU, n);
    uint32_t* vorder = (uint32_t*)malloc((size_t)V * sizeof(uint32_t));
    uint32_t* new_id = (uint32_t*)malloc((size_t)V * sizeof(uint32_t));
    seeded_order(orc_mix_seed(seed, 0x9e47ULL), V, vorder);
    for (uint32_t i = 0; i < V; ++i) new_id[vorder[i]] = i;
    uint32_t* eorder = (uint32_t*)malloc(n * sizeof(uint32_t));
    seeded_order(orc_mix_seed(seed, 0x5917ULL), n, eorder);
    uint32_t* sh = (uint32_t*)malloc(3 * n * sizeof(uint32_t));
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t e = eorder[i];
        sh[3 * i] = new_id[lower_bound32(U, V, raw[3 * e])];
        sh[3 * i + 1] = lower_bound32(RU, R, raw[3 * e + 1]);
        sh[3 * i + 2] = new_id[lower_bound32(U, V, raw[3 * e + 2])];
    }
    const uint64_t n_train = (uint64_t)((double)train_frac * (double)n);
    uint64_t n_valid = (uint64_t)((double)valid_frac * (double)n);
    if (n_valid > n - n_train) n_valid = n - n_train;
    const uint64_t n_test = n - n_train - n_valid;
    /* stable counting sort of the train split by bucket */
    const uint32_t nb = p * p;
    memset(offsets, 0, (nb + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < n_train; ++i) ++offsets[part_of(sh[3 * i], V, p) * p + part_of(sh[3 * i + 2], V, p) + 1];
    for (uint32_t b = 0; b < nb; ++b) offsets[b + 1] += offsets[b];
    uint64_t* at = (uint64_t*)malloc((nb + 1) * sizeof(uint64_t));
    memcpy(at, offsets, (nb + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < n_train; ++i) {
        const uint64_t k = at[part_of(sh[3 * i], V, p) * p + part_of(sh[3 * i + 2], V, p)]++;
        memcpy(train_out + 3 * k, sh + 3 * i, 12);
    }
    if (valid_out) memcpy(valid_out, sh + 3 * n_train, n_valid * 12);
    if (test_out) memcpy(test_out, sh + 3 * (n_train + n_valid), n_test * 12);
    if (node_tokens)
        for (uint32_t i = 0; i < V; ++i) node_tokens[i] = U[vorder[i]];
    if (rel_tokens) memcpy(rel_tokens, RU, (size_t)R * 4);
    counts[0] = n_train;
    counts[1] = n_valid;
    counts[2] = n_test;
    *num_nodes = V;
    *num_rel = R;
    free(U);
    free(RU);
    free(vorder);
    free(new_id);
    free(eorder);
    free(sh);
    free(at);
}

/* ---------------------------------------------------------------- synthetic graphs
 * The benchmark graph generator, restated for the CPU arm so that it never loads the product library.
 * Edge e is a pure function of (seed, e) — the definition ember_graph_generate implements
 * (paper_2101_08358_b200/csrc/graph.cu:1-9): power-law source ranks w(r) ∝ (r+1)^-0.9 by inverse CDF,
 * Zipf(1) relations, with probability 0.9 a power-law destination inside community pi_r(comm(src))
 * (comm = rank mod K, pi_r affine on Z_K), else global; ranks become ids through a keyed 4-round
 * Feistel permutation with cycle walking. */
typedef struct {
    uint64_t V, seed;
    uint32_t R, K, half;
    double train, valid;
} orc_gen;

static double g_u01(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

static uint64_t g_powerlaw(double u, uint64_t n) {
    const double a = pow((double)n + 1.0, 0.1) - 1.0;
    const double x = pow(1.0 + u * a, 10.0);
    const uint64_t r = x < 1.0 ? 0 : (uint64_t)x - 1;
    return r >= n ? n - 1 : r;
}

static uint32_t g_zipf(double u, uint32_t R) {
    const double x = exp(u * log((double)R + 1.0));
    const uint32_t r = x < 1.0 ? 0 : (uint32_t)x - 1;
    return r >= R ? R - 1 : r;
}

static uint64_t g_feistel(uint64_t x, const orc_gen* g) {
    const uint64_t mask = (1ULL << g->half) - 1;
    do {
        uint64_t l = x >> g->half, r = x & mask;
        for (uint32_t round = 0; round < 4; ++round) {
            const uint64_t f = orc_splitmix64(r ^ orc_mix_seed(g->seed, 0xfe15ULL + round)) & mask;
            const uint64_t nl = r;
            r = l ^ f;
            l = nl;
        }
        x = (l << g->half) | r;
    } while (x >= g->V);
    return x;
}

static void g_edge(const orc_gen* g, uint64_t e, uint32_t* out3, uint8_t* split) {
    const uint64_t h = orc_mix_seed(g->seed, e);
    const uint64_t src = g_powerlaw(g_u01(orc_splitmix64(h + 1)), g->V);
    const uint32_t rel = g->R <= 1 ? 0u : g_zipf(g_u01(orc_splitmix64(h + 2)), g->R);
    uint64_t dst;
    if (g_u01(orc_splitmix64(h + 3)) < 0.9) {
        const uint64_t c = src & (g->K - 1);
        uint64_t c2 = c;
        if (g->R > 1) {
            const uint64_t hr = orc_mix_seed(g->seed ^ 0x7e1aULL, rel);
            const uint64_t a = 2 * (hr % (g->K / 2 > 0 ? g->K / 2 : 1)) + 1;
            c2 = (a * c + (orc_splitmix64(hr) & (g->K - 1))) & (g->K - 1);
        }
        const uint64_t members = (g->V - c2 + g->K - 1) / g->K;
        dst = c2 + g->K * g_powerlaw(g_u01(orc_splitmix64(h + 4)), members);
    } else {
        dst = g_powerlaw(g_u01(orc_splitmix64(h + 4)), g->V);
    }
    out3[0] = (uint32_t)g_feistel(src, g);
    out3[1] = rel;
    out3[2] = (uint32_t)g_feistel(dst, g);
    if (split) {
        const double us = g_u01(orc_splitmix64(h + 5));
        *split = us < g->train ? 0 : (us < g->train + g->valid ? 1 : 2);
    }
}

void orc_graph_generate(uint64_t V, uint32_t R, uint64_t first, uint64_t n, uint64_t seed, float train_frac,
                        float valid_frac, uint32_t* edges, uint8_t* split) {
    orc_gen g;
    g.V = V;
    g.R = R;
    g.K = 1;
    while (g.K < 1024 && (uint64_t)g.K * 8 <= V) g.K <<= 1;
    g.seed = seed;
    uint32_t bits = 1;
    while ((1ULL << bits) < V) ++bits;
    g.half = (bits + 1) / 2;
    g.train = train_frac; /* float -> double, as the device generator widens them */
    g.valid = valid_frac;
#pragma omp parallel for schedule(static, 65536)
    for (int64_t e = 0; e < (int64_t)n; ++e) g_edge(&g, first + (uint64_t)e, edges + 3 * e, split ? split + e : NULL);
}

/* bucket_edges of the edges whose split byte is `which` (split NULL: all edges):
 * stable counting sort by (part(src), part(dst)); out: the selected edges bucketed, offsets[p*p+1]. */
uint64_t orc_graph_bucket(uint64_t V, uint32_t p, const uint32_t* edges, const uint8_t* split, uint8_t which,
                          uint64_t n, uint32_t* out, uint64_t* offsets) {
    const uint32_t nb = p * p;
    memset(offsets, 0, ((size_t)nb + 1) * sizeof(uint64_t));
    for (uint64_t e = 0; e < n; ++e)
        if (!split || split[e] == which) ++offsets[part_of(edges[3 * e], V, p) * p + part_of(edges[3 * e + 2], V, p) + 1];
    for (uint32_t b = 0; b < nb; ++b) offsets[b + 1] += offsets[b];
    uint64_t* at = (uint64_t*)malloc(((size_t)nb + 1) * sizeof(uint64_t));
    memcpy(at, offsets, ((size_t)nb + 1) * sizeof(uint64_t));
    for (uint64_t e = 0; e < n; ++e) {
        if (split && split[e] != which) continue;
        const uint64_t k = at[part_of(edges[3 * e], V, p) * p + part_of(edges[3 * e + 2], V, p)]++;
        memcpy(out + 3 * k, edges + 3 * e, 12);
    }
    free(at);
    return offsets[nb];
}

/* ---------------------------------------------------------------- the CPU trainer's step on partitions
 * Marius's CPU path for one batch of bucket (i, j) with partitions i and j resident in host memory
 * (Algorithm 1; getCpuParameters / updateCpuParameters):
 * sample_negatives -> unique node ids of the batch (dedupe) -> gather their rows into a compact
 * parameter slice -> loss_and_grad -> Adagrad of the relations and of the touched node rows in place. */
static int u32_cmp_q(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}

double orc_train_batch_parts(const orc_model* m, uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket,
                             const uint32_t* bucket_edges, uint64_t bucket_n, uint64_t batch_begin, uint32_t nb,
                             uint64_t first_i, uint64_t rows_i, float* theta_i, float* acc_i, uint64_t first_j,
                             uint64_t rows_j, float* theta_j, float* acc_j, float* rel_theta, float* rel_acc,
                             uint32_t* n_unique_out) {
    const uint32_t d = m->dim;
    const uint32_t chunks = m->num_chunks ? m->num_chunks : 1;
    const uint64_t nneg = (uint64_t)chunks * 2 * m->num_negatives;
    const uint32_t* batch = bucket_edges + 3 * batch_begin;
    uint32_t* negs = (uint32_t*)malloc((nneg ? nneg : 1) * sizeof(uint32_t));
    /* negatives: destination side from partition j, source side from partition i */
    orc_sample_negatives(m, epoch, bucket_step, batch_in_bucket, bucket_edges, bucket_n, first_i, rows_i, first_j,
                         rows_j, negs);
    const uint64_t cap = 2 * (uint64_t)nb + nneg;
    uint32_t* uniq = (uint32_t*)malloc(cap * sizeof(uint32_t));
    for (uint32_t e = 0; e < nb; ++e) {
        uniq[e] = batch[3 * e];
        uniq[nb + e] = batch[3 * e + 2];
    }
    memcpy(uniq + 2 * (uint64_t)nb, negs, nneg * sizeof(uint32_t));
    qsort(uniq, cap, sizeof(uint32_t), u32_cmp_q);
    uint32_t nu = 0;
    for (uint64_t k = 0; k < cap; ++k)
        if (k == 0 || uniq[k] != uniq[k - 1]) uniq[nu++] = uniq[k];
    /* compact ids and the gathered parameter slice */
    uint32_t* cb = (uint32_t*)malloc((size_t)nb * 3 * sizeof(uint32_t));
    uint32_t* cn = (uint32_t*)malloc((nneg ? nneg : 1) * sizeof(uint32_t));
    float* slice = (float*)malloc((size_t)nu * d * sizeof(float));
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)nb; ++e) {
        cb[3 * e] = lower_bound32(uniq, nu, batch[3 * e]);
        cb[3 * e + 1] = batch[3 * e + 1];
        cb[3 * e + 2] = lower_bound32(uniq, nu, batch[3 * e + 2]);
    }
    for (uint64_t k = 0; k < nneg; ++k) cn[k] = lower_bound32(uniq, nu, negs[k]);
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < (int64_t)nu; ++u) {
        const uint64_t id = uniq[u];
        const float* src = id - first_i < rows_i ? theta_i + (id - first_i) * d : theta_j + (id - first_j) * d;
        memcpy(slice + (uint64_t)u * d, src, d * sizeof(float));
    }
    uint32_t* ids = (uint32_t*)malloc(cap * sizeof(uint32_t));
    float* rows = (float*)malloc(cap * d * sizeof(float));
    uint32_t* rids = (uint32_t*)malloc((size_t)(nb ? nb : 1) * sizeof(uint32_t));
    float* rrows = (float*)malloc((size_t)(nb ? nb : 1) * d * sizeof(float));
    uint32_t ng = 0, nr = 0;
    const double loss =
        orc_loss_and_grad(m, cb, nb, cn, slice, rel_theta, NULL, NULL, ids, rows, &ng, rids, rrows, &nr);
    if (nr) orc_adagrad_apply(d, m->lr, m->eps, rids, rrows, nr, rel_theta, rel_acc);
    /* node Adagrad straight into the partition tables (compact id -> global id -> partition row) */
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < (int64_t)ng; ++u) {
        const uint64_t id = uniq[ids[u]];
        const int in_i = id - first_i < rows_i;
        float* th = in_i ? theta_i + (id - first_i) * d : theta_j + (id - first_j) * d;
        float* ac = in_i ? acc_i + (id - first_i) * d : acc_j + (id - first_j) * d;
        const float* g = rows + (uint64_t)u * d;
        for (uint32_t k = 0; k < d; ++k) {
            const float a = ac[k] + g[k] * g[k];
            ac[k] = a;
            th[k] -= m->lr * g[k] / (sqrtf(a) + m->eps);
        }
    }
    if (n_unique_out) *n_unique_out = nu;
    free(negs);
    free(uniq);
    free(cb);
    free(cn);
    free(slice);
    free(ids);
    free(rows);
    free(rids);
    free(rrows);
    return loss;
}
