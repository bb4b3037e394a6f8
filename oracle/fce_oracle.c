/*
 * fce_oracle.c — CPU restatement of the reference fused-LCE path (T = float).
 *
 * TEST INFRASTRUCTURE ONLY (see fce_oracle.h).  Citations are relative to the
 * reference tree proj/include/fusedce/.  Build: gcc -std=c11 -O2
 * -ffp-contract=off -fopenmp (Makefile target oracle/liboracle.so).
 */
#include "fce_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_D_TILE 64 /* ExecPolicy::d_tile default, exec.hpp:17-21 */
#define ORC_SKIP (-2) /* detail::kSkipPosition, fused_forward.hpp:39 */

/* ------------------------------------------------------ instance.hpp:15-25 */
uint64_t orc_splitmix64(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

double orc_splitmix_unit(uint64_t* state) {
    return (double)(orc_splitmix64(state) >> 11) * 0x1.0p-53;
}

/* ---------------------------------------------------------- bf16.hpp:14-36 */
float orc_round_bf16(float x) {
    if (isnan(x)) return x;
    uint32_t bits;
    memcpy(&bits, &x, 4);
    const uint32_t lsb = (bits >> 16) & 1u;
    bits += 0x7FFFu + lsb; /* round half to even */
    bits &= 0xFFFF0000u;
    float y;
    memcpy(&y, &bits, 4);
    return y;
}

int orc_is_bf16_value(float x) { return isnan(x) || orc_round_bf16(x) == x; }

/* ------------------------------------------------------ instance.hpp:38-85 */
int orc_make_instance(size_t n, size_t d, size_t v, uint64_t seed, int64_t ignore_index,
                      double ignore_fraction, int round, float* hidden, float* weight,
                      int64_t* targets) {
    if (n == 0 || d == 0 || v == 0) return ORC_EMPTY_INPUT;
    const double scale = 1.0 / sqrt((double)d);
    uint64_t hs = seed;
    if (hidden)
        for (size_t i = 0; i < n * d; ++i) {
            float x = (float)((2.0 * orc_splitmix_unit(&hs) - 1.0) * scale);
            hidden[i] = round ? orc_round_bf16(x) : x;
        }
    uint64_t ws = seed ^ 0xA5A5A5A5A5A5A5A5ull;
    if (weight)
        for (size_t i = 0; i < v * d; ++i) {
            float x = (float)((2.0 * orc_splitmix_unit(&ws) - 1.0) * scale);
            weight[i] = round ? orc_round_bf16(x) : x;
        }
    if (targets) {
        uint64_t ts = seed ^ 0x5A5A5A5A5A5A5A5Aull;
        for (size_t i = 0; i < n; ++i) targets[i] = (int64_t)(orc_splitmix64(&ts) % (uint64_t)v);
        if (ignore_fraction > 0.0) {
            uint64_t is = seed ^ 0x3C3C3C3C3C3C3C3Cull;
            for (size_t i = 0; i < n; ++i)
                if (orc_splitmix_unit(&is) < ignore_fraction) targets[i] = ignore_index;
        }
    }
    return ORC_OK;
}

/* --------------------------------------------------- detail/kernels.hpp:11-61 */
static float dot_block(const float* a, const float* b, size_t n) {
    enum { L = 8 };
    float acc0[L] = {0}, acc1[L] = {0};
    size_t i = 0;
    for (; i + 2 * L <= n; i += 2 * L) {
        for (size_t k = 0; k < L; ++k) acc0[k] += a[i + k] * b[i + k];
        for (size_t k = 0; k < L; ++k) acc1[k] += a[i + L + k] * b[i + L + k];
    }
    for (; i + L <= n; i += L)
        for (size_t k = 0; k < L; ++k) acc0[k] += a[i + k] * b[i + k];
    float tail = 0.f;
    for (; i < n; ++i) tail += a[i] * b[i];
    for (size_t k = 0; k < L; ++k) acc0[k] += acc1[k];
    float sum = 0.f;
    for (size_t k = 0; k < L; ++k) sum += acc0[k];
    return sum + tail;
}

float orc_dot(const float* a, const float* b, size_t n, size_t d_tile) {
    if (n <= d_tile) return dot_block(a, b, n);
    float total = 0.f;
    size_t base = 0;
    for (; base + d_tile <= n; base += d_tile) total += dot_block(a + base, b + base, d_tile);
    if (base < n) total += dot_block(a + base, b + base, n - base);
    return total;
}

/* ---------------------------------------------------- softmax_stats.hpp:14-75 */
static orc_stats stats_identity(void) {
    orc_stats s;
    s.m = -INFINITY;
    s.a = 0.f;
    s.z_target = 0.f;
    s.found = 0;
    return s;
}

void orc_stats_update(orc_stats* s, float z) {
    if (z > s->m) {
        s->a = s->a * expf(s->m - z) + 1.f;
        s->m = z;
    } else {
        s->a += expf(z - s->m);
    }
}

float orc_stats_logsumexp(const orc_stats* s) { return s->m + logf(s->a); }

float orc_stats_loss(const orc_stats* s) { return (s->m - s->z_target) + logf(s->a); }

int orc_merge_stats(const orc_stats* s1, const orc_stats* s2, orc_stats* out) {
    if (s1->found && s2->found) return ORC_DUPLICATE_TARGET;
    orc_stats o = stats_identity();
    o.m = s1->m > s2->m ? s1->m : s2->m;
    float a = 0.f;
    if (s1->a != 0.f) a += s1->a * expf(s1->m - o.m);
    if (s2->a != 0.f) a += s2->a * expf(s2->m - o.m);
    o.a = a;
    if (s1->found) {
        o.z_target = s1->z_target;
        o.found = 1;
    } else if (s2->found) {
        o.z_target = s2->z_target;
        o.found = 1;
    }
    *out = o;
    return ORC_OK;
}

/* ------------------------------------------------------------ exec.hpp:25-41 */
int orc_partition_ranges(size_t total, size_t parts, size_t* out_lo, size_t* out_hi) {
    if (parts == 0) return ORC_INVALID_LAYOUT;
    const size_t base = total / parts, extra = total % parts;
    size_t lo = 0;
    for (size_t p = 0; p < parts; ++p) {
        const size_t len = base + (p < extra ? 1 : 0);
        out_lo[p] = lo;
        out_hi[p] = lo + len;
        lo += len;
    }
    return ORC_OK;
}

/* ----------------------------------------------------- dense_matrix.hpp:182-211 */
static int validate(size_t n, size_t d, size_t v, const int64_t* targets, int has_ignore,
                    int64_t ignore_index, size_t v_total) {
    if (n == 0 || d == 0 || v == 0) return ORC_EMPTY_INPUT;
    for (size_t i = 0; i < n; ++i) {
        if (has_ignore && targets[i] == ignore_index) continue;
        if (targets[i] < 0 || (size_t)targets[i] >= v_total) return ORC_TARGET_OUT_OF_RANGE;
    }
    return ORC_OK;
}

static size_t count_valid(const int64_t* targets, size_t n, int has_ignore, int64_t ignore_index) {
    if (!has_ignore) return n;
    size_t c = 0;
    for (size_t i = 0; i < n; ++i) c += targets[i] != ignore_index;
    return c;
}

/* ------------------------------------------------------ reduction.hpp:37-54 */
float orc_reduce_losses(const float* rows, size_t n, int reduction, size_t valid_count) {
    float sum = 0.f;
    for (size_t i = 0; i < n; ++i) sum += rows[i];
    if (reduction == ORC_MEAN) sum = valid_count > 0 ? sum / (float)valid_count : 0.f;
    return sum;
}

/* ---------------------------------------------------- fused_forward.hpp:47-131
 * accumulate_stats_block streams, per row, v ascending over [lo, hi): the
 * vocab_tile blocking only reorders rows, never the per-row update order, so
 * it is dropped here.  forward_core merges window partials in ascending
 * window order (112-123); window == V degenerates to one merge with the
 * identity, which is exact. */
static int forward_impl(const float* hidden, const float* weight, size_t n, size_t d, size_t v,
                        size_t v_offset, const int64_t* targets, int has_ignore,
                        int64_t ignore_index, int reduction, size_t window, int threads,
                        orc_stats* stats, float* loss_rows, float* loss_reduced, int partial);

int orc_fused_forward(const float* hidden, const float* weight, size_t n, size_t d, size_t v,
                      size_t v_offset, const int64_t* targets, int has_ignore, int64_t ignore_index,
                      int reduction, size_t window, int threads, orc_stats* stats,
                      float* loss_rows, float* loss_reduced) {
    return forward_impl(hidden, weight, n, d, v, v_offset, targets, has_ignore, ignore_index,
                        reduction, window, threads, stats, loss_rows, loss_reduced, 0);
}

int orc_rank_partial(const float* hidden, const float* weight_shard, size_t n, size_t d,
                     size_t v_rows, size_t v_offset, const int64_t* targets, int has_ignore,
                     int64_t ignore_index, int threads, orc_stats* stats) {
    return forward_impl(hidden, weight_shard, n, d, v_rows, v_offset, targets, has_ignore,
                        ignore_index, ORC_NONE, 0, threads, stats, NULL, NULL, 1);
}

static int forward_impl(const float* hidden, const float* weight, size_t n, size_t d, size_t v,
                        size_t v_offset, const int64_t* targets, int has_ignore,
                        int64_t ignore_index, int reduction, size_t window, int threads,
                        orc_stats* stats, float* loss_rows, float* loss_reduced, int partial) {
    /* fused_forward validates against V; a TP rank partial
     * (parallel_sim.hpp:165-181) leaves the global check to tp_forward. */
    if (!partial && v_offset == 0) {
        int st = validate(n, d, v, targets, has_ignore, ignore_index, v);
        if (st) return st;
    } else if (n == 0 || d == 0 || v == 0) {
        return ORC_EMPTY_INPUT;
    }
    const size_t win = window == 0 ? v : (window < v ? window : v);
    (void)threads;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
    for (long long ii = 0; ii < (long long)n; ++ii) {
        const size_t i = (size_t)ii;
        orc_stats merged = stats_identity();
        float loss = 0.f;
        const int skip = has_ignore && targets[i] == ignore_index;
        if (!skip) {
            const int64_t want = targets[i] - (int64_t)v_offset;
            const float* h = hidden + i * d;
            for (size_t lo = 0; lo < v; lo += win) {
                const size_t hi = lo + win < v ? lo + win : v;
                orc_stats s = stats_identity();
                for (size_t c = lo; c < hi; ++c) {
                    const float z = orc_dot(h, weight + c * d, d, ORC_D_TILE);
                    orc_stats_update(&s, z);
                    if ((int64_t)c == want) {
                        s.z_target = z;
                        s.found = 1;
                    }
                }
                orc_stats out;
                orc_merge_stats(&merged, &s, &out); /* disjoint windows: no duplicate */
                merged = out;
            }
            loss = orc_stats_loss(&merged);
        }
        if (stats) stats[i] = merged;
        if (loss_rows) loss_rows[i] = loss;
    }
    if (loss_reduced && reduction != ORC_NONE) {
        float* tmp = loss_rows;
        if (!tmp) return ORC_INVALID_LAYOUT;
        *loss_reduced = orc_reduce_losses(tmp, n, reduction,
                                          count_valid(targets, n, has_ignore, ignore_index));
    }
    return ORC_OK;
}

/* --------------------------------------------------- fused_backward.hpp:26-140 */
static float gamma_of(size_t i, const int64_t* targets, int has_ignore, int64_t ignore_index,
                      int reduction, float up, const float* up_rows, size_t valid) {
    /* effective_upstream, reduction.hpp:101-126 */
    if (has_ignore && targets[i] == ignore_index) return 0.f;
    if (reduction == ORC_NONE) return up_rows[i];
    if (reduction == ORC_MEAN) return valid > 0 ? up / (float)valid : 0.f;
    return up;
}

int orc_fused_backward(const float* hidden, const float* weight, size_t n, size_t d, size_t v,
                       size_t v_offset, size_t v_total, const int64_t* targets, int has_ignore,
                       int64_t ignore_index, const orc_stats* stats, int reduction,
                       float upstream_scalar, const float* upstream_rows, int threads,
                       float* dhidden, float* dweight) {
    /* validate_problem against the global vocabulary (tp_backward validates
     * shards against the merged stats, parallel_sim.hpp:246-260) */
    int st = validate(n, d, v, targets, has_ignore, ignore_index, v_total ? v_total : v);
    if (st) return st;
    /* require_stats, fused_backward.hpp:58-73 */
    for (size_t i = 0; i < n; ++i) {
        if (has_ignore && targets[i] == ignore_index) continue;
        if (!stats[i].found || !(stats[i].a > 0.f)) return ORC_MISSING_STATS;
    }
    /* check_upstream, reduction.hpp:81-97 */
    if (reduction == ORC_NONE && !upstream_rows) return ORC_INCONSISTENT_UPSTREAM;
    if (reduction != ORC_NONE && upstream_rows) return ORC_INCONSISTENT_UPSTREAM;
    const size_t valid = count_valid(targets, n, has_ignore, ignore_index);

    /* dH rows: ascending v per row */
    if (dhidden) {
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
        for (long long ii = 0; ii < (long long)n; ++ii) {
            const size_t i = (size_t)ii;
            float* dh = dhidden + i * d;
            memset(dh, 0, sizeof(float) * d);
            if (has_ignore && targets[i] == ignore_index) continue;
            const float* h = hidden + i * d;
            const float m = stats[i].m, a = stats[i].a;
            const float scale =
                gamma_of(i, targets, has_ignore, ignore_index, reduction, upstream_scalar, upstream_rows, valid);
            const int64_t want = targets[i] - (int64_t)v_offset;
            for (size_t c = 0; c < v; ++c) {
                const float z = orc_dot(h, weight + c * d, d, ORC_D_TILE);
                const float p = expf(z - m) / a;
                const float g = scale * (p - ((int64_t)c == want ? 1.f : 0.f));
                const float* w = weight + c * d;
                for (size_t k = 0; k < d; ++k) dh[k] += g * w[k];
            }
        }
    }
    /* dW rows: ascending n per vocab row */
    if (dweight) {
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
        for (long long cc = 0; cc < (long long)v; ++cc) {
            const size_t c = (size_t)cc;
            float* dw = dweight + c * d;
            memset(dw, 0, sizeof(float) * d);
            const float* w = weight + c * d;
            for (size_t i = 0; i < n; ++i) {
                if (has_ignore && targets[i] == ignore_index) continue;
                const float* h = hidden + i * d;
                const float m = stats[i].m, a = stats[i].a;
                const float scale = gamma_of(i, targets, has_ignore, ignore_index, reduction,
                                             upstream_scalar, upstream_rows, valid);
                const int64_t want = targets[i] - (int64_t)v_offset;
                const float z = orc_dot(h, w, d, ORC_D_TILE);
                const float p = expf(z - m) / a;
                const float g = scale * (p - ((int64_t)c == want ? 1.f : 0.f));
                for (size_t k = 0; k < d; ++k) dw[k] += g * h[k];
            }
        }
    }
    return ORC_OK;
}
