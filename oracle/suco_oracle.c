/* TEST INFRASTRUCTURE ONLY — CPU oracle restating the SuCo reference path.
 * See suco_oracle.h for the contract. Compiled with -ffp-contract=off so that
 * every fp64 product and sum rounds separately, as in the reference's x86-64
 * build (which emits no FMA). Parity pinned in tests/test_oracle.py. */
#define _GNU_SOURCE
#include "suco_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

enum { SO_OK = 0, SO_INTERNAL = 1, SO_CONFIG = 2, SO_FORMAT = 3, SO_INCOMPAT = 4, SO_CONTRACT = 5 };

static _Thread_local char g_err[512];

const char* so_last_error(void) { return g_err; }

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

/* ------------------------------------------------------------------ rng */

/* rng.hpp:14-19 */
uint64_t so_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* rng.hpp:22-24 */
uint64_t so_derive_seed(uint64_t seed, uint64_t stream) {
    return so_splitmix64(seed ^ so_splitmix64(stream));
}

/* std::mt19937_64 (the reference's engine, rng.hpp:4/:27): the published
 * MT19937-64 recurrence with its standard tempering constants. */
void so_mt_seed(so_mt* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i) {
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    }
    g->idx = 312;
}

uint64_t so_mt_next(so_mt* g) {
    if (g->idx >= 312) {
        const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* rng.hpp:27-33: rejection below (2^64 - bound) % bound */
uint64_t so_uniform_below(so_mt* g, uint64_t bound) {
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
        const uint64_t r = so_mt_next(g);
        if (r >= threshold) return r % bound;
    }
}

/* rng.hpp:36-38 */
double so_uniform_unit(so_mt* g) { return (double)(so_mt_next(g) >> 11) * 0x1.0p-53; }

/* rng.hpp:41-47 (Box-Muller on the 53-bit uniforms) */
double so_normal_unit(so_mt* g) {
    double u1 = so_uniform_unit(g);
    while (u1 <= 0.0) u1 = so_uniform_unit(g);
    const double u2 = so_uniform_unit(g);
    const double two_pi = 6.283185307179586476925286766559;
    return sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
}

/* core.cpp:42-50 */
uint64_t so_fnv1a(const void* bytes, uint64_t len, uint64_t seed) {
    const unsigned char* p = (const unsigned char*)bytes;
    uint64_t h = seed;
    for (uint64_t i = 0; i < len; ++i) {
        h ^= p[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* ------------------------------------------------------------- synthetic */

/* tests/support/synthetic.cpp:12-29 */
int so_clustered(uint64_t n, uint32_t d, uint32_t clusters, uint64_t seed, double lo, double hi,
                 double sigma, int quantize_u8, float* out) {
    so_mt g;
    so_mt_seed(&g, seed);
    double* centers = malloc(sizeof(double) * (size_t)clusters * d);
    if (!centers) return fail(SO_INTERNAL, "out of memory");
    for (size_t i = 0; i < (size_t)clusters * d; ++i) centers[i] = lo + so_uniform_unit(&g) * (hi - lo);
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t c = so_uniform_below(&g, clusters);
        const double* center = centers + c * d;
        for (uint32_t j = 0; j < d; ++j) {
            double v = center[j] + sigma * so_normal_unit(&g);
            if (quantize_u8) {
                v = round(v);
                v = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
            }
            out[i * d + j] = (float)v;
        }
    }
    free(centers);
    return SO_OK;
}

/* tests/support/synthetic.cpp:35-42 (float arithmetic throughout) */
int so_uniform(uint64_t n, uint32_t d, uint64_t seed, float lo, float hi, float* out) {
    so_mt g;
    so_mt_seed(&g, seed);
    const float span = hi - lo;
    for (uint64_t i = 0; i < n * d; ++i) {
        const float u = (float)so_uniform_unit(&g);
        out[i] = lo + u * span;
    }
    return SO_OK;
}

static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

/* io.cpp:212-252: partial Fisher-Yates; both parts in ascending original-id order */
int so_hold_out(const float* data, uint64_t n, uint32_t d, uint64_t count, uint64_t seed,
                float* base_out, float* query_out) {
    if (count >= n) {
        return fail(SO_CONFIG, "cannot hold out %llu of %llu points; at least one base point must remain",
                    (unsigned long long)count, (unsigned long long)n);
    }
    uint32_t* ids = malloc(sizeof(uint32_t) * n);
    if (!ids) return fail(SO_INTERNAL, "out of memory");
    for (uint64_t i = 0; i < n; ++i) ids[i] = (uint32_t)i;
    so_mt g;
    so_mt_seed(&g, seed);
    for (uint64_t i = 0; i < count; ++i) {
        const uint64_t j = i + so_uniform_below(&g, n - i);
        const uint32_t t = ids[i];
        ids[i] = ids[j];
        ids[j] = t;
    }
    qsort(ids, count, sizeof(uint32_t), cmp_u32);
    qsort(ids + count, n - count, sizeof(uint32_t), cmp_u32);
    for (uint64_t i = 0; i < count; ++i) memcpy(query_out + i * d, data + (uint64_t)ids[i] * d, 4 * d);
    for (uint64_t i = count; i < n; ++i) {
        memcpy(base_out + (i - count) * d, data + (uint64_t)ids[i] * d, 4 * d);
    }
    free(ids);
    return SO_OK;
}

/* ------------------------------------------------------- collision params */

/* sc_linear.cpp:18-22 */
static double snapped_product(double ratio, uint64_t n) {
    const double product = ratio * (double)n;
    const double nearest = round(product);
    return fabs(product - nearest) <= 1e-6 ? nearest : product;
}

/* sc_linear.cpp:39-42 */
uint64_t so_collision_count(double alpha, uint64_t n) {
    const uint64_t c = (uint64_t)floor(snapped_product(alpha, n));
    return c < 1 ? 1 : c;
}

/* sc_linear.cpp:44-47 */
uint64_t so_candidate_count(double beta, uint64_t n, uint64_t k) {
    const uint64_t c = (uint64_t)ceil(snapped_product(beta, n));
    return c > k ? c : k;
}

/* sc_linear.cpp:26-37 */
int so_validate_params(double alpha, double beta, uint32_t k, uint64_t n) {
    if (!(alpha > 0.0) || alpha > 1.0) return fail(SO_CONFIG, "alpha must be in (0, 1], got %f", alpha);
    if (!(beta > 0.0) || beta > 1.0) return fail(SO_CONFIG, "beta must be in (0, 1], got %f", beta);
    if (k < 1 || k > n) {
        return fail(SO_CONFIG, "k must be in [1, n]; got k = %u with n = %llu", k, (unsigned long long)n);
    }
    return SO_OK;
}

/* ------------------------------------------------------------- subspaces */

/* subspace.cpp:10-44 */
int so_sample_subspaces(uint32_t d, uint32_t ns, uint32_t mode, uint64_t seed, uint32_t* dims_out,
                        uint32_t* sizes_out, uint32_t* split_out) {
    if (ns < 2) return fail(SO_CONFIG, "sample_subspaces: need at least 2 subspaces, got %u", ns);
    const uint32_t s = d / ns;
    if (s < 2) {
        return fail(SO_CONFIG, "sample_subspaces: floor(d/num_subspaces) = %u leaves a subspace half empty", s);
    }
    for (uint32_t i = 0; i < d; ++i) dims_out[i] = i;
    if (mode == 1) { /* rng.hpp:50-56 Fisher-Yates from the back */
        so_mt g;
        so_mt_seed(&g, seed);
        for (uint64_t i = d; i > 1; --i) {
            const uint64_t j = so_uniform_below(&g, i);
            const uint32_t t = dims_out[i - 1];
            dims_out[i - 1] = dims_out[j];
            dims_out[j] = t;
        }
    }
    for (uint32_t i = 0; i < ns; ++i) {
        const uint32_t begin = s * i;
        const uint32_t end = (i + 1 == ns) ? d : s * (i + 1);
        sizes_out[i] = end - begin;
        split_out[i] = (end - begin) / 2;
    }
    return SO_OK;
}

/* ---------------------------------------------------------------- kernel */

/* core.hpp:66-84: four strided accumulators, tail into acc0, (a0+a1)+(a2+a3) */
double so_sqdist4(const float* a, const float* b, size_t len) {
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0, acc3 = 0.0;
    size_t i = 0;
    for (; i + 4 <= len; i += 4) {
        const double d0 = (double)a[i] - (double)b[i];
        const double d1 = (double)a[i + 1] - (double)b[i + 1];
        const double d2 = (double)a[i + 2] - (double)b[i + 2];
        const double d3 = (double)a[i + 3] - (double)b[i + 3];
        acc0 += d0 * d0;
        acc1 += d1 * d1;
        acc2 += d2 * d2;
        acc3 += d3 * d3;
    }
    for (; i < len; ++i) {
        const double dd = (double)a[i] - (double)b[i];
        acc0 += dd * dd;
    }
    return (acc0 + acc1) + (acc2 + acc3);
}

/* ---------------------------------------------------------------- kmeans */

/* kmeans.cpp:19-33: strict '<' so ties keep the lower cluster id */
static uint32_t nearest(const float* p, const float* cent, uint32_t k, uint32_t dim, double* best_out) {
    uint32_t best = 0;
    double bd = INFINITY;
    for (uint32_t c = 0; c < k; ++c) {
        const double dist = so_sqdist4(p, cent + (size_t)c * dim, dim);
        if (dist < bd) {
            bd = dist;
            best = c;
        }
    }
    *best_out = bd;
    return best;
}

/* kmeans.cpp:38-54: WCSS partials per 4096-point chunk combined in chunk order */
static double assign_all(const float* pts, uint64_t n, uint32_t dim, const float* cent, uint32_t k,
                         uint32_t* assign) {
    double wcss = 0.0;
    for (uint64_t lo = 0; lo < n; lo += 4096) {
        const uint64_t hi = lo + 4096 < n ? lo + 4096 : n;
        double acc = 0.0;
        for (uint64_t i = lo; i < hi; ++i) {
            double dist;
            assign[i] = nearest(pts + i * dim, cent, k, dim, &dist);
            acc += dist;
        }
        wcss += acc;
    }
    return wcss;
}

/* kmeans.cpp:58-114: k-means++ seeding with serial fp64 folds */
static void kmeanspp(const float* pts, uint64_t n, uint32_t dim, uint32_t k, so_mt* g, float* cent,
                     double* min_dist, unsigned char* chosen) {
    for (uint64_t i = 0; i < n; ++i) {
        min_dist[i] = INFINITY;
        chosen[i] = 0;
    }
    uint64_t pick = so_uniform_below(g, n);
    for (uint32_t c = 0;; ++c) {
        /* place(c, pick) kmeans.cpp:64-72 */
        const float* src = pts + pick * dim;
        memcpy(cent + (size_t)c * dim, src, 4 * (size_t)dim);
        chosen[pick] = 1;
        for (uint64_t i = 0; i < n; ++i) {
            const double dist = so_sqdist4(pts + i * dim, src, dim);
            if (dist < min_dist[i]) min_dist[i] = dist;
        }
        if (c + 1 == k) break;
        double total = 0.0;
        for (uint64_t i = 0; i < n; ++i) total += min_dist[i];
        pick = n;
        if (total > 0.0) {
            const double target = so_uniform_unit(g) * total;
            double cum = 0.0;
            for (uint64_t i = 0; i < n; ++i) {
                cum += min_dist[i];
                if (cum > target) {
                    pick = i;
                    break;
                }
            }
            if (pick == n) {
                for (uint64_t i = n; i-- > 0;) {
                    if (min_dist[i] > 0.0) {
                        pick = i;
                        break;
                    }
                }
            }
        }
        if (pick == n) {
            for (uint64_t i = 0; i < n; ++i) {
                if (!chosen[i]) {
                    pick = i;
                    break;
                }
            }
            if (pick == n) pick = 0;
        }
    }
}

/* kmeans.cpp:118-194 */
int so_kmeans(const float* pts, uint64_t n, uint32_t dim, uint32_t k, uint32_t iters, uint64_t seed,
              float* cent, uint32_t* assign, uint32_t* repaired, uint32_t* nrepaired, double* wcss) {
    if (k < 1) return fail(SO_CONFIG, "kmeans: k must be >= 1");
    if (iters < 1) return fail(SO_CONFIG, "kmeans: iterations must be >= 1");
    if (n < k) return fail(SO_CONFIG, "kmeans: n = %llu is smaller than k = %u", (unsigned long long)n, k);
    double* min_dist = malloc(sizeof(double) * n);
    unsigned char* chosen = malloc(n);
    double* sums = malloc(sizeof(double) * (size_t)k * dim);
    uint64_t* counts = malloc(sizeof(uint64_t) * k);
    if (!min_dist || !chosen || !sums || !counts) {
        free(min_dist), free(chosen), free(sums), free(counts);
        return fail(SO_INTERNAL, "out of memory");
    }
    so_mt g;
    so_mt_seed(&g, seed);
    kmeanspp(pts, n, dim, k, &g, cent, min_dist, chosen);
    uint32_t nrep = 0;
    for (uint32_t it = 0; it < iters; ++it) {
        const double w = assign_all(pts, n, dim, cent, k, assign);
        if (wcss) wcss[it] = w;
        /* update: serial sums in point order (kmeans.cpp:153-168) */
        memset(sums, 0, sizeof(double) * (size_t)k * dim);
        memset(counts, 0, sizeof(uint64_t) * k);
        for (uint64_t i = 0; i < n; ++i) {
            const uint32_t c = assign[i];
            double* dst = sums + (size_t)c * dim;
            const float* src = pts + i * dim;
            for (uint32_t j = 0; j < dim; ++j) dst[j] += src[j];
            ++counts[c];
        }
        for (uint32_t c = 0; c < k; ++c) {
            if (counts[c] == 0) continue;
            const double inv = 1.0 / (double)counts[c];
            for (uint32_t j = 0; j < dim; ++j) {
                cent[(size_t)c * dim + j] = (float)(sums[(size_t)c * dim + j] * inv);
            }
        }
        /* empty-cluster repair: farthest from the stale centroid, strict '>' (kmeans.cpp:172-188) */
        for (uint32_t c = 0; c < k; ++c) {
            if (counts[c] != 0) continue;
            const float* stale = cent + (size_t)c * dim;
            uint64_t far = 0;
            double fd = -1.0;
            for (uint64_t i = 0; i < n; ++i) {
                const double dist = so_sqdist4(pts + i * dim, stale, dim);
                if (dist > fd) {
                    fd = dist;
                    far = i;
                }
            }
            memcpy(cent + (size_t)c * dim, pts + far * dim, 4 * (size_t)dim);
            if (repaired) repaired[nrep] = c;
            ++nrep;
        }
    }
    assign_all(pts, n, dim, cent, k, assign);
    if (nrepaired) *nrepaired = nrep;
    free(min_dist), free(chosen), free(sums), free(counts);
    return SO_OK;
}

/* ------------------------------------------------------------------- IMI */

/* index.cpp:69-96: counting sort, ids ascending within a cell */
int so_build_imi(const uint32_t* first, const uint32_t* second, uint64_t n, uint32_t k_half,
                 uint64_t* offsets, uint32_t* ids) {
    if (k_half < 1) return fail(SO_CONTRACT, "build_imi: k_half must be >= 1");
    const uint64_t cells = (uint64_t)k_half * k_half;
    memset(offsets, 0, sizeof(uint64_t) * (cells + 1));
    for (uint64_t i = 0; i < n; ++i) {
        if (first[i] >= k_half || second[i] >= k_half) {
            return fail(SO_CONTRACT, "assignment out of range at point %llu", (unsigned long long)i);
        }
        ++offsets[(uint64_t)first[i] * k_half + second[i] + 1];
    }
    for (uint64_t c = 1; c <= cells; ++c) offsets[c] += offsets[c - 1];
    uint64_t* cursor = malloc(sizeof(uint64_t) * cells);
    if (!cursor) return fail(SO_INTERNAL, "out of memory");
    memcpy(cursor, offsets, sizeof(uint64_t) * cells);
    for (uint64_t i = 0; i < n; ++i) ids[cursor[(uint64_t)first[i] * k_half + second[i]]++] = (uint32_t)i;
    free(cursor);
    return SO_OK;
}

/* ----------------------------------------------------------------- index */

struct so_index {
    uint64_t n, seed;
    uint32_t d, ns, k_half, iters, mode;
    uint32_t* dims;  /* d: concatenated per-subspace dimension lists */
    uint32_t* start; /* ns: first position of subspace i in dims */
    uint32_t* size;  /* ns */
    uint32_t* split; /* ns: first-half dimension count */
    float** cent1;   /* ns x (k_half x h1) */
    float** cent2;
    uint64_t** offsets; /* ns x (K+1) */
    uint32_t** ids;     /* ns x n */
};

void so_index_free(so_index* x) {
    if (!x) return;
    for (uint32_t s = 0; s < x->ns; ++s) {
        if (x->cent1) free(x->cent1[s]);
        if (x->cent2) free(x->cent2[s]);
        if (x->offsets) free(x->offsets[s]);
        if (x->ids) free(x->ids[s]);
    }
    free(x->cent1), free(x->cent2), free(x->offsets), free(x->ids);
    free(x->dims), free(x->start), free(x->size), free(x->split);
    free(x);
}

static so_index* index_alloc(uint32_t d, uint32_t ns) {
    so_index* x = calloc(1, sizeof(so_index));
    if (!x) return NULL;
    x->d = d;
    x->ns = ns;
    x->dims = calloc(d, 4);
    x->start = calloc(ns, 4);
    x->size = calloc(ns, 4);
    x->split = calloc(ns, 4);
    x->cent1 = calloc(ns, sizeof(float*));
    x->cent2 = calloc(ns, sizeof(float*));
    x->offsets = calloc(ns, sizeof(uint64_t*));
    x->ids = calloc(ns, sizeof(uint32_t*));
    if (!x->dims || !x->start || !x->size || !x->split || !x->cent1 || !x->cent2 || !x->offsets || !x->ids) {
        so_index_free(x);
        return NULL;
    }
    return x;
}

int so_index_info(const so_index* x, uint64_t* n, uint32_t* d, uint32_t* ns, uint32_t* k_half) {
    *n = x->n;
    *d = x->d;
    *ns = x->ns;
    *k_half = x->k_half;
    return SO_OK;
}

static uint32_t half_dim(const so_index* x, uint32_t s, int half) {
    return half == 0 ? x->split[s] : x->size[s] - x->split[s];
}

/* subspace.cpp:83-92 */
static void project(const so_index* x, const float* point, uint32_t s, int half, float* out) {
    const uint32_t lo = half == 0 ? 0 : x->split[s];
    const uint32_t hi = half == 0 ? x->split[s] : x->size[s];
    const uint32_t* dims = x->dims + x->start[s];
    for (uint32_t k = lo; k < hi; ++k) out[k - lo] = point[dims[k]];
}

typedef struct {
    const so_index* x;
    const float* data;
    uint64_t n;
    uint32_t* const* assign; /* 2*ns arrays */
    const uint32_t* train;   /* sampled build: ascending training-row ids (NULL: every row trains) */
    uint64_t n_train;
    int rc;
    char err[512];
    unsigned next;
    pthread_mutex_t mu;
} build_ctx;

/* one (subspace, half) job of index.cpp:120-137 */
static int build_job(build_ctx* b, unsigned job) {
    const so_index* x = b->x;
    const uint32_t s = job / 2;
    const int half = (int)(job % 2);
    const uint32_t h = half_dim(x, s, half);
    const uint64_t n = b->train ? b->n_train : b->n;
    float* proj = malloc(sizeof(float) * n * h);
    if (!proj) return fail(SO_INTERNAL, "out of memory");
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t row = b->train ? b->train[i] : i;
        project(x, b->data + row * x->d, s, half, proj + i * h);
    }
    float* cent = malloc(sizeof(float) * (size_t)x->k_half * h);
    uint32_t* kassign = b->train ? malloc(sizeof(uint32_t) * n) : b->assign[job];
    int rc = kassign ? so_kmeans(proj, n, h, x->k_half, x->iters, so_derive_seed(x->seed, job), cent, kassign, NULL,
                                 NULL, NULL)
                     : fail(SO_INTERNAL, "out of memory");
    free(proj);
    if (b->train) {
        /* sampled build: every row goes to its nearest trained centroid, kmeans.cpp:19-33's rule
           (the same rule as the k-means final assignment pass, kmeans.cpp:190-191) */
        float* tmp = malloc(sizeof(float) * (h ? h : 1));
        if (!tmp && !rc) rc = fail(SO_INTERNAL, "out of memory");
        for (uint64_t i = 0; !rc && i < b->n; ++i) {
            double dist;
            project(x, b->data + i * x->d, s, half, tmp);
            b->assign[job][i] = nearest(tmp, cent, x->k_half, h, &dist);
        }
        free(tmp);
        free(kassign);
    }
    if (half == 0) x->cent1[s] = cent;
    else x->cent2[s] = cent;
    return rc;
}

static void* build_worker(void* arg) {
    build_ctx* b = arg;
    for (;;) {
        pthread_mutex_lock(&b->mu);
        const unsigned job = b->next++;
        const int stop = b->rc != 0;
        pthread_mutex_unlock(&b->mu);
        if (stop || job >= 2 * b->x->ns) return NULL;
        const int rc = build_job(b, job);
        if (rc) {
            pthread_mutex_lock(&b->mu);
            if (!b->rc) {
                b->rc = rc;
                snprintf(b->err, sizeof b->err, "%s", g_err);
            }
            pthread_mutex_unlock(&b->mu);
        }
    }
}

static int check_dataset(const float* data, uint64_t n, uint32_t d) {
    /* core.cpp:8-21 */
    if (n < 1 || d < 1) return fail(SO_CONTRACT, "dataset requires n >= 1 and d >= 1");
    for (uint64_t i = 0; i < n * d; ++i) {
        if (!isfinite(data[i])) return fail(SO_CONTRACT, "dataset component %llu is not finite", (unsigned long long)i);
    }
    return SO_OK;
}

/* index.cpp:98-145; train != NULL: the sampled build (see so_build_index_sampled) */
static int build_index_impl(const float* data, uint64_t n, uint32_t d, uint32_t ns, uint32_t k_half, uint32_t iters,
                            uint64_t seed, uint32_t mode, unsigned threads, const uint32_t* train, uint64_t n_train,
                            so_index** out) {
    int rc = check_dataset(data, n, d);
    if (rc) return rc;
    if (k_half < 1) return fail(SO_CONFIG, "k_half must be >= 1");
    if (iters < 1) return fail(SO_CONFIG, "iterations must be >= 1");
    const uint64_t n_fit = train ? n_train : n;
    if (n_fit < k_half) {
        return fail(SO_CONFIG, "%s has n = %llu points, fewer than k_half = %u", train ? "training sample" : "dataset",
                    (unsigned long long)n_fit, k_half);
    }
    if (n > 0xFFFFFFFFULL) return fail(SO_CONTRACT, "dataset exceeds 32-bit point-id capacity");
    for (uint64_t i = 0; train && i < n_train; ++i) {
        if (train[i] >= n || (i && train[i] <= train[i - 1])) {
            return fail(SO_CONTRACT, "training ids must be strictly ascending and < n (entry %llu)",
                        (unsigned long long)i);
        }
    }
    if (ns < 2) return fail(SO_CONFIG, "sample_subspaces: need at least 2 subspaces, got %u", ns);
    so_index* x = index_alloc(d, ns);
    if (!x) return fail(SO_INTERNAL, "out of memory");
    x->n = n;
    x->seed = seed;
    x->k_half = k_half;
    x->iters = iters;
    x->mode = mode;
    rc = so_sample_subspaces(d, ns, mode, seed, x->dims, x->size, x->split);
    if (rc) {
        so_index_free(x);
        return rc;
    }
    for (uint32_t s = 1; s < ns; ++s) x->start[s] = x->start[s - 1] + x->size[s - 1];

    uint32_t** assign = calloc(2 * ns, sizeof(uint32_t*));
    for (uint32_t j = 0; j < 2 * ns; ++j) assign[j] = malloc(sizeof(uint32_t) * n);
    build_ctx b = {.x = x, .data = data, .n = n, .assign = assign, .train = train, .n_train = n_train, .rc = 0,
                   .next = 0};
    pthread_mutex_init(&b.mu, NULL);
    unsigned nt = threads == 0 ? 8 : threads;
    if (nt > 2 * ns) nt = 2 * ns;
    pthread_t* th = malloc(sizeof(pthread_t) * nt);
    for (unsigned t = 0; t < nt; ++t) pthread_create(&th[t], NULL, build_worker, &b);
    for (unsigned t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&b.mu);
    rc = b.rc;
    if (rc) snprintf(g_err, sizeof g_err, "%s", b.err);
    const uint64_t cells = (uint64_t)k_half * k_half;
    for (uint32_t s = 0; !rc && s < ns; ++s) {
        x->offsets[s] = malloc(sizeof(uint64_t) * (cells + 1));
        x->ids[s] = malloc(sizeof(uint32_t) * n);
        rc = so_build_imi(assign[2 * s], assign[2 * s + 1], n, k_half, x->offsets[s], x->ids[s]);
    }
    for (uint32_t j = 0; j < 2 * ns; ++j) free(assign[j]);
    free(assign);
    if (rc) {
        so_index_free(x);
        return rc;
    }
    *out = x;
    return SO_OK;
}

int so_build_index(const float* data, uint64_t n, uint32_t d, uint32_t ns, uint32_t k_half, uint32_t iters,
                   uint64_t seed, uint32_t mode, unsigned threads, so_index** out) {
    return build_index_impl(data, n, d, ns, k_half, iters, seed, mode, threads, NULL, 0, out);
}

int so_build_index_sampled(const float* data, uint64_t n, uint32_t d, uint32_t ns, uint32_t k_half, uint32_t iters,
                           uint64_t seed, uint32_t mode, const uint32_t* train, uint64_t n_train, unsigned threads,
                           so_index** out) {
    if (!train) return fail(SO_CONTRACT, "training ids are null");
    return build_index_impl(data, n, d, ns, k_half, iters, seed, mode, threads, train, n_train, out);
}

/* ------------------------------------------------------------ persistence */

typedef struct {
    unsigned char* buf;
    uint64_t cap, pos;
} wbuf;

static void put32(wbuf* w, uint32_t v) {
    if (w->buf && w->pos + 4 <= w->cap) {
        for (int i = 0; i < 4; ++i) w->buf[w->pos + i] = (unsigned char)(v >> (8 * i));
    }
    w->pos += 4;
}
static void put64(wbuf* w, uint64_t v) {
    put32(w, (uint32_t)v);
    put32(w, (uint32_t)(v >> 32));
}
static void putf(wbuf* w, float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    put32(w, u);
}

/* index.cpp:147-170 (format: README.md:138-146) */
int so_serialize_index(const so_index* x, unsigned char* buf, uint64_t cap, uint64_t* len) {
    wbuf w = {buf, cap, 0};
    if (buf && cap >= 4) memcpy(buf, "SUCO", 4);
    w.pos = 4;
    put32(&w, 1);
    put64(&w, x->n);
    put32(&w, x->d);
    put32(&w, x->ns);
    put32(&w, x->k_half);
    put32(&w, x->iters);
    put64(&w, x->seed);
    put32(&w, x->mode);
    for (uint32_t s = 0; s < x->ns; ++s) {
        put32(&w, x->size[s]);
        for (uint32_t j = 0; j < x->size[s]; ++j) put32(&w, x->dims[x->start[s] + j]);
    }
    const uint64_t cells = (uint64_t)x->k_half * x->k_half;
    for (uint32_t s = 0; s < x->ns; ++s) {
        const uint64_t c1 = (uint64_t)x->k_half * half_dim(x, s, 0), c2 = (uint64_t)x->k_half * half_dim(x, s, 1);
        for (uint64_t i = 0; i < c1; ++i) putf(&w, x->cent1[s][i]);
        for (uint64_t i = 0; i < c2; ++i) putf(&w, x->cent2[s][i]);
        for (uint64_t i = 0; i <= cells; ++i) put64(&w, x->offsets[s][i]);
        for (uint64_t i = 0; i < x->n; ++i) put32(&w, x->ids[s][i]);
    }
    *len = w.pos;
    if (buf && cap < w.pos) return fail(SO_CONTRACT, "serialize: buffer too small");
    return SO_OK;
}

typedef struct {
    const unsigned char* p;
    uint64_t len, pos;
    const char* section;
} rbuf;

static int need(rbuf* r, uint64_t count, const char* section) {
    if (r->len - r->pos < count) {
        return fail(SO_FORMAT, "index file truncated in section '%s' at byte offset %llu", section,
                    (unsigned long long)r->pos);
    }
    return SO_OK;
}
static int get32(rbuf* r, const char* section, uint32_t* v) {
    const int rc = need(r, 4, section);
    if (rc) return rc;
    *v = (uint32_t)r->p[r->pos] | ((uint32_t)r->p[r->pos + 1] << 8) | ((uint32_t)r->p[r->pos + 2] << 16) |
         ((uint32_t)r->p[r->pos + 3] << 24);
    r->pos += 4;
    return SO_OK;
}
static int get64(rbuf* r, const char* section, uint64_t* v) {
    uint32_t lo, hi;
    int rc = get32(r, section, &lo);
    if (!rc) rc = get32(r, section, &hi);
    if (!rc) *v = (uint64_t)lo | ((uint64_t)hi << 32);
    return rc;
}

/* index.cpp:191-293: every violation is a CorruptIndexError naming its section */
int so_deserialize_index(const unsigned char* bytes, uint64_t len, so_index** out) {
    rbuf r = {bytes, len, 0, ""};
    int rc;
    so_index* x = NULL;
    unsigned char* seen = NULL;
    if ((rc = need(&r, 4, "magic"))) return rc;
    if (memcmp(bytes, "SUCO", 4) != 0) return fail(SO_FORMAT, "index section 'magic': bad magic bytes");
    r.pos = 4;
    uint32_t version, d, ns, k_half, iters, mode;
    uint64_t n, seed;
    if ((rc = get32(&r, "version", &version))) return rc;
    if (version != 1) return fail(SO_FORMAT, "index section 'version': unsupported format version %u", version);
    if ((rc = get64(&r, "header", &n)) || (rc = get32(&r, "header", &d)) || (rc = get32(&r, "header", &ns)) ||
        (rc = get32(&r, "header", &k_half)) || (rc = get32(&r, "header", &iters)) ||
        (rc = get64(&r, "header", &seed)) || (rc = get32(&r, "header", &mode))) {
        return rc;
    }
    if (n < 1) return fail(SO_FORMAT, "index section 'header': n must be >= 1");
    if (n > 0xFFFFFFFFULL) return fail(SO_FORMAT, "index section 'header': n exceeds 32-bit point-id capacity");
    if (d < 1) return fail(SO_FORMAT, "index section 'header': d must be >= 1");
    if (ns < 2) return fail(SO_FORMAT, "index section 'header': subspace count must be >= 2");
    if (k_half < 1) return fail(SO_FORMAT, "index section 'header': k_half must be >= 1");
    if (iters < 1) return fail(SO_FORMAT, "index section 'header': iterations must be >= 1");
    if (n < k_half) return fail(SO_FORMAT, "index section 'header': n smaller than k_half");
    if (mode > 1) return fail(SO_FORMAT, "index section 'header': unknown subspace mode %u", mode);

    x = index_alloc(d, ns);
    seen = calloc(d > n ? d : n, 1);
    if (!x || !seen) {
        rc = fail(SO_INTERNAL, "out of memory");
        goto done;
    }
    x->n = n, x->seed = seed, x->k_half = k_half, x->iters = iters, x->mode = mode;
    uint32_t pos = 0;
    for (uint32_t s = 0; s < ns; ++s) {
        uint32_t count;
        if ((rc = get32(&r, "layout", &count))) goto done;
        if (count < 2) {
            rc = fail(SO_FORMAT, "index section 'layout': subspace %u has < 2 dimensions", s);
            goto done;
        }
        x->start[s] = pos;
        x->size[s] = count;
        x->split[s] = count / 2;
        for (uint32_t j = 0; j < count; ++j) {
            uint32_t dim;
            if ((rc = get32(&r, "layout", &dim))) goto done;
            if (dim >= d) {
                rc = fail(SO_FORMAT, "index section 'layout': dimension index %u >= d", dim);
                goto done;
            }
            if (seen[dim]) {
                rc = fail(SO_FORMAT, "index section 'layout': dimension %u repeated", dim);
                goto done;
            }
            seen[dim] = 1;
            x->dims[pos++] = dim;
        }
    }
    for (uint32_t dim = 0; dim < d; ++dim) {
        if (!seen[dim]) {
            rc = fail(SO_FORMAT, "index section 'layout': dimension %u missing", dim);
            goto done;
        }
    }
    const uint64_t cells = (uint64_t)k_half * k_half;
    for (uint32_t s = 0; s < ns; ++s) {
        const uint64_t c1 = (uint64_t)k_half * half_dim(x, s, 0), c2 = (uint64_t)k_half * half_dim(x, s, 1);
        x->cent1[s] = malloc(4 * c1);
        x->cent2[s] = malloc(4 * c2);
        x->offsets[s] = malloc(8 * (cells + 1));
        x->ids[s] = malloc(4 * n);
        for (uint64_t i = 0; i < c1 + c2; ++i) {
            uint32_t u;
            if ((rc = get32(&r, "centroids", &u))) goto done;
            float f;
            memcpy(&f, &u, 4);
            if (!isfinite(f)) {
                rc = fail(SO_FORMAT, "index section 'centroids': non-finite centroid value");
                goto done;
            }
            if (i < c1) x->cent1[s][i] = f;
            else x->cent2[s][i - c1] = f;
        }
        for (uint64_t c = 0; c <= cells; ++c) {
            if ((rc = get64(&r, "imi offsets", &x->offsets[s][c]))) goto done;
            if (c == 0 && x->offsets[s][0] != 0) {
                rc = fail(SO_FORMAT, "index section 'imi offsets': first offset must be 0");
                goto done;
            }
            if (c > 0 && x->offsets[s][c] < x->offsets[s][c - 1]) {
                rc = fail(SO_FORMAT, "index section 'imi offsets': offsets decrease at cell %llu",
                          (unsigned long long)(c - 1));
                goto done;
            }
        }
        if (x->offsets[s][cells] != n) {
            rc = fail(SO_FORMAT, "index section 'imi offsets': offsets do not cover n points");
            goto done;
        }
        memset(seen, 0, n);
        for (uint64_t i = 0; i < n; ++i) {
            uint32_t id;
            if ((rc = get32(&r, "imi ids", &id))) goto done;
            if (id >= n) {
                rc = fail(SO_FORMAT, "index section 'imi ids': point id %u >= n", id);
                goto done;
            }
            if (seen[id]) {
                rc = fail(SO_FORMAT, "index section 'imi ids': point id %u repeated", id);
                goto done;
            }
            seen[id] = 1;
            x->ids[s][i] = id;
        }
    }
    if (r.pos != len) {
        rc = fail(SO_FORMAT, "index section 'trailer': %llu trailing bytes", (unsigned long long)(len - r.pos));
        goto done;
    }
    rc = SO_OK;
done:
    free(seen);
    if (rc) so_index_free(x);
    else *out = x;
    return rc;
}

/* ------------------------------------------------------------------ query */

typedef struct {
    double d;
    uint32_t id;
} dist_id;

static int cmp_dist_id(const void* a, const void* b) {
    const dist_id* x = a;
    const dist_id* y = b;
    if (x->d != y->d) return x->d < y->d ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

/* query.cpp:42-64: true Euclidean (sqrt), order by (dist, id) */
int so_centroid_distances(const float* q, uint32_t dim, const float* cent, uint32_t k_half, double* dists,
                          uint32_t* order) {
    if (k_half < 1) return fail(SO_CONTRACT, "k_half must be >= 1");
    if (dim == 0) return fail(SO_CONTRACT, "query half is empty");
    dist_id* tmp = malloc(sizeof(dist_id) * k_half);
    if (!tmp) return fail(SO_INTERNAL, "out of memory");
    for (uint32_t c = 0; c < k_half; ++c) {
        dists[c] = sqrt(so_sqdist4(cent + (size_t)c * dim, q, dim));
        tmp[c].d = dists[c];
        tmp[c].id = c;
    }
    qsort(tmp, k_half, sizeof(dist_id), cmp_dist_id);
    for (uint32_t c = 0; c < k_half; ++c) order[c] = tmp[c].id;
    free(tmp);
    return SO_OK;
}

typedef struct {
    double sum;
    uint32_t i, j;
} cell_key;

static int cmp_cell(const void* a, const void* b) {
    const cell_key* x = a;
    const cell_key* y = b;
    if (x->sum != y->sum) return x->sum < y->sum ? -1 : 1;
    if (x->i != y->i) return x->i < y->i ? -1 : 1;
    return (x->j > y->j) - (x->j < y->j);
}

/* query.cpp:66-121 (kind 0: Dynamic Activation) and oracles.cpp:63-88 (kind 2:
 * sort every cell by (sum, rank1, rank2) and cut). check_traversal_args
 * query.cpp:16-30 first. */
int so_traverse(int kind, double alpha, uint64_t n, const double* d1, const uint32_t* o1, const double* d2,
                const uint32_t* o2, uint32_t k, const uint64_t* offsets, uint32_t* c1, uint32_t* c2,
                uint64_t* cum, double* sums, uint64_t cap, uint64_t* count) {
    if (!(alpha > 0.0) || alpha > 1.0) return fail(SO_CONTRACT, "alpha must be in (0, 1]");
    if (k < 1) return fail(SO_CONTRACT, "imi has no cells");
    const uint64_t cells = (uint64_t)k * k;
    if (offsets[cells] != n) {
        return fail(SO_CONTRACT, "imi holds %llu ids but n = %llu", (unsigned long long)offsets[cells],
                    (unsigned long long)n);
    }
    const uint64_t target = so_collision_count(alpha, n);
    double* r1 = malloc(8 * (size_t)k);
    double* r2 = malloc(8 * (size_t)k);
    for (uint32_t i = 0; i < k; ++i) {
        r1[i] = d1[o1[i]];
        r2[i] = d2[o2[i]];
    }
    uint64_t got = 0, cumulative = 0;
    int rc = SO_OK;
#define EMIT(ci, cj, s)                                                         \
    do {                                                                        \
        const uint32_t a_ = o1[ci], b_ = o2[cj];                                \
        cumulative += offsets[(uint64_t)a_ * k + b_ + 1] - offsets[(uint64_t)a_ * k + b_]; \
        if (got < cap) {                                                        \
            c1[got] = a_;                                                       \
            c2[got] = b_;                                                       \
            cum[got] = cumulative;                                              \
            sums[got] = (s);                                                    \
        }                                                                       \
        ++got;                                                                  \
    } while (0)
    if (kind == 0) {
        uint32_t* cur = calloc(k, 4);
        double* act = malloc(8 * (size_t)k);
        for (uint32_t i = 0; i < k; ++i) act[i] = INFINITY;
        act[0] = r1[0] + r2[0];
        uint32_t activated = 1;
        while (cumulative < target) {
            uint32_t pos = 0;
            double best = act[0];
            for (uint32_t i = 1; i < activated; ++i) {
                if (act[i] < best) {
                    best = act[i];
                    pos = i;
                }
            }
            if (best == INFINITY) break;
            const uint32_t j = cur[pos];
            EMIT(pos, j, best);
            if (j == 0 && activated < k) {
                act[activated] = r1[activated] + r2[0];
                ++activated;
            }
            if (j + 1 == k) {
                act[pos] = INFINITY;
            } else {
                cur[pos] = j + 1;
                act[pos] = r1[pos] + r2[j + 1];
            }
        }
        free(cur), free(act);
    } else {
        cell_key* all = malloc(sizeof(cell_key) * cells);
        for (uint32_t i = 0; i < k; ++i) {
            for (uint32_t j = 0; j < k; ++j) all[(uint64_t)i * k + j] = (cell_key){r1[i] + r2[j], i, j};
        }
        qsort(all, cells, sizeof(cell_key), cmp_cell);
        for (uint64_t c = 0; c < cells; ++c) {
            EMIT(all[c].i, all[c].j, all[c].sum);
            if (cumulative >= target) break;
        }
        free(all);
    }
#undef EMIT
    free(r1), free(r2);
    *count = got;
    if (got > cap) rc = fail(SO_CONTRACT, "cell output capacity too small");
    return rc;
}

/* query.cpp:159-197 */
int so_rerank(const float* data, uint64_t n, uint32_t d, const float* query, uint32_t qlen, const uint32_t* cands,
              uint64_t m, uint32_t k, uint32_t* ids, double* dists, uint32_t* count) {
    if (qlen != d) return fail(SO_CONTRACT, "query length %u does not match dataset d = %u", qlen, d);
    if (k < 1) return fail(SO_CONTRACT, "k must be >= 1");
    if (m < k) return fail(SO_CONTRACT, "k = %u exceeds the %llu candidates", k, (unsigned long long)m);
    dist_id* s = malloc(sizeof(dist_id) * m);
    if (!s) return fail(SO_INTERNAL, "out of memory");
    for (uint64_t i = 0; i < m; ++i) {
        if (cands[i] >= n) {
            free(s);
            return fail(SO_CONTRACT, "candidate id %u out of range", cands[i]);
        }
        s[i].id = cands[i];
        s[i].d = so_sqdist4(data + (uint64_t)cands[i] * d, query, d);
    }
    qsort(s, m, sizeof(dist_id), cmp_dist_id);
    for (uint32_t i = 0; i < k; ++i) {
        ids[i] = s[i].id;
        dists[i] = sqrt(s[i].d);
    }
    *count = k;
    free(s);
    return SO_OK;
}

typedef struct {
    uint32_t score, id;
} score_id;

static int cmp_score_id(const void* a, const void* b) {
    const score_id* x = a;
    const score_id* y = b;
    if (x->score != y->score) return x->score > y->score ? -1 : 1;
    return (x->id > y->id) - (x->id < y->id);
}

typedef struct {
    uint32_t* scores; /* n */
    uint32_t* touched;
    uint64_t ntouched;
    float* half;
    uint32_t* o1;
    uint32_t* o2;
    double* dd1;
    double* dd2;
    uint32_t* c1;
    uint32_t* c2;
    uint64_t* cum;
    double* sums;
    uint32_t* cands;
    score_id* sel;
} scratch;

static int scratch_init(scratch* s, const so_index* x) {
    memset(s, 0, sizeof *s);
    const uint64_t cells = (uint64_t)x->k_half * x->k_half;
    s->scores = calloc(x->n, 4);
    s->touched = malloc(4 * x->n);
    s->half = malloc(4 * (size_t)x->d);
    s->o1 = malloc(4 * (size_t)x->k_half);
    s->o2 = malloc(4 * (size_t)x->k_half);
    s->dd1 = malloc(8 * (size_t)x->k_half);
    s->dd2 = malloc(8 * (size_t)x->k_half);
    s->c1 = malloc(4 * cells);
    s->c2 = malloc(4 * cells);
    s->cum = malloc(8 * cells);
    s->sums = malloc(8 * cells);
    s->cands = malloc(4 * x->n);
    s->sel = malloc(sizeof(score_id) * x->n);
    return (s->scores && s->touched && s->half && s->o1 && s->o2 && s->dd1 && s->dd2 && s->c1 && s->c2 && s->cum &&
            s->sums && s->cands && s->sel)
               ? SO_OK
               : fail(SO_INTERNAL, "out of memory");
}

static void scratch_free(scratch* s) {
    free(s->scores), free(s->touched), free(s->half), free(s->o1), free(s->o2), free(s->dd1), free(s->dd2);
    free(s->c1), free(s->c2), free(s->cum), free(s->sums), free(s->cands), free(s->sel);
}

/* query.cpp:199-253: scores, then the top-m candidate set by (score desc,
 * id asc) — here by an explicit sort, an independent formulation of the
 * reference's nth_element/fill. Leaves m candidates in s->cands. */
static int query_candidates(const so_index* x, const float* data, uint64_t n, uint32_t d, const float* query,
                            uint32_t qlen, double alpha, double beta, uint32_t k, scratch* s, uint64_t* m_out,
                            uint32_t* cells_per_subspace, uint64_t* cumulative) {
    (void)data;
    if (x->n != n) {
        return fail(SO_INCOMPAT, "index was built from n = %llu points but dataset has n = %llu",
                    (unsigned long long)x->n, (unsigned long long)n);
    }
    if (x->d != d) return fail(SO_INCOMPAT, "index was built for d = %u but dataset has d = %u", x->d, d);
    if (qlen != d) return fail(SO_CONTRACT, "query length %u does not match dataset d = %u", qlen, d);
    int rc = so_validate_params(alpha, beta, k, n);
    if (rc) return rc;
    for (uint64_t t = 0; t < s->ntouched; ++t) s->scores[s->touched[t]] = 0;
    s->ntouched = 0;
    const uint64_t cells = (uint64_t)x->k_half * x->k_half;
    for (uint32_t si = 0; si < x->ns; ++si) {
        const uint32_t h1 = half_dim(x, si, 0), h2 = half_dim(x, si, 1);
        project(x, query, si, 0, s->half);
        so_centroid_distances(s->half, h1, x->cent1[si], x->k_half, s->dd1, s->o1);
        project(x, query, si, 1, s->half);
        so_centroid_distances(s->half, h2, x->cent2[si], x->k_half, s->dd2, s->o2);
        uint64_t nc;
        rc = so_traverse(0, alpha, n, s->dd1, s->o1, s->dd2, s->o2, x->k_half, x->offsets[si], s->c1, s->c2,
                         s->cum, s->sums, cells, &nc);
        if (rc) return rc;
        if (cells_per_subspace) cells_per_subspace[si] = (uint32_t)nc;
        if (cumulative) cumulative[si] = nc ? s->cum[nc - 1] : 0;
        for (uint64_t c = 0; c < nc; ++c) {
            const uint64_t cell = (uint64_t)s->c1[c] * x->k_half + s->c2[c];
            for (uint64_t p = x->offsets[si][cell]; p < x->offsets[si][cell + 1]; ++p) {
                const uint32_t id = x->ids[si][p];
                if (s->scores[id]++ == 0) s->touched[s->ntouched++] = id;
            }
        }
    }
    const uint64_t m = so_candidate_count(beta, n, k);
    uint64_t got = 0;
    if (s->ntouched >= m) {
        for (uint64_t t = 0; t < s->ntouched; ++t) s->sel[t] = (score_id){s->scores[s->touched[t]], s->touched[t]};
        qsort(s->sel, s->ntouched, sizeof(score_id), cmp_score_id);
        for (uint64_t t = 0; t < m; ++t) s->cands[got++] = s->sel[t].id;
    } else {
        for (uint64_t t = 0; t < s->ntouched; ++t) s->cands[got++] = s->touched[t];
        for (uint64_t id = 0; got < m && id < n; ++id) {
            if (s->scores[id] == 0) s->cands[got++] = (uint32_t)id;
        }
    }
    *m_out = m;
    return SO_OK;
}

int so_query_intermediates(const so_index* x, const float* data, uint64_t n, uint32_t d, const float* query,
                           uint32_t qlen, double alpha, double beta, uint32_t k, uint32_t* scores, uint32_t* cands,
                           uint64_t* m_out, uint32_t* cells_per_subspace, uint64_t* cumulative) {
    scratch s;
    int rc = scratch_init(&s, x);
    if (!rc) rc = query_candidates(x, data, n, d, query, qlen, alpha, beta, k, &s, m_out, cells_per_subspace, cumulative);
    if (!rc) {
        memcpy(scores, s.scores, 4 * n);
        memcpy(cands, s.cands, 4 * *m_out);
        qsort(cands, *m_out, 4, cmp_u32);
    }
    scratch_free(&s);
    return rc;
}

typedef struct {
    const so_index* x;
    const float* data;
    uint64_t n;
    uint32_t d;
    const float* queries;
    uint64_t nq;
    uint32_t qlen;
    double alpha, beta;
    uint32_t k;
    uint32_t* ids;
    double* dists;
    uint32_t* counts;
    uint64_t next;
    int rc;
    char err[512];
    pthread_mutex_t mu;
} batch_ctx;

static void* batch_worker(void* arg) {
    batch_ctx* b = arg;
    scratch s;
    if (scratch_init(&s, b->x)) {
        pthread_mutex_lock(&b->mu);
        if (!b->rc) b->rc = SO_INTERNAL, snprintf(b->err, sizeof b->err, "%s", g_err);
        pthread_mutex_unlock(&b->mu);
        scratch_free(&s);
        return NULL;
    }
    for (;;) {
        pthread_mutex_lock(&b->mu);
        const uint64_t q = b->next++;
        const int stop = b->rc != 0;
        pthread_mutex_unlock(&b->mu);
        if (stop || q >= b->nq) break;
        uint64_t m;
        int rc = query_candidates(b->x, b->data, b->n, b->d, b->queries + q * b->qlen, b->qlen, b->alpha, b->beta,
                                  b->k, &s, &m, NULL, NULL);
        if (!rc) {
            rc = so_rerank(b->data, b->n, b->d, b->queries + q * b->qlen, b->qlen, s.cands, m, b->k,
                           b->ids + q * b->k, b->dists + q * b->k, b->counts + q);
        }
        if (rc) {
            pthread_mutex_lock(&b->mu);
            if (!b->rc) b->rc = rc, snprintf(b->err, sizeof b->err, "%s", g_err);
            pthread_mutex_unlock(&b->mu);
            break;
        }
    }
    scratch_free(&s);
    return NULL;
}

int so_knn_query_batch(const so_index* x, const float* data, uint64_t n, uint32_t d, const float* queries,
                       uint64_t nq, uint32_t qlen, double alpha, double beta, uint32_t k, unsigned threads,
                       uint32_t* ids, double* dists, uint32_t* counts, double* wall_s) {
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    batch_ctx b = {.x = x, .data = data, .n = n, .d = d, .queries = queries, .nq = nq, .qlen = qlen,
                   .alpha = alpha, .beta = beta, .k = k, .ids = ids, .dists = dists, .counts = counts};
    pthread_mutex_init(&b.mu, NULL);
    unsigned nt = threads == 0 ? 1 : threads;
    if (nt > nq) nt = nq ? (unsigned)nq : 1;
    pthread_t* th = malloc(sizeof(pthread_t) * nt);
    for (unsigned t = 0; t < nt; ++t) pthread_create(&th[t], NULL, batch_worker, &b);
    for (unsigned t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&b.mu);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    if (wall_s) *wall_s = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    if (b.rc) snprintf(g_err, sizeof g_err, "%s", b.err);
    return b.rc;
}
