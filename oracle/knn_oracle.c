/*
 * knn_oracle.c -- CPU restatement of the reference k-NN algorithm.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * engine: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path never calls it and
 * has no CPU fallback.
 *
 * It restates, in plain C, the arithmetic and selection contract of the
 * reference tknn library (paths relative to /root/reference/proj):
 *   - SplitMix64 + unit floats ........ include/knn/rng.hpp:13-23
 *   - generate_dataset ................ src/io.cpp:57-62
 *   - metric steps + fold ............. include/knn/distance.hpp:41-65, 98-105
 *   - Neighbor order .................. include/knn/heap.hpp:21-24
 *   - NeighborHeap push/sift/drain .... src/heap.cpp:18-64
 *   - brute_force_knn ................. src/oracle.cpp:10-42
 *   - the KNN_DOUBLE_ACCUM fold and brute force (types.hpp:9-13)
 * plus the SURVEY §8(d)(iii) sampled-row oracle (exact top-k for a subset of
 * query rows, multithreaded over rows), which produces the same lists as
 * brute_force_knn for those rows because the bounded heap keeps the k smallest
 * of a total order regardless of push order.
 *
 * "cosine" is not a reference built-in; it restates the custom fold SURVEY
 * §8(d) registers for config C4: step acc + u*v, finalize 1 - acc.
 *
 * Build with -ffp-contract=off (as the reference CMakeLists.txt:15-20 does):
 * every step is a separately rounded sub/mul/add.
 *
 * Pinned against (tests/test_oracle_pin.py): the reference's own KATs
 * (test_io.cpp:44-64, test_oracle.cpp:45-66, test_distance.cpp), the golden
 * fixtures in tests/golden/ produced by the compiled reference, and -- when
 * oracle/_ref was built -- the reference library itself on random instances.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* KO_MANHATTAN and KO_ROOT_SQUARES restate the custom functors the
 * reference's own tests register: test_distance.cpp:134-145 (acc +
 * dist_t(fabs(u - v))) and :166-178 (the sqeuclidean step, finalize sqrt). */
enum { KO_HELLINGER = 0, KO_SQEUCLIDEAN = 1, KO_COSINE = 2, KO_MANHATTAN = 3, KO_ROOT_SQUARES = 4 };

/* ---- rng.hpp:13-23 ---------------------------------------------------- */
uint64_t ko_splitmix64_next(uint64_t *state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

float ko_next_unit_float(uint64_t *state) {
    return (float)(ko_splitmix64_next(state) >> 40) * 0x1.0p-24f;
}

/* ---- io.cpp:57-62: row-major values from one stream ------------------- */
void ko_generate(uint32_t n, uint32_t d, uint64_t seed, float *out) {
    uint64_t s = seed;
    const size_t total = (size_t)n * d;
    for (size_t i = 0; i < total; ++i) out[i] = ko_next_unit_float(&s);
}

/* Elements [first, first + count) of the same stream.  next() only adds the
 * Weyl increment to the state (rng.hpp:13-14), so the state before element i
 * is seed + i * 0x9e3779b97f4a7c15 (mod 2^64): jump there, then step as
 * ko_generate does.  Pinned against ko_generate in tests/test_oracle_pin.py. */
void ko_generate_at(uint64_t seed, uint64_t first, uint64_t count, float *out) {
    uint64_t s = seed + first * 0x9e3779b97f4a7c15ull;
    for (uint64_t i = 0; i < count; ++i) out[i] = ko_next_unit_float(&s);
}

/* ---- distance.hpp:41-65 (+ cosine custom fold), fold 98-105 ----------- */
float ko_fold(int metric, const float *u, const float *v, uint32_t d) {
    float acc = 0.0f;
    switch (metric) {
    case KO_HELLINGER:
        for (uint32_t j = 0; j < d; ++j) {
            const float t = sqrtf(u[j]) - sqrtf(v[j]);
            acc = acc + t * t;
        }
        return acc;
    case KO_SQEUCLIDEAN:
        for (uint32_t j = 0; j < d; ++j) {
            const float t = u[j] - v[j];
            acc = acc + t * t;
        }
        return acc;
    case KO_COSINE:
        for (uint32_t j = 0; j < d; ++j) acc = acc + u[j] * v[j];
        return 1.0f - acc;
    case KO_MANHATTAN:
        for (uint32_t j = 0; j < d; ++j) acc = acc + fabsf(u[j] - v[j]);
        return acc;
    case KO_ROOT_SQUARES:
        for (uint32_t j = 0; j < d; ++j) {
            const float t = u[j] - v[j];
            acc = acc + t * t;
        }
        return sqrtf(acc);
    default:
        return NAN;
    }
}

/* ---- heap.hpp:16-27 Neighbor, heap.cpp:18-64 NeighborHeap ------------- */
typedef struct {
    float distance;
    uint32_t index;
} ko_neighbor;

static int nb_less(ko_neighbor a, ko_neighbor b) {
    if (a.distance != b.distance) return a.distance < b.distance;
    return a.index < b.index;
}

typedef struct {
    uint32_t capacity;
    uint32_t size;
    ko_neighbor *e;
} ko_heap;

static void heap_sift_up(ko_heap *h, size_t i) {
    while (i > 0) {
        const size_t parent = (i - 1) / 2;
        if (!nb_less(h->e[parent], h->e[i])) break;
        ko_neighbor t = h->e[parent];
        h->e[parent] = h->e[i];
        h->e[i] = t;
        i = parent;
    }
}

static void heap_sift_down(ko_heap *h, size_t i, size_t limit) {
    for (;;) {
        const size_t left = 2 * i + 1;
        if (left >= limit) break;
        size_t largest = left;
        const size_t right = left + 1;
        if (right < limit && nb_less(h->e[largest], h->e[right])) largest = right;
        if (!nb_less(h->e[i], h->e[largest])) break;
        ko_neighbor t = h->e[i];
        h->e[i] = h->e[largest];
        h->e[largest] = t;
        i = largest;
    }
}

static int heap_push(ko_heap *h, ko_neighbor c) {
    if (h->size < h->capacity) {
        h->e[h->size++] = c;
        heap_sift_up(h, h->size - 1);
        return 1;
    }
    if (nb_less(c, h->e[0])) {
        h->e[0] = c;
        heap_sift_down(h, 0, h->size);
        return 1;
    }
    return 0;
}

/* In-place heapsort (heap.cpp:32-42): leaves e[0..size) ascending. */
static void heap_drain_sorted(ko_heap *h) {
    for (size_t m = h->size; m > 1; --m) {
        ko_neighbor t = h->e[0];
        h->e[0] = h->e[m - 1];
        h->e[m - 1] = t;
        heap_sift_down(h, 0, m - 1);
    }
}

/* Exposed for the heap-property tests (SPEC heap_push / drain examples).
 * Pushes `count` candidates into a heap of `capacity` and writes the drained
 * ascending contents; returns how many were written. */
uint32_t ko_heap_stream(uint32_t capacity, const float *dist, const uint32_t *index,
                        uint32_t count, float *out_dist, uint32_t *out_index) {
    ko_heap h = {capacity, 0, (ko_neighbor *)malloc(sizeof(ko_neighbor) * capacity)};
    for (uint32_t i = 0; i < count; ++i) {
        ko_neighbor c = {dist[i], index[i]};
        heap_push(&h, c);
    }
    heap_drain_sorted(&h);
    for (uint32_t i = 0; i < h.size; ++i) {
        out_dist[i] = h.e[i].distance;
        out_index[i] = h.e[i].index;
    }
    const uint32_t n = h.size;
    free(h.e);
    return n;
}

/* ---- oracle.cpp:10-42 brute_force_knn -------------------------------- */
/* Outputs are row-major n x min(k, n-1). Returns 0, or 2 for a bad k/n. */
int ko_brute_force(const float *x, uint32_t n, uint32_t d, uint32_t k, int metric,
                   uint32_t *out_index, float *out_dist, uint64_t *pair_evaluations) {
    if (k < 1 || n < 2 || d < 1) return 2;
    const uint32_t cap = k < n - 1 ? k : n - 1;
    ko_neighbor *store = (ko_neighbor *)malloc(sizeof(ko_neighbor) * (size_t)n * cap);
    ko_heap *heaps = (ko_heap *)malloc(sizeof(ko_heap) * n);
    if (!store || !heaps) {
        free(store);
        free(heaps);
        return 4;
    }
    for (uint32_t i = 0; i < n; ++i) {
        heaps[i].capacity = cap;
        heaps[i].size = 0;
        heaps[i].e = store + (size_t)i * cap;
    }
    uint64_t pairs = 0;
    for (uint32_t xi = 1; xi < n; ++xi) {
        const float *vx = x + (size_t)xi * d;
        for (uint32_t y = 0; y < xi; ++y) {
            const float dist = ko_fold(metric, vx, x + (size_t)y * d, d);
            ko_neighbor a = {dist, xi}, b = {dist, y};
            heap_push(&heaps[y], a);
            heap_push(&heaps[xi], b);
            ++pairs;
        }
    }
    for (uint32_t i = 0; i < n; ++i) {
        heap_drain_sorted(&heaps[i]);
        for (uint32_t j = 0; j < cap; ++j) {
            out_index[(size_t)i * cap + j] = heaps[i].e[j].index;
            out_dist[(size_t)i * cap + j] = heaps[i].e[j].distance;
        }
    }
    if (pair_evaluations) *pair_evaluations = pairs;
    free(store);
    free(heaps);
    return 0;
}

/* ---- KNN_DOUBLE_ACCUM build (types.hpp:9-13: dist_t = double) --------- */
/* distance.hpp:49-52 / :59-62 with dist_t = double: t stays a float
 * (su - sv rounded in single precision); acc + dist_t(t) * dist_t(t) in
 * double.  Hellinger stages sqrtf once per coordinate (distance.hpp:47). */
double ko_fold_f64(int metric, const float *u, const float *v, uint32_t d) {
    double acc = 0.0;
    switch (metric) {
    case KO_HELLINGER:
        for (uint32_t j = 0; j < d; ++j) {
            const float t = sqrtf(u[j]) - sqrtf(v[j]);
            acc = acc + (double)t * (double)t;
        }
        return acc;
    case KO_SQEUCLIDEAN:
        for (uint32_t j = 0; j < d; ++j) {
            const float t = u[j] - v[j];
            acc = acc + (double)t * (double)t;
        }
        return acc;
    case KO_COSINE:
        for (uint32_t j = 0; j < d; ++j) acc = acc + (double)u[j] * (double)v[j];
        return 1.0 - acc;
    case KO_MANHATTAN:
        for (uint32_t j = 0; j < d; ++j) acc = acc + (double)fabsf(u[j] - v[j]);
        return acc;
    case KO_ROOT_SQUARES:
        for (uint32_t j = 0; j < d; ++j) {
            const float t = u[j] - v[j];
            acc = acc + (double)t * (double)t;
        }
        return sqrt(acc);
    default:
        return NAN;
    }
}

typedef struct {
    double distance;
    uint32_t index;
} ko_neighbor64;

static int nb64_cmp(const void *pa, const void *pb) {
    const ko_neighbor64 *a = (const ko_neighbor64 *)pa, *b = (const ko_neighbor64 *)pb;
    if (a->distance != b->distance) return a->distance < b->distance ? -1 : 1;
    return a->index < b->index ? -1 : (a->index > b->index);
}

/* brute_force_knn (oracle.cpp:10-42) in the double build.  Each row's list is
 * the min(k, n-1) smallest of its n-1 (distance, index) pairs in Neighbor
 * order (heap.hpp:21-24); the bounded heap keeps exactly those whatever the
 * push order (acceptance criterion 6), so this selects them by sorting.  The
 * distance of {x, y} is fold(v_x, v_y) with x > y, as oracle.cpp:27. */
int ko_brute_force_f64(const float *x, uint32_t n, uint32_t d, uint32_t k, int metric,
                       uint32_t *out_index, double *out_dist) {
    if (k < 1 || n < 2 || d < 1) return 2;
    const uint32_t cap = k < n - 1 ? k : n - 1;
    ko_neighbor64 *row = (ko_neighbor64 *)malloc(sizeof(ko_neighbor64) * n);
    if (!row) return 4;
    for (uint32_t q = 0; q < n; ++q) {
        uint32_t m = 0;
        for (uint32_t y = 0; y < n; ++y) {
            if (y == q) continue;
            const uint32_t hi = y > q ? y : q, lo = y > q ? q : y;
            row[m].distance = ko_fold_f64(metric, x + (size_t)hi * d, x + (size_t)lo * d, d);
            row[m].index = y;
            ++m;
        }
        qsort(row, m, sizeof(ko_neighbor64), nb64_cmp);
        for (uint32_t j = 0; j < cap; ++j) {
            out_index[(size_t)q * cap + j] = row[j].index;
            out_dist[(size_t)q * cap + j] = row[j].distance;
        }
    }
    free(row);
    return 0;
}

/* The double build's lists for a subset of query rows (same selection as
 * ko_brute_force_f64, row by row). Outputs are nrows x min(k, n-1). */
int ko_rows_topk_f64(const float *x, uint32_t n, uint32_t d, uint32_t k, int metric, const uint32_t *rows,
                     uint32_t nrows, uint32_t *out_index, double *out_dist) {
    if (k < 1 || n < 2 || d < 1) return 2;
    const uint32_t cap = k < n - 1 ? k : n - 1;
    ko_neighbor64 *row = (ko_neighbor64 *)malloc(sizeof(ko_neighbor64) * n);
    if (!row) return 4;
    for (uint32_t r = 0; r < nrows; ++r) {
        const uint32_t q = rows[r];
        uint32_t m = 0;
        for (uint32_t y = 0; y < n; ++y) {
            if (y == q) continue;
            const uint32_t hi = y > q ? y : q, lo = y > q ? q : y;
            row[m].distance = ko_fold_f64(metric, x + (size_t)hi * d, x + (size_t)lo * d, d);
            row[m].index = y;
            ++m;
        }
        qsort(row, m, sizeof(ko_neighbor64), nb64_cmp);
        for (uint32_t j = 0; j < cap; ++j) {
            out_index[(size_t)r * cap + j] = row[j].index;
            out_dist[(size_t)r * cap + j] = row[j].distance;
        }
    }
    free(row);
    return 0;
}

/* ---- sampled-row oracle ---------------------------- */
typedef struct {
    const float *x;
    uint32_t n, d, cap;
    int metric;
    const uint32_t *rows;
    uint32_t nrows;
    uint32_t *out_index;
    float *out_dist;
    uint32_t next; /* work counter, guarded by mu */
    pthread_mutex_t mu;
} rows_job;

static void rows_one(rows_job *j, uint32_t r, ko_neighbor *buf) {
    const uint32_t q = j->rows[r];
    ko_heap h = {j->cap, 0, buf};
    const float *vq = j->x + (size_t)q * j->d;
    for (uint32_t i = 0; i < j->n; ++i) {
        if (i == q) continue;
        /* Reference argument order: the larger index first (oracle.cpp:24-26). */
        const float *vi = j->x + (size_t)i * j->d;
        const float dist = i > q ? ko_fold(j->metric, vi, vq, j->d)
                                 : ko_fold(j->metric, vq, vi, j->d);
        ko_neighbor c = {dist, i};
        heap_push(&h, c);
    }
    heap_drain_sorted(&h);
    for (uint32_t t = 0; t < j->cap; ++t) {
        j->out_index[(size_t)r * j->cap + t] = h.e[t].index;
        j->out_dist[(size_t)r * j->cap + t] = h.e[t].distance;
    }
}

static void *rows_worker(void *arg) {
    rows_job *j = (rows_job *)arg;
    ko_neighbor *buf = (ko_neighbor *)malloc(sizeof(ko_neighbor) * j->cap);
    for (;;) {
        pthread_mutex_lock(&j->mu);
        const uint32_t r = j->next++;
        pthread_mutex_unlock(&j->mu);
        if (r >= j->nrows) break;
        rows_one(j, r, buf);
    }
    free(buf);
    return NULL;
}

/* Exact top-min(k, n-1) lists for the query rows `rows[0..nrows)`, computed
 * with `threads` POSIX threads. Outputs are nrows x min(k, n-1). */
int ko_rows_topk(const float *x, uint32_t n, uint32_t d, uint32_t k, int metric,
                 const uint32_t *rows, uint32_t nrows, uint32_t threads,
                 uint32_t *out_index, float *out_dist) {
    if (k < 1 || n < 2 || d < 1) return 2;
    for (uint32_t r = 0; r < nrows; ++r)
        if (rows[r] >= n) return 2;
    rows_job j;
    j.x = x;
    j.n = n;
    j.d = d;
    j.cap = k < n - 1 ? k : n - 1;
    j.metric = metric;
    j.rows = rows;
    j.nrows = nrows;
    j.out_index = out_index;
    j.out_dist = out_dist;
    j.next = 0;
    pthread_mutex_init(&j.mu, NULL);
    if (threads < 1) threads = 1;
    pthread_t *tids = (pthread_t *)malloc(sizeof(pthread_t) * threads);
    for (uint32_t t = 0; t < threads; ++t) pthread_create(&tids[t], NULL, rows_worker, &j);
    for (uint32_t t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
    free(tids);
    pthread_mutex_destroy(&j.mu);
    return 0;
}
