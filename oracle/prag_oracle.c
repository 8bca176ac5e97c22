/*
 * prag_oracle.c -- TEST INFRASTRUCTURE ONLY (see prag_oracle.h).
 *
 * Op-for-op CPU restatement of the reference hot path. Every function cites
 * the reference lines it follows (paths relative to
 * /root/reference/proj/include/prag/). Build flags (oracle/Makefile) mirror the
 * reference's CMake Release flags (-O3 -DNDEBUG, no -march) plus
 * -ffp-contract=off so no FMA contraction can change a rounding.
 *
 * Selection note: the reference sorts ALL candidates by (distance, chunk_id)
 * and truncates (annindex.hpp:54-60, :313) and sorts all nlist
 * (distance, list) pairs (annindex.hpp:277-281). Both keys are strict total
 * orders over distinct elements, so any exact selection of the first k under
 * that order yields the identical sequence; we use a bounded heap for the
 * candidates to keep large parity cases fast.
 */
#include "prag_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static void set_err(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

const char* ora_last_error(void) { return g_err; }

/* common.hpp:73-80: sequential fp32 fold of (a-b)^2. */
float ora_squared_l2(const float* a, const float* b, size_t d) {
    float acc = 0.0f;
    for (size_t i = 0; i < d; ++i) {
        float diff = a[i] - b[i];
        acc += diff * diff;
    }
    return acc;
}

/* ---- SplitMix64 (common.hpp:33-64) and hash_combine (common.hpp:66-71) ---- */
uint64_t ora_splitmix_next(uint64_t* state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static double splitmix_double(uint64_t* s) {
    return (double)(ora_splitmix_next(s) >> 11) * 0x1.0p-53;
}

double ora_splitmix_gaussian(uint64_t* s) {
    double u1 = splitmix_double(s);
    double u2 = splitmix_double(s);
    while (u1 <= 0.0) u1 = splitmix_double(s);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

uint64_t ora_hash_combine(uint64_t a, uint64_t b) {
    uint64_t z = a + 0x9e3779b97f4a7c15ULL + (b << 6) + (b >> 2);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void ora_random_vectors(uint64_t seed, uint64_t n, uint32_t d, float* out) {
    uint64_t s = seed;
    for (uint64_t i = 0; i < n * (uint64_t)d; ++i) out[i] = (float)ora_splitmix_gaussian(&s);
}

/* ---- PRAGIX01 loader: annindex.hpp:361-411 (read_pod: tokendb.hpp:176-185) ---- */
static int read_exact(FILE* f, void* dst, size_t n) { return fread(dst, 1, n, f) == n; }

void ora_free_index(ora_index* idx) {
    if (!idx) return;
    free(idx->centroids);
    free(idx->codewords);
    free(idx->list_off);
    free(idx->ids);
    free(idx->codes);
    free(idx);
}

int ora_load_index(const char* path, ora_index** out) {
    *out = NULL;
    FILE* f = fopen(path, "rb");
    if (!f) {
        set_err("cannot open for reading: %s", path);
        return ORA_FORMAT;
    }
    char magic[8];
    if (!read_exact(f, magic, 8) || memcmp(magic, "PRAGIX01", 8) != 0) {
        fclose(f);
        set_err("bad index magic at offset 0 in %s", path);
        return ORA_FORMAT;
    }
    uint64_t offset = 8;
    uint32_t hdr[4];
    static const char* names[4] = {"version", "nlist", "d", "n_subquantizers"};
    for (int i = 0; i < 4; ++i) {
        if (!read_exact(f, &hdr[i], 4)) {
            fclose(f);
            set_err("truncated or unreadable %s at offset %llu", names[i], (unsigned long long)offset);
            return ORA_FORMAT;
        }
        offset += 4;
        if (i == 0 && hdr[0] != 1) {
            fclose(f);
            set_err("unsupported index version %u in %s", hdr[0], path);
            return ORA_FORMAT;
        }
    }
    ora_index* idx = (ora_index*)calloc(1, sizeof *idx);
    idx->nlist = hdr[1];
    idx->d = hdr[2];
    idx->nsq = hdr[3];
    if (idx->nsq == 0 || idx->d % idx->nsq != 0) {
        fclose(f);
        free(idx);
        set_err("invalid n_subquantizers in %s", path);
        return ORA_FORMAT;
    }
    idx->sub_dim = idx->d / idx->nsq;
    size_t nc = (size_t)idx->nlist * idx->d;
    idx->centroids = (float*)malloc((nc ? nc : 1) * sizeof(float));
    for (uint32_t c = 0; c < idx->nlist; ++c) {
        if (!read_exact(f, idx->centroids + (size_t)c * idx->d, idx->d * sizeof(float))) {
            set_err("truncated centroids at offset %llu", (unsigned long long)offset);
            goto fail;
        }
        offset += idx->d * sizeof(float);
    }
    size_t nw = (size_t)idx->nsq * 256 * idx->sub_dim;
    idx->codewords = (float*)malloc((nw ? nw : 1) * sizeof(float));
    for (size_t w = 0; w < (size_t)idx->nsq * 256; ++w) {
        if (!read_exact(f, idx->codewords + w * idx->sub_dim, idx->sub_dim * sizeof(float))) {
            set_err("truncated codebook at offset %llu", (unsigned long long)offset);
            goto fail;
        }
        offset += idx->sub_dim * sizeof(float);
    }
    idx->list_off = (uint64_t*)calloc((size_t)idx->nlist + 1, sizeof(uint64_t));
    {
        uint64_t cap = 1024, total = 0;
        idx->ids = (uint64_t*)malloc(cap * sizeof(uint64_t));
        idx->codes = (uint8_t*)malloc(cap * idx->nsq);
        for (uint32_t l = 0; l < idx->nlist; ++l) {
            uint64_t len;
            if (!read_exact(f, &len, 8)) {
                set_err("truncated or unreadable posting list length at offset %llu",
                        (unsigned long long)offset);
                goto fail;
            }
            offset += 8;
            for (uint64_t e = 0; e < len; ++e) {
                if (total == cap) {
                    cap *= 2;
                    idx->ids = (uint64_t*)realloc(idx->ids, cap * sizeof(uint64_t));
                    idx->codes = (uint8_t*)realloc(idx->codes, cap * idx->nsq);
                }
                if (!read_exact(f, &idx->ids[total], 8)) {
                    set_err("truncated or unreadable posting chunk_id at offset %llu",
                            (unsigned long long)offset);
                    goto fail;
                }
                offset += 8;
                if (!read_exact(f, idx->codes + total * idx->nsq, idx->nsq)) {
                    set_err("truncated posting code at offset %llu", (unsigned long long)offset);
                    goto fail;
                }
                offset += idx->nsq;
                ++total;
            }
            idx->list_off[l + 1] = total;
        }
        idx->ntotal = total;
    }
    fclose(f);
    *out = idx;
    return ORA_OK;
fail:
    fclose(f);
    ora_free_index(idx);
    return ORA_FORMAT;
}

/* ---- selection helpers ---- */
typedef struct {
    float dist;
    uint64_t id;
} scored;

static int scored_less(const scored* a, const scored* b) {
    /* annindex.hpp:55-58 */
    if (a->dist != b->dist) return a->dist < b->dist;
    return a->id < b->id;
}

static int scored_cmp(const void* pa, const void* pb) {
    const scored* a = (const scored*)pa;
    const scored* b = (const scored*)pb;
    if (scored_less(a, b)) return -1;
    if (scored_less(b, a)) return 1;
    return 0;
}

/* bounded max-heap of the k best (smallest) scored items */
typedef struct {
    scored* h;
    uint32_t n, k;
} topk_heap;

static void heap_push(topk_heap* t, scored s) {
    if (t->n < t->k) {
        uint32_t i = t->n++;
        t->h[i] = s;
        while (i > 0) {
            uint32_t p = (i - 1) / 2;
            if (scored_less(&t->h[p], &t->h[i])) {
                scored tmp = t->h[p];
                t->h[p] = t->h[i];
                t->h[i] = tmp;
                i = p;
            } else {
                break;
            }
        }
        return;
    }
    if (!scored_less(&s, &t->h[0])) return;
    t->h[0] = s;
    uint32_t i = 0;
    for (;;) {
        uint32_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < t->n && scored_less(&t->h[m], &t->h[l])) m = l;
        if (r < t->n && scored_less(&t->h[m], &t->h[r])) m = r;
        if (m == i) break;
        scored tmp = t->h[m];
        t->h[m] = t->h[i];
        t->h[i] = tmp;
        i = m;
    }
}

typedef struct {
    float dist;
    uint32_t list;
} list_pair;

static int list_pair_cmp(const void* pa, const void* pb) {
    /* std::pair<float, uint32_t> operator< as used by annindex.hpp:281 */
    const list_pair* a = (const list_pair*)pa;
    const list_pair* b = (const list_pair*)pb;
    if (a->dist < b->dist) return -1;
    if (b->dist < a->dist) return 1;
    return (a->list > b->list) - (a->list < b->list);
}

int ora_probe_lists(const ora_index* idx, const float* query, uint32_t nprobe, uint32_t* out_lists,
                    float* out_dist) {
    if (nprobe < 1 || nprobe > idx->nlist) {
        set_err("search: nprobe out of [1, nlist]");
        return ORA_CONFIG;
    }
    list_pair* order = (list_pair*)malloc(sizeof(list_pair) * idx->nlist);
    for (uint32_t c = 0; c < idx->nlist; ++c) {
        order[c].dist = ora_squared_l2(query, idx->centroids + (size_t)c * idx->d, idx->d);
        order[c].list = c;
    }
    qsort(order, idx->nlist, sizeof(list_pair), list_pair_cmp);
    for (uint32_t p = 0; p < nprobe; ++p) {
        out_lists[p] = order[p].list;
        if (out_dist) out_dist[p] = order[p].dist;
    }
    free(order);
    return ORA_OK;
}

/* annindex.hpp:262-315, exact_rerank = false. */
int ora_search(const ora_index* idx, const float* query, uint32_t nprobe, uint32_t k,
               uint64_t* out_ids, float* out_dist, uint32_t* out_count,
               uint64_t* out_scanned_vectors, uint32_t* out_scanned_lists) {
    if (k < 1) { /* :265 */
        set_err("search: k must be >= 1");
        return ORA_CONFIG;
    }
    if (nprobe < 1 || nprobe > idx->nlist) { /* :266-268 */
        set_err("search: nprobe out of [1, nlist]");
        return ORA_CONFIG;
    }
    const uint32_t d = idx->d, nsq = idx->nsq, sub_dim = idx->sub_dim;
    uint32_t* lists = (uint32_t*)malloc(sizeof(uint32_t) * nprobe);
    ora_probe_lists(idx, query, nprobe, lists, NULL); /* :277-281 */

    float* table = (float*)malloc(sizeof(float) * (size_t)nsq * 256 + 4);
    float* residual = (float*)malloc(sizeof(float) * d + 4);
    topk_heap heap = {(scored*)malloc(sizeof(scored) * k), 0, k};
    uint64_t scanned = 0;
    for (uint32_t p = 0; p < nprobe; ++p) { /* :287 */
        uint32_t list = lists[p];
        uint64_t b = idx->list_off[list], e = idx->list_off[list + 1];
        if (b == e) continue; /* :290 */
        const float* cen = idx->centroids + (size_t)list * d;
        for (uint32_t j = 0; j < d; ++j) residual[j] = query[j] - cen[j]; /* :292 */
        for (uint32_t sq = 0; sq < nsq; ++sq) {                             /* :293-299 */
            const float* sub = residual + (size_t)sq * sub_dim;
            const float* words = idx->codewords + (size_t)sq * 256 * sub_dim;
            for (uint32_t code = 0; code < 256; ++code)
                table[sq * 256 + code] = ora_squared_l2(sub, words + (size_t)code * sub_dim, sub_dim);
        }
        for (uint64_t i = b; i < e; ++i) { /* :300-304 */
            const uint8_t* code = idx->codes + i * nsq;
            float dist = 0.0f;
            for (uint32_t sq = 0; sq < nsq; ++sq) dist += table[sq * 256 + code[sq]];
            scored s = {dist, idx->ids[i]};
            heap_push(&heap, s);
        }
        scanned += e - b; /* :305 */
    }
    /* :313 sort_and_truncate */
    qsort(heap.h, heap.n, sizeof(scored), scored_cmp);
    for (uint32_t i = 0; i < heap.n; ++i) {
        out_ids[i] = heap.h[i].id;
        out_dist[i] = heap.h[i].dist;
    }
    *out_count = heap.n;
    if (out_scanned_vectors) *out_scanned_vectors = scanned;
    if (out_scanned_lists) *out_scanned_lists = nprobe; /* :284 */
    free(heap.h);
    free(residual);
    free(table);
    free(lists);
    return ORA_OK;
}

typedef struct {
    const ora_index* idx;
    const float* queries;
    uint32_t nq, nprobe, k;
    uint64_t* ids;
    float* dist;
    uint32_t* count;
    uint64_t* scanned;
    int next;
    pthread_mutex_t mu;
    int status;
} batch_ctx;

static void* batch_worker(void* arg) {
    batch_ctx* c = (batch_ctx*)arg;
    for (;;) {
        pthread_mutex_lock(&c->mu);
        int q = c->next++;
        pthread_mutex_unlock(&c->mu);
        if (q >= (int)c->nq) break;
        int rc = ora_search(c->idx, c->queries + (size_t)q * c->idx->d, c->nprobe, c->k,
                            c->ids + (size_t)q * c->k, c->dist + (size_t)q * c->k, c->count + q,
                            c->scanned ? c->scanned + q : NULL, NULL);
        if (rc) c->status = rc;
    }
    return NULL;
}

int ora_search_batch(const ora_index* idx, const float* queries, uint32_t nq, uint32_t nprobe,
                     uint32_t k, uint64_t* out_ids, float* out_dist, uint32_t* out_count,
                     uint64_t* out_scanned_vectors, int threads) {
    if (k < 1) {
        set_err("search: k must be >= 1");
        return ORA_CONFIG;
    }
    if (nprobe < 1 || nprobe > idx->nlist) {
        set_err("search: nprobe out of [1, nlist]");
        return ORA_CONFIG;
    }
    batch_ctx c = {idx, queries, nq, nprobe, k, out_ids, out_dist, out_count, out_scanned_vectors,
                   0, PTHREAD_MUTEX_INITIALIZER, 0};
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, batch_worker, &c);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    return c.status;
}

/* annindex.hpp:244-257 */
int ora_brute_force(const float* vecs, uint64_t n, uint32_t d, const float* query, uint32_t k,
                    uint64_t* out_ids, float* out_dist, uint32_t* out_count) {
    if (k < 1) {
        set_err("brute_force_search: k must be >= 1");
        return ORA_CONFIG;
    }
    topk_heap heap = {(scored*)malloc(sizeof(scored) * k), 0, k};
    for (uint64_t i = 0; i < n; ++i) {
        scored s = {ora_squared_l2(vecs + i * d, query, d), i};
        heap_push(&heap, s);
    }
    qsort(heap.h, heap.n, sizeof(scored), scored_cmp);
    for (uint32_t i = 0; i < heap.n; ++i) {
        out_ids[i] = heap.h[i].id;
        out_dist[i] = heap.h[i].dist;
    }
    *out_count = heap.n;
    free(heap.h);
    return ORA_OK;
}

/* Shard merge: the global top-k is the top-k of the union of per-shard
 * top-k lists, because each candidate's distance depends only on its own
 * (query, list, code). */
int ora_merge_topk(const uint64_t* ids, const float* dist, const uint32_t* count, uint32_t nparts,
                   uint32_t kin, uint32_t k, uint64_t* out_ids, float* out_dist, uint32_t* out_count) {
    topk_heap heap = {(scored*)malloc(sizeof(scored) * (k ? k : 1)), 0, k};
    for (uint32_t p = 0; p < nparts; ++p)
        for (uint32_t i = 0; i < count[p] && i < kin; ++i) {
            scored s = {dist[(size_t)p * kin + i], ids[(size_t)p * kin + i]};
            heap_push(&heap, s);
        }
    qsort(heap.h, heap.n, sizeof(scored), scored_cmp);
    for (uint32_t i = 0; i < heap.n; ++i) {
        out_ids[i] = heap.h[i].id;
        out_dist[i] = heap.h[i].dist;
    }
    *out_count = heap.n;
    free(heap.h);
    return ORA_OK;
}

/* ---- performance model: perfmodel.hpp:53-85, :148-157 ---- */
void ora_least_squares(const double* x, const double* y, size_t n, double* slope, double* intercept,
                       double* max_abs_residual, double* r_squared) {
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    for (size_t i = 0; i < n; ++i) {
        sx += x[i];
        sy += y[i];
        sxx += x[i] * x[i];
        sxy += x[i] * y[i];
    }
    double denom = n * sxx - sx * sx;
    double s = 0.0, b;
    if (denom == 0.0) {
        b = sy / n;
    } else {
        s = (n * sxy - sx * sy) / denom;
        b = (sy - s * sx) / n;
    }
    double ss_res = 0.0, ss_tot = 0.0, mean_y = sy / n, mar = 0.0;
    for (size_t i = 0; i < n; ++i) {
        double r = y[i] - (s * x[i] + b);
        if (fabs(r) > mar) mar = fabs(r);
        ss_res += r * r;
        ss_tot += (y[i] - mean_y) * (y[i] - mean_y);
    }
    *slope = s;
    *intercept = b;
    if (max_abs_residual) *max_abs_residual = mar;
    if (r_squared) *r_squared = ss_tot > 0.0 ? 1.0 - ss_res / ss_tot : 1.0;
}

static int dbl_cmp(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

double ora_median(const double* v, size_t n) {
    double* c = (double*)malloc(sizeof(double) * (n ? n : 1));
    memcpy(c, v, sizeof(double) * n);
    qsort(c, n, sizeof(double), dbl_cmp);
    double m = n % 2 ? c[n / 2] : 0.5 * (c[n / 2 - 1] + c[n / 2]);
    free(c);
    return m;
}

uint32_t ora_select_nprobe(double slope_s, double intercept_s, double budget_s, uint32_t nlist,
                           double safety_margin) {
    if (budget_s <= 0.0) return 1;
    double limit = budget_s * (1.0 - safety_margin);
    if (slope_s * 1 + intercept_s > limit) return 1;
    if (slope_s <= 0.0) return nlist;
    double max_n = (limit - intercept_s) / slope_s;
    if (max_n >= (double)nlist) return nlist;
    double f = floor(max_n + 1e-9);
    return (uint32_t)(f > 1.0 ? f : 1.0);
}

/* ------------------------------------------------------------------ build
 * prag::train_index (annindex.hpp:164-241) and its kmeans
 * (annindex.hpp:62-130), restated over flat arrays. Outputs the flattened
 * IvfIndex/PqCodebook (list-major, each list in vector order). */

/* annindex.hpp:64-130: k-means++ seeding then Lloyd; pts[i] points at a row
 * of `dim` floats; centroids out [k][dim]. */
static int ora_kmeans(const float* const* pts, uint64_t n, uint32_t dim, uint32_t k, uint64_t seed, int iters,
                      float* cent) {
    if (n < k) {
        set_err("kmeans: fewer points than clusters");
        return ORA_CONFIG;
    }
    uint64_t st = seed;
    float* md = malloc(n * sizeof(float));
    for (uint64_t i = 0; i < n; ++i) md[i] = 3.402823466e+38f; /* FLT_MAX */
    uint64_t first = ora_splitmix_next(&st) % n;
    memcpy(cent, pts[first], dim * sizeof(float));
    for (uint32_t t = 1; t < k; ++t) {
        const float* last = cent + (size_t)(t - 1) * dim;
        double total = 0.0;
        for (uint64_t i = 0; i < n; ++i) {
            float dsq = ora_squared_l2(pts[i], last, dim);
            if (dsq < md[i]) md[i] = dsq;
            total += md[i];
        }
        uint64_t pick = 0;
        if (total > 0.0) {
            double r = splitmix_double(&st) * total;
            double acc = 0.0;
            for (uint64_t i = 0; i < n; ++i) {
                acc += md[i];
                if (acc >= r) {
                    pick = i;
                    break;
                }
            }
        } else {
            pick = ora_splitmix_next(&st) % n;
        }
        memcpy(cent + (size_t)t * dim, pts[pick], dim * sizeof(float));
    }
    free(md);
    uint32_t* asg = calloc(n, sizeof(uint32_t));
    float* adist = calloc(n, sizeof(float));
    double* sums = malloc((size_t)k * dim * sizeof(double));
    uint64_t* cnt = malloc((size_t)k * sizeof(uint64_t));
    for (int it = 0; it < iters; ++it) {
        for (uint64_t i = 0; i < n; ++i) {
            float best = 3.402823466e+38f;
            uint32_t bc = 0;
            for (uint32_t c = 0; c < k; ++c) {
                float dsq = ora_squared_l2(pts[i], cent + (size_t)c * dim, dim);
                if (dsq < best) {
                    best = dsq;
                    bc = c;
                }
            }
            asg[i] = bc;
            adist[i] = best;
        }
        memset(sums, 0, (size_t)k * dim * sizeof(double));
        memset(cnt, 0, (size_t)k * sizeof(uint64_t));
        for (uint64_t i = 0; i < n; ++i) {
            ++cnt[asg[i]];
            double* s = sums + (size_t)asg[i] * dim;
            for (uint32_t j = 0; j < dim; ++j) s[j] += pts[i][j];
        }
        for (uint32_t c = 0; c < k; ++c) {
            float* dst = cent + (size_t)c * dim;
            if (cnt[c] == 0) {
                uint64_t far = 0;
                float far_d = -1.0f;
                for (uint64_t i = 0; i < n; ++i)
                    if (adist[i] > far_d) {
                        far_d = adist[i];
                        far = i;
                    }
                memcpy(dst, pts[far], dim * sizeof(float));
                adist[far] = 0.0f;
            } else {
                for (uint32_t j = 0; j < dim; ++j) dst[j] = (float)(sums[(size_t)c * dim + j] / (double)cnt[c]);
            }
        }
    }
    free(asg);
    free(adist);
    free(sums);
    free(cnt);
    return ORA_OK;
}

int ora_train_index(const float* vecs, uint64_t n, uint32_t d, uint32_t nlist, uint32_t n_subquantizers,
                    uint64_t seed, int iters, uint64_t sample_cap, float* centroids, float* codewords,
                    uint64_t* list_off, uint64_t* ids, uint8_t* codes) {
    if (n == 0) {
        set_err("train_index: empty embedding set");
        return ORA_CONFIG;
    }
    if (n < nlist) {
        set_err("train_index: nlist exceeds number of vectors");
        return ORA_CONFIG;
    }
    uint32_t nsq = n_subquantizers ? n_subquantizers : (d / 4 > 1 ? d / 4 : 1);
    if (d % nsq != 0) {
        set_err("train_index: d not divisible by n_subquantizers");
        return ORA_CONFIG;
    }
    uint32_t sub = d / nsq;
    /* training_sample (annindex.hpp:134-145) */
    uint64_t* idx = malloc(n * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) idx[i] = i;
    uint64_t ns = n;
    if (n > sample_cap) {
        uint64_t st = seed ^ 0x5a5a;
        for (uint64_t i = 0; i < sample_cap; ++i) {
            uint64_t j = i + ora_splitmix_next(&st) % (n - i);
            uint64_t t = idx[i];
            idx[i] = idx[j];
            idx[j] = t;
        }
        ns = sample_cap;
    }
    const float** sp = malloc((ns ? ns : 1) * sizeof(float*));
    for (uint64_t i = 0; i < ns; ++i) sp[i] = vecs + idx[i] * d;
    int rc = ora_kmeans(sp, ns, d, nlist, seed, iters, centroids);
    if (rc) {
        free(idx);
        free(sp);
        return rc;
    }
    /* assignment + residuals (annindex.hpp:195-202) */
    uint32_t* asg = malloc(n * sizeof(uint32_t));
    float* res = malloc(n * d * sizeof(float));
    for (uint64_t i = 0; i < n; ++i) {
        const float* v = vecs + i * d;
        float best = 3.402823466e+38f;
        uint32_t bc = 0;
        for (uint32_t c = 0; c < nlist; ++c) {
            float dsq = ora_squared_l2(v, centroids + (size_t)c * d, d);
            if (dsq < best) {
                best = dsq;
                bc = c;
            }
        }
        asg[i] = bc;
        for (uint32_t j = 0; j < d; ++j) res[i * d + j] = v[j] - centroids[(size_t)bc * d + j];
    }
    /* PQ codebooks (annindex.hpp:209-218) */
    uint64_t pq = n < 256 ? n : 256;
    uint64_t clusters = pq < ns ? pq : ns;
    memset(codewords, 0, (size_t)nsq * 256 * sub * sizeof(float));
    for (uint32_t q = 0; q < nsq; ++q) {
        for (uint64_t i = 0; i < ns; ++i) sp[i] = res + idx[i] * d + (size_t)q * sub;
        rc = ora_kmeans(sp, ns, sub, (uint32_t)clusters, ora_hash_combine(seed, q + 1), iters,
                        codewords + (size_t)q * 256 * sub);
        if (rc) break;
    }
    if (!rc) {
        /* postings in vector order (annindex.hpp:222-238) */
        memset(list_off, 0, (nlist + 1) * sizeof(uint64_t));
        for (uint64_t i = 0; i < n; ++i) ++list_off[asg[i] + 1];
        for (uint32_t l = 0; l < nlist; ++l) list_off[l + 1] += list_off[l];
        uint64_t* fill = malloc((nlist + 1) * sizeof(uint64_t));
        memcpy(fill, list_off, (nlist + 1) * sizeof(uint64_t));
        for (uint64_t i = 0; i < n; ++i) {
            uint64_t at = fill[asg[i]]++;
            ids[at] = i;
            for (uint32_t q = 0; q < nsq; ++q) {
                const float* s = res + i * d + (size_t)q * sub;
                float best = 3.402823466e+38f;
                uint32_t bc = 0;
                for (uint32_t c = 0; c < pq; ++c) {
                    float dsq = ora_squared_l2(s, codewords + ((size_t)q * 256 + c) * sub, sub);
                    if (dsq < best) {
                        best = dsq;
                        bc = c;
                    }
                }
                codes[at * nsq + q] = (uint8_t)bc;
            }
        }
        free(fill);
    }
    free(idx);
    free(sp);
    free(asg);
    free(res);
    return rc;
}
