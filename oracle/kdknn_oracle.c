/*
 * kdknn_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * CPU restatement, in plain C, of the reference `kdknn` package's hot path:
 * the per-rank kd-tree build (pkg/src/kdknn/local_tree.py + median.py) and the
 * exact KNN traversal (pkg/src/kdknn/local_query.py), plus the brute-force
 * top-k oracle of pkg/tests/conftest.py:8-18.  Every function cites the
 * reference file:line it follows.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 *
 * Parity pin: the fixtures under tests/golden/ were produced by importing the real reference
 * (tests/golden/make_golden.py); tests/test_oracle_golden.py checks this file
 * against them byte for byte (tree arrays, packed ids/coords, KNN outputs).
 *
 * Arithmetic contract: binary64, no FMA contraction (compile with
 * -ffp-contract=off), ascending-dimension accumulation -- identical to the
 * numba kernels (fastmath off) of the reference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GAMMA 0x9E3779B97F4A7C15ULL
#define SALT_VARIANCE 0ULL     /* local_tree.py:44 */
#define SALT_MEDIAN_BASE 1ULL  /* local_tree.py:45 */
#define PAR_NODE_MIN (1 << 17) /* nodes this big use threaded histogram/partition */

/* ------------------------------------------------------------------ RNG --- */
/* median.py:51-56 _mix64 (SplitMix64 finaliser) */
static inline uint64_t mix64(uint64_t z) {
    z = z + GAMMA;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* median.py:59-66 _rng_next */
static inline uint64_t rng_next(uint64_t *state) {
    *state = *state + GAMMA;
    uint64_t z = *state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* median.py:69-71 _node_seed */
uint64_t kdo_node_seed(uint64_t seed, uint64_t path, uint64_t salt) {
    return mix64(seed ^ mix64(path) ^ mix64(salt * GAMMA));
}

/* ------------------------------------------------- Fisher-Yates sampling --- */
/* median.py:74-85 _sample_indices: m distinct indices of [0,n) by a partial
 * Fisher-Yates over arange(n).  The reference materialises arange(n); this
 * restatement keeps only the touched slots in an open-addressed map, which
 * yields the identical draw (step j swaps slots j and r = j + z mod (n-j);
 * slot j is final after step j). */
typedef struct { int64_t *keys; int64_t *vals; int64_t cap; } fy_map;

static void fy_map_init(fy_map *h, int64_t m) {
    int64_t cap = 16;
    while (cap < 4 * m + 16) cap <<= 1;
    h->cap = cap;
    h->keys = (int64_t *)malloc(sizeof(int64_t) * cap);
    h->vals = (int64_t *)malloc(sizeof(int64_t) * cap);
    for (int64_t i = 0; i < cap; i++) h->keys[i] = -1;
}
static void fy_map_free(fy_map *h) { free(h->keys); free(h->vals); }
static inline int64_t fy_slot(const fy_map *h, int64_t key) {
    uint64_t s = mix64((uint64_t)key) & (uint64_t)(h->cap - 1);
    while (h->keys[s] != -1 && h->keys[s] != key) s = (s + 1) & (uint64_t)(h->cap - 1);
    return (int64_t)s;
}
static inline int64_t fy_get(const fy_map *h, int64_t key) {
    int64_t s = fy_slot(h, key);
    return h->keys[s] == -1 ? key : h->vals[s];
}
static inline void fy_set(fy_map *h, int64_t key, int64_t v) {
    int64_t s = fy_slot(h, key);
    h->keys[s] = key;
    h->vals[s] = v;
}

void kdo_sample_indices(int64_t n, int64_t m, uint64_t seed, int64_t *out) {
    fy_map h;
    fy_map_init(&h, m);
    uint64_t state = seed;
    for (int64_t j = 0; j < m; j++) {
        uint64_t z = rng_next(&state);
        int64_t r = j + (int64_t)(z % (uint64_t)(n - j));
        int64_t vj = fy_get(&h, j), vr = fy_get(&h, r);
        fy_set(&h, j, vr);
        fy_set(&h, r, vj);
        out[j] = vr;
    }
    fy_map_free(&h);
}

/* ------------------------------------------------------- histogram/select --- */
/* median.py:99-117 _locate == number of boundaries <= v (searchsorted right;
 * equivalence pinned by reference tests/test_median.py:89-108). */
static inline int64_t locate(const double *b, int64_t nb, double v) {
    int64_t lo = 0, hi = nb;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (b[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* median.py:128-140 _histogram (counts[nb+1], equals[nb]) */
void kdo_histogram(const double *values, int64_t n, const double *b, int64_t nb,
                   int64_t *counts, int64_t *equals) {
    memset(counts, 0, sizeof(int64_t) * (nb + 1));
    if (equals) memset(equals, 0, sizeof(int64_t) * nb);
    for (int64_t i = 0; i < n; i++) {
        int64_t k = locate(b, nb, values[i]);
        counts[k]++;
        if (equals && k > 0 && b[k - 1] == values[i]) equals[k - 1]++;
    }
}

/* median.py:143-166 _select_median: closest cumulative fraction to 0.5 in
 * binary64, strict < so ties go to the lower boundary. */
int64_t kdo_select_median(int64_t nb, const int64_t *counts, int64_t *below_out) {
    int64_t total = 0;
    for (int64_t b = 0; b <= nb; b++) total += counts[b];
    *below_out = 0;
    if (total <= 0 || nb == 0) return -1;
    int64_t best = -1, cum = 0, best_below = 0;
    double best_diff = INFINITY;
    for (int64_t i = 0; i < nb; i++) {
        cum += counts[i];
        double diff = fabs((double)cum / (double)total - 0.5);
        if (diff < best_diff) { best_diff = diff; best = i; best_below = cum; }
    }
    *below_out = best_below;
    return best;
}

static int cmp_double(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

/* np.unique (sort + keep first of each run of equal values) */
static int64_t unique_sorted(double *v, int64_t n) {
    if (n == 0) return 0;
    qsort(v, (size_t)n, sizeof(double), cmp_double);
    int64_t w = 1;
    for (int64_t i = 1; i < n; i++)
        if (v[i] != v[w - 1]) v[w++] = v[i];
    return w;
}

/* ------------------------------------------------------------ tree build --- */
typedef struct {
    const double *coords; /* (D, N) row-major: coords[d*N + i] */
    int64_t N;
    int D;
    int64_t *idx;
    int64_t *scratch;
    uint64_t seed;
    int64_t bucket, vsample, msample;
} build_ctx;

/* local_tree.py:111-132 _dim_ssd: sequential f64 mean / sum of squared devs
 * over the Fisher-Yates variance sample, in draw order. */
static void dim_ssd(const build_ctx *c, int64_t start, int64_t end, uint64_t seed, double *ssd) {
    int64_t n = end - start;
    int64_t take = c->vsample < n ? c->vsample : n;
    int64_t *picked = (int64_t *)malloc(sizeof(int64_t) * take);
    kdo_sample_indices(n, take, seed, picked);
    for (int d = 0; d < c->D; d++) {
        const double *row = c->coords + (int64_t)d * c->N;
        double mean = 0.0;
        for (int64_t j = 0; j < take; j++) mean += row[c->idx[start + picked[j]]];
        mean /= (double)take;
        double s = 0.0;
        for (int64_t j = 0; j < take; j++) {
            double diff = row[c->idx[start + picked[j]]] - mean;
            s += diff * diff;
        }
        ssd[d] = s;
    }
    free(picked);
}

static void histogram_par(const double *values, int64_t n, const double *b, int64_t nb,
                          int64_t *counts) {
    memset(counts, 0, sizeof(int64_t) * (nb + 1));
#ifdef _OPENMP
    if (n >= PAR_NODE_MIN && !omp_in_parallel() && omp_get_max_threads() > 1) {
#pragma omp parallel
        {
            int64_t *loc = (int64_t *)calloc((size_t)(nb + 1), sizeof(int64_t));
#pragma omp for schedule(static)
            for (int64_t i = 0; i < n; i++) loc[locate(b, nb, values[i])]++;
#pragma omp critical
            for (int64_t k = 0; k <= nb; k++) counts[k] += loc[k];
            free(loc);
        }
        return;
    }
#endif
    for (int64_t i = 0; i < n; i++) counts[locate(b, nb, values[i])]++;
}

/* local_tree.py:135-180 _choose_split.  Returns 0 (valid split) or 1
 * (degenerate leaf: every dimension constant over the node). */
static int choose_split(const build_ctx *c, int64_t start, int64_t end, uint64_t path,
                        int *dim_out, double *val_out) {
    int64_t n = end - start;
    int D = c->D;
    double ssd[64];
    int order[64];
    dim_ssd(c, start, end, kdo_node_seed(c->seed, path, SALT_VARIANCE), ssd);
    /* np.argsort(-ssd, kind="mergesort"): stable, descending variance */
    for (int d = 0; d < D; d++) order[d] = d;
    for (int a = 1; a < D; a++) {
        int t = order[a], p = a - 1;
        while (p >= 0 && -ssd[order[p]] > -ssd[t]) { order[p + 1] = order[p]; p--; }
        order[p + 1] = t;
    }
    double *values = (double *)malloc(sizeof(double) * n);
    int64_t m = c->msample < n ? c->msample : n;
    int64_t *picked = (int64_t *)malloc(sizeof(int64_t) * m);
    double *bnd = (double *)malloc(sizeof(double) * m);
    int64_t *counts = (int64_t *)malloc(sizeof(int64_t) * (m + 1));
    int status = 1;
    for (int t = 0; t < D; t++) {
        int d = order[t];
        const double *row = c->coords + (int64_t)d * c->N;
        for (int64_t i = 0; i < n; i++) values[i] = row[c->idx[start + i]];
        /* median.py:88-96 _sample_from + np.unique + _histogram + _select_median */
        kdo_sample_indices(n, m, kdo_node_seed(c->seed, path, SALT_MEDIAN_BASE + (uint64_t)d), picked);
        for (int64_t j = 0; j < m; j++) bnd[j] = values[picked[j]];
        int64_t nb = unique_sorted(bnd, m);
        histogram_par(values, n, bnd, nb, counts);
        int64_t below;
        int64_t bi = kdo_select_median(nb, counts, &below);
        if (bi >= 0 && 0 < below && below < n) {
            *dim_out = d; *val_out = bnd[bi]; status = 0; break;
        }
        /* local_tree.py:162-177 exact fallback: distinct value whose
         * below-count is closest to n/2 (minimum value excluded) */
        qsort(values, (size_t)n, sizeof(double), cmp_double);
        double half = (double)n * 0.5, best_diff = 0.0, best_val = 0.0;
        int found = 0;
        for (int64_t i = 1; i < n; i++) {
            if (values[i] != values[i - 1]) {
                double diff = fabs((double)i - half);
                if (!found || diff < best_diff) { found = 1; best_diff = diff; best_val = values[i]; }
            }
        }
        if (found) { *dim_out = d; *val_out = best_val; status = 0; break; }
    }
    free(values); free(picked); free(bnd); free(counts);
    return status;
}

/* local_tree.py:183-206 _partition_stable (coord < value first, ties right) */
static int64_t partition_stable(const build_ctx *c, int64_t start, int64_t end, int dim,
                                double value, int64_t *scratch) {
    const double *row = c->coords + (int64_t)dim * c->N;
    int64_t *idx = c->idx;
    int64_t n = end - start;
#ifdef _OPENMP
    if (n >= PAR_NODE_MIN && !omp_in_parallel() && omp_get_max_threads() > 1) {
        /* local_tree.py:408-433 chunked count/scatter/copy: same stable result */
        int maxt = omp_get_max_threads();
        int64_t *lc = (int64_t *)calloc((size_t)maxt + 1, sizeof(int64_t));
        int64_t nl_total = 0;
#pragma omp parallel num_threads(maxt)
        {
            int nth = omp_get_num_threads();
            int t = omp_get_thread_num();
            int64_t chunk = (n + nth - 1) / nth;
            int64_t lo = start + (int64_t)t * chunk, hi = lo + chunk;
            if (lo > end) lo = end;
            if (hi > end) hi = end;
            int64_t cnt = 0;
            for (int64_t i = lo; i < hi; i++) cnt += row[idx[i]] < value;
            lc[t + 1] = cnt;
#pragma omp barrier
#pragma omp single
            {
                for (int k = 1; k <= nth; k++) lc[k] += lc[k - 1];
                nl_total = lc[nth];
            }
            int64_t lp = lc[t], rp = nl_total + (lo - start) - lc[t];
            for (int64_t i = lo; i < hi; i++) {
                int64_t j = idx[i];
                if (row[j] < value) scratch[lp++] = j; else scratch[rp++] = j;
            }
#pragma omp barrier
            for (int64_t i = lo; i < hi; i++) idx[i] = scratch[i - start];
        }
        free(lc);
        return nl_total;
    }
#endif
    int64_t nl = 0;
    for (int64_t i = start; i < end; i++) nl += row[idx[i]] < value;
    int64_t li = 0, ri = nl;
    for (int64_t i = start; i < end; i++) {
        int64_t j = idx[i];
        if (row[j] < value) scratch[li++] = j; else scratch[ri++] = j;
    }
    memcpy(idx + start, scratch, sizeof(int64_t) * n);
    return nl;
}

/* Linked node store (children by index), renumbered to preorder at the end
 * exactly like local_tree.py:320-374 _renumber_preorder. */
typedef struct {
    int32_t *dim; double *val; int64_t *left; int64_t *right; int64_t *count;
    int64_t used, cap;
} nodes_t;

static void nodes_init(nodes_t *s, int64_t cap) {
    s->cap = cap > 1 ? cap : 1;
    s->used = 0;
    s->dim = (int32_t *)malloc(sizeof(int32_t) * s->cap);
    s->val = (double *)malloc(sizeof(double) * s->cap);
    s->left = (int64_t *)malloc(sizeof(int64_t) * s->cap);
    s->right = (int64_t *)malloc(sizeof(int64_t) * s->cap);
    s->count = (int64_t *)malloc(sizeof(int64_t) * s->cap);
}
static void nodes_free(nodes_t *s) { free(s->dim); free(s->val); free(s->left); free(s->right); free(s->count); }

/* local_tree.py:236-317 _build_subtree (DFS, left child numbered first) */
static void build_dfs(const build_ctx *c, nodes_t *s, int64_t slot, int64_t start, int64_t end,
                      uint64_t path, int64_t *scratch) {
    int64_t n = end - start;
    s->count[slot] = n;
    int dim = -1;
    double value = 0.0;
    int leaf = n <= c->bucket;
    if (!leaf && choose_split(c, start, end, path, &dim, &value) == 1) leaf = 1;
    if (leaf) {
        s->dim[slot] = -1; s->val[slot] = 0.0; s->left[slot] = start; s->right[slot] = n;
        return;
    }
    int64_t nl = partition_stable(c, start, end, dim, value, scratch);
    s->dim[slot] = dim; s->val[slot] = value;
    int64_t ls = s->used++, rs = s->used++;
    s->left[slot] = ls; s->right[slot] = rs;
    build_dfs(c, s, ls, start, start + nl, path * 2ULL, scratch);
    build_dfs(c, s, rs, start + nl, end, path * 2ULL + 1ULL, scratch);
}

typedef struct {
    int32_t *node_dim; double *node_value; int32_t *node_left; int32_t *node_right;
    int64_t *node_count; int64_t *perm; int64_t n_nodes; int64_t depth; int64_t n;
} kdo_tree;

/* preorder renumbering + depth (local_tree.py:320-374) */
static void renumber(const nodes_t *s, kdo_tree *t) {
    int64_t nn = s->used;
    t->n_nodes = nn;
    t->node_dim = (int32_t *)malloc(sizeof(int32_t) * (nn ? nn : 1));
    t->node_value = (double *)malloc(sizeof(double) * (nn ? nn : 1));
    t->node_left = (int32_t *)malloc(sizeof(int32_t) * (nn ? nn : 1));
    t->node_right = (int32_t *)malloc(sizeof(int32_t) * (nn ? nn : 1));
    t->node_count = (int64_t *)malloc(sizeof(int64_t) * (nn ? nn : 1));
    t->depth = 0;
    if (!nn) return;
    int64_t *st_old = (int64_t *)malloc(sizeof(int64_t) * (nn + 1));
    int64_t *st_par = (int64_t *)malloc(sizeof(int64_t) * (nn + 1));
    int8_t *st_left = (int8_t *)malloc(nn + 1);
    int64_t *st_dep = (int64_t *)malloc(sizeof(int64_t) * (nn + 1));
    int64_t sp = 0, cursor = 0;
    st_old[0] = 0; st_par[0] = -1; st_left[0] = 0; st_dep[0] = 0; sp = 1;
    while (sp > 0) {
        sp--;
        int64_t old = st_old[sp], par = st_par[sp], d = st_dep[sp];
        int isl = st_left[sp];
        int64_t nw = cursor++;
        if (par >= 0) { if (isl) t->node_left[par] = (int32_t)nw; else t->node_right[par] = (int32_t)nw; }
        if (d > t->depth) t->depth = d;
        t->node_dim[nw] = s->dim[old];
        t->node_value[nw] = s->val[old];
        t->node_count[nw] = s->count[old];
        if (s->dim[old] < 0) {
            t->node_left[nw] = (int32_t)s->left[old];
            t->node_right[nw] = (int32_t)s->right[old];
        } else {
            st_old[sp] = s->right[old]; st_par[sp] = nw; st_left[sp] = 0; st_dep[sp] = d + 1; sp++;
            st_old[sp] = s->left[old]; st_par[sp] = nw; st_left[sp] = 1; st_dep[sp] = d + 1; sp++;
        }
    }
    free(st_old); free(st_par); free(st_left); free(st_dep);
}

typedef struct { int64_t start, end; uint64_t path; int64_t slot; } task_t;

/* local_tree.py:436-574 build_local_tree.  Breadth-first over the top levels
 * (threaded histogram/partition inside big nodes), then one depth-first task
 * per frontier subtree; the preorder result does not depend on nthreads. */
kdo_tree *kdo_build(const double *coords, int64_t n, int D, int64_t bucket, int64_t local_sample_m,
                    int64_t variance_sample, uint64_t seed, int nthreads) {
    if (D < 1 || D > 64) return NULL;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
    int nt = omp_get_max_threads();
#else
    int nt = 1;
    (void)nthreads;
#endif
    kdo_tree *t = (kdo_tree *)calloc(1, sizeof(kdo_tree));
    t->n = n;
    t->perm = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t i = 0; i < n; i++) t->perm[i] = i;
    if (n == 0) { nodes_t s; nodes_init(&s, 1); renumber(&s, t); nodes_free(&s); return t; }
    build_ctx c = {coords, n, D, t->perm, NULL, seed, bucket, variance_sample, local_sample_m};
    int64_t *scratch = (int64_t *)malloc(sizeof(int64_t) * n);
    c.scratch = scratch;

    nodes_t top;
    nodes_init(&top, 1024);
    int64_t threshold = (int64_t)nt * 10;
    task_t *front = (task_t *)malloc(sizeof(task_t));
    int64_t nf = 1;
    front[0].start = 0; front[0].end = n; front[0].path = 1; front[0].slot = 0;
    top.used = 1;
    while (nf > 0 && nf < threshold && nt > 1) {
        task_t *next = (task_t *)malloc(sizeof(task_t) * 2 * nf);
        int64_t nn = 0;
        for (int64_t f = 0; f < nf; f++) {
            task_t tk = front[f];
            if (top.used + 2 > top.cap) {
                top.cap *= 2;
                top.dim = realloc(top.dim, sizeof(int32_t) * top.cap);
                top.val = realloc(top.val, sizeof(double) * top.cap);
                top.left = realloc(top.left, sizeof(int64_t) * top.cap);
                top.right = realloc(top.right, sizeof(int64_t) * top.cap);
                top.count = realloc(top.count, sizeof(int64_t) * top.cap);
            }
            int64_t sz = tk.end - tk.start;
            top.count[tk.slot] = sz;
            int dim = -1; double value = 0.0;
            int leaf = sz <= bucket;
            if (!leaf && choose_split(&c, tk.start, tk.end, tk.path, &dim, &value) == 1) leaf = 1;
            if (leaf) {
                top.dim[tk.slot] = -1; top.val[tk.slot] = 0.0;
                top.left[tk.slot] = tk.start; top.right[tk.slot] = sz;
                continue;
            }
            int64_t nl = partition_stable(&c, tk.start, tk.end, dim, value, scratch);
            top.dim[tk.slot] = dim; top.val[tk.slot] = value;
            int64_t ls = top.used++, rs = top.used++;
            top.left[tk.slot] = ls; top.right[tk.slot] = rs;
            next[nn].start = tk.start; next[nn].end = tk.start + nl; next[nn].path = tk.path * 2ULL; next[nn].slot = ls; nn++;
            next[nn].start = tk.start + nl; next[nn].end = tk.end; next[nn].path = tk.path * 2ULL + 1ULL; next[nn].slot = rs; nn++;
        }
        free(front);
        front = next;
        nf = nn;
    }
    /* depth-first tasks, each into a private store */
    nodes_t *sub = (nodes_t *)calloc((size_t)(nf ? nf : 1), sizeof(nodes_t));
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t f = 0; f < nf; f++) {
        int64_t sz = front[f].end - front[f].start;
        nodes_init(&sub[f], 2 * sz + 1);
        sub[f].used = 1;
        build_dfs(&c, &sub[f], 0, front[f].start, front[f].end, front[f].path, scratch + front[f].start);
    }
    /* stitch: frontier slot f is replaced by task f's root (local_tree.py:530-560) */
    int64_t total = top.used;
    for (int64_t f = 0; f < nf; f++) total += sub[f].used - 1;
    nodes_t all;
    nodes_init(&all, total);
    all.used = total;
    memcpy(all.dim, top.dim, sizeof(int32_t) * top.used);
    memcpy(all.val, top.val, sizeof(double) * top.used);
    memcpy(all.left, top.left, sizeof(int64_t) * top.used);
    memcpy(all.right, top.right, sizeof(int64_t) * top.used);
    memcpy(all.count, top.count, sizeof(int64_t) * top.used);
    int64_t off = top.used;
    for (int64_t f = 0; f < nf; f++) {
        nodes_t *s = &sub[f];
        /* local slot 0 -> frontier slot; local slot i>0 -> off + i - 1 */
        for (int64_t i = 0; i < s->used; i++) {
            int64_t g = i == 0 ? front[f].slot : off + i - 1;
            all.dim[g] = s->dim[i]; all.val[g] = s->val[i]; all.count[g] = s->count[i];
            if (s->dim[i] >= 0) {
                all.left[g] = s->left[i] == 0 ? front[f].slot : off + s->left[i] - 1;
                all.right[g] = s->right[i] == 0 ? front[f].slot : off + s->right[i] - 1;
            } else {
                all.left[g] = s->left[i]; all.right[g] = s->right[i];
            }
        }
        off += s->used - 1;
        nodes_free(s);
    }
    free(sub); free(front); nodes_free(&top);
    renumber(&all, t);
    nodes_free(&all);
    free(scratch);
    return t;
}

int64_t kdo_tree_n_nodes(const kdo_tree *t) { return t->n_nodes; }
int64_t kdo_tree_depth(const kdo_tree *t) { return t->depth; }

/* copy out: node arrays + the bucket permutation (pack_buckets order,
 * local_tree.py:402-405) */
void kdo_tree_export(const kdo_tree *t, int32_t *dim, double *val, int32_t *left, int32_t *right,
                     int64_t *count, int64_t *perm) {
    memcpy(dim, t->node_dim, sizeof(int32_t) * t->n_nodes);
    memcpy(val, t->node_value, sizeof(double) * t->n_nodes);
    memcpy(left, t->node_left, sizeof(int32_t) * t->n_nodes);
    memcpy(right, t->node_right, sizeof(int32_t) * t->n_nodes);
    memcpy(count, t->node_count, sizeof(int64_t) * t->n_nodes);
    memcpy(perm, t->perm, sizeof(int64_t) * t->n);
}

void kdo_tree_free(kdo_tree *t) {
    if (!t) return;
    free(t->node_dim); free(t->node_value); free(t->node_left); free(t->node_right);
    free(t->node_count); free(t->perm); free(t);
}

/* ----------------------------------------------------------- KNN query --- */
/* local_query.py:36-49 _heap_push (max-heap on lexicographic (d, id)) */
static inline int64_t heap_push(double *hd, uint64_t *hid, int64_t hsize, double d, uint64_t pid) {
    int64_t i = hsize;
    hd[i] = d; hid[i] = pid;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (hd[p] < hd[i] || (hd[p] == hd[i] && hid[p] < hid[i])) {
            double td = hd[p]; hd[p] = hd[i]; hd[i] = td;
            uint64_t ti = hid[p]; hid[p] = hid[i]; hid[i] = ti;
            i = p;
        } else break;
    }
    return hsize + 1;
}

/* local_query.py:52-69 _heap_replace_root */
static inline void heap_replace_root(double *hd, uint64_t *hid, int64_t hsize, double d, uint64_t pid) {
    hd[0] = d; hid[0] = pid;
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, big = i;
        if (l < hsize && (hd[l] > hd[big] || (hd[l] == hd[big] && hid[l] > hid[big]))) big = l;
        if (r < hsize && (hd[r] > hd[big] || (hd[r] == hd[big] && hid[r] > hid[big]))) big = r;
        if (big == i) break;
        double td = hd[big]; hd[big] = hd[i]; hd[i] = td;
        uint64_t ti = hid[big]; hid[big] = hid[i]; hid[i] = ti;
        i = big;
    }
}

/* local_query.py:72-172 _knn_kernel (Algorithm 1): explicit stack, prune
 * `bound >= r'`, far bound = bound - old_off^2 + new_off^2, near child
 * pushed last; leaves are never bound-checked.  coords is the packed (D, n)
 * array, queries (nq, D) row-major. */
void kdo_knn(const int32_t *node_dim, const double *node_value, const int32_t *node_left,
             const int32_t *node_right, int64_t n_nodes, const double *coords, int64_t n,
             const uint64_t *ids, int D, int64_t depth, const double *queries, int64_t nq,
             int64_t k, const double *radii, double *out_d, uint64_t *out_ids, int64_t *out_counts,
             int64_t *out_counters, int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    int64_t cap = depth + 2;
#pragma omp parallel
    {
        int64_t *st_node = (int64_t *)malloc(sizeof(int64_t) * cap);
        double *st_bound = (double *)malloc(sizeof(double) * cap);
        double *st_off = (double *)malloc(sizeof(double) * cap * D);
        double *cur = (double *)malloc(sizeof(double) * D);
        double *hd = (double *)malloc(sizeof(double) * k);
        uint64_t *hid = (uint64_t *)malloc(sizeof(uint64_t) * k);
#pragma omp for schedule(dynamic, 512)
        for (int64_t qi = 0; qi < nq; qi++) {
            int64_t c0 = 0, c1 = 0, c2 = 0;
            if (n_nodes == 0) {
                out_counts[qi] = 0;
                if (out_counters) { out_counters[qi * 3] = 0; out_counters[qi * 3 + 1] = 0; out_counters[qi * 3 + 2] = 0; }
                continue;
            }
            const double *q = queries + qi * D;
            double r_prime = radii[qi];
            int64_t hsize = 0, sp = 0;
            st_node[0] = 0; st_bound[0] = 0.0;
            for (int d = 0; d < D; d++) st_off[d] = 0.0;
            sp = 1;
            while (sp > 0) {
                sp--;
                int64_t node = st_node[sp];
                double bound = st_bound[sp];
                for (int d = 0; d < D; d++) cur[d] = st_off[sp * D + d];
                c0++;
                int dim = node_dim[node];
                if (dim < 0) {
                    int64_t start = node_left[node], len = node_right[node];
                    c1++; c2 += len;
                    for (int64_t i = start; i < start + len; i++) {
                        double dist = 0.0;
                        for (int d = 0; d < D; d++) {
                            double diff = coords[(int64_t)d * n + i] - q[d];
                            dist += diff * diff;
                        }
                        if (hsize < k) {
                            if (dist < r_prime) {
                                hsize = heap_push(hd, hid, hsize, dist, ids[i]);
                                if (hsize == k) r_prime = hd[0];
                            }
                        } else if (dist < hd[0] || (dist == hd[0] && ids[i] < hid[0])) {
                            heap_replace_root(hd, hid, hsize, dist, ids[i]);
                            r_prime = hd[0];
                        }
                    }
                    continue;
                }
                if (bound >= r_prime) continue;
                double v = node_value[node], qd = q[dim], new_off = qd - v;
                int64_t near, far;
                if (qd < v) { near = node_left[node]; far = node_right[node]; }
                else { near = node_right[node]; far = node_left[node]; }
                double old_off = cur[dim];
                double far_bound = bound - old_off * old_off + new_off * new_off;
                if (far_bound < r_prime) {
                    st_node[sp] = far; st_bound[sp] = far_bound;
                    for (int d = 0; d < D; d++) st_off[sp * D + d] = cur[d];
                    st_off[sp * D + dim] = new_off;
                    sp++;
                }
                st_node[sp] = near; st_bound[sp] = bound;
                for (int d = 0; d < D; d++) st_off[sp * D + d] = cur[d];
                sp++;
            }
            /* drain max-first into the tail -> ascending (d, id) */
            out_counts[qi] = hsize;
            int64_t j = hsize;
            while (hsize > 0) {
                j--;
                out_d[qi * k + j] = hd[0];
                out_ids[qi * k + j] = hid[0];
                hsize--;
                if (hsize > 0) heap_replace_root(hd, hid, hsize, hd[hsize], hid[hsize]);
            }
            if (out_counters) { out_counters[qi * 3] = c0; out_counters[qi * 3 + 1] = c1; out_counters[qi * 3 + 2] = c2; }
        }
        free(st_node); free(st_bound); free(st_off); free(cur); free(hd); free(hid);
    }
}

/* ------------------------------------------------------------ brute force --- */
/* pkg/tests/conftest.py:8-18 oracle_topk: linear scan with the
 * core.py:199-228 distance, strict radius filter, lexsort((ids, dists))[:k].
 * coords is (D, n) row-major. */
void kdo_brute_knn(const double *coords, int64_t n, const uint64_t *ids, int D, const double *queries,
                   int64_t nq, int64_t k, const double *radii, double *out_d, uint64_t *out_ids,
                   int64_t *out_counts, int nthreads) {
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
#pragma omp parallel for schedule(dynamic, 4)
    for (int64_t qi = 0; qi < nq; qi++) {
        const double *q = queries + qi * D;
        double r = radii ? radii[qi] : INFINITY;
        double *bd = out_d + qi * k;
        uint64_t *bi = out_ids + qi * k;
        int64_t cnt = 0;
        for (int64_t i = 0; i < n; i++) {
            double dist = 0.0;
            for (int d = 0; d < D; d++) {
                double diff = coords[(int64_t)d * n + i] - q[d];
                dist += diff * diff;
            }
            if (!(dist < r)) continue;
            uint64_t id = ids[i];
            if (cnt == k && !(dist < bd[k - 1] || (dist == bd[k - 1] && id < bi[k - 1]))) continue;
            int64_t p = cnt < k ? cnt : k - 1;
            while (p > 0 && (dist < bd[p - 1] || (dist == bd[p - 1] && id < bi[p - 1]))) {
                bd[p] = bd[p - 1]; bi[p] = bi[p - 1]; p--;
            }
            bd[p] = dist; bi[p] = id;
            if (cnt < k) cnt++;
        }
        out_counts[qi] = cnt;
    }
}
