/*
 * medtree_oracle.c -- CPU restatement of the reference running-median
 * algorithm (interval-occurrences trees, "IOT"), used ONLY as test
 * infrastructure: the parity checker for the CUDA path and the timed CPU
 * baseline in bench.py.  Nothing in the product path links or calls this.
 *
 * Parity pinned: tests/test_oracle.py checks this code against golden
 * vectors produced by the reference package itself (tests/golden/, made by
 * tests/golden/make_golden.py importing /root/reference/pkg/src/medtree) and
 * against the SHA-256 digest published in BASELINE.md.
 *
 * Every function follows the reference numba kernels in
 *   /root/reference/pkg/src/medtree/_kernels.py  (cited as K:line)
 * and the band driver in
 *   /root/reference/pkg/src/medtree/engine.py    (cited as E:line).
 * Op tallies (counting=True) are not restated: they never change results
 * (K:1-8, reference tests/test_engine.py:226-240).
 *
 * Counter layout (K:3-6): slot 0 = top count, slots 1.. = explicit left
 * nodes in flat preorder (node, left subtree, right-hanging subtree).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ------------------------------------------------------------ columns */

/* K:31-66 col_add_u / col_remove_u: d bisection steps, left-branch counts. */
static inline void col_step_u(int32_t *col, int v, int d, int32_t delta)
{
    int64_t pos = 1, lo = 0, w = (int64_t)1 << d;
    for (int i = 0; i < d; ++i) {
        w >>= 1;
        if (v < lo + w) {
            col[pos] += delta;
            pos += 1;
        } else {
            lo += w;
            pos += w;
        }
    }
}

/* K:69-112 col_add_a / col_remove_a: stored splits, leaf + precision stops. */
static inline void col_step_a(int32_t *col, int v, const int64_t *up,
                              const uint8_t *leaf, const int64_t *span,
                              int64_t n_values, int64_t precision, int32_t delta)
{
    int64_t pos = 1, hi = n_values;
    for (;;) {
        int64_t s = up[pos];
        if (v < s) {
            col[pos] += delta;
            if (leaf[pos] != 0) return;
            hi = s;
            pos += 1;
        } else {
            int64_t nxt = pos + span[pos];
            if (hi - s <= precision) return;
            pos = nxt;
        }
    }
}

typedef struct {
    int adaptive;            /* 0: uniform bisection, 1: stored topology */
    int d;                   /* bit depth */
    int levels;              /* uniform descent depth (E:32-35) */
    const int64_t *up;       /* adaptive topology arrays (topology.py:214-264) */
    const uint8_t *leaf;
    const int64_t *span;
    int64_t slots;
    int64_t n_values;
    int64_t precision;
    int64_t max_error;
} topo_t;

static inline void col_step(const topo_t *t, int32_t *col, int v, int32_t delta)
{
    if (t->adaptive)
        col_step_a(col, v, t->up, t->leaf, t->span, t->n_values, t->precision, delta);
    else
        col_step_u(col, v, t->d, delta);
}

/* K:115-140 advance_col_*: drop clamp(y-h2-1), take clamp(y+h2). */
static inline void advance_col(const topo_t *t, int32_t *col, const uint16_t *img,
                               int H, int W, int c, int y, int h2)
{
    int y_out = y - h2 - 1;
    if (y_out < 0) y_out = 0;
    int y_in = y + h2;
    if (y_in > H - 1) y_in = H - 1;
    col_step(t, col, img[(int64_t)y_out * W + c], -1);
    col_step(t, col, img[(int64_t)y_in * W + c], +1);
}

/* ------------------------------------------------------- window tree */

typedef struct {
    int64_t *win, *lastx;
    uint8_t *valid;
    int32_t *cols;           /* [W][slots], reference layout (engine.py:74) */
    int64_t slots;
} state_t;

/* K:145-194 sync_node: hit / replay g<n column steps / rebuild. */
static inline int64_t sync_node(state_t *s, int64_t k, int x, int n, int h2, int W)
{
    if (s->valid[k]) {
        int64_t g = x - s->lastx[k];
        if (g == 0) return s->win[k];
        if (g < n) {
            int64_t c = s->win[k];
            for (int64_t p = s->lastx[k] + 1; p <= x; ++p) {
                int64_t cin = p + h2;
                if (cin > W - 1) cin = W - 1;
                int64_t cout = p - h2 - 1;
                if (cout < 0) cout = 0;
                c += (int64_t)s->cols[cin * s->slots + k] - s->cols[cout * s->slots + k];
            }
            s->win[k] = c;
            s->lastx[k] = x;
            return c;
        }
    }
    int64_t sum = 0;
    for (int j = -h2; j <= h2; ++j) {
        int64_t cc = (int64_t)x + j;
        if (cc < 0) cc = 0;
        else if (cc > W - 1) cc = W - 1;
        sum += s->cols[cc * s->slots + k];
    }
    s->win[k] = sum;
    s->valid[k] = 1;
    s->lastx[k] = x;
    return sum;
}

/* K:197-210 rebuild_all (mode "unconditional", row start). */
static void rebuild_all(state_t *s, int x, int h2, int W)
{
    for (int64_t k = 1; k < s->slots; ++k) {
        int64_t sum = 0;
        for (int j = -h2; j <= h2; ++j) {
            int64_t cc = (int64_t)x + j;
            if (cc < 0) cc = 0;
            else if (cc > W - 1) cc = W - 1;
            sum += s->cols[cc * s->slots + k];
        }
        s->win[k] = sum;
    }
}

/* K:213-224 shift_all (mode "unconditional", horizontal step). */
static void shift_all(state_t *s, int x, int h2, int W)
{
    int64_t cin = (int64_t)x + h2;
    if (cin > W - 1) cin = W - 1;
    int64_t cout = (int64_t)x - h2 - 1;
    if (cout < 0) cout = 0;
    for (int64_t k = 1; k < s->slots; ++k)
        s->win[k] += (int64_t)s->cols[cin * s->slots + k] - s->cols[cout * s->slots + k];
}

static inline int64_t node_count(state_t *s, int on_demand, int64_t pos, int x,
                                 int n, int h2, int W)
{
    return on_demand ? sync_node(s, pos, x, n, h2, W) : s->win[pos];
}

/* K:229-253 extract_u: `levels` bisection steps; returns interval lower bound. */
static inline int64_t extract_u(state_t *s, const topo_t *t, int on_demand, int x,
                                int n, int h2, int W, int64_t r)
{
    int64_t acc = 0, pos = 1, lo = 0, w = (int64_t)1 << t->d;
    for (int i = 0; i < t->levels; ++i) {
        w >>= 1;
        int64_t below = acc + node_count(s, on_demand, pos, x, n, h2, W);
        if (r <= below) {
            pos += 1;
        } else {
            acc = below;
            lo += w;
            pos += w;
        }
    }
    return lo;
}

/* K:256-289 extract_a: descent until width <= max_error or a leaf. */
static inline int64_t extract_a(state_t *s, const topo_t *t, int on_demand, int x,
                                int n, int h2, int W, int64_t r)
{
    int64_t acc = 0, pos = 1, lo = 0, hi = t->n_values;
    while (hi - lo > t->max_error) {
        int64_t sp = t->up[pos];
        int64_t below = acc + node_count(s, on_demand, pos, x, n, h2, W);
        if (r <= below) {
            hi = sp;
            if (t->leaf[pos] != 0) break;
            pos += 1;
        } else {
            acc = below;
            int64_t nxt = pos + t->span[pos];
            lo = sp;
            if (hi - lo <= t->precision) break;
            pos = nxt;
        }
    }
    return lo;
}

/* K:294-323 init_columns_*: columns hold the span of a virtual row -1. */
static void init_columns(const topo_t *t, state_t *s, const uint16_t *img,
                         int H, int W, int n, int h2)
{
    for (int x = 0; x < W; ++x) {
        int32_t *col = s->cols + (int64_t)x * s->slots;
        col[0] = n;
        for (int j = -h2; j <= h2; ++j) {
            int y = j - 1;
            if (y < 0) y = 0;
            else if (y > H - 1) y = H - 1;
            col_step(t, col, img[(int64_t)y * W + x], +1);
        }
    }
}

/* K:326-388 run_frame_u / run_frame_a: the frame driver. */
static void run_frame(const topo_t *t, state_t *s, const uint16_t *img,
                      uint16_t *out, int H, int W, int n, int64_t r, int on_demand)
{
    int h2 = n / 2;
    memset(s->cols, 0, sizeof(int32_t) * (size_t)W * (size_t)s->slots);
    memset(s->win, 0, sizeof(int64_t) * (size_t)s->slots);
    memset(s->lastx, 0, sizeof(int64_t) * (size_t)s->slots);
    memset(s->valid, 0, (size_t)s->slots);
    s->win[0] = (int64_t)n * n;
    init_columns(t, s, img, H, W, n, h2);
    for (int y = 0; y < H; ++y) {
        int top = h2 < W - 1 ? h2 : W - 1;
        for (int c = 0; c <= top; ++c)
            advance_col(t, s->cols + (int64_t)c * s->slots, img, H, W, c, y, h2);
        if (on_demand)
            memset(s->valid, 0, (size_t)s->slots);
        else
            rebuild_all(s, 0, h2, W);
        for (int x = 0; x < W; ++x) {
            if (x > 0) {
                if (x + h2 <= W - 1)
                    advance_col(t, s->cols + (int64_t)(x + h2) * s->slots, img, H, W,
                                x + h2, y, h2);
                if (!on_demand) shift_all(s, x, h2, W);
            }
            int64_t v = t->adaptive ? extract_a(s, t, on_demand, x, n, h2, W, r)
                                    : extract_u(s, t, on_demand, x, n, h2, W, r);
            out[(int64_t)y * W + x] = (uint16_t)v;
        }
    }
}

/* ------------------------------------------------------ band driver */

typedef struct {
    const topo_t *t;
    const uint16_t *img;
    uint16_t *out;
    int H, W, n, on_demand;
    int64_t r;
    int64_t a, b;            /* output rows [a, b) of this band */
    int status;
} band_job_t;

static void *band_worker(void *arg)
{
    band_job_t *j = (band_job_t *)arg;
    int h2 = j->n / 2;
    /* E:252-260: halo = h2 rows, clamped at the global edges */
    int64_t top = j->a - h2 > 0 ? j->a - h2 : 0;
    int64_t bottom = j->b + h2 < j->H ? j->b + h2 : j->H;
    int subH = (int)(bottom - top);
    state_t s;
    s.slots = j->t->slots;
    s.cols = (int32_t *)malloc(sizeof(int32_t) * (size_t)j->W * (size_t)s.slots);
    s.win = (int64_t *)malloc(sizeof(int64_t) * (size_t)s.slots);
    s.lastx = (int64_t *)malloc(sizeof(int64_t) * (size_t)s.slots);
    s.valid = (uint8_t *)malloc((size_t)s.slots);
    uint16_t *sub_out = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)subH * (size_t)j->W);
    if (!s.cols || !s.win || !s.lastx || !s.valid || !sub_out) {
        j->status = -1;
    } else {
        run_frame(j->t, &s, j->img + top * j->W, sub_out, subH, j->W, j->n, j->r,
                  j->on_demand);
        memcpy(j->out + j->a * j->W, sub_out + (j->a - top) * j->W,
               sizeof(uint16_t) * (size_t)(j->b - j->a) * (size_t)j->W);
        j->status = 0;
    }
    free(s.cols);
    free(s.win);
    free(s.lastx);
    free(s.valid);
    free(sub_out);
    return NULL;
}

/*
 * Public oracle entry.  img/out: uint16 row-major [H][W] (the reference
 * works on a uint16 copy, E:70).  mode_adaptive selects run_frame_a with the
 * caller's topology arrays; on_demand=0 is mode "unconditional".  bands
 * follows E:243-262 (linspace edges, h2 halo rows); `threads` bands run
 * concurrently (the reference runs them serially -- results are identical,
 * reference tests/test_engine.py:243-256).  Returns 0 or -1 (out of memory).
 */
int mto_filter(const uint16_t *img, int H, int W, uint16_t *out, int n, int d,
               int levels, int64_t rank, int on_demand, int mode_adaptive,
               const int64_t *up, const uint8_t *leaf, const int64_t *span,
               int64_t slots, int64_t precision, int64_t max_error,
               int bands, int threads)
{
    topo_t t;
    t.adaptive = mode_adaptive;
    t.d = d;
    t.levels = levels;
    t.up = up;
    t.leaf = leaf;
    t.span = span;
    t.n_values = (int64_t)1 << d;
    t.slots = mode_adaptive ? slots : t.n_values;
    t.precision = precision;
    t.max_error = max_error;

    if (bands < 1) bands = 1;
    if (bands > H) bands = H;
    if (threads < 1) threads = 1;
    band_job_t *jobs = (band_job_t *)calloc((size_t)bands, sizeof(band_job_t));
    if (!jobs) return -1;
    int njobs = 0;
    for (int i = 0; i < bands; ++i) {
        /* numpy.linspace(0, H, bands+1, dtype=int): floor(i*H/bands) */
        int64_t a = (int64_t)((double)H * i / bands);
        int64_t b = (int64_t)((double)H * (i + 1) / bands);
        if (i == bands - 1) b = H;
        if (a == b) continue;
        band_job_t *j = &jobs[njobs++];
        j->t = &t;
        j->img = img;
        j->out = out;
        j->H = H;
        j->W = W;
        j->n = n;
        j->on_demand = on_demand;
        j->r = rank;
        j->a = a;
        j->b = b;
        j->status = 0;
    }
    int status = 0;
    for (int base = 0; base < njobs; base += threads) {
        int cnt = njobs - base < threads ? njobs - base : threads;
        pthread_t *tids = (pthread_t *)calloc((size_t)cnt, sizeof(pthread_t));
        int *started = (int *)calloc((size_t)cnt, sizeof(int));
        for (int i = 0; i < cnt; ++i) {
            if (cnt == 1 || pthread_create(&tids[i], NULL, band_worker, &jobs[base + i]) != 0) {
                band_worker(&jobs[base + i]);
            } else {
                started[i] = 1;
            }
        }
        for (int i = 0; i < cnt; ++i)
            if (started[i]) pthread_join(tids[i], NULL);
        for (int i = 0; i < cnt; ++i)
            if (jobs[base + i].status) status = -1;
        free(tids);
        free(started);
    }
    free(jobs);
    return status;
}
