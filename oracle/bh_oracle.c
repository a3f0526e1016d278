/*
 * bh_oracle.c -- plain, slow, fp64 CPU Barnes-Hut oracle.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_1109_5190_b200/csrc); neither includes the other.
 *
 * What it computes follows the paper step by step, in the paper's order, with
 * the readings of DESIGN.md §3 where the paper is
 * silent.  Citations are to /root/reference/PAPER.md (the paper) and
 * SPEC.md (the CPU program spec, used only for interfaces / test ideas).
 *
 *  1. Root cube + Morton keys          (§1 "hierarchy of cube
 *     structures ... recursive algorithm"; reading L10: fp32 op sequence)
 *  2. Stable sort of keys               (reading L13: ties -> user index)
 *  3. Octree by recursive insertion      ("subdivides the cubes
 *     until there is one particle per sub-cube"; L9: 21-level cap, buckets)
 *  4. Mass / centre of mass bottom-up    ("compute center of
 *     mass"; L14: fp64 sequential child-order sums)
 *  5. Per-particle recursive walk       (§3: a remote cluster
 *     is one body iff D > r/theta; L1-L5: r = cell side, D to the COM, strict,
 *     cells containing the target are opened)
 *  6. Plummer-softened Newtonian force  (PAPER.md:52-53 gravity; L6/L7)
 *  7. Leapfrog (kick-drift, deferred closing kick)  (PAPER.md:461-463
 *     "compute the next iteration values"; L8)
 *  8. O(N^2) direct sum                 (SPEC.md:213-221 accel_direct)
 *  9. Optional quadrupole moments       ("incorporating
 *     multipole moments" as future work; reading L25 of
 *     DESIGN.md §3): traceless Q about each cell's centre of mass, combined
 *     bottom-up in child order by the parallel-axis rule, and the softened
 *     monopole + quadrupole field of every accepted cell
 *
 * Parity pins: every function here is checked by tests/test_oracle_pins.py
 * against closed forms, brute force on tiny inputs and the worked example
 * of SURVEY.md §8(c) (Fig. 2 analogue) -- see DESIGN.md §4.
 *
 * Compile with -ffp-contract=off: every fp32 and fp64 operation below is a
 * single IEEE round-to-nearest operation (x86-64 SSE).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXLEVEL 21 /* 63-bit keys: 21 three-bit digits (L9) */

enum { OR_OK = 0, OR_ERR_ARG = -1, OR_ERR_OOM = -3, OR_ERR_NONFINITE = -5 };

typedef struct onode {
    struct onode *child[8]; /* internal node: children by Morton digit     */
    int level;              /* 0 = root cube                                */
    int is_leaf;            /* single particle leaf or level-21 bucket       */
    int64_t nmemb;          /* particles stored in a leaf/bucket             */
    int64_t cap;            /* capacity of memb[] (buckets grow)             */
    int64_t *memb;          /* sorted positions of leaf/bucket members       */
    int64_t inl;            /* inline storage for the first member           */
    int64_t first, count;   /* sorted range covered (set by DFS numbering)   */
    double M, MX[3], com[3];
    double Q[6];            /* traceless quadrupole about com: xx yy zz xy xz yz */
} onode;

typedef struct oracle_ctx {
    int64_t n;
    double *mass, *pos, *vel; /* fp64 state, user order */
    double theta, eps, G, dt;
    int multipole; /* 1: monopole cells (the paper's method), 2: + quadrupole */
    int64_t k; /* steps taken (0: next kick is the half kick) */
    /* tree state (valid after oracle_build) */
    int built;
    float lo[3], L, scale;
    uint64_t *key;       /* key of user particle i */
    int64_t *perm;       /* sorted position -> user index */
    int64_t *rank;       /* user index -> sorted position (k_i) */
    onode *pool;
    int64_t pool_used, pool_cap;
    onode *root;
    int64_t n_nodes; /* exported nodes (internal + leaves + buckets) */
    char err[256];
} oracle_ctx;

/* ---------------------------------------------------------------- step 1 */
/* Root cube and keys, reading L10: in fp32, no FMA,
 * lo_a = min x_a, L = max_a(max x_a - lo_a), scale = 2^21 / L,
 * q_a = min(2^21-1, (uint32) floorf((x_a - lo_a) * scale)); L == 0 or a
 * non-finite scale -> scale = 0.  key: x-major 3-bit interleave, bit by bit. */
static void root_cube(int64_t n, const float *p32, float lo[3], float *L, float *scale) {
    float hi[3];
    for (int a = 0; a < 3; a++) { lo[a] = p32[a]; hi[a] = p32[a]; }
    for (int64_t i = 1; i < n; i++)
        for (int a = 0; a < 3; a++) {
            float x = p32[3 * i + a];
            if (x < lo[a]) lo[a] = x;
            if (x > hi[a]) hi[a] = x;
        }
    float Lm = 0.0f;
    for (int a = 0; a < 3; a++) {
        float e = hi[a] - lo[a];
        if (e > Lm) Lm = e;
    }
    *L = Lm;
    float s = 2097152.0f / Lm;
    if (Lm == 0.0f || !isfinite(s)) s = 0.0f;
    *scale = s;
}

static uint32_t quantise(float x, float lo, float scale) {
    float t = (x - lo) * scale;
    float f = floorf(t);
    uint32_t q = (uint32_t)f;
    if (q > 2097151u) q = 2097151u;
    return q;
}

static uint64_t interleave(uint32_t qx, uint32_t qy, uint32_t qz) {
    uint64_t key = 0;
    for (int b = 0; b < MAXLEVEL; b++) {
        key |= (uint64_t)((qx >> b) & 1u) << (3 * b + 2);
        key |= (uint64_t)((qy >> b) & 1u) << (3 * b + 1);
        key |= (uint64_t)((qz >> b) & 1u) << (3 * b);
    }
    return key;
}

/* ---------------------------------------------------------------- step 2 */
/* Stable sort by key == sort by (key, user index): reading L13. */
static const uint64_t *g_sort_keys;
static int cmp_key_index(const void *a, const void *b) {
    int64_t i = *(const int64_t *)a, j = *(const int64_t *)b;
    uint64_t ki = g_sort_keys[i], kj = g_sort_keys[j];
    if (ki < kj) return -1;
    if (ki > kj) return 1;
    return (i < j) ? -1 : (i > j);
}

/* ---------------------------------------------------------------- step 3 */
static onode *new_node(oracle_ctx *c, int level) {
    if (c->pool_used == c->pool_cap) return NULL;
    onode *nd = &c->pool[c->pool_used++];
    memset(nd, 0, sizeof(*nd));
    nd->level = level;
    return nd;
}

static int digit(uint64_t key, int level_of_child) {
    /* digit selecting the child at level `level_of_child` (1..21) */
    return (int)((key >> (3 * (MAXLEVEL - level_of_child))) & 7u);
}

static void leaf_free(onode *nd) {
    if (nd->memb && nd->memb != &nd->inl) free(nd->memb);
    nd->memb = NULL; nd->nmemb = 0; nd->cap = 0;
}

static int leaf_push(onode *nd, int64_t sp) {
    if (nd->cap == 0) { nd->memb = &nd->inl; nd->cap = 1; }
    if (nd->nmemb == nd->cap) {
        int64_t nc = 2 * nd->cap;
        int64_t *m = (int64_t *)malloc((size_t)nc * sizeof(int64_t));
        if (!m) return -1;
        memcpy(m, nd->memb, (size_t)nd->nmemb * sizeof(int64_t));
        if (nd->memb != &nd->inl) free(nd->memb);
        nd->memb = m;
        nd->cap = nc;
    }
    nd->memb[nd->nmemb++] = sp;
    return 0;
}

/* Insert sorted particle sp (user index perm[sp]) below node nd.  A cell
 * holding >= 2 particles at level < 21 is subdivided by key digit; a level-21
 * cell with >= 2 particles is a bucket leaf (L9). */
static int insert(oracle_ctx *c, onode *nd, int64_t sp) {
    for (;;) {
        if (nd->is_leaf) {
            if (nd->level == MAXLEVEL) return leaf_push(nd, sp); /* bucket */
            /* subdivide: push the resident particle one level down */
            int64_t old = nd->memb[0];
            leaf_free(nd);
            nd->is_leaf = 0;
            int d = digit(c->key[c->perm[old]], nd->level + 1);
            onode *ch = new_node(c, nd->level + 1);
            if (!ch) return -2;
            ch->is_leaf = 1;
            if (leaf_push(ch, old)) return -1;
            nd->child[d] = ch;
            continue; /* retry inserting sp into the now-internal node */
        }
        int d = digit(c->key[c->perm[sp]], nd->level + 1);
        if (!nd->child[d]) {
            onode *ch = new_node(c, nd->level + 1);
            if (!ch) return -2;
            ch->is_leaf = 1;
            nd->child[d] = ch;
            return leaf_push(ch, sp);
        }
        nd = nd->child[d];
    }
}

/* DFS pre-order numbering (children in digit order): first/count per node. */
static int64_t number_dfs(onode *nd, int64_t *next_first) {
    int64_t nodes = 1;
    nd->first = *next_first;
    if (nd->is_leaf) {
        *next_first += nd->nmemb;
    } else {
        for (int d = 0; d < 8; d++)
            if (nd->child[d]) nodes += number_dfs(nd->child[d], next_first);
    }
    nd->count = *next_first - nd->first;
    return nodes;
}

/* ---------------------------------------------------------------- step 4 */
/* Moments (L14): leaf M = m, MX = m*x (exact in fp64); internal node and
 * bucket: sequential left-to-right sums over children in digit order (bucket
 * members in sorted order) starting from 0; com = MX / M. */
/* Step 9.  The traceless quadrupole of a point mass m at offset y from the
 * expansion centre, m (3 y y^T - |y|^2 I), added to Q in the order xx yy zz xy
 * xz yz; a cell's Q about its centre of mass is the sum over its children in
 * digit order of (child Q about the child's com) + (the child's mass at the
 * offset d = com_child - com) -- the parallel-axis rule, exact because each
 * child's mass dipole about its own com vanishes.  Particles (single leaves,
 * bucket members) are point masses with Q = 0 about themselves. */
static void add_point_quad(double *Q, double m, const double *y) {
    double r2 = y[0] * y[0];
    r2 = r2 + y[1] * y[1];
    r2 = r2 + y[2] * y[2];
    Q[0] = Q[0] + m * (3.0 * y[0] * y[0] - r2);
    Q[1] = Q[1] + m * (3.0 * y[1] * y[1] - r2);
    Q[2] = Q[2] + m * (3.0 * y[2] * y[2] - r2);
    Q[3] = Q[3] + m * (3.0 * y[0] * y[1]);
    Q[4] = Q[4] + m * (3.0 * y[0] * y[2]);
    Q[5] = Q[5] + m * (3.0 * y[1] * y[2]);
}

static void quadrupole(oracle_ctx *c, onode *nd) {
    for (int k = 0; k < 6; k++) nd->Q[k] = 0.0;
    if (nd->is_leaf) {
        for (int64_t t = 0; t < nd->nmemb; t++) {
            int64_t u = c->perm[nd->memb[t]];
            double y[3];
            for (int a = 0; a < 3; a++) y[a] = c->pos[3 * u + a] - nd->com[a];
            add_point_quad(nd->Q, c->mass[u], y);
        }
        return;
    }
    for (int d = 0; d < 8; d++) {
        onode *ch = nd->child[d];
        if (!ch) continue;
        for (int k = 0; k < 6; k++) nd->Q[k] = nd->Q[k] + ch->Q[k];
        double y[3];
        for (int a = 0; a < 3; a++) y[a] = ch->com[a] - nd->com[a];
        add_point_quad(nd->Q, ch->M, y);
    }
}

static void moments(oracle_ctx *c, onode *nd) {
    nd->M = 0.0;
    nd->MX[0] = nd->MX[1] = nd->MX[2] = 0.0;
    if (nd->is_leaf) {
        for (int64_t t = 0; t < nd->nmemb; t++) {
            int64_t u = c->perm[nd->memb[t]];
            double m = c->mass[u];
            nd->M = nd->M + m;
            for (int a = 0; a < 3; a++) nd->MX[a] = nd->MX[a] + m * c->pos[3 * u + a];
        }
    } else {
        for (int d = 0; d < 8; d++) {
            onode *ch = nd->child[d];
            if (!ch) continue;
            moments(c, ch);
            nd->M = nd->M + ch->M;
            for (int a = 0; a < 3; a++) nd->MX[a] = nd->MX[a] + ch->MX[a];
        }
    }
    for (int a = 0; a < 3; a++) nd->com[a] = nd->MX[a] / nd->M;
    if (c->multipole >= 2) quadrupole(c, nd);
}

/* ---------------------------------------------------------------- steps 5-6 */
typedef struct {
    double x[3];   /* target position (fp64 state) */
    int64_t ki;    /* target sorted position */
    double acc[3]; /* sum of contributions (without G) */
    int64_t count; /* interactions */
    int nonfinite;
} walker;

/* d^2 = ((cx-x)^2 + (cy-y)^2) + (cz-z)^2 with this association (L23/§8c). */
static double dist2(const double *src, const double *x) {
    double dx = src[0] - x[0], dy = src[1] - x[1], dz = src[2] - x[2];
    double d2 = dx * dx;
    d2 = d2 + dy * dy;
    d2 = d2 + dz * dz;
    return d2;
}

/* One contribution (src - x) * m / (r^2 + eps^2)^(3/2), Plummer-softened
 * Newtonian gravity (L6). */
static void contribute(const oracle_ctx *c, walker *w, double m, const double *src) {
    double r2 = dist2(src, w->x) + c->eps * c->eps;
    if (r2 == 0.0) { w->nonfinite = 1; return; }
    double inv3 = 1.0 / (r2 * sqrt(r2));
    for (int a = 0; a < 3; a++) w->acc[a] = w->acc[a] + (src[a] - w->x[a]) * m * inv3;
    w->count++;
}

/* An accepted cell with multipole = 2: the monopole contribution, then the
 * quadrupole field of the softened potential -(G/2) r^T Q r / r_e^5 (r = x -
 * com, r_e^2 = |r|^2 + eps^2), written with dr = com - x:
 *   a_q = -(Q dr) / r_e^5 + (5/2) (dr^T Q dr) dr / r_e^7        (G applied last) */
static void contribute_cell(const oracle_ctx *c, walker *w, const onode *nd) {
    contribute(c, w, nd->M, nd->com);
    if (c->multipole < 2) return;
    double dr[3];
    for (int a = 0; a < 3; a++) dr[a] = nd->com[a] - w->x[a];
    double r2 = dist2(nd->com, w->x) + c->eps * c->eps;
    if (r2 == 0.0) { w->nonfinite = 1; return; }
    const double *Q = nd->Q;
    double q[3];
    q[0] = Q[0] * dr[0] + Q[3] * dr[1] + Q[4] * dr[2];
    q[1] = Q[3] * dr[0] + Q[1] * dr[1] + Q[5] * dr[2];
    q[2] = Q[4] * dr[0] + Q[5] * dr[1] + Q[2] * dr[2];
    double s = q[0] * dr[0] + q[1] * dr[1] + q[2] * dr[2];
    double inv2 = 1.0 / r2, inv = sqrt(inv2);
    double inv5 = inv2 * inv2 * inv, inv7 = inv5 * inv2;
    for (int a = 0; a < 3; a++) w->acc[a] = w->acc[a] - q[a] * inv5 + 2.5 * s * inv7 * dr[a];
}

static void contribute_particle(const oracle_ctx *c, walker *w, int64_t sp) {
    int64_t u = c->perm[sp];
    contribute(c, w, c->mass[u], &c->pos[3 * u]);
}

/* MAC ("treated as a single body only if D is greater than
 * r/theta"), reading L1-L4: accept iff s_l^2 < theta^2 * d^2 (strict, fp64),
 * s_l = L * 2^-l the cell side, d measured to the centre of mass. */
static int mac_accept(const oracle_ctx *c, const onode *nd, const double *x) {
    double s = ldexp((double)c->L, -nd->level);
    double s2 = s * s;
    double th2 = c->theta * c->theta;
    double d2 = dist2(nd->com, x);
    return s2 < th2 * d2;
}

static void walk(const oracle_ctx *c, const onode *nd, walker *w) {
    if (nd->is_leaf && nd->nmemb == 1) {
        /* single-particle leaf: j != i contributes, j == i is skipped */
        if (nd->memb[0] != w->ki) contribute_particle(c, w, nd->memb[0]);
        return;
    }
    int contains = nd->first <= w->ki && w->ki < nd->first + nd->count;
    /* L5: a cell containing the target is never accepted */
    if (!contains && mac_accept(c, nd, w->x)) {
        contribute_cell(c, w, nd);
        return;
    }
    if (nd->is_leaf) { /* bucket: its children are its member particles */
        for (int64_t t = 0; t < nd->nmemb; t++)
            if (nd->memb[t] != w->ki) contribute_particle(c, w, nd->memb[t]);
        return;
    }
    for (int d = 0; d < 8; d++)
        if (nd->child[d]) walk(c, nd->child[d], w);
}

/* ---------------------------------------------------------------- API */
static void free_tree(oracle_ctx *c) {
    if (c->pool) {
        for (int64_t t = 0; t < c->pool_used; t++) leaf_free(&c->pool[t]);
        free(c->pool);
    }
    c->pool = NULL; c->pool_used = c->pool_cap = 0; c->root = NULL;
    c->built = 0;
}

oracle_ctx *oracle_create(int64_t n, const double *mass, const double *pos, const double *vel,
                          double theta, double eps, double G, double dt, int64_t k0) {
    if (n < 1 || !mass || !pos) return NULL;
    oracle_ctx *c = (oracle_ctx *)calloc(1, sizeof(oracle_ctx));
    if (!c) return NULL;
    c->n = n;
    c->mass = (double *)malloc((size_t)n * sizeof(double));
    c->pos = (double *)malloc((size_t)n * 3 * sizeof(double));
    c->vel = (double *)calloc((size_t)n * 3, sizeof(double));
    c->key = (uint64_t *)malloc((size_t)n * sizeof(uint64_t));
    c->perm = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    c->rank = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    if (!c->mass || !c->pos || !c->vel || !c->key || !c->perm || !c->rank) return NULL;
    memcpy(c->mass, mass, (size_t)n * sizeof(double));
    memcpy(c->pos, pos, (size_t)n * 3 * sizeof(double));
    if (vel) memcpy(c->vel, vel, (size_t)n * 3 * sizeof(double));
    c->theta = theta; c->eps = eps; c->G = G; c->dt = dt; c->k = k0;
    c->multipole = 1;
    return c;
}

/* Multipole order of accepted cells (1 = the paper's monopole, default;
 * 2 = + quadrupole).  Takes effect at the next oracle_build. */
int oracle_set_multipole(oracle_ctx *c, int order) {
    if (!c || order < 1 || order > 2) return OR_ERR_ARG;
    c->multipole = order;
    c->built = 0;
    return OR_OK;
}

/* Quadrupoles of the exported nodes (DFS order as oracle_get_tree), Q[6] each
 * (xx yy zz xy xz yz); returns the node count. */
static void export_quad(const onode *nd, double *Q, int64_t *at) {
    for (int k = 0; k < 6; k++) Q[6 * *at + k] = nd->Q[k];
    (*at)++;
    if (nd->is_leaf) return;
    for (int d = 0; d < 8; d++)
        if (nd->child[d]) export_quad(nd->child[d], Q, at);
}

int64_t oracle_get_quadrupoles(const oracle_ctx *c, double *Q, int64_t cap) {
    if (!c->built || c->multipole < 2) return -1;
    if (!Q || cap < c->n_nodes) return c->n_nodes;
    int64_t at = 0;
    export_quad(c->root, Q, &at);
    return at;
}

void oracle_destroy(oracle_ctx *c) {
    if (!c) return;
    free_tree(c);
    free(c->mass); free(c->pos); free(c->vel); free(c->key); free(c->perm); free(c->rank);
    free(c);
}

const char *oracle_last_error(const oracle_ctx *c) { return c ? c->err : "null ctx"; }

/* Steps 1-4 on the current state: keys from fp32(x), sort, tree, moments. */
int oracle_build(oracle_ctx *c) {
    int64_t n = c->n;
    free_tree(c);
    float *p32 = (float *)malloc((size_t)n * 3 * sizeof(float));
    if (!p32) return OR_ERR_OOM;
    for (int64_t i = 0; i < 3 * n; i++) {
        p32[i] = (float)c->pos[i];
        if (!isfinite(p32[i])) {
            free(p32);
            snprintf(c->err, sizeof c->err, "non-finite position at particle %lld", (long long)(i / 3));
            return OR_ERR_NONFINITE;
        }
    }
    root_cube(n, p32, c->lo, &c->L, &c->scale);
    for (int64_t i = 0; i < n; i++) {
        uint32_t q[3];
        for (int a = 0; a < 3; a++) q[a] = quantise(p32[3 * i + a], c->lo[a], c->scale);
        c->key[i] = interleave(q[0], q[1], q[2]);
    }
    free(p32);
    for (int64_t i = 0; i < n; i++) c->perm[i] = i;
    g_sort_keys = c->key;
    qsort(c->perm, (size_t)n, sizeof(int64_t), cmp_key_index);
    for (int64_t s = 0; s < n; s++) c->rank[c->perm[s]] = s;

    /* pool: worst case 22 nodes per particle (a 21-level chain + leaf) */
    int64_t cap = 2 * n + 64;
    for (;;) {
        c->pool = (onode *)malloc((size_t)cap * sizeof(onode));
        if (!c->pool) return OR_ERR_OOM;
        c->pool_cap = cap; c->pool_used = 0;
        c->root = new_node(c, 0);
        c->root->is_leaf = 1;
        int rc = 0;
        if (leaf_push(c->root, 0)) rc = -1;
        for (int64_t s = 1; s < n && rc == 0; s++) rc = insert(c, c->root, s);
        if (rc == 0) break;
        free_tree(c);
        if (rc == -1) return OR_ERR_OOM;
        cap *= 2; /* pool exhausted: retry larger */
    }
    int64_t nf = 0;
    c->n_nodes = number_dfs(c->root, &nf);
    moments(c, c->root);
    c->built = 1;
    return OR_OK;
}

int oracle_root(const oracle_ctx *c, float *lo3, float *L, float *scale) {
    if (!c->built) return OR_ERR_ARG;
    for (int a = 0; a < 3; a++) lo3[a] = c->lo[a];
    *L = c->L; *scale = c->scale;
    return OR_OK;
}

/* keys_sorted[s], perm[s] = user index at sorted position s */
int oracle_get_keys(const oracle_ctx *c, uint64_t *keys_sorted, int64_t *perm) {
    if (!c->built) return OR_ERR_ARG;
    for (int64_t s = 0; s < c->n; s++) {
        perm[s] = c->perm[s];
        keys_sorted[s] = c->key[c->perm[s]];
    }
    return OR_OK;
}

typedef struct { uint8_t *level; int64_t *first, *count; double *M, *MX; int64_t at, cap; } exporter;
static void export_dfs(const onode *nd, exporter *e) {
    if (e->at < e->cap) {
        e->level[e->at] = (uint8_t)nd->level;
        e->first[e->at] = nd->first;
        e->count[e->at] = nd->count;
        if (e->M) e->M[e->at] = nd->M;
        if (e->MX) for (int a = 0; a < 3; a++) e->MX[3 * e->at + a] = nd->MX[a];
    }
    e->at++;
    if (!nd->is_leaf)
        for (int d = 0; d < 8; d++)
            if (nd->child[d]) export_dfs(nd->child[d], e);
}

/* DFS pre-order export (level, first, count[, M, MX]); returns node count. */
int64_t oracle_get_tree(const oracle_ctx *c, uint8_t *level, int64_t *first, int64_t *count,
                        double *M, double *MX, int64_t cap) {
    if (!c->built) return -1;
    exporter e = {level, first, count, M, MX, 0, cap};
    export_dfs(c->root, &e);
    return e.at;
}

/* Accelerations (with G) and interaction counts for `nt` targets given by
 * user index (targets == NULL: all particles, nt ignored). */
int oracle_forces(oracle_ctx *c, int64_t nt, const int64_t *targets, double *acc, int64_t *count) {
    if (!c->built) return OR_ERR_ARG;
    int64_t total = targets ? nt : c->n;
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(| : bad)
    for (int64_t t = 0; t < total; t++) {
        int64_t i = targets ? targets[t] : t;
        walker w;
        memset(&w, 0, sizeof w);
        for (int a = 0; a < 3; a++) w.x[a] = c->pos[3 * i + a];
        w.ki = c->rank[i];
        walk(c, c->root, &w);
        for (int a = 0; a < 3; a++) acc[3 * t + a] = c->G * w.acc[a];
        if (count) count[t] = w.count;
        bad |= w.nonfinite;
    }
    if (bad) {
        snprintf(c->err, sizeof c->err, "eps == 0 and coincident particles: infinite force");
        return OR_ERR_NONFINITE;
    }
    return OR_OK;
}

/* Leapfrog (L8) of one particle: k == 0: v += a dt/2, else v += a dt; then
 * x += v dt (fp64). */
static void leapfrog(const oracle_ctx *c, const double *x, const double *v, const double *a, double *xo,
                     double *vo) {
    double kick = (c->k == 0) ? 0.5 * c->dt : c->dt;
    for (int d = 0; d < 3; d++) {
        vo[d] = v[d] + a[d] * kick;
        xo[d] = x[d] + vo[d] * c->dt;
    }
}

/* One step of `nt` targets only (user indices), without changing the state:
 * the tree of the current state (built if needed), the targets' forces, and
 * their leapfrog update into pos_out / vel_out [nt][3].  The teacher-forced
 * trajectory check of the large configurations: the oracle's step from the
 * GPU's state at step k, on sampled particles (reading L24). */
int oracle_step_targets(oracle_ctx *c, int64_t nt, const int64_t *targets, double *pos_out, double *vel_out,
                        int64_t *count) {
    if (nt < 0 || (nt > 0 && !targets)) return OR_ERR_ARG;
    if (!c->built) {
        int rc = oracle_build(c);
        if (rc) return rc;
    }
    double *acc = (double *)malloc((size_t)(nt > 0 ? nt : 1) * 3 * sizeof(double));
    if (!acc) return OR_ERR_OOM;
    int rc = oracle_forces(c, nt, targets, acc, count);
    if (rc == OR_OK)
        for (int64_t t = 0; t < nt; t++) {
            int64_t i = targets[t];
            leapfrog(c, &c->pos[3 * i], &c->vel[3 * i], &acc[3 * t], &pos_out[3 * t], &vel_out[3 * t]);
        }
    free(acc);
    return rc;
}

/* Leapfrog (L8): k == 0: v += a dt/2, else v += a dt; then x += v dt.  One
 * tree and one walk per step; velocities are staggered v_{k-1/2}. */
int oracle_step(oracle_ctx *c, int64_t nsteps, int64_t *interactions) {
    int64_t n = c->n;
    double *acc = (double *)malloc((size_t)n * 3 * sizeof(double));
    int64_t *cnt = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    if (!acc || !cnt) { free(acc); free(cnt); return OR_ERR_OOM; }
    int rc = OR_OK;
    for (int64_t st = 0; st < nsteps; st++) {
        rc = oracle_build(c);
        if (rc) break;
        rc = oracle_forces(c, 0, NULL, acc, cnt);
        if (rc) break;
        int64_t tot = 0;
        for (int64_t i = 0; i < n; i++) {
            leapfrog(c, &c->pos[3 * i], &c->vel[3 * i], &acc[3 * i], &c->pos[3 * i], &c->vel[3 * i]);
            tot += cnt[i];
        }
        if (interactions) interactions[st] = tot;
        c->k++;
    }
    free(acc); free(cnt);
    return rc;
}

int oracle_get_state(const oracle_ctx *c, double *pos, double *vel) {
    if (pos) memcpy(pos, c->pos, (size_t)c->n * 3 * sizeof(double));
    if (vel) memcpy(vel, c->vel, (size_t)c->n * 3 * sizeof(double));
    return OR_OK;
}

/* O(N^2) direct sum: softened pairwise sum over all j != i
 * in ascending j order, times G. */
int oracle_direct(int64_t n, const double *mass, const double *pos, double eps, double G,
                  int64_t nt, const int64_t *targets, double *acc) {
    int64_t total = targets ? nt : n;
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t t = 0; t < total; t++) {
        int64_t i = targets ? targets[t] : t;
        double s[3] = {0.0, 0.0, 0.0};
        for (int64_t j = 0; j < n; j++) {
            if (j == i) continue;
            double r2 = dist2(&pos[3 * j], &pos[3 * i]) + eps * eps;
            if (r2 == 0.0) { bad = 1; continue; }
            double inv3 = 1.0 / (r2 * sqrt(r2));
            for (int a = 0; a < 3; a++) s[a] = s[a] + (pos[3 * j + a] - pos[3 * i + a]) * mass[j] * inv3;
        }
        for (int a = 0; a < 3; a++) acc[3 * t + a] = G * s[a];
    }
    return bad ? OR_ERR_NONFINITE : OR_OK;
}

/* Exposed for the exhaustive interleave / quantisation pins. */
uint64_t oracle_interleave(uint32_t qx, uint32_t qy, uint32_t qz) { return interleave(qx, qy, qz); }
uint32_t oracle_quantise(float x, float lo, float scale) { return quantise(x, lo, scale); }
