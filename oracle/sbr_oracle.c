/*
 * sbr_oracle.c -- CPU restatement of the reference SBR trace-integrate path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py; the product path (paper_2604_09243_b200)
 * never links or calls it.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Parity pin: the functions below are checked bit-for-bit against golden
 * vectors produced by running the reference package itself
 * (tests/golden/make_golden.py, numba 0.65 / numpy 2.3.5); see
 * tests/test_oracle_golden.py.
 *
 * Every routine restates one reference function; the reference location is
 * given as pkg/src/sbr/<file>:<line>.  Arithmetic follows the reference
 * operand association exactly and is compiled with -ffp-contract=off so no
 * a*b+c is fused (numba/LLVM never contracts).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EINVAL 2
#define ORC_ENOMEM 12

typedef struct {
    /* BVH in the reference preorder layout (bvh.py:58-88) */
    const double *nmin, *nmax;      /* (M,3) node boxes (float32 boxes upcast) */
    const int32_t *first, *count;   /* node_first / node_count */
    const int32_t *order;           /* tri_order */
    int64_t nnodes;
    int32_t stack_depth;            /* bvh.params.max_depth + 2 (bvh.py:381) */
    /* mesh SoA (geometry.py:88-127) */
    const double *v0, *v1, *v2, *normals;
    int64_t ntri;
    int32_t single;                 /* 1: float32 mesh -> float32 edge subtraction */
} orc_scene;

typedef struct {
    int64_t pops;       /* node pops (visits) */
    int64_t boxes;      /* _aabb_hit calls */
    int64_t tris;       /* _tri_hit_t calls */
    int64_t internal;   /* internal-node expansions */
    int64_t queries;    /* _traverse calls */
} orc_counters;

/* ---------------------------------------------------------------------- */
/* geometry.py:326-355  _tri_hit_t : edge-inclusive Moller-Trumbore          */
/* ---------------------------------------------------------------------- */
static inline double orc_tri_hit(const orc_scene *s, int64_t ti,
                                 double ox, double oy, double oz,
                                 double dx, double dy, double dz,
                                 double t_min, double t_max)
{
    const double *a = s->v0 + 3 * ti, *b = s->v1 + 3 * ti, *c = s->v2 + 3 * ti;
    double ax = a[0], ay = a[1], az = a[2];
    double e1x, e1y, e1z, e2x, e2y, e2z;
    if (s->single) {
        /* float32 arrays: numba subtracts in float32 */
        e1x = (double)((float)b[0] - (float)ax);
        e1y = (double)((float)b[1] - (float)ay);
        e1z = (double)((float)b[2] - (float)az);
        e2x = (double)((float)c[0] - (float)ax);
        e2y = (double)((float)c[1] - (float)ay);
        e2z = (double)((float)c[2] - (float)az);
    } else {
        e1x = b[0] - ax; e1y = b[1] - ay; e1z = b[2] - az;
        e2x = c[0] - ax; e2y = c[1] - ay; e2z = c[2] - az;
    }
    double px = dy * e2z - dz * e2y;
    double py = dz * e2x - dx * e2z;
    double pz = dx * e2y - dy * e2x;
    double det = e1x * px + e1y * py + e1z * pz;
    if (det == 0.0) return -1.0;
    double inv = 1.0 / det;
    double tx = ox - ax, ty = oy - ay, tz = oz - az;
    double u = (tx * px + ty * py + tz * pz) * inv;
    if (u < 0.0 || u > 1.0) return -1.0;
    double qx = ty * e1z - tz * e1y;
    double qy = tz * e1x - tx * e1z;
    double qz = tx * e1y - ty * e1x;
    double v = (dx * qx + dy * qy + dz * qz) * inv;
    if (v < 0.0 || u + v > 1.0) return -1.0;
    double t = (e2x * qx + e2y * qy + e2z * qz) * inv;
    if (t <= t_min || t > t_max) return -1.0;
    return t;
}

/* ---------------------------------------------------------------------- */
/* geometry.py:358-391  _aabb_hit : slab test, entry clamped to 0           */
/* ---------------------------------------------------------------------- */
static inline int orc_box_hit(const orc_scene *s, int64_t ni,
                              const double o[3], const double inv[3],
                              double t_max, double *entry)
{
    double t_near = 0.0, t_far = t_max;
    for (int ax = 0; ax < 3; ++ax) {
        double lo = s->nmin[3 * ni + ax], hi = s->nmax[3 * ni + ax];
        if (isinf(inv[ax])) {
            if (o[ax] < lo || o[ax] > hi) { *entry = 0.0; return 0; }
        } else {
            double t1 = (lo - o[ax]) * inv[ax];
            double t2 = (hi - o[ax]) * inv[ax];
            if (t1 > t2) { double tmp = t1; t1 = t2; t2 = tmp; }
            if (t1 > t_near) t_near = t1;
            if (t2 < t_far) t_far = t2;
            if (t_near > t_far) { *entry = 0.0; return 0; }
        }
    }
    *entry = t_near;
    return 1;
}

/* ---------------------------------------------------------------------- */
/* bvh.py:306-362  _traverse : explicit stack, near-first, (t,id) lexmin     */
/* ---------------------------------------------------------------------- */
static int64_t orc_traverse(const orc_scene *s, const double o[3],
                            const double d[3], double t_min, double t_max,
                            int32_t *stack, double *t_out, int64_t *visits_out,
                            orc_counters *cnt)
{
    double best_t = t_max;
    int64_t best = -1, visits = 0;
    double inv[3];
    for (int a = 0; a < 3; ++a) inv[a] = d[a] != 0.0 ? 1.0 / d[a] : INFINITY;
    int sp = 0;
    stack[sp++] = 0;
    if (cnt) cnt->queries++;
    while (sp > 0) {
        int32_t node = stack[--sp];
        visits++;
        double e;
        if (cnt) cnt->boxes++;
        if (!orc_box_hit(s, node, o, inv, best_t, &e) || e > best_t) continue;
        int32_t c = s->count[node];
        if (c > 0) {
            int32_t f = s->first[node];
            for (int32_t k = f; k < f + c; ++k) {
                int32_t ti = s->order[k];
                if (cnt) cnt->tris++;
                double t = orc_tri_hit(s, ti, o[0], o[1], o[2], d[0], d[1], d[2],
                                       t_min, best_t);
                if (t > 0.0 && (t < best_t || (t == best_t && ti < best))) {
                    best_t = t;
                    best = ti;
                }
            }
        } else {
            int32_t l = node + 1, r = s->first[node];
            double el, er;
            if (cnt) { cnt->boxes += 2; cnt->internal++; }
            int hl = orc_box_hit(s, l, o, inv, best_t, &el);
            int hr = orc_box_hit(s, r, o, inv, best_t, &er);
            if (hl && hr) {
                if (el <= er) { stack[sp++] = r; stack[sp++] = l; }
                else          { stack[sp++] = l; stack[sp++] = r; }
            } else if (hl) {
                stack[sp++] = l;
            } else if (hr) {
                stack[sp++] = r;
            }
        }
    }
    if (cnt) cnt->pops += visits;
    *t_out = best_t;
    if (visits_out) *visits_out = visits;
    return best;
}

static int orc_threads(int want)
{
#ifdef _OPENMP
    if (want <= 0) want = omp_get_max_threads();
    return want;
#else
    (void)want;
    return 1;
#endif
}

/* bvh.py:365-378 + 407-423  closest_hit_batch */
int orc_closest_hit_batch(const orc_scene *s, const double *o, const double *d,
                          int64_t n, double t_min, double t_max,
                          int64_t *tri, double *t, int64_t *visits,
                          orc_counters *counters, int nthreads)
{
    int nt = orc_threads(nthreads);
    int64_t p = 0, b = 0, tr = 0, in = 0, q = 0;
    int failed = 0;
#pragma omp parallel num_threads(nt) reduction(+:p,b,tr,in,q)
    {
        int32_t *stack = (int32_t *)malloc(sizeof(int32_t) * (size_t)s->stack_depth);
        orc_counters c = {0, 0, 0, 0, 0};
        if (!stack) {
#pragma omp atomic write
            failed = 1;
        } else {
#pragma omp for schedule(dynamic, 256)
            for (int64_t r = 0; r < n; ++r) {
                tri[r] = orc_traverse(s, o + 3 * r, d + 3 * r, t_min, t_max, stack,
                                      t + r, visits ? visits + r : NULL,
                                      counters ? &c : NULL);
            }
            free(stack);
        }
        p += c.pops; b += c.boxes; tr += c.tris; in += c.internal; q += c.queries;
    }
    if (counters) {
        counters->pops = p; counters->boxes = b; counters->tris = tr;
        counters->internal = in; counters->queries = q;
    }
    return failed ? ORC_ENOMEM : ORC_OK;
}

/* tests/meshes.py:51-86  brute-force linear scan (the c5 oracle) */
int orc_brute_force_batch(const orc_scene *s, const double *o, const double *d,
                          int64_t n, double t_min, double t_max,
                          int64_t *tri, double *t, int nthreads)
{
    int nt = orc_threads(nthreads);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 64)
    for (int64_t r = 0; r < n; ++r) {
        double best_t = t_max;
        int64_t best = -1;
        const double *oo = o + 3 * r, *dd = d + 3 * r;
        for (int64_t ti = 0; ti < s->ntri; ++ti) {
            double h = orc_tri_hit(s, ti, oo[0], oo[1], oo[2], dd[0], dd[1], dd[2],
                                   t_min, best_t);
            if (h > 0.0 && (h < best_t || (h == best_t && ti < best))) {
                best_t = h;
                best = ti;
            }
        }
        tri[r] = best;
        t[r] = best_t;
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* transport.py:276-327  _trace_one : bounce loop + escape probe            */
/* ---------------------------------------------------------------------- */
typedef struct {
    uint8_t valid, escaped;
    int32_t bounces;
    double n0[3], path, out_dir[3];
} orc_record;

static void orc_trace_one(const orc_scene *s, double o[3], double d[3],
                          int32_t max_bounces, double eps, int strict,
                          int32_t *stack, orc_record *rec, int32_t *ids,
                          orc_counters *cnt)
{
    double path = 0.0, n0x = 0.0, n0y = 0.0, n0z = 0.0;
    int32_t bounces = 0;
    int valid = 0, escaped = 0;
    for (int32_t it = 0; it < max_bounces; ++it) {
        double t;
        int64_t tri = orc_traverse(s, o, d, 0.0, INFINITY, stack, &t, NULL, cnt);
        if (tri < 0) { escaped = 1; break; }
        const double *nn = s->normals + 3 * tri;
        double nx = nn[0], ny = nn[1], nz = nn[2];
        double nd = nx * d[0] + ny * d[1] + nz * d[2];
        if (nd > 0.0) {
            if (strict && bounces == 0) {
                rec->valid = 0; rec->escaped = 1; rec->bounces = 0;
                rec->n0[0] = rec->n0[1] = rec->n0[2] = 0.0; rec->path = 0.0;
                rec->out_dir[0] = d[0]; rec->out_dir[1] = d[1]; rec->out_dir[2] = d[2];
                return;
            }
            nx = -nx; ny = -ny; nz = -nz; nd = -nd;
        }
        if (ids) ids[it] = (int32_t)tri;
        double hx = o[0] + t * d[0], hy = o[1] + t * d[1], hz = o[2] + t * d[2];
        path += t;
        bounces += 1;
        if (bounces == 1) { n0x = nx; n0y = ny; n0z = nz; valid = 1; }
        d[0] -= 2.0 * nd * nx;
        d[1] -= 2.0 * nd * ny;
        d[2] -= 2.0 * nd * nz;
        o[0] = hx + eps * nx;
        o[1] = hy + eps * ny;
        o[2] = hz + eps * nz;
    }
    if (valid && !escaped) {
        double t;
        int64_t tri = orc_traverse(s, o, d, 0.0, INFINITY, stack, &t, NULL, cnt);
        escaped = tri < 0;
    }
    rec->valid = (uint8_t)valid; rec->escaped = (uint8_t)escaped;
    rec->bounces = bounces; rec->path = path;
    rec->n0[0] = n0x; rec->n0[1] = n0y; rec->n0[2] = n0z;
    rec->out_dir[0] = d[0]; rec->out_dir[1] = d[1]; rec->out_dir[2] = d[2];
}

static void orc_store(int64_t r, const orc_record *rec, uint8_t *valid,
                      double *n0, double *path, int32_t *bounces,
                      uint8_t *escaped, double *out_dir)
{
    valid[r] = rec->valid;
    n0[3 * r] = rec->n0[0]; n0[3 * r + 1] = rec->n0[1]; n0[3 * r + 2] = rec->n0[2];
    path[r] = rec->path;
    bounces[r] = rec->bounces;
    escaped[r] = rec->escaped;
    out_dir[3 * r] = rec->out_dir[0]; out_dir[3 * r + 1] = rec->out_dir[1];
    out_dir[3 * r + 2] = rec->out_dir[2];
}

/* transport.py:330-356 + 375-422  _trace_rows / trace_grid.
 * ids (optional): n * max_bounces int32, -1 padded -- hit triangle per bounce
 * (the F4 ID-recording extension; not part of the reference HitRecords).
 * Rows [i_begin, i_end) only, so bench can time a bounded sample. */
int orc_trace_grid(const orc_scene *s, const double corner[3], const double u[3],
                   const double v[3], const double k[3], double spacing,
                   int64_t n_u, int64_t n_v, int64_t i_begin, int64_t i_end,
                   int32_t max_bounces, double eps, int32_t strict,
                   uint8_t *valid, double *n0, double *path, int32_t *bounces,
                   uint8_t *escaped, double *out_dir, int32_t *ids,
                   orc_counters *counters, int nthreads)
{
    int nt = orc_threads(nthreads);
    int64_t p = 0, b = 0, tr = 0, in = 0, q = 0;
    (void)n_u;
#pragma omp parallel num_threads(nt) reduction(+:p,b,tr,in,q)
    {
        int32_t *stack = (int32_t *)malloc(sizeof(int32_t) * (size_t)s->stack_depth);
        orc_counters c = {0, 0, 0, 0, 0};
#pragma omp for schedule(dynamic, 1)
        for (int64_t i = i_begin; i < i_end; ++i) {
            double bx = corner[0] + (i + 0.5) * spacing * u[0];
            double by = corner[1] + (i + 0.5) * spacing * u[1];
            double bz = corner[2] + (i + 0.5) * spacing * u[2];
            for (int64_t j = 0; j < n_v; ++j) {
                double o[3], d[3];
                o[0] = bx + (j + 0.5) * spacing * v[0];
                o[1] = by + (j + 0.5) * spacing * v[1];
                o[2] = bz + (j + 0.5) * spacing * v[2];
                d[0] = k[0]; d[1] = k[1]; d[2] = k[2];
                int64_t r = i * n_v + j, slot = r - i_begin * n_v;
                int32_t *rid = NULL;
                if (ids) {
                    rid = ids + slot * max_bounces;
                    for (int32_t z = 0; z < max_bounces; ++z) rid[z] = -1;
                }
                orc_record rec;
                orc_trace_one(s, o, d, max_bounces, eps, strict, stack, &rec, rid,
                              counters ? &c : NULL);
                orc_store(slot, &rec, valid, n0, path, bounces, escaped, out_dir);
            }
        }
        free(stack);
        p += c.pops; b += c.boxes; tr += c.tris; in += c.internal; q += c.queries;
    }
    if (counters) {
        counters->pops = p; counters->boxes = b; counters->tris = tr;
        counters->internal = in; counters->queries = q;
    }
    return ORC_OK;
}

/* transport.py:359-372  trace_ray, batched over an explicit ray list */
int orc_trace_rays(const orc_scene *s, const double *origins, const double *dirs,
                   int64_t n, int32_t max_bounces, double eps, int32_t strict,
                   uint8_t *valid, double *n0, double *path, int32_t *bounces,
                   uint8_t *escaped, double *out_dir, int32_t *ids, int nthreads)
{
    int nt = orc_threads(nthreads);
#pragma omp parallel num_threads(nt)
    {
        int32_t *stack = (int32_t *)malloc(sizeof(int32_t) * (size_t)s->stack_depth);
#pragma omp for schedule(dynamic, 64)
        for (int64_t r = 0; r < n; ++r) {
            double o[3] = {origins[3 * r], origins[3 * r + 1], origins[3 * r + 2]};
            double d[3] = {dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2]};
            int32_t *rid = NULL;
            if (ids) {
                rid = ids + r * max_bounces;
                for (int32_t z = 0; z < max_bounces; ++z) rid[z] = -1;
            }
            orc_record rec;
            orc_trace_one(s, o, d, max_bounces, eps, strict, stack, &rec, rid, NULL);
            orc_store(r, &rec, valid, n0, path, bounces, escaped, out_dir);
        }
        free(stack);
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* Record hash (parity at 1e9-ray scale): the same function as the device's */
/* record_hash (paper_2604_09243_b200/csrc/pipeline.h) -- a splitmix64 chain */
/* over r, ids[0..B) (-1 padded), valid|escaped<<8|N<<16, n0, R, out_dir.   */
/* Segment hash = wrapping sum over the segment's rays.                     */
/* ---------------------------------------------------------------------- */
static inline uint64_t orc_mix(uint64_t z)
{
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

static inline uint64_t orc_dbits(double x)
{
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
}

uint64_t orc_record_hash(int64_t r, const int32_t *ids, int32_t max_bounces,
                         const orc_record *rec)
{
    uint64_t h = orc_mix((uint64_t)r);
    for (int32_t b = 0; b < max_bounces; ++b) h = orc_mix(h ^ (uint64_t)(uint32_t)ids[b]);
    h = orc_mix(h ^ ((uint64_t)rec->valid | ((uint64_t)rec->escaped << 8) |
                     ((uint64_t)(uint32_t)rec->bounces << 16)));
    h = orc_mix(h ^ orc_dbits(rec->n0[0]));
    h = orc_mix(h ^ orc_dbits(rec->n0[1]));
    h = orc_mix(h ^ orc_dbits(rec->n0[2]));
    h = orc_mix(h ^ orc_dbits(rec->path));
    h = orc_mix(h ^ orc_dbits(rec->out_dir[0]));
    h = orc_mix(h ^ orc_dbits(rec->out_dir[1]));
    h = orc_mix(h ^ orc_dbits(rec->out_dir[2]));
    return h;
}

/* trace_grid rows [i_begin, i_end) reduced to per-segment record hashes
 * (seg_hash: ceil(n_u*n_v/seg_rays) entries, zeroed here) */
int orc_trace_grid_hash(const orc_scene *s, const double corner[3], const double u[3],
                        const double v[3], const double k[3], double spacing,
                        int64_t n_u, int64_t n_v, int64_t i_begin, int64_t i_end,
                        int32_t max_bounces, double eps, int32_t strict,
                        int64_t seg_rays, uint64_t *seg_hash, int nthreads)
{
    int nt = orc_threads(nthreads);
    const int64_t nseg = (n_u * n_v + seg_rays - 1) / seg_rays;
    memset(seg_hash, 0, sizeof(uint64_t) * (size_t)nseg);
    int failed = 0;
#pragma omp parallel num_threads(nt)
    {
        int32_t *stack = (int32_t *)malloc(sizeof(int32_t) * (size_t)s->stack_depth);
        int32_t *ids = (int32_t *)malloc(sizeof(int32_t) * (size_t)max_bounces);
        uint64_t *loc = (uint64_t *)calloc((size_t)nseg, sizeof(uint64_t));
        if (!stack || !ids || !loc) {
#pragma omp atomic write
            failed = 1;
        } else {
#pragma omp for schedule(dynamic, 1)
            for (int64_t i = i_begin; i < i_end; ++i) {
                double bx = corner[0] + (i + 0.5) * spacing * u[0];
                double by = corner[1] + (i + 0.5) * spacing * u[1];
                double bz = corner[2] + (i + 0.5) * spacing * u[2];
                for (int64_t j = 0; j < n_v; ++j) {
                    double o[3], d[3];
                    o[0] = bx + (j + 0.5) * spacing * v[0];
                    o[1] = by + (j + 0.5) * spacing * v[1];
                    o[2] = bz + (j + 0.5) * spacing * v[2];
                    d[0] = k[0]; d[1] = k[1]; d[2] = k[2];
                    for (int32_t z = 0; z < max_bounces; ++z) ids[z] = -1;
                    orc_record rec;
                    orc_trace_one(s, o, d, max_bounces, eps, strict, stack, &rec, ids, NULL);
                    const int64_t r = i * n_v + j;
                    loc[r / seg_rays] += orc_record_hash(r, ids, max_bounces, &rec);
                }
            }
#pragma omp critical
            for (int64_t q = 0; q < nseg; ++q) seg_hash[q] += loc[q];
        }
        free(stack);
        free(ids);
        free(loc);
    }
    return failed ? ORC_ENOMEM : ORC_OK;
}

/* hashes of materialised records (rays r_base + [0, n)) */
void orc_records_hash(int64_t n, int64_t r_base, int32_t max_bounces, const uint8_t *valid,
                      const double *n0, const double *path, const int32_t *bounces,
                      const uint8_t *escaped, const double *out_dir, const int32_t *ids,
                      int64_t seg_rays, uint64_t *seg_hash)
{
    for (int64_t w = 0; w < n; ++w) {
        orc_record rec;
        rec.valid = valid[w]; rec.escaped = escaped[w]; rec.bounces = bounces[w];
        rec.path = path[w];
        for (int a = 0; a < 3; ++a) { rec.n0[a] = n0[3 * w + a]; rec.out_dir[a] = out_dir[3 * w + a]; }
        const int64_t r = r_base + w;
        seg_hash[r / seg_rays] += orc_record_hash(r, ids + w * max_bounces, max_bounces, &rec);
    }
}

/* ---------------------------------------------------------------------- */
/* Tree-independence classifier.  A query is ROBUST when the */
/* linear-scan winner W (lexicographic (t, id) minimum over every accepting */
/* triangle, tests/meshes.py:51-86 brute force) has its hit point o + t d   */
/* inside W's own AABB by a relative margin of 1e-9 on every axis where the */
/* box has extent (on flat axes the ray must cross the plane, |d_k| >= 1e-9)*/
/* and no other accepting triangle has t <= t_W (1 + 1e-9).  Then every     */
/* traversal whose culling is conservative -- the reference's _traverse on  */
/* any tree (bvh.py:306-362), the GPU BVH4 kernel, the raster pass --       */
/* returns W.  A ray is robust when every query of its walk is.             */
/* ---------------------------------------------------------------------- */
static int orc_query_robust(const orc_scene *s, const double o[3], const double d[3],
                            int64_t *w_out, double *t_out)
{
    double best_t = INFINITY;
    int64_t best = -1;
    for (int64_t ti = 0; ti < s->ntri; ++ti) {
        double h = orc_tri_hit(s, ti, o[0], o[1], o[2], d[0], d[1], d[2], 0.0, best_t);
        if (h > 0.0 && (h < best_t || (h == best_t && ti < best))) {
            best_t = h;
            best = ti;
        }
    }
    *w_out = best;
    *t_out = best_t;
    if (best < 0) return 1;
    const double lim = best_t * (1.0 + 1e-9) + 1e-300;
    for (int64_t ti = 0; ti < s->ntri; ++ti) {
        if (ti == best) continue;
        double h = orc_tri_hit(s, ti, o[0], o[1], o[2], d[0], d[1], d[2], 0.0, lim);
        if (h > 0.0) return 0;     /* near-tie (edge / vertex / coplanar) */
    }
    const double *a = s->v0 + 3 * best, *b = s->v1 + 3 * best, *c = s->v2 + 3 * best;
    const double dn = fabs(d[0]) + fabs(d[1]) + fabs(d[2]);
    for (int ax = 0; ax < 3; ++ax) {
        double lo = fmin(fmin(a[ax], b[ax]), c[ax]), hi = fmax(fmax(a[ax], b[ax]), c[ax]);
        if (s->single) {   /* bvh.py:286-290 boxes of float32 meshes */
            lo = (double)nextafterf((float)lo, -INFINITY);
            hi = (double)nextafterf((float)hi, INFINITY);
        }
        const double hp = o[ax] + best_t * d[ax];
        const double mu = 1e-9 * (fabs(lo) + fabs(hi) + fabs(o[ax]) + fabs(best_t * d[ax])) + 1e-300;
        if (hi - lo > 2.0 * mu) {
            if (!(hp >= lo + mu && hp <= hi - mu)) return 0;
        } else {
            if (!(fabs(d[ax]) >= 1e-9 * dn)) return 0;
            if (!(fabs(hp - 0.5 * (lo + hi)) <= mu + 0.5 * (hi - lo))) return 0;
        }
    }
    return 1;
}

/* per ray of rows [i_begin, i_end): robust[r] = 1 if every query of the
 * walk (transport.py:276-327, driven by the linear-scan winners) is robust;
 * prim_tri / prim_t (optional): the linear-scan answer of query 0 */
int orc_classify_grid(const orc_scene *s, const double corner[3], const double u[3],
                      const double v[3], const double k[3], double spacing,
                      int64_t n_v, int64_t i_begin, int64_t i_end, int32_t max_bounces,
                      double eps, int32_t strict, uint8_t *robust, int64_t *prim_tri,
                      double *prim_t, int nthreads)
{
    int nt = orc_threads(nthreads);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 16)
    for (int64_t r = i_begin * n_v; r < i_end * n_v; ++r) {
        const int64_t i = r / n_v, j = r - i * n_v, slot = r - i_begin * n_v;
        double o[3], d[3];
        for (int a = 0; a < 3; ++a) {
            double bx = corner[a] + (i + 0.5) * spacing * u[a];
            o[a] = bx + (j + 0.5) * spacing * v[a];
            d[a] = k[a];
        }
        int ok = 1, bounces = 0, valid = 0, escaped = 0;
        for (int32_t it = 0; it < max_bounces && ok; ++it) {
            int64_t tri;
            double t;
            ok = orc_query_robust(s, o, d, &tri, &t);
            if (it == 0) {
                if (prim_tri) prim_tri[slot] = tri;
                if (prim_t) prim_t[slot] = t;
            }
            if (!ok) break;
            if (tri < 0) { escaped = 1; break; }
            const double *nn = s->normals + 3 * tri;
            double nx = nn[0], ny = nn[1], nz = nn[2];
            double nd = nx * d[0] + ny * d[1] + nz * d[2];
            if (nd > 0.0) {
                if (strict && bounces == 0) { escaped = 1; valid = 0; break; }
                nx = -nx; ny = -ny; nz = -nz; nd = -nd;
            }
            double hx = o[0] + t * d[0], hy = o[1] + t * d[1], hz = o[2] + t * d[2];
            bounces += 1;
            valid = 1;
            d[0] -= 2.0 * nd * nx;
            d[1] -= 2.0 * nd * ny;
            d[2] -= 2.0 * nd * nz;
            o[0] = hx + eps * nx;
            o[1] = hy + eps * ny;
            o[2] = hz + eps * nz;
        }
        if (ok && valid && !escaped) {
            int64_t tri;
            double t;
            ok = orc_query_robust(s, o, d, &tri, &t);
        }
        robust[slot] = (uint8_t)ok;
    }
    return ORC_OK;
}

/* single queries (closest_hit_batch rays) */
int orc_classify_rays(const orc_scene *s, const double *o, const double *d, int64_t n,
                      uint8_t *robust, int nthreads)
{
    int nt = orc_threads(nthreads);
#pragma omp parallel for num_threads(nt) schedule(dynamic, 16)
    for (int64_t r = 0; r < n; ++r) {
        int64_t tri;
        double t;
        robust[r] = (uint8_t)orc_query_robust(s, o + 3 * r, d + 3 * r, &tri, &t);
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* po.py:59-80  pairwise_sum : adjacent-pair tree, odd tail carried          */
/* ---------------------------------------------------------------------- */
void orc_pairwise_sum(double *work /* (n,2) in/out scratch */, int64_t n,
                      double out[2])
{
    if (n == 0) { out[0] = 0.0; out[1] = 0.0; return; }
    while (n > 1) {
        int64_t half = n / 2;
        for (int64_t i = 0; i < half; ++i) {
            double re = work[4 * i] + work[4 * i + 2];
            double im = work[4 * i + 1] + work[4 * i + 3];
            work[2 * i] = re;
            work[2 * i + 1] = im;
        }
        if (n % 2) {
            work[2 * half] = work[2 * (n - 1)];
            work[2 * half + 1] = work[2 * (n - 1) + 1];
            n = half + 1;
        } else {
            n = half;
        }
    }
    out[0] = work[0];
    out[1] = work[1];
}

/* ---------------------------------------------------------------------- */
/* po.py:83-113  accumulate : selection (compaction) + PO terms + pairwise   */
/* Returns ORC_OK, or 4 (NumericalError) with *bad_index set.               */
/* ---------------------------------------------------------------------- */
int orc_accumulate(const uint8_t *valid, const double *n0, const double *path,
                   const int32_t *bounces, const uint8_t *escaped, int64_t n,
                   const double k_inc[3], double k, double cell_area,
                   double gamma, int32_t count_trapped, double out[2],
                   int64_t *bad_index)
{
    double *work = (double *)malloc(sizeof(double) * 2 * (size_t)(n > 0 ? n : 1));
    if (!work) return ORC_ENOMEM;
    /* coef = 1j * k * dA / (4 pi); coef * 2.0 -> (0, (k*dA/(4pi))*2) */
    double cim = k * cell_area / (4.0 * M_PI);
    int64_t m = 0;
    *bad_index = -1;
    for (int64_t r = 0; r < n; ++r) {
        if (!valid[r]) continue;
        if (!count_trapped && !escaped[r]) continue;
        double c = -(n0[3 * r] * k_inc[0] + n0[3 * r + 1] * k_inc[1]
                     + n0[3 * r + 2] * k_inc[2]);
        if (!(c > 0.0)) continue;
        /* (coef*2.0) * cos * gamma**N * exp(-2j k R) */
        double a = cim * 2.0 * c * pow(gamma, (double)bounces[r]);
        double ph = -2.0 * k * path[r];
        double re = -a * sin(ph);   /* j*a*(cos ph + j sin ph) = (-a sin, a cos) */
        double im = a * cos(ph);
        if (!isfinite(re) || !isfinite(im)) {
            *bad_index = r;
            free(work);
            return 4;
        }
        work[2 * m] = re;
        work[2 * m + 1] = im;
        ++m;
    }
    orc_pairwise_sum(work, m, out);
    free(work);
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* bvh.py:124-299  build : median / binned-SAH recursive preorder emit       */
/* ---------------------------------------------------------------------- */
typedef struct {
    const double *tmin, *tmax, *cent;  /* (T,3) */
    int split_sah, n_leaf, bins, max_depth;
    double c_t, c_i;
    double *nmin, *nmax;
    int32_t *first, *count, *order;
    int64_t nn, cursor;
    int32_t depth_seen;
    int64_t *scratch;                   /* T entries */
    double *keys;                       /* T entries */
    int32_t *bin_of;                    /* T entries */
} orc_builder;

static double orc_sa(const double lo[3], const double hi[3])
{
    double d0 = hi[0] - lo[0], d1 = hi[1] - lo[1], d2 = hi[2] - lo[2];
    return 2.0 * (d0 * d1 + d1 * d2 + d2 * d0);
}

/* stable merge sort of idx[0..n) by keys[pos] (ties keep position order);
 * equivalent to np.lexsort((arange(n), c[:, axis])) in bvh.py:149 */
static void orc_msort(int64_t *idx, double *key, int64_t n, int64_t *tmpi,
                      double *tmpk)
{
    if (n < 2) return;
    int64_t h = n / 2;
    orc_msort(idx, key, h, tmpi, tmpk);
    orc_msort(idx + h, key + h, n - h, tmpi, tmpk);
    int64_t i = 0, j = h, o = 0;
    while (i < h && j < n) {
        if (key[j] < key[i]) { tmpi[o] = idx[j]; tmpk[o++] = key[j++]; }
        else                 { tmpi[o] = idx[i]; tmpk[o++] = key[i++]; }
    }
    while (i < h) { tmpi[o] = idx[i]; tmpk[o++] = key[i++]; }
    while (j < n) { tmpi[o] = idx[j]; tmpk[o++] = key[j++]; }
    memcpy(idx, tmpi, sizeof(int64_t) * (size_t)n);
    memcpy(key, tmpk, sizeof(double) * (size_t)n);
}

/* bvh.py:154-215 binned_sah_split; returns 1 and partitions idx in place
 * (left block first, both order-preserving) with *nl set, else 0. */
static int orc_sah_split(orc_builder *B, int64_t *idx, int64_t n,
                         const double box_lo[3], const double box_hi[3],
                         int64_t *nl_out)
{
    int nb = B->bins;
    double sa_p = orc_sa(box_lo, box_hi);
    if (sa_p < 1e-300) sa_p = 1e-300;
    int have = 0, best_axis = -1, best_b = -1;
    double best_cost = 0.0;
    int64_t *cnt = (int64_t *)calloc((size_t)nb, sizeof(int64_t));
    double *bmin = (double *)malloc(sizeof(double) * 3 * (size_t)nb);
    double *bmax = (double *)malloc(sizeof(double) * 3 * (size_t)nb);
    double *lmin = (double *)malloc(sizeof(double) * 3 * (size_t)nb);
    double *lmax = (double *)malloc(sizeof(double) * 3 * (size_t)nb);
    double *rmin = (double *)malloc(sizeof(double) * 3 * (size_t)nb);
    double *rmax = (double *)malloc(sizeof(double) * 3 * (size_t)nb);
    int64_t *ln = (int64_t *)malloc(sizeof(int64_t) * (size_t)nb);
    int64_t *rn = (int64_t *)malloc(sizeof(int64_t) * (size_t)nb);
    double best_scale = 0.0, best_lo = 0.0;
    for (int axis = 0; axis < 3; ++axis) {
        double c_lo = INFINITY, c_hi = -INFINITY;
        for (int64_t i = 0; i < n; ++i) {
            double c = B->cent[3 * idx[i] + axis];
            if (c < c_lo) c_lo = c;
            if (c > c_hi) c_hi = c;
        }
        if (c_hi <= c_lo) continue;
        double scale = nb / (c_hi - c_lo);
        memset(cnt, 0, sizeof(int64_t) * (size_t)nb);
        for (int q = 0; q < 3 * nb; ++q) { bmin[q] = INFINITY; bmax[q] = -INFINITY; }
        for (int64_t i = 0; i < n; ++i) {
            int64_t t = idx[i];
            int64_t bi = (int64_t)(scale * (B->cent[3 * t + axis] - c_lo));
            if (bi > nb - 1) bi = nb - 1;
            cnt[bi]++;
            for (int a = 0; a < 3; ++a) {
                if (B->tmin[3 * t + a] < bmin[3 * bi + a]) bmin[3 * bi + a] = B->tmin[3 * t + a];
                if (B->tmax[3 * t + a] > bmax[3 * bi + a]) bmax[3 * bi + a] = B->tmax[3 * t + a];
            }
        }
        /* prefix / suffix sweeps (np.cumsum / minimum.accumulate) */
        int64_t acc = 0;
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int b = 0; b < nb; ++b) {
            acc += cnt[b];
            for (int a = 0; a < 3; ++a) {
                if (bmin[3 * b + a] < lo[a]) lo[a] = bmin[3 * b + a];
                if (bmax[3 * b + a] > hi[a]) hi[a] = bmax[3 * b + a];
                lmin[3 * b + a] = lo[a]; lmax[3 * b + a] = hi[a];
            }
            ln[b] = acc;
        }
        acc = 0;
        double rlo[3] = {INFINITY, INFINITY, INFINITY}, rhi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int b = nb - 1; b >= 0; --b) {
            acc += cnt[b];
            for (int a = 0; a < 3; ++a) {
                if (bmin[3 * b + a] < rlo[a]) rlo[a] = bmin[3 * b + a];
                if (bmax[3 * b + a] > rhi[a]) rhi[a] = bmax[3 * b + a];
                rmin[3 * b + a] = rlo[a]; rmax[3 * b + a] = rhi[a];
            }
            rn[b] = acc;
        }
        for (int b = 0; b < nb - 1; ++b) {
            int64_t nl = ln[b], nr = rn[b + 1];
            if (nl == 0 || nr == 0) continue;
            double sal = orc_sa(lmin + 3 * b, lmax + 3 * b);
            double sar = orc_sa(rmin + 3 * (b + 1), rmax + 3 * (b + 1));
            /* bvh.py:124-127 sah_cost, left-to-right association */
            double cost = B->c_t + (sal / sa_p) * (double)nl * B->c_i
                          + (sar / sa_p) * (double)nr * B->c_i;
            if (!have || cost < best_cost) {
                have = 1; best_cost = cost; best_axis = axis; best_b = b;
                best_scale = scale; best_lo = c_lo;
            }
        }
    }
    free(cnt); free(bmin); free(bmax); free(lmin); free(lmax);
    free(rmin); free(rmax); free(ln); free(rn);
    if (!have) return 0;
    if (best_cost >= (double)n * B->c_i && n <= 4 * (int64_t)B->n_leaf) return 0;
    /* stable partition by bin <= boundary */
    int64_t *tmp = B->scratch;
    int64_t nl = 0, nr = 0;
    for (int64_t i = 0; i < n; ++i) {
        int64_t t = idx[i];
        int64_t bi = (int64_t)(best_scale * (B->cent[3 * t + best_axis] - best_lo));
        if (bi > nb - 1) bi = nb - 1;
        if (bi <= best_b) idx[nl++] = t; else tmp[nr++] = t;
    }
    memcpy(idx + nl, tmp, sizeof(int64_t) * (size_t)nr);
    *nl_out = nl;
    return 1;
}

/* bvh.py:135-151 median_split */
static int orc_median_split(orc_builder *B, int64_t *idx, int64_t n,
                            const double box_lo[3], const double box_hi[3],
                            int64_t *nl_out)
{
    int all_same = 1;
    const double *c0 = B->cent + 3 * idx[0];
    for (int64_t i = 1; i < n && all_same; ++i) {
        const double *c = B->cent + 3 * idx[i];
        if (c[0] != c0[0] || c[1] != c0[1] || c[2] != c0[2]) all_same = 0;
    }
    if (all_same) return 0;
    int axis = 0;
    double ext0 = box_hi[0] - box_lo[0], ext1 = box_hi[1] - box_lo[1],
           ext2 = box_hi[2] - box_lo[2];
    double best = ext0;
    if (ext1 > best) { best = ext1; axis = 1; }
    if (ext2 > best) { axis = 2; }
    double *key = B->keys;
    for (int64_t i = 0; i < n; ++i) key[i] = B->cent[3 * idx[i] + axis];
    double *tmpk = (double *)malloc(sizeof(double) * (size_t)n);
    orc_msort(idx, key, n, B->scratch, tmpk);
    free(tmpk);
    *nl_out = n / 2;
    return 1;
}

static int64_t orc_emit(orc_builder *B, int64_t *idx, int64_t n, int depth)
{
    if (depth > B->depth_seen) B->depth_seen = depth;
    int64_t me = B->nn++;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a) {
            double x = B->tmin[3 * idx[i] + a], y = B->tmax[3 * idx[i] + a];
            if (x < lo[a]) lo[a] = x;
            if (y > hi[a]) hi[a] = y;
        }
    }
    for (int a = 0; a < 3; ++a) { B->nmin[3 * me + a] = lo[a]; B->nmax[3 * me + a] = hi[a]; }
    int64_t nl = 0;
    int split = 0;
    if (n > B->n_leaf && depth < B->max_depth) {
        split = B->split_sah ? orc_sah_split(B, idx, n, lo, hi, &nl)
                             : orc_median_split(B, idx, n, lo, hi, &nl);
    }
    if (!split) {
        B->first[me] = (int32_t)B->cursor;
        B->count[me] = (int32_t)n;
        for (int64_t i = 0; i < n; ++i) B->order[B->cursor + i] = (int32_t)idx[i];
        B->cursor += n;
    } else {
        orc_emit(B, idx, nl, depth + 1);
        int64_t right = orc_emit(B, idx + nl, n - nl, depth + 1);
        B->first[me] = (int32_t)right;
        B->count[me] = 0;
    }
    return me;
}

/* Output arrays must hold 2*ntri-1 nodes.  single=1 applies the float32
 * outward nextafter rounding of bvh.py:286-290. */
int orc_build(const double *v0, const double *v1, const double *v2, int64_t ntri,
              int32_t split_sah, int32_t n_leaf, int32_t bins, double c_t,
              double c_i, int32_t max_depth, int32_t single,
              double *nmin, double *nmax, int32_t *first, int32_t *count,
              int32_t *order, int64_t *nnodes, int32_t *depth_seen)
{
    if (ntri < 1) return ORC_EINVAL;
    double *tmin = (double *)malloc(sizeof(double) * 3 * (size_t)ntri);
    double *tmax = (double *)malloc(sizeof(double) * 3 * (size_t)ntri);
    double *cent = (double *)malloc(sizeof(double) * 3 * (size_t)ntri);
    int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)ntri);
    int64_t *scratch = (int64_t *)malloc(sizeof(int64_t) * (size_t)ntri);
    double *keys = (double *)malloc(sizeof(double) * (size_t)ntri);
    if (!tmin || !tmax || !cent || !idx || !scratch || !keys) return ORC_ENOMEM;
    for (int64_t t = 0; t < ntri; ++t) {
        for (int a = 0; a < 3; ++a) {
            double x = v0[3 * t + a], y = v1[3 * t + a], z = v2[3 * t + a];
            double lo = fmin(fmin(x, y), z), hi = fmax(fmax(x, y), z);
            tmin[3 * t + a] = lo; tmax[3 * t + a] = hi;
            cent[3 * t + a] = (lo + hi) * 0.5;
        }
        idx[t] = t;
    }
    orc_builder B = {tmin, tmax, cent, split_sah, n_leaf, bins, max_depth, c_t, c_i,
                     nmin, nmax, first, count, order, 0, 0, 0, scratch, keys, NULL};
    orc_emit(&B, idx, ntri, 0);
    if (single) {
        for (int64_t q = 0; q < 3 * B.nn; ++q) {
            nmin[q] = (double)nextafterf((float)nmin[q], -INFINITY);
            nmax[q] = (double)nextafterf((float)nmax[q], INFINITY);
        }
    }
    *nnodes = B.nn;
    *depth_seen = B.depth_seen;
    free(tmin); free(tmax); free(cent); free(idx); free(scratch); free(keys);
    return ORC_OK;
}

/* geometry.py:394-409 ray_triangle_intersect over independent (ray, tri)
 * pairs: tri r is (v0[r], v1[r], v2[r]).  Returns t or -1 per pair. */
int orc_tri_hit_pairs(const double *v0, const double *v1, const double *v2,
                      const double *o, const double *d, int64_t n,
                      double t_min, double t_max, int32_t single, double *t)
{
    orc_scene s;
    memset(&s, 0, sizeof(s));
    s.v0 = v0; s.v1 = v1; s.v2 = v2; s.ntri = n; s.single = single;
    for (int64_t r = 0; r < n; ++r)
        t[r] = orc_tri_hit(&s, r, o[3 * r], o[3 * r + 1], o[3 * r + 2],
                           d[3 * r], d[3 * r + 1], d[3 * r + 2], t_min, t_max);
    return ORC_OK;
}
