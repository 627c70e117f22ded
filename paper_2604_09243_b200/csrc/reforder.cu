// reforder.cu -- reference-order traversal: bvh.py:306-362 _traverse replayed
// operation by operation on the reference tree.
//
// The fast path (raster pass + k_trace_persistent) returns, for every query,
// the lexicographic (t, id) minimum over the triangles its conservative
// culling reaches.  That equals the reference whenever the winning
// triangle's hit point lies robustly inside its own box and no other
// accepting triangle ties it within rounding (then EVERY
// conservative traversal, the reference's included, returns it).  For the
// remaining rays -- near-edge-on triangles whose rounding-dominated
// Moller-Trumbore determinant accepts rays outside the triangle's box, and
// edge/vertex near-ties -- the reference's own answer depends on its tree and
// its visit order (bvh.py:329-342: slab tests against best_t).  This mode
// reproduces that order exactly, so it matches the reference bit for bit on
// every ray, those included:
//   * the reference-layout tree (nodes_min/max FP64, node_first/count,
//     tri_order) of a GPU SAH/median build or an upload, triangles in
//     original order;
//   * _aabb_hit (geometry.py:358-391) in FP64: inv = 1/d (inf for d == 0),
//     the parallel-slab rule, t1/t2 swap, entry clamped at 0, culling
//     against best_t; float32 meshes' boxes rounded outward to float32 as
//     bvh.py:286-290 does;
//   * children pushed far-first with the e_l <= e_r tie rule, explicit
//     int32 stack (bvh.py:338-360);
//   * the exact FP64 Moller-Trumbore (sbr_device.cuh tri_hit_exact).
// One thread per ray, no persistence: this is the validation / tie-exact
// mode (sbr_ctx_set_traversal), not the throughput path.
#include "pipeline.h"

namespace sbr {

constexpr int kRefStack = 256;   // entries; the reference needs max_depth_seen + 1

__device__ __forceinline__ double ref_plane(const RefView &V, const double *a, int64_t i,
                                            bool lo)
{
    const double x = __ldg(a + i);
    if (!V.round_f32) return x;
    const float f = __double2float_rn(x);
    return (double)nextafterf(f, lo ? -INFINITY : INFINITY);
}

// geometry.py:358-391 _aabb_hit
__device__ __forceinline__ bool ref_box(const RefView &V, int64_t ni, const double o[3],
                                        const double inv[3], const bool par[3], double t_max,
                                        double &entry)
{
    double t_near = 0.0, t_far = t_max;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        const double lo = ref_plane(V, V.nmin, 3 * ni + ax, true);
        const double hi = ref_plane(V, V.nmax, 3 * ni + ax, false);
        if (par[ax]) {
            if (o[ax] < lo || o[ax] > hi) return false;
        } else {
            double t1 = DM(DS(lo, o[ax]), inv[ax]);
            double t2 = DM(DS(hi, o[ax]), inv[ax]);
            if (t1 > t2) {
                const double tmp = t1;
                t1 = t2;
                t2 = tmp;
            }
            if (t1 > t_near) t_near = t1;
            if (t2 < t_far) t_far = t2;
            if (t_near > t_far) return false;
        }
    }
    entry = t_near;
    return true;
}

__device__ __forceinline__ TriF64 ref_tri(const RefView &V, int ti)
{
    const double *p = V.verts + 9 * (int64_t)ti;
    TriF64 T;
    T.ax = __ldg(p); T.ay = __ldg(p + 1); T.az = __ldg(p + 2);
    if (V.single) {   // float32 arrays subtract in float32
        T.e1x = __fsub_rn((float)__ldg(p + 3), (float)T.ax);
        T.e1y = __fsub_rn((float)__ldg(p + 4), (float)T.ay);
        T.e1z = __fsub_rn((float)__ldg(p + 5), (float)T.az);
        T.e2x = __fsub_rn((float)__ldg(p + 6), (float)T.ax);
        T.e2y = __fsub_rn((float)__ldg(p + 7), (float)T.ay);
        T.e2z = __fsub_rn((float)__ldg(p + 8), (float)T.az);
    } else {
        T.e1x = DS(__ldg(p + 3), T.ax); T.e1y = DS(__ldg(p + 4), T.ay);
        T.e1z = DS(__ldg(p + 5), T.az);
        T.e2x = DS(__ldg(p + 6), T.ax); T.e2y = DS(__ldg(p + 7), T.ay);
        T.e2z = DS(__ldg(p + 8), T.az);
    }
    T.id = ti;
    return T;
}

// bvh.py:306-362 _traverse: (triangle or -1, t, visits)
__device__ int ref_traverse(const RefView &V, const double o[3], const double d[3], double t_min,
                            double t_max, int *stack, double &t_out, int64_t &visits,
                            bool f32rays = false)
{
    double best_t = t_max;
    int best = -1;
    int64_t vis = 0;
    double inv[3];
    bool par[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        inv[a] = d[a] != 0.0 ? __drcp_rn(d[a]) : __longlong_as_double(0x7ff0000000000000LL);
        par[a] = isinf(inv[a]);   // bvh.py: inv == +-inf (also 1/subnormal overflow)
    }
    stack[0] = 0;
    int sp = 1;
    while (sp > 0) {
        const int node = stack[--sp];
        ++vis;
        double entry;
        if (!ref_box(V, node, o, inv, par, best_t, entry) || entry > best_t) continue;
        const int cnt = __ldg(V.count + node);
        if (cnt > 0) {
            const int first = __ldg(V.first + node);
            for (int k = first; k < first + cnt; ++k) {
                const int ti = __ldg(V.order + k);
                const TriF64 T = ref_tri(V, ti);
                const double t =
                    f32rays ? tri_hit_f32rays(T, o[0], o[1], o[2], d[0], d[1], d[2], t_min, best_t)
                            : tri_hit_exact(T, o[0], o[1], o[2], d[0], d[1], d[2], t_min, best_t);
                if (t > 0.0 && (t < best_t || (t == best_t && ti < best))) {
                    best_t = t;
                    best = ti;
                }
            }
        } else {
            const int left = node + 1, right = __ldg(V.first + node);
            double el = 0.0, er = 0.0;
            const bool hl = ref_box(V, left, o, inv, par, best_t, el);
            const bool hr = ref_box(V, right, o, inv, par, best_t, er);
            if (hl && hr) {
                if (el <= er) {
                    stack[sp++] = right;
                    stack[sp++] = left;
                } else {
                    stack[sp++] = left;
                    stack[sp++] = right;
                }
            } else if (hl) {
                stack[sp++] = left;
            } else if (hr) {
                stack[sp++] = right;
            }
        }
    }
    t_out = best_t;
    visits = vis;
    return best;
}

__global__ void k_closest_ref(RefView V, const double *orig, const double *dirs, int64_t n,
                              double t_min, double t_max, int64_t *tri, double *t_out,
                              int64_t *visits)
{
    int stack[kRefStack];
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        // float32 mesh: closest_hit_batch casts the rays to float32 too
        auto f = [&](double x) { return V.single ? (double)__double2float_rn(x) : x; };
        const double o[3] = {f(orig[3 * r]), f(orig[3 * r + 1]), f(orig[3 * r + 2])};
        const double d[3] = {f(dirs[3 * r]), f(dirs[3 * r + 1]), f(dirs[3 * r + 2])};
        double t;
        int64_t vis;
        const int b = ref_traverse(V, o, d, t_min, t_max, stack, t, vis, V.single != 0);
        tri[r] = b;
        t_out[r] = t;
        if (visits) visits[r] = vis;
    }
}

// transport.py:276-327 _trace_one over ref_traverse (same FP64 operation
// sequence as k_trace_persistent's query completion)
template <int MODE>
__global__ void k_trace_ref(RefView V, TraceCfg cfg, const GridDev *grids, const UnitDev *units,
                            int n_units, const double *orig, const double *dirs, int64_t n,
                            int64_t r_base, FullOut full, SlotRec *slots)
{
    int stack[kRefStack];
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < n;
         w += (int64_t)gridDim.x * blockDim.x) {
        double o[3], d[3];
        int64_t r = w;
        if (MODE == kModeSolve) {
            const int ui = find_unit(units, n_units, w);
            const UnitDev U = units[ui];
            r = U.ray_begin + (w - U.slot_base);
            const GridDev &G = grids[U.grid];
            bool real = r < U.ray_end;
            if (real && !(cfg.allow_aliasing || !(G.spacing > cfg.spacing_limit))) {
                atomicOr(cfg.error_flag, 1u);
                real = false;
            }
            if (!real) {
                SlotRec z;
                z.R = 0.0; z.cosv = 0.f; z.meta = 0u;
                slots[w] = z;
                continue;
            }
            grid_origin(G, r, o[0], o[1], o[2]);
            d[0] = G.k[0]; d[1] = G.k[1]; d[2] = G.k[2];
        } else if (MODE == kModeGrid) {
            r = w + r_base;
            grid_origin(*grids, r, o[0], o[1], o[2]);
            d[0] = grids->k[0]; d[1] = grids->k[1]; d[2] = grids->k[2];
        } else {
            for (int a = 0; a < 3; ++a) {
                o[a] = orig[3 * w + a];
                d[a] = dirs[3 * w + a];
            }
        }
        const bool hash = MODE != kModeSolve && full.seg_hash;
        int32_t *ids = (MODE != kModeSolve && !hash && full.ids)
                           ? full.ids + w * (int64_t)cfg.max_bounces
                           : nullptr;
        if (ids)
            for (int b = 0; b < cfg.max_bounces; ++b) ids[b] = -1;
        unsigned long long hid = hash ? hash_mix((unsigned long long)r) : 0ULL;
        double path = 0.0, n0x = 0.0, n0y = 0.0, n0z = 0.0, cosd = 0.0;
        int bounces = 0;
        bool valid = false, escaped = false, strict_out = false;
        for (int it = 0; it < cfg.max_bounces; ++it) {
            double t;
            int64_t vis;
            const int tri = ref_traverse(V, o, d, 0.0, inf, stack, t, vis);
            if (tri < 0) {
                escaped = true;
                break;
            }
            const double *nn = cfg.B.normals + 3 * (int64_t)tri;
            double nx = __ldg(nn), ny = __ldg(nn + 1), nz = __ldg(nn + 2);
            double nd = DA(DA(DM(nx, d[0]), DM(ny, d[1])), DM(nz, d[2]));
            if (nd > 0.0) {
                if (cfg.strict && bounces == 0) {   // transport.py:306-307
                    strict_out = true;
                    break;
                }
                nx = -nx; ny = -ny; nz = -nz; nd = -nd;
            }
            if (ids) ids[it] = tri;
            if (hash) hid = hash_mix(hid ^ (unsigned long long)(unsigned int)tri);
            const double hx = DA(o[0], DM(t, d[0])), hy = DA(o[1], DM(t, d[1])),
                         hz = DA(o[2], DM(t, d[2]));
            path = DA(path, t);
            bounces += 1;
            if (bounces == 1) {
                n0x = nx; n0y = ny; n0z = nz;
                cosd = -nd;
                valid = true;
            }
            const double s = DM(2.0, nd);
            d[0] = DS(d[0], DM(s, nx));
            d[1] = DS(d[1], DM(s, ny));
            d[2] = DS(d[2], DM(s, nz));
            o[0] = DA(hx, DM(cfg.eps, nx));
            o[1] = DA(hy, DM(cfg.eps, ny));
            o[2] = DA(hz, DM(cfg.eps, nz));
        }
        if (strict_out) {
            valid = false;
            bounces = 0;
            path = 0.0;
            n0x = n0y = n0z = 0.0;
            escaped = true;
        } else if (valid && !escaped) {   // escape probe (transport.py:319-326)
            double t;
            int64_t vis;
            escaped = ref_traverse(V, o, d, 0.0, inf, stack, t, vis) < 0;
        }
        if (MODE == kModeSolve) {
            const double c = valid ? cosd : 0.0;
            const bool sel = valid && (escaped || cfg.count_trapped) && c > 0.0;
            SlotRec rec;
            rec.R = path;
            rec.cosv = (float)c;
            rec.meta = (uint32_t)bounces | kMetaActive | (valid ? kMetaValid : 0u) |
                       (escaped ? kMetaEscaped : 0u) | (sel ? kMetaSel : 0u);
            slots[w] = rec;
        } else if (hash) {
            const unsigned long long h = record_hash(hid, bounces, cfg.max_bounces, valid,
                                                     escaped, n0x, n0y, n0z, path, d[0], d[1],
                                                     d[2]);
            atomicAdd(full.seg_hash + r / full.seg_rays, h);
        } else {
            full.valid[w] = valid ? 1 : 0;
            full.escaped[w] = escaped ? 1 : 0;
            full.bounces[w] = bounces;
            full.path[w] = path;
            full.n0[3 * w] = n0x; full.n0[3 * w + 1] = n0y; full.n0[3 * w + 2] = n0z;
            full.out_dir[3 * w] = d[0]; full.out_dir[3 * w + 1] = d[1];
            full.out_dir[3 * w + 2] = d[2];
        }
    }
}

static int ref_blocks(int64_t n)
{
    const int64_t want = (n + 127) / 128;
    return (int)(want < 65535 ? (want > 0 ? want : 1) : 65535);
}

cudaError_t launch_closest_ref(const RefView &V, const double *d_orig, const double *d_dirs,
                               int64_t n, double t_min, double t_max, int64_t *d_tri,
                               double *d_t, int64_t *d_visits, cudaStream_t st,
                               const LaunchStats &ls)
{
    if (n == 0) return cudaSuccess;
    k_closest_ref<<<ref_blocks(n), 128, 0, st>>>(V, d_orig, d_dirs, n, t_min, t_max, d_tri, d_t,
                                                 d_visits);
    ++*ls.launches;
    return cudaGetLastError();
}

cudaError_t launch_trace_ref(const RefView &V, const TraceCfg &cfg, const GridDev *d_grids,
                             const double *d_orig, const double *d_dirs, int64_t n,
                             int64_t r_base, const FullOut &out, const UnitDev *d_units,
                             SlotRec *d_slots, int n_units, cudaStream_t st,
                             const LaunchStats &ls)
{
    if (n == 0) return cudaSuccess;
    const int nb = ref_blocks(n);
    if (d_slots)
        k_trace_ref<kModeSolve><<<nb, 128, 0, st>>>(V, cfg, d_grids, d_units, n_units, nullptr,
                                                   nullptr, n, 0, out, d_slots);
    else if (d_grids)
        k_trace_ref<kModeGrid><<<nb, 128, 0, st>>>(V, cfg, d_grids, nullptr, 0, nullptr, nullptr,
                                                  n, r_base, out, nullptr);
    else
        k_trace_ref<kModeList><<<nb, 128, 0, st>>>(V, cfg, nullptr, nullptr, 0, d_orig, d_dirs,
                                                  n, 0, out, nullptr);
    ++*ls.launches;
    return cudaGetLastError();
}

}  // namespace sbr
