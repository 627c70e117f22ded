// traverse.cuh -- closest-hit / any-hit BVH traversal and the multi-bounce
// ray walk, as device functions shared by every trace kernel.
//
// Reference semantics:
//   closest_hit()  == bvh.py:306-362 _traverse (result only; the visit
//                     count is this tree's node fetches);
//   trace_ray_walk == transport.py:276-327 _trace_one, operation for
//                     operation in FP64 round-to-nearest intrinsics.
#pragma once

#include "sbr_device.cuh"

namespace sbr {

struct StackEntry {
    int ref;
    float tn;
};

// Closest hit in (t_min, best_t]; best_t is in/out.  Returns the original
// triangle id or -1.  ANY: stop at the first accepted triangle (escape
// probe, transport.py:319-326, only needs hit / no hit).
template <int STORAGE, bool ANY>
__device__ __forceinline__ int closest_hit(const BvhView &B, double ox, double oy,
                                           double oz, double dx, double dy,
                                           double dz, double t_min,
                                           double &best_t, int &visits)
{
    StackEntry stack[kStack];
    int sp = 0;
    const RayBox rb = make_raybox(B, ox, oy, oz, dx, dy, dz);
    float tmax = __double2float_ru(best_t);
    int best = -1;
    int ref = B.root;
    while (true) {
        if (ref >= 0) {
            ++visits;
            int rr[4];
            float tt[4];
            const int n = node4_visit(B.nodes4 + ref, rb, tmax, rr, tt);
            if (n > 0) {
#pragma unroll
                for (int c = 3; c >= 1; --c)
                    if (c < n) {
                        stack[sp].ref = rr[c];
                        stack[sp].tn = tt[c];
                        ++sp;
                    }
                ref = rr[0];
                continue;
            }
        } else {
            ++visits;
            const int first = leaf_first(ref), cnt = leaf_count(ref);
            for (int k = first; k < first + cnt; ++k) {
                TriF64 T = load_tri<STORAGE>(B, k);
                double t = tri_hit_exact(T, ox, oy, oz, dx, dy, dz, t_min, best_t);
                if (t > 0.0 && (t < best_t || (t == best_t && T.id < best))) {
                    best_t = t;
                    best = T.id;
                    tmax = __double2float_ru(t);
                    if (ANY) return best;
                }
            }
        }
        // pop the next node whose entry distance is still within best_t
        bool found = false;
        while (sp > 0) {
            --sp;
            if (stack[sp].tn <= tmax) {
                ref = stack[sp].ref;
                found = true;
                break;
            }
        }
        if (!found) break;
    }
    return best;
}

struct RayResult {
    bool valid, escaped;
    int bounces;
    double n0x, n0y, n0z, path, dx, dy, dz;
    int queries;
};

// transport.py:276-327.  ids (optional, stride 1) receives the hit
// triangle of every accepted bounce.
template <int STORAGE>
__device__ __forceinline__ RayResult trace_ray_walk(const BvhView &B, double ox,
                                                    double oy, double oz,
                                                    double dx, double dy,
                                                    double dz, int max_bounces,
                                                    double eps, bool strict,
                                                    int *ids, int &visits)
{
    RayResult R;
    R.valid = false; R.escaped = false; R.bounces = 0;
    R.n0x = R.n0y = R.n0z = 0.0; R.path = 0.0; R.queries = 0;
    for (int it = 0; it < max_bounces; ++it) {
        double t = __longlong_as_double(0x7ff0000000000000LL);  // +inf
        ++R.queries;
        int tri = closest_hit<STORAGE, false>(B, ox, oy, oz, dx, dy, dz, 0.0, t, visits);
        if (tri < 0) { R.escaped = true; break; }
        const double *n = B.normals + 3 * (int64_t)tri;
        double nx = __ldg(n), ny = __ldg(n + 1), nz = __ldg(n + 2);
        double nd = DA(DA(DM(nx, dx), DM(ny, dy)), DM(nz, dz));
        if (nd > 0.0) {
            if (strict && R.bounces == 0) {
                R.valid = false; R.escaped = true; R.bounces = 0;
                R.n0x = R.n0y = R.n0z = 0.0; R.path = 0.0;
                R.dx = dx; R.dy = dy; R.dz = dz;
                return R;
            }
            nx = -nx; ny = -ny; nz = -nz; nd = -nd;
        }
        if (ids) ids[it] = tri;
        double hx = DA(ox, DM(t, dx)), hy = DA(oy, DM(t, dy)), hz = DA(oz, DM(t, dz));
        R.path = DA(R.path, t);
        R.bounces += 1;
        if (R.bounces == 1) { R.n0x = nx; R.n0y = ny; R.n0z = nz; R.valid = true; }
        double s = DM(2.0, nd);
        dx = DS(dx, DM(s, nx));
        dy = DS(dy, DM(s, ny));
        dz = DS(dz, DM(s, nz));
        ox = DA(hx, DM(eps, nx));
        oy = DA(hy, DM(eps, ny));
        oz = DA(hz, DM(eps, nz));
    }
    if (R.valid && !R.escaped) {
        double t = __longlong_as_double(0x7ff0000000000000LL);
        ++R.queries;
        int tri = closest_hit<STORAGE, true>(B, ox, oy, oz, dx, dy, dz, 0.0, t, visits);
        R.escaped = tri < 0;
    }
    R.dx = dx; R.dy = dy; R.dz = dz;
    return R;
}

}  // namespace sbr
