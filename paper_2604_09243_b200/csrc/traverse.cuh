// traverse.cuh -- closest-hit / any-hit BVH traversal and the multi-bounce
// ray walk, as device functions shared by every trace kernel.
//
// Reference semantics:
//   closest_hit()  == bvh.py:306-362 _traverse (result only; the visit
//                     count is this tree's node fetches).  The multi-bounce
//                     walk lives in trace_persistent.cuh.
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
template <int STORAGE, bool ANY, bool F32RAYS = false>
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
                double t = F32RAYS ? tri_hit_f32rays(T, ox, oy, oz, dx, dy, dz, t_min, best_t)
                                   : tri_hit_exact(T, ox, oy, oz, dx, dy, dz, t_min, best_t);
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

}  // namespace sbr
