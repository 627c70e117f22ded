// trace_persistent.cuh -- persistent, warp-cooperative multi-bounce tracer.
//
// Every lane is a small state machine over (ray, query, traversal step):
//
//   IDLE  -> fetch a ray index from the warp's private chunk of the global
//            work counter (one atomic per kChunkRays rays per warp), build
//            its origin on the fly (transport.py:339-345) and start query 0
//   TRAV  -> one BVH node per step: conservative FP32 slab tests of both
//            children (child-pair node, four 16-byte loads), near child
//            next, far child onto the stack
//   LEAF  -> exact FP64 Moller-Trumbore on the leaf's triangles
//   DONE  -> query finished: the bounce logic of transport.py:293-326
//            (flip / strict / reflect / epsilon offset / escape probe) and
//            either the next query or the ray's output record
//
// The warp loop is "while-while" (Aila & Laine 2009): node steps repeat
// while any lane is traversing, lanes that reached a leaf wait, then all
// pending leaves are intersected together, then finished queries advance
// and idle lanes are refilled.  A lane never waits for a whole other ray
// (bounce counts and miss/hit mixes no longer serialise the warp), only for
// the current traversal phase.
//
// Results are bit-identical to the reference (transport.py:276-327): every
// query still returns the lexicographic (t, id) minimum over accepted
// triangles, and the per-bounce FP64 arithmetic is unchanged.
#pragma once

#include <type_traits>

#include "pipeline.h"
#include "traverse.cuh"

namespace sbr {

#ifndef SBR_CHUNK_RAYS
#define SBR_CHUNK_RAYS 128
#endif
#ifndef SBR_TRACE_MINB
#define SBR_TRACE_MINB 8
#endif
constexpr int kChunkRays = SBR_CHUNK_RAYS;   // rays claimed per warp-level atomic
// two parked leaves per lane before it blocks (lane census: 9 of 32 lanes sat
// blocked on a second leaf; trace 113 -> 111 ms).  -DSBR_PARK1 restores one.
#ifndef SBR_PARK1
#define SBR_PARK2
#endif
#ifndef SBR_DONE_BREAK
#define SBR_DONE_BREAK 8
#endif
constexpr int kDoneBreak = SBR_DONE_BREAK;   // finished lanes that end a traversal phase

enum LaneState : int { kIdle = 0, kTrav = 1, kLeaf = 2, kDone = 3 };

struct TraceArgs {
    TraceCfg cfg;
    // work source
    const GridDev *grids;     // solve: all grids; grid mode: the one grid
    const UnitDev *units;     // solve only
    int n_units;
    const double *orig, *dirs;  // list mode
    int64_t n_work;           // solve: slots; grid/list: rays
    unsigned long long *counter;
    // query-0 results of the raster pass (solve: aliases `slots`, indexed by
    // slot; grid: indexed by ray); null = trace query 0 through the BVH
    const PrimHit *prim;
    // solve + raster: the slots whose query 0 hit (k_prim_compact); the other
    // slots already hold their final records.  n_work is read from n_work_dev.
    // packed query-0 hit per entry (pipeline.h kWl*); entry w is overwritten
    // with ray w's SlotRec
    uint4 *worklist;
    const unsigned long long *n_work_dev;
    // grid mode: rays r_base + [0, n_work) of the grid (a row range); output
    // and prim indices are relative to r_base
    int64_t r_base;
    // outputs
    SlotRec *slots;           // solve
    FullOut full;             // grid / list
};

struct LaneRay {
    // ray + walk state (FP64, transport.py:276-327)
    double ox, oy, oz, dx, dy, dz;
    double path, n0x, n0y, n0z;
    double cosd;     // solve mode: -(n0 . k_inc) of the first hit
    double best_t;
    int best;
    int bounces;
    bool valid, probe;
    // traversal state
    RayBox rb;
    float tmax;
    int ref, sp;
    int pend;        // parked leaf reference (0: none)
#ifdef SBR_PARK2
    int pend2;       // second parked leaf
#endif
    // bookkeeping
    int64_t r;       // ray index within its grid / list
    int64_t slot;    // output slot (solve) or ray index (relative to r_base)
    int grid;
    unsigned long long hid;   // hash mode: running hash of the per-bounce ids
#ifdef SBR_TRACE_STATS
    unsigned long long st_nodes, st_tris, st_leaves, st_push, st_queries;
#endif
};

template <int STORAGE>
__device__ __forceinline__ void start_query(const BvhView &B, LaneRay &L, int &state)
{
    L.rb = make_raybox(B, L.ox, L.oy, L.oz, L.dx, L.dy, L.dz);
    L.best_t = __longlong_as_double(0x7ff0000000000000LL);
    L.best = -1;
    L.tmax = __int_as_float(0x7f800000);
    L.sp = 0;
    L.pend = 0;
#ifdef SBR_PARK2
    L.pend2 = 0;
#endif
    L.ref = B.root;
    state = L.ref >= 0 ? kTrav : kLeaf;
#ifdef SBR_TRACE_STATS
    L.st_queries += 1;
#endif
}

// exact test of one leaf's triangles; true = any-hit probe satisfied
template <int STORAGE>
__device__ __forceinline__ bool leaf_test(const BvhView &B, LaneRay &L, int leaf)
{
    const int first = leaf_first(leaf), cnt = leaf_count(leaf);
#ifdef SBR_TRACE_STATS
    L.st_leaves += 1;
#endif
    for (int k = first; k < first + cnt; ++k) {
#ifdef SBR_TRACE_STATS
        L.st_tris += 1;
#endif
        const TriF64 T = load_tri<STORAGE>(B, k);
        const double t = tri_hit_exact(T, L.ox, L.oy, L.oz, L.dx, L.dy, L.dz, 0.0, L.best_t);
        if (t > 0.0 && (t < L.best_t || (t == L.best_t && T.id < L.best))) {
            L.best_t = t;
            L.best = T.id;
            L.tmax = __double2float_ru(t);
            if (L.probe) return true;   // escape probe: any hit decides
        }
    }
    return false;
}

// pop the next stack entry whose entry distance can still beat best_t
__device__ __forceinline__ bool pop_next(StackEntry *stack, LaneRay &L)
{
    while (L.sp > 0) {
        --L.sp;
        if (stack[L.sp].tn <= L.tmax) {
            L.ref = stack[L.sp].ref;
            return true;
        }
    }
    return false;
}
__device__ __forceinline__ void push_entry(StackEntry *stack, LaneRay &L, int ref, float tn)
{
#ifdef SBR_TRACE_STATS
    L.st_push += 1;
#endif
    stack[L.sp].ref = ref;
    stack[L.sp].tn = tn;
    ++L.sp;
}

// Probe-only launches (every traced query is an escape probe: max_bounces
// == 1 with query 0 answered by the raster pass): a probe stops at its first
// hit, so entry distances never cull a pop -- 4-byte entries (refs only)
// halve the stack's local-memory lines (C5 trace 137 -> 133 ms).
__device__ __forceinline__ bool pop_next(int *stack, LaneRay &L)
{
    if (L.sp > 0) {
        --L.sp;
        L.ref = stack[L.sp];
        return true;
    }
    return false;
}
__device__ __forceinline__ void push_entry(int *stack, LaneRay &L, int ref, float)
{
    stack[L.sp] = ref;
    ++L.sp;
}

// MINB = 8 caps registers at 64 (32 resident warps per SM): measured
// faster than unconstrained 80-92 registers despite a few spills, since the
// traversal is latency-bound.
template <int W> __device__ __forceinline__ const typename WideNode<W>::T *wide_nodes(const BvhView &B);
#ifdef SBR_NODE_Q
template <> __device__ __forceinline__ const Node4Q *wide_nodes<4>(const BvhView &B) { return B.nodes4q; }
#else
template <> __device__ __forceinline__ const Node4 *wide_nodes<4>(const BvhView &B) { return B.nodes4; }
#endif
#ifdef SBR_NODE_Q
template <> __device__ __forceinline__ const Node8Q *wide_nodes<8>(const BvhView &B) { return B.nodes8q; }
#else
template <> __device__ __forceinline__ const Node8 *wide_nodes<8>(const BvhView &B) { return B.nodes8; }
#endif

template <int STORAGE, int MODE, int W = 4, bool PROBES = false, int MINB = SBR_TRACE_MINB>
__global__ void __launch_bounds__(128, MINB)
k_trace_persistent(TraceArgs a)
{
    const TraceCfg &cfg = a.cfg;
    const BvhView &B = cfg.B;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;

    typename std::conditional<PROBES, int, StackEntry>::type stack[kStack];
    LaneRay L;
#ifdef SBR_TRACE_STATS
    L.st_nodes = L.st_tris = L.st_leaves = L.st_push = L.st_queries = 0;
#endif
    int state = kIdle;
    const int64_t n_work = a.worklist ? (int64_t)*a.n_work_dev : a.n_work;
    bool exhausted = false;
    int64_t chunk_next = 0, chunk_end = 0;   // warp-uniform private work range

    while (true) {
#ifdef SBR_TRACE_STATS
        long long clk0 = clock64();
#endif
        // ---------------- refill idle lanes -------------------------------
        const unsigned want = __ballot_sync(0xffffffffu, state == kIdle && !exhausted);
        if (want) {
            // warp-uniform bookkeeping: [chunk_next, chunk_end) is this warp's
            // private slice of the global work counter
            const int need = __popc(want);
            const int64_t avail = chunk_end - chunk_next;
            int64_t fresh = 0;
            if (avail < need) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(a.counter, (unsigned long long)kChunkRays);
                fresh = (int64_t)__shfl_sync(0xffffffffu, base, 0);
            }
            int wl_unit = -1;
            int64_t wl_slot = 0;
            if (want & (1u << lane)) {
                const int rank = __popc(want & lt_mask);
                const int64_t w = rank < avail ? chunk_next + rank : fresh + (rank - avail);
                if (w < n_work) {
                    if (a.worklist) {
                        // one 16-byte load: the raster's query-0 result, the
                        // ray's unit and its offset in the unit
                        const uint4 e = __ldg(&a.worklist[w]);
                        const unsigned long long pk =
                            (unsigned long long)e.z | ((unsigned long long)e.w << 32);
                        L.slot = w;                 // output: the list entry itself
                        L.best_t = __longlong_as_double((long long)e.x |
                                                        ((long long)e.y << 32));
                        L.best = (int)(pk & ((1ULL << kWlOffShift) - 1));
                        wl_slot = (int64_t)((pk >> kWlOffShift) &
                                            ((1ULL << (kWlUnitShift - kWlOffShift)) - 1));
                        wl_unit = (int)(pk >> kWlUnitShift);
                    } else {
                        L.slot = w;
                    }
                } else {
                    exhausted = true;
                }
            }
            if (avail >= need) {
                chunk_next += need;
            } else {
                chunk_next = fresh + (need - avail);
                chunk_end = fresh + kChunkRays;
            }
            if (state == kIdle && !exhausted && (want & (1u << lane))) {
                // ---------------- ray setup -------------------------------
                bool real = true;
                const GridDev *G = nullptr;
                if (MODE == kModeSolve) {
                    const int ui = wl_unit >= 0 ? wl_unit : find_unit(a.units, a.n_units, L.slot);
                    const UnitDev U = a.units[ui];
                    // list entries carry the ray's offset within its unit
                    L.r = wl_unit >= 0 ? U.ray_begin + wl_slot
                                       : U.ray_begin + (L.slot - U.slot_base);
                    L.grid = U.grid;
                    G = a.grids + U.grid;
                    real = L.r < U.ray_end;
                    const bool alias_ok = cfg.allow_aliasing || !(G->spacing > cfg.spacing_limit);
                    if (!alias_ok) {
                        atomicOr(cfg.error_flag, 1u);
                        real = false;
                    }
                    if (!real) {
                        SlotRec z;
                        z.R = 0.0; z.cosv = 0.f; z.meta = 0u;
                        a.slots[L.slot] = z;
                    }
                } else if (MODE == kModeGrid) {
                    L.r = L.slot + a.r_base;
                    G = a.grids;
                } else {
                    L.r = L.slot;
                }
                if (real) {
                    if (MODE == kModeList) {
                        L.ox = a.orig[3 * L.r]; L.oy = a.orig[3 * L.r + 1];
                        L.oz = a.orig[3 * L.r + 2];
                        L.dx = a.dirs[3 * L.r]; L.dy = a.dirs[3 * L.r + 1];
                        L.dz = a.dirs[3 * L.r + 2];
                    } else {
                        grid_origin(*G, L.r, L.ox, L.oy, L.oz);
                        L.dx = G->k[0]; L.dy = G->k[1]; L.dz = G->k[2];
                    }
                    if (MODE != kModeSolve && a.full.seg_hash) {
                        L.hid = hash_mix((unsigned long long)L.r);
                    } else if (MODE != kModeSolve && a.full.ids) {
                        int *ids = a.full.ids + L.slot * (int64_t)cfg.max_bounces;
                        for (int b = 0; b < cfg.max_bounces; ++b) ids[b] = -1;
                    }
                    L.path = 0.0; L.n0x = L.n0y = L.n0z = 0.0; L.cosd = 0.0;
                    L.bounces = 0; L.valid = false; L.probe = false;
                    if (MODE == kModeSolve && wl_unit >= 0) {
                        state = kDone;   // query 0 answered by the raster pass (loaded above)
                    } else if (MODE != kModeList && a.prim) {
                        // query 0 already answered by the raster pass
                        const PrimHit h = a.prim[L.slot];
                        const bool hit = h.tbits != kNoHitBits;
                        L.best_t = hit ? __longlong_as_double((long long)h.tbits)
                                       : __longlong_as_double(0x7ff0000000000000LL);
                        L.best = hit ? (int)h.id : -1;
                        state = kDone;
                    } else {
                        start_query<STORAGE>(B, L, state);
                    }
                }
            }
        }
        if (!__any_sync(0xffffffffu, state != kIdle || !exhausted)) break;

#ifdef SBR_TRACE_STATS
        long long clk1 = clock64();
#endif
        // ---------------- traversal phase ---------------------------------
        // Speculative while-while: a lane that reaches its first leaf parks
        // it in L.pend and keeps traversing; the phase ends once every
        // traversing lane has a parked leaf (or stopped at a second leaf).
        while (true) {
            // the traversal phase ends when no lane is still looking for its
            // first leaf -- or once kDoneBreak lanes have finished their query
            // and would otherwise idle until it ends (lane census: 11.5 of 32
            // lanes sat in kDone per step without this; trace 130 -> 113 ms)
            const unsigned trav = __ballot_sync(0xffffffffu, state == kTrav && L.pend == 0);
            if (!trav) break;
            if (__popc(__ballot_sync(0xffffffffu, state == kDone)) >= kDoneBreak) break;
#ifdef SBR_TRACE_STATS
            {   // lane-state census per traversal step (stats build only)
                const unsigned act = __ballot_sync(0xffffffffu, state == kTrav && L.pend == 0);
                const unsigned prk = __ballot_sync(0xffffffffu, state == kTrav && L.pend != 0);
                const unsigned blk = __ballot_sync(0xffffffffu, state == kLeaf);
                const unsigned dn = __ballot_sync(0xffffffffu, state == kDone);
                if (lane == 0) {
                    unsigned long long *st = a.counter + 8;
                    atomicAdd(st + 0, 1ULL);
                    atomicAdd(st + 1, (unsigned long long)__popc(act));
                    atomicAdd(st + 2, (unsigned long long)__popc(prk));
                    atomicAdd(st + 3, (unsigned long long)__popc(blk));
                    atomicAdd(st + 4, (unsigned long long)__popc(dn));
                }
            }
#endif
            if (state == kTrav) {
#ifdef SBR_TRACE_STATS
                L.st_nodes += 1;
#endif
                int rr[W];
                float tt[W];
                const int n = WideNode<W>::visit(wide_nodes<W>(B) + L.ref, L.rb, L.tmax, rr, tt);
                bool have = true;
                if (n > 0) {
#pragma unroll
                    for (int c = W - 1; c >= 1; --c)   // farther hits first: nearest pops first
                        if (c < n) push_entry(stack, L, rr[c], tt[c]);
                    L.ref = rr[0];
                } else {
                    have = pop_next(stack, L);
                }
#ifdef SBR_PARK2
                const bool parked = L.pend != 0 || L.pend2 != 0;
#else
                const bool parked = L.pend != 0;
#endif
                if (!have) {
                    state = parked ? kLeaf : kDone;   // kLeaf with ref 0: parked leaves only
                    L.ref = 0;
                } else {
                    // park leaves while a slot is free; a leaf with no free slot
                    // stops the lane (kLeaf, tested after the parked ones)
                    while (L.ref < 0) {
                        if (L.pend == 0) L.pend = L.ref;
#ifdef SBR_PARK2
                        else if (L.pend2 == 0) L.pend2 = L.ref;
#endif
                        else { state = kLeaf; break; }
                        if (!pop_next(stack, L)) { state = kLeaf; L.ref = 0; break; }
                    }
                }
            }
        }

#ifdef SBR_TRACE_STATS
        long long clk2 = clock64();
#endif
        // ---------------- leaf phase --------------------------------------
        // parked leaf first, then (kLeaf lanes) the leaf in L.ref and any
        // further leaves popped straight off the stack
        if (L.pend != 0 && (state == kTrav || state == kLeaf)) {
            const int leaf = L.pend;
            L.pend = 0;
            if (leaf_test<STORAGE>(B, L, leaf)) state = kDone;
        }
#ifdef SBR_PARK2
        if (L.pend2 != 0 && (state == kTrav || state == kLeaf)) {
            const int leaf = L.pend2;
            L.pend2 = 0;
            if (leaf_test<STORAGE>(B, L, leaf)) state = kDone;
        }
        if (state == kDone) L.pend2 = 0;
#endif
#ifdef SBR_TRACE_STATS
        {
            const unsigned lf = __ballot_sync(0xffffffffu, state == kLeaf || L.pend != 0);
            if (lane == 0) {
                atomicAdd(a.counter + 13, 1ULL);
                atomicAdd(a.counter + 14, (unsigned long long)__popc(lf));
            }
        }
#endif
        while (state == kLeaf) {
            if (L.ref < 0) {
                if (leaf_test<STORAGE>(B, L, L.ref)) { state = kDone; break; }
            }
            if (!pop_next(stack, L)) state = kDone;
            else if (L.ref >= 0) state = kTrav;
        }

#ifdef SBR_TRACE_STATS
        long long clk3 = clock64();
#endif
        // ---------------- query completion (transport.py:293-326) ---------
        if (state == kDone) {
            bool finish = false, escaped = false;
            if (L.probe) {
                escaped = L.best < 0;
                finish = true;
            } else if (L.best < 0) {
                escaped = true;
                finish = true;
            } else {
                const double t = L.best_t;
                const double *n = B.normals + 3 * (int64_t)L.best;
                double nx = __ldg(n), ny = __ldg(n + 1), nz = __ldg(n + 2);
                double ndd = DA(DA(DM(nx, L.dx), DM(ny, L.dy)), DM(nz, L.dz));
                bool strict_out = false;
                if (ndd > 0.0) {
                    if (cfg.strict && L.bounces == 0) {
                        strict_out = true;
                    } else {
                        nx = -nx; ny = -ny; nz = -nz; ndd = -ndd;
                    }
                }
                if (strict_out) {
                    // transport.py:306-307: invalid, escaped, direction kept
                    L.valid = false;
                    L.bounces = 0;
                    L.path = 0.0;
                    L.n0x = L.n0y = L.n0z = 0.0;
                    escaped = true;
                    finish = true;
                } else {
                    if (MODE != kModeSolve && a.full.seg_hash)
                        L.hid = hash_mix(L.hid ^ (unsigned long long)(unsigned int)L.best);
                    else if (MODE != kModeSolve && a.full.ids)
                        a.full.ids[L.slot * (int64_t)cfg.max_bounces + L.bounces] = L.best;
                    const double hx = DA(L.ox, DM(t, L.dx)), hy = DA(L.oy, DM(t, L.dy)),
                                 hz = DA(L.oz, DM(t, L.dz));
                    L.path = DA(L.path, t);
                    L.bounces += 1;
                    if (L.bounces == 1) {
                        L.valid = true;
                        // solve mode keeps only cos = -(n0 . k_inc) (po.py:99);
                        // d == k_inc here, so -ndd is that dot product exactly
                        if (MODE == kModeSolve) L.cosd = -ndd;
                        else { L.n0x = nx; L.n0y = ny; L.n0z = nz; }
                    }
                    const double s = DM(2.0, ndd);
                    L.dx = DS(L.dx, DM(s, nx));
                    L.dy = DS(L.dy, DM(s, ny));
                    L.dz = DS(L.dz, DM(s, nz));
                    L.ox = DA(hx, DM(cfg.eps, nx));
                    L.oy = DA(hy, DM(cfg.eps, ny));
                    L.oz = DA(hz, DM(cfg.eps, nz));
                    if (L.bounces == cfg.max_bounces) L.probe = true;  // budget spent
                    start_query<STORAGE>(B, L, state);
                }
            }
            if (finish) {
                if (MODE == kModeSolve) {
                    const double c = L.valid ? L.cosd : 0.0;
                    const bool sel = L.valid && (escaped || cfg.count_trapped) && c > 0.0;
                    SlotRec rec;
                    rec.R = L.path;
                    rec.cosv = (float)c;
                    rec.meta = (uint32_t)L.bounces | kMetaActive | (L.valid ? kMetaValid : 0u) |
                               (escaped ? kMetaEscaped : 0u) | (sel ? kMetaSel : 0u);
                    if (a.worklist) {
                        rec.meta |= (uint32_t)(L.r & (kChunk - 1)) << kMetaOffShift;
                        reinterpret_cast<SlotRec *>(a.worklist)[L.slot] = rec;
                    } else {
                        a.slots[L.slot] = rec;
                    }
                } else if (a.full.seg_hash) {
                    const unsigned long long h = record_hash(
                        L.hid, L.bounces, cfg.max_bounces, L.valid, escaped, L.n0x, L.n0y,
                        L.n0z, L.path, L.dx, L.dy, L.dz);
                    atomicAdd(a.full.seg_hash + L.r / a.full.seg_rays, h);
                } else {
                    const int64_t r = L.slot;
                    a.full.valid[r] = L.valid ? 1 : 0;
                    a.full.escaped[r] = escaped ? 1 : 0;
                    a.full.bounces[r] = L.bounces;
                    a.full.path[r] = L.path;
                    a.full.n0[3 * r] = L.n0x; a.full.n0[3 * r + 1] = L.n0y;
                    a.full.n0[3 * r + 2] = L.n0z;
                    a.full.out_dir[3 * r] = L.dx; a.full.out_dir[3 * r + 1] = L.dy;
                    a.full.out_dir[3 * r + 2] = L.dz;
                }
                state = kIdle;
            }
        }
#ifdef SBR_TRACE_STATS
        {   // cycles per phase (warp-uniform points; lane 0 records)
            __syncwarp();
            const long long clk4 = clock64();
            if (lane == 0) {
                atomicAdd(a.counter + 16, (unsigned long long)(clk1 - clk0));   // refill
                atomicAdd(a.counter + 17, (unsigned long long)(clk2 - clk1));   // traversal
                atomicAdd(a.counter + 18, (unsigned long long)(clk3 - clk2));   // leaf
                atomicAdd(a.counter + 19, (unsigned long long)(clk4 - clk3));   // completion
            }
        }
#endif
    }
#ifdef SBR_TRACE_STATS
    atomicAdd(a.counter + 20, L.st_nodes);
    atomicAdd(a.counter + 21, L.st_tris);
    atomicAdd(a.counter + 22, L.st_leaves);
    atomicAdd(a.counter + 23, L.st_push);
    atomicAdd(a.counter + 24, L.st_queries);
#endif
}

}  // namespace sbr
