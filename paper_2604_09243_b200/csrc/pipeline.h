// pipeline.h -- launch wrappers of the trace / compaction+PO / reduce kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sbr_device.cuh"

namespace sbr {

constexpr int kChunk = 1024;        // ray slots per PO block (compaction tile)
constexpr int kSegChunks = 512;     // chunks per segment -> 2^19 rays
constexpr int64_t kSegRays = (int64_t)kChunk * kSegChunks;

// One incident direction (ApertureGrid, transport.py:84-127).
struct GridDev {
    double corner[3], u[3], v[3], k[3];
    double spacing;
    int64_t n_v;
    int64_t n_rays;
    // derived on the host (grid_derive): rows, and per axis the raster's
    // magnitude bound |corner| + n_u ds |u| + n_v ds |v| (primary.cu)
    int64_t n_u;
    double rbound[3];
};

inline void grid_derive(GridDev &g)
{
    g.n_u = g.n_v > 0 ? g.n_rays / g.n_v : 0;
    const double su = (double)g.n_u * g.spacing, sv = (double)g.n_v * g.spacing;
    for (int a = 0; a < 3; ++a) {
        const double c = g.corner[a] < 0 ? -g.corner[a] : g.corner[a];
        const double u = g.u[a] < 0 ? -g.u[a] : g.u[a];
        const double v = g.v[a] < 0 ? -g.v[a] : g.v[a];
        g.rbound[a] = (c + su * u + sv * v) * (1.0 + 1e-12);
    }
}

// Unit of work: rays [ray_begin, ray_end) of grid `grid` (segment `seg`),
// occupying slots [slot_base, slot_base + roundup(len, kChunk)) of a batch.
struct UnitDev {
    int grid;
    int seg;
    int64_t ray_begin, ray_end;
    int64_t slot_base;
    int64_t seg_out;    // global segment row of the partial output
};

// Compact per-ray record of the solve path (16 B).
struct __align__(16) SlotRec {
    double R;          // accumulated path length (FP64)
    float cosv;        // -(n0 . k_inc)
    uint32_t meta;     // bits 0-15 bounces | flags below
};
constexpr uint32_t kMetaValid = 1u << 16;
constexpr uint32_t kMetaEscaped = 1u << 17;
constexpr uint32_t kMetaSel = 1u << 18;
constexpr uint32_t kMetaActive = 1u << 19;
constexpr uint32_t kMetaBounceMask = 0xffffu;
// list-mode records (written over work-list entries) carry the ray's offset
// within its 1024-slot chunk in bits 20..29 (r mod 1024: units are chunk-
// and segment-aligned), for the NumericalError record index
constexpr int kMetaOffShift = 20;

// Work-list entry (16 B) of a primary hit, written by k_prim_compact:
//   x, y = bits of the query-0 t; z, w = id | (ray offset in its unit) << 25
//   | (unit index in the batch) << 44 -- ids < 2^25 (kMaxTriangles), unit
//   offsets < 2^19 (kSegRays), units per batch < 2^20 (run_units).
// The trace kernel overwrites the entry with the ray's SlotRec.
constexpr int kWlOffShift = 25;
constexpr int kWlUnitShift = 44;
constexpr int kMaxBatchUnits = 1 << 20;
// meta of an all-ones slot (a PrimHit that no triangle reached): a finished
// primary miss -- no real record has bits 20..31 set
constexpr uint32_t kMissMeta = 0xffffffffu;

// Primary-visibility result of one ray (query 0), written by the raster
// pass (128-bit compare-and-swap minimum) and read by the trace kernel.  Aliases the
// SlotRec of the same slot in the fused solve: tbits <-> R, id <-> meta.
// All-ones = no hit (the buffer is memset to 0xff before the pass).
struct __align__(16) PrimHit {
    unsigned long long tbits;   // bits of the closest accepted t (> 0, finite)
    unsigned int pad;
    unsigned int id;            // smallest triangle id among hits at that t
};
static_assert(sizeof(PrimHit) == sizeof(SlotRec), "PrimHit aliases SlotRec");
constexpr unsigned long long kNoHitBits = ~0ULL;

enum TraceMode : int { kModeSolve = 0, kModeGrid = 1, kModeList = 2 };

// unit owning a slot (units sorted by slot_base)
__device__ inline int find_unit(const UnitDev *u, int n, int64_t slot)
{
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (__ldg(&u[mid].slot_base) <= slot) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// origin of ray r = i * n_v + j exactly as transport.py:339-345 builds it:
// bx = corner + ((i+.5) ds) u, ox = bx + ((j+.5) ds) v (no FMA contraction)
__device__ inline void grid_origin(const GridDev &g, int64_t r, double &ox,
                                            double &oy, double &oz)
{
    int64_t i, j;
    if ((uint64_t)r < 0xffffffffULL) {   // 32-bit division (apertures < 2^32 rays)
        const uint32_t q = (uint32_t)r / (uint32_t)g.n_v;
        i = q;
        j = r - (int64_t)q * g.n_v;
    } else {
        i = r / g.n_v;
        j = r - i * g.n_v;
    }
    double si = DM(DA((double)i, 0.5), g.spacing);
    double sj = DM(DA((double)j, 0.5), g.spacing);
    double bx = DA(g.corner[0], DM(si, g.u[0]));
    double by = DA(g.corner[1], DM(si, g.u[1]));
    double bz = DA(g.corner[2], DM(si, g.u[2]));
    ox = DA(bx, DM(sj, g.v[0]));
    oy = DA(by, DM(sj, g.v[1]));
    oz = DA(bz, DM(sj, g.v[2]));
}

struct TraceCfg {
    BvhView B;
    int storage;
    int max_bounces;
    double eps;
    int strict;
    int count_trapped;
    int allow_aliasing;
    double spacing_limit;       // lambda_min / sampling_factor (<= 0: no rule)
    unsigned int *error_flag;   // device: bit 0 = sampling rule violated
};

struct LaunchStats {
    int64_t *launches;
    int num_sms;
};

// ---- trace ---------------------------------------------------------------
// prim_from_slots: query 0 of every ray was resolved by launch_raster into
// the slots (PrimHit aliasing), the kernel starts at the first bounce.
// worklist (raster mode): slots still to trace, count in *d_nwork.
cudaError_t launch_trace_solve(const TraceCfg &cfg, const GridDev *d_grids,
                               const UnitDev *d_units, int n_units, int64_t n_slots,
                               SlotRec *d_slots, unsigned long long *d_counter,
                               bool prim_from_slots, uint4 *d_worklist,
                               const unsigned long long *d_nwork, cudaStream_t st,
                               const LaunchStats &ls);

// After the raster pass: final records for padding / aliasing-rejected /
// missed slots, and the list of slots whose query 0 hit (warp-ordered).
// d_chunk_hits[c] = (first list entry, count) of chunk c's hits (list mode of
// launch_po); misses and padding slots are left untouched (all-ones)
cudaError_t launch_prim_compact(const TraceCfg &cfg, const GridDev *d_grids,
                                const UnitDev *d_units, int n_units, int64_t n_slots,
                                SlotRec *d_slots, const unsigned int *d_hitmap,
                                const int *d_chunk_unit, uint4 *d_worklist,
                                unsigned long long *d_nwork, uint2 *d_chunk_hits,
                                cudaStream_t st, const LaunchStats &ls);
cudaError_t launch_chunk_units(const UnitDev *d_units, int n_units, int *d_chunk_unit,
                               cudaStream_t st, const LaunchStats &ls);

struct FullOut {
    uint8_t *valid;
    double *n0;
    double *path;
    int32_t *bounces;
    uint8_t *escaped;
    double *out_dir;
    int32_t *ids;      // may be null
    // hash mode (grid only): no per-ray stores; record_hash() of every ray is
    // added into seg_hash[r / seg_rays] (r = ray index in the grid)
    unsigned long long *seg_hash;
    int64_t seg_rays;
};

// Per-ray record hash (a checksum of every HitRecords field plus the
// per-bounce ids, -1 padded to max_bounces), shared with the oracle
// (oracle/sbr_oracle.c orc_record_hash): splitmix64 finaliser chained over
//   r, ids[0..B), flags (valid | escaped << 8 | N << 16), n0 xyz, R, out_dir xyz.
// A segment's hash is the wrapping sum over its rays, so it is independent
// of execution order.
__host__ __device__ inline unsigned long long hash_mix(unsigned long long z)
{
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ unsigned long long dbits(double x)
{
    return (unsigned long long)__double_as_longlong(x);
}
// hid = ids folded so far (hash_mix(r) then hash_mix(h ^ id) per recorded
// bounce); n_ids = bounces recorded
__device__ __forceinline__ unsigned long long record_hash(unsigned long long hid, int n_ids,
                                                          int max_bounces, bool valid,
                                                          bool escaped, double n0x, double n0y,
                                                          double n0z, double path, double ox,
                                                          double oy, double oz)
{
    for (int b = n_ids; b < max_bounces; ++b) hid = hash_mix(hid ^ 0xffffffffULL);
    unsigned long long h = hash_mix(hid ^ ((unsigned long long)(valid ? 1 : 0) |
                                           ((unsigned long long)(escaped ? 1 : 0) << 8) |
                                           ((unsigned long long)(unsigned int)n_ids << 16)));
    h = hash_mix(h ^ dbits(n0x));
    h = hash_mix(h ^ dbits(n0y));
    h = hash_mix(h ^ dbits(n0z));
    h = hash_mix(h ^ dbits(path));
    h = hash_mix(h ^ dbits(ox));
    h = hash_mix(h ^ dbits(oy));
    h = hash_mix(h ^ dbits(oz));
    return h;
}

// grid != null: rays from the grid; else origins/dirs arrays
// d_prim (grid mode only, may be null): query-0 results from launch_raster
// grid mode traces rays r_base + [0, n) of the grid
cudaError_t launch_trace_full(const TraceCfg &cfg, const GridDev *d_grid,
                              const double *d_orig, const double *d_dirs, int64_t n,
                              int64_t r_base, const FullOut &out, const PrimHit *d_prim,
                              unsigned long long *d_counter, cudaStream_t st,
                              const LaunchStats &ls);

// ---- reference-order traversal (reforder.cu) --------------------------------
// The reference-layout tree (bvh.py:58-88) and the mesh in original order.
struct RefView {
    const double *nmin, *nmax;       // (N,3)
    const int32_t *first, *count, *order;
    int round_f32;                   // boxes rounded outward to float32 (bvh.py:286-290)
    const double *verts;             // (T,9) original order
    int single;                      // float32 edge subtraction (storage kSingle)
};
cudaError_t launch_closest_ref(const RefView &V, const double *d_orig, const double *d_dirs,
                               int64_t n, double t_min, double t_max, int64_t *d_tri,
                               double *d_t, int64_t *d_visits, cudaStream_t st,
                               const LaunchStats &ls);
// d_slots != null: solve mode over n slots of d_units; else grid (d_grids)
// or list mode like launch_trace_full
cudaError_t launch_trace_ref(const RefView &V, const TraceCfg &cfg, const GridDev *d_grids,
                             const double *d_orig, const double *d_dirs, int64_t n,
                             int64_t r_base, const FullOut &out, const UnitDev *d_units,
                             SlotRec *d_slots, int n_units, cudaStream_t st,
                             const LaunchStats &ls);

cudaError_t launch_closest(const BvhView &B, int storage, const double *d_orig,
                           const double *d_dirs, int64_t n, double t_min, double t_max,
                           int64_t *d_tri, double *d_t, int64_t *d_visits, cudaStream_t st,
                           const LaunchStats &ls);

// ---- primary visibility (raster pass) -------------------------------------
// The primary rays of an aperture form a regular orthographic grid with one
// direction, so query 0 of every ray is answered per TRIANGLE instead of per
// ray: each (grid, triangle) pair enumerates the grid cells of a region
// proven to hold every cell its test can accept and runs the same exact
// FP64 Moller-Trumbore test on each (origin built exactly as the launcher
// builds it).  A 128-bit compare-and-swap keeps the lexicographic (t, id)
// minimum of bvh.py:340 per ray, independent of execution order.
struct RasterArgs {
    BvhView B;
    int storage;
    int64_t ntri;              // triangles (leaf-order slots)
    const GridDev *grids;
    const int *bgrids;         // grids of this batch
    int nbg;
    const int64_t *seg_base;   // (ngrids+1) first global segment row of each grid
    const int64_t *seg_slot;   // per global segment row: slot - ray index, or kNoSlot
    PrimHit *prim;
    unsigned int *hitmap;          // 1 bit per slot, set on a slot's first hit (or null)
    unsigned long long *counter;   // work counter (zeroed by launch_raster)
    int sparse;                    // some segments of the batch's grids are not in it
    int4 *big;                     // queue of big-triangle chunks (grid, tri, chunk, setup)
    unsigned long long *nbig;      // its fill counter
    int64_t big_cap;               // its capacity (items beyond it stay in k_raster)
    // set-ups of queued triangles (kRasterSetupBytes each), computed once in
    // k_raster and read by every chunk of the triangle (-1 in the queue
    // entry: table full, the chunk recomputes it)
    unsigned char *setups;
    unsigned long long *nsetup;
    int64_t setup_cap;
    int64_t row_lo, row_hi;        // rows [row_lo, row_hi) only (a partial trace_grid)
    // accumulating counters (may be null): [0] candidate cells tested,
    // [1] WIDE (ill-conditioned) pairs, [2] chunk-queue overflows
    unsigned long long *stats;
};
constexpr int kRasterSetupBytes = 256;
constexpr int64_t kNoSlot = INT64_MIN;   // segment not in this batch / shard
cudaError_t launch_raster(const RasterArgs &a, cudaStream_t st, const LaunchStats &ls);

// ---- integrate ------------------------------------------------------------
cudaError_t launch_records_to_slots(const uint8_t *valid, const double *n0,
                                    const double *path, const int32_t *bounces,
                                    const uint8_t *escaped, int64_t n, double kx,
                                    double ky, double kz, int count_trapped,
                                    int64_t n_slots, SlotRec *slots, cudaStream_t st,
                                    const LaunchStats &ls);

// dkturn != 0: the nk wavenumbers are equally spaced, (k[f+1]-k[f]) / pi
// d_list != null (raster pass): list mode -- each chunk reads only its hits'
// records, which the trace kernel wrote over their work-list entries
// (d_chunk_hits: the chunk's run of the list); otherwise every slot is read
cudaError_t launch_po(SlotRec *d_slots, const UnitDev *d_units, int n_units,
                      const uint4 *d_list, const uint2 *d_chunk_hits,
                      int64_t n_chunks, const double *d_k2, int nk, double dkturn,
                      const double *d_gpow,
                      int max_bounces, double2 *d_chunk_part, int64_t *d_diag,
                      unsigned long long *d_bad, unsigned long long *d_counter,
                      const int *d_chunk_unit, cudaStream_t st, const LaunchStats &ls);

cudaError_t launch_seg_reduce(const double2 *d_chunk_part, const UnitDev *d_units,
                              int n_units, int nk, double2 *d_seg_part, cudaStream_t st,
                              const LaunchStats &ls);

cudaError_t launch_finalize(const double2 *d_seg_part, const int64_t *d_seg_base,
                            int ngrids, int nk, const double *d_scale, double2 *d_amp,
                            cudaStream_t st, const LaunchStats &ls);

// ---- packed reduce buffer (sbr_solve_shard_packed / sbr_finalize_packed) ---
cudaError_t launch_pack_diag(const int64_t *d_diag, int ng, int stride, int nranks, int rank,
                             double *d_tail, cudaStream_t st, const LaunchStats &ls);
cudaError_t launch_unpack_diag(const double *d_tail, int ng, int stride, int nranks,
                               int64_t *d_diag, cudaStream_t st, const LaunchStats &ls);

// ---- scalar predicates ------------------------------------------------------
cudaError_t launch_tri_pairs(const double *v0, const double *v1, const double *v2,
                             const double *o, const double *d, int64_t n, double t_min,
                             double t_max, int single, double *t_out, cudaStream_t st,
                             const LaunchStats &ls);
cudaError_t launch_box_pairs(const double *lo, const double *hi, const double *o,
                             const double *inv, int64_t n, double t_max, uint8_t *hit,
                             double *entry, cudaStream_t st, const LaunchStats &ls);

// Best-of-5 read bandwidth of a `bytes` buffer re-read `reps` times through L2.
cudaError_t probe_l2_read(int64_t bytes, int reps, int num_sms, cudaStream_t st, double *gbs);

}  // namespace sbr
