/*
 * sbr200.h -- C ABI of the B200-native SBR trace-integrate library
 * (libsbr200.so, built from paper_2604_09243_b200/csrc for sm_100a).
 *
 * This is the drop-in boundary for the reference package's hot path.  The
 * reference (pkg/src/sbr, Python + numba) has no formal FFI; its de-facto
 * kernel interface is the numba signature of
 *   _trace_rows(nodes_min, nodes_max, node_first, node_count, tri_order,
 *               v0, v1, v2, normals, corner, uvec, vvec, kvec, spacing, n_v,
 *               i_start, i_end, max_bounces, eps, strict, stack_depth, out*6)
 *   (pkg/src/sbr/transport.py:330-335)
 * plus the module functions re-exported by pkg/src/sbr/__init__.py:10-46.
 * Each entry point below names the reference interface it replaces.
 *
 * Conventions
 *  - All pointers are plain host pointers owned by the caller unless the
 *    parameter name ends in `_dev` (a device pointer on the context's GPU).
 *    Arrays are C-contiguous; (N,3) arrays are row-major xyz triples.
 *  - Every function returns an sbr_status; on failure sbr_last_error()
 *    returns a thread-local message.  Status codes mirror the reference
 *    exception mapping (pkg/src/sbr/errors.py:8-17, cli.py:196-205):
 *    SBR_EINVAL -> ValidationError, SBR_ENUMERIC -> NumericalError.
 *  - Results are a pure function of the inputs: no dependence on launch
 *    configuration, GPU count or scheduling (reference "workers"
 *    invariance, pkg/src/sbr/sweep.py:5-8).
 *  - Handles are not thread-safe across threads without external locking;
 *    use one context per GPU (one process per GPU in the sweep driver).
 */
#ifndef SBR200_H
#define SBR200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SBR200_ABI_VERSION 3

typedef enum {
    SBR_OK = 0,
    SBR_EINVAL = 2,    /* ValidationError (errors.py:12) */
    SBR_EIO = 3,       /* OSError */
    SBR_ENUMERIC = 4,  /* NumericalError (errors.py:16) */
    SBR_ENOTSUP = 5,   /* input outside the native fast path (caller falls back to the
                          reference-equivalent Python reader; host I/O only) */
    SBR_ECUDA = 10,    /* CUDA runtime failure */
    SBR_ENCCL = 11,    /* NCCL unavailable or a collective failed */
    SBR_ENOMEM = 12    /* device or host allocation failure */
} sbr_status;

/* Triangle storage on device (geometry.py:88-127 Mesh precision). */
typedef enum {
    SBR_STORAGE_AUTO = 0,      /* F32_EXACT if every coordinate is float32-representable, else F64 */
    SBR_STORAGE_F32_EXACT = 1, /* float32 storage, lossless; FP64 edges (== reference precision="double") */
    SBR_STORAGE_F64 = 2,       /* float64 storage (72 B/triangle) */
    SBR_STORAGE_SINGLE = 3     /* reference precision="single": float32 vertices AND float32 edge
                                  subtraction, FP64 ray state */
} sbr_storage;

typedef struct sbr_ctx sbr_ctx;
typedef struct sbr_mesh sbr_mesh;
typedef struct sbr_bvh sbr_bvh;

/* Replaces bvh.py:22-49 BuildParams.
 *  SBR_SPLIT_SAH / SBR_SPLIT_MEDIAN: the reference's binned-SAH
 *                  (bvh.py:154-215) or median-split (bvh.py:135-151) tree,
 *                  built on the GPU level by level and identical node for
 *                  node (sbr_bvh_export returns it verbatim);
 *  SBR_SPLIT_LBVH: a GPU LBVH (Morton order; fastest build).
 * Closest-hit results do not depend on the tree. */
enum { SBR_SPLIT_MEDIAN = 0, SBR_SPLIT_SAH = 1, SBR_SPLIT_LBVH = 2 };
typedef struct {
    int32_t split_rule;     /* SBR_SPLIT_* */
    int32_t n_leaf;         /* >= 1 (LBVH: <= 63) */
    int32_t max_depth;      /* SAH: depth limit, reference default 64 */
    int32_t bins_per_axis;  /* SAH: 2..64, 0 -> 16 */
    double c_t, c_i;        /* SAH cost constants, <= 0 -> 1.0 */
} sbr_build_params;

/* One incident direction's launch grid (transport.py:84-127 ApertureGrid).
 * Ray (i,j) starts at corner + ((i+.5)*spacing)*u + ((j+.5)*spacing)*v
 * and travels along k (transport.py:339-345). */
typedef struct {
    double corner[3], u[3], v[3], k[3];
    double spacing;
    double cell_area;
    int64_t n_u, n_v;
} sbr_grid;

/* transport.py:215-239 TraceParams + the sampling rule of
 * transport.py:75-81 (checked again on device by the launcher). */
typedef struct {
    int32_t max_bounces;      /* >= 1 */
    int32_t strict;           /* strict_orientation */
    int32_t allow_aliasing;   /* skip the spacing <= lambda_min / factor rule */
    int32_t reserved;
    double eps;               /* resolved epsilon (> 0) */
    double lambda_min;        /* shortest wavelength of the solve (0: no check) */
    double sampling_factor;   /* 5.0 by default */
} sbr_trace_params;

/* Per-solve diagnostics (sweep.py:256-259): arrays of length ngrids,
 * hist is ngrids*(max_bounces+1).  Any pointer may be NULL. */
typedef struct {
    int64_t *valid_rays;
    int32_t *max_bounce;
    int64_t *hist;
    int64_t *queries;         /* closest-hit queries = sum(N_i + 1) */
} sbr_diag;

const char *sbr_last_error(void);
int sbr_abi_version(void);

/* ---- context ---------------------------------------------------------- */
int sbr_ctx_create(int device, sbr_ctx **out);
int sbr_ctx_destroy(sbr_ctx *ctx);
int sbr_ctx_synchronize(sbr_ctx *ctx);
/* Release the context's grow-only scratch (solve slots and work list, build
 * workspaces, staging and pinned upload buffers) back to the device pool;
 * the next call re-grows what it needs.  Meshes and trees are untouched. */
int sbr_ctx_trim(sbr_ctx *ctx);
/* Stream the library launches on (cudaStream_t as void*). */
int sbr_ctx_stream(sbr_ctx *ctx, void **stream_out);
/* Number of kernels this context has launched (instrumentation). */
int sbr_ctx_launch_count(sbr_ctx *ctx, int64_t *count_out);

/* Traversal order of every query entry point (closest hit, trace_grid*,
 * trace_rays, solve*):
 *  SBR_TRAVERSAL_FAST (default): query 0 of aperture rays by the raster
 *    pass (the exact linear-scan answer), later queries by the persistent
 *    BVH4 kernel.  Bit-identical to the reference on every query whose
 *    winning triangle's hit point lies robustly inside its box with no
 *    accepting triangle tied within rounding.
 *  SBR_TRAVERSAL_REFERENCE: every query replays bvh.py:306-362 _traverse on
 *    the reference tree (FP64 slabs, far-first pushes, best_t culling) --
 *    bit-identical to the reference on every ray, including near-edge-on
 *    and edge/vertex tie rays; needs a SAH/median build or an uploaded
 *    tree (SBR_EINVAL otherwise).  Visit counts equal the reference's. */
enum { SBR_TRAVERSAL_FAST = 0, SBR_TRAVERSAL_REFERENCE = 1 };
int sbr_ctx_set_traversal(sbr_ctx *ctx, int32_t mode);
int sbr_ctx_get_traversal(sbr_ctx *ctx, int32_t *mode);

/* Per-kernel CUDA-event timing of the solve pipeline (trace kernel and
 * compaction+PO kernel), accumulated over calls; enabling resets it. */
int sbr_ctx_profile(sbr_ctx *ctx, int32_t enable);
int sbr_ctx_kernel_stats(sbr_ctx *ctx, double *trace_ms, int64_t *trace_launches,
                         double *po_ms, int64_t *po_launches);
/* Accumulated time of the primary-visibility raster pass (memset + two
 * sweeps) that precedes each trace launch; trace_ms excludes it. */
int sbr_ctx_raster_stats(sbr_ctx *ctx, double *raster_ms);
/* Read and clear the raster pass's counters, accumulated since the last
 * call: {candidate cells tested, ill-conditioned (WIDE) (grid, triangle)
 * pairs, chunk-queue overflows}. */
int sbr_ctx_raster_counters(sbr_ctx *ctx, int64_t out[3]);
/* Accumulated per-stage times of the solve pipeline with profiling on:
 * ms = {raster pass (incl. any slot memset), hit-list compaction, trace
 * kernel, compaction+PO kernel}. */
int sbr_ctx_stage_ms(sbr_ctx *ctx, double ms[4]);
/* Instrumentation: read bandwidth (GB/s) of a `bytes` buffer re-read `reps`
 * times from L2 (16-byte ld.global.cg, 8 CTAs/SM, best of 5). */
int sbr_probe_l2_bandwidth(sbr_ctx *ctx, int64_t bytes, int32_t reps, double *gbs);
/* Instrumented builds only (-DSBR_TRACE_STATS): read and clear n <= 24
 * lane-state counters of the trace kernel (zeros otherwise). */
int sbr_ctx_debug_counters(sbr_ctx *ctx, int64_t *out, int32_t n);
/* Device allocations the library holds right now (all contexts, meshes,
 * trees, scratch): for leak checks -- destroying every handle returns both
 * counts to zero. */
int sbr_debug_live_allocations(int64_t *count, int64_t *bytes);

/* ---- mesh: geometry.py:130-180 mesh_from_soup output -> device --------- */
int sbr_mesh_create(sbr_ctx *ctx, const double *v0, const double *v1,
                    const double *v2, const double *normals, int64_t ntri,
                    int32_t storage, sbr_mesh **out);
int sbr_mesh_destroy(sbr_mesh *mesh);
/* aabb = {min x,y,z, max x,y,z}; storage = resolved sbr_storage. */
int sbr_mesh_info(const sbr_mesh *mesh, int64_t *ntri, int32_t *storage,
                  double aabb[6]);

/* ---- BVH: bvh.py:218-299 build (GPU LBVH) ------------------------------ */
int sbr_bvh_build(sbr_ctx *ctx, const sbr_mesh *mesh,
                  const sbr_build_params *params, sbr_bvh **out);
/* Upload a reference-layout tree (bvh.py:58-88): preorder, left child
 * = i+1, node_first = right child (internal) or first index (leaf). */
int sbr_bvh_upload(sbr_ctx *ctx, const sbr_mesh *mesh, const double *nodes_min,
                   const double *nodes_max, const int32_t *node_first,
                   const int32_t *node_count, const int32_t *tri_order,
                   int64_t nnodes, sbr_bvh **out);
/* Size of the reference-layout export. */
int sbr_bvh_info(const sbr_bvh *bvh, int64_t *nnodes_export,
                 int64_t *nnodes_device, int32_t *max_depth);
/* Export into the reference layout so bvh.py:90-121 Bvh.validate() and
 * the CPU _traverse can consume it.  Arrays sized by sbr_bvh_info. */
int sbr_bvh_export(const sbr_bvh *bvh, double *nodes_min, double *nodes_max,
                   int32_t *node_first, int32_t *node_count, int32_t *tri_order);
int sbr_bvh_destroy(sbr_bvh *bvh);

/* ---- queries ------------------------------------------------------------ */
/* bvh.py:407-423 closest_hit_batch: tri (-1 on miss), t, node visits. */
int sbr_closest_hit(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                    const double *origins, const double *dirs, int64_t n,
                    double t_min, double t_max, int64_t *tri, double *t,
                    int64_t *visits);

/* geometry.py:394-409 ray_triangle_intersect over n independent
 * (ray, triangle) pairs (pair r uses triangle v0[r],v1[r],v2[r]);
 * t[r] = hit distance in (t_min, t_max] or -1.  single=1 evaluates the
 * reference float32 variant (float32 edge subtraction). */
int sbr_tri_hit_pairs(sbr_ctx *ctx, const double *v0, const double *v1,
                      const double *v2, const double *origins, const double *dirs,
                      int64_t n, double t_min, double t_max, int32_t single,
                      double *t);

/* geometry.py:412-425 ray_aabb_intersect (FP64 slab, geometry.py:358-391)
 * over n independent (ray, box) pairs; dir_inv holds reciprocals with
 * +-inf for zero components. */
int sbr_aabb_hit_pairs(sbr_ctx *ctx, const double *box_min, const double *box_max,
                       const double *origins, const double *dir_inv, int64_t n,
                       double t_max, uint8_t *hit, double *entry);

/* transport.py:375-422 trace_grid -> HitRecords (transport.py:251-273).
 * tri_ids (optional, n*max_bounces, -1 padded) records the hit triangle of
 * every bounce (the per-ray id parity channel). */
int sbr_trace_grid(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                   const sbr_grid *grid, const sbr_trace_params *params,
                   uint8_t *valid, double *normal0, double *path,
                   int32_t *bounces, uint8_t *escaped, double *out_dir,
                   int32_t *tri_ids);

/* transport.py:330-356 _trace_rows(i_start, i_end): rows [i_begin, i_end)
 * of the grid only; outputs hold (i_end - i_begin) * n_v records starting at
 * ray i_begin * n_v (the reference's per-worker row split). */
int sbr_trace_grid_rows(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                        const sbr_grid *grid, const sbr_trace_params *params,
                        int64_t i_begin, int64_t i_end, uint8_t *valid,
                        double *normal0, double *path, int32_t *bounces,
                        uint8_t *escaped, double *out_dir, int32_t *tri_ids);

/* Record checksums of rows [i_begin, i_end) without materialising records
 * (parity at 1e9-ray scale): seg_hash[s] = wrapping sum over rays r of
 * segment s (r / seg_rays == s, r over the whole grid, ceil(n_u*n_v /
 * seg_rays) entries) of a splitmix64 chain over r, the per-bounce triangle
 * ids (-1 padded to max_bounces), valid | escaped << 8 | bounces << 16,
 * normal0 xyz, path, out_dir xyz (bit patterns).  oracle/sbr_oracle.c
 * orc_trace_grid_hash computes the same function on the CPU. */
int sbr_trace_grid_hash(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                        const sbr_grid *grid, const sbr_trace_params *params,
                        int64_t i_begin, int64_t i_end, int64_t seg_rays,
                        uint64_t *seg_hash);

/* transport.py:359-372 trace_ray over an explicit ray list. */
int sbr_trace_rays(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                   const double *origins, const double *dirs, int64_t n,
                   const sbr_trace_params *params, uint8_t *valid,
                   double *normal0, double *path, int32_t *bounces,
                   uint8_t *escaped, double *out_dir, int32_t *tri_ids);

/* po.py:83-113 accumulate over host HitRecords (multi-frequency):
 * amp[f] = complex amplitude for wavenumber k[f], interleaved re,im.
 * On a non-finite term returns SBR_ENUMERIC with *bad_index = record. */
int sbr_accumulate(sbr_ctx *ctx, const uint8_t *valid, const double *normal0,
                   const double *path, const int32_t *bounces,
                   const uint8_t *escaped, int64_t n, const double k_inc[3],
                   const double *k, int32_t nk, double cell_area, double gamma,
                   int32_t count_trapped, double *amp, int64_t *bad_index);

/* ---- fused pipeline: sweep.py:240-263 solve_direction over many grids --
 * trace -> warp-ballot compaction -> PO integral -> deterministic reduce.
 * amp is ngrids*nk*2 (re,im) for wavenumbers k[0..nk).  Records never
 * leave the GPU. */
int sbr_solve(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
              const sbr_grid *grids, int32_t ngrids,
              const sbr_trace_params *params, const double *k, int32_t nk,
              double gamma, int32_t count_trapped, double *amp,
              sbr_diag *diag);

/* ---- sharded solve (multi-GPU; one process per GPU) ---------------------
 * Work is cut into fixed units of (grid g, segment s) where a segment is
 * SBR_SEGMENT_RAYS consecutive ray indices r = i*n_v + j of grid g.
 * shard_mode 0: unit (g,s) belongs to rank g % nranks (angle sharding);
 * shard_mode 1: unit index u (row-major over all units) belongs to rank
 *               u % nranks (ray-tile sharding).
 * The call writes FP64 segment partial sums into seg_dev (layout from
 * sbr_segment_layout: nseg_total*nk*2 doubles, zero for foreign units) and
 * integer diagnostics into diag_dev (ngrids*(3+max_bounces+1) int64:
 * valid, queries, max_bounce, hist...).  Summing seg_dev and diag_dev
 * element-wise over ranks (one NCCL reduce; max_bounce via a MAX reduce on
 * its rows) and calling sbr_finalize yields bit-identical results to
 * sbr_solve for any nranks. */
#define SBR_SEGMENT_RAYS (1 << 19)
int sbr_segment_layout(const sbr_grid *grids, int32_t ngrids,
                       int64_t *seg_base /* ngrids+1 */);
int sbr_solve_shard(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                    const sbr_grid *grids, int32_t ngrids,
                    const sbr_trace_params *params, const double *k, int32_t nk,
                    double gamma, int32_t count_trapped, int32_t rank,
                    int32_t nranks, int32_t shard_mode, double *seg_dev,
                    int64_t *diag_dev);
int sbr_finalize(sbr_ctx *ctx, const sbr_grid *grids, int32_t ngrids,
                 const double *k, int32_t nk, int32_t max_bounces,
                 const double *seg_dev, const int64_t *diag_dev, double *amp,
                 sbr_diag *diag);

/* ---- one-collective sharding -------------------------------------------
 * The same units as sbr_solve_shard, but partials AND diagnostics go into
 * ONE float64 device buffer of sbr_packed_layout() doubles:
 *   [segment partials (nseg*nk*2)][diagnostics (ngrids*(3+B+1)), integers
 *   as doubles, max-bounce column 0][max-bounce slots (ngrids*nranks), this
 *   rank's value in its own slot]
 * so a single element-wise SUM over ranks (one ncclReduce) is exact
 * (disjoint support; integers < 2^53) and sbr_finalize_packed takes the
 * max over the slots.  Bit-identical to sbr_solve for any nranks. */
int sbr_packed_layout(const sbr_grid *grids, int32_t ngrids, int32_t nk,
                      int32_t max_bounces, int32_t nranks, int64_t *count);
int sbr_solve_shard_packed(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                           const sbr_grid *grids, int32_t ngrids,
                           const sbr_trace_params *params, const double *k, int32_t nk,
                           double gamma, int32_t count_trapped, int32_t rank,
                           int32_t nranks, int32_t shard_mode, double *buf_dev);
int sbr_finalize_packed(sbr_ctx *ctx, const sbr_grid *grids, int32_t ngrids,
                        const double *k, int32_t nk, int32_t max_bounces, int32_t nranks,
                        const double *buf_dev, double *amp, sbr_diag *diag);

/* NCCL communicator of a context (one process per GPU; replaces the paper's
 * MPI layer).  libnccl is loaded at run time: the library
 * itself never needs it, these calls return SBR_ENCCL when it is absent.
 * Rank 0 calls sbr_comm_unique_id and ships the 128 bytes to the others
 * (any out-of-band channel: MPI, a file, torch.distributed, a socket). */
int sbr_comm_version(int32_t *nccl_version);
int sbr_comm_unique_id(uint8_t id[128]);
int sbr_comm_init(sbr_ctx *ctx, int32_t nranks, int32_t rank, const uint8_t id[128]);
int sbr_comm_destroy(sbr_ctx *ctx);
/* in-place ncclReduce(sum, float64) of a device buffer to `root` */
int sbr_reduce_sum_f64(sbr_ctx *ctx, double *buf_dev, int64_t count, int32_t root);
/* sweep.py:296-370 run_sweep's solve across the communicator's ranks: shard
 * (mode as sbr_solve_shard) -> one ncclReduce of the packed buffer ->
 * finalize on `root` (amp/diag written there only; other ranks may pass
 * NULL). */
int sbr_solve_distributed(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                          const sbr_grid *grids, int32_t ngrids,
                          const sbr_trace_params *params, const double *k, int32_t nk,
                          double gamma, int32_t count_trapped, int32_t shard_mode,
                          int32_t root, double *amp, sbr_diag *diag);

/* ---- mesh I/O (host only, no GPU needed) ---------------------------------
 * geometry.py:190-241 load_mesh: parse a Wavefront OBJ ("v"/"f" records,
 * 1-based or negative indices, polygons fan-triangulated).  `label` is the
 * path text used in error messages (reference wording).  SBR_EINVAL carries
 * the reference's ValidationError message; SBR_ENOTSUP means the file uses
 * number syntax only Python's float()/int() define (underscores, hex,
 * non-ASCII) and must be read by the Python loop. */
typedef struct sbr_obj sbr_obj;
int sbr_obj_read(const char *path, const char *label, sbr_obj **out);
int sbr_obj_info(const sbr_obj *obj, int64_t *nverts, int64_t *ntris);
/* verts (nverts,3) f64, tris (ntris,3) i64 vertex indices, labels (ntris) i64
 * source face numbers; any pointer may be NULL. */
int sbr_obj_copy(const sbr_obj *obj, double *verts, int64_t *tris, int64_t *labels);
int sbr_obj_free(sbr_obj *obj);
/* geometry.py:244-265 save_obj: exactly-equal corners share a "v" line
 * (first-seen order, "%.17g"), then one "f a b c" per triangle. */
int sbr_obj_write(const char *path, const double *v0, const double *v1, const double *v2,
                  int64_t ntri);
/* transport.py:425-436 dump_hits_csv: one "i,j,valid,nx,ny,nz,R,N" row per
 * ray of an n_u x n_v grid's HitRecords (record r = i*n_v + j), "%.9g". */
int sbr_dump_hits_csv(const char *path, int64_t n_u, int64_t n_v, const uint8_t *valid,
                      const double *normal0, const double *path_len, const int32_t *bounces);

#ifdef __cplusplus
}
#endif
#endif /* SBR200_H */
