// sahbuild.cu -- the reference's binned-SAH BVH (bvh.py:124-299), built on
// the GPU level by level, node for node identical to the reference tree.
//
// The reference recursion (emit -> binned_sah_split -> stable partition,
// preorder numbering) is order-independent except for the partition, which
// is stable.  Every per-node quantity is a min/max/count reduction (exact in
// any order) or a short FP64 formula evaluated once per node, so the tree can
// be built breadth-first with all nodes of a level in parallel:
//   level loop (host):
//     element -> active segment: written by the previous level's
//                    k_partition (median splits: k_seg_of, a binary search)
//     k_bounds       node box + centroid bounds per segment (ordered-int
//                    atomicMin/Max on doubles: exact)
//     k_bin          per (segment, axis, bin) counts + child-box bounds
//     k_select       one warp per segment, a lane per (axis, boundary)
//                    candidate: the reference's SAH sweep, cost formula with
//                    the reference's association, tie to the lowest (axis,
//                    boundary), leaf rule (bvh.py:154-215)
//     k_small        segments of <= kSmallSeg triangles skip the three
//                    kernels above: one warp loads the triangles, reduces
//                    the bounds and evaluates every (axis, boundary) in a
//                    lane of its own, with no bins in memory
//     scan           stable partition ranks (CUB exclusive sum over flags)
//     k_partition    left block first, both order-preserving (bvh.py:213-214)
//     k_children     BFS node ids of the children, next level's segments
//   then subtree sizes bottom-up and preorder ids top-down give the
//   reference's node numbering (left child = i + 1, node_first = right child
//   or leaf start); leaves' triangle ranges are already in preorder.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sahbuild.h"

namespace sbr {

#define CK(x)                                                     \
    do {                                                          \
        cudaError_t e_ = (x);                                     \
        if (e_ != cudaSuccess) return e_;                         \
    } while (0)

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

__device__ __forceinline__ unsigned long long ordd(double x)
{
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double unordd(unsigned long long u)
{
    const unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffULL) : ~u;
    return __longlong_as_double((long long)b);
}
constexpr unsigned long long kOrdPosInf = 0xfff0000000000000ULL;   // ordd(+inf)
constexpr unsigned long long kOrdNegInf = 0x000fffffffffffffULL;   // ordd(-inf)

// per-triangle bounds: tri_min, tri_max, centroid = (min + max) * 0.5
// (bvh.py:227-231), AoS of 9 doubles
__global__ void k_tri_bounds(const double *__restrict__ verts, int64_t n,
                             double *__restrict__ tb, int *__restrict__ idx,
                             int *__restrict__ eseg)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const double *v = verts + 9 * t;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double lo = fmin(fmin(v[a], v[3 + a]), v[6 + a]);
        const double hi = fmax(fmax(v[a], v[3 + a]), v[6 + a]);
        tb[9 * t + a] = lo;
        tb[9 * t + 3 + a] = hi;
        tb[9 * t + 6 + a] = __dmul_rn(__dadd_rn(lo, hi), 0.5);
    }
    idx[t] = (int)t;
    eseg[t] = 0;   // level 0: one segment (later levels: k_partition)
}



constexpr int kSmallSeg = 32;   // segments this small are handled by k_small

__global__ void k_seg_init(SegAcc *__restrict__ acc, unsigned int *__restrict__ cnt,
                           unsigned long long *__restrict__ bbox, int S, int64_t nslots,
                           const int64_t *__restrict__ sc, int64_t slots_per_seg)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < S) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            acc[i].box[q] = kOrdPosInf; acc[i].box[3 + q] = kOrdNegInf;
            acc[i].cb[q] = kOrdPosInf; acc[i].cb[3 + q] = kOrdNegInf;
        }
    }
    if (i < nslots && sc[i / slots_per_seg] > kSmallSeg) {   // small segments: no bins
        cnt[i] = 0u;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            bbox[6 * i + q] = kOrdPosInf;
            bbox[6 * i + 3 + q] = kOrdNegInf;
        }
    }
}

__global__ void k_seg_of(const int64_t *__restrict__ sb, const int64_t *__restrict__ sc, int S,
                         int64_t n, int *__restrict__ eseg)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int lo = 0, hi = S - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (sb[mid] <= i) lo = mid; else hi = mid - 1;
    }
    eseg[i] = (S > 0 && sb[lo] <= i && i < sb[lo] + sc[lo]) ? lo : -1;
}

// Work tiles of the per-element kernels: a block takes kTile consecutive
// elements.  Active segments are contiguous and ordered in element order, so
// a tile spans segments [s_lo, s_hi]; when that is at most kLocalSegs (all
// levels near the root, where every element hits the same few addresses)
// the block reduces into shared memory first and flushes once per value.
constexpr int kTile = 1024;
constexpr int kTileThreads = 256;
constexpr int kLocalSegs = 4;

// [s_lo, s_hi] of the tile's elements that belong to a segment handled by
// the bin kernels (s_hi < 0: none); block-uniform result
__device__ __forceinline__ void tile_range(const int *__restrict__ eseg,
                                           const int64_t *__restrict__ sc, int64_t t0,
                                           int64_t t1, int skip_small, int *srange, int &s_lo,
                                           int &s_hi)
{
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) { srange[0] = 0x7fffffff; srange[1] = -1; }
    __syncthreads();
    int mn = 0x7fffffff, mx = -1;
    for (int64_t i = t0 + tid; i < t1; i += blockDim.x) {
        const int s = eseg[i];
        if (s >= 0 && !(skip_small && sc[s] <= kSmallSeg)) { mn = min(mn, s); mx = max(mx, s); }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0 && mx >= 0) { atomicMin(&srange[0], mn); atomicMax(&srange[1], mx); }
    __syncthreads();
    s_lo = srange[0];
    s_hi = srange[1];
}

// node box + centroid bounds: a warp-segmented pre-reduction per run of
// equal segment ids, then shared (few segments per tile) or global
// ordered-integer atomics -- min/max, exact in any order
__global__ void __launch_bounds__(kTileThreads)
k_bounds(const double *__restrict__ tb, const int *__restrict__ idx,
         const int *__restrict__ eseg, int64_t n, SegAcc *__restrict__ acc,
         const int64_t *__restrict__ sc, int skip_small)
{
    __shared__ unsigned long long sacc[kLocalSegs][12];
    __shared__ int srange[2];
    const int tid = threadIdx.x, lane = tid & 31;
    const int64_t t0 = (int64_t)blockIdx.x * kTile;
    const int64_t t1 = t0 + kTile < n ? t0 + kTile : n;
    int s_lo, s_hi;
    tile_range(eseg, sc, t0, t1, skip_small, srange, s_lo, s_hi);
    if (s_hi < 0) return;                               // block-uniform
    const bool local = s_hi - s_lo < kLocalSegs;
    if (local && tid < kLocalSegs * 12) {
        const int q = tid % 12;
        sacc[tid / 12][q] = (q < 3 || (q >= 6 && q < 9)) ? kOrdPosInf : kOrdNegInf;
    }
    __syncthreads();
    for (int64_t i = t0 + tid; i - lane < t1; i += blockDim.x) {
        int s = i < t1 ? eseg[i] : -1;
        if (skip_small && s >= 0 && sc[s] <= kSmallSeg) s = -1;   // k_small's
        unsigned long long v[12];
        if (s >= 0) {
            const double *b = tb + 9 * (int64_t)idx[i];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                v[q] = ordd(b[q]);            // tri_min   -> min
                v[3 + q] = ordd(b[3 + q]);    // tri_max   -> max
                v[6 + q] = ordd(b[6 + q]);    // centroid  -> min
                v[9 + q] = v[6 + q];          // centroid  -> max
            }
        } else {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                v[q] = kOrdPosInf; v[3 + q] = kOrdNegInf;
                v[6 + q] = kOrdPosInf; v[9 + q] = kOrdNegInf;
            }
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int so = __shfl_down_sync(0xffffffffu, s, o);
            const bool same = lane + o < 32 && so == s;
#pragma unroll
            for (int q = 0; q < 12; ++q) {
                const unsigned long long w = __shfl_down_sync(0xffffffffu, v[q], o);
                if (same) {
                    const bool is_min = (q < 3) || (q >= 6 && q < 9);
                    v[q] = is_min ? (w < v[q] ? w : v[q]) : (w > v[q] ? w : v[q]);
                }
            }
        }
        const int sp = __shfl_up_sync(0xffffffffu, s, 1);
        if (s >= 0 && (lane == 0 || sp != s)) {      // head of its run
            if (local) {
                unsigned long long *L = sacc[s - s_lo];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    atomicMin(&L[q], v[q]);
                    atomicMax(&L[3 + q], v[3 + q]);
                    atomicMin(&L[6 + q], v[6 + q]);
                    atomicMax(&L[9 + q], v[9 + q]);
                }
            } else {
                SegAcc &A = acc[s];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    atomicMin(&A.box[q], v[q]);
                    atomicMax(&A.box[3 + q], v[3 + q]);
                    atomicMin(&A.cb[q], v[6 + q]);
                    atomicMax(&A.cb[3 + q], v[9 + q]);
                }
            }
        }
    }
    if (local) {
        __syncthreads();
        if (tid < (s_hi - s_lo + 1) * 12) {
            const int ls = tid / 12, q = tid % 12;
            const int s = s_lo + ls;
            if (!(skip_small && sc[s] <= kSmallSeg)) {
                const unsigned long long x = sacc[ls][q];
                SegAcc &A = acc[s];
                if (q < 3) atomicMin(&A.box[q], x);
                else if (q < 6) atomicMax(&A.box[q], x);
                else if (q < 9) atomicMin(&A.cb[q - 6], x);
                else atomicMax(&A.cb[q - 6], x);
            }
        }
    }
}

// bin index of a centroid coordinate (bvh.py:181-182): min(int64(scale *
// (c - c_lo)), bins - 1), scale = bins / (c_hi - c_lo)
__device__ __forceinline__ int bin_of(double c, double c_lo, double scale, int nbins)
{
    const long long b = (long long)__dmul_rn(scale, __dsub_rn(c, c_lo));
    return b > nbins - 1 ? nbins - 1 : (int)b;
}

__global__ void __launch_bounds__(kTileThreads)
k_bin(const double *__restrict__ tb, const int *__restrict__ idx,
      const int *__restrict__ eseg, int64_t n, const SegAcc *__restrict__ acc, int nbins,
      int R, unsigned int *__restrict__ cnt, unsigned long long *__restrict__ bbox,
      const int64_t *__restrict__ sc)
{
    const int tid = threadIdx.x;
    const int64_t t0 = (int64_t)blockIdx.x * kTile;
    const int64_t t1 = t0 + kTile < n ? t0 + kTile : n;
    // near the root few segments share every bin: R replicas (chosen by
    // block) spread the global atomics; k_select merges them (exact).
    // Consecutive elements mostly fall into the same bin (the order is
    // spatially coherent), so each axis first reduces runs of lanes with
    // equal (segment, bin) in registers and only run heads touch memory,
    // with fire-and-forget global min / max (shared-memory 64-bit min / max
    // are CAS loops: a block-local pre-reduction was slower).
    const int rep = blockIdx.x % R;
    const int lane = tid & 31;
    for (int64_t i = t0 + tid; i - lane < t1; i += blockDim.x) {
        int s = i < t1 ? eseg[i] : -1;
        if (s >= 0 && sc[s] <= kSmallSeg) s = -1;
        if (!__any_sync(0xffffffffu, s >= 0)) continue;   // all k_small's (deep levels)
        unsigned long long bx[6];
        double cen[3];
        if (s >= 0) {
            const double *b = tb + 9 * (int64_t)idx[i];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                bx[q] = ordd(b[q]);
                bx[3 + q] = ordd(b[3 + q]);
                cen[q] = b[6 + q];
            }
        } else {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                bx[q] = kOrdPosInf;
                bx[3 + q] = kOrdNegInf;
                cen[q] = 0.0;
            }
        }
        const SegAcc *A = acc + (s >= 0 ? s : 0);
#pragma unroll 1
        for (int axis = 0; axis < 3; ++axis) {
            int bi = -1;
            if (s >= 0) {
                const double c_lo = unordd(A->cb[axis]), c_hi = unordd(A->cb[3 + axis]);
                if (c_hi > c_lo)                                // bvh.py:177-178
                    bi = bin_of(cen[axis], c_lo, __ddiv_rn((double)nbins, __dsub_rn(c_hi, c_lo)),
                                nbins);
            }
            unsigned int c = bi >= 0 ? 1u : 0u;
            unsigned long long v[6];
#pragma unroll
            for (int q = 0; q < 6; ++q) v[q] = bx[q];
            // runs of equal (segment, bin): bins are not monotone along the
            // elements, so lanes compare run starts, not keys
            const int sp = __shfl_up_sync(0xffffffffu, s, 1);
            const int bp = __shfl_up_sync(0xffffffffu, bi, 1);
            const bool head = lane == 0 || sp != s || bp != bi;
            const unsigned heads = __ballot_sync(0xffffffffu, head);
            const int rs = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int ro = __shfl_down_sync(0xffffffffu, rs, o);
                const unsigned int co = __shfl_down_sync(0xffffffffu, c, o);
                const bool same = lane + o < 32 && ro == rs;
                if (same) c += co;
#pragma unroll
                for (int q = 0; q < 6; ++q) {
                    const unsigned long long w = __shfl_down_sync(0xffffffffu, v[q], o);
                    if (same) v[q] = q < 3 ? (w < v[q] ? w : v[q]) : (w > v[q] ? w : v[q]);
                }
            }
            if (bi >= 0 && head) {                                  // head of its run
                const int64_t slot = (((int64_t)s * R + rep) * 3 + axis) * nbins + bi;
                unsigned int *cp = cnt + slot;
                unsigned long long *bb = bbox + 6 * slot;
                atomicAdd(cp, c);
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    atomicMin(&bb[q], v[q]);
                    atomicMax(&bb[3 + q], v[3 + q]);
                }
            }
        }
    }
}

// _box_surface_area (bvh.py:130-132): 2 * (d0 d1 + d1 d2 + d2 d0)
__device__ __forceinline__ double sa_of(const double lo[3], const double hi[3])
{
    const double d0 = __dsub_rn(hi[0], lo[0]), d1 = __dsub_rn(hi[1], lo[1]),
                 d2 = __dsub_rn(hi[2], lo[2]);
    return __dmul_rn(2.0, __dadd_rn(__dadd_rn(__dmul_rn(d0, d1), __dmul_rn(d1, d2)),
                                    __dmul_rn(d2, d0)));
}



// one warp per segment: node box out, split decision (bvh.py:154-215 and
// the leaf test of bvh.py:253-262).  Lanes merge the bin replicas, lanes
// 0..2 sweep one axis each, lane 0 picks the first minimum in (axis,
// boundary) order -- the reference's strict-< scan order.
constexpr int kSelWarps = 4;

__global__ void __launch_bounds__(kSelWarps * 32)
k_select(const SegAcc *__restrict__ acc, const unsigned int *__restrict__ cnt,
         const unsigned long long *__restrict__ bbox, const int64_t *__restrict__ sc,
         const int *__restrict__ snode, int S, int R, int depth, SahParams P,
         double *__restrict__ node_box, SegSplit *__restrict__ out,
         int *__restrict__ split_flag)
{
    __shared__ int64_t sbc[kSelWarps][3][kSahMaxBins];
    __shared__ double smn[kSelWarps][3][3][kSahMaxBins], smx[kSelWarps][3][3][kSahMaxBins];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * kSelWarps + w;
    if (s >= S || sc[s] <= kSmallSeg) return;         // warp-uniform; small: k_small
    const SegAcc &A = acc[s];
    double lo[3], hi[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        lo[q] = unordd(A.box[q]);
        hi[q] = unordd(A.box[3 + q]);
    }
    if (lane == 0) {
        double *nb = node_box + 6 * (int64_t)snode[s];
#pragma unroll
        for (int q = 0; q < 3; ++q) { nb[q] = lo[q]; nb[3 + q] = hi[q]; }
    }
    SegSplit r;
    r.split = 0; r.axis = -1; r.boundary = -1; r.c_lo = 0.0; r.scale = 0.0; r.nl = 0;
    const int64_t n = sc[s];
    const int B = P.bins;
    if (n > P.n_leaf && depth < P.max_depth) {
        // merge the replicas of every (axis, bin) (exact: min / max / sum)
        for (int idx = lane; idx < 3 * B; idx += 32) {
            const int axis = idx / B, b = idx - axis * B;
            unsigned long long mn[3] = {kOrdPosInf, kOrdPosInf, kOrdPosInf};
            unsigned long long mx[3] = {kOrdNegInf, kOrdNegInf, kOrdNegInf};
            int64_t c = 0;
#pragma unroll 4
            for (int rep = 0; rep < R; ++rep) {
                const int64_t slot = (((int64_t)s * R + rep) * 3 + axis) * B + b;
                const unsigned long long *bb = bbox + 6 * slot;
                c += cnt[slot];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    mn[q] = bb[q] < mn[q] ? bb[q] : mn[q];
                    mx[q] = bb[3 + q] > mx[q] ? bb[3 + q] : mx[q];
                }
            }
            sbc[w][axis][b] = c;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                smn[w][q][axis][b] = unordd(mn[q]);
                smx[w][q][axis][b] = unordd(mx[q]);
            }
        }
        __syncwarp();
        double sa_p = sa_of(lo, hi);
        if (!(sa_p >= 1e-300)) sa_p = 1e-300;          // max(sa, 1e-300)
        // every (axis, boundary) candidate in a lane of its own: the child
        // boxes are unions over bins (exact in any order), so the counts,
        // boxes and costs are those of the reference's running sweep; the
        // warp then takes the first minimum in (axis, boundary) order, the
        // reference's strict-< scan (bvh.py:175-207)
        bool ok[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) ok[q] = unordd(A.cb[3 + q]) > unordd(A.cb[q]);   // bvh.py:177-178
        bool have = false;
        double best = 0.0;
        int best_c = 0x7fffffff;
        long long best_nl = 0;
        const int ncand = 3 * (B - 1);
        for (int cand = lane; cand < ncand; cand += 32) {
            const int axis = cand / (B - 1), b = cand - axis * (B - 1);
            if (!ok[axis]) continue;
            double l3[3] = {INFINITY, INFINITY, INFINITY}, h3[3] = {-INFINITY, -INFINITY, -INFINITY};
            double r3[3] = {INFINITY, INFINITY, INFINITY}, g3[3] = {-INFINITY, -INFINITY, -INFINITY};
            long long ln = 0, nr = 0;
            for (int k = 0; k < B; ++k) {
                const long long c = sbc[w][axis][k];
                if (k <= b) {
                    ln += c;
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        l3[q] = fmin(l3[q], smn[w][q][axis][k]);
                        h3[q] = fmax(h3[q], smx[w][q][axis][k]);
                    }
                } else {
                    nr += c;
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        r3[q] = fmin(r3[q], smn[w][q][axis][k]);
                        g3[q] = fmax(g3[q], smx[w][q][axis][k]);
                    }
                }
            }
            if (ln == 0 || nr == 0) continue;
            const double sal = sa_of(l3, h3), sar = sa_of(r3, g3);
            // sah_cost (bvh.py:124-127): c_t + (sal/sa_p) n_l c_i + (sar/sa_p) n_r c_i
            const double cost = __dadd_rn(
                __dadd_rn(P.c_t, __dmul_rn(__dmul_rn(__ddiv_rn(sal, sa_p), (double)ln), P.c_i)),
                __dmul_rn(__dmul_rn(__ddiv_rn(sar, sa_p), (double)nr), P.c_i));
            if (!have || cost < best) {   // candidates ascend per lane: keeps the first
                have = true;
                best = cost;
                best_c = cand;
                best_nl = ln;
            }
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const int oh = __shfl_xor_sync(0xffffffffu, (int)have, o);
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oc = __shfl_xor_sync(0xffffffffu, best_c, o);
            const long long on = __shfl_xor_sync(0xffffffffu, best_nl, o);
            if (oh && (!have || ob < best || (ob == best && oc < best_c))) {
                have = true; best = ob; best_c = oc; best_nl = on;
            }
        }
        if (lane == 0) {
            if (have) {
                r.axis = best_c / (B - 1);
                r.boundary = best_c - r.axis * (B - 1);
                r.nl = best_nl;
                const double c_lo = unordd(A.cb[r.axis]), c_hi = unordd(A.cb[3 + r.axis]);
                r.c_lo = c_lo;
                r.scale = __ddiv_rn((double)B, __dsub_rn(c_hi, c_lo));
            }
            // bvh.py:210-211: no admissible split, or not worth it for a small node
            if (have && !(best >= __dmul_rn((double)n, P.c_i) && n <= 4 * (int64_t)P.n_leaf))
                r.split = 1;
        }
    }
    if (lane == 0) {
        out[s] = r;
        split_flag[s] = r.split;
    }
}

// Segments of at most kSmallSeg triangles (most of the deep levels): one
// warp per segment, no bins in memory.  Lane l holds triangle l; the node
// box and centroid bounds are butterfly reductions on the same ordered
// integers k_bounds uses (bit-identical boxes, -0.0 < +0.0 included).  Each
// (axis, boundary) candidate then gets a lane that unions the triangles on
// either side: the same counts and the same child boxes as the bin sweep of
// k_select (a union over bins is a union over their triangles; signed zeros
// cannot change a surface area), hence the same costs, and the warp picks
// the first minimum in (axis, boundary) order as the reference scan does.
constexpr int kSmallWarps = 4;

__global__ void __launch_bounds__(kSmallWarps * 32)
k_small(const double *__restrict__ tb, const int *__restrict__ idx,
        const int64_t *__restrict__ sb, const int64_t *__restrict__ sc,
        const int *__restrict__ snode, int S, int depth, SahParams P,
        double *__restrict__ node_box, SegSplit *__restrict__ out, int *__restrict__ split_flag)
{
    __shared__ double sbox[kSmallWarps][6][kSmallSeg];
    __shared__ unsigned char sbin[kSmallWarps][3][kSmallSeg];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s = blockIdx.x * kSmallWarps + w;
    if (s >= S) return;
    const int64_t n64 = sc[s];
    if (n64 > kSmallSeg) return;                      // warp-uniform
    const int n = (int)n64;
    unsigned long long v[12];
    double c[3] = {0.0, 0.0, 0.0};
    if (lane < n) {
        const double *b = tb + 9 * (int64_t)idx[sb[s] + lane];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            sbox[w][q][lane] = b[q];
            sbox[w][3 + q][lane] = b[3 + q];
            c[q] = b[6 + q];
            v[q] = ordd(b[q]);
            v[3 + q] = ordd(b[3 + q]);
            v[6 + q] = ordd(c[q]);
            v[9 + q] = v[6 + q];
        }
    } else {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            v[q] = kOrdPosInf; v[3 + q] = kOrdNegInf;
            v[6 + q] = kOrdPosInf; v[9 + q] = kOrdNegInf;
        }
    }
    // butterfly over the 2^ceil(log2 n) lanes that hold triangles: lane 0
    // (and its group) ends with the full reduction; the other lanes get it
    // by broadcast when they take part in the candidate sweep
    const bool leaf = !(n > P.n_leaf && depth < P.max_depth);
    const int span = n <= 1 ? 1 : 1 << (32 - __clz(n - 1));
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        if (o >= span) break;                          // warp-uniform
#pragma unroll
        for (int q = 0; q < 12; ++q) {
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, v[q], o);
            const bool is_min = (q < 3) || (q >= 6 && q < 9);
            v[q] = is_min ? (x < v[q] ? x : v[q]) : (x > v[q] ? x : v[q]);
        }
    }
    if (!leaf && span < 32) {
#pragma unroll
        for (int q = 0; q < 12; ++q) v[q] = __shfl_sync(0xffffffffu, v[q], 0);
    }
    double lo[3], hi[3], clo[3], chi[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        lo[q] = unordd(v[q]); hi[q] = unordd(v[3 + q]);
        clo[q] = unordd(v[6 + q]); chi[q] = unordd(v[9 + q]);
    }
    if (lane == 0) {
        double *nb = node_box + 6 * (int64_t)snode[s];
#pragma unroll
        for (int q = 0; q < 3; ++q) { nb[q] = lo[q]; nb[3 + q] = hi[q]; }
    }
    SegSplit r;
    r.split = 0; r.axis = -1; r.boundary = -1; r.c_lo = 0.0; r.scale = 0.0; r.nl = 0;
    const int B = P.bins;
    if (!leaf) {
        double scale[3];
        unsigned occ[3];   // bins holding a triangle (B <= 32)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            scale[q] = chi[q] > clo[q] ? __ddiv_rn((double)B, __dsub_rn(chi[q], clo[q])) : 0.0;
            const int bq = lane < n ? bin_of(c[q], clo[q], scale[q], B) : 0;
            if (lane < n) sbin[w][q][lane] = (unsigned char)bq;
            occ[q] = __reduce_or_sync(0xffffffffu, lane < n && bq < 32 ? 1u << bq : 0u);
        }
        __syncwarp();
        double sa_p = sa_of(lo, hi);
        if (!(sa_p >= 1e-300)) sa_p = 1e-300;          // max(sa, 1e-300)
        // Boundary b moves exactly the triangles of bin b to the left, so a
        // boundary after an empty bin repeats the previous partition (same
        // cost, later in the scan: never chosen) or has an empty side.  With
        // B <= 32 only the boundaries after occupied bins are evaluated,
        // packed onto the lanes (one round instead of two for n <= 10).
        const bool packed = B <= 32;
        const unsigned bmask = B >= 33 ? 0xffffffffu : (1u << (B - 1)) - 1u;
        int nc[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) nc[q] = chi[q] > clo[q] ? __popc(occ[q] & bmask) : 0;
        // best candidate of this lane over the rounds: (have, cost, index)
        bool have = false;
        double best = 0.0;
        int best_c = 0x7fffffff, best_nl = 0;
        const int ncand = packed ? nc[0] + nc[1] + nc[2] : 3 * (B - 1);
        for (int k = lane; k < ncand; k += 32) {
            int axis, b;
            if (packed) {   // k-th occupied boundary in (axis, boundary) order
                axis = k < nc[0] ? 0 : (k < nc[0] + nc[1] ? 1 : 2);
                const int kk = k - (axis > 0 ? nc[0] : 0) - (axis > 1 ? nc[1] : 0);
                b = (int)__fns(occ[axis] & bmask, 0, kk + 1);
            } else {
                axis = k / (B - 1);
                b = k - axis * (B - 1);
            }
            const int cand = axis * (B - 1) + b;
            if (!(chi[axis] > clo[axis])) continue;     // bvh.py:177-178
            double l3[3] = {INFINITY, INFINITY, INFINITY}, h3[3] = {-INFINITY, -INFINITY, -INFINITY};
            double r3[3] = {INFINITY, INFINITY, INFINITY}, g3[3] = {-INFINITY, -INFINITY, -INFINITY};
            int ln = 0;
            for (int t = 0; t < n; ++t) {
                if (sbin[w][axis][t] <= b) {
                    ++ln;
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        l3[q] = fmin(l3[q], sbox[w][q][t]);
                        h3[q] = fmax(h3[q], sbox[w][3 + q][t]);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        r3[q] = fmin(r3[q], sbox[w][q][t]);
                        g3[q] = fmax(g3[q], sbox[w][3 + q][t]);
                    }
                }
            }
            const int nr = n - ln;
            if (ln == 0 || nr == 0) continue;
            const double sal = sa_of(l3, h3), sar = sa_of(r3, g3);
            // sah_cost (bvh.py:124-127), same association as k_select
            const double cost = __dadd_rn(
                __dadd_rn(P.c_t, __dmul_rn(__dmul_rn(__ddiv_rn(sal, sa_p), (double)ln), P.c_i)),
                __dmul_rn(__dmul_rn(__ddiv_rn(sar, sa_p), (double)nr), P.c_i));
            if (!have || cost < best) {   // candidates ascend per lane: keeps the first
                have = true;
                best = cost;
                best_c = cand;
                best_nl = ln;
            }
        }
        // warp argmin: lowest cost, then lowest candidate index
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const int oh = __shfl_xor_sync(0xffffffffu, (int)have, o);
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oc = __shfl_xor_sync(0xffffffffu, best_c, o);
            const int on = __shfl_xor_sync(0xffffffffu, best_nl, o);
            if (oh && (!have || ob < best || (ob == best && oc < best_c))) {
                have = true; best = ob; best_c = oc; best_nl = on;
            }
        }
        if (have) {
            r.axis = best_c / (B - 1);
            r.boundary = best_c - r.axis * (B - 1);
            r.nl = best_nl;
            r.c_lo = clo[r.axis];
            r.scale = scale[r.axis];
        }
        // bvh.py:210-211: no admissible split, or not worth it for a small node
        if (have && !(best >= __dmul_rn((double)n, P.c_i) && n <= 4 * (int64_t)P.n_leaf))
            r.split = 1;
    }
    if (lane == 0) {
        out[s] = r;
        split_flag[s] = r.split;
    }
}

// median split (bvh.py:135-151): split along the longest axis of the node box
// (np.argmax: first maximum) unless every centroid coincides; the left child
// takes the n // 2 first elements of the stable (centroid, position) order
__global__ void k_select_median(const SegAcc *__restrict__ acc, const int64_t *__restrict__ sc,
                                const int *__restrict__ snode, int S, int depth, SahParams P,
                                double *__restrict__ node_box, SegSplit *__restrict__ out,
                                int *__restrict__ split_flag)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const SegAcc &A = acc[s];
    double lo[3], hi[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        lo[q] = unordd(A.box[q]);
        hi[q] = unordd(A.box[3 + q]);
    }
    double *nb = node_box + 6 * (int64_t)snode[s];
#pragma unroll
    for (int q = 0; q < 3; ++q) { nb[q] = lo[q]; nb[3 + q] = hi[q]; }
    SegSplit r;
    r.split = 0; r.axis = -1; r.boundary = -1; r.c_lo = 0.0; r.scale = 0.0; r.nl = 0;
    const int64_t n = sc[s];
    bool same = true;
#pragma unroll
    for (int q = 0; q < 3; ++q) same = same && A.cb[q] == A.cb[3 + q];
    if (n > P.n_leaf && depth < P.max_depth && !same) {
        const double e0 = __dsub_rn(hi[0], lo[0]), e1 = __dsub_rn(hi[1], lo[1]),
                     e2 = __dsub_rn(hi[2], lo[2]);
        int axis = 0;
        double best = e0;
        if (e1 > best) { best = e1; axis = 1; }
        if (e2 > best) axis = 2;
        r.split = 1;
        r.axis = axis;
        r.nl = n / 2;
    }
    out[s] = r;
    split_flag[s] = r.split;
}

// sort keys (centroid on the split axis; -0.0 folded onto +0.0 as np.lexsort
// compares them equal) for elements of split segments
__global__ void k_median_keys(const double *__restrict__ tb, const int *__restrict__ idx,
                              const int *__restrict__ eseg, int64_t n,
                              const SegSplit *__restrict__ sp, double *__restrict__ key)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int s = eseg[i];
    key[i] = (s >= 0 && sp[s].split) ? tb[9 * (int64_t)idx[i] + 6 + sp[s].axis] + 0.0 : 0.0;
}

__global__ void k_split_offsets(int S, const int *__restrict__ sflag, const int *__restrict__ crank,
                                const int64_t *__restrict__ sb, const int64_t *__restrict__ sc,
                                int64_t *__restrict__ beg, int64_t *__restrict__ end)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S || !sflag[s]) return;
    beg[crank[s]] = sb[s];
    end[crank[s]] = sb[s] + sc[s];
}

__global__ void k_flags(const double *__restrict__ tb, const int *__restrict__ idx,
                        const int *__restrict__ eseg, int64_t n,
                        const SegSplit *__restrict__ sp, int nbins, int *__restrict__ flag)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int s = eseg[i];
    int f = 0;
    if (s >= 0 && sp[s].split) {
        const SegSplit &r = sp[s];
        const double c = tb[9 * (int64_t)idx[i] + 6 + r.axis];
        f = bin_of(c, r.c_lo, r.scale, nbins) <= r.boundary;
    }
    flag[i] = f;
}

// also the next level's element -> segment map: the children of split
// segment s are segments 2 crank[s] (left) and 2 crank[s] + 1 (k_children),
// elements of unsplit segments belong to none
__global__ void k_partition(const int *__restrict__ idx, const int *__restrict__ eseg,
                            int64_t n, const SegSplit *__restrict__ sp,
                            const int64_t *__restrict__ sb, const int *__restrict__ flag,
                            const int *__restrict__ rank, const int *__restrict__ crank,
                            int *__restrict__ out, int *__restrict__ eseg_next)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int s = eseg[i];
    int64_t dst = i;
    int ns = -1;
    if (s >= 0 && sp[s].split) {
        const int64_t b = sb[s];
        const int64_t left = (int64_t)rank[i] - rank[b];       // flags before i in segment
        dst = flag[i] ? b + left : b + sp[s].nl + ((i - b) - left);
        ns = 2 * crank[s] + (flag[i] ? 0 : 1);
    }
    out[dst] = idx[i];
    eseg_next[dst] = ns;
}

// children of split segments -> next level; leaves recorded
__global__ void k_children(int S, const SegSplit *__restrict__ sp, const int *__restrict__ crank,
                           const int64_t *__restrict__ sb, const int64_t *__restrict__ sc,
                           const int *__restrict__ snode, int node_base,
                           int *__restrict__ left, int *__restrict__ right,
                           int64_t *__restrict__ leaf_first, int64_t *__restrict__ leaf_count,
                           int64_t *__restrict__ nsb, int64_t *__restrict__ nsc,
                           int *__restrict__ nsnode)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const int me = snode[s];
    if (!sp[s].split) {
        left[me] = -1;
        right[me] = -1;
        leaf_first[me] = sb[s];
        leaf_count[me] = sc[s];
        return;
    }
    const int k = crank[s];                 // index among split segments
    const int l = node_base + 2 * k, r = l + 1;
    left[me] = l;
    right[me] = r;
    leaf_count[me] = 0;
    nsb[2 * k] = sb[s];
    nsc[2 * k] = sp[s].nl;
    nsnode[2 * k] = l;
    nsb[2 * k + 1] = sb[s] + sp[s].nl;
    nsc[2 * k + 1] = sc[s] - sp[s].nl;
    nsnode[2 * k + 1] = r;
}

__global__ void k_sizes(int a, int b, const int *__restrict__ left, const int *__restrict__ right,
                        int64_t *__restrict__ size)
{
    const int i = a + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= b) return;
    size[i] = left[i] < 0 ? 1 : 1 + size[left[i]] + size[right[i]];
}

__global__ void k_preorder(int a, int b, const int *__restrict__ left,
                           const int *__restrict__ right, const int64_t *__restrict__ size,
                           int64_t *__restrict__ pre)
{
    const int i = a + blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= b || left[i] < 0) return;
    pre[left[i]] = pre[i] + 1;
    pre[right[i]] = pre[i] + 1 + size[left[i]];
}

__global__ void k_emit_ref(int N, const int64_t *__restrict__ pre, const double *__restrict__ box,
                           const int *__restrict__ right, const int64_t *__restrict__ lf,
                           const int64_t *__restrict__ lc, double *__restrict__ nmin,
                           double *__restrict__ nmax, int32_t *__restrict__ first,
                           int32_t *__restrict__ count)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int64_t p = pre[i];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        nmin[3 * p + q] = box[6 * (int64_t)i + q];
        nmax[3 * p + q] = box[6 * (int64_t)i + 3 + q];
    }
    if (right[i] < 0) {
        first[p] = (int32_t)lf[i];
        count[p] = (int32_t)lc[i];
    } else {
        first[p] = (int32_t)pre[right[i]];
        count[p] = 0;
    }
}

// reference-layout tree (device) -> child-pair BVH2 nodes for traversal:
// one Node per internal reference node, numbered by an exclusive scan of the
// internal flags (root stays 0); boxes relative to the frame, rounded
// outward to float exactly as the host UploadBuilder does
__global__ void k_ref_flags(int N, const int32_t *__restrict__ count, int *__restrict__ flag,
                            int *__restrict__ big)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    flag[i] = count[i] == 0;
    if (count[i] > kMaxLeafCount) atomicOr(big, 1);
}

__global__ void k_ref_nodes(int N, const double *__restrict__ nmin, const double *__restrict__ nmax,
                            const int32_t *__restrict__ first, const int32_t *__restrict__ count,
                            const int *__restrict__ rank, double3 frame, Node *__restrict__ out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N || count[i] != 0) return;
    const int kids[2] = {i + 1, first[i]};
    float b[2][6];
    int ref[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const int k = kids[c];
        const double f[3] = {frame.x, frame.y, frame.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            b[c][a] = nextafterf(__double2float_rn(nmin[3 * (int64_t)k + a] - f[a]), -INFINITY);
            b[c][3 + a] = nextafterf(__double2float_rn(nmax[3 * (int64_t)k + a] - f[a]), INFINITY);
        }
        ref[c] = count[k] > 0 ? leaf_ref(first[k], count[k]) : rank[k];
    }
    Node nd;
    nd.a = make_float4(b[0][0], b[0][1], b[0][2], b[0][3]);
    nd.b = make_float4(b[0][4], b[0][5], b[1][0], b[1][1]);
    nd.c = make_float4(b[1][2], b[1][3], b[1][4], b[1][5]);
    nd.d = make_int4(ref[0], ref[1], 0, 0);
    out[rank[i]] = nd;
}

cudaError_t ref_to_bvh2(const SahTree &t, const double frame[3], SahWork &w, LbvhOutput &out,
                        bool &host_needed, cudaStream_t st, int64_t *launches)
{
    const int N = (int)t.nnodes;
    host_needed = false;
    CK(w.flag.reserve(N + 1));
    CK(w.rank.reserve(N + 1));
    CK(w.big.reserve(1));
    CK(cudaMemsetAsync(w.big.p, 0, sizeof(int), st));
    CK(cudaMemsetAsync(w.flag.p + N, 0, sizeof(int), st));
    k_ref_flags<<<nblk(N, 256), 256, 0, st>>>(N, t.count.p, w.flag.p, w.big.p);
    size_t need = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, need, w.flag.p, w.rank.p, N + 1, st));
    CK(w.scan_tmp.reserve(need));
    CK(cub::DeviceScan::ExclusiveSum(w.scan_tmp.p, need, w.flag.p, w.rank.p, N + 1, st));
    int big = 0, internal = 0, root_count = 0;
    CK(cudaMemcpyAsync(&big, w.big.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&internal, w.rank.p + N, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&root_count, t.count.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (big || root_count > 0) {           // leaf > 63 triangles or a leaf root
        host_needed = true;
        return cudaSuccess;
    }
    CK(out.nodes.alloc(internal));
    k_ref_nodes<<<nblk(N, 256), 256, 0, st>>>(N, t.nmin.p, t.nmax.p, t.first.p, t.count.p,
                                              w.rank.p, make_double3(frame[0], frame[1], frame[2]),
                                              out.nodes.p);
    *launches += 3;
    CK(cudaGetLastError());
    out.nnodes = internal;
    out.root = 0;
    out.max_depth = t.max_depth;
    return cudaSuccess;
}

cudaError_t sah_build(const double *d_verts, int64_t n, const SahParams &P, SahTree &out,
                      SahWork &w, cudaStream_t st, int64_t *launches)
{
    if (n < 1 || P.bins < 2 || P.bins > kSahMaxBins) return cudaErrorInvalidValue;
    const int T = 256;
    const int B = P.bins;
    const int64_t max_nodes = 2 * n;   // binary tree with >= 1 triangle per leaf
    CK(w.tb.reserve(9 * (size_t)n));
    CK(w.idx.reserve(n)); CK(w.idx2.reserve(n)); CK(w.eseg.reserve(n)); CK(w.eseg2.reserve(n));
    CK(w.flag.reserve(n + 1)); CK(w.rank.reserve(n + 1));
    CK(w.node_box.reserve(6 * (size_t)max_nodes));
    CK(w.left.reserve(max_nodes)); CK(w.right.reserve(max_nodes));
    CK(w.lf.reserve(max_nodes)); CK(w.lc.reserve(max_nodes));
    CK(w.size.reserve(max_nodes)); CK(w.pre.reserve(max_nodes));
    CK(w.sb.reserve(n)); CK(w.sc.reserve(n)); CK(w.nsb.reserve(n)); CK(w.nsc.reserve(n));
    CK(w.snode.reserve(n)); CK(w.nsnode.reserve(n));
    CK(w.crank.reserve(n + 1)); CK(w.sflag.reserve(n + 1));
    CK(w.acc.reserve(n)); CK(w.sp.reserve(n));
    size_t scan_bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int *)nullptr, (int *)nullptr,
                                     (int)(n + 1), st));
    CK(w.scan_tmp.reserve(scan_bytes));
    scan_bytes = w.scan_tmp.bytes();
    int *idx = w.idx.p, *idx2 = w.idx2.p;
    int64_t *sb = w.sb.p, *sc = w.sc.p, *nsb = w.nsb.p, *nsc = w.nsc.p;
    int *snode = w.snode.p, *nsnode = w.nsnode.p;

    int *eseg = w.eseg.p, *eseg2 = w.eseg2.p;
    k_tri_bounds<<<nblk(n, T), T, 0, st>>>(d_verts, n, w.tb.p, idx, eseg);
    ++*launches;
    const int64_t zero64 = 0;
    const int zero = 0;
    CK(cudaMemcpyAsync(sb, &zero64, 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(sc, &n, 8, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(snode, &zero, 4, cudaMemcpyHostToDevice, st));
    int S = 1, node_count = 1, depth = 0;
    std::vector<int> level_start{0};
    const bool timing = getenv("SBR_SAH_TIMING") != nullptr;
    while (S > 0) {
        cudaEvent_t lv0 = nullptr, lv1 = nullptr;
        if (timing) {
            cudaEventCreate(&lv0); cudaEventCreate(&lv1);
            cudaEventRecord(lv0, st);
        }
        // bin replicas near the root (k_bin spreads its run heads over them,
        // k_select merges them): 8 measured best of 1..32 (build 7.15 ->
        // 6.96 ms against 32; fewer replicas to merge in k_select's warp)
        const int R = S >= 4096 ? 1 : std::min(8, 4096 / S);
        const int64_t nslots = (int64_t)S * R * 3 * B;
        // grow geometrically so a build allocates O(log) times
        if ((size_t)nslots > w.cnt.n) {
            const size_t cap = std::max<size_t>((size_t)nslots, 2 * w.cnt.n);
            CK(w.cnt.alloc(cap));
            CK(w.bbox.alloc(6 * cap));
        }
        k_seg_init<<<nblk(std::max<int64_t>(nslots, S), T), T, 0, st>>>(
            w.acc.p, w.cnt.p, w.bbox.p, S, nslots, sc, (int64_t)R * 3 * B);
        if (P.median && depth > 0) {   // SAH levels get the map from k_partition
            k_seg_of<<<nblk(n, T), T, 0, st>>>(sb, sc, S, n, eseg);
            ++*launches;
        }
        k_bounds<<<nblk(n, kTile), kTileThreads, 0, st>>>(w.tb.p, idx, eseg, n, w.acc.p, sc,
                                                          !P.median);
        CK(cudaMemsetAsync(w.sflag.p + S, 0, sizeof(int), st));
        if (!P.median) {
            k_bin<<<nblk(n, kTile), kTileThreads, 0, st>>>(w.tb.p, idx, eseg, n, w.acc.p, B,
                                                           R, w.cnt.p, w.bbox.p, sc);
            k_select<<<nblk(S, kSelWarps), kSelWarps * 32, 0, st>>>(
                w.acc.p, w.cnt.p, w.bbox.p, sc, snode, S, R, depth, P, w.node_box.p, w.sp.p,
                w.sflag.p);
            k_small<<<nblk(S, kSmallWarps), kSmallWarps * 32, 0, st>>>(
                w.tb.p, idx, sb, sc, snode, S, depth, P, w.node_box.p, w.sp.p, w.sflag.p);
            ++*launches;
        } else {
            k_select_median<<<nblk(S, 128), 128, 0, st>>>(w.acc.p, sc, snode, S, depth, P,
                                                          w.node_box.p, w.sp.p, w.sflag.p);
        }
        // split flags of the segments -> child slots (exclusive scan; the
        // extra element S receives the total)
        CK(cub::DeviceScan::ExclusiveSum(w.scan_tmp.p, scan_bytes, w.sflag.p, w.crank.p, S + 1,
                                         st));
        if (!P.median) {
            k_flags<<<nblk(n, T), T, 0, st>>>(w.tb.p, idx, eseg, n, w.sp.p, B, w.flag.p);
            CK(cub::DeviceScan::ExclusiveSum(w.scan_tmp.p, scan_bytes, w.flag.p, w.rank.p,
                                             (int)n, st));
            k_partition<<<nblk(n, T), T, 0, st>>>(idx, eseg, n, w.sp.p, sb, w.flag.p,
                                                  w.rank.p, w.crank.p, idx2, eseg2);
            std::swap(eseg, eseg2);
        } else {
            // stable sort of each split segment by its centroid key; the
            // other positions keep their order
            int nsp = 0;
            CK(cudaMemcpyAsync(&nsp, w.crank.p + S, sizeof(int), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            CK(cudaMemcpyAsync(idx2, idx, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
            if (nsp > 0) {
                CK(w.key.reserve(n)); CK(w.key2.reserve(n));
                CK(w.sbeg.reserve(nsp)); CK(w.send.reserve(nsp));
                k_median_keys<<<nblk(n, T), T, 0, st>>>(w.tb.p, idx, eseg, n, w.sp.p,
                                                        w.key.p);
                k_split_offsets<<<nblk(S, 128), 128, 0, st>>>(S, w.sflag.p, w.crank.p, sb, sc,
                                                              w.sbeg.p, w.send.p);
                size_t need = 0;
                CK(cub::DeviceSegmentedSort::StableSortPairs(
                    nullptr, need, w.key.p, w.key2.p, idx, idx2, (int)n, nsp, w.sbeg.p, w.send.p,
                    st));
                CK(w.sort_tmp.reserve(need));
                CK(cub::DeviceSegmentedSort::StableSortPairs(
                    w.sort_tmp.p, need, w.key.p, w.key2.p, idx, idx2, (int)n, nsp, w.sbeg.p,
                    w.send.p, st));
            }
        }
        std::swap(idx, idx2);
        k_children<<<nblk(S, 128), 128, 0, st>>>(S, w.sp.p, w.crank.p, sb, sc, snode, node_count,
                                                 w.left.p, w.right.p, w.lf.p, w.lc.p, nsb, nsc,
                                                 nsnode);
        *launches += 8;
        CK(cudaGetLastError());
        int nsplit = 0;
        CK(cudaMemcpyAsync(&nsplit, w.crank.p + S, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (timing) {
            cudaEventRecord(lv1, st);
            cudaEventSynchronize(lv1);
            float m = 0.f;
            cudaEventElapsedTime(&m, lv0, lv1);
            fprintf(stderr, "[sah] level %d: %d segments, %d split, %.3f ms\n", depth, S, nsplit, m);
            cudaEventDestroy(lv0); cudaEventDestroy(lv1);
        }
        std::swap(sb, nsb);
        std::swap(sc, nsc);
        std::swap(snode, nsnode);
        level_start.push_back(node_count);
        node_count += 2 * nsplit;
        S = 2 * nsplit;
        if (S > 0) ++depth;
    }
    const int N = node_count;
    const int L = (int)level_start.size() - 1;
    for (int l = L - 1; l >= 0; --l) {
        const int a = level_start[l], b = level_start[l + 1];
        if (b > a) k_sizes<<<nblk(b - a, T), T, 0, st>>>(a, b, w.left.p, w.right.p, w.size.p);
    }
    CK(cudaMemsetAsync(w.pre.p, 0, 8, st));
    for (int l = 0; l < L; ++l) {
        const int a = level_start[l], b = level_start[l + 1];
        if (b > a)
            k_preorder<<<nblk(b - a, T), T, 0, st>>>(a, b, w.left.p, w.right.p, w.size.p, w.pre.p);
    }
    CK(out.nmin.alloc(3 * (size_t)N)); CK(out.nmax.alloc(3 * (size_t)N));
    CK(out.first.alloc(N)); CK(out.count.alloc(N)); CK(out.order.alloc(n));
    k_emit_ref<<<nblk(N, T), T, 0, st>>>(N, w.pre.p, w.node_box.p, w.right.p, w.lf.p, w.lc.p,
                                         out.nmin.p, out.nmax.p, out.first.p, out.count.p);
    CK(cudaMemcpyAsync(out.order.p, idx, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));
    *launches += 2 * L + 1;
    CK(cudaGetLastError());
    out.nnodes = N;
    out.max_depth = depth;
    return cudaSuccess;
}

}  // namespace sbr
