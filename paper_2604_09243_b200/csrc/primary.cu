// primary.cu -- primary visibility by rasterising triangles into the launch
// grid (query 0 of every ray, transport.py:293-296 with t_min = 0, t_max = inf).
//
// All primary rays of one aperture share the direction k and start on a
// regular grid: origin(i, j) = corner + ((i+.5) ds) u + ((j+.5) ds) v
// (transport.py:339-345).  A ray can only be accepted by a triangle's
// Moller-Trumbore test if it passes through the triangle (edge-inclusive, up
// to rounding far below a cell), i.e. if its cell centre lies in the
// triangle's projection onto the aperture plane.  So instead of one BVH
// traversal per ray, every (grid, triangle) pair enumerates the cells of its
// projected bounding box widened by kMargin cells and evaluates the SAME exact
// FP64 test on each (bit-identical origin; d x e2 and 1/det hoisted: they do
// not depend on the origin).  The closest hit is the lexicographic minimum
// of (t, id) over accepted triangles (bvh.py:340), order-independent, so a
// 128-bit compare-and-swap minimum on (t bits, id) produces it exactly
// (t > 0, so IEEE bits order as t).  Misses cost nothing.
//
// Work layout: a warp owns 32 (grid, triangle) items of ONE grid (triangles
// padded per grid to a multiple of 32).  Lanes set up their triangle, a warp
// scan of the candidate counts flattens the 32 bounding boxes into one
// candidate list, and the warp walks that list 32 candidates at a time with
// the triangle set-ups read from shared memory -- full lanes regardless of
// how unevenly the triangles cover the grid.
#include "pipeline.h"

namespace sbr {

constexpr double kMargin = 0.01;   // cells; >> every projection rounding error
constexpr int kRasterThreads = 256;
constexpr int kRasterWarps = kRasterThreads / 32;
constexpr long long kBigTri = 2048;     // candidates above which a triangle is chunked
constexpr long long kBigChunk = 1024;   // candidates per big-triangle work item

struct __align__(16) RasterTri {
    double ax, ay, az, e1x, e1y, e1z, e2x, e2y, e2z, px, py, pz, det, inv;
    long long i0, j0;
    long long excl;      // first flattened candidate index of this triangle
    int cols, id;
};

struct __align__(16) U128 {
    unsigned long long lo, hi;
};

// (t bits, id) lexicographic minimum into a PrimHit (layout: tbits | pad, id)
__device__ __forceinline__ void prim_min(PrimHit *h, unsigned long long bits, unsigned int id)
{
    U128 *p = reinterpret_cast<U128 *>(h);
    // pre-check with one plain 16-byte load; a stale (cached) value is safe:
    // entries only ever decrease, and the CAS re-validates
    U128 cur = *p;
    U128 nv;
    nv.lo = bits;
    nv.hi = 0xffffffffULL | ((unsigned long long)id << 32);
    while (bits < cur.lo || (bits == cur.lo && id < (unsigned int)(cur.hi >> 32))) {
        const U128 prev = atomicCAS(p, cur, nv);
        if (prev.lo == cur.lo && prev.hi == cur.hi) break;
        cur = prev;
    }
}

// Candidate rectangle of one (grid, triangle): the cells whose centre lies
// in the triangle's projected bounding box widened by kMargin.  count == 0:
// the triangle cannot be hit (det == 0, geometry.py:339) or lies outside.
struct RasterSetup {
    TriF64 T;
    TriDir P;
    double inv;
    long long i0, j0, count;
    int cols;
    double pa[3], pb[3];   // projected vertices in cell units (row a, column b)
};

__device__ __forceinline__ RasterSetup raster_setup(const TriF64 &T, const GridDev &G)
{
    RasterSetup S;
    S.T = T;
    S.count = 0;
    S.P = tri_dir(T, G.k[0], G.k[1], G.k[2]);
    if (S.P.det == 0.0) return S;
    const int64_t n_v = G.n_v, n_u = G.n_rays / n_v;
    const double isp = 1.0 / G.spacing;
    const double rx = T.ax - G.corner[0], ry = T.ay - G.corner[1], rz = T.az - G.corner[2];
    const double a0 = (rx * G.u[0] + ry * G.u[1] + rz * G.u[2]) * isp - 0.5;
    const double b0 = (rx * G.v[0] + ry * G.v[1] + rz * G.v[2]) * isp - 0.5;
    const double a1 = a0 + (T.e1x * G.u[0] + T.e1y * G.u[1] + T.e1z * G.u[2]) * isp;
    const double b1 = b0 + (T.e1x * G.v[0] + T.e1y * G.v[1] + T.e1z * G.v[2]) * isp;
    const double a2 = a0 + (T.e2x * G.u[0] + T.e2y * G.u[1] + T.e2z * G.u[2]) * isp;
    const double b2 = b0 + (T.e2x * G.v[0] + T.e2y * G.v[1] + T.e2z * G.v[2]) * isp;
    S.pa[0] = a0; S.pa[1] = a1; S.pa[2] = a2;
    S.pb[0] = b0; S.pb[1] = b1; S.pb[2] = b2;
    const double alo = fmin(fmin(a0, a1), a2) - kMargin;
    const double ahi = fmax(fmax(a0, a1), a2) + kMargin;
    const double blo = fmin(fmin(b0, b1), b2) - kMargin;
    const double bhi = fmax(fmax(b0, b1), b2) + kMargin;
    if (!(ahi >= 0.0 && bhi >= 0.0 && alo <= (double)(n_u - 1) && blo <= (double)(n_v - 1)))
        return S;                               // outside the aperture (or non-finite)
    const int64_t i0 = alo <= 0.0 ? 0 : (int64_t)ceil(alo);
    const int64_t i1 = ahi >= (double)(n_u - 1) ? n_u - 1 : (int64_t)floor(ahi);
    const int64_t j0 = blo <= 0.0 ? 0 : (int64_t)ceil(blo);
    const int64_t j1 = bhi >= (double)(n_v - 1) ? n_v - 1 : (int64_t)floor(bhi);
    const int64_t rows = i1 - i0 + 1, cols = j1 - j0 + 1;
    if (rows <= 0 || cols <= 0) return S;
    S.i0 = i0;
    S.j0 = j0;
    S.cols = (int)cols;
    S.count = rows * cols;
    S.inv = __drcp_rn(S.P.det);                 // == IEEE 1.0 / det
    return S;
}

// Sharded launches (a.sparse): shrink the candidate rectangle to the rows
// between the first and the last owned segment it touches (count 0: none
// owned).  Only cells raster_cell would skip anyway are dropped; k_raster and
// k_raster_big apply it identically, so chunk indices agree.
__device__ __forceinline__ void trim_owned(RasterSetup &S, const GridDev &G, const int64_t *segs)
{
    if (S.count == 0) return;
    const int64_t rows = S.count / S.cols;
    const int64_t r0 = S.i0 * G.n_v + S.j0;
    const int64_t r1 = (S.i0 + rows - 1) * G.n_v + S.j0 + S.cols - 1;
    int64_t qf = -1, ql = -1;
    for (int64_t q = r0 / kSegRays; q <= r1 / kSegRays; ++q)
        if (__ldg(&segs[q]) != kNoSlot) {
            if (qf < 0) qf = q;
            ql = q;
        }
    if (qf < 0) {
        S.count = 0;
        return;
    }
    const int64_t fa = (qf * kSegRays) / G.n_v, fb = ((ql + 1) * kSegRays - 1) / G.n_v;
    const int64_t a = fa > S.i0 ? fa : S.i0;
    const int64_t b = fb < S.i0 + rows - 1 ? fb : S.i0 + rows - 1;
    S.i0 = a;
    S.count = (b - a + 1) * S.cols;
}

__device__ __forceinline__ void split_cell(long long local, int cols, long long &li, long long &lj)
{
    if (local < 0x7fffffffLL) {
        const unsigned l32 = (unsigned)local, c32 = (unsigned)cols;
        li = l32 / c32;
        lj = l32 - (unsigned)li * c32;
    } else {
        li = local / cols;
        lj = local - li * cols;
    }
}

// Exact test of ray (i, j) against one triangle; records the hit.
__device__ __forceinline__ void raster_cell(const RasterArgs &a, const GridDev &G,
                                            const int64_t *seg, const TriF64 &T,
                                            const TriDir &P, double inv, int id, int64_t i,
                                            int64_t j)
{
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    const int64_t r = i * G.n_v + j;
    // sharded / partial batches: skip cells of segments this launch does not
    // own before doing any arithmetic
    const int64_t off = __ldg(&seg[r / kSegRays]);
    if (a.sparse && off == kNoSlot) return;
    // origin exactly as the launcher builds it (pipeline.cu grid_origin)
    const double sp = G.spacing;
    const double si = DM(DA((double)i, 0.5), sp);
    const double sj = DM(DA((double)j, 0.5), sp);
    const double ox = DA(DA(G.corner[0], DM(si, G.u[0])), DM(sj, G.v[0]));
    const double oy = DA(DA(G.corner[1], DM(si, G.u[1])), DM(sj, G.v[1]));
    const double oz = DA(DA(G.corner[2], DM(si, G.u[2])), DM(sj, G.v[2]));
    const double t = tri_hit_origin<true>(T, P, inv, ox, oy, oz, G.k[0], G.k[1], G.k[2], 0.0,
                                          inf);
    if (t > 0.0 && t < inf && off != kNoSlot)
        prim_min(a.prim + (off + r), (unsigned long long)__double_as_longlong(t),
                 (unsigned int)id);
}

// Column extent of the cells of row a within kMargin (L-inf) of the
// projected triangle: the b-range of the triangle clipped to the band
// |a' - a| <= kMargin (its extreme points are vertices inside the band or
// edge / band-boundary crossings), widened by kMargin.  The exact test can
// only accept cells within rounding (<< kMargin) of the triangle, so this
// span holds every cell the bounding box would have offered that can hit.
__device__ __forceinline__ void row_span(const RasterSetup &S, double a, double &blo, double &bhi)
{
    double lo = __longlong_as_double(0x7ff0000000000000LL), hi = -lo;
    const double c[2] = {a - kMargin, a + kMargin};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int k1 = k == 2 ? 0 : k + 1;
        if (S.pa[k] >= c[0] && S.pa[k] <= c[1]) { lo = fmin(lo, S.pb[k]); hi = fmax(hi, S.pb[k]); }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const double d0 = S.pa[k] - c[e], d1 = S.pa[k1] - c[e];
            if ((d0 < 0.0 && d1 > 0.0) || (d0 > 0.0 && d1 < 0.0)) {
                const double t = d0 / (d0 - d1);   // in (0, 1)
                const double b = S.pb[k] + t * (S.pb[k1] - S.pb[k]);
                lo = fmin(lo, b);
                hi = fmax(hi, b);
            }
        }
    }
    blo = lo - kMargin;
    bhi = hi + kMargin;
}

// Persistent: each warp pulls its next 32-triangle item from a global
// counter, so uneven candidate counts never leave warps idle.  A triangle
// with more than kBigTri candidates is not walked here: it is queued as
// kBigChunk-candidate chunks for k_raster_big, so no warp ever holds a huge
// triangle at the tail of the launch.
template <int STORAGE>
__global__ void __launch_bounds__(kRasterThreads, 4)
k_raster(RasterArgs a, int64_t ntri_pad)
{
    __shared__ RasterTri st[kRasterWarps][32];
    __shared__ int scan[kRasterWarps][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t warps_total = (int64_t)a.nbg * (ntri_pad / 32);
    while (true) {
        unsigned long long got = 0;
        if (lane == 0) got = atomicAdd(a.counter, 1ULL);
        const int64_t wg = (int64_t)__shfl_sync(0xffffffffu, got, 0);
        if (wg >= warps_total) break;
        const int64_t item = wg * 32 + lane;
        const int gl = (int)(item / ntri_pad);           // warp-uniform
        const int64_t tri = item - (int64_t)gl * ntri_pad;
        const int g = __ldg(&a.bgrids[gl]);
        const GridDev &G = a.grids[g];
        // ---- per-lane triangle set-up and candidate rectangle ----------
        long long count = 0;
        RasterTri &R = st[wib][lane];
        if (tri < a.ntri) {
            RasterSetup S = raster_setup(load_tri<STORAGE>(a.B, (int)tri), G);
            if (a.sparse) trim_owned(S, G, a.seg_slot + __ldg(&a.seg_base[g]));
            count = S.count;
            if (count > kBigTri && a.big) {
                const long long nch = (count + kBigChunk - 1) / kBigChunk;
                // sharded / partial batches: queue only chunks whose rows touch
                // a segment of this launch (ray-tile shards skip 7/8 of them)
                const int64_t *segs = a.seg_slot + __ldg(&a.seg_base[g]);
                auto owned = [&](long long c) {
                    if (!a.sparse) return true;
                    const long long c1 = (c + 1) * kBigChunk < count ? (c + 1) * kBigChunk : count;
                    const int64_t r0 = (S.i0 + c * kBigChunk / S.cols) * G.n_v + S.j0;
                    const int64_t r1 = (S.i0 + (c1 - 1) / S.cols) * G.n_v + S.j0 + S.cols - 1;
                    for (int64_t q = r0 / kSegRays; q <= r1 / kSegRays; ++q)
                        if (__ldg(&segs[q]) != kNoSlot) return true;
                    return false;
                };
                long long nown = 0;
                for (long long c = 0; c < nch; ++c) nown += owned(c);
                const unsigned long long at =
                    nown ? atomicAdd(a.nbig, (unsigned long long)nown) : 0ULL;
                if (at + nown <= (unsigned long long)a.big_cap) {
                    long long w = 0;
                    for (long long c = 0; c < nch; ++c)
                        if (owned(c)) a.big[at + w++] = make_int4(gl, (int)tri, (int)c, 0);
                    count = 0;                          // walked by k_raster_big
                }
            }
            if (count) {
                R.ax = S.T.ax; R.ay = S.T.ay; R.az = S.T.az;
                R.e1x = S.T.e1x; R.e1y = S.T.e1y; R.e1z = S.T.e1z;
                R.e2x = S.T.e2x; R.e2y = S.T.e2y; R.e2z = S.T.e2z;
                R.px = S.P.px; R.py = S.P.py; R.pz = S.P.pz; R.det = S.P.det;
                R.inv = S.inv;
                R.i0 = S.i0; R.j0 = S.j0; R.cols = S.cols; R.id = S.T.id;
            }
        }
        // ---- warp scan of candidate counts --------------------------------
        long long incl = count;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const long long total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0) continue;
        if (count) R.excl = incl - count;
        const int64_t *seg = a.seg_slot + __ldg(&a.seg_base[g]);
        // walk the flattened list in windows of 2^30 so the prefix search
        // runs on 32-bit values (one window unless a triangle is enormous)
        constexpr long long kWin = 1LL << 30;
        for (long long win = 0; win < total; win += kWin) {
            long long v = incl - win;
            v = v < 0 ? 0 : (v > kWin ? kWin : v);
            __syncwarp();
            scan[wib][lane] = (int)v;
            __syncwarp();
            const int wtotal = (int)((total - win) < kWin ? (total - win) : kWin);
            for (int base = 0; base < wtotal; base += 32) {
                const int c = base + lane;
                if (c >= wtotal) continue;
                // owner = first lane whose clipped inclusive prefix exceeds c
                int lo = 0;
#pragma unroll
                for (int step = 16; step > 0; step >>= 1)
                    if (scan[wib][lo + step - 1] <= c) lo += step;
                const RasterTri &Q = st[wib][lo];
                long long li, lj;
                split_cell((long long)c + win - Q.excl, Q.cols, li, lj);
                TriF64 T;
                T.ax = Q.ax; T.ay = Q.ay; T.az = Q.az;
                T.e1x = Q.e1x; T.e1y = Q.e1y; T.e1z = Q.e1z;
                T.e2x = Q.e2x; T.e2y = Q.e2y; T.e2z = Q.e2z;
                TriDir P;
                P.px = Q.px; P.py = Q.py; P.pz = Q.pz; P.det = Q.det;
                raster_cell(a, G, seg, T, P, Q.inv, Q.id, Q.i0 + li, Q.j0 + lj);
            }
        }
        __syncwarp();
    }
}

// Chunks of big triangles: a warp takes one chunk (kBigChunk candidates of
// one triangle), recomputes the (identical) set-up and walks 32 cells at a
// time.
template <int STORAGE>
__global__ void __launch_bounds__(kRasterThreads, 4)
k_raster_big(RasterArgs a)
{
    const int lane = threadIdx.x & 31;
    const unsigned long long nbig = *a.nbig;
    const unsigned long long n = nbig < (unsigned long long)a.big_cap ? nbig : a.big_cap;
    while (true) {
        unsigned long long got = 0;
        if (lane == 0) got = atomicAdd(a.counter, 1ULL);
        const unsigned long long w = __shfl_sync(0xffffffffu, got, 0);
        if (w >= n) break;
        const int4 it = a.big[w];
        const int g = __ldg(&a.bgrids[it.x]);
        const GridDev &G = a.grids[g];
        RasterSetup S = raster_setup(load_tri<STORAGE>(a.B, it.y), G);
        const int64_t *seg = a.seg_slot + __ldg(&a.seg_base[g]);
        if (a.sparse) trim_owned(S, G, seg);
        const long long c0 = (long long)it.z * kBigChunk;
        const long long c1 = c0 + kBigChunk < S.count ? c0 + kBigChunk : S.count;
        if (c0 >= c1) continue;
        // the chunk's rows, 32 at a time: lane r takes row r's cells that
        // lie within kMargin of the triangle (not the whole box row), then
        // the warp walks the concatenated spans 32 cells at a time
        const long long row_a = c0 / S.cols, row_b = (c1 - 1) / S.cols;
        for (long long rbase = row_a; rbase <= row_b; rbase += 32) {
            const long long li = rbase + lane;
            long long jl = 0, jr = -1;
            if (li <= row_b) {
                const long long wl = li == row_a ? c0 % S.cols : 0;
                const long long wr = li == row_b ? (c1 - 1) % S.cols : S.cols - 1;
                double blo, bhi;
                row_span(S, (double)(S.i0 + li), blo, bhi);
                const long long sl = blo > (double)(S.j0 + wl) ? (long long)ceil(blo) - S.j0 : wl;
                const long long sr = bhi < (double)(S.j0 + wr) ? (long long)floor(bhi) - S.j0 : wr;
                jl = sl;
                jr = sr;
            }
            const int cnt = jr >= jl ? (int)(jr - jl + 1) : 0;
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            const int excl = incl - cnt;
            const int jl32 = (int)jl;
            for (int base = 0; base < total; base += 32) {
                const int c = base + lane;
                int owner = 0;   // first lane whose inclusive count exceeds c
#pragma unroll
                for (int st = 16; st >= 1; st >>= 1)
                    if (__shfl_sync(0xffffffffu, incl, owner + st - 1) <= c) owner += st;
                const int oex = __shfl_sync(0xffffffffu, excl, owner);
                const int ojl = __shfl_sync(0xffffffffu, jl32, owner);
                if (c < total)
                    raster_cell(a, G, seg, S.T, S.P, S.inv, S.T.id, S.i0 + rbase + owner,
                                S.j0 + ojl + (c - oex));
            }
        }
    }
}

template <int S>
static int persistent_raster_blocks(int num_sms, bool big)
{
    int per_sm = 0;
    const cudaError_t e =
        big ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_raster_big<S>,
                                                            kRasterThreads, 0)
            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_raster<S>,
                                                            kRasterThreads, 0);
    return (e != cudaSuccess || per_sm < 1 ? 1 : per_sm) * num_sms;
}

template <int S>
static void raster_dispatch(const RasterArgs &a, cudaStream_t st, int num_sms)
{
    const int64_t ntri_pad = (a.ntri + 31) / 32 * 32;
    const int64_t warps = (int64_t)a.nbg * (ntri_pad / 32);
    int64_t blocks = (warps + kRasterWarps - 1) / kRasterWarps;
    const int64_t cap = persistent_raster_blocks<S>(num_sms, false);
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    k_raster<S><<<(unsigned)blocks, kRasterThreads, 0, st>>>(a, ntri_pad);
    if (a.big) {
        cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), st);
        k_raster_big<S><<<persistent_raster_blocks<S>(num_sms, true), kRasterThreads, 0, st>>>(a);
    }
}

cudaError_t launch_raster(const RasterArgs &a, cudaStream_t st, const LaunchStats &ls)
{
    if (a.nbg == 0 || a.ntri == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), st);
    if (e == cudaSuccess && a.big)
        e = cudaMemsetAsync(a.nbig, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    if (a.storage == kF64) raster_dispatch<kF64>(a, st, ls.num_sms);
    else if (a.storage == kSingle) raster_dispatch<kSingle>(a, st, ls.num_sms);
    else raster_dispatch<kF32Exact>(a, st, ls.num_sms);
    *ls.launches += a.big ? 2 : 1;
    return cudaGetLastError();
}

}  // namespace sbr
