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

// Persistent: each warp pulls its next 32-triangle item from a global
// counter, so uneven candidate counts never leave warps idle.
template <int STORAGE>
__global__ void __launch_bounds__(kRasterThreads, 4)
k_raster(RasterArgs a, int64_t ntri_pad)
{
    __shared__ RasterTri st[kRasterWarps][32];
    __shared__ int scan[kRasterWarps][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
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
        const double dx = G.k[0], dy = G.k[1], dz = G.k[2];
        const double sp = G.spacing;
        const int64_t n_v = G.n_v, n_u = G.n_rays / n_v;
        // ---- per-lane triangle set-up and candidate rectangle ----------
        long long count = 0;
        RasterTri &R = st[wib][lane];
        if (tri < a.ntri) {
            const TriF64 T = load_tri<STORAGE>(a.B, (int)tri);
            const TriDir P = tri_dir(T, dx, dy, dz);
            if (P.det != 0.0) {                    // geometry.py:339: never accepted
                const double isp = 1.0 / sp;
                const double rx = T.ax - G.corner[0], ry = T.ay - G.corner[1],
                             rz = T.az - G.corner[2];
                const double a0 = (rx * G.u[0] + ry * G.u[1] + rz * G.u[2]) * isp - 0.5;
                const double b0 = (rx * G.v[0] + ry * G.v[1] + rz * G.v[2]) * isp - 0.5;
                const double a1 = a0 + (T.e1x * G.u[0] + T.e1y * G.u[1] + T.e1z * G.u[2]) * isp;
                const double b1 = b0 + (T.e1x * G.v[0] + T.e1y * G.v[1] + T.e1z * G.v[2]) * isp;
                const double a2 = a0 + (T.e2x * G.u[0] + T.e2y * G.u[1] + T.e2z * G.u[2]) * isp;
                const double b2 = b0 + (T.e2x * G.v[0] + T.e2y * G.v[1] + T.e2z * G.v[2]) * isp;
                const double alo = fmin(fmin(a0, a1), a2) - kMargin;
                const double ahi = fmax(fmax(a0, a1), a2) + kMargin;
                const double blo = fmin(fmin(b0, b1), b2) - kMargin;
                const double bhi = fmax(fmax(b0, b1), b2) + kMargin;
                if (ahi >= 0.0 && bhi >= 0.0 && alo <= (double)(n_u - 1) &&
                    blo <= (double)(n_v - 1)) {
                    const int64_t i0 = alo <= 0.0 ? 0 : (int64_t)ceil(alo);
                    const int64_t i1 = ahi >= (double)(n_u - 1) ? n_u - 1 : (int64_t)floor(ahi);
                    const int64_t j0 = blo <= 0.0 ? 0 : (int64_t)ceil(blo);
                    const int64_t j1 = bhi >= (double)(n_v - 1) ? n_v - 1 : (int64_t)floor(bhi);
                    const int64_t rows = i1 - i0 + 1, cols = j1 - j0 + 1;
                    if (rows > 0 && cols > 0) {
                        count = rows * cols;
                        R.ax = T.ax; R.ay = T.ay; R.az = T.az;
                        R.e1x = T.e1x; R.e1y = T.e1y; R.e1z = T.e1z;
                        R.e2x = T.e2x; R.e2y = T.e2y; R.e2z = T.e2z;
                        R.px = P.px; R.py = P.py; R.pz = P.pz; R.det = P.det;
                        R.inv = __drcp_rn(P.det);    // == IEEE 1.0 / det
                        R.i0 = i0; R.j0 = j0; R.cols = (int)cols; R.id = T.id;
                    }
                }
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
                const long long local = (long long)c + win - Q.excl;
                long long li, lj;
                if (local < 0x7fffffffLL) {
                    const unsigned l32 = (unsigned)local, c32 = (unsigned)Q.cols;
                    li = l32 / c32;
                    lj = l32 - (unsigned)li * c32;
                } else {
                    li = local / Q.cols;
                    lj = local - li * Q.cols;
                }
                const int64_t i = Q.i0 + li, j = Q.j0 + lj;
                // origin exactly as the launcher builds it (pipeline.cu grid_origin)
                const double si = DM(DA((double)i, 0.5), sp);
                const double sj = DM(DA((double)j, 0.5), sp);
                const double ox = DA(DA(G.corner[0], DM(si, G.u[0])), DM(sj, G.v[0]));
                const double oy = DA(DA(G.corner[1], DM(si, G.u[1])), DM(sj, G.v[1]));
                const double oz = DA(DA(G.corner[2], DM(si, G.u[2])), DM(sj, G.v[2]));
                TriF64 T;
                T.ax = Q.ax; T.ay = Q.ay; T.az = Q.az;
                T.e1x = Q.e1x; T.e1y = Q.e1y; T.e1z = Q.e1z;
                T.e2x = Q.e2x; T.e2y = Q.e2y; T.e2z = Q.e2z;
                TriDir P;
                P.px = Q.px; P.py = Q.py; P.pz = Q.pz; P.det = Q.det;
                const double t = tri_hit_origin<true>(T, P, Q.inv, ox, oy, oz, dx, dy, dz,
                                                      0.0, inf);
                if (t > 0.0 && t < inf) {
                    const int64_t r = i * n_v + j;
                    const int64_t off = __ldg(&seg[r / kSegRays]);
                    if (off != kNoSlot)
                        prim_min(a.prim + (off + r), (unsigned long long)__double_as_longlong(t),
                                 (unsigned int)Q.id);
                }
            }
        }
        __syncwarp();
    }
}

template <int S>
static void raster_dispatch(const RasterArgs &a, cudaStream_t st, int num_sms)
{
    const int64_t ntri_pad = (a.ntri + 31) / 32 * 32;
    const int64_t warps = (int64_t)a.nbg * (ntri_pad / 32);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_raster<S>, kRasterThreads, 0) !=
            cudaSuccess || per_sm < 1)
        per_sm = 1;
    int64_t blocks = (warps + kRasterWarps - 1) / kRasterWarps;
    if (blocks > (int64_t)per_sm * num_sms) blocks = (int64_t)per_sm * num_sms;
    if (blocks < 1) blocks = 1;
    k_raster<S><<<(unsigned)blocks, kRasterThreads, 0, st>>>(a, ntri_pad);
}

cudaError_t launch_raster(const RasterArgs &a, cudaStream_t st, const LaunchStats &ls)
{
    if (a.nbg == 0 || a.ntri == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(a.counter, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    if (a.storage == kF64) raster_dispatch<kF64>(a, st, ls.num_sms);
    else if (a.storage == kSingle) raster_dispatch<kSingle>(a, st, ls.num_sms);
    else raster_dispatch<kF32Exact>(a, st, ls.num_sms);
    *ls.launches += 1;
    return cudaGetLastError();
}

}  // namespace sbr
