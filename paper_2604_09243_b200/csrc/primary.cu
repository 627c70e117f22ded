// primary.cu -- primary visibility by rasterising triangles into the launch
// grid (query 0 of every ray, transport.py:293-296 with t_min = 0, t_max = inf).
//
// All primary rays of one aperture share the direction k and start on a
// regular grid: origin(i, j) = corner + ((i+.5) ds) u + ((j+.5) ds) v
// (transport.py:339-345).  So instead of one BVH traversal per ray, every
// (grid, triangle) pair enumerates a candidate set of cells PROVEN to
// contain every cell its Moller-Trumbore test can accept (see "Candidate
// region" below; it covers near-edge-on triangles whose rounding-dominated
// det accepts rays far outside the triangle) and evaluates the SAME exact
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

// Candidate region (why the raster pass is exactly the linear scan).
// Möller-Trumbore accepts a ray o only if its rounded numerators pass
//   sigma*un in [0, D(1+3e)],  sigma*vn >= 0,  sigma*(un+vn) <= D(1+4e)
// (sigma = sign det, D = |det|, e = 2^-53; an underflowed product is covered
// by an absolute 1e-290).  un and vn differ from the exact affine functions
//   F(o) = sigma (o - a).p          (p = d x e2 as computed, geometry.py:336)
//   G(o) = sigma (o - a).(e1 x d)   (= sigma d.((o - a) x e1), geometry.py:347)
// by at most a few ulp of the magnitude sums Mp = sum_k |p_k| R_k and
// Mr = sum_k (|e1 x d| terms)_k R_k, where R_k bounds |o_k|, |a_k| and
// |o_k - a_k| over the aperture; the same bound also absorbs the rounding of
// the origin (pipeline.cu grid_origin) and of the cell-space coefficients
// below.  With Eu = 64e Mp and Ev = 64e Mr (about 3x the worst first-order
// sum) every accepted cell (i, j) satisfies, for the cell-space affine forms
//   F(i, j) = f0 + fi i + fj j,  G(i, j) = g0 + gi i + gj j,
//   F >= -Eu,   G >= -Ev,   F + G <= H = D(1 + 16e) + Eu + Ev.
// That triangle of cells is a superset of the accepting set for EVERY
// triangle, including near-edge-on ones whose rounding-dominated det lets
// Möller-Trumbore accept rays far outside the triangle: there the region is
// a long thin strip (the two edge forms are almost parallel), clipped by
// the aperture.  Cells outside it cannot be accepted, so query 0 from this
// pass is the reference's documented semantics, the lexicographic (t, id)
// minimum over EVERY accepting triangle -- "identical to a linear scan"
// (bvh.py:394-395) -- with no tree and no padding involved.
//   Well-conditioned pairs (the region's three vertices are stable under
// rounding): candidates = the vertices' bounding box (widened by their error
// bound), walked as a rectangle, or as per-row spans of the three
// half-planes for big triangles.  Otherwise (WIDE): the bounding box of the
// two edge strips clipped to the aperture, walked as spans along the
// box's shorter side (one column through a grid-aligned edge-on panel, not
// every row), always through the chunk queue.
constexpr double kEps = 1.1102230246251565e-16;   // 2^-53
constexpr double kTiny = 1e-290;
#ifndef SBR_RASTER_MINB
#define SBR_RASTER_MINB 4
#endif
#ifndef SBR_RASTER_CLAIM
#define SBR_RASTER_CLAIM 4
#endif
constexpr int kRasterClaim = SBR_RASTER_CLAIM;   // warp items per work-counter atomic
#ifndef SBR_BIG_CLAIM
#define SBR_BIG_CLAIM 2
#endif
constexpr int kBigClaim = SBR_BIG_CLAIM;         // big-triangle chunks per atomic
constexpr int kRasterThreads = 256;
constexpr int kRasterWarps = kRasterThreads / 32;
#ifndef SBR_BIG_TRI
#define SBR_BIG_TRI 512   // C5 8-rank shard raster 6.4 -> 4.9 ms, C5 32.6 -> 29.6 ms
#endif
constexpr long long kBigTri = SBR_BIG_TRI;   // candidates above which a triangle is chunked
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

// (t bits, id) lexicographic minimum into a PrimHit (layout: tbits | pad, id).
// The thread whose CAS replaces the all-ones "no hit" marks the slot in the
// hit bitmap (one fire-and-forget OR per hit ray), so the compaction reads
// only the slots that were hit.
__device__ __forceinline__ void prim_min(PrimHit *h, unsigned long long bits, unsigned int id,
                                         unsigned int *hitmap, int64_t slot)
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
        if (prev.lo == cur.lo && prev.hi == cur.hi) {
            if (hitmap && cur.lo == kNoHitBits)
                atomicOr(hitmap + (slot >> 5), 1u << (unsigned)(slot & 31));
            break;
        }
        cur = prev;
    }
}

// Candidates of one (grid, triangle).  The bounding box [i0, i0+rows) x
// [j0, j0+cols) is walked line by line: lines are rows (trans = 0) or
// columns (trans = 1), each clipped to the half-plane span.  count == 0: the
// triangle cannot be hit (det == 0, geometry.py:339) or lies outside.
struct RasterSetup {
    TriF64 T;
    TriDir P;
    double inv;
    long long i0, j0, rows, count;
    int cols;
    int trans, wide;
    int span;        // chunk by lines (32 per chunk), walking each line's span
    double f0, fi, fj, g0, gi, gj, eu, ev, h, err;
};
static_assert(sizeof(RasterSetup) <= kRasterSetupBytes, "set-up table slot");

// Candidate box of an ill-conditioned (WIDE) pair: the boxes of the two edge
// strips -Eu <= F <= H + Ev and -Ev <= G <= H + Eu, clipped to the aperture.
// Rare (204 of C4's 354M pairs), so kept out of line: its registers do not
// weigh on the common path.  Returns false when the region is empty.
__device__ __forceinline__ bool wide_region(const RasterSetup &S, int64_t n_u, int64_t n_v,
                                         double &alo_o, double &ahi_o, double &blo_o,
                                         double &bhi_o)
{
    double alo, ahi, blo, bhi;
    alo = 0.0; ahi = (double)(n_u - 1);
    blo = 0.0; bhi = (double)(n_v - 1);
    const double xs[3] = {S.f0, S.fi, S.fj}, ys[3] = {S.g0, S.gi, S.gj};
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const double *c = s ? ys : xs;
        const double lo = s ? -S.ev : -S.eu, hi = s ? S.h + S.eu : S.h + S.ev;
        // column range over the aperture's rows (extremes at the end rows)
        if (c[2] != 0.0) {
            double mn = INFINITY, mx = -INFINITY;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const double x = e ? (double)(n_u - 1) : 0.0;
                const double q0 = (lo - c[0] - c[1] * x) / c[2];
                const double q1 = (hi - c[0] - c[1] * x) / c[2];
                const double w = (S.err + 8.0 * kEps * (fabs(lo) + fabs(hi) + fabs(c[0]) +
                                                        fabs(c[1] * x))) / fabs(c[2]);
                mn = fmin(mn, fmin(q0, q1) - w);
                mx = fmax(mx, fmax(q0, q1) + w);
            }
            blo = fmax(blo, mn - 1e-9 * (1.0 + fabs(mn)));
            bhi = fmin(bhi, mx + 1e-9 * (1.0 + fabs(mx)));
        }
        // row range over the aperture's columns
        if (c[1] != 0.0) {
            double mn = INFINITY, mx = -INFINITY;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const double y = e ? (double)(n_v - 1) : 0.0;
                const double q0 = (lo - c[0] - c[2] * y) / c[1];
                const double q1 = (hi - c[0] - c[2] * y) / c[1];
                const double w = (S.err + 8.0 * kEps * (fabs(lo) + fabs(hi) + fabs(c[0]) +
                                                        fabs(c[2] * y))) / fabs(c[1]);
                mn = fmin(mn, fmin(q0, q1) - w);
                mx = fmax(mx, fmax(q0, q1) + w);
            }
            alo = fmax(alo, mn - 1e-9 * (1.0 + fabs(mn)));
            ahi = fmin(ahi, mx + 1e-9 * (1.0 + fabs(mx)));
        }
    }
    if (!(alo <= ahi && blo <= bhi)) return false;   // NaN-safe: empty
    alo_o = alo; ahi_o = ahi; blo_o = blo; bhi_o = bhi;
    return true;
}

__device__ __forceinline__ RasterSetup raster_setup(const TriF64 &T, const GridDev &G,
                                                    int64_t row_lo, int64_t row_hi)
{
    RasterSetup S;
    S.T = T;
    S.count = 0;
    S.P = tri_dir(T, G.k[0], G.k[1], G.k[2]);
    if (S.P.det == 0.0) return S;
    const int64_t n_v = G.n_v, n_u = G.n_u;
    const double dx = G.k[0], dy = G.k[1], dz = G.k[2];
    const double sg = S.P.det > 0.0 ? 1.0 : -1.0;
    const double D = fabs(S.P.det);
    // r = e1 x d, so that G(o) = (o - a) . r
    const double rx = T.e1y * dz - T.e1z * dy;
    const double ry = T.e1z * dx - T.e1x * dz;
    const double rz = T.e1x * dy - T.e1y * dx;
    const double Rx = G.rbound[0] + fabs(T.ax);
    const double Ry = G.rbound[1] + fabs(T.ay);
    const double Rz = G.rbound[2] + fabs(T.az);
    const double Mp = fabs(S.P.px) * Rx + fabs(S.P.py) * Ry + fabs(S.P.pz) * Rz;
    const double Mr = (fabs(T.e1y * dz) + fabs(T.e1z * dy)) * Rx +
                      (fabs(T.e1z * dx) + fabs(T.e1x * dz)) * Ry +
                      (fabs(T.e1x * dy) + fabs(T.e1y * dx)) * Rz;
    S.eu = 64.0 * kEps * Mp + kTiny;
    S.ev = 64.0 * kEps * Mr + kTiny;
    S.h = D * (1.0 + 16.0 * kEps) + S.eu + S.ev;
    // evaluation slack of any form at any cell of the aperture
    S.err = 16.0 * kEps * (Mp + Mr + D) + kTiny;
    // cell-space forms: o*(i, j) = corner + (i+.5) ds u + (j+.5) ds v
    const double cx = G.corner[0] - T.ax, cy = G.corner[1] - T.ay, cz = G.corner[2] - T.az;
    const double sp = G.spacing;
    S.fi = sg * sp * (G.u[0] * S.P.px + G.u[1] * S.P.py + G.u[2] * S.P.pz);
    S.fj = sg * sp * (G.v[0] * S.P.px + G.v[1] * S.P.py + G.v[2] * S.P.pz);
    S.f0 = sg * (cx * S.P.px + cy * S.P.py + cz * S.P.pz) + 0.5 * (S.fi + S.fj);
    S.gi = sg * sp * (G.u[0] * rx + G.u[1] * ry + G.u[2] * rz);
    S.gj = sg * sp * (G.v[0] * rx + G.v[1] * ry + G.v[2] * rz);
    S.g0 = sg * (cx * rx + cy * ry + cz * rz) + 0.5 * (S.gi + S.gj);
    if (!(isfinite(S.f0) && isfinite(S.g0) && isfinite(S.h) && isfinite(S.fi) &&
          isfinite(S.fj) && isfinite(S.gi) && isfinite(S.gj)))
        return S;   // non-finite geometry: the exact test accepts nothing finite
    double alo, ahi, blo, bhi;
    double area = INFINITY;   // of the candidate region, in cells
    // ---- well-conditioned: the region's vertices by Cramer's rule --------
    // vertex 0 solves M x = (-Eu - f0, -Ev - g0) with M = [fi fj; gi gj];
    // vertices 1 and 2 add M^-1 (0, L) and M^-1 (L, 0), L = H + Eu + Ev (the
    // region's legs in (F, G)).  One bound per axis covers all three: the
    // first-order error of the 2x2 solve (relative error of det2 <= 2e kd /
    // |det2|, numerators a few ulp of their magnitude sums), the rounded
    // reciprocal and the vertex additions -- each x4 or more
    const double det2 = S.fi * S.gj - S.fj * S.gi;
    const double kd = fabs(S.fi * S.gj) + fabs(S.fj * S.gi);
    S.wide = 1;
    if (fabs(det2) > 1e-6 * kd) {
        const double L = S.h + S.eu + S.ev;
        const double inv2 = 1.0 / det2, ainv2 = fabs(inv2);
        const double nf = -S.eu - S.f0, ng = -S.ev - S.g0;
        const double a0 = (nf * S.gj - S.fj * ng) * inv2;
        const double b0 = (S.fi * ng - S.gi * nf) * inv2;
        const double La = L * inv2;
        const double a1 = a0 - S.fj * La, b1 = b0 + S.fi * La;
        const double a2 = a0 + S.gj * La, b2 = b0 - S.gi * La;
        const double amax = fmax(fmax(fabs(a0), fabs(a1)), fabs(a2));
        const double bmax = fmax(fmax(fabs(b0), fabs(b1)), fabs(b2));
        const double mf = fabs(S.f0) + S.eu + L, mg = fabs(S.g0) + S.ev + L;
        const double ea = 16.0 * kEps * ((amax * kd + mf * fabs(S.gj) + fabs(S.fj) * mg) *
                                             ainv2 * (1.0 + 16.0 * kEps) + 2.0 * amax);
        const double eb = 16.0 * kEps * ((bmax * kd + mg * fabs(S.fi) + fabs(S.gi) * mf) *
                                             ainv2 * (1.0 + 16.0 * kEps) + 2.0 * bmax);
        if (fmax(ea, eb) <= 0.25 && amax < 1e300 && bmax < 1e300) {   // NaN fails too
            S.wide = 0;
            // the region is the (F, G) triangle with legs L, mapped to cells
            // through a Jacobian of det2
            area = 0.5 * L * L * ainv2;
            const double wa = ea + 1e-9 * (1.0 + amax), wb = eb + 1e-9 * (1.0 + bmax);
            alo = fmin(fmin(a0, a1), a2) - wa;
            ahi = fmax(fmax(a0, a1), a2) + wa;
            blo = fmin(fmin(b0, b1), b2) - wb;
            bhi = fmax(fmax(b0, b1), b2) + wb;
        }
    }
    if (S.wide && !wide_region(S, n_u, n_v, alo, ahi, blo, bhi)) return S;
    if (!(ahi >= 0.0 && bhi >= 0.0 && alo <= (double)(n_u - 1) && blo <= (double)(n_v - 1)))
        return S;                               // outside the aperture (or non-finite)
    int64_t i0 = alo <= 0.0 ? 0 : __double2ll_ru(alo);
    int64_t i1 = ahi >= (double)(n_u - 1) ? n_u - 1 : __double2ll_rd(ahi);
    if (i0 < row_lo) i0 = row_lo;               // row window of a partial trace
    if (i1 > row_hi - 1) i1 = row_hi - 1;
    const int64_t j0 = blo <= 0.0 ? 0 : __double2ll_ru(blo);
    const int64_t j1 = bhi >= (double)(n_v - 1) ? n_v - 1 : __double2ll_rd(bhi);
    const int64_t rows = i1 - i0 + 1, cols = j1 - j0 + 1;
    if (rows <= 0 || cols <= 0) return S;
    S.i0 = i0;
    S.j0 = j0;
    S.rows = rows;
    S.cols = (int)cols;
    // Span mode: a region much smaller than its bounding box (the long thin
    // sliver of a nearly edge-on triangle, or a WIDE strip) is chunked by
    // lines and walked span by span -- bounding-box chunks would enumerate
    // (and queue) the whole box, up to hundreds of millions of cells
    S.span = S.wide ||
             (double)rows * (double)cols > 4.0 * (area + (double)rows + (double)cols + 256.0);
    S.trans = S.span && cols < rows;
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
    const int64_t rows = S.rows;
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
    S.rows = b - a + 1;
    S.trans = S.trans && S.cols < S.rows;
    S.count = S.rows * S.cols;
}

// chunks of a queued pair: span mode = 32 lines each, else kBigChunk cells
// of the bounding box in line-major order
__device__ __forceinline__ long long span_lines(const RasterSetup &S)
{
    return S.trans ? (long long)S.cols : S.rows;
}
__device__ __forceinline__ long long big_chunks(const RasterSetup &S)
{
    return S.span ? (span_lines(S) + 31) / 32 : (S.count + kBigChunk - 1) / kBigChunk;
}
// Ray-tile shards (sparse launches): a well-conditioned pair's chunks are
// its pieces in the 2^19-ray segments it touches (chunk c = segment qa + c),
// so a rank queues and walks exactly the pieces of the segments it owns
__device__ __forceinline__ bool seg_chunks(const RasterArgs &a, const RasterSetup &S)
{
    return a.sparse && !S.trans && !S.span;
}
__device__ __forceinline__ void seg_range(const RasterSetup &S, int64_t n_v, int64_t &qa,
                                          int64_t &qb)
{
    qa = (S.i0 * n_v + S.j0) / kSegRays;
    qb = ((S.i0 + S.rows - 1) * n_v + S.j0 + S.cols - 1) / kSegRays;
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
                 (unsigned int)id, a.hitmap, off + r);
}

// Span of line x (a row i, or a column j when S.trans) inside the candidate
// region: the three half-planes F + Eu >= 0, G + Ev >= 0, H - F - G >= 0
// solved for the other index, each widened by its evaluation slack.
__device__ __forceinline__ void line_span(const RasterSetup &S, double x, double &lo, double &hi)
{
    const double fa = S.trans ? S.fj : S.fi, fb = S.trans ? S.fi : S.fj;
    const double ga = S.trans ? S.gj : S.gi, gb = S.trans ? S.gi : S.gj;
    const double k0[3] = {S.f0 + S.eu, S.g0 + S.ev, S.h - S.f0 - S.g0};
    const double kx[3] = {fa, ga, -(fa + ga)};
    const double ky[3] = {fb, gb, -(fb + gb)};
    lo = -INFINITY;
    hi = INFINITY;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        // need k0 + kx x + ky y >= 0
        const double num = k0[c] + kx[c] * x;
        const double w = S.err + 8.0 * kEps * (fabs(k0[c]) + fabs(kx[c] * x) + S.h);
        if (ky[c] > 0.0) {
            const double y = (-num - w) / ky[c];
            lo = fmax(lo, y - 1e-9 * (1.0 + fabs(y)));
        } else if (ky[c] < 0.0) {
            const double y = (-num - w) / ky[c];
            hi = fmin(hi, y + 1e-9 * (1.0 + fabs(y)));
        } else if (num + w < 0.0) {
            lo = INFINITY;   // the whole line fails this half-plane
        }
    }
}

// Persistent: each warp pulls its next 32-triangle item from a global
// counter, so uneven candidate counts never leave warps idle.  A triangle
// with more than kBigTri candidates is not walked here: it is queued as
// kBigChunk-candidate chunks for k_raster_big, so no warp ever holds a huge
// triangle at the tail of the launch.
template <int STORAGE>
__global__ void __launch_bounds__(kRasterThreads, SBR_RASTER_MINB)
k_raster(RasterArgs a, int64_t ntri_pad, int claim)
{
    __shared__ RasterTri st[kRasterWarps][32];
    __shared__ int scan[kRasterWarps][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t warps_total = (int64_t)a.nbg * (ntri_pad / 32);
    // a warp claims `claim` consecutive items per atomic: one counter shared
    // by every warp of the GPU serialises its atomics at L2 (C4 raster 43 ->
    // 37 ms with 4); 1 when there are few items per warp (load balance)
    int64_t wg = 0, wg_end = 0;
    while (true) {
        if (wg >= wg_end) {
            unsigned long long got = 0;
            if (lane == 0) got = atomicAdd(a.counter, (unsigned long long)claim);
            wg = (int64_t)__shfl_sync(0xffffffffu, got, 0);
            wg_end = wg + claim;
        }
        if (wg >= warps_total) break;
        const int64_t item = wg * 32 + lane;
        ++wg;
        const int gl = (int)(item / ntri_pad);           // warp-uniform
        const int64_t tri = item - (int64_t)gl * ntri_pad;
        const int g = __ldg(&a.bgrids[gl]);
        const GridDev &G = a.grids[g];
        // ---- per-lane triangle set-up and candidate rectangle ----------
        long long count = 0;
        RasterTri &R = st[wib][lane];
        if (tri < a.ntri) {
            RasterSetup S = raster_setup(load_tri<STORAGE>(a.B, (int)tri), G, a.row_lo, a.row_hi);
            if (a.sparse) trim_owned(S, G, a.seg_slot + __ldg(&a.seg_base[g]));
            count = S.count;
            if (S.wide && count && a.stats) atomicAdd(a.stats + 1, 1ULL);
            if (count > kBigTri && a.big) {
                const bool segm = seg_chunks(a, S);
                int64_t qa = 0, qb = 0;
                if (segm) seg_range(S, G.n_v, qa, qb);
                const long long nch = segm ? qb - qa + 1 : big_chunks(S);
                // sharded / partial batches: queue only chunks whose rows touch
                // a segment of this launch (ray-tile shards skip 7/8 of them);
                // column-major (trans) chunks span every row: always queued
                const int64_t *segs = a.seg_slot + __ldg(&a.seg_base[g]);
                auto owned = [&](long long c) {
                    if (segm) return __ldg(&segs[qa + c]) != kNoSlot;
                    if (!a.sparse || S.trans) return true;
                    int64_t r0, r1;
                    if (S.span) {
                        const long long la = 32 * c;
                        const long long lb = la + 31 < S.rows - 1 ? la + 31 : S.rows - 1;
                        r0 = (S.i0 + la) * G.n_v + S.j0;
                        r1 = (S.i0 + lb) * G.n_v + S.j0 + S.cols - 1;
                    } else {
                        const long long c1 =
                            (c + 1) * kBigChunk < count ? (c + 1) * kBigChunk : count;
                        r0 = (S.i0 + c * kBigChunk / S.cols) * G.n_v + S.j0;
                        r1 = (S.i0 + (c1 - 1) / S.cols) * G.n_v + S.j0 + S.cols - 1;
                    }
                    for (int64_t q = r0 / kSegRays; q <= r1 / kSegRays; ++q)
                        if (__ldg(&segs[q]) != kNoSlot) return true;
                    return false;
                };
                long long nown = 0;
                for (long long c = 0; c < nch; ++c) nown += owned(c);
                const unsigned long long at =
                    nown ? atomicAdd(a.nbig, (unsigned long long)nown) : 0ULL;
                const unsigned long long cap = (unsigned long long)a.big_cap;
                if (at + nown <= cap) {
                    // publish the set-up once for all of the triangle's chunks
                    int si = -1;
                    if (nown > 1 && a.setups) {
                        const unsigned long long k = atomicAdd(a.nsetup, 1ULL);
                        if (k < (unsigned long long)a.setup_cap) {
                            si = (int)k;
                            *reinterpret_cast<RasterSetup *>(a.setups +
                                                             (size_t)k * kRasterSetupBytes) = S;
                        }
                    }
                    long long w = 0;
                    for (long long c = 0; c < nch; ++c)
                        if (owned(c)) a.big[at + w++] = make_int4(gl, (int)tri, (int)c, si);
                    count = 0;                          // walked by k_raster_big
                } else {
                    // the reservation straddles the queue's end: publish no
                    // work in its in-range part (k_raster_big walks every
                    // entry below min(nbig, cap)) and walk the triangle's box
                    // here -- exact, but slow for span-mode regions (the
                    // queue holds 16M chunks; C5 needs ~3.7M)
                    for (unsigned long long w = at; w < cap; ++w) a.big[w] = make_int4(-1, 0, 0, 0);
                    if (a.stats) atomicAdd(a.stats + 2, 1ULL);
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
        if (lane == 0 && a.stats) atomicAdd(a.stats, (unsigned long long)total);
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

// Chunks of big (or WIDE) triangles: a warp takes one chunk (kBigChunk
// candidates of one triangle's bounding box, line-major), recomputes the
// (identical) set-up and walks the chunk's lines 32 at a time: lane r takes
// line r's cells inside the half-plane span (not the whole box line), then
// the warp walks the concatenated spans 32 cells at a time.
template <int STORAGE>
__global__ void __launch_bounds__(kRasterThreads, SBR_RASTER_MINB)
k_raster_big(RasterArgs a)
{
    const int lane = threadIdx.x & 31;
    const unsigned long long nbig = *a.nbig;
    const unsigned long long n = nbig < (unsigned long long)a.big_cap ? nbig : a.big_cap;
    unsigned long long w_next = 0, w_end = 0;   // claimed kBigClaim chunks at a time
    while (true) {
        if (w_next >= w_end) {
            unsigned long long got = 0;
            if (lane == 0) got = atomicAdd(a.counter, (unsigned long long)kBigClaim);
            w_next = __shfl_sync(0xffffffffu, got, 0);
            w_end = w_next + kBigClaim;
        }
        const unsigned long long w = w_next++;
        if (w >= n) break;
        const int4 it = a.big[w];
        if (it.x < 0) continue;                 // unpublished (overflowed reservation)
        const int g = __ldg(&a.bgrids[it.x]);
        const GridDev &G = a.grids[g];
        const int64_t *seg = a.seg_slot + __ldg(&a.seg_base[g]);
        RasterSetup S;
        if (it.w >= 0) {   // published by k_raster (already trimmed to owned rows)
            S = *reinterpret_cast<const RasterSetup *>(a.setups +
                                                       (size_t)it.w * kRasterSetupBytes);
        } else {
            S = raster_setup(load_tri<STORAGE>(a.B, it.y), G, a.row_lo, a.row_hi);
            if (a.sparse) trim_owned(S, G, seg);
        }
        const long long width = S.trans ? S.rows : (long long)S.cols;   // cells per line
        const long long l0 = S.trans ? S.j0 : S.i0, m0 = S.trans ? S.i0 : S.j0;
        long long c0, c1, line_a, line_b;
        const bool segm = seg_chunks(a, S);
        int64_t seg_lo = 0, seg_hi = -1;
        if (segm) {     // the rows of one segment (clipped to it per line below)
            int64_t qa, qb;
            seg_range(S, G.n_v, qa, qb);
            const int64_t q = qa + it.z;
            seg_lo = q * kSegRays;
            seg_hi = seg_lo + kSegRays - 1;
            const int64_t ra = seg_lo / G.n_v, rz = seg_hi / G.n_v;
            line_a = (ra > S.i0 ? ra : S.i0) - S.i0;
            line_b = (rz < S.i0 + S.rows - 1 ? rz : S.i0 + S.rows - 1) - S.i0;
            if (line_a > line_b) continue;
            c0 = line_a * width;
            c1 = (line_b + 1) * width;
        } else if (S.span) {   // 32 whole lines
            line_a = 32LL * it.z;
            line_b = line_a + 31 < span_lines(S) - 1 ? line_a + 31 : span_lines(S) - 1;
            if (line_a > line_b) continue;
            c0 = line_a * width;
            c1 = (line_b + 1) * width;
        } else {
            c0 = (long long)it.z * kBigChunk;
            c1 = c0 + kBigChunk < S.count ? c0 + kBigChunk : S.count;
            if (c0 >= c1) continue;
            line_a = c0 / width;
            line_b = (c1 - 1) / width;
        }
        for (long long lbase = line_a; lbase <= line_b; lbase += 32) {
            const long long li = lbase + lane;
            long long ml = 0, mr = -1;
            if (li <= line_b) {
                const long long wl = li == line_a ? c0 % width : 0;
                const long long wr = li == line_b ? (c1 - 1) % width : width - 1;
                double lo, hi;
                line_span(S, (double)(l0 + li), lo, hi);
                if (lo <= (double)(m0 + wr) && hi >= (double)(m0 + wl)) {
                    ml = lo > (double)(m0 + wl) ? (long long)ceil(lo) - m0 : wl;
                    mr = hi < (double)(m0 + wr) ? (long long)floor(hi) - m0 : wr;
                }
                if (segm && mr >= ml) {   // exactly this chunk's segment
                    const int64_t rb = (l0 + li) * G.n_v + m0;
                    if (seg_lo - rb > ml) ml = seg_lo - rb;
                    if (seg_hi - rb < mr) mr = seg_hi - rb;
                } else if (a.sparse && !S.trans && mr >= ml) {
                    // ray-tile shards: a row meets at most two segments (n_v <
                    // kSegRays); keep only the cells of the owned one(s)
                    const int64_t rb = (l0 + li) * G.n_v + m0;
                    const int64_t qa = (rb + ml) / kSegRays, qb = (rb + mr) / kSegRays;
                    const bool oa = __ldg(&seg[qa]) != kNoSlot;
                    const bool ob = qb == qa ? oa : __ldg(&seg[qb]) != kNoSlot;
                    if (!oa && !ob) {
                        mr = ml - 1;
                    } else if (!oa) {
                        ml = qb * kSegRays - rb;
                    } else if (!ob) {
                        mr = qb * kSegRays - 1 - rb;
                    }
                }
            }
            const int cnt = mr >= ml ? (int)(mr - ml + 1) : 0;
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            if (lane == 0 && a.stats && total) atomicAdd(a.stats, (unsigned long long)total);
            const int excl = incl - cnt;
            const int ml32 = (int)ml;
            for (int base = 0; base < total; base += 32) {
                const int c = base + lane;
                int owner = 0;   // first lane whose inclusive count exceeds c
#pragma unroll
                for (int st = 16; st >= 1; st >>= 1)
                    if (__shfl_sync(0xffffffffu, incl, owner + st - 1) <= c) owner += st;
                const int oex = __shfl_sync(0xffffffffu, excl, owner);
                const int oml = __shfl_sync(0xffffffffu, ml32, owner);
                if (c < total) {
                    const long long line = l0 + lbase + owner, m = m0 + oml + (c - oex);
                    raster_cell(a, G, seg, S.T, S.P, S.inv, S.T.id, S.trans ? m : line,
                                S.trans ? line : m);
                }
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
    const int claim = warps >= (int64_t)64 * blocks * kRasterWarps ? kRasterClaim : 1;
    k_raster<S><<<(unsigned)blocks, kRasterThreads, 0, st>>>(a, ntri_pad, claim);
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
    if (e == cudaSuccess && a.setups)
        e = cudaMemsetAsync(a.nsetup, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    if (a.storage == kF64) raster_dispatch<kF64>(a, st, ls.num_sms);
    else if (a.storage == kSingle) raster_dispatch<kSingle>(a, st, ls.num_sms);
    else raster_dispatch<kF32Exact>(a, st, ls.num_sms);
    *ls.launches += a.big ? 2 : 1;
    return cudaGetLastError();
}

}  // namespace sbr
