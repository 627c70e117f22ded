// sbr_device.cuh -- device data layout and the exact/conservative
// intersection primitives shared by the trace, LBVH and PO kernels.
//
// Exactness contract: the closest hit of a query is the
// lexicographic minimum of (t, triangle id) over every triangle whose
// Moller-Trumbore test accepts the ray (pkg/src/sbr/bvh.py:340).  That set
// does not depend on the tree, so any BVH whose box culling is conservative
// returns the reference result bit-for-bit, provided the per-triangle
// arithmetic is bit-identical.  Hence:
//   * tri_hit_exact() mirrors geometry.py:326-355 operation by operation
//     with explicit round-to-nearest FP64 intrinsics (no FMA contraction,
//     identical association);
//   * box tests run in FP32 on outward-rounded boxes with a per-ray padding
//     (RayBox) that dominates every rounding error of the FP32 slab test,
//     so they only ever cull boxes that cannot contain an accepted hit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sbr {

// ---------------------------------------------------------------------------
// Node / triangle layout in HBM
// ---------------------------------------------------------------------------
// Child-pair BVH2 node, 64 B = four 16-byte loads:
//   a = (c0.lo.x, c0.lo.y, c0.lo.z, c0.hi.x)
//   b = (c0.hi.y, c0.hi.z, c1.lo.x, c1.lo.y)
//   c = (c1.lo.z, c1.hi.x, c1.hi.y, c1.hi.z)
//   d = (ref0, ref1, -, -)
// Boxes are FP32, relative to the scene centre (BvhView::c*), rounded
// outward.  A child reference >= 0 is an internal node index; < 0 is a leaf
// encoding (first triangle slot, count) -- see leaf_ref().
struct __align__(16) Node {
    float4 a, b, c;
    int4 d;
};

// 4-wide node, 128 B = one cache line = eight 16-byte loads, boxes SoA by
// axis so the four slab tests vectorise naturally:
//   lox, loy, loz, hix, hiy, hiz (4 children each), ref (4 child refs)
// An absent child has ref == kEmptyRef and is never hit.
struct __align__(128) Node4 {
    float4 lox, loy, loz, hix, hiy, hiz;
    int4 ref;
    int4 pad;
};
constexpr int kEmptyRef = 0x7fffffff;

// 4-wide node with 8-bit quantised child boxes, 64 B (half a line, four
// loads instead of eight).  Per axis a: plane = p_a + q * 2^e_a with the
// child box rounded OUTWARD onto that grid at build time (k_quantize4);
// the slab test folds the decode into its fma (node4q_visit).
struct __align__(64) Node4Q {
    float px, py, pz;     // quantisation origin (box frame)
    unsigned int exps;    // biased float exponents of the scales: ex | ey << 8 | ez << 16
    int4 ref;
    unsigned int q[6];    // planes lox loy loz hix hiy hiz; child k in byte k
    unsigned int pad[2];
};
static_assert(sizeof(Node4Q) == 64, "Node4Q is half a line");

// 8-wide node with quantised child boxes, 96 B (three sectors): header,
// eight refs, six planes of eight bytes (plane j in q[2j], q[2j+1]).
struct __align__(32) Node8Q {
    float px, py, pz;
    unsigned int exps;
    int4 ref[2];
    unsigned int q[12];
};
static_assert(sizeof(Node8Q) == 96, "Node8Q is three sectors");

// 8-wide node, 256 B = two cache lines: the same SoA planes with eight
// children each (two float4 per plane), eight refs, padding.
struct __align__(128) Node8 {
    float4 lox[2], loy[2], loz[2], hix[2], hiy[2], hiz[2];
    int4 ref[2];
    int4 pad[2];
};
static_assert(sizeof(Node8) == 256, "Node8 is two lines");

constexpr int kLeafCountShift = 25;
constexpr int kLeafFirstMask = (1 << kLeafCountShift) - 1;
constexpr int kMaxLeafCount = 63;
constexpr int64_t kMaxTriangles = (int64_t)1 << kLeafCountShift;
constexpr int kStack = 96;   // traversal stack entries (<= 3 per BVH4 level)
constexpr int kMaxDepth4 = 31;  // deepest BVH4 level accepted (3 * 31 + 1 < kStack)

__host__ __device__ inline int leaf_ref(int first, int count)
{
    return (int)(0x80000000u | ((unsigned)count << kLeafCountShift) | (unsigned)first);
}
__host__ __device__ inline int leaf_first(int ref) { return ref & kLeafFirstMask; }
__host__ __device__ inline int leaf_count(int ref) { return (ref >> kLeafCountShift) & kMaxLeafCount; }

// Triangle storage in leaf order.
//   F32 (float32-representable vertices): 3 x float4 = 48 B
//     t0 = (v0.x v0.y v0.z v1.x) t1 = (v1.y v1.z v2.x v2.y) t2 = (v2.z id - -)
//   F64: 5 x double2 = 80 B: (v0.x v0.y)(v0.z v1.x)(v1.y v1.z)(v2.x v2.y)(v2.z id)
enum Storage : int { kF32Exact = 1, kF64 = 2, kSingle = 3 };

struct BvhView {
    const Node *nodes;       // binary tree (build / export)
    const Node4 *nodes4;     // 4-wide tree (traversal)
    const Node4Q *nodes4q;   // the same tree with quantised child boxes
    const Node8 *nodes8;     // 8-wide tree (traversal when width == 8)
    const Node8Q *nodes8q;   // the same with quantised child boxes
    int width;               // 4 or 8: which wide tree the trace kernel walks
    const float4 *tri32;
    const double2 *tri64;
    const double *normals;   // (T,3), original triangle order
    double cx, cy, cz;       // box frame origin
    float scale;             // max |box coordinate| in the box frame
    int root;                // root reference (internal node 0, or a leaf)
};

// ---------------------------------------------------------------------------
// Exact FP64 Moller-Trumbore (geometry.py:326-355)
// ---------------------------------------------------------------------------
#define DM(a, b) __dmul_rn((a), (b))
#define DA(a, b) __dadd_rn((a), (b))
#define DS(a, b) __dsub_rn((a), (b))

struct TriF64 {
    double ax, ay, az, e1x, e1y, e1z, e2x, e2y, e2z;
    int id;
};

template <int STORAGE>
__device__ __forceinline__ TriF64 load_tri(const BvhView &B, int k)
{
    TriF64 r;
    if (STORAGE == kF64) {
        const double2 *p = B.tri64 + 5 * (int64_t)k;
        double2 q0 = __ldg(p), q1 = __ldg(p + 1), q2 = __ldg(p + 2),
                q3 = __ldg(p + 3), q4 = __ldg(p + 4);
        r.ax = q0.x; r.ay = q0.y; r.az = q1.x;
        r.e1x = DS(q1.y, r.ax); r.e1y = DS(q2.x, r.ay); r.e1z = DS(q2.y, r.az);
        r.e2x = DS(q3.x, r.ax); r.e2y = DS(q3.y, r.ay); r.e2z = DS(q4.x, r.az);
        r.id = (int)__double_as_longlong(q4.y);
    } else {
        const float4 *p = B.tri32 + 3 * (int64_t)k;
        float4 t0 = __ldg(p), t1 = __ldg(p + 1), t2 = __ldg(p + 2);
        r.ax = t0.x; r.ay = t0.y; r.az = t0.z;
        if (STORAGE == kSingle) {
            // reference precision="single": float32 arrays subtract in float32
            r.e1x = __fsub_rn(t0.w, t0.x); r.e1y = __fsub_rn(t1.x, t0.y);
            r.e1z = __fsub_rn(t1.y, t0.z);
            r.e2x = __fsub_rn(t1.z, t0.x); r.e2y = __fsub_rn(t1.w, t0.y);
            r.e2z = __fsub_rn(t2.x, t0.z);
        } else {
            r.e1x = DS((double)t0.w, r.ax); r.e1y = DS((double)t1.x, r.ay);
            r.e1z = DS((double)t1.y, r.az);
            r.e2x = DS((double)t1.z, r.ax); r.e2y = DS((double)t1.w, r.ay);
            r.e2z = DS((double)t2.x, r.az);
        }
        r.id = __float_as_int(t2.y);
    }
    return r;
}

// Direction-only part of the test: p = d x e2 and det = e1 . p
// (geometry.py:336-339).  Identical for every ray of one aperture, so the
// primary-visibility pass hoists it out of its per-cell loop.
struct TriDir {
    double px, py, pz, det;
};

__device__ __forceinline__ TriDir tri_dir(const TriF64 &T, double dx, double dy, double dz)
{
    TriDir r;
    r.px = DS(DM(dy, T.e2z), DM(dz, T.e2y));
    r.py = DS(DM(dz, T.e2x), DM(dx, T.e2z));
    r.pz = DS(DM(dx, T.e2y), DM(dy, T.e2x));
    r.det = DA(DA(DM(T.e1x, r.px), DM(T.e1y, r.py)), DM(T.e1z, r.pz));
    return r;
}

// Origin-dependent part (geometry.py:340-355) for det != 0.  HAVE_INV: the
// caller passes inv == __drcp_rn(det) (== IEEE 1.0 / det); otherwise it is
// computed here, after the division-free pre-filters.
template <bool HAVE_INV>
__device__ __forceinline__ double tri_hit_origin(const TriF64 &T, const TriDir &P, double inv,
                                                 double ox, double oy, double oz, double dx,
                                                 double dy, double dz, double t_min,
                                                 double t_max)
{
    const double det = P.det;
    double tx = DS(ox, T.ax), ty = DS(oy, T.ay), tz = DS(oz, T.az);
    double un = DA(DA(DM(tx, P.px), DM(ty, P.py)), DM(tz, P.pz));
    // Division-free pre-filters.  They only reject rays the exact test below
    // rejects too: with 1e-150 < |un|, |det| < 1e150 the rounded product
    // un * fl(1/det) is a normal number carrying the sign of un*det, so
    // opposite signs mean u < 0; |un| > 2|det| means u > 1 after rounding.
    const double adet = fabs(det);
    const bool safe = adet < 1e150;
    if (safe && fabs(un) > 1e-150 && ((un < 0.0) != (det < 0.0))) return -1.0;
    if (safe && fabs(un) > 2.0 * adet) return -1.0;
    double qx = DS(DM(ty, T.e1z), DM(tz, T.e1y));
    double qy = DS(DM(tz, T.e1x), DM(tx, T.e1z));
    double qz = DS(DM(tx, T.e1y), DM(ty, T.e1x));
    double vn = DA(DA(DM(dx, qx), DM(dy, qy)), DM(dz, qz));
    if (safe && fabs(vn) > 1e-150 && ((vn < 0.0) != (det < 0.0))) return -1.0;
    // exact reference sequence (geometry.py:340-352)
    if (!HAVE_INV) inv = __drcp_rn(det);  // == IEEE 1.0 / det
    double u = DM(un, inv);
    if (u < 0.0 || u > 1.0) return -1.0;
    double v = DM(vn, inv);
    if (v < 0.0 || DA(u, v) > 1.0) return -1.0;
    double t = DM(DA(DA(DM(T.e2x, qx), DM(T.e2y, qy)), DM(T.e2z, qz)), inv);
    if (t <= t_min || t > t_max) return -1.0;
    return t;
}

// Returns t in (t_min, t_max] or -1.0 (edge-inclusive), bit-identical to
// the reference.  Operand association: a*b + c*d + e*f == (ab + cd) + ef.
__device__ __forceinline__ double tri_hit_exact(const TriF64 &T, double ox,
                                                double oy, double oz, double dx,
                                                double dy, double dz,
                                                double t_min, double t_max)
{
    const TriDir P = tri_dir(T, dx, dy, dz);
    if (P.det == 0.0) return -1.0;
    return tri_hit_origin<false>(T, P, 0.0, ox, oy, oz, dx, dy, dz, t_min, t_max);
}

// Closest-hit queries on a float32 mesh (reference closest_hit /
// closest_hit_batch, bvh.py:395-423, cast the RAYS to the mesh dtype too):
// numba then evaluates _tri_hit_t (geometry.py:326-355) with float32
// vertices and rays -- edges, p, det, the t-vector, q and the three dot
// products in float32 (no contraction) -- and only inv_det = 1.0 / det (a
// float64 literal) and the products with it in float64.  T comes from
// load_tri<kSingle> (float32 values held exactly in doubles); o and d must
// be float32-representable.
__device__ __forceinline__ double tri_hit_f32rays(const TriF64 &T, double oxd, double oyd,
                                                  double ozd, double dxd, double dyd,
                                                  double dzd, double t_min, double t_max)
{
#define FM(a, b) __fmul_rn((a), (b))
#define FA(a, b) __fadd_rn((a), (b))
#define FS(a, b) __fsub_rn((a), (b))
    const float ox = (float)oxd, oy = (float)oyd, oz = (float)ozd;
    const float dx = (float)dxd, dy = (float)dyd, dz = (float)dzd;
    const float ax = (float)T.ax, ay = (float)T.ay, az = (float)T.az;
    const float e1x = (float)T.e1x, e1y = (float)T.e1y, e1z = (float)T.e1z;
    const float e2x = (float)T.e2x, e2y = (float)T.e2y, e2z = (float)T.e2z;
    const float px = FS(FM(dy, e2z), FM(dz, e2y));
    const float py = FS(FM(dz, e2x), FM(dx, e2z));
    const float pz = FS(FM(dx, e2y), FM(dy, e2x));
    const float det = FA(FA(FM(e1x, px), FM(e1y, py)), FM(e1z, pz));
    if (det == 0.0f) return -1.0;
    const double inv = __drcp_rn((double)det);   // == IEEE 1.0 / det in float64
    const float tx = FS(ox, ax), ty = FS(oy, ay), tz = FS(oz, az);
    const double u = DM((double)FA(FA(FM(tx, px), FM(ty, py)), FM(tz, pz)), inv);
    if (u < 0.0 || u > 1.0) return -1.0;
    const float qx = FS(FM(ty, e1z), FM(tz, e1y));
    const float qy = FS(FM(tz, e1x), FM(tx, e1z));
    const float qz = FS(FM(tx, e1y), FM(ty, e1x));
    const double v = DM((double)FA(FA(FM(dx, qx), FM(dy, qy)), FM(dz, qz)), inv);
    if (v < 0.0 || DA(u, v) > 1.0) return -1.0;
    const double t = DM((double)FA(FA(FM(e2x, qx), FM(e2y, qy)), FM(e2z, qz)), inv);
    if (t <= t_min || t > t_max) return -1.0;
    return t;
#undef FM
#undef FA
#undef FS
}

// ---------------------------------------------------------------------------
// Conservative FP32 slab test
// ---------------------------------------------------------------------------
// For each axis the padded slab [lo - delta, hi + delta] is evaluated as
//   t_lo = fma(lo, inv, off_lo), off_lo = -(o' + delta) * inv
//   t_hi = fma(hi, inv, off_hi), off_hi = -(o' - delta) * inv
// (the near plane of the pair is lo for inv >= 0, hi otherwise)
// with o' = fl32(o - c).  Every rounding error (origin conversion, the
// reciprocal, the offsets, the fma) is a position error bounded by a few
// ulp of (|o'| + scale); delta = 2^-17 (|o'|_inf + scale) exceeds that by
// more than 10x, so the computed interval contains the exact interval of
// the unpadded box: culling is conservative, never result-changing.
struct RayBox {
    float ix, iy, iz;
    float nx, ny, nz;   // offsets of the near planes (off_lo if inv >= 0 else off_hi)
    float fx, fy, fz;   // offsets of the far planes
    int sel;            // float4 index of the near plane per axis: x | y << 3 | z << 6
};

__device__ __forceinline__ float safe_dir(float d)
{
    return fabsf(d) < 1e-20f ? (d < 0.f ? -1e-20f : 1e-20f) : d;
}

__device__ __forceinline__ RayBox make_raybox(const BvhView &B, double ox, double oy,
                                              double oz, double dx, double dy,
                                              double dz)
{
    RayBox r;
    const float fx = __double2float_rn(ox - B.cx);
    const float fy = __double2float_rn(oy - B.cy);
    const float fz = __double2float_rn(oz - B.cz);
    const float m = fmaxf(fmaxf(fabsf(fx), fabsf(fy)), fabsf(fz));
    const float delta = (m + B.scale) * 7.62939453125e-06f;  // 2^-17
    r.ix = __frcp_rn(safe_dir(__double2float_rn(dx)));   // correctly rounded 1/d
    r.iy = __frcp_rn(safe_dir(__double2float_rn(dy)));
    r.iz = __frcp_rn(safe_dir(__double2float_rn(dz)));
    const float lx = -(fx + delta) * r.ix, hx = -(fx - delta) * r.ix;
    const float ly = -(fy + delta) * r.iy, hy = -(fy - delta) * r.iy;
    const float lz = -(fz + delta) * r.iz, hz = -(fz - delta) * r.iz;
    // near plane = lo for a positive component, hi for a negative one;
    // Node4 float4 order: lox loy loz hix hiy hiz -> indices 0..5
    const bool sx = r.ix < 0.f, sy = r.iy < 0.f, sz = r.iz < 0.f;
    r.nx = sx ? hx : lx; r.fx = sx ? lx : hx;
    r.ny = sy ? hy : ly; r.fy = sy ? ly : hy;
    r.nz = sz ? hz : lz; r.fz = sz ? lz : hz;
    r.sel = (sx ? 3 : 0) | (sy ? 4 : 1) << 3 | (sz ? 5 : 2) << 6;
    return r;
}

// 4-element compare-exchange on (key, ref) pairs
__device__ __forceinline__ void cswap(float &ka, int &va, float &kb, int &vb)
{
    const bool s = kb < ka;
    const float k = s ? kb : ka;
    kb = s ? ka : kb;
    ka = k;
    const int v = s ? vb : va;
    vb = s ? va : vb;
    va = v;
}

// Visit one BVH4 node: slab-test its four children against the padded
// boxes (only the ray's near planes give entry distances and its far planes
// exit distances, so no per-axis min/max) and return the hit children
// ordered near -> far by entry distance; the count is the return value.
__device__ __forceinline__ int node4_visit(const Node4 *np, const RayBox &r, float tmax,
                                           int ref[4], float tn[4])
{
    const float4 *q = reinterpret_cast<const float4 *>(np);
    const int nxi = r.sel & 7, nyi = (r.sel >> 3) & 7, nzi = (r.sel >> 6) & 7;
    const float4 nxv = __ldg(q + nxi), fxv = __ldg(q + (3 - nxi));
    const float4 nyv = __ldg(q + nyi), fyv = __ldg(q + (5 - nyi));
    const float4 nzv = __ldg(q + nzi), fzv = __ldg(q + (7 - nzi));
    const int4 rf = __ldg(&np->ref);
    const float inf = __int_as_float(0x7f800000);
#define SBR_SLAB(c, k)                                                                     \
    {                                                                                      \
        const float a = fmaxf(fmaxf(fmaf(nxv.c, r.ix, r.nx), fmaf(nyv.c, r.iy, r.ny)),     \
                              fmaxf(fmaf(nzv.c, r.iz, r.nz), 0.0f));                       \
        const float b = fminf(fminf(fmaf(fxv.c, r.ix, r.fx), fmaf(fyv.c, r.iy, r.fy)),     \
                              fminf(fmaf(fzv.c, r.iz, r.fz), tmax));                       \
        tn[k] = (a <= b && rf.c != kEmptyRef) ? a : inf;                                   \
    }
    SBR_SLAB(x, 0)
    SBR_SLAB(y, 1)
    SBR_SLAB(z, 2)
    SBR_SLAB(w, 3)
#undef SBR_SLAB
    const int n = (tn[0] != inf) + (tn[1] != inf) + (tn[2] != inf) + (tn[3] != inf);
    ref[0] = rf.x; ref[1] = rf.y; ref[2] = rf.z; ref[3] = rf.w;
    // 4-element sorting network, misses (+inf) sink to the end
    cswap(tn[0], ref[0], tn[1], ref[1]);
    cswap(tn[2], ref[2], tn[3], ref[3]);
    cswap(tn[0], ref[0], tn[2], ref[2]);
    cswap(tn[1], ref[1], tn[3], ref[3]);
    cswap(tn[1], ref[1], tn[2], ref[2]);
    return n;
}

// Visit one BVH8 node: eight padded slab tests (two float4 per plane), hit
// children sorted near -> far by an optimal 19-comparator network; misses
// (+inf) sink to the end.  Returns the hit count.
__device__ __forceinline__ int node8_visit(const Node8 *np, const RayBox &r, float tmax,
                                           int ref[8], float tn[8])
{
    const float4 *q = reinterpret_cast<const float4 *>(np);
    const int nxi = r.sel & 7, nyi = (r.sel >> 3) & 7, nzi = (r.sel >> 6) & 7;
    const float inf = __int_as_float(0x7f800000);
    int n = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const float4 nxv = __ldg(q + 2 * nxi + h), fxv = __ldg(q + 2 * (3 - nxi) + h);
        const float4 nyv = __ldg(q + 2 * nyi + h), fyv = __ldg(q + 2 * (5 - nyi) + h);
        const float4 nzv = __ldg(q + 2 * nzi + h), fzv = __ldg(q + 2 * (7 - nzi) + h);
        const int4 rf = __ldg(&np->ref[h]);
#define SBR_SLAB8(c, k)                                                                    \
        {                                                                                  \
            const float a = fmaxf(fmaxf(fmaf(nxv.c, r.ix, r.nx), fmaf(nyv.c, r.iy, r.ny)), \
                                  fmaxf(fmaf(nzv.c, r.iz, r.nz), 0.0f));                   \
            const float b = fminf(fminf(fmaf(fxv.c, r.ix, r.fx), fmaf(fyv.c, r.iy, r.fy)), \
                                  fminf(fmaf(fzv.c, r.iz, r.fz), tmax));                   \
            tn[4 * h + k] = (a <= b && rf.c != kEmptyRef) ? a : inf;                       \
            ref[4 * h + k] = rf.c;                                                         \
            n += tn[4 * h + k] != inf;                                                     \
        }
        SBR_SLAB8(x, 0)
        SBR_SLAB8(y, 1)
        SBR_SLAB8(z, 2)
        SBR_SLAB8(w, 3)
#undef SBR_SLAB8
    }
#define SBR_CS(i, j) cswap(tn[i], ref[i], tn[j], ref[j]);
    SBR_CS(0, 2) SBR_CS(1, 3) SBR_CS(4, 6) SBR_CS(5, 7)
    SBR_CS(0, 4) SBR_CS(1, 5) SBR_CS(2, 6) SBR_CS(3, 7)
    SBR_CS(0, 1) SBR_CS(2, 3) SBR_CS(4, 5) SBR_CS(6, 7)
    SBR_CS(2, 4) SBR_CS(3, 5)
    SBR_CS(1, 4) SBR_CS(3, 6)
    SBR_CS(1, 2) SBR_CS(3, 4) SBR_CS(5, 6)
#undef SBR_CS
    return n;
}

// byte k of w as an exact float (0x4B0000kk = 2^23 + k)
__device__ __forceinline__ float qbyte(unsigned int w, int k)
{
    return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7540 | k)) - 8388608.0f;
}

// Visit one quantised BVH4 node.  t = fma(q, 2^e inv, fma(p, inv, off)):
// the exact plane p + q 2^e (outward-rounded, so it contains the child box)
// times inv plus the padded offset, with two roundings where node4_visit has
// one -- a few ulp of (|o'| + scale), still far inside the 2^-17 padding.
__device__ __forceinline__ int node4q_visit(const Node4Q *np, const RayBox &r, float tmax,
                                            int ref[4], float tn[4])
{
    const uint4 h = __ldg(reinterpret_cast<const uint4 *>(np));
    const int4 rf = __ldg(&np->ref);
    const uint4 qa = __ldg(reinterpret_cast<const uint4 *>(np->q));
    const uint2 qb = __ldg(reinterpret_cast<const uint2 *>(np->q + 4));
    const float px = __uint_as_float(h.x), py = __uint_as_float(h.y), pz = __uint_as_float(h.z);
    const float ax = __uint_as_float((h.w & 0xffu) << 23) * r.ix;
    const float ay = __uint_as_float(((h.w >> 8) & 0xffu) << 23) * r.iy;
    const float az = __uint_as_float(((h.w >> 16) & 0xffu) << 23) * r.iz;
    const float bnx = fmaf(px, r.ix, r.nx), bfx = fmaf(px, r.ix, r.fx);
    const float bny = fmaf(py, r.iy, r.ny), bfy = fmaf(py, r.iy, r.fy);
    const float bnz = fmaf(pz, r.iz, r.nz), bfz = fmaf(pz, r.iz, r.fz);
    // near plane per axis: lo when the float4 index in sel is the lo one
    const bool lx = (r.sel & 7) == 0, ly = ((r.sel >> 3) & 7) == 1, lz = ((r.sel >> 6) & 7) == 2;
    const unsigned int wnx = lx ? qa.x : qa.w, wfx = lx ? qa.w : qa.x;
    const unsigned int wny = ly ? qa.y : qb.x, wfy = ly ? qb.x : qa.y;
    const unsigned int wnz = lz ? qa.z : qb.y, wfz = lz ? qb.y : qa.z;
    const float inf = __int_as_float(0x7f800000);
    const int rr[4] = {rf.x, rf.y, rf.z, rf.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float a = fmaxf(fmaxf(fmaf(qbyte(wnx, k), ax, bnx), fmaf(qbyte(wny, k), ay, bny)),
                              fmaxf(fmaf(qbyte(wnz, k), az, bnz), 0.0f));
        const float b = fminf(fminf(fmaf(qbyte(wfx, k), ax, bfx), fmaf(qbyte(wfy, k), ay, bfy)),
                              fminf(fmaf(qbyte(wfz, k), az, bfz), tmax));
        tn[k] = (a <= b && rr[k] != kEmptyRef) ? a : inf;
        ref[k] = rr[k];
    }
    const int n = (tn[0] != inf) + (tn[1] != inf) + (tn[2] != inf) + (tn[3] != inf);
    cswap(tn[0], ref[0], tn[1], ref[1]);
    cswap(tn[2], ref[2], tn[3], ref[3]);
    cswap(tn[0], ref[0], tn[2], ref[2]);
    cswap(tn[1], ref[1], tn[3], ref[3]);
    cswap(tn[1], ref[1], tn[2], ref[2]);
    return n;
}

// Visit one quantised BVH8 node (decode as node4q_visit), hit children
// sorted near -> far by the 19-comparator network of node8_visit.
__device__ __forceinline__ int node8q_visit(const Node8Q *np, const RayBox &r, float tmax,
                                            int ref[8], float tn[8])
{
    const uint4 h = __ldg(reinterpret_cast<const uint4 *>(np));
    const int4 r0 = __ldg(&np->ref[0]), r1 = __ldg(&np->ref[1]);
    const uint4 qa = __ldg(reinterpret_cast<const uint4 *>(np->q));
    const uint4 qb = __ldg(reinterpret_cast<const uint4 *>(np->q + 4));
    const uint4 qc = __ldg(reinterpret_cast<const uint4 *>(np->q + 8));
    // planes: lox = (qa.x, qa.y), loy = (qa.z, qa.w), loz = (qb.x, qb.y),
    //         hix = (qb.z, qb.w), hiy = (qc.x, qc.y), hiz = (qc.z, qc.w)
    const float px = __uint_as_float(h.x), py = __uint_as_float(h.y), pz = __uint_as_float(h.z);
    const float ax = __uint_as_float((h.w & 0xffu) << 23) * r.ix;
    const float ay = __uint_as_float(((h.w >> 8) & 0xffu) << 23) * r.iy;
    const float az = __uint_as_float(((h.w >> 16) & 0xffu) << 23) * r.iz;
    const float bnx = fmaf(px, r.ix, r.nx), bfx = fmaf(px, r.ix, r.fx);
    const float bny = fmaf(py, r.iy, r.ny), bfy = fmaf(py, r.iy, r.fy);
    const float bnz = fmaf(pz, r.iz, r.nz), bfz = fmaf(pz, r.iz, r.fz);
    const bool lx = (r.sel & 7) == 0, ly = ((r.sel >> 3) & 7) == 1, lz = ((r.sel >> 6) & 7) == 2;
    const unsigned int wnx[2] = {lx ? qa.x : qb.z, lx ? qa.y : qb.w};
    const unsigned int wfx[2] = {lx ? qb.z : qa.x, lx ? qb.w : qa.y};
    const unsigned int wny[2] = {ly ? qa.z : qc.x, ly ? qa.w : qc.y};
    const unsigned int wfy[2] = {ly ? qc.x : qa.z, ly ? qc.y : qa.w};
    const unsigned int wnz[2] = {lz ? qb.x : qc.z, lz ? qb.y : qc.w};
    const unsigned int wfz[2] = {lz ? qc.z : qb.x, lz ? qc.w : qb.y};
    const float inf = __int_as_float(0x7f800000);
    const int rr[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    int n = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int hh = k >> 2, kk = k & 3;
        const float a = fmaxf(fmaxf(fmaf(qbyte(wnx[hh], kk), ax, bnx), fmaf(qbyte(wny[hh], kk), ay, bny)),
                              fmaxf(fmaf(qbyte(wnz[hh], kk), az, bnz), 0.0f));
        const float b = fminf(fminf(fmaf(qbyte(wfx[hh], kk), ax, bfx), fmaf(qbyte(wfy[hh], kk), ay, bfy)),
                              fminf(fmaf(qbyte(wfz[hh], kk), az, bfz), tmax));
        tn[k] = (a <= b && rr[k] != kEmptyRef) ? a : inf;
        ref[k] = rr[k];
        n += tn[k] != inf;
    }
#define SBR_CS(i, j) cswap(tn[i], ref[i], tn[j], ref[j]);
    SBR_CS(0, 2) SBR_CS(1, 3) SBR_CS(4, 6) SBR_CS(5, 7)
    SBR_CS(0, 4) SBR_CS(1, 5) SBR_CS(2, 6) SBR_CS(3, 7)
    SBR_CS(0, 1) SBR_CS(2, 3) SBR_CS(4, 5) SBR_CS(6, 7)
    SBR_CS(2, 4) SBR_CS(3, 5)
    SBR_CS(1, 4) SBR_CS(3, 6)
    SBR_CS(1, 2) SBR_CS(3, 4) SBR_CS(5, 6)
#undef SBR_CS
    return n;
}

// width-generic visit used by the traversal loops
template <int W> struct WideNode;
template <> struct WideNode<4> {
#ifdef SBR_NODE_Q
    using T = Node4Q;
    static __device__ __forceinline__ int visit(const Node4Q *p, const RayBox &r, float tmax,
                                                int *ref, float *tn)
    {
        return node4q_visit(p, r, tmax, ref, tn);
    }
#else
    using T = Node4;
    static __device__ __forceinline__ int visit(const Node4 *p, const RayBox &r, float tmax,
                                                int *ref, float *tn)
    {
        return node4_visit(p, r, tmax, ref, tn);
    }
#endif
};
template <> struct WideNode<8> {
#ifdef SBR_NODE_Q
    using T = Node8Q;
    static __device__ __forceinline__ int visit(const Node8Q *p, const RayBox &r, float tmax,
                                                int *ref, float *tn)
    {
        return node8q_visit(p, r, tmax, ref, tn);
    }
#else
    using T = Node8;
    static __device__ __forceinline__ int visit(const Node8 *p, const RayBox &r, float tmax,
                                                int *ref, float *tn)
    {
        return node8_visit(p, r, tmax, ref, tn);
    }
#endif
};

}  // namespace sbr
