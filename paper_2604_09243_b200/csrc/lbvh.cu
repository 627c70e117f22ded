// lbvh.cu -- GPU LBVH build (replaces the serial recursive build of
// pkg/src/sbr/bvh.py:218-299).
//
// Pipeline (one stream, all on device):
//   1. k_morton    : triangle AABB (FP64, exact), centroid = box centre
//                    (bvh.py:229-231), 63-bit Morton code over the centroid
//                    bounds; value = triangle index.
//   2. CUB radix sort of (code, index) pairs (stable: equal codes keep
//      index order, so the tree is deterministic).
//   3. k_karras    : binary radix tree (Karras 2012) with index tie-break
//                    for duplicate codes; internal node i covers a
//                    contiguous range of sorted primitives.
//   4. k_refit     : bottom-up FP64 box union with arrival counters
//                    (exact min/max -> order independent -> deterministic).
//   5. k_emit      : internal nodes whose range exceeds n_leaf are kept and
//                    relabelled by prefix sum; every smaller subtree
//                    collapses into one leaf of <= n_leaf triangles.  Child
//                    boxes are written as FP32 in the scene frame, rounded
//                    outward.
//   6. k_pack_tris : triangles gathered into leaf order (48 B FP32-exact or
//                    80 B FP64 records with the original id embedded).
#include <cstring>

#include <cub/cub.cuh>
#include <cstdlib>

#include "lbvh.h"

namespace sbr {

__device__ __forceinline__ uint64_t spread21(uint64_t x)
{
    x &= 0x1fffffULL;
    x = (x | x << 32) & 0x1f00000000ffffULL;
    x = (x | x << 16) & 0x1f0000ff0000ffULL;
    x = (x | x << 8) & 0x100f00f00f00f00fULL;
    x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
    x = (x | x << 2) & 0x1249249249249249ULL;
    return x;
}

__global__ void k_morton(const double *__restrict__ verts, int64_t n, double3 cmin,
                         double3 cinv, double *__restrict__ tri_box,
                         uint64_t *__restrict__ keys, int *__restrict__ vals)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double *v = verts + 9 * i;
    double lo[3], hi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = fmin(fmin(v[a], v[3 + a]), v[6 + a]);
        hi[a] = fmax(fmax(v[a], v[3 + a]), v[6 + a]);
        tri_box[6 * i + a] = lo[a];
        tri_box[6 * i + 3 + a] = hi[a];
    }
    const double scale = 2097151.0;  // 2^21 - 1
    double c[3] = {(lo[0] + hi[0]) * 0.5, (lo[1] + hi[1]) * 0.5, (lo[2] + hi[2]) * 0.5};
    double q[3] = {(c[0] - cmin.x) * cinv.x, (c[1] - cmin.y) * cinv.y, (c[2] - cmin.z) * cinv.z};
    uint64_t code = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double s = fmin(fmax(q[a] * scale, 0.0), scale);
        code |= spread21((uint64_t)s) << (2 - a);
    }
    keys[i] = code;
    vals[i] = (int)i;
}

__device__ __forceinline__ int delta(const uint64_t *k, int64_t n, int64_t i, int64_t j)
{
    if (j < 0 || j >= n) return -1;
    uint64_t a = k[i], b = k[j];
    if (a == b) return 64 + __clzll((long long)(i ^ j));
    return __clzll((long long)(a ^ b));
}

// child encoding in the radix tree: >= 0 internal node, < 0 -(leaf + 1)
__global__ void k_karras(const uint64_t *__restrict__ keys, int64_t n,
                         int2 *__restrict__ child, int2 *__restrict__ range,
                         int *__restrict__ parent)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    int d = (delta(keys, n, i, i + 1) - delta(keys, n, i, i - 1)) >= 0 ? 1 : -1;
    int dmin = delta(keys, n, i, i - d);
    int64_t lmax = 2;
    while (delta(keys, n, i, i + lmax * d) > dmin) lmax *= 2;
    int64_t l = 0;
    for (int64_t t = lmax / 2; t >= 1; t /= 2)
        if (delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
    int64_t j = i + l * d;
    int dnode = delta(keys, n, i, j);
    int64_t s = 0;
    int64_t len = l;
    // binary search for the split position
    int64_t t = (len + 1) / 2;
    while (true) {
        if (delta(keys, n, i, i + (s + t) * d) > dnode) s += t;
        if (t == 1) break;
        t = (t + 1) / 2;
    }
    int64_t gamma = i + s * d + (d < 0 ? -1 : 0);
    int64_t lo = i < j ? i : j, hi = i < j ? j : i;
    int left = (lo == gamma) ? -(int)(gamma + 1) : (int)gamma;
    int right = (hi == gamma + 1) ? -(int)(gamma + 2) : (int)(gamma + 1);
    child[i] = make_int2(left, right);
    range[i] = make_int2((int)lo, (int)hi);
    // parent array: internal nodes at [0, n-1), leaves at n-1 + leaf
    parent[left >= 0 ? left : (n - 1) + (-left - 1)] = (int)i;
    parent[right >= 0 ? right : (n - 1) + (-right - 1)] = (int)i;
}

__global__ void k_refit(const double *__restrict__ tri_box, const int *__restrict__ vals,
                        int64_t n, const int2 *__restrict__ child,
                        const int *__restrict__ parent, double *__restrict__ node_box,
                        int *__restrict__ arrive)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t node = parent[(n - 1) + i];
    while (true) {
        __threadfence();
        if (atomicAdd(&arrive[node], 1) == 0) return;  // sibling not done yet
        __threadfence();
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        int2 c = child[node];
        int cs[2] = {c.x, c.y};
        for (int q = 0; q < 2; ++q) {
            const double *b;
            if (cs[q] >= 0) b = node_box + 6 * (int64_t)cs[q];
            else b = tri_box + 6 * (int64_t)vals[-cs[q] - 1];
            for (int a = 0; a < 3; ++a) {
                double x = *((volatile const double *)(b + a));
                double y = *((volatile const double *)(b + 3 + a));
                lo[a] = fmin(lo[a], x);
                hi[a] = fmax(hi[a], y);
            }
        }
        for (int a = 0; a < 3; ++a) {
            node_box[6 * node + a] = lo[a];
            node_box[6 * node + 3 + a] = hi[a];
        }
        if (node == 0) return;
        node = parent[node];
    }
}

__global__ void k_keep(const int2 *__restrict__ range, int64_t n, int n_leaf,
                       int *__restrict__ keep)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    int2 r = range[i];
    keep[i] = (r.y - r.x + 1) > n_leaf ? 1 : 0;
}

__device__ __forceinline__ void rel_box(const double *b, double3 c, float out[6])
{
    out[0] = __double2float_rd(b[0] - c.x);
    out[1] = __double2float_rd(b[1] - c.y);
    out[2] = __double2float_rd(b[2] - c.z);
    out[3] = __double2float_ru(b[3] - c.x);
    out[4] = __double2float_ru(b[4] - c.y);
    out[5] = __double2float_ru(b[5] - c.z);
}

__global__ void k_emit(const int2 *__restrict__ child, const int2 *__restrict__ range,
                       const int *__restrict__ keep, const int *__restrict__ relabel,
                       const double *__restrict__ node_box,
                       const double *__restrict__ tri_box, const int *__restrict__ vals,
                       int64_t n, double3 c, Node *__restrict__ out)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n - 1 || !keep[i]) return;
    int2 ch = child[i];
    int cs[2] = {ch.x, ch.y};
    int refs[2];
    float bx[2][6];
    for (int q = 0; q < 2; ++q) {
        int cc = cs[q];
        if (cc >= 0) {
            rel_box(node_box + 6 * (int64_t)cc, c, bx[q]);
            if (keep[cc]) {
                refs[q] = relabel[cc];
            } else {
                int2 r = range[cc];
                refs[q] = leaf_ref(r.x, r.y - r.x + 1);
            }
        } else {
            int leaf = -cc - 1;
            rel_box(tri_box + 6 * (int64_t)vals[leaf], c, bx[q]);
            refs[q] = leaf_ref(leaf, 1);
        }
    }
    Node nd;
    nd.a = make_float4(bx[0][0], bx[0][1], bx[0][2], bx[0][3]);
    nd.b = make_float4(bx[0][4], bx[0][5], bx[1][0], bx[1][1]);
    nd.c = make_float4(bx[1][2], bx[1][3], bx[1][4], bx[1][5]);
    nd.d = make_int4(refs[0], refs[1], 0, 0);
    out[relabel[i]] = nd;
}

__global__ void k_depth(const int *__restrict__ keep, const int *__restrict__ parent,
                        int64_t n, int *__restrict__ max_depth)
{
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n - 1 || !keep[i]) return;
    int d = 0;
    int64_t node = i;
    while (node != 0) {
        node = parent[node];
        ++d;
    }
    atomicMax(max_depth, d);
}

__global__ void k_pack_tris(const double *__restrict__ verts, const int *__restrict__ order,
                            int64_t n, int storage, float4 *__restrict__ tri32,
                            double2 *__restrict__ tri64)
{
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    int id = order[k];
    const double *v = verts + 9 * (int64_t)id;
    if (storage == kF64) {
        double2 *p = tri64 + 5 * k;
        p[0] = make_double2(v[0], v[1]);
        p[1] = make_double2(v[2], v[3]);
        p[2] = make_double2(v[4], v[5]);
        p[3] = make_double2(v[6], v[7]);
        p[4] = make_double2(v[8], __longlong_as_double((long long)id));
    } else {
        float4 *p = tri32 + 3 * k;
        p[0] = make_float4((float)v[0], (float)v[1], (float)v[2], (float)v[3]);
        p[1] = make_float4((float)v[4], (float)v[5], (float)v[6], (float)v[7]);
        p[2] = make_float4((float)v[8], __int_as_float(id), 0.f, 0.f);
    }
}

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

#define CK(x)                                                     \
    do {                                                          \
        cudaError_t e_ = (x);                                     \
        if (e_ != cudaSuccess) return e_;                         \
    } while (0)

// ---------------------------------------------------------------------------
// mesh ingest: SoA -> (T,9) records + bounds / flags reductions
// ---------------------------------------------------------------------------
// order-preserving map double -> uint64 so atomicMin/Max work on doubles
__device__ __forceinline__ unsigned long long ord_of(double x)
{
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
static inline double unord(unsigned long long u)
{
    const unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffULL) : ~u;
    double x;
    memcpy(&x, &b, sizeof(x));
    return x;
}

// red[0..5] = min (lo xyz, centroid lo xyz), red[6..11] = max, red[12] =
// non-finite flag, red[13] = not-float32-representable flag
__global__ void k_ingest(const double *__restrict__ soa, int64_t n, double *__restrict__ verts,
                         unsigned long long *__restrict__ red)
{
    double mn[6], mx[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) { mn[q] = INFINITY; mx[q] = -INFINITY; }
    bool bad = false, not32 = false;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        double v[9];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double x = soa[c * 3 * n + 3 * t + a];
                v[3 * c + a] = x;
                bad |= !isfinite(x);
                not32 |= (double)(float)x != x;
            }
#pragma unroll
        for (int q = 0; q < 9; ++q) verts[9 * t + q] = v[q];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const double lo = fmin(fmin(v[a], v[3 + a]), v[6 + a]);
            const double hi = fmax(fmax(v[a], v[3 + a]), v[6 + a]);
            const double cc = (lo + hi) * 0.5;
            mn[a] = fmin(mn[a], lo); mx[a] = fmax(mx[a], hi);
            mn[3 + a] = fmin(mn[3 + a], cc); mx[3 + a] = fmax(mx[3 + a], cc);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            mn[q] = fmin(mn[q], __shfl_xor_sync(0xffffffffu, mn[q], o));
            mx[q] = fmax(mx[q], __shfl_xor_sync(0xffffffffu, mx[q], o));
        }
    }
    bad = __any_sync(0xffffffffu, bad);
    not32 = __any_sync(0xffffffffu, not32);
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            atomicMin(&red[q], ord_of(mn[q]));
            atomicMax(&red[6 + q], ord_of(mx[q]));
        }
        if (bad) atomicOr(&red[12], 1ULL);
        if (not32) atomicOr(&red[13], 1ULL);
    }
}

cudaError_t mesh_ingest(const double *d_soa, int64_t ntri, double *d_verts, MeshIngest &out,
                        cudaStream_t st, int64_t *launches)
{
    DevBuf<unsigned long long> red(14);
    CK(red.status());
    unsigned long long init[14];
    for (int q = 0; q < 6; ++q) { init[q] = ~0ULL; init[6 + q] = 0ULL; }
    init[12] = init[13] = 0ULL;
    CK(cudaMemcpyAsync(red.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    int64_t want = (ntri + 255) / 256;
    unsigned nb = (unsigned)(want < 4096 ? (want > 0 ? want : 1) : 4096);
    k_ingest<<<nb, 256, 0, st>>>(d_soa, ntri, d_verts, red.p);
    ++*launches;
    CK(cudaGetLastError());
    unsigned long long res[14];
    CK(cudaMemcpyAsync(res, red.p, sizeof(res), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int a = 0; a < 3; ++a) {
        out.lo[a] = unord(res[a]);
        out.clo[a] = unord(res[3 + a]);
        out.hi[a] = unord(res[6 + a]);
        out.chi[a] = unord(res[9 + a]);
    }
    out.finite = res[12] == 0ULL;
    out.all_f32 = res[13] == 0ULL;
    return cudaSuccess;
}

cudaError_t lbvh_build(const LbvhInput &in, LbvhOutput &out, Arena &ws, cudaStream_t st,
                       int64_t *launches)
{
    const int64_t n = in.ntri;
    const int T = 256;
    const int64_t ni = n > 1 ? n - 1 : 1;
    // one grow-only workspace for every temporary (no per-build cudaMalloc)
    size_t sort_bytes = 0, scan_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (uint64_t *)nullptr,
                                       (uint64_t *)nullptr, (int *)nullptr, (int *)nullptr,
                                       (int)n, 0, 63, st));
    CK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int *)nullptr, (int *)nullptr,
                                     (int)ni, st));
    const size_t need = 256 * 20 + 48 * n + 16 * n + 8 * n + sort_bytes + 16 * ni + 8 * n +
                        12 * ni + 48 * ni + 4 + scan_bytes;
    CK(ws.reserve(need));
    double *tri_box = ws.take<double>(6 * n);
    uint64_t *keys = ws.take<uint64_t>(n), *keys2 = ws.take<uint64_t>(n);
    int *vals = ws.take<int>(n), *order = ws.take<int>(n);
    unsigned char *sort_tmp = ws.take<unsigned char>(sort_bytes);

    double3 cmin = make_double3(in.cmin[0], in.cmin[1], in.cmin[2]);
    double ext[3] = {in.cmax[0] - in.cmin[0], in.cmax[1] - in.cmin[1], in.cmax[2] - in.cmin[2]};
    double3 cinv = make_double3(ext[0] > 0 ? 1.0 / ext[0] : 0.0, ext[1] > 0 ? 1.0 / ext[1] : 0.0,
                                ext[2] > 0 ? 1.0 / ext[2] : 0.0);
    k_morton<<<nblk(n, T), T, 0, st>>>(in.d_verts, n, cmin, cinv, tri_box, keys, vals);
    ++*launches;
    CK(cudaGetLastError());

    CK(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, keys, keys2, vals, order, (int)n,
                                       0, 63, st));
    ++*launches;

    out.n_leaf_slots = n;
    out.storage = in.storage;
    double3 c = make_double3(in.frame[0], in.frame[1], in.frame[2]);

    // triangles in leaf order
    if (in.storage == kF64) {
        CK(out.tri64.alloc(5 * n));
    } else {
        CK(out.tri32.alloc(3 * n));
    }
    k_pack_tris<<<nblk(n, T), T, 0, st>>>(in.d_verts, order, n, in.storage, out.tri32.p,
                                          out.tri64.p);
    ++*launches;
    CK(cudaGetLastError());
    CK(out.leaf_ids.alloc(n));
    CK(cudaMemcpyAsync(out.leaf_ids.p, order, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));

    if (n <= in.n_leaf) {
        // single leaf: node 0 carries the leaf in both child slots
        double lo[3], hi[3];
        for (int a = 0; a < 3; ++a) { lo[a] = in.aabb[a]; hi[a] = in.aabb[3 + a]; }
        Node nd;
        float b[6];
        for (int a = 0; a < 3; ++a) {
            b[a] = (float)(lo[a] - in.frame[a]);
            b[3 + a] = (float)(hi[a] - in.frame[a]);
            b[a] = nextafterf(b[a], -INFINITY);
            b[3 + a] = nextafterf(b[3 + a], INFINITY);
        }
        nd.a = make_float4(b[0], b[1], b[2], b[3]);
        nd.b = make_float4(b[4], b[5], b[0], b[1]);
        nd.c = make_float4(b[2], b[3], b[4], b[5]);
        int r = leaf_ref(0, (int)n);
        nd.d = make_int4(r, r, 0, 0);
        CK(out.nodes.alloc(1));
        CK(cudaMemcpyAsync(out.nodes.p, &nd, sizeof(Node), cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
        out.nnodes = 1;
        out.root = 0;
        out.max_depth = 0;
        return cudaSuccess;
    }

    int2 *child = ws.take<int2>(ni), *range = ws.take<int2>(ni);
    int *parent = ws.take<int>(2 * n - 1), *arrive = ws.take<int>(ni);
    int *keep = ws.take<int>(ni), *relabel = ws.take<int>(ni), *dmax = ws.take<int>(1);
    double *node_box = ws.take<double>(6 * ni);
    unsigned char *scan_tmp = ws.take<unsigned char>(scan_bytes);

    k_karras<<<nblk(ni, T), T, 0, st>>>(keys2, n, child, range, parent);
    ++*launches;
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(arrive, 0, sizeof(int) * ni, st));
    k_refit<<<nblk(n, T), T, 0, st>>>(tri_box, order, n, child, parent, node_box, arrive);
    ++*launches;
    CK(cudaGetLastError());
    k_keep<<<nblk(ni, T), T, 0, st>>>(range, n, in.n_leaf, keep);
    ++*launches;
    CK(cudaGetLastError());

    CK(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, keep, relabel, (int)ni, st));
    ++*launches;
    int last_keep = 0, last_rel = 0;
    CK(cudaMemcpyAsync(&last_keep, keep + ni - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&last_rel, relabel + ni - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int64_t nk = (int64_t)last_keep + last_rel;
    CK(out.nodes.alloc(nk));
    k_emit<<<nblk(ni, T), T, 0, st>>>(child, range, keep, relabel, node_box, tri_box, order, n,
                                      c, out.nodes.p);
    ++*launches;
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(dmax, 0, sizeof(int), st));
    k_depth<<<nblk(ni, T), T, 0, st>>>(keep, parent, n, dmax);
    ++*launches;
    CK(cudaGetLastError());
    int depth = 0;
    CK(cudaMemcpyAsync(&depth, dmax, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    out.nnodes = nk;
    out.root = 0;
    out.max_depth = depth;
    return cudaSuccess;
}

cudaError_t pack_tris(const double *d_verts, const int *d_order, int64_t n, int storage,
                      LbvhOutput &out, cudaStream_t st, int64_t *launches)
{
    if (storage == kF64) {
        CK(out.tri64.alloc(5 * n));
    } else {
        CK(out.tri32.alloc(3 * n));
    }
    k_pack_tris<<<nblk(n, 256), 256, 0, st>>>(d_verts, d_order, n, storage, out.tri32.p,
                                              out.tri64.p);
    ++*launches;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// BVH2 -> BVH4 collapse (level by level, deterministic)
// ---------------------------------------------------------------------------
template <int W> struct PlainNode;
template <> struct PlainNode<4> { using T = Node4; };
template <> struct PlainNode<8> { using T = Node8; };
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
__device__ __forceinline__ void child_box(const Node &n, int which, float b[6])
{
    if (which == 0) {
        b[0] = n.a.x; b[1] = n.a.y; b[2] = n.a.z; b[3] = n.a.w; b[4] = n.b.x; b[5] = n.b.y;
    } else {
        b[0] = n.b.z; b[1] = n.b.w; b[2] = n.c.x; b[3] = n.c.y; b[4] = n.c.z; b[5] = n.c.w;
    }
}

__device__ __forceinline__ float half_area(const float b[6])
{
    const float dx = b[3] - b[0], dy = b[4] - b[1], dz = b[5] - b[2];
    return dx * dy + dy * dz + dz * dx;
}

// pass A: open up to W descendants of each item (greedily the child with the
// largest surface area), count internal ones
template <int W>
__global__ void k_collapse_open(const Node *__restrict__ bvh2, const int *__restrict__ items,
                                int n_items, int *__restrict__ cref, float *__restrict__ cbox,
                                int *__restrict__ cnt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_items) return;
    const Node x = bvh2[items[i]];
    int ref[W];
    float box[W][6];
    ref[0] = x.d.x;
    ref[1] = x.d.y;
    child_box(x, 0, box[0]);
    child_box(x, 1, box[1]);
    int n = 2;
    while (n < W) {
        int pick = -1;
        float best = -1.f;
        for (int k = 0; k < n; ++k)
            if (ref[k] >= 0) {
                const float a = half_area(box[k]);
                if (a > best) { best = a; pick = k; }
            }
        if (pick < 0) break;
        const Node y = bvh2[ref[pick]];
        ref[pick] = y.d.x;
        child_box(y, 0, box[pick]);
        ref[n] = y.d.y;
        child_box(y, 1, box[n]);
        ++n;
    }
    int internal = 0;
    for (int k = 0; k < W; ++k) {
        const bool have = k < n;
        cref[W * i + k] = have ? ref[k] : kEmptyRef;
        for (int q = 0; q < 6; ++q) cbox[6 * W * i + 6 * k + q] = have ? box[k][q] : 0.f;
        internal += (have && ref[k] >= 0) ? 1 : 0;
    }
    cnt[i] = internal;
}

// pass B: write the wide nodes, allocate (by prefix offset) and enqueue the
// internal children as the next level
template <int W>
__global__ void k_collapse_emit(const int *__restrict__ cref, const float *__restrict__ cbox,
                                const int *__restrict__ off, const int *__restrict__ out_idx,
                                int n_items, int next_base,
                                typename PlainNode<W>::T *__restrict__ out,
                                int *__restrict__ next_items, int *__restrict__ next_out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_items) return;
    float pl[6][W];     // lox loy loz hix hiy hiz planes
    int r[W];
    int j = off[i];
    for (int k = 0; k < W; ++k) {
        int c = cref[W * i + k];
        for (int q = 0; q < 6; ++q) pl[q][k] = cbox[6 * W * i + 6 * k + q];
        if (c >= 0 && c != kEmptyRef) {
            next_items[j] = c;
            next_out[j] = next_base + j;
            c = next_base + j;
            ++j;
        }
        r[k] = c;
    }
    // SoA planes: W/4 float4 per plane, then W/4 int4 refs, then padding
    typename PlainNode<W>::T nd;
    float4 *f = reinterpret_cast<float4 *>(&nd);
    for (int q = 0; q < 6; ++q)
        for (int h = 0; h < W / 4; ++h)
            f[q * (W / 4) + h] = make_float4(pl[q][4 * h], pl[q][4 * h + 1], pl[q][4 * h + 2],
                                             pl[q][4 * h + 3]);
    int4 *ri = reinterpret_cast<int4 *>(f + 6 * (W / 4));
    for (int h = 0; h < W / 4; ++h) {
        ri[h] = make_int4(r[4 * h], r[4 * h + 1], r[4 * h + 2], r[4 * h + 3]);
        ri[W / 4 + h] = make_int4(0, 0, 0, 0);
    }
    out[out_idx[i]] = nd;
}

template <int W>
static cudaError_t collapse_wide(LbvhOutput &out, typename PlainNode<W>::T **dst, int64_t &nn,
                                 int &depth, Arena &ws, cudaStream_t st, int64_t *launches)
{
    const int n2 = (int)out.nnodes;
    size_t scan_bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int *)nullptr, (int *)nullptr, n2,
                                     st));
    CK(ws.reserve(256 * 12 + (size_t)n2 * (4 * 4 + W * 4 + 6 * W * 4 + 4 * 2) + scan_bytes + 64));
    int *items[2] = {ws.take<int>(n2), ws.take<int>(n2)};
    int *outs[2] = {ws.take<int>(n2), ws.take<int>(n2)};
    int *cref = ws.take<int>((size_t)W * n2);
    float *cbox = ws.take<float>((size_t)6 * W * n2);
    int *cnt = ws.take<int>(n2), *off = ws.take<int>(n2);
    unsigned char *scan_tmp = ws.take<unsigned char>(scan_bytes);
    const int zero = 0;
    CK(cudaMemcpyAsync(items[0], &out.root, sizeof(int), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(outs[0], &zero, sizeof(int), cudaMemcpyHostToDevice, st));
    int n_items = 1, next_base = 1, level = 0, cur = 0;
    while (n_items > 0) {
        const unsigned nb = (unsigned)((n_items + 127) / 128);
        k_collapse_open<W><<<nb, 128, 0, st>>>(out.nodes.p, items[cur], n_items, cref, cbox, cnt);
        ++*launches;
        CK(cudaGetLastError());
        CK(cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, cnt, off, n_items, st));
        ++*launches;
        k_collapse_emit<W><<<nb, 128, 0, st>>>(cref, cbox, off, outs[cur], n_items, next_base,
                                               *dst, items[cur ^ 1], outs[cur ^ 1]);
        ++*launches;
        CK(cudaGetLastError());
        int last_off = 0, last_cnt = 0;
        CK(cudaMemcpyAsync(&last_off, off + n_items - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&last_cnt, cnt + n_items - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const int total = last_off + last_cnt;
        next_base += total;
        n_items = total;
        cur ^= 1;
        ++level;
    }
    nn = next_base;
    depth = level - 1;
    return cudaSuccess;
}

// Node4 / Node8 -> quantised node: per axis the origin p = min child lo (a
// float) and the smallest power-of-two step 2^e with 255 * 2^e >= max child
// hi - p; child planes are rounded outward (floor / ceil, exact in FP64).
template <int W> struct QNode;
template <> struct QNode<4> { using T = Node4Q; };
template <> struct QNode<8> { using T = Node8Q; };

template <int W>
__global__ void k_quantize(const typename PlainNode<W>::T *__restrict__ in, int64_t n,
                           typename QNode<W>::T *__restrict__ out)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    // plain layout: 6 planes of W floats, then W refs
    const float *pl = reinterpret_cast<const float *>(in + i);
    const int *rf = reinterpret_cast<const int *>(pl + 6 * W);
    typename QNode<W>::T Q;
    float p[3];
    unsigned int exps = 0;
    unsigned int qw[6][W / 4];
    for (int a = 0; a < 3; ++a) {
        float mn = INFINITY, mx = -INFINITY;
        for (int k = 0; k < W; ++k)
            if (rf[k] != kEmptyRef) { mn = fminf(mn, pl[a * W + k]); mx = fmaxf(mx, pl[(3 + a) * W + k]); }
        if (!(mn <= mx)) { mn = 0.f; mx = 0.f; }
        p[a] = mn;
        const double ext = (double)mx - (double)mn;    // exact
        int e = -100;
        while ((double)255 * ldexp(1.0, e) < ext) ++e;
        exps |= (unsigned int)(e + 127) << (8 * a);
        for (int h = 0; h < W / 4; ++h) { qw[a][h] = 0u; qw[3 + a][h] = 0u; }
        for (int k = 0; k < W; ++k) {
            unsigned int ql = 0u, qh = 0u;
            if (rf[k] != kEmptyRef) {
                ql = (unsigned int)floor(ldexp((double)pl[a * W + k] - (double)mn, -e));
                qh = (unsigned int)ceil(ldexp((double)pl[(3 + a) * W + k] - (double)mn, -e));
                qh = qh > 255u ? 255u : qh;
            }
            qw[a][k >> 2] |= ql << (8 * (k & 3));
            qw[3 + a][k >> 2] |= qh << (8 * (k & 3));
        }
    }
    Q.px = p[0]; Q.py = p[1]; Q.pz = p[2];
    Q.exps = exps;
    int *qr = reinterpret_cast<int *>(&Q.ref);
    for (int k = 0; k < W; ++k) qr[k] = rf[k];
    for (int j = 0; j < 6; ++j)
        for (int h = 0; h < W / 4; ++h) Q.q[j * (W / 4) + h] = qw[j][h];
    if (W == 4) reinterpret_cast<unsigned int *>(&Q)[14] = reinterpret_cast<unsigned int *>(&Q)[15] = 0u;
    out[i] = Q;
}

// the traversal tree width: 4 unless SBR_WIDTH=8
int traversal_width()
{
    const char *s = getenv("SBR_WIDTH");
    return (s && atoi(s) == 8) ? 8 : 4;
}

cudaError_t collapse_bvh4(LbvhOutput &out, Arena &ws, cudaStream_t st, int64_t *launches)
{
    const int n2 = (int)out.nnodes;
    CK(out.nodes4.alloc(n2));
    Node4 *p4 = out.nodes4.p;
    CK(collapse_wide<4>(out, &p4, out.nnodes4, out.depth4, ws, st, launches));
#ifdef SBR_NODE_Q
    // quantised boxes (-DSBR_NODE_Q): measured neutral at width 4, 9% faster
    // than the 256 B nodes at width 8 (profiles/experiments)
    CK(out.nodes4q.alloc((size_t)out.nnodes4));
    k_quantize<4><<<(unsigned)((out.nnodes4 + 127) / 128), 128, 0, st>>>(p4, out.nnodes4,
                                                                      out.nodes4q.p);
    ++*launches;
    CK(cudaGetLastError());
#endif
    out.width = traversal_width();
    if (out.width == 8) {
        CK(out.nodes8.alloc(n2));
        Node8 *p8 = out.nodes8.p;
        int d8 = 0;
        CK(collapse_wide<8>(out, &p8, out.nnodes8, d8, ws, st, launches));
#ifdef SBR_NODE_Q
        CK(out.nodes8q.alloc((size_t)out.nnodes8));
        k_quantize<8><<<(unsigned)((out.nnodes8 + 127) / 128), 128, 0, st>>>(p8, out.nnodes8,
                                                                          out.nodes8q.p);
        ++*launches;
        CK(cudaGetLastError());
#endif
        out.depth8 = d8;
    }
    return cudaSuccess;
}

}  // namespace sbr
