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
#include <cub/cub.cuh>

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

cudaError_t lbvh_build(const LbvhInput &in, LbvhOutput &out, cudaStream_t st,
                       int64_t *launches)
{
    const int64_t n = in.ntri;
    const int T = 256;
    DevBuf<double> tri_box(6 * n);
    DevBuf<uint64_t> keys(n), keys2(n);
    DevBuf<int> vals(n), order(n);
    CK(tri_box.status()); CK(keys.status()); CK(keys2.status());
    CK(vals.status()); CK(order.status());

    double3 cmin = make_double3(in.cmin[0], in.cmin[1], in.cmin[2]);
    double ext[3] = {in.cmax[0] - in.cmin[0], in.cmax[1] - in.cmin[1], in.cmax[2] - in.cmin[2]};
    double3 cinv = make_double3(ext[0] > 0 ? 1.0 / ext[0] : 0.0, ext[1] > 0 ? 1.0 / ext[1] : 0.0,
                                ext[2] > 0 ? 1.0 / ext[2] : 0.0);
    k_morton<<<nblk(n, T), T, 0, st>>>(in.d_verts, n, cmin, cinv, tri_box.p, keys.p, vals.p);
    ++*launches;
    CK(cudaGetLastError());

    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, keys2.p, vals.p, order.p,
                                       (int)n, 0, 63, st));
    DevBuf<unsigned char> tmp(tmp_bytes);
    CK(tmp.status());
    CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, keys2.p, vals.p, order.p,
                                       (int)n, 0, 63, st));
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
    k_pack_tris<<<nblk(n, T), T, 0, st>>>(in.d_verts, order.p, n, in.storage, out.tri32.p,
                                          out.tri64.p);
    ++*launches;
    CK(cudaGetLastError());
    CK(out.leaf_ids.alloc(n));
    CK(cudaMemcpyAsync(out.leaf_ids.p, order.p, sizeof(int) * n, cudaMemcpyDeviceToDevice, st));

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

    const int64_t ni = n - 1;
    DevBuf<int2> child(ni), range(ni);
    DevBuf<int> parent(2 * n - 1), arrive(ni), keep(ni), relabel(ni), dmax(1);
    DevBuf<double> node_box(6 * ni);
    CK(child.status()); CK(range.status()); CK(parent.status()); CK(arrive.status());
    CK(keep.status()); CK(relabel.status()); CK(node_box.status()); CK(dmax.status());

    k_karras<<<nblk(ni, T), T, 0, st>>>(keys2.p, n, child.p, range.p, parent.p);
    ++*launches;
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(arrive.p, 0, sizeof(int) * ni, st));
    k_refit<<<nblk(n, T), T, 0, st>>>(tri_box.p, order.p, n, child.p, parent.p, node_box.p,
                                      arrive.p);
    ++*launches;
    CK(cudaGetLastError());
    k_keep<<<nblk(ni, T), T, 0, st>>>(range.p, n, in.n_leaf, keep.p);
    ++*launches;
    CK(cudaGetLastError());

    size_t scan_bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, keep.p, relabel.p, (int)ni, st));
    DevBuf<unsigned char> scan_tmp(scan_bytes);
    CK(scan_tmp.status());
    CK(cub::DeviceScan::ExclusiveSum(scan_tmp.p, scan_bytes, keep.p, relabel.p, (int)ni, st));
    ++*launches;
    int last_keep = 0, last_rel = 0;
    CK(cudaMemcpyAsync(&last_keep, keep.p + ni - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&last_rel, relabel.p + ni - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int64_t nk = (int64_t)last_keep + last_rel;
    CK(out.nodes.alloc(nk));
    k_emit<<<nblk(ni, T), T, 0, st>>>(child.p, range.p, keep.p, relabel.p, node_box.p,
                                      tri_box.p, order.p, n, c, out.nodes.p);
    ++*launches;
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(dmax.p, 0, sizeof(int), st));
    k_depth<<<nblk(ni, T), T, 0, st>>>(keep.p, parent.p, n, dmax.p);
    ++*launches;
    CK(cudaGetLastError());
    int depth = 0;
    CK(cudaMemcpyAsync(&depth, dmax.p, sizeof(int), cudaMemcpyDeviceToHost, st));
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

}  // namespace sbr
