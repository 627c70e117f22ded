// sahbuild.h -- GPU construction of the reference binned-SAH tree.
#pragma once

#include "lbvh.h"

namespace sbr {

constexpr int kSahMaxBins = 64;

struct SahParams {          // bvh.py:22-49 BuildParams
    int n_leaf;
    int max_depth;
    int bins;               // bins_per_axis, 2..kSahMaxBins
    double c_t, c_i;
    int median = 0;         // 1: the reference median split (bvh.py:135-151) instead of SAH
};

// The tree in the reference's preorder layout (bvh.py:58-88), on device:
// nodes (nnodes,3) boxes, node_first/node_count, tri_order.
struct SahTree {
    DevBuf<double> nmin, nmax;
    DevBuf<int32_t> first, count, order;
    int64_t nnodes = 0;
    int max_depth = 0;
};

// per active segment (node under construction) of one level
struct SegAcc {                      // per active segment (node)
    unsigned long long box[6];       // lo xyz (min), hi xyz (max), ordered
    unsigned long long cb[6];        // centroid lo xyz, hi xyz
};

struct SegSplit {
    int split;          // 1: internal (children at the next level)
    int axis, boundary;
    double c_lo, scale;
    int64_t nl;
};

// grow-only scratch of the builder (kept by the context across builds)
struct SahWork {
    DevBuf<double> tb, node_box;
    DevBuf<int> idx, idx2, eseg, eseg2, flag, rank, left, right, snode, nsnode, crank, sflag, big;
    DevBuf<int64_t> lf, lc, size, pre, sb, sc, nsb, nsc;
    DevBuf<unsigned int> cnt;
    DevBuf<unsigned long long> bbox;
    DevBuf<SegAcc> acc;
    DevBuf<SegSplit> sp;
    DevBuf<unsigned char> scan_tmp;
    // median split: per-element keys / values and split-segment offsets
    DevBuf<double> key, key2;
    DevBuf<int64_t> sbeg, send;
    DevBuf<unsigned char> sort_tmp;
};

// d_verts: (T,9) FP64 vertices in original triangle order.  Leaves the tree
// on the stream (not synchronised).
cudaError_t sah_build(const double *d_verts, int64_t n, const SahParams &P, SahTree &out,
                      SahWork &w, cudaStream_t st, int64_t *launches);

// Child-pair traversal nodes from the reference layout on the device.
// host_needed: a leaf holds > kMaxLeafCount triangles or the root is a leaf
// (use the host converter instead).
cudaError_t ref_to_bvh2(const SahTree &t, const double frame[3], SahWork &w, LbvhOutput &out,
                        bool &host_needed, cudaStream_t st, int64_t *launches);

}  // namespace sbr
