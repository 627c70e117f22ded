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
};

// The tree in the reference's preorder layout (bvh.py:58-88), on device:
// nodes (nnodes,3) boxes, node_first/node_count, tri_order.
struct SahTree {
    DevBuf<double> nmin, nmax;
    DevBuf<int32_t> first, count, order;
    int64_t nnodes = 0;
    int max_depth = 0;
};

// d_verts: (T,9) FP64 vertices in original triangle order.
cudaError_t sah_build(const double *d_verts, int64_t n, const SahParams &P, SahTree &out,
                      cudaStream_t st, int64_t *launches);

}  // namespace sbr
