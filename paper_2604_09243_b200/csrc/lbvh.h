// lbvh.h -- host-side declarations shared by the library translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sbr_device.cuh"

namespace sbr {

// Owning device buffer (RAII, move-only).
template <class T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaError_t err = cudaSuccess;

    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : p(o.p), n(o.n), err(o.err) { o.p = nullptr; o.n = 0; }
    DevBuf &operator=(DevBuf &&o) noexcept
    {
        if (this != &o) {
            release();
            p = o.p; n = o.n; err = o.err;
            o.p = nullptr; o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }

    cudaError_t alloc(size_t count)
    {
        release();
        err = cudaSuccess;
        if (count) {
            err = cudaMalloc((void **)&p, sizeof(T) * count);
            if (err != cudaSuccess) p = nullptr;
        }
        n = p ? count : 0;
        return err;
    }
    // grow-only reuse for scratch
    cudaError_t reserve(size_t count)
    {
        if (count <= n && p) return cudaSuccess;
        return alloc(count);
    }
    cudaError_t status() const { return err; }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
};

struct LbvhInput {
    const double *d_verts;   // (T, 9): v0 xyz, v1 xyz, v2 xyz (original order)
    int64_t ntri;
    int storage;             // kF32Exact / kF64 / kSingle
    int n_leaf;
    double cmin[3], cmax[3]; // centroid bounds
    double aabb[6];          // mesh AABB
    double frame[3];         // box frame origin (scene centre)
};

struct LbvhOutput {
    DevBuf<Node> nodes;
    DevBuf<float4> tri32;
    DevBuf<double2> tri64;
    DevBuf<int> leaf_ids;    // leaf slot -> original triangle id
    int64_t nnodes = 0;
    int64_t n_leaf_slots = 0;
    int root = 0;
    int max_depth = 0;
    int storage = 0;
};

cudaError_t lbvh_build(const LbvhInput &in, LbvhOutput &out, cudaStream_t st,
                       int64_t *launches);
cudaError_t pack_tris(const double *d_verts, const int *d_order, int64_t n, int storage,
                      LbvhOutput &out, cudaStream_t st, int64_t *launches);

}  // namespace sbr
