// lbvh.h -- host-side declarations shared by the library translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "sbr_device.cuh"

namespace sbr {

// Device allocations go through the device's stream-ordered memory pool on
// the library stream of that device's context (registered by sbr_ctx_create,
// release threshold = keep everything): allocating and freeing meshes, trees
// and scratch never synchronises the device or returns pages to the driver
// (plain cudaMalloc/cudaFree cost 10-300 ms spikes per sweep on 1M-triangle
// scenes).  Without a context on the device, plain cudaMalloc/cudaFree.
cudaStream_t alloc_stream(int device);   // capi.cu; nullptr if no context

void count_alloc(int64_t bytes);        // capi.cu: live-allocation counters
inline cudaError_t dev_alloc(void **p, size_t bytes, int &device)
{
    cudaGetDevice(&device);
    cudaStream_t s = alloc_stream(device);
    const cudaError_t e = s ? cudaMallocAsync(p, bytes, s) : cudaMalloc(p, bytes);
    if (e == cudaSuccess) count_alloc((int64_t)bytes);
    return e;
}
inline void dev_free(void *p, int device, size_t bytes)
{
    cudaStream_t s = alloc_stream(device);
    if (s) cudaFreeAsync(p, s);
    else cudaFree(p);
    count_alloc(-(int64_t)bytes);
}

// Owning device buffer (RAII, move-only).
template <class T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaError_t err = cudaSuccess;
    int device = 0;

    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : p(o.p), n(o.n), err(o.err), device(o.device)
    {
        o.p = nullptr; o.n = 0;
    }
    DevBuf &operator=(DevBuf &&o) noexcept
    {
        if (this != &o) {
            release();
            p = o.p; n = o.n; err = o.err; device = o.device;
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
            err = dev_alloc((void **)&p, sizeof(T) * count, device);
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
        if (p) dev_free(p, device, n * sizeof(T));
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
};

// Grow-only device workspace carved into 256-byte aligned sub-buffers.
struct Arena {
    DevBuf<unsigned char> buf;
    size_t off = 0;
    cudaError_t reserve(size_t bytes)
    {
        off = 0;
        return buf.reserve(bytes);
    }
    template <class T>
    T *take(size_t count)
    {
        const size_t at = (off + 255) & ~(size_t)255;
        off = at + count * sizeof(T);
        return reinterpret_cast<T *>(buf.p + at);
    }
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
    // 4-wide traversal tree collapsed from `nodes` (level order, root 0)
    DevBuf<Node4> nodes4;
    DevBuf<Node4Q> nodes4q;  // nodes4 with quantised boxes (same indices)
    int64_t nnodes4 = 0;
    int depth4 = 0;
    // optional 8-wide traversal tree (SBR_WIDTH=8)
    DevBuf<Node8> nodes8;
    DevBuf<Node8Q> nodes8q;
    int64_t nnodes8 = 0;
    int depth8 = 0;
    int width = 4;
};

// Collapse the binary tree in out.nodes into out.nodes4: every BVH4 node
// adopts up to four descendants, greedily opening the child with the
// largest box surface area; deterministic (prefix-sum allocation).
cudaError_t collapse_bvh4(LbvhOutput &out, Arena &ws, cudaStream_t st, int64_t *launches);

// Device-side mesh ingest: soa = [v0 (T,3) | v1 (T,3) | v2 (T,3)] -> verts
// (T,9) plus the reductions the builder needs; synchronises the stream.
struct MeshIngest {
    double lo[3], hi[3], clo[3], chi[3];
    bool finite, all_f32;
};
cudaError_t mesh_ingest(const double *d_soa, int64_t ntri, double *d_verts, MeshIngest &out,
                        cudaStream_t st, int64_t *launches);

cudaError_t lbvh_build(const LbvhInput &in, LbvhOutput &out, Arena &ws, cudaStream_t st,
                       int64_t *launches);
cudaError_t pack_tris(const double *d_verts, const int *d_order, int64_t n, int storage,
                      LbvhOutput &out, cudaStream_t st, int64_t *launches);

}  // namespace sbr
