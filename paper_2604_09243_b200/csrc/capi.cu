// capi.cu -- the extern "C" boundary (include/sbr200.h): handles, argument
// validation, host<->device staging and the batched solve orchestration.
#include <chrono>
#include <condition_variable>
#include <dlfcn.h>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <algorithm>
#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sbr200.h"
#include "lbvh.h"
#include "pipeline.h"
#include "sahbuild.h"
#include <nccl.h>   // types and enums only: libnccl is dlopen-ed (comm section)

using namespace sbr;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

static int vfail(int code, const char *fmt, va_list ap)
{
    char buf[1024];
    vsnprintf(buf, sizeof(buf), fmt, ap);
    g_err = buf;
    return code;
}

static int fail(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    const int rc = vfail(code, fmt, ap);
    va_end(ap);
    return rc;
}

// shared with the other translation units (objio.cpp)
int sbr_fail(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    const int rc = vfail(code, fmt, ap);
    va_end(ap);
    return rc;
}

#define CUDA_TRY(x)                                                                     \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess)                                                          \
            return fail(e_ == cudaErrorMemoryAllocation ? SBR_ENOMEM : SBR_ECUDA,       \
                        "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__,  \
                        __LINE__);                                                      \
    } while (0)

#define REQUIRE(cond, ...)                       \
    do {                                         \
        if (!(cond)) return fail(SBR_EINVAL, __VA_ARGS__); \
    } while (0)

extern "C" const char *sbr_last_error(void) { return g_err.c_str(); }
extern "C" int sbr_abi_version(void) { return SBR200_ABI_VERSION; }

// ---------------------------------------------------------------------------
// handles
// ---------------------------------------------------------------------------
// Persistent host copy workers for upload_host: spawning threads per chunk
// cost ~0.3 ms a chunk, more than the 16 MB copy itself.
struct CopyPool {
    std::vector<std::thread> th;
    std::mutex m;
    std::condition_variable go, done;
    uint64_t gen = 0;
    int pending = 0;
    bool stop = false;
    unsigned char *dst = nullptr;
    const unsigned char *src = nullptr;
    size_t n = 0, part = 0;

    int workers() const { return (int)th.size() + 1; }
    void start(int nth)
    {
        for (int t = 1; t < nth; ++t)
            th.emplace_back([this, t] {
                uint64_t seen = 0;
                for (;;) {
                    size_t a, z;
                    unsigned char *d;
                    const unsigned char *s;
                    {
                        std::unique_lock<std::mutex> lk(m);
                        go.wait(lk, [&] { return stop || gen != seen; });
                        if (stop) return;
                        seen = gen;
                        a = std::min(n, t * part), z = std::min(n, a + part);
                        d = dst, s = src;
                    }
                    if (z > a) memcpy(d + a, s + a, z - a);
                    std::lock_guard<std::mutex> lk(m);
                    if (--pending == 0) done.notify_one();
                }
            });
    }
    // memcpy(d, s, bytes) split over the workers and the calling thread
    void copy(unsigned char *d, const unsigned char *s, size_t bytes)
    {
        const int w = workers();
        const size_t p = (bytes + w - 1) / w;
        if (w > 1) {
            std::lock_guard<std::mutex> lk(m);
            dst = d, src = s, n = bytes, part = p, pending = w - 1, ++gen;
            go.notify_all();
        }
        memcpy(d, s, std::min(bytes, p));
        if (w > 1) {
            std::unique_lock<std::mutex> lk(m);
            done.wait(lk, [&] { return pending == 0; });
        }
    }
    ~CopyPool()
    {
        {
            std::lock_guard<std::mutex> lk(m);
            stop = true;
        }
        go.notify_all();
        for (auto &t : th) t.join();
    }
};

struct sbr_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 148;
    int64_t launches = 0;
    std::mutex mu;
    int traversal = SBR_TRAVERSAL_FAST;   // sbr_ctx_set_traversal
    void *comm = nullptr;                 // ncclComm_t (sbr_comm_init)
    int comm_rank = 0, comm_size = 0;
    DevBuf<unsigned long long> counter;
    DevBuf<unsigned int> err_flag;
    DevBuf<unsigned long long> bad;
    // solve scratch (grow-only)
    DevBuf<SlotRec> slots;
    DevBuf<UnitDev> units;
    DevBuf<GridDev> grids;
    DevBuf<double2> chunk_part;
    DevBuf<double2> seg_part;
    DevBuf<int64_t> diag;
    DevBuf<int64_t> seg_base;
    DevBuf<int64_t> seg_slot;    // raster pass: global segment row -> slot offset
    DevBuf<int> bgrids;          // raster pass: grids of the current batch
    // raster pass: (slot, unit) of every slot whose query 0 hit; the trace
    // kernel overwrites entry w with that ray's SlotRec (k_po reads them)
    DevBuf<uint4> worklist;
    DevBuf<uint2> chunk_hits;               // raster pass: per chunk (list start, count)
    // slots [0, clean_slots) hold all-ones (the raster pass's "no hit"): list
    // mode PO restores that after every batch, so only growth needs a memset
    int64_t clean_slots = 0;
    DevBuf<unsigned long long> nwork;
    DevBuf<unsigned int> hitmap;            // raster pass: 1 bit per slot, first hit
    DevBuf<int> chunk_unit;                 // batch chunk -> unit index
    DevBuf<int4> big;                       // raster pass: big-triangle chunk queue
    DevBuf<unsigned long long> nbig;
    DevBuf<unsigned char> setups;           // raster pass: set-ups of queued triangles
    DevBuf<unsigned long long> nsetup;
    DevBuf<double> k2, gpow, scale;
    double dkturn = 0.0;         // uniform wavenumber step in turns (0: not uniform)
    DevBuf<double2> amp;
    DevBuf<double> stage;        // host->device staging (mesh ingest, records)
    // pinned double buffer for large host->device uploads (upload_host)
    unsigned char *pin[2] = {nullptr, nullptr};
    cudaEvent_t pin_ev[2] = {nullptr, nullptr};
    CopyPool copiers;            // host threads filling the pinned buffers
    Arena ws;                    // LBVH build workspace
    SahWork sah;                 // SAH build workspace
    // optional per-kernel CUDA-event timing of the solve pipeline
    bool profile = false;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    double trace_ms = 0.0, po_ms = 0.0, raster_ms = 0.0, compact_ms = 0.0;
    int64_t trace_n = 0, po_n = 0;
    LaunchStats stats() { return LaunchStats{&launches, num_sms}; }
    ~sbr_ctx()
    {
        for (auto &e : ev)
            if (e) cudaEventDestroy(e);
        for (int b = 0; b < 2; ++b) {
            if (pin[b]) cudaFreeHost(pin[b]);
            if (pin_ev[b]) cudaEventDestroy(pin_ev[b]);
        }
    }
};

struct sbr_mesh {
    sbr_ctx *ctx = nullptr;
    int64_t ntri = 0;
    int storage = kF64;
    double aabb[6];
    double cmin[3], cmax[3];
    DevBuf<double> verts;    // (T,9) original order
    DevBuf<double> normals;  // (T,3)
};

struct sbr_bvh {
    sbr_ctx *ctx = nullptr;
    const sbr_mesh *mesh = nullptr;
    LbvhOutput out;
    // reference-layout tree when this BVH IS a reference tree (GPU SAH build
    // or upload): exported verbatim; ref_depth < 0 otherwise
    // (host copies filled lazily from ref_dev on export)
    SahTree ref_dev;
    std::vector<double> ref_nmin, ref_nmax;
    std::vector<int32_t> ref_first, ref_count, ref_order;
    int ref_depth = -1;
    int ref_round_f32 = 0;     // GPU-built tree of a float32 mesh: replica rounds boxes
    int ref_tree_depth = -1;   // depth of ref_dev (reference-order traversal stack bound)
    // BVH4 deeper than the fast kernels' stack (kMaxDepth4): every traversal
    // of this tree replays the reference order on the reference tree instead
    // (reforder.cu, stack bound 255; the reference itself allows max_depth + 2)
    bool deep = false;
    double frame[3];
    float scale = 0.f;
    BvhView view() const
    {
        BvhView v;
        v.nodes = out.nodes.p;
        v.nodes4 = out.nodes4.p;
        v.nodes4q = out.nodes4q.p;
        v.nodes8 = out.nodes8.p;
        v.nodes8q = out.nodes8q.p;
        v.width = out.width;
        v.tri32 = out.tri32.p;
        v.tri64 = out.tri64.p;
        v.normals = mesh->normals.p;
        v.cx = frame[0]; v.cy = frame[1]; v.cz = frame[2];
        v.scale = scale;
        v.root = out.root;
        return v;
    }
};

static int set_device(sbr_ctx *ctx)
{
    CUDA_TRY(cudaSetDevice(ctx->device));
    return SBR_OK;
}

// the 4-wide traversal pushes <= 3 entries per level: bound the depth by the
// per-thread stack (kStack); deletes the handle on failure
static int check_depth(sbr_bvh *b)
{
    if (b->out.width == 8 && 7 * b->out.depth8 + 1 >= kStack) b->out.width = 4;  // stack bound
    if (b->out.depth4 <= kMaxDepth4) return SBR_OK;
    const int d = b->out.depth4;
    delete b;
    return fail(SBR_EINVAL, "BVH4 depth %d exceeds the traversal stack limit (%d)", d,
                kMaxDepth4);
}

// library stream per device for the stream-ordered allocator (lbvh.h)
static std::mutex g_alloc_mu;
static cudaStream_t g_alloc_stream[128];

cudaStream_t sbr::alloc_stream(int device)
{
    if (device < 0 || device >= 128) return nullptr;
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    return g_alloc_stream[device];
}

extern "C" int sbr_ctx_create(int device, sbr_ctx **out)
{
    REQUIRE(out, "out is NULL");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    REQUIRE(device >= 0 && device < ndev, "device %d out of range (have %d)", device, ndev);
    sbr_ctx *ctx = new sbr_ctx();
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) {
        cudaMemPool_t pool;
        e = cudaDeviceGetDefaultMemPool(&pool, device);
        uint64_t keep = UINT64_MAX;
        if (e == cudaSuccess) e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        if (e == cudaSuccess && device < 128) {
            std::lock_guard<std::mutex> lk(g_alloc_mu);
            if (!g_alloc_stream[device]) g_alloc_stream[device] = ctx->stream;
        }
    }
    // [0] trace, [1] raster work, [2..4] raster counters, [8..] stats builds
    if (e == cudaSuccess) e = ctx->counter.alloc(32);
    if (e == cudaSuccess) e = cudaMemsetAsync(ctx->counter.p, 0, 32 * sizeof(unsigned long long),
                                              ctx->stream);
    if (e == cudaSuccess) e = ctx->err_flag.alloc(1);
    if (e == cudaSuccess) e = ctx->bad.alloc(1);
    if (e != cudaSuccess) {
        delete ctx;
        return fail(SBR_ECUDA, "context creation failed: %s", cudaGetErrorString(e));
    }
    *out = ctx;
    return SBR_OK;
}

extern "C" int sbr_ctx_destroy(sbr_ctx *ctx)
{
    if (!ctx) return SBR_OK;
    sbr_comm_destroy(ctx);
    const int dev = ctx->device;
    cudaStream_t s = ctx->stream;
    cudaSetDevice(dev);
    if (s) cudaStreamSynchronize(s);
    delete ctx;               // its buffers are freed (stream-ordered) first
    if (s) {
        cudaStreamSynchronize(s);
        {
            std::lock_guard<std::mutex> lk(g_alloc_mu);
            if (dev < 128 && g_alloc_stream[dev] == s) g_alloc_stream[dev] = nullptr;
        }
        cudaStreamDestroy(s);
    }
    return SBR_OK;
}

extern "C" int sbr_ctx_synchronize(sbr_ctx *ctx)
{
    REQUIRE(ctx, "ctx is NULL");
    if (int rc = set_device(ctx)) return rc;
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return SBR_OK;
}

extern "C" int sbr_ctx_trim(sbr_ctx *ctx)
{
    REQUIRE(ctx, "ctx is NULL");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    ctx->slots.release(); ctx->units.release(); ctx->grids.release();
    ctx->clean_slots = 0;
    ctx->chunk_hits.release();
    ctx->chunk_part.release(); ctx->seg_part.release(); ctx->diag.release();
    ctx->seg_base.release(); ctx->seg_slot.release(); ctx->bgrids.release();
    ctx->worklist.release(); ctx->big.release(); ctx->setups.release(); ctx->hitmap.release();
    ctx->chunk_unit.release();
    ctx->amp.release(); ctx->stage.release();
    ctx->ws.buf.release();
    ctx->ws.off = 0;
    ctx->sah = SahWork();
    for (int b = 0; b < 2; ++b) {
        if (ctx->pin[b]) cudaFreeHost(ctx->pin[b]);
        if (ctx->pin_ev[b]) cudaEventDestroy(ctx->pin_ev[b]);
        ctx->pin[b] = nullptr;
        ctx->pin_ev[b] = nullptr;
    }
    // hand the freed blocks back to the device (release threshold is "keep")
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess)
        cudaMemPoolTrimTo(pool, 0);
    return SBR_OK;
}

extern "C" int sbr_ctx_stream(sbr_ctx *ctx, void **stream_out)
{
    REQUIRE(ctx && stream_out, "NULL argument");
    *stream_out = (void *)ctx->stream;
    return SBR_OK;
}

extern "C" int sbr_ctx_launch_count(sbr_ctx *ctx, int64_t *count_out)
{
    REQUIRE(ctx && count_out, "NULL argument");
    *count_out = ctx->launches;
    return SBR_OK;
}

// ---------------------------------------------------------------------------
// mesh
// ---------------------------------------------------------------------------
// Host (pageable) -> device upload through two pinned 16 MB chunks: the
// persistent copy workers (CopyPool) copy chunk k+1 into one pinned buffer
// while the DMA engine moves chunk k from the other (pageable cudaMemcpy runs
// at ~10 GB/s and serialises the staging copy with the transfer).
static constexpr size_t kPinChunk = (size_t)16 << 20;
static constexpr unsigned kCopyThreads = 4;   // B200 box: 4 beat 1, 2, 8, 12, 16

static cudaError_t upload_host(sbr_ctx *ctx, void *dst, const void *src, size_t bytes)
{
    if (bytes < ((size_t)4 << 20))
        return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream);
    for (int b = 0; b < 2; ++b) {
        if (!ctx->pin[b]) {
            cudaError_t e = cudaHostAlloc((void **)&ctx->pin[b], kPinChunk, cudaHostAllocDefault);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->pin_ev[b], cudaEventDisableTiming);
            if (e != cudaSuccess) {
                if (ctx->pin[b]) cudaFreeHost(ctx->pin[b]);
                ctx->pin[b] = nullptr;
                cudaGetLastError();
                return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream);
            }
            cudaEventRecord(ctx->pin_ev[b], ctx->stream);
        }
    }
    if (ctx->copiers.th.empty()) {
        const unsigned hw = std::thread::hardware_concurrency();
        ctx->copiers.start((int)std::max(1u, std::min(kCopyThreads, hw ? hw : 1u)));
    }
    const unsigned char *s = static_cast<const unsigned char *>(src);
    unsigned char *d = static_cast<unsigned char *>(dst);
    int b = 0;
    for (size_t off = 0; off < bytes; off += kPinChunk, b ^= 1) {
        const size_t n = std::min(kPinChunk, bytes - off);
        cudaError_t e = cudaEventSynchronize(ctx->pin_ev[b]);   // buffer b free again
        if (e != cudaSuccess) return e;
        ctx->copiers.copy(ctx->pin[b], s + off, n);
        e = cudaMemcpyAsync(d + off, ctx->pin[b], n, cudaMemcpyHostToDevice, ctx->stream);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->pin_ev[b], ctx->stream);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

extern "C" int sbr_mesh_create(sbr_ctx *ctx, const double *v0, const double *v1,
                               const double *v2, const double *normals, int64_t ntri,
                               int32_t storage, sbr_mesh **out)
{
    REQUIRE(ctx && v0 && v1 && v2 && normals && out, "NULL argument");
    REQUIRE(ntri >= 1, "mesh has no triangles");
    REQUIRE(ntri < kMaxTriangles, "mesh has %lld triangles; the device layout supports < %lld",
            (long long)ntri, (long long)kMaxTriangles);
    REQUIRE(storage >= SBR_STORAGE_AUTO && storage <= SBR_STORAGE_SINGLE, "bad storage %d",
            storage);
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    // Raw SoA upload, then one device pass interleaves the (T,9) vertex
    // records and reduces the AABB, centroid bounds and the finite /
    // float32-representable flags (no host-side loop over the mesh).
    sbr_mesh *m = new sbr_mesh();
    m->ctx = ctx;
    m->ntri = ntri;
    MeshIngest ing;
    cudaError_t e = m->verts.alloc((size_t)ntri * 9);
    if (e == cudaSuccess) e = m->normals.alloc((size_t)ntri * 3);
    if (e == cudaSuccess) e = ctx->stage.reserve((size_t)ntri * 9);
    if (e == cudaSuccess) e = upload_host(ctx, ctx->stage.p, v0, 24 * ntri);
    if (e == cudaSuccess) e = upload_host(ctx, ctx->stage.p + 3 * ntri, v1, 24 * ntri);
    if (e == cudaSuccess) e = upload_host(ctx, ctx->stage.p + 6 * ntri, v2, 24 * ntri);
    if (e == cudaSuccess) e = upload_host(ctx, m->normals.p, normals, sizeof(double) * 3 * ntri);
    if (e == cudaSuccess)
        e = mesh_ingest(ctx->stage.p, ntri, m->verts.p, ing, ctx->stream, &ctx->launches);
    if (e != cudaSuccess) {
        delete m;
        return fail(e == cudaErrorMemoryAllocation ? SBR_ENOMEM : SBR_ECUDA, "mesh upload: %s",
                    cudaGetErrorString(e));
    }
    if (!ing.finite) {
        delete m;
        return fail(SBR_EINVAL, "mesh has non-finite vertex coordinates");
    }
    int st = storage;
    if (st == SBR_STORAGE_AUTO) st = ing.all_f32 ? SBR_STORAGE_F32_EXACT : SBR_STORAGE_F64;
    if ((st == SBR_STORAGE_F32_EXACT || st == SBR_STORAGE_SINGLE) && !ing.all_f32) {
        delete m;
        return fail(SBR_EINVAL, "storage requires float32-representable vertices");
    }
    m->storage = st;
    for (int a = 0; a < 3; ++a) {
        m->aabb[a] = ing.lo[a]; m->aabb[3 + a] = ing.hi[a];
        m->cmin[a] = ing.clo[a]; m->cmax[a] = ing.chi[a];
    }
    *out = m;
    return SBR_OK;
}

extern "C" int sbr_mesh_destroy(sbr_mesh *mesh)
{
    if (!mesh) return SBR_OK;
    cudaSetDevice(mesh->ctx->device);
    delete mesh;
    return SBR_OK;
}

extern "C" int sbr_mesh_info(const sbr_mesh *mesh, int64_t *ntri, int32_t *storage,
                             double aabb[6])
{
    REQUIRE(mesh, "mesh is NULL");
    if (ntri) *ntri = mesh->ntri;
    if (storage) *storage = mesh->storage;
    if (aabb) memcpy(aabb, mesh->aabb, sizeof(double) * 6);
    return SBR_OK;
}

// ---------------------------------------------------------------------------
// BVH
// ---------------------------------------------------------------------------
static void set_frame(sbr_bvh *b, const sbr_mesh *m)
{
    double s = 0.0;
    for (int a = 0; a < 3; ++a) {
        b->frame[a] = 0.5 * (m->aabb[a] + m->aabb[3 + a]);
        s = fmax(s, fmax(fabs(m->aabb[a] - b->frame[a]), fabs(m->aabb[3 + a] - b->frame[a])));
    }
    b->scale = (float)s * 1.0001f + 1e-30f;
}

static int build_sah(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_build_params *params,
                     sbr_bvh *b);

extern "C" int sbr_bvh_build(sbr_ctx *ctx, const sbr_mesh *mesh,
                             const sbr_build_params *params, sbr_bvh **out)
{
    REQUIRE(ctx && mesh && out, "NULL argument");
    int n_leaf = params ? params->n_leaf : 4;
    REQUIRE(n_leaf >= 1, "n_leaf must be >= 1, got %d", n_leaf);
    const int rule = params ? params->split_rule : SBR_SPLIT_SAH;
    REQUIRE(rule == SBR_SPLIT_MEDIAN || rule == SBR_SPLIT_SAH || rule == SBR_SPLIT_LBVH,
            "unknown split rule %d", rule);
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    sbr_bvh *b = new sbr_bvh();
    b->ctx = ctx;
    b->mesh = mesh;
    if (rule == SBR_SPLIT_SAH || rule == SBR_SPLIT_MEDIAN) {
        sbr_build_params p = *params;
        if (int rc = build_sah(ctx, mesh, &p, b)) {
            delete b;
            return rc;
        }
        *out = b;
        return SBR_OK;
    }
    REQUIRE(n_leaf <= kMaxLeafCount, "the LBVH builder supports n_leaf <= %d, got %d",
            kMaxLeafCount, n_leaf);
    set_frame(b, mesh);
    LbvhInput in;
    in.d_verts = mesh->verts.p;
    in.ntri = mesh->ntri;
    in.storage = mesh->storage;
    in.n_leaf = n_leaf;
    for (int a = 0; a < 3; ++a) {
        in.cmin[a] = mesh->cmin[a]; in.cmax[a] = mesh->cmax[a];
        in.frame[a] = b->frame[a];
    }
    memcpy(in.aabb, mesh->aabb, sizeof(in.aabb));
    cudaError_t e = lbvh_build(in, b->out, ctx->ws, ctx->stream, &ctx->launches);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e == cudaSuccess) e = collapse_bvh4(b->out, ctx->ws, ctx->stream, &ctx->launches);
    if (e != cudaSuccess) {
        delete b;
        return fail(e == cudaErrorMemoryAllocation ? SBR_ENOMEM : SBR_ECUDA, "LBVH build: %s",
                    cudaGetErrorString(e));
    }
    if (int rc = check_depth(b)) return rc;
    *out = b;
    return SBR_OK;
}

// host conversion of a reference preorder tree into child-pair nodes
struct UploadBuilder {
    const double *nmin, *nmax;
    const int32_t *first, *count;
    int64_t nn;
    double frame[3];
    std::vector<Node> nodes;
    int max_depth = 0;
    bool ok = true;
    std::string why;

    void rel(const double *lo, const double *hi, float out[6]) const
    {
        for (int a = 0; a < 3; ++a) {
            float l = (float)(lo[a] - frame[a]), h = (float)(hi[a] - frame[a]);
            out[a] = nextafterf(l, -INFINITY);
            out[3 + a] = nextafterf(h, INFINITY);
        }
    }
    // reference for a leaf range; splits ranges > kMaxLeafCount into a
    // balanced subtree of internal nodes sharing the leaf box
    int leaf_range(int f, int c, const float box[6], int depth)
    {
        if (c <= kMaxLeafCount) return leaf_ref(f, c);
        int me = (int)nodes.size();
        nodes.push_back(Node());
        max_depth = std::max(max_depth, depth);
        int h = c / 2;
        int l = leaf_range(f, h, box, depth + 1);
        int r = leaf_range(f + h, c - h, box, depth + 1);
        Node nd;
        nd.a = make_float4(box[0], box[1], box[2], box[3]);
        nd.b = make_float4(box[4], box[5], box[0], box[1]);
        nd.c = make_float4(box[2], box[3], box[4], box[5]);
        nd.d = make_int4(l, r, 0, 0);
        nodes[me] = nd;
        return me;
    }
    int child_ref(int64_t i, int depth, float box[6])
    {
        rel(nmin + 3 * i, nmax + 3 * i, box);
        if (count[i] > 0) return leaf_range(first[i], count[i], box, depth);
        return internal(i, depth);
    }
    int internal(int64_t i, int depth)
    {
        if (!ok) return 0;
        int64_t l = i + 1, r = first[i];
        if (!(l > 0 && l < nn && r > 0 && r < nn)) {
            ok = false;
            why = "bad child index";
            return 0;
        }
        int me = (int)nodes.size();
        nodes.push_back(Node());
        max_depth = std::max(max_depth, depth);
        float bl[6], br[6];
        int rl = child_ref(l, depth + 1, bl);
        int rr = child_ref(r, depth + 1, br);
        Node nd;
        nd.a = make_float4(bl[0], bl[1], bl[2], bl[3]);
        nd.b = make_float4(bl[4], bl[5], br[0], br[1]);
        nd.c = make_float4(br[2], br[3], br[4], br[5]);
        nd.d = make_int4(rl, rr, 0, 0);
        nodes[me] = nd;
        return me;
    }
};

// reference-layout tree -> device BVH2 (+ BVH4) into a fresh sbr_bvh;
// the caller holds ctx->mu and has validated the permutation
static int upload_ref_tree(sbr_ctx *ctx, const sbr_mesh *mesh, const double *nodes_min,
                           const double *nodes_max, const int32_t *node_first,
                           const int32_t *node_count, const int32_t *tri_order,
                           int64_t nnodes, sbr_bvh *b)
{
    set_frame(b, mesh);
    UploadBuilder U{nodes_min, nodes_max, node_first, node_count, nnodes,
                    {b->frame[0], b->frame[1], b->frame[2]}};
    if (node_count[0] > 0) {
        // root is a leaf: wrap it in a node carrying the leaf twice
        float box[6];
        U.rel(nodes_min, nodes_max, box);
        U.nodes.push_back(Node());
        int r = U.leaf_range(node_first[0], node_count[0], box, 1);
        Node nd;
        nd.a = make_float4(box[0], box[1], box[2], box[3]);
        nd.b = make_float4(box[4], box[5], box[0], box[1]);
        nd.c = make_float4(box[2], box[3], box[4], box[5]);
        nd.d = make_int4(r, r, 0, 0);
        U.nodes[0] = nd;
    } else {
        U.internal(0, 0);
    }
    if (!U.ok) return fail(SBR_EINVAL, "invalid BVH: %s", U.why.c_str());
    DevBuf<int> order(mesh->ntri);
    cudaError_t e = order.status();
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(order.p, tri_order, sizeof(int) * mesh->ntri, cudaMemcpyHostToDevice,
                            ctx->stream);
    if (e == cudaSuccess)
        e = pack_tris(mesh->verts.p, order.p, mesh->ntri, mesh->storage, b->out, ctx->stream,
                      &ctx->launches);
    if (e == cudaSuccess) e = b->out.leaf_ids.alloc(mesh->ntri);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(b->out.leaf_ids.p, order.p, sizeof(int) * mesh->ntri,
                            cudaMemcpyDeviceToDevice, ctx->stream);
    if (e == cudaSuccess) e = b->out.nodes.alloc(U.nodes.size());
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(b->out.nodes.p, U.nodes.data(), sizeof(Node) * U.nodes.size(),
                            cudaMemcpyHostToDevice, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return fail(SBR_ECUDA, "BVH upload: %s", cudaGetErrorString(e));
    b->out.nnodes = (int64_t)U.nodes.size();
    b->out.n_leaf_slots = mesh->ntri;
    b->out.root = 0;
    b->out.max_depth = U.max_depth;
    b->out.storage = mesh->storage;
    e = collapse_bvh4(b->out, ctx->ws, ctx->stream, &ctx->launches);
    if (e != cudaSuccess) return fail(SBR_ECUDA, "BVH upload: %s", cudaGetErrorString(e));
    if (b->out.width == 8 && 7 * b->out.depth8 + 1 >= kStack) b->out.width = 4;  // stack bound
    b->deep = b->out.depth4 > kMaxDepth4;   // checked against the reference tree by the caller
    return SBR_OK;
}

// A deep tree (BVH4 depth > kMaxDepth4) is walked in reference order on its
// reference tree; without one (LBVH) or beyond that kernel's stack: EINVAL.
static int deep_ok(const sbr_bvh *b)
{
    if (!b->deep) return SBR_OK;
    if (b->ref_dev.nnodes > 0 && b->ref_tree_depth >= 0 && b->ref_tree_depth + 1 < 256)
        return SBR_OK;
    return fail(SBR_EINVAL, "BVH4 depth %d exceeds the traversal stack limit (%d) and no "
                "reference tree of depth < 255 is available", b->out.depth4, kMaxDepth4);
}

static bool use_ref(const sbr_ctx *ctx, const sbr_bvh *bvh)
{
    return ctx->traversal == SBR_TRAVERSAL_REFERENCE || bvh->deep;
}

extern "C" int sbr_bvh_upload(sbr_ctx *ctx, const sbr_mesh *mesh, const double *nodes_min,
                              const double *nodes_max, const int32_t *node_first,
                              const int32_t *node_count, const int32_t *tri_order,
                              int64_t nnodes, sbr_bvh **out)
{
    REQUIRE(ctx && mesh && nodes_min && nodes_max && node_first && node_count && tri_order && out,
            "NULL argument");
    REQUIRE(nnodes >= 1, "empty tree");
    // permutation check (bvh.py:95-97)
    std::vector<char> seen((size_t)mesh->ntri, 0);
    for (int64_t k = 0; k < mesh->ntri; ++k) {
        int32_t t = tri_order[k];
        REQUIRE(t >= 0 && t < mesh->ntri && !seen[t], "tri_order is not a permutation");
        seen[t] = 1;
    }
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    sbr_bvh *b = new sbr_bvh();
    b->ctx = ctx;
    b->mesh = mesh;
    if (int rc = upload_ref_tree(ctx, mesh, nodes_min, nodes_max, node_first, node_count,
                                 tri_order, nnodes, b)) {
        delete b;
        return rc;
    }
    // device copy of the layout itself for reference-order traversal
    // (bvh.py:306-362 replayed as given: no further box rounding)
    {
        SahTree &T = b->ref_dev;
        const size_t N = (size_t)nnodes, Tn = (size_t)mesh->ntri;
        cudaError_t e = T.nmin.alloc(3 * N);
        if (e == cudaSuccess) e = T.nmax.alloc(3 * N);
        if (e == cudaSuccess) e = T.first.alloc(N);
        if (e == cudaSuccess) e = T.count.alloc(N);
        if (e == cudaSuccess) e = T.order.alloc(Tn);
        cudaStream_t st = ctx->stream;
        if (e == cudaSuccess) e = cudaMemcpyAsync(T.nmin.p, nodes_min, 24 * N, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(T.nmax.p, nodes_max, 24 * N, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(T.first.p, node_first, 4 * N, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(T.count.p, node_count, 4 * N, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(T.order.p, tri_order, 4 * Tn, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            delete b;
            return fail(SBR_ECUDA, "BVH upload: %s", cudaGetErrorString(e));
        }
        T.nnodes = (int64_t)nnodes;
        // depth by walking the preorder layout (children of i: i+1, first[i])
        std::vector<int> depth(N, 0);
        int md = 0;
        for (size_t i = 0; i < N; ++i) {
            md = depth[i] > md ? depth[i] : md;
            if (node_count[i] == 0) {
                const int32_t l = (int32_t)i + 1, r = node_first[i];
                if (l > 0 && (size_t)l < N) depth[l] = depth[i] + 1;
                if (r > 0 && (size_t)r < N) depth[r] = depth[i] + 1;
            }
        }
        T.max_depth = md;
        b->ref_tree_depth = md;
    }
    if (int rc = deep_ok(b)) {
        delete b;
        return rc;
    }
    *out = b;
    return SBR_OK;
}

// GPU build of the reference binned-SAH tree (sahbuild.cu): the reference
// layout stays on the device (exported verbatim on request) and is converted
// to traversal nodes on the device
static int ref_download(const sbr_bvh *bvh);

static int build_sah(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_build_params *params,
                     sbr_bvh *b)
{
    SahParams P;
    P.n_leaf = params->n_leaf;
    P.max_depth = params->max_depth > 0 ? params->max_depth : 64;
    P.bins = params->bins_per_axis > 0 ? params->bins_per_axis : 16;
    P.c_t = params->c_t > 0.0 ? params->c_t : 1.0;
    P.c_i = params->c_i > 0.0 ? params->c_i : 1.0;
    P.median = params->split_rule == SBR_SPLIT_MEDIAN;
    REQUIRE(P.median || (P.bins >= 2 && P.bins <= kSahMaxBins),
            "bins_per_axis must be in [2, %d]", kSahMaxBins);
    const bool timing = getenv("SBR_SAH_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point z) {
        return std::chrono::duration<double, std::milli>(z - a).count();
    };
    const auto t0 = now();
    SahTree &T = b->ref_dev;
    cudaError_t e = sah_build(mesh->verts.p, mesh->ntri, P, T, ctx->sah, ctx->stream,
                              &ctx->launches);
    if (e != cudaSuccess)
        return fail(e == cudaErrorMemoryAllocation ? SBR_ENOMEM : SBR_ECUDA, "SAH build: %s",
                    cudaGetErrorString(e));
    b->ref_depth = T.max_depth;
    b->ref_tree_depth = T.max_depth;
    b->ref_round_f32 = mesh->storage == kSingle;
    set_frame(b, mesh);
    bool host = false;
    e = ref_to_bvh2(T, b->frame, ctx->sah, b->out, host, ctx->stream, &ctx->launches);
    if (e != cudaSuccess) return fail(SBR_ECUDA, "SAH build: %s", cudaGetErrorString(e));
    const auto t1 = now();
    if (host) {   // big leaves / leaf root: the host converter splits them
        if (int rc = ref_download(b)) return rc;
        const int rc = upload_ref_tree(ctx, mesh, b->ref_nmin.data(), b->ref_nmax.data(),
                                       b->ref_first.data(), b->ref_count.data(),
                                       b->ref_order.data(), (int64_t)b->ref_first.size(), b);
        b->out.max_depth = T.max_depth;
        return rc ? rc : deep_ok(b);
    }
    e = pack_tris(mesh->verts.p, T.order.p, mesh->ntri, mesh->storage, b->out, ctx->stream,
                  &ctx->launches);
    if (e == cudaSuccess) e = b->out.leaf_ids.alloc(mesh->ntri);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(b->out.leaf_ids.p, T.order.p, sizeof(int) * mesh->ntri,
                            cudaMemcpyDeviceToDevice, ctx->stream);
    b->out.n_leaf_slots = mesh->ntri;
    b->out.storage = mesh->storage;
    if (e == cudaSuccess) e = collapse_bvh4(b->out, ctx->ws, ctx->stream, &ctx->launches);
    if (e != cudaSuccess) return fail(SBR_ECUDA, "SAH build: %s", cudaGetErrorString(e));
    if (timing)
        fprintf(stderr, "[sah] build+convert %.2f ms, pack+bvh4 %.2f ms, nodes %lld\n",
                ms(t0, t1), ms(t1, now()), (long long)T.nnodes);
    if (b->out.width == 8 && 7 * b->out.depth8 + 1 >= kStack) b->out.width = 4;  // stack bound
    b->deep = b->out.depth4 > kMaxDepth4;
    return deep_ok(b);
}

static int ref_download(const sbr_bvh *bvh)
{
    sbr_bvh *b = const_cast<sbr_bvh *>(bvh);
    if (!b->ref_first.empty() || b->ref_dev.nnodes == 0) return SBR_OK;
    const size_t N = (size_t)b->ref_dev.nnodes;
    const size_t T = (size_t)b->mesh->ntri;
    b->ref_nmin.resize(3 * N);
    b->ref_nmax.resize(3 * N);
    b->ref_first.resize(N);
    b->ref_count.resize(N);
    b->ref_order.resize(T);
    CUDA_TRY(cudaSetDevice(b->ctx->device));
    cudaStream_t st = b->ctx->stream;
    CUDA_TRY(cudaMemcpyAsync(b->ref_nmin.data(), b->ref_dev.nmin.p, 24 * N, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(b->ref_nmax.data(), b->ref_dev.nmax.p, 24 * N, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(b->ref_first.data(), b->ref_dev.first.p, 4 * N, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(b->ref_count.data(), b->ref_dev.count.p, 4 * N, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(b->ref_order.data(), b->ref_dev.order.p, 4 * T, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return SBR_OK;
}

// ---- export to the reference preorder layout -------------------------------
struct Exporter {
    const std::vector<Node> &nodes;
    const double *frame;
    std::vector<double> nmin, nmax;
    std::vector<int32_t> first, count;

    static void box_of(const Node &n, int which, float b[6])
    {
        if (which == 0) {
            b[0] = n.a.x; b[1] = n.a.y; b[2] = n.a.z; b[3] = n.a.w; b[4] = n.b.x; b[5] = n.b.y;
        } else {
            b[0] = n.b.z; b[1] = n.b.w; b[2] = n.c.x; b[3] = n.c.y; b[4] = n.c.z; b[5] = n.c.w;
        }
    }
    int64_t emit_box(const float b[6], const float b2[6])
    {
        int64_t me = (int64_t)first.size();
        for (int a = 0; a < 3; ++a) {
            double lo = (double)b[a], hi = (double)b[3 + a];
            if (b2) { lo = fmin(lo, (double)b2[a]); hi = fmax(hi, (double)b2[3 + a]); }
            nmin.push_back(lo + frame[a]);
            nmax.push_back(hi + frame[a]);
        }
        first.push_back(0);
        count.push_back(0);
        return me;
    }
    // preorder emit of reference `ref` with box b; returns node index
    int64_t emit(int ref, const float b[6])
    {
        int64_t me = emit_box(b, nullptr);
        if (ref < 0) {
            first[me] = leaf_first(ref);
            count[me] = leaf_count(ref);
            return me;
        }
        const Node &n = nodes[ref];
        float bl[6], br[6];
        box_of(n, 0, bl);
        box_of(n, 1, br);
        emit(n.d.x, bl);
        int64_t r = emit(n.d.y, br);
        first[me] = (int32_t)r;
        count[me] = 0;
        return me;
    }
};

static int export_tree(const sbr_bvh *b, std::vector<Node> &nodes, Exporter **ex)
{
    nodes.resize(b->out.nnodes);
    CUDA_TRY(cudaMemcpyAsync(nodes.data(), b->out.nodes.p, sizeof(Node) * nodes.size(),
                             cudaMemcpyDeviceToHost, b->ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(b->ctx->stream));
    Exporter *E = new Exporter{nodes, b->frame, {}, {}, {}, {}};
    const Node &r = nodes[0];
    float bl[6], br[6], root[6];
    Exporter::box_of(r, 0, bl);
    Exporter::box_of(r, 1, br);
    for (int a = 0; a < 3; ++a) {
        root[a] = fminf(bl[a], br[a]);
        root[3 + a] = fmaxf(bl[3 + a], br[3 + a]);
    }
    if (r.d.x == r.d.y) {
        E->emit(r.d.x, root);  // single-leaf tree
    } else {
        int64_t me = E->emit_box(root, nullptr);
        E->emit(r.d.x, bl);
        int64_t right = E->emit(r.d.y, br);
        E->first[me] = (int32_t)right;
        E->count[me] = 0;
    }
    *ex = E;
    return SBR_OK;
}

extern "C" int sbr_bvh_info(const sbr_bvh *bvh, int64_t *nnodes_export, int64_t *nnodes_device,
                            int32_t *max_depth)
{
    REQUIRE(bvh, "bvh is NULL");
    if (nnodes_device) *nnodes_device = bvh->out.nnodes;
    if (bvh->ref_depth >= 0) {
        if (max_depth) *max_depth = bvh->ref_depth;
        if (nnodes_export) *nnodes_export = bvh->ref_dev.nnodes ? bvh->ref_dev.nnodes
                                                                : (int64_t)bvh->ref_first.size();
        return SBR_OK;
    }
    if (max_depth) *max_depth = bvh->out.max_depth + 1;
    if (nnodes_export) {
        if (int rc = set_device(bvh->ctx)) return rc;
        std::vector<Node> nodes;
        Exporter *E = nullptr;
        if (int rc = export_tree(bvh, nodes, &E)) return rc;
        *nnodes_export = (int64_t)E->first.size();
        delete E;
    }
    return SBR_OK;
}

extern "C" int sbr_bvh_export(const sbr_bvh *bvh, double *nodes_min, double *nodes_max,
                              int32_t *node_first, int32_t *node_count, int32_t *tri_order)
{
    REQUIRE(bvh && nodes_min && nodes_max && node_first && node_count && tri_order,
            "NULL argument");
    if (bvh->ref_depth >= 0) {
        if (int rc = ref_download(bvh)) return rc;
        memcpy(nodes_min, bvh->ref_nmin.data(), sizeof(double) * bvh->ref_nmin.size());
        memcpy(nodes_max, bvh->ref_nmax.data(), sizeof(double) * bvh->ref_nmax.size());
        memcpy(node_first, bvh->ref_first.data(), sizeof(int32_t) * bvh->ref_first.size());
        memcpy(node_count, bvh->ref_count.data(), sizeof(int32_t) * bvh->ref_count.size());
        memcpy(tri_order, bvh->ref_order.data(), sizeof(int32_t) * bvh->ref_order.size());
        return SBR_OK;
    }
    if (int rc = set_device(bvh->ctx)) return rc;
    std::vector<Node> nodes;
    Exporter *E = nullptr;
    if (int rc = export_tree(bvh, nodes, &E)) return rc;
    memcpy(nodes_min, E->nmin.data(), sizeof(double) * E->nmin.size());
    memcpy(nodes_max, E->nmax.data(), sizeof(double) * E->nmax.size());
    memcpy(node_first, E->first.data(), sizeof(int32_t) * E->first.size());
    memcpy(node_count, E->count.data(), sizeof(int32_t) * E->count.size());
    delete E;
    CUDA_TRY(cudaMemcpyAsync(tri_order, bvh->out.leaf_ids.p, sizeof(int32_t) * bvh->mesh->ntri,
                             cudaMemcpyDeviceToHost, bvh->ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(bvh->ctx->stream));
    return SBR_OK;
}

extern "C" int sbr_bvh_destroy(sbr_bvh *bvh)
{
    if (!bvh) return SBR_OK;
    cudaSetDevice(bvh->ctx->device);
    delete bvh;
    return SBR_OK;
}

// ---------------------------------------------------------------------------
// queries
// ---------------------------------------------------------------------------
static int check_pair(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh)
{
    REQUIRE(ctx && mesh && bvh, "NULL handle");
    REQUIRE(bvh->mesh == mesh, "BVH was built for a different mesh");
    REQUIRE(mesh->ctx == ctx && bvh->ctx == ctx, "handles belong to another context");
    return SBR_OK;
}

static RefView ref_view(const sbr_bvh *b)
{
    RefView v;
    v.nmin = b->ref_dev.nmin.p;
    v.nmax = b->ref_dev.nmax.p;
    v.first = b->ref_dev.first.p;
    v.count = b->ref_dev.count.p;
    v.order = b->ref_dev.order.p;
    v.round_f32 = b->ref_round_f32;
    v.verts = b->mesh->verts.p;
    v.single = b->mesh->storage == kSingle;
    return v;
}

// reference-order traversal needs the reference-layout tree on the device
static int check_ref_mode(const sbr_ctx *ctx, const sbr_bvh *bvh)
{
    if (!use_ref(ctx, bvh)) return SBR_OK;
    REQUIRE(bvh->ref_dev.nnodes > 0,
            "reference-order traversal needs the reference tree (split_rule 'sah' or 'median', "
            "or an uploaded tree)");
    REQUIRE(bvh->ref_tree_depth >= 0 && bvh->ref_tree_depth + 1 < 256,
            "tree depth %d exceeds the reference-order traversal stack (255)",
            bvh->ref_tree_depth);
    return SBR_OK;
}

extern "C" int sbr_ctx_set_traversal(sbr_ctx *ctx, int32_t mode)
{
    REQUIRE(ctx, "ctx is NULL");
    REQUIRE(mode == SBR_TRAVERSAL_FAST || mode == SBR_TRAVERSAL_REFERENCE,
            "unknown traversal mode %d", (int)mode);
    std::lock_guard<std::mutex> lk(ctx->mu);
    ctx->traversal = mode;
    return SBR_OK;
}

extern "C" int sbr_ctx_get_traversal(sbr_ctx *ctx, int32_t *mode)
{
    REQUIRE(ctx && mode, "NULL argument");
    *mode = ctx->traversal;
    return SBR_OK;
}

// Query 0 of aperture rays: rasterised per triangle or traced through the
// BVH like every other query.  Both give the same bits.  The raster pass
// hands each warp 32 triangles of one grid, so it needs many (grid,
// triangle) pairs to fill the GPU: below ~512 warps of work (a handful of
// large triangles, e.g. corner reflectors) the BVH path is faster.
// SBR_PRIMARY=raster|bvh forces a path (A/B measurement, parity tests).
static bool raster_primary(int64_t ntri, int64_t ngrids)
{
    const char *s = getenv("SBR_PRIMARY");
    if (s && std::strcmp(s, "bvh") == 0) return false;
    if (s && std::strcmp(s, "raster") == 0) return true;
    return ngrids * ((ntri + 31) / 32) >= 512;
}

static RasterArgs raster_args(const sbr_bvh *bvh, const GridDev *grids, const int *bgrids,
                              int nbg, const int64_t *seg_base, const int64_t *seg_slot,
                              PrimHit *prim)
{
    RasterArgs r;
    r.B = bvh->view();
    r.storage = bvh->mesh->storage;
    r.ntri = bvh->mesh->ntri;
    r.grids = grids;
    r.bgrids = bgrids;
    r.nbg = nbg;
    r.seg_base = seg_base;
    r.seg_slot = seg_slot;
    r.prim = prim;
    r.counter = nullptr;
    r.sparse = 0;
    r.big = nullptr;
    r.nbig = nullptr;
    r.big_cap = 0;
    r.setups = nullptr;
    r.nsetup = nullptr;
    r.setup_cap = 0;
    r.hitmap = nullptr;
    r.row_lo = 0;
    r.row_hi = INT64_MAX;
    r.stats = nullptr;
    return r;
}

// big-triangle chunk queue of the raster pass (grow-only, 4M items = 64 MB);
// SBR_BIG_CAP (tests) shrinks it to force the overflow path
// rays: ray slots of the launch.  Queued chunks run at about rays / 256
// (C5: 3.7M for 1.0e9 rays), so the queue holds rays / 64 (64k .. 16M) and
// the set-up table rays / 512 triangles (16k .. 2M) -- sized to the launch,
// not to the largest workload.  Overflow stays exact (walked in k_raster).
static cudaError_t attach_big_queue(sbr_ctx *ctx, RasterArgs &ra, int64_t rays)
{
    size_t cap = (size_t)std::min<int64_t>((int64_t)1 << 24,
                                           std::max<int64_t>((int64_t)1 << 16, rays / 64));
    if (const char *s = getenv("SBR_BIG_CAP")) {
        const long long v = atoll(s);
        if (v >= 1 && v < (long long)cap) cap = (size_t)v;
    }
    cudaError_t e = ctx->big.reserve(cap);
    if (e == cudaSuccess) e = ctx->nbig.reserve(1);
    if (e != cudaSuccess) return e;
    ra.big = ctx->big.p;
    ra.nbig = ctx->nbig.p;
    ra.big_cap = (int64_t)cap;
    const size_t scap = (size_t)std::min<int64_t>((int64_t)1 << 21,
                                                  std::max<int64_t>((int64_t)1 << 14, rays / 512));
    e = ctx->setups.reserve(scap * kRasterSetupBytes);
    if (e == cudaSuccess) e = ctx->nsetup.reserve(1);
    if (e != cudaSuccess) return e;
    ra.setups = ctx->setups.p;
    ra.nsetup = ctx->nsetup.p;
    ra.setup_cap = (int64_t)scap;
    return cudaSuccess;
}

static TraceCfg make_cfg(const sbr_bvh *bvh, const sbr_trace_params *p, sbr_ctx *ctx)
{
    TraceCfg c;
    c.B = bvh->view();
    c.storage = bvh->mesh->storage;
    c.max_bounces = p->max_bounces;
    c.eps = p->eps;
    c.strict = p->strict;
    c.count_trapped = 0;
    c.allow_aliasing = p->allow_aliasing;
    c.spacing_limit = (p->lambda_min > 0.0 && p->sampling_factor > 0.0)
                          ? p->lambda_min / p->sampling_factor
                          : INFINITY;
    c.error_flag = ctx->err_flag.p;
    return c;
}

static int check_params(const sbr_trace_params *p)
{
    REQUIRE(p, "params is NULL");
    REQUIRE(p->max_bounces >= 1, "max_bounces must be >= 1");
    REQUIRE(p->max_bounces <= 0xffff, "max_bounces too large");
    REQUIRE(p->eps > 0.0 && std::isfinite(p->eps), "epsilon must be positive");
    return SBR_OK;
}

extern "C" int sbr_closest_hit(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                               const double *origins, const double *dirs, int64_t n,
                               double t_min, double t_max, int64_t *tri, double *t,
                               int64_t *visits)
{
    if (int rc = check_pair(ctx, mesh, bvh)) return rc;
    REQUIRE(n >= 0, "negative ray count");
    if (n == 0) return SBR_OK;
    REQUIRE(origins && dirs && tri && t, "NULL argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    DevBuf<double> o(3 * n), d(3 * n), tt(n);
    DevBuf<int64_t> ti(n), vi(n);
    CUDA_TRY(o.status()); CUDA_TRY(d.status()); CUDA_TRY(tt.status());
    CUDA_TRY(ti.status()); CUDA_TRY(vi.status());
    cudaStream_t st = ctx->stream;
    CUDA_TRY(cudaMemcpyAsync(o.p, origins, 24 * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d.p, dirs, 24 * n, cudaMemcpyHostToDevice, st));
    if (int rc = check_ref_mode(ctx, bvh)) return rc;
    if (use_ref(ctx, bvh))
        CUDA_TRY(launch_closest_ref(ref_view(bvh), o.p, d.p, n, t_min, t_max, ti.p, tt.p, vi.p,
                                    st, ctx->stats()));
    else
        CUDA_TRY(launch_closest(bvh->view(), mesh->storage, o.p, d.p, n, t_min, t_max, ti.p,
                                tt.p, vi.p, st, ctx->stats()));
    CUDA_TRY(cudaMemcpyAsync(tri, ti.p, 8 * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(t, tt.p, 8 * n, cudaMemcpyDeviceToHost, st));
    if (visits) CUDA_TRY(cudaMemcpyAsync(visits, vi.p, 8 * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return SBR_OK;
}

// Shared body of sbr_trace_grid[_rows|_hash] and sbr_trace_rays.  Grid mode
// traces rows [i_begin, i_end) of the grid (records indexed from
// i_begin * n_v); seg_hash != NULL selects hash mode (no per-ray outputs:
// per-segment record hashes, segment = seg_rays consecutive ray indices of
// the whole grid).
static int trace_full_common(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                             const sbr_grid *grid, const double *origins, const double *dirs,
                             int64_t n_list, int64_t i_begin, int64_t i_end,
                             const sbr_trace_params *params, uint8_t *valid,
                             double *normal0, double *path, int32_t *bounces, uint8_t *escaped,
                             double *out_dir, int32_t *tri_ids, uint64_t *seg_hash,
                             int64_t seg_rays)
{
    if (int rc = check_pair(ctx, mesh, bvh)) return rc;
    if (int rc = check_params(params)) return rc;
    const bool hash = seg_hash != nullptr;
    REQUIRE(hash || (valid && normal0 && path && bounces && escaped && out_dir), "NULL output");
    const int64_t n = grid ? (i_end - i_begin) * grid->n_v : n_list;
    const int64_t r_base = grid ? i_begin * grid->n_v : 0;
    const int64_t n_grid = grid ? grid->n_u * grid->n_v : 0;
    const int64_t nhash = hash ? (n_grid + seg_rays - 1) / seg_rays : 0;
    if (hash) std::memset(seg_hash, 0, sizeof(uint64_t) * nhash);
    if (n == 0) return SBR_OK;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    if (int rc = check_ref_mode(ctx, bvh)) return rc;
    cudaStream_t st = ctx->stream;
    const int B = params->max_bounces;
    const int64_t m = hash ? 0 : n;
    DevBuf<uint8_t> dv(m), de(m);
    DevBuf<double> dn(3 * m), dp(m), dd(3 * m), o, d;
    DevBuf<int32_t> db(m), di;
    DevBuf<unsigned long long> dh;
    DevBuf<GridDev> dg;
    CUDA_TRY(dv.status()); CUDA_TRY(de.status()); CUDA_TRY(dn.status()); CUDA_TRY(dp.status());
    CUDA_TRY(dd.status()); CUDA_TRY(db.status());
    if (tri_ids && !hash) CUDA_TRY(di.alloc((size_t)n * B));
    if (hash) {
        CUDA_TRY(dh.alloc(nhash));
        CUDA_TRY(cudaMemsetAsync(dh.p, 0, 8 * nhash, st));
    }
    if (grid) {
        GridDev g;
        for (int a = 0; a < 3; ++a) {
            g.corner[a] = grid->corner[a]; g.u[a] = grid->u[a];
            g.v[a] = grid->v[a]; g.k[a] = grid->k[a];
        }
        g.spacing = grid->spacing;
        g.n_v = grid->n_v;
        g.n_rays = n_grid;
        grid_derive(g);
        CUDA_TRY(dg.alloc(1));
        CUDA_TRY(cudaMemcpyAsync(dg.p, &g, sizeof(g), cudaMemcpyHostToDevice, st));
    } else {
        CUDA_TRY(o.alloc(3 * n));
        CUDA_TRY(d.alloc(3 * n));
        CUDA_TRY(cudaMemcpyAsync(o.p, origins, 24 * n, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(d.p, dirs, 24 * n, cudaMemcpyHostToDevice, st));
    }
    TraceCfg cfg = make_cfg(bvh, params, ctx);
    FullOut fo{dv.p, dn.p, dp.p, db.p, de.p, dd.p, (tri_ids && !hash) ? di.p : nullptr,
               hash ? dh.p : nullptr, seg_rays};
    if (use_ref(ctx, bvh)) {
        CUDA_TRY(launch_trace_ref(ref_view(bvh), cfg, dg.p, o.p, d.p, n, r_base, fo, nullptr,
                                  nullptr, 0, st, ctx->stats()));
    } else {
        DevBuf<PrimHit> prim;
        DevBuf<int64_t> dsb(2), dss;
        DevBuf<int> dbg(1);
        if (grid && raster_primary(mesh->ntri, 1)) {
            // one grid, prim index = ray index - r_base for every segment
            const int64_t nseg = (n_grid + kSegRays - 1) / kSegRays;
            std::vector<int64_t> sb{0, nseg}, ss(nseg, -r_base);
            const int bg = 0;
            CUDA_TRY(prim.alloc(n));
            CUDA_TRY(dss.alloc(nseg));
            CUDA_TRY(dsb.status()); CUDA_TRY(dbg.status());
            CUDA_TRY(cudaMemcpyAsync(dsb.p, sb.data(), 16, cudaMemcpyHostToDevice, st));
            CUDA_TRY(cudaMemcpyAsync(dss.p, ss.data(), 8 * nseg, cudaMemcpyHostToDevice, st));
            CUDA_TRY(cudaMemcpyAsync(dbg.p, &bg, 4, cudaMemcpyHostToDevice, st));
            CUDA_TRY(cudaMemsetAsync(prim.p, 0xff, sizeof(PrimHit) * n, st));
            RasterArgs ra = raster_args(bvh, dg.p, dbg.p, 1, dsb.p, dss.p, prim.p);
            ra.counter = ctx->counter.p + 1;
            ra.stats = ctx->counter.p + 2;
            ra.row_lo = i_begin;
            ra.row_hi = i_end;
            CUDA_TRY(attach_big_queue(ctx, ra, n));
            CUDA_TRY(launch_raster(ra, st, ctx->stats()));
        }
        CUDA_TRY(launch_trace_full(cfg, dg.p, o.p, d.p, n, r_base, fo, prim.p, ctx->counter.p,
                                   st, ctx->stats()));
        CUDA_TRY(cudaStreamSynchronize(st));   // scratch tables die with this scope
    }
    if (hash) {
        CUDA_TRY(cudaMemcpyAsync(seg_hash, dh.p, 8 * nhash, cudaMemcpyDeviceToHost, st));
    } else {
        CUDA_TRY(cudaMemcpyAsync(valid, dv.p, n, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(escaped, de.p, n, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(normal0, dn.p, 24 * n, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(path, dp.p, 8 * n, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(out_dir, dd.p, 24 * n, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(bounces, db.p, 4 * n, cudaMemcpyDeviceToHost, st));
        if (tri_ids)
            CUDA_TRY(cudaMemcpyAsync(tri_ids, di.p, sizeof(int32_t) * n * B,
                                     cudaMemcpyDeviceToHost, st));
    }
    CUDA_TRY(cudaStreamSynchronize(st));
    return SBR_OK;
}

static int check_grid(const sbr_grid *grid)
{
    REQUIRE(grid, "grid is NULL");
    REQUIRE(grid->n_u >= 1 && grid->n_v >= 1 && grid->spacing > 0.0, "invalid grid");
    return SBR_OK;
}

extern "C" int sbr_trace_grid(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                              const sbr_grid *grid, const sbr_trace_params *params,
                              uint8_t *valid, double *normal0, double *path, int32_t *bounces,
                              uint8_t *escaped, double *out_dir, int32_t *tri_ids)
{
    if (int rc = check_grid(grid)) return rc;
    return trace_full_common(ctx, mesh, bvh, grid, nullptr, nullptr, 0, 0, grid->n_u, params,
                             valid, normal0, path, bounces, escaped, out_dir, tri_ids, nullptr,
                             0);
}

extern "C" int sbr_trace_grid_rows(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                                   const sbr_grid *grid, const sbr_trace_params *params,
                                   int64_t i_begin, int64_t i_end, uint8_t *valid,
                                   double *normal0, double *path, int32_t *bounces,
                                   uint8_t *escaped, double *out_dir, int32_t *tri_ids)
{
    if (int rc = check_grid(grid)) return rc;
    REQUIRE(0 <= i_begin && i_begin <= i_end && i_end <= grid->n_u, "row range out of bounds");
    return trace_full_common(ctx, mesh, bvh, grid, nullptr, nullptr, 0, i_begin, i_end, params,
                             valid, normal0, path, bounces, escaped, out_dir, tri_ids, nullptr,
                             0);
}

extern "C" int sbr_trace_grid_hash(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                                   const sbr_grid *grid, const sbr_trace_params *params,
                                   int64_t i_begin, int64_t i_end, int64_t seg_rays,
                                   uint64_t *seg_hash)
{
    if (int rc = check_grid(grid)) return rc;
    REQUIRE(0 <= i_begin && i_begin <= i_end && i_end <= grid->n_u, "row range out of bounds");
    REQUIRE(seg_rays >= 1 && seg_hash, "bad hash output");
    return trace_full_common(ctx, mesh, bvh, grid, nullptr, nullptr, 0, i_begin, i_end, params,
                             nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                             seg_hash, seg_rays);
}

extern "C" int sbr_trace_rays(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                              const double *origins, const double *dirs, int64_t n,
                              const sbr_trace_params *params, uint8_t *valid, double *normal0,
                              double *path, int32_t *bounces, uint8_t *escaped,
                              double *out_dir, int32_t *tri_ids)
{
    REQUIRE(n >= 0, "negative ray count");
    REQUIRE(n == 0 || (origins && dirs), "NULL rays");
    return trace_full_common(ctx, mesh, bvh, nullptr, origins, dirs, n, 0, 0, params, valid,
                             normal0, path, bounces, escaped, out_dir, tri_ids, nullptr, 0);
}

// ---------------------------------------------------------------------------
// integrate + fused solve
// ---------------------------------------------------------------------------
static int64_t seg_count(int64_t n_rays) { return (n_rays + kSegRays - 1) / kSegRays; }
static int64_t round_chunk(int64_t n) { return (n + kChunk - 1) / kChunk * kChunk; }

extern "C" int sbr_segment_layout(const sbr_grid *grids, int32_t ngrids, int64_t *seg_base)
{
    REQUIRE(grids && seg_base && ngrids >= 0, "bad arguments");
    seg_base[0] = 0;
    for (int g = 0; g < ngrids; ++g)
        seg_base[g + 1] = seg_base[g] + seg_count(grids[g].n_u * grids[g].n_v);
    return SBR_OK;
}

// slots (16 B each) staged per batch: up to 2^30 (16 GB, a whole C4 sweep in
// one persistent launch, so the kernels drain once per solve); run_units
// halves the budget when the device cannot hold a batch.  (Sizing it from
// cudaMemGetInfo made the batching depend on what the allocator pools
// happened to hold.)  SBR_SLOT_BUDGET overrides (tests use tiny budgets to
// prove results do not depend on batching).
static int64_t slot_budget()
{
    const char *s = getenv("SBR_SLOT_BUDGET");
    int64_t v = s ? atoll(s) : ((int64_t)1 << 30);
    if (v < kChunk) v = kChunk;
    // work-list entries and the raster's slot arithmetic hold 32-bit slots
    if (v > ((int64_t)1 << 31)) v = (int64_t)1 << 31;
    return round_chunk(v);
}

// k (wavenumbers) -> device 2k table, and gamma^N host table (po.py:107
// evaluates gamma ** N with libm pow: same as the host pow here).
static int upload_freqs(sbr_ctx *ctx, const double *k, int nk, double gamma, int B)
{
    std::vector<double> k2(nk), gp(B + 1);
    for (int f = 0; f < nk; ++f) k2[f] = k[f] / M_PI;   // phase 2kR in turns = (k/pi) R
    // equally spaced wavenumbers (a linspace frequency sweep) enable the
    // rotation recurrence of k_po
    ctx->dkturn = 0.0;
    if (nk > 1) {
        const double dk = (k[nk - 1] - k[0]) / (nk - 1);
        bool uniform = dk != 0.0;
        for (int f = 0; f < nk && uniform; ++f)
            uniform = std::fabs(k[f] - (k[0] + f * dk)) <= 1e-13 * std::fabs(k[f]);
        if (uniform) ctx->dkturn = dk / M_PI;
    }
    for (int b = 0; b <= B; ++b) gp[b] = pow(gamma, (double)b);
    CUDA_TRY(ctx->k2.reserve(nk));
    CUDA_TRY(ctx->gpow.reserve(B + 1));
    CUDA_TRY(cudaMemcpyAsync(ctx->k2.p, k2.data(), 8 * nk, cudaMemcpyHostToDevice, ctx->stream));
    CUDA_TRY(cudaMemcpyAsync(ctx->gpow.p, gp.data(), 8 * (B + 1), cudaMemcpyHostToDevice,
                             ctx->stream));
    return SBR_OK;
}

// Runs the batched trace -> PO -> segment pipeline over `units` (all on
// ctx->stream); writes segment partials into seg_dev and diagnostics into
// diag_dev (both pre-zeroed by the caller).
static int run_units(sbr_ctx *ctx, const sbr_bvh *bvh, const std::vector<UnitDev> &all_units,
                     const std::vector<int64_t> &seg_base, int nk, const TraceCfg &cfg,
                     double2 *seg_dev, int64_t *diag_dev)
{
    cudaStream_t st = ctx->stream;
    int64_t budget = slot_budget();
    const int ngrids = (int)seg_base.size() - 1;
    const bool refmode = use_ref(ctx, bvh);
    const bool raster = !refmode && raster_primary(bvh->mesh->ntri, ngrids);
    std::vector<int64_t> seg_slot;
    std::vector<int> bgrids;
    if (raster) {
        CUDA_TRY(ctx->seg_base.reserve(seg_base.size()));
        CUDA_TRY(cudaMemcpyAsync(ctx->seg_base.p, seg_base.data(), 8 * seg_base.size(),
                                 cudaMemcpyHostToDevice, st));
        CUDA_TRY(ctx->seg_slot.reserve(seg_base[ngrids]));
        CUDA_TRY(ctx->bgrids.reserve(ngrids));
    }
    size_t u0 = 0;
    std::vector<UnitDev> batch;
    while (u0 < all_units.size()) {
        batch.clear();
        int64_t slots = 0;
        size_t u1 = u0;
        while (u1 < all_units.size()) {
            UnitDev u = all_units[u1];
            int64_t need = round_chunk(u.ray_end - u.ray_begin);
            if (!batch.empty() && (slots + need > budget || (int64_t)batch.size() >= kMaxBatchUnits))
                break;   // work-list entries hold the unit index in 20 bits
            u.slot_base = slots;
            slots += need;
            batch.push_back(u);
            ++u1;
        }
        {   // device memory for the batch; on exhaustion retry with half the slots
            const void *before = ctx->slots.p;
            cudaError_t e = ctx->slots.reserve(slots);
            if (ctx->slots.p != before) ctx->clean_slots = 0;   // fresh memory
            if (e == cudaSuccess && raster) e = ctx->worklist.reserve(slots);
            if (e == cudaSuccess && raster) e = ctx->hitmap.reserve((slots + 31) / 32);
            if (e == cudaSuccess && raster) e = ctx->chunk_hits.reserve(slots / kChunk);
            if (e == cudaSuccess) e = ctx->chunk_part.reserve((size_t)(slots / kChunk) * nk);
            if (e == cudaErrorMemoryAllocation && budget > ((int64_t)1 << 22)) {
                cudaGetLastError();
                ctx->slots.release();
                ctx->worklist.release();
                ctx->hitmap.release();
                ctx->chunk_hits.release();
                ctx->chunk_part.release();
                ctx->clean_slots = 0;
                budget = round_chunk(budget / 2);
                continue;
            }
            CUDA_TRY(e);
        }
        CUDA_TRY(ctx->units.reserve(batch.size()));
        CUDA_TRY(cudaMemcpyAsync(ctx->units.p, batch.data(), sizeof(UnitDev) * batch.size(),
                                 cudaMemcpyHostToDevice, st));
        CUDA_TRY(ctx->chunk_unit.reserve(slots / kChunk));
        CUDA_TRY(launch_chunk_units(ctx->units.p, (int)batch.size(), ctx->chunk_unit.p, st,
                                    ctx->stats()));
        if (ctx->profile) CUDA_TRY(cudaEventRecord(ctx->ev[0], st));
        // the batch's slots are all-ones after a list-mode PO; anything
        // else (BVH primary, reference order, an error) leaves them dirty
        static const bool force_memset = getenv("SBR_FORCE_MEMSET") != nullptr;  // A/B only
        const int64_t clean = force_memset ? 0 : ctx->clean_slots;
        ctx->clean_slots = 0;
        if (raster) {
            seg_slot.assign(seg_base[ngrids], kNoSlot);
            bgrids.clear();
            for (const UnitDev &u : batch) {
                seg_slot[u.seg_out] = u.slot_base - u.ray_begin;
                if (bgrids.empty() || bgrids.back() != u.grid) bgrids.push_back(u.grid);
            }
            CUDA_TRY(cudaMemcpyAsync(ctx->seg_slot.p, seg_slot.data(), 8 * seg_slot.size(),
                                     cudaMemcpyHostToDevice, st));
            CUDA_TRY(cudaMemcpyAsync(ctx->bgrids.p, bgrids.data(), 4 * bgrids.size(),
                                     cudaMemcpyHostToDevice, st));
            if (clean < slots)
                CUDA_TRY(cudaMemsetAsync(ctx->slots.p + clean, 0xff,
                                         sizeof(SlotRec) * (slots - clean), st));
            CUDA_TRY(cudaMemsetAsync(ctx->hitmap.p, 0, sizeof(unsigned) * ((slots + 31) / 32), st));
            RasterArgs ra = raster_args(bvh, ctx->grids.p, ctx->bgrids.p, (int)bgrids.size(),
                                        ctx->seg_base.p, ctx->seg_slot.p,
                                        reinterpret_cast<PrimHit *>(ctx->slots.p));
            ra.hitmap = ctx->hitmap.p;
            ra.counter = ctx->counter.p + 1;
            ra.stats = ctx->counter.p + 2;
            CUDA_TRY(attach_big_queue(ctx, ra, slots));
            for (int g : bgrids)       // a grid of the batch with a segment outside it
                for (int64_t q = seg_base[g]; q < seg_base[g + 1] && !ra.sparse; ++q)
                    ra.sparse = seg_slot[q] == kNoSlot;
            CUDA_TRY(launch_raster(ra, st, ctx->stats()));
        }
        if (ctx->profile) CUDA_TRY(cudaEventRecord(ctx->ev[4], st));
        if (raster) {
            CUDA_TRY(ctx->worklist.reserve(slots));
            CUDA_TRY(ctx->nwork.reserve(1));
            CUDA_TRY(launch_prim_compact(cfg, ctx->grids.p, ctx->units.p, (int)batch.size(),
                                         slots, ctx->slots.p, ctx->hitmap.p, ctx->chunk_unit.p,
                                         ctx->worklist.p, ctx->nwork.p, ctx->chunk_hits.p, st,
                                         ctx->stats()));
        }
        if (ctx->profile) CUDA_TRY(cudaEventRecord(ctx->ev[3], st));
        if (refmode) {
            const FullOut none{};
            CUDA_TRY(launch_trace_ref(ref_view(bvh), cfg, ctx->grids.p, nullptr, nullptr, slots,
                                      0, none, ctx->units.p, ctx->slots.p, (int)batch.size(), st,
                                      ctx->stats()));
        } else {
            CUDA_TRY(launch_trace_solve(cfg, ctx->grids.p, ctx->units.p, (int)batch.size(),
                                        slots, ctx->slots.p, ctx->counter.p, raster,
                                        raster ? ctx->worklist.p : nullptr,
                                        raster ? ctx->nwork.p : nullptr, st, ctx->stats()));
        }
        if (ctx->profile) CUDA_TRY(cudaEventRecord(ctx->ev[1], st));
        CUDA_TRY(launch_po(ctx->slots.p, ctx->units.p, (int)batch.size(),
                           raster ? ctx->worklist.p : nullptr,
                           raster ? ctx->chunk_hits.p : nullptr, slots / kChunk, ctx->k2.p, nk,
                           ctx->dkturn, ctx->gpow.p, cfg.max_bounces, ctx->chunk_part.p,
                           diag_dev, ctx->bad.p, ctx->counter.p + 5, ctx->chunk_unit.p, st,
                           ctx->stats()));
        if (ctx->profile) CUDA_TRY(cudaEventRecord(ctx->ev[2], st));
        CUDA_TRY(launch_seg_reduce(ctx->chunk_part.p, ctx->units.p, (int)batch.size(), nk,
                                   seg_dev, st, ctx->stats()));
        // the units buffer is rewritten by the next batch: keep batches ordered
        CUDA_TRY(cudaStreamSynchronize(st));
        // the trace kernel reset every hit slot it consumed: all-ones again
        if (raster) ctx->clean_slots = std::max(clean, slots);
        if (ctx->profile) {
            float a = 0.f, b = 0.f;
            float c = 0.f;
            float cc = 0.f;
            CUDA_TRY(cudaEventElapsedTime(&c, ctx->ev[0], ctx->ev[4]));
            CUDA_TRY(cudaEventElapsedTime(&cc, ctx->ev[4], ctx->ev[3]));
            ctx->compact_ms += cc;
            CUDA_TRY(cudaEventElapsedTime(&a, ctx->ev[3], ctx->ev[1]));
            CUDA_TRY(cudaEventElapsedTime(&b, ctx->ev[1], ctx->ev[2]));
            ctx->raster_ms += c;
            ctx->trace_ms += a;
            ctx->po_ms += b;
            ctx->trace_n += 1;
            ctx->po_n += 1;
        }
        u0 = u1;
    }
    return SBR_OK;
}

static int upload_grids(sbr_ctx *ctx, const sbr_grid *grids, int ngrids)
{
    std::vector<GridDev> g(ngrids);
    for (int i = 0; i < ngrids; ++i) {
        for (int a = 0; a < 3; ++a) {
            g[i].corner[a] = grids[i].corner[a]; g[i].u[a] = grids[i].u[a];
            g[i].v[a] = grids[i].v[a]; g[i].k[a] = grids[i].k[a];
        }
        g[i].spacing = grids[i].spacing;
        g[i].n_v = grids[i].n_v;
        g[i].n_rays = grids[i].n_u * grids[i].n_v;
        grid_derive(g[i]);
    }
    CUDA_TRY(ctx->grids.reserve(ngrids));
    CUDA_TRY(cudaMemcpyAsync(ctx->grids.p, g.data(), sizeof(GridDev) * ngrids,
                             cudaMemcpyHostToDevice, ctx->stream));
    return SBR_OK;
}

static int check_grids(const sbr_grid *grids, int ngrids)
{
    REQUIRE(grids && ngrids >= 1, "no grids");
    for (int g = 0; g < ngrids; ++g) {
        REQUIRE(grids[g].n_u >= 1 && grids[g].n_v >= 1, "grid %d: empty", g);
        REQUIRE(grids[g].spacing > 0.0 && grids[g].cell_area > 0.0, "grid %d: bad spacing", g);
    }
    return SBR_OK;
}

static int check_sampling(const sbr_grid *grids, int ngrids, const sbr_trace_params *p)
{
    if (p->allow_aliasing || !(p->lambda_min > 0.0)) return SBR_OK;
    const double limit = p->lambda_min / p->sampling_factor;
    for (int g = 0; g < ngrids; ++g)
        REQUIRE(grids[g].spacing <= limit,
                "ray spacing %g exceeds wavelength/%g = %g (ratio %.3f); pass allow_aliasing "
                "to override",
                grids[g].spacing, p->sampling_factor, limit,
                grids[g].spacing * p->sampling_factor / p->lambda_min);
    return SBR_OK;
}

static int solve_shard_locked(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                              const sbr_grid *grids, int32_t ngrids,
                              const sbr_trace_params *params, const double *k, int32_t nk,
                              double gamma, int32_t count_trapped, int32_t rank, int32_t nranks,
                              int32_t shard_mode, double2 *seg_dev, int64_t *diag_dev)
{
    cudaStream_t st = ctx->stream;
    std::vector<int64_t> seg_base(ngrids + 1);
    sbr_segment_layout(grids, ngrids, seg_base.data());
    const int B = params->max_bounces;
    const int64_t dstride = 3 + B + 1;
    CUDA_TRY(cudaMemsetAsync(seg_dev, 0, sizeof(double2) * seg_base[ngrids] * nk, st));
    CUDA_TRY(cudaMemsetAsync(diag_dev, 0, sizeof(int64_t) * ngrids * dstride, st));
    CUDA_TRY(cudaMemsetAsync(ctx->err_flag.p, 0, sizeof(unsigned int), st));
    CUDA_TRY(cudaMemsetAsync(ctx->bad.p, 0xff, sizeof(unsigned long long), st));
    if (int rc = upload_grids(ctx, grids, ngrids)) return rc;
    if (int rc = upload_freqs(ctx, k, nk, gamma, B)) return rc;
    std::vector<UnitDev> units;
    int64_t uidx = 0;
    for (int g = 0; g < ngrids; ++g) {
        const int64_t n = grids[g].n_u * grids[g].n_v;
        for (int64_t s = 0; s < seg_base[g + 1] - seg_base[g]; ++s, ++uidx) {
            const int owner = shard_mode == 0 ? (g % nranks) : (int)(uidx % nranks);
            if (owner != rank) continue;
            UnitDev u;
            u.grid = g;
            u.seg = (int)s;
            u.ray_begin = s * kSegRays;
            u.ray_end = std::min(n, (s + 1) * kSegRays);
            u.slot_base = 0;
            u.seg_out = seg_base[g] + s;
            units.push_back(u);
        }
    }
    TraceCfg cfg = make_cfg(bvh, params, ctx);
    cfg.count_trapped = count_trapped;
    if (int rc = run_units(ctx, bvh, units, seg_base, nk, cfg, seg_dev, diag_dev)) return rc;
    unsigned int flag = 0;
    unsigned long long bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&flag, ctx->err_flag.p, sizeof(flag), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&bad, ctx->bad.p, sizeof(bad), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (flag & 1u) return fail(SBR_EINVAL, "device launcher: ray spacing violates the sampling rule");
    if (bad != ~0ULL)
        return fail(SBR_ENUMERIC, "non-finite contribution at record index %llu", bad);
    return SBR_OK;
}

static int validate_solve(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                          const sbr_grid *grids, int32_t ngrids, const sbr_trace_params *params,
                          const double *k, int32_t nk, double gamma)
{
    if (int rc = check_pair(ctx, mesh, bvh)) return rc;
    if (int rc = check_params(params)) return rc;
    if (int rc = check_grids(grids, ngrids)) return rc;
    REQUIRE(k && nk >= 1 && nk <= 65535, "need 1..65535 wavenumbers");
    for (int f = 0; f < nk; ++f) REQUIRE(k[f] > 0.0 && std::isfinite(k[f]), "bad wavenumber");
    REQUIRE(std::fabs(gamma) <= 1.0, "|gamma| must be <= 1");
    if (int rc = check_ref_mode(ctx, bvh)) return rc;
    return check_sampling(grids, ngrids, params);
}

extern "C" int sbr_solve_shard(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                               const sbr_grid *grids, int32_t ngrids,
                               const sbr_trace_params *params, const double *k, int32_t nk,
                               double gamma, int32_t count_trapped, int32_t rank,
                               int32_t nranks, int32_t shard_mode, double *seg_dev,
                               int64_t *diag_dev)
{
    if (int rc = validate_solve(ctx, mesh, bvh, grids, ngrids, params, k, nk, gamma)) return rc;
    REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank %d / %d", rank, nranks);
    REQUIRE(shard_mode == 0 || shard_mode == 1, "bad shard_mode");
    REQUIRE(seg_dev && diag_dev, "NULL device buffers");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    return solve_shard_locked(ctx, mesh, bvh, grids, ngrids, params, k, nk, gamma, count_trapped,
                              rank, nranks, shard_mode, (double2 *)seg_dev, diag_dev);
}

static int finalize_locked(sbr_ctx *ctx, const sbr_grid *grids, int32_t ngrids, const double *k,
                           int32_t nk, int32_t B, const double2 *seg_dev, const int64_t *diag_dev,
                           double *amp, sbr_diag *diag)
{
    cudaStream_t st = ctx->stream;
    std::vector<int64_t> seg_base(ngrids + 1);
    sbr_segment_layout(grids, ngrids, seg_base.data());
    std::vector<double> scale((size_t)ngrids * nk);
    for (int g = 0; g < ngrids; ++g)
        for (int f = 0; f < nk; ++f)
            scale[(size_t)g * nk + f] = k[f] * grids[g].cell_area / (4.0 * M_PI);
    CUDA_TRY(ctx->seg_base.reserve(ngrids + 1));
    CUDA_TRY(ctx->scale.reserve(scale.size()));
    CUDA_TRY(ctx->amp.reserve(scale.size()));
    CUDA_TRY(cudaMemcpyAsync(ctx->seg_base.p, seg_base.data(), 8 * (ngrids + 1),
                             cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(ctx->scale.p, scale.data(), 8 * scale.size(), cudaMemcpyHostToDevice,
                             st));
    CUDA_TRY(launch_finalize(seg_dev, ctx->seg_base.p, ngrids, nk, ctx->scale.p, ctx->amp.p, st,
                             ctx->stats()));
    CUDA_TRY(cudaMemcpyAsync(amp, ctx->amp.p, sizeof(double2) * scale.size(),
                             cudaMemcpyDeviceToHost, st));
    const int64_t dstride = 3 + B + 1;
    std::vector<int64_t> dg((size_t)ngrids * dstride);
    CUDA_TRY(cudaMemcpyAsync(dg.data(), diag_dev, 8 * dg.size(), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (diag) {
        for (int g = 0; g < ngrids; ++g) {
            const int64_t *row = dg.data() + (size_t)g * dstride;
            if (diag->valid_rays) diag->valid_rays[g] = row[0];
            if (diag->queries) diag->queries[g] = row[1];
            if (diag->max_bounce) diag->max_bounce[g] = (int32_t)row[2];
            if (diag->hist)
                for (int b = 0; b <= B; ++b) diag->hist[(size_t)g * (B + 1) + b] = row[3 + b];
        }
    }
    return SBR_OK;
}

// ---------------------------------------------------------------------------
// one-collective sharding: packed reduce buffer + NCCL (replaces the paper's
// MPI layer; the reference's worker pool over angles,
// sweep.py:327-349)
// ---------------------------------------------------------------------------
static int64_t packed_count(const sbr_grid *grids, int32_t ngrids, int32_t nk, int32_t B,
                            int32_t nranks)
{
    std::vector<int64_t> seg_base(ngrids + 1);
    sbr_segment_layout(grids, ngrids, seg_base.data());
    return seg_base[ngrids] * nk * 2 + (int64_t)ngrids * (3 + B + 1 + nranks);
}

extern "C" int sbr_packed_layout(const sbr_grid *grids, int32_t ngrids, int32_t nk,
                                 int32_t max_bounces, int32_t nranks, int64_t *count)
{
    REQUIRE(grids && count && ngrids >= 1 && nk >= 1 && max_bounces >= 1 && nranks >= 1,
            "bad arguments");
    *count = packed_count(grids, ngrids, nk, max_bounces, nranks);
    return SBR_OK;
}

extern "C" int sbr_solve_shard_packed(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                                      const sbr_grid *grids, int32_t ngrids,
                                      const sbr_trace_params *params, const double *k,
                                      int32_t nk, double gamma, int32_t count_trapped,
                                      int32_t rank, int32_t nranks, int32_t shard_mode,
                                      double *buf_dev)
{
    if (int rc = validate_solve(ctx, mesh, bvh, grids, ngrids, params, k, nk, gamma)) return rc;
    REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank %d / %d", rank, nranks);
    REQUIRE(shard_mode == 0 || shard_mode == 1, "bad shard_mode");
    REQUIRE(buf_dev, "NULL device buffer");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    const int B = params->max_bounces, stride = 3 + B + 1;
    std::vector<int64_t> seg_base(ngrids + 1);
    sbr_segment_layout(grids, ngrids, seg_base.data());
    CUDA_TRY(ctx->diag.reserve((size_t)ngrids * stride));
    if (int rc = solve_shard_locked(ctx, mesh, bvh, grids, ngrids, params, k, nk, gamma,
                                    count_trapped, rank, nranks, shard_mode, (double2 *)buf_dev,
                                    ctx->diag.p))
        return rc;
    CUDA_TRY(launch_pack_diag(ctx->diag.p, ngrids, stride, nranks, rank,
                              buf_dev + seg_base[ngrids] * nk * 2, ctx->stream, ctx->stats()));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return SBR_OK;
}

static int finalize_packed_locked(sbr_ctx *ctx, const sbr_grid *grids, int32_t ngrids,
                                  const double *k, int32_t nk, int32_t B, int32_t nranks,
                                  const double *buf_dev, double *amp, sbr_diag *diag)
{
    const int stride = 3 + B + 1;
    std::vector<int64_t> seg_base(ngrids + 1);
    sbr_segment_layout(grids, ngrids, seg_base.data());
    DevBuf<int64_t> dg((size_t)ngrids * stride);
    CUDA_TRY(dg.status());
    CUDA_TRY(launch_unpack_diag(buf_dev + seg_base[ngrids] * nk * 2, ngrids, stride, nranks,
                                dg.p, ctx->stream, ctx->stats()));
    return finalize_locked(ctx, grids, ngrids, k, nk, B, (const double2 *)buf_dev, dg.p, amp,
                           diag);
}

extern "C" int sbr_finalize_packed(sbr_ctx *ctx, const sbr_grid *grids, int32_t ngrids,
                                   const double *k, int32_t nk, int32_t max_bounces,
                                   int32_t nranks, const double *buf_dev, double *amp,
                                   sbr_diag *diag)
{
    REQUIRE(ctx && amp && buf_dev, "NULL argument");
    if (int rc = check_grids(grids, ngrids)) return rc;
    REQUIRE(k && nk >= 1 && nk <= 65535, "need 1..65535 wavenumbers");
    REQUIRE(max_bounces >= 1 && nranks >= 1, "bad max_bounces / nranks");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    return finalize_packed_locked(ctx, grids, ngrids, k, nk, max_bounces, nranks, buf_dev, amp,
                                  diag);
}

// ---- NCCL, loaded at run time (no link-time dependency: the library still
// loads on a host without NCCL; only the comm entry points need it).  The
// first libnccl.so.2 already in the process (e.g. torch's) wins, else the
// system's; SBR_NCCL_LIB names another.
struct NcclApi {
    bool tried = false;
    void *h = nullptr;
    std::string why;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclReduce) reduce = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    decltype(&ncclGetVersion) version = nullptr;
};
static std::mutex g_nccl_mu;
static NcclApi g_nccl;

static const NcclApi *nccl_api()
{
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.tried) return g_nccl.h ? &g_nccl : nullptr;
    g_nccl.tried = true;
    const char *env = getenv("SBR_NCCL_LIB");
    const char *cands[] = {env, "libnccl.so.2", "libnccl.so",
                           "/usr/lib/x86_64-linux-gnu/libnccl.so.2"};
    for (const char *c : cands) {
        if (!c) continue;
        g_nccl.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
        if (g_nccl.h) break;
        g_nccl.why = dlerror();
    }
    if (!g_nccl.h) return nullptr;
#define SBR_NCCL_SYM(f, n) g_nccl.f = (decltype(g_nccl.f))dlsym(g_nccl.h, n)
    SBR_NCCL_SYM(get_unique_id, "ncclGetUniqueId");
    SBR_NCCL_SYM(init_rank, "ncclCommInitRank");
    SBR_NCCL_SYM(destroy, "ncclCommDestroy");
    SBR_NCCL_SYM(reduce, "ncclReduce");
    SBR_NCCL_SYM(error_string, "ncclGetErrorString");
    SBR_NCCL_SYM(version, "ncclGetVersion");
#undef SBR_NCCL_SYM
    if (!(g_nccl.get_unique_id && g_nccl.init_rank && g_nccl.destroy && g_nccl.reduce &&
          g_nccl.error_string && g_nccl.version)) {
        g_nccl.why = "libnccl lacks a required symbol";
        dlclose(g_nccl.h);
        g_nccl.h = nullptr;
        return nullptr;
    }
    return &g_nccl;
}

#define NCCL_TRY(api, x)                                                               \
    do {                                                                               \
        ncclResult_t r_ = (x);                                                         \
        if (r_ != ncclSuccess)                                                         \
            return fail(SBR_ENCCL, "%s failed: %s", #x, (api)->error_string(r_));      \
    } while (0)

extern "C" int sbr_comm_version(int32_t *version)
{
    REQUIRE(version, "NULL argument");
    const NcclApi *api = nccl_api();
    if (!api) return fail(SBR_ENCCL, "NCCL unavailable: %s", g_nccl.why.c_str());
    int v = 0;
    NCCL_TRY(api, api->version(&v));
    *version = v;
    return SBR_OK;
}

extern "C" int sbr_comm_unique_id(uint8_t id[128])
{
    REQUIRE(id, "NULL argument");
    const NcclApi *api = nccl_api();
    if (!api) return fail(SBR_ENCCL, "NCCL unavailable: %s", g_nccl.why.c_str());
    ncclUniqueId u;
    NCCL_TRY(api, api->get_unique_id(&u));
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    memcpy(id, &u, 128);
    return SBR_OK;
}

extern "C" int sbr_comm_init(sbr_ctx *ctx, int32_t nranks, int32_t rank, const uint8_t id[128])
{
    REQUIRE(ctx && id, "NULL argument");
    REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank %d / %d", rank, nranks);
    const NcclApi *api = nccl_api();
    if (!api) return fail(SBR_ENCCL, "NCCL unavailable: %s", g_nccl.why.c_str());
    std::lock_guard<std::mutex> lk(ctx->mu);
    REQUIRE(!ctx->comm, "context already has a communicator");
    if (int rc = set_device(ctx)) return rc;
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclComm_t c = nullptr;
    NCCL_TRY(api, api->init_rank(&c, nranks, u, rank));
    ctx->comm = c;
    ctx->comm_rank = rank;
    ctx->comm_size = nranks;
    return SBR_OK;
}

extern "C" int sbr_comm_destroy(sbr_ctx *ctx)
{
    REQUIRE(ctx, "ctx is NULL");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (!ctx->comm) return SBR_OK;
    const NcclApi *api = nccl_api();
    if (int rc = set_device(ctx)) return rc;
    ncclComm_t c = (ncclComm_t)ctx->comm;
    ctx->comm = nullptr;
    if (api) NCCL_TRY(api, api->destroy(c));
    return SBR_OK;
}

static int reduce_locked(sbr_ctx *ctx, double *buf_dev, int64_t count, int32_t root)
{
    REQUIRE(ctx->comm, "no communicator: call sbr_comm_init first");
    REQUIRE(root >= 0 && root < ctx->comm_size, "bad root %d", root);
    const NcclApi *api = nccl_api();
    NCCL_TRY(api, api->reduce(buf_dev, buf_dev, (size_t)count, ncclFloat64, ncclSum, root,
                              (ncclComm_t)ctx->comm, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return SBR_OK;
}

extern "C" int sbr_reduce_sum_f64(sbr_ctx *ctx, double *buf_dev, int64_t count, int32_t root)
{
    REQUIRE(ctx && (buf_dev || count == 0) && count >= 0, "bad arguments");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    return reduce_locked(ctx, buf_dev, count, root);
}

extern "C" int sbr_solve_distributed(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                                     const sbr_grid *grids, int32_t ngrids,
                                     const sbr_trace_params *params, const double *k,
                                     int32_t nk, double gamma, int32_t count_trapped,
                                     int32_t shard_mode, int32_t root, double *amp,
                                     sbr_diag *diag)
{
    REQUIRE(ctx && ctx->comm, "no communicator: call sbr_comm_init first");
    if (int rc = validate_solve(ctx, mesh, bvh, grids, ngrids, params, k, nk, gamma)) return rc;
    const int64_t count = packed_count(grids, ngrids, nk, params->max_bounces, ctx->comm_size);
    DevBuf<double> buf;
    {
        std::lock_guard<std::mutex> lk(ctx->mu);
        if (int rc = set_device(ctx)) return rc;
        CUDA_TRY(buf.alloc((size_t)count));
    }
    if (int rc = sbr_solve_shard_packed(ctx, mesh, bvh, grids, ngrids, params, k, nk, gamma,
                                        count_trapped, ctx->comm_rank, ctx->comm_size,
                                        shard_mode, buf.p))
        return rc;
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = reduce_locked(ctx, buf.p, count, root)) return rc;
    if (ctx->comm_rank != root) return SBR_OK;
    REQUIRE(amp, "NULL amp on the root");
    return finalize_packed_locked(ctx, grids, ngrids, k, nk, params->max_bounces,
                                  ctx->comm_size, buf.p, amp, diag);
}

extern "C" int sbr_finalize(sbr_ctx *ctx, const sbr_grid *grids, int32_t ngrids,
                            const double *k, int32_t nk, int32_t max_bounces,
                            const double *seg_dev, const int64_t *diag_dev, double *amp,
                            sbr_diag *diag)
{
    REQUIRE(ctx && amp && seg_dev && diag_dev, "NULL argument");
    if (int rc = check_grids(grids, ngrids)) return rc;
    REQUIRE(k && nk >= 1 && nk <= 65535, "need 1..65535 wavenumbers");
    REQUIRE(max_bounces >= 1, "max_bounces must be >= 1");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    return finalize_locked(ctx, grids, ngrids, k, nk, max_bounces, (const double2 *)seg_dev,
                           diag_dev, amp, diag);
}

extern "C" int sbr_solve(sbr_ctx *ctx, const sbr_mesh *mesh, const sbr_bvh *bvh,
                         const sbr_grid *grids, int32_t ngrids, const sbr_trace_params *params,
                         const double *k, int32_t nk, double gamma, int32_t count_trapped,
                         double *amp, sbr_diag *diag)
{
    if (int rc = validate_solve(ctx, mesh, bvh, grids, ngrids, params, k, nk, gamma)) return rc;
    REQUIRE(amp, "amp is NULL");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    std::vector<int64_t> seg_base(ngrids + 1);
    sbr_segment_layout(grids, ngrids, seg_base.data());
    const int B = params->max_bounces;
    CUDA_TRY(ctx->seg_part.reserve((size_t)seg_base[ngrids] * nk));
    CUDA_TRY(ctx->diag.reserve((size_t)ngrids * (3 + B + 1)));
    if (int rc = solve_shard_locked(ctx, mesh, bvh, grids, ngrids, params, k, nk, gamma,
                                    count_trapped, 0, 1, 0, ctx->seg_part.p, ctx->diag.p))
        return rc;
    return finalize_locked(ctx, grids, ngrids, k, nk, B, ctx->seg_part.p, ctx->diag.p, amp, diag);
}

extern "C" int sbr_accumulate(sbr_ctx *ctx, const uint8_t *valid, const double *normal0,
                              const double *path, const int32_t *bounces, const uint8_t *escaped,
                              int64_t n, const double k_inc[3], const double *k, int32_t nk,
                              double cell_area, double gamma, int32_t count_trapped, double *amp,
                              int64_t *bad_index)
{
    REQUIRE(ctx && amp && k_inc && k && nk >= 1, "NULL argument");
    REQUIRE(nk <= 65535, "at most 65535 wavenumbers");
    REQUIRE(n >= 0, "negative record count");
    REQUIRE(cell_area > 0.0, "cell_area must be positive");
    REQUIRE(std::fabs(gamma) <= 1.0, "|gamma| must be <= 1");
    if (bad_index) *bad_index = -1;
    if (n == 0) {
        for (int f = 0; f < 2 * nk; ++f) amp[f] = 0.0;
        return SBR_OK;
    }
    REQUIRE(valid && normal0 && path && bounces && escaped, "NULL records");
    int maxb = 0;
    for (int64_t r = 0; r < n; ++r) {
        REQUIRE(bounces[r] >= 0 && bounces[r] <= 0xffff, "bounce count out of range at %lld",
                (long long)r);
        maxb = std::max(maxb, (int)bounces[r]);
    }
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    cudaStream_t st = ctx->stream;
    const int64_t nseg = seg_count(n);
    const int64_t n_slots = nseg * kSegRays;  // one unit per segment
    std::vector<UnitDev> units(nseg);
    int64_t slots_used = 0;
    for (int64_t s = 0; s < nseg; ++s) {
        units[s].grid = 0;
        units[s].seg = (int)s;
        units[s].ray_begin = s * kSegRays;
        units[s].ray_end = std::min(n, (s + 1) * kSegRays);
        units[s].slot_base = s * kSegRays;
        units[s].seg_out = s;
        slots_used = units[s].slot_base + round_chunk(units[s].ray_end - units[s].ray_begin);
    }
    (void)n_slots;
    DevBuf<uint8_t> dv(n), de(n);
    DevBuf<double> dn(3 * n), dp(n);
    DevBuf<int32_t> db(n);
    CUDA_TRY(dv.status()); CUDA_TRY(de.status()); CUDA_TRY(dn.status()); CUDA_TRY(dp.status());
    CUDA_TRY(db.status());
    CUDA_TRY(cudaMemcpyAsync(dv.p, valid, n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(de.p, escaped, n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dn.p, normal0, 24 * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dp.p, path, 8 * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(db.p, bounces, 4 * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx->slots.reserve(slots_used));
    CUDA_TRY(ctx->units.reserve(nseg));
    CUDA_TRY(ctx->chunk_part.reserve((size_t)(slots_used / kChunk) * nk));
    CUDA_TRY(ctx->seg_part.reserve((size_t)nseg * nk));
    CUDA_TRY(ctx->diag.reserve(3 + maxb + 1));
    CUDA_TRY(cudaMemsetAsync(ctx->diag.p, 0, 8 * (3 + maxb + 1), st));
    CUDA_TRY(cudaMemsetAsync(ctx->bad.p, 0xff, sizeof(unsigned long long), st));
    CUDA_TRY(cudaMemcpyAsync(ctx->units.p, units.data(), sizeof(UnitDev) * nseg,
                             cudaMemcpyHostToDevice, st));
    if (int rc = upload_freqs(ctx, k, nk, gamma, maxb)) return rc;
    ctx->clean_slots = 0;   // the records overwrite the raster's all-ones slots
    CUDA_TRY(launch_records_to_slots(dv.p, dn.p, dp.p, db.p, de.p, n, k_inc[0], k_inc[1],
                                     k_inc[2], count_trapped, slots_used, ctx->slots.p, st,
                                     ctx->stats()));
    CUDA_TRY(launch_po(ctx->slots.p, ctx->units.p, (int)nseg, nullptr, nullptr,
                       slots_used / kChunk, ctx->k2.p, nk,
                       ctx->dkturn, ctx->gpow.p, maxb, ctx->chunk_part.p, ctx->diag.p, ctx->bad.p,
                       ctx->counter.p + 5, nullptr, st, ctx->stats()));
    CUDA_TRY(launch_seg_reduce(ctx->chunk_part.p, ctx->units.p, (int)nseg, nk, ctx->seg_part.p, st,
                               ctx->stats()));
    sbr_grid g;
    memset(&g, 0, sizeof(g));
    g.n_u = n;
    g.n_v = 1;
    g.spacing = 1.0;
    g.cell_area = cell_area;
    unsigned long long bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&bad, ctx->bad.p, sizeof(bad), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (bad != ~0ULL) {
        if (bad_index) *bad_index = (int64_t)bad;
        return fail(SBR_ENUMERIC, "non-finite contribution at record index %llu", bad);
    }
    return finalize_locked(ctx, &g, 1, k, nk, maxb, ctx->seg_part.p, ctx->diag.p, amp, nullptr);
}

// ---------------------------------------------------------------------------
// scalar predicates
// ---------------------------------------------------------------------------
extern "C" int sbr_tri_hit_pairs(sbr_ctx *ctx, const double *v0, const double *v1,
                                 const double *v2, const double *origins, const double *dirs,
                                 int64_t n, double t_min, double t_max, int32_t single,
                                 double *t)
{
    REQUIRE(ctx, "ctx is NULL");
    REQUIRE(n >= 0, "negative count");
    if (n == 0) return SBR_OK;
    REQUIRE(v0 && v1 && v2 && origins && dirs && t, "NULL argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    cudaStream_t st = ctx->stream;
    DevBuf<double> a(3 * n), b(3 * n), c(3 * n), o(3 * n), d(3 * n), tt(n);
    CUDA_TRY(a.status()); CUDA_TRY(b.status()); CUDA_TRY(c.status());
    CUDA_TRY(o.status()); CUDA_TRY(d.status()); CUDA_TRY(tt.status());
    CUDA_TRY(cudaMemcpyAsync(a.p, v0, 24 * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(b.p, v1, 24 * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(c.p, v2, 24 * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(o.p, origins, 24 * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(d.p, dirs, 24 * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(launch_tri_pairs(a.p, b.p, c.p, o.p, d.p, n, t_min, t_max, single, tt.p, st,
                              ctx->stats()));
    CUDA_TRY(cudaMemcpyAsync(t, tt.p, 8 * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return SBR_OK;
}

extern "C" int sbr_aabb_hit_pairs(sbr_ctx *ctx, const double *box_min, const double *box_max,
                                  const double *origins, const double *dir_inv, int64_t n,
                                  double t_max, uint8_t *hit, double *entry)
{
    REQUIRE(ctx, "ctx is NULL");
    REQUIRE(n >= 0, "negative count");
    if (n == 0) return SBR_OK;
    REQUIRE(box_min && box_max && origins && dir_inv && hit && entry, "NULL argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    cudaStream_t st = ctx->stream;
    DevBuf<double> lo(3 * n), hi(3 * n), o(3 * n), iv(3 * n), en(n);
    DevBuf<uint8_t> h(n);
    CUDA_TRY(lo.status()); CUDA_TRY(hi.status()); CUDA_TRY(o.status());
    CUDA_TRY(iv.status()); CUDA_TRY(en.status()); CUDA_TRY(h.status());
    CUDA_TRY(cudaMemcpyAsync(lo.p, box_min, 24 * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(hi.p, box_max, 24 * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(o.p, origins, 24 * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(iv.p, dir_inv, 24 * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(launch_box_pairs(lo.p, hi.p, o.p, iv.p, n, t_max, h.p, en.p, st, ctx->stats()));
    CUDA_TRY(cudaMemcpyAsync(hit, h.p, n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(entry, en.p, 8 * n, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return SBR_OK;
}

// ---------------------------------------------------------------------------
// instrumentation
// ---------------------------------------------------------------------------
extern "C" int sbr_ctx_profile(sbr_ctx *ctx, int32_t enable)
{
    REQUIRE(ctx, "ctx is NULL");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    if (enable && !ctx->ev[0])
        for (auto &e : ctx->ev) CUDA_TRY(cudaEventCreate(&e));
    ctx->profile = enable != 0;
    ctx->trace_ms = ctx->po_ms = ctx->raster_ms = ctx->compact_ms = 0.0;
    ctx->trace_n = ctx->po_n = 0;
    return SBR_OK;
}

extern "C" int sbr_probe_l2_bandwidth(sbr_ctx *ctx, int64_t bytes, int32_t reps, double *gbs)
{
    REQUIRE(ctx && gbs && bytes >= (1 << 20) && reps >= 1, "bad arguments");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    CUDA_TRY(probe_l2_read(bytes, reps, ctx->num_sms, ctx->stream, gbs));
    return SBR_OK;
}

// Instrumented builds (-DSBR_TRACE_STATS) accumulate lane-state counters in
// counter[8..31]; this reads and clears them (all zero in normal builds).
static std::atomic<int64_t> g_live_allocs{0}, g_live_bytes{0};

void sbr::count_alloc(int64_t bytes)
{
    g_live_allocs += bytes >= 0 ? 1 : -1;
    g_live_bytes += bytes;
}

extern "C" int sbr_debug_live_allocations(int64_t *count, int64_t *bytes)
{
    REQUIRE(count && bytes, "NULL argument");
    *count = g_live_allocs.load();
    *bytes = g_live_bytes.load();
    return SBR_OK;
}

extern "C" int sbr_ctx_debug_counters(sbr_ctx *ctx, int64_t *out, int32_t n)
{
    REQUIRE(ctx && out && n >= 0 && n <= 24, "bad arguments");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    CUDA_TRY(cudaMemcpyAsync(out, ctx->counter.p + 8, sizeof(int64_t) * n, cudaMemcpyDeviceToHost,
                             ctx->stream));
    CUDA_TRY(cudaMemsetAsync(ctx->counter.p + 8, 0, sizeof(int64_t) * 24, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return SBR_OK;
}

extern "C" int sbr_ctx_raster_stats(sbr_ctx *ctx, double *raster_ms)
{
    REQUIRE(ctx && raster_ms, "NULL argument");
    *raster_ms = ctx->raster_ms;
    return SBR_OK;
}

extern "C" int sbr_ctx_raster_counters(sbr_ctx *ctx, int64_t out[3])
{
    REQUIRE(ctx && out, "NULL argument");
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (int rc = set_device(ctx)) return rc;
    CUDA_TRY(cudaMemcpyAsync(out, ctx->counter.p + 2, 3 * sizeof(int64_t), cudaMemcpyDeviceToHost,
                             ctx->stream));
    CUDA_TRY(cudaMemsetAsync(ctx->counter.p + 2, 0, 3 * sizeof(int64_t), ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return SBR_OK;
}

extern "C" int sbr_ctx_stage_ms(sbr_ctx *ctx, double ms[4])
{
    REQUIRE(ctx && ms, "NULL argument");
    ms[0] = ctx->raster_ms;
    ms[1] = ctx->compact_ms;
    ms[2] = ctx->trace_ms;
    ms[3] = ctx->po_ms;
    return SBR_OK;
}

extern "C" int sbr_ctx_kernel_stats(sbr_ctx *ctx, double *trace_ms, int64_t *trace_launches,
                                    double *po_ms, int64_t *po_launches)
{
    REQUIRE(ctx, "ctx is NULL");
    if (trace_ms) *trace_ms = ctx->trace_ms;
    if (trace_launches) *trace_launches = ctx->trace_n;
    if (po_ms) *po_ms = ctx->po_ms;
    if (po_launches) *po_launches = ctx->po_n;
    return SBR_OK;
}
