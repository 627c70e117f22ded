// pipeline.cu -- the hot path: ray launch + multi-bounce traversal,
// warp-ballot compaction + physical-optics integral, deterministic reduce.
//
//   k_trace_persistent (trace_persistent.cuh) persistent warps with per-lane
//                  ray refill; each lane computes its ray origin on the fly
//                  from the grid scalars (transport.py:339-345, no launch
//                  record is materialised), walks up to B bounces
//                  (transport.py:276-327) and stores a 16-byte SlotRec.
//   k_po           one block per 1024-slot chunk: coalesced SlotRec loads,
//                  warp __ballot_sync + popc + block scan compact the
//                  selected records (po.py:96-101) into shared memory in
//                  slot order, then evaluates (po.py:105-108)
//                    term_f = j k_f dA/4pi * 2 cos Gamma^N exp(-2j k_f R)
//                  for nk wavenumbers: phase in turns reduced exactly in
//                  FP64; FP64 sincospi + lane sums per wavenumber, or (a
//                  uniform sweep) SFU __sincosf anchors + FP32 rotations and
//                  lane sums; warp shuffle tree, fixed cross-warp order.
//   k_seg_reduce / k_finalize  fixed pairwise trees (po.py:59-80 shape)
//                  over chunk -> segment -> grid partials: results are
//                  bit-stable and independent of GPU count.
#include <cstdlib>

#include "pipeline.h"
#include "traverse.cuh"

namespace sbr {

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------


__device__ __forceinline__ int64_t warp_fetch(unsigned long long *counter)
{
    unsigned long long item = 0;
    if ((threadIdx.x & 31) == 0) item = atomicAdd(counter, 1ULL);
    return (int64_t)__shfl_sync(0xffffffffu, item, 0);
}

// ---------------------------------------------------------------------------
// trace kernels
// ---------------------------------------------------------------------------
constexpr int kTraceThreads = 128;

}  // namespace sbr
#include "trace_persistent.cuh"
namespace sbr {

template <int STORAGE>
__global__ void __launch_bounds__(kTraceThreads)
k_closest(BvhView B, const double *__restrict__ orig, const double *__restrict__ dirs,
          int64_t n, double t_min, double t_max, int64_t *__restrict__ tri,
          double *__restrict__ t_out, int64_t *__restrict__ visits_out)
{
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        double t = t_max;
        int visits = 0;
        int id;
        if (STORAGE == kSingle) {   // float32 mesh: the reference casts the rays too
            auto f = [](double x) { return (double)__double2float_rn(x); };
            id = closest_hit<STORAGE, false, true>(B, f(orig[3 * r]), f(orig[3 * r + 1]),
                                                   f(orig[3 * r + 2]), f(dirs[3 * r]),
                                                   f(dirs[3 * r + 1]), f(dirs[3 * r + 2]), t_min,
                                                   t, visits);
        } else {
            id = closest_hit<STORAGE, false>(B, orig[3 * r], orig[3 * r + 1], orig[3 * r + 2],
                                             dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2],
                                             t_min, t, visits);
        }
        tri[r] = id;
        t_out[r] = t;
        visits_out[r] = visits;
    }
}

// ---------------------------------------------------------------------------
// records -> slots (sbr_accumulate on host HitRecords)
// ---------------------------------------------------------------------------
__global__ void k_records_to_slots(const uint8_t *__restrict__ valid,
                                   const double *__restrict__ n0,
                                   const double *__restrict__ path,
                                   const int32_t *__restrict__ bounces,
                                   const uint8_t *__restrict__ escaped, int64_t n, double kx,
                                   double ky, double kz, int count_trapped, int64_t n_slots,
                                   SlotRec *__restrict__ slots)
{
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n_slots;
         r += (int64_t)gridDim.x * blockDim.x) {
        SlotRec rec;
        rec.R = 0.0; rec.cosv = 0.f; rec.meta = 0u;
        if (r < n) {
            bool v = valid[r] != 0, e = escaped[r] != 0;
            double c = -DA(DA(DM(n0[3 * r], kx), DM(n0[3 * r + 1], ky)), DM(n0[3 * r + 2], kz));
            bool sel = v && (e || count_trapped) && c > 0.0;
            int b = bounces[r];
            rec.R = path[r];
            rec.cosv = (float)c;
            rec.meta = ((uint32_t)b & kMetaBounceMask) | kMetaActive | (v ? kMetaValid : 0u) |
                       (e ? kMetaEscaped : 0u) | (sel ? kMetaSel : 0u);
        }
        slots[r] = rec;
    }
}

// ---------------------------------------------------------------------------
// compaction + PO
// ---------------------------------------------------------------------------
constexpr int kPoThreads = 256;
constexpr int kPoWarps = kPoThreads / 32;
constexpr int kPerThread = kChunk / kPoThreads;   // 4
constexpr int kMaxHist = 64;                      // bounce histogram bins in smem

// ROT: equally spaced wavenumbers, phases by rotation recurrence (FPT > 1)
template <int FPT, bool ROT>
__global__ void __launch_bounds__(kPoThreads)
k_po(SlotRec *__restrict__ slots, const UnitDev *__restrict__ units, int n_units,
     const uint4 *__restrict__ list, const uint2 *__restrict__ chunk_hits,
     const double *__restrict__ kturn, int nk, double dkturn, const double *__restrict__ gpow,
     int max_bounces,
     double2 *__restrict__ chunk_part, int64_t *__restrict__ diag,
     unsigned long long *__restrict__ bad)
{
    __shared__ double2 srec[kChunk];                 // compacted (R, w)
    __shared__ float2 srot[ROT ? kChunk : 1];        // per record: sincos of the k step
    __shared__ int wcount[kPerThread][kPoWarps];
    __shared__ int wbase[kPerThread][kPoWarps];
    __shared__ int s_total;
    // per-chunk counters fit 32 bits: native shared atomics (64-bit shared
    // atomics are CAS loops -- measured as the top PO stall)
    __shared__ unsigned int s_hist[kMaxHist];
    __shared__ unsigned int s_valid, s_queries, s_maxb;
    __shared__ double2 red[kPoWarps][FPT];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t chunk = blockIdx.x;
    const int64_t slot0 = chunk * kChunk;
    const int ui = find_unit(units, n_units, slot0);
    const UnitDev U = units[ui];
    const int nb = max_bounces + 1;
    const int64_t dstride = 3 + nb;

    if (tid < kMaxHist) s_hist[tid] = 0u;
    if (tid == 0) { s_valid = 0u; s_queries = 0u; s_maxb = 0u; }

    // ---- load + ballot ----
    // list mode (raster pass): only the chunk's primary hits are read -- the
    // records the trace kernel wrote over the chunk's run of the hit list,
    // in slot order, contiguous; the chunk's other real slots are primary
    // misses (one query, invalid, nothing to integrate), never touched
    uint2 run = make_uint2(0u, 0u);
    if (list) run = __ldg(&chunk_hits[chunk]);
    SlotRec rec[kPerThread];
    unsigned selmask = 0;
    unsigned long long my_q = 0;
    unsigned my_maxb = 0;
    int my_valid = 0;
#pragma unroll
    for (int q = 0; q < kPerThread; ++q) {
        const int e = q * kPoThreads + tid;
        SlotRec r;
        if (list) {
            if (e < (int)run.y) {
                r = reinterpret_cast<const SlotRec *>(list)[run.x + e];
            } else {
                r.R = 0.0; r.cosv = 0.f; r.meta = 0u;
            }
        } else {
            r = slots[slot0 + e];
            if (r.meta == kMissMeta) {   // primary miss left by k_prim_compact
                r.R = 0.0;
                r.cosv = 0.f;
                r.meta = kMetaActive | kMetaEscaped;
            }
        }
        rec[q] = r;
        const bool sel = (r.meta & kMetaSel) != 0;
        const unsigned bal = __ballot_sync(0xffffffffu, sel);
        if (lane == 0) wcount[q][warp] = __popc(bal);
        if (sel) selmask |= 1u << q;
        if (r.meta & kMetaActive) {
            const unsigned b = r.meta & kMetaBounceMask;
            my_q += b + 1;
            my_maxb = max(my_maxb, b);
        }
        if (r.meta & kMetaValid) ++my_valid;
    }
    __syncthreads();
    // exclusive scan over (q, warp) in slot order
    if (warp == 0) {
        int carry = 0;
        for (int base = 0; base < kPerThread * kPoWarps; base += 32) {
            const int idx = base + lane;
            const int v = idx < kPerThread * kPoWarps ? (&wcount[0][0])[idx] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (idx < kPerThread * kPoWarps) (&wbase[0][0])[idx] = carry + incl - v;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) s_total = carry;
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int q = 0; q < kPerThread; ++q) {
        const bool sel = (selmask >> q) & 1u;
        const unsigned bal = __ballot_sync(0xffffffffu, sel);
        if (sel) {
            const SlotRec r = rec[q];
            const int pos = wbase[q][warp] + __popc(bal & lt);
            const unsigned b = r.meta & kMetaBounceMask;
            const double w = 2.0 * (double)r.cosv * gpow[b];
            srec[pos] = make_double2(r.R, w);
            if (!isfinite(r.R) || !isfinite(w)) {
                const int64_t sl = list ? slot0 + ((r.meta >> kMetaOffShift) & (kChunk - 1))
                                        : slot0 + q * kPoThreads + tid;
                const int64_t ridx = U.ray_begin + (sl - U.slot_base);
                atomicMin(bad, (unsigned long long)ridx);
            }
        }
        {   // bounce histogram of valid rays: one atomic per distinct value
            const bool v = (rec[q].meta & kMetaValid) != 0;
            const unsigned b = v ? (rec[q].meta & kMetaBounceMask) : 0xffffffffu;
            const unsigned peers = __match_any_sync(0xffffffffu, b);
            if (v && lane == __ffs(peers) - 1) {
                if (b < (unsigned)kMaxHist) atomicAdd(&s_hist[b], (unsigned)__popc(peers));
                else if (diag)
                    atomicAdd((unsigned long long *)&diag[(int64_t)U.grid * dstride + 3 + b],
                              (unsigned long long)__popc(peers));
            }
        }
    }
    // diagnostics: warp reductions then one atomic per warp
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        my_q += __shfl_xor_sync(0xffffffffu, my_q, o);
        my_valid += __shfl_xor_sync(0xffffffffu, my_valid, o);
        my_maxb = max(my_maxb, __shfl_xor_sync(0xffffffffu, my_maxb, o));
    }
    if (lane == 0) {
        atomicAdd(&s_queries, (unsigned)my_q);
        atomicAdd(&s_valid, (unsigned)my_valid);
        atomicMax(&s_maxb, my_maxb);
    }
    if (list && tid == 0) {   // the chunk's primary misses: one query each
        const int64_t first_r = U.ray_begin + (slot0 - U.slot_base);
        int64_t real = U.ray_end - first_r;
        real = real < 0 ? 0 : (real > kChunk ? kChunk : real);
        atomicAdd(&s_queries, (unsigned)(real - (int64_t)run.y));
    }
    __syncthreads();
    if (diag) {
        int64_t *dg = diag + (int64_t)U.grid * dstride;
        if (tid == 0) {
            if (s_valid) atomicAdd((unsigned long long *)&dg[0], (unsigned long long)s_valid);
            atomicAdd((unsigned long long *)&dg[1], (unsigned long long)s_queries);
            atomicMax((unsigned long long *)&dg[2], (unsigned long long)s_maxb);
        }
        if (tid < nb && tid < kMaxHist && s_hist[tid])
            atomicAdd((unsigned long long *)&dg[3 + tid], (unsigned long long)s_hist[tid]);
    }

    // ---- PO terms ----
    const int M = s_total;
    if (ROT) {
        // the phase step between neighbouring wavenumbers is the same for
        // every frequency group: its SFU sincos once per record, shared by the
        // group warps (was once per record and group)
        for (int m = tid; m < M; m += kPoThreads) {
            const double dt = dkturn * srec[m].x;
            float ds, dc;
            __sincosf((float)(dt - rint(dt)) * 6.28318530717958648f, &ds, &dc);
            srot[m] = make_float2(ds, dc);
        }
        __syncthreads();
    }
    const int G = (nk + FPT - 1) / FPT;        // frequency groups
    // warps per group; one wavenumber: one warp (lane m mod 32 sums the m-th
    // selected record -- the sum k_po_list forms in list mode)
    const int wpg = (G >= kPoWarps || FPT == 1) ? 1 : kPoWarps / G;
    const int passes = (G + kPoWarps - 1) / kPoWarps;
    for (int pass = 0; pass < passes; ++pass) {
        int grp, sub;
        if (G >= kPoWarps) { grp = pass * kPoWarps + warp; sub = 0; }
        else { grp = warp / wpg; sub = warp % wpg; }
        const bool active = grp < G && (G >= kPoWarps || warp < G * wpg);
        // phase 2 k R in turns: tau = (k / pi) R, reduced exactly in FP64
        // (tau - rint(tau) has no rounding error), then one float conversion
        double kk[FPT];
        double sred[FPT], cred[FPT];   // this lane's sums (FP64)
#pragma unroll
        for (int f = 0; f < FPT; ++f) {
            const int fi = grp * FPT + f;
            kk[f] = (active && fi < nk) ? kturn[fi] : 0.0;
            sred[f] = 0.0;
            cred[f] = 0.0;
        }
        if (ROT && active) {
            // __sincosf on the SFU; a lane's <= 32 terms per chunk accumulate
            // in FP32 (error comparable to the SFU's)
            float sacc[FPT], cacc[FPT];
#pragma unroll
            for (int f = 0; f < FPT; ++f) { sacc[f] = 0.f; cacc[f] = 0.f; }
            // equally spaced wavenumbers: one SFU sincos for the group's first
            // phase and one for the step, then FPT-1 exact-phase rotations
            // (FP32 complex products, error <= FPT ulps), re-anchored per group
            for (int m = sub * 32 + lane; m < M; m += wpg * 32) {
                const double2 rw = srec[m];
                const float wf = (float)rw.y;
                const double t0 = kk[0] * rw.x;
                const float2 rot = srot[m];
                const float ds = rot.x, dc = rot.y;
                float sn, cs;
                __sincosf((float)(t0 - rint(t0)) * 6.28318530717958648f, &sn, &cs);
#pragma unroll
                for (int f = 0; f < FPT; ++f) {
                    sacc[f] = fmaf(wf, sn, sacc[f]);
                    cacc[f] = fmaf(wf, cs, cacc[f]);
                    const float s2 = fmaf(sn, dc, cs * ds);
                    cs = fmaf(cs, dc, -sn * ds);
                    sn = s2;
                }
            }
#pragma unroll
            for (int f = 0; f < FPT; ++f) { sred[f] = (double)sacc[f]; cred[f] = (double)cacc[f]; }
        } else if (!ROT && active) {
            // per-frequency phases in FP64: sincospi of twice the exactly
            // reduced fraction (2 pi folded into the function), FP64 lane
            // sums -- the field follows the reference's complex128 sum to
            // ~1e-12 even at deep nulls, where any FP32 phase (1e-7 per term)
            // breaks a 1e-4 relative tolerance (scripts/parity_full_configs.py)
            for (int m = sub * 32 + lane; m < M; m += wpg * 32) {
                const double2 rw = srec[m];
#pragma unroll
                for (int f = 0; f < FPT; ++f) {
                    const double tau = kk[f] * rw.x;
                    double sn, cs;
                    sincospi(2.0 * (tau - rint(tau)), &sn, &cs);
                    sred[f] = fma(rw.y, sn, sred[f]);
                    cred[f] = fma(rw.y, cs, cred[f]);
                }
            }
        }
#pragma unroll
        for (int f = 0; f < FPT; ++f) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sred[f] += __shfl_xor_sync(0xffffffffu, sred[f], o);
                cred[f] += __shfl_xor_sync(0xffffffffu, cred[f], o);
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int f = 0; f < FPT; ++f) red[warp][f] = make_double2(sred[f], cred[f]);
        }
        __syncthreads();
        // fixed-order cross-warp combine; one thread per (group, f)
        const int groups_now = G >= kPoWarps ? min(kPoWarps, G - pass * kPoWarps) : G;
        if (tid < groups_now * FPT) {
            const int gl = tid / FPT, f = tid % FPT;
            const int g = G >= kPoWarps ? pass * kPoWarps + gl : gl;
            const int fi = g * FPT + f;
            if (fi < nk) {
                double2 acc = make_double2(0.0, 0.0);
                const int nsub = G >= kPoWarps ? 1 : wpg;
                for (int s = 0; s < nsub; ++s) {
                    const int w = G >= kPoWarps ? gl : gl * wpg + s;
                    acc.x += red[w][f].x;
                    acc.y += red[w][f].y;
                }
                chunk_part[chunk * nk + fi] = acc;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// PO over the hit list (raster mode, one wavenumber): one warp per chunk
// ---------------------------------------------------------------------------
// After the raster pass a chunk's only records with anything to integrate
// are its primary hits, which the trace kernel wrote contiguously over the
// chunk's run of the hit list (chunk_hits).  A warp integrates one chunk
// with no block barriers and no full-chunk staging: the m-th SELECTED record
// of the chunk (slot order) goes to lane m mod 32 (a 32-entry shared-memory
// hand-off per batch of 32 records), each lane sums its terms in order in
// FP64, and a fixed xor-shuffle tree gives the partial -- exactly the sum
// k_po forms for the same chunk (one warp per wavenumber group there), so
// list and slot modes agree bit for bit.  Warps pull runs of kPoSuper
// consecutive chunks; the per-grid diagnostics (valid rays, queries, max
// bounce, bounce histogram) accumulate per warp and are flushed when the
// grid changes.
constexpr int kPoListThreads = 256;
constexpr int kPoListWarps = kPoListThreads / 32;
constexpr int kPoSuper = 16;

__global__ void __launch_bounds__(kPoListThreads)
k_po_list(const UnitDev *__restrict__ units, int n_units, const uint4 *__restrict__ list,
          const uint2 *__restrict__ chunk_hits, int64_t n_chunks,
          const double *__restrict__ kturn, const double *__restrict__ gpow, int max_bounces,
          double2 *__restrict__ chunk_part, int64_t *__restrict__ diag,
          unsigned long long *__restrict__ bad, unsigned long long *__restrict__ counter,
          const int *__restrict__ chunk_unit)
{
    __shared__ unsigned int s_hist[kPoListWarps][kMaxHist];
    __shared__ double2 xfer[kPoListWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const int nb = max_bounces + 1;
    const int64_t dstride = 3 + nb;
    const double kk = __ldg(&kturn[0]);
    const SlotRec *recs = reinterpret_cast<const SlotRec *>(list);
    for (int b = lane; b < kMaxHist; b += 32) s_hist[warp][b] = 0u;
    __syncwarp();
    int cur_grid = -1;
    unsigned long long acc_q = 0;
    unsigned int acc_valid = 0, acc_maxb = 0;
    auto flush = [&]() {
        unsigned long long q = acc_q;
        unsigned int v = acc_valid, m = acc_maxb;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            q += __shfl_xor_sync(0xffffffffu, q, o);
            v += __shfl_xor_sync(0xffffffffu, v, o);
            m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        }
        __syncwarp();
        if (cur_grid >= 0 && diag) {
            int64_t *dg = diag + (int64_t)cur_grid * dstride;
            if (lane == 0) {
                if (v) atomicAdd((unsigned long long *)&dg[0], (unsigned long long)v);
                if (q) atomicAdd((unsigned long long *)&dg[1], q);
                atomicMax((unsigned long long *)&dg[2], (unsigned long long)m);
            }
            for (int b = lane; b < nb && b < kMaxHist; b += 32)
                if (s_hist[warp][b])
                    atomicAdd((unsigned long long *)&dg[3 + b], (unsigned long long)s_hist[warp][b]);
        }
        __syncwarp();
        for (int b = lane; b < kMaxHist; b += 32) s_hist[warp][b] = 0u;
        __syncwarp();
        acc_q = 0;
        acc_valid = 0;
        acc_maxb = 0;
    };
    while (true) {
        unsigned long long got = 0;
        if (lane == 0) got = atomicAdd(counter, (unsigned long long)kPoSuper);
        const int64_t c0 = (int64_t)__shfl_sync(0xffffffffu, got, 0);
        if (c0 >= n_chunks) break;
        const int64_t c1 = c0 + kPoSuper < n_chunks ? c0 + kPoSuper : n_chunks;
        for (int64_t chunk = c0; chunk < c1; ++chunk) {
            const int64_t slot0 = chunk * kChunk;
            const int ui = chunk_unit ? __ldg(&chunk_unit[chunk]) : find_unit(units, n_units, slot0);
            const UnitDev U = units[ui];
            if (U.grid != cur_grid) {
                flush();
                cur_grid = U.grid;
            }
            const uint2 run = __ldg(&chunk_hits[chunk]);
            if (lane == 0) {   // the chunk's primary misses: one query each
                const int64_t first_r = U.ray_begin + (slot0 - U.slot_base);
                int64_t real = U.ray_end - first_r;
                real = real < 0 ? 0 : (real > kChunk ? kChunk : real);
                acc_q += (unsigned long long)(real - (int64_t)run.y);
            }
            const int nrec = (int)run.y;
            double sred = 0.0, cred = 0.0;
            int m_base = 0;   // selected records handed out so far
            for (int base = 0; base < nrec; base += 32) {
                const int e = base + lane;
                SlotRec r;
                if (e < nrec) {
                    r = recs[run.x + e];
                } else {
                    r.R = 0.0; r.cosv = 0.f; r.meta = 0u;
                }
                const unsigned b = r.meta & kMetaBounceMask;
                if (r.meta & kMetaActive) {
                    acc_q += b + 1;
                    acc_maxb = max(acc_maxb, b);
                }
                const bool v = (r.meta & kMetaValid) != 0;
                acc_valid += v ? 1u : 0u;
                {   // bounce histogram: one shared atomic per distinct value
                    const unsigned key = v ? b : 0xffffffffu;
                    const unsigned peers = __match_any_sync(0xffffffffu, key);
                    if (v && lane == __ffs(peers) - 1) {
                        if (b < (unsigned)kMaxHist)
                            atomicAdd(&s_hist[warp][b], (unsigned)__popc(peers));
                        else if (diag)
                            atomicAdd((unsigned long long *)&diag[(int64_t)U.grid * dstride + 3 + b],
                                      (unsigned long long)__popc(peers));
                    }
                }
                const bool sel = (r.meta & kMetaSel) != 0;
                const unsigned bal = __ballot_sync(0xffffffffu, sel);
                const int cnt = __popc(bal);
                if (sel) {
                    const double w = 2.0 * (double)r.cosv * __ldg(&gpow[b]);
                    if (!isfinite(r.R) || !isfinite(w)) {
                        const int64_t sl = slot0 + ((r.meta >> kMetaOffShift) & (kChunk - 1));
                        atomicMin(bad, (unsigned long long)(U.ray_begin + (sl - U.slot_base)));
                    }
                    xfer[warp][(m_base + __popc(bal & lt)) & 31] = make_double2(r.R, w);
                }
                __syncwarp();
                if (((lane - m_base) & 31) < cnt) {
                    const double2 rw = xfer[warp][lane];
                    // phase 2 k R in turns, reduced exactly in FP64; FP64
                    // sincospi (2 pi folded in), FP64 lane sums (as k_po)
                    const double tau = kk * rw.x;
                    double sn, cs;
                    sincospi(2.0 * (tau - rint(tau)), &sn, &cs);
                    sred = fma(rw.y, sn, sred);
                    cred = fma(rw.y, cs, cred);
                }
                __syncwarp();
                m_base += cnt;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sred += __shfl_xor_sync(0xffffffffu, sred, o);
                cred += __shfl_xor_sync(0xffffffffu, cred, o);
            }
            if (lane == 0) chunk_part[chunk] = make_double2(0.0 + sred, 0.0 + cred);
        }
    }
    flush();
}

// chunk -> unit table of a batch (units are chunk-aligned): one load instead
// of a binary search over the units in the compaction and PO kernels
__global__ void k_chunk_units(const UnitDev *__restrict__ units, int n_units,
                              int *__restrict__ chunk_unit)
{
    const int u = blockIdx.x;
    if (u >= n_units) return;
    const UnitDev U = units[u];
    const int64_t c0 = U.slot_base / kChunk;
    const int64_t nc = (U.ray_end - U.ray_begin + kChunk - 1) / kChunk;
    for (int64_t c = threadIdx.x; c < nc; c += blockDim.x) chunk_unit[c0 + c] = u;
}

cudaError_t launch_chunk_units(const UnitDev *d_units, int n_units, int *d_chunk_unit,
                               cudaStream_t st, const LaunchStats &ls)
{
    if (n_units <= 0) return cudaSuccess;
    k_chunk_units<<<n_units, 256, 0, st>>>(d_units, n_units, d_chunk_unit);
    ++*ls.launches;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// hit-list compaction after the raster pass
// ---------------------------------------------------------------------------
// A slot whose primary ray missed is finished (transport.py:294-296: miss on
// query 0 -> escaped, invalid, N = 0); its all-ones PrimHit stays in place as
// that record (k_po decodes kMissMeta), so the trace kernel only ever
// receives rays with work left and misses cost no write.  Hits are appended to the
// work list 32 slots (one warp ballot) at a time, so consecutive list entries
// are neighbouring rays of one aperture: coherent first bounces.
constexpr int kCompactThreads = 256;
constexpr int kCompactPer = 4;                        // slots per thread per tile
constexpr int kCompactTile = kCompactThreads * kCompactPer;   // == kChunk

__global__ void __launch_bounds__(kCompactThreads)
k_prim_compact(TraceCfg cfg, const GridDev *__restrict__ grids,
               const UnitDev *__restrict__ units, int n_units, int64_t n_slots,
               SlotRec *__restrict__ slots, const unsigned int *__restrict__ hitmap,
               const int *__restrict__ chunk_unit, uint4 *__restrict__ list,
               unsigned long long *__restrict__ nlist, uint2 *__restrict__ chunk_hits)
{
    constexpr int W = kCompactThreads / 32;
    __shared__ int cnt[kCompactPer][W];
    __shared__ int pos[kCompactPer][W];
    __shared__ unsigned long long s_at;
    __shared__ int s_gcnt[W], s_gat[W];
    __shared__ unsigned long long s_gbase;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // tiles strided over the blocks: at any moment the blocks work on one
    // window of neighbouring tiles, so the list comes out close to aperture
    // order (coherent first bounces for the trace kernel)
    const int64_t ntiles = (n_slots + kCompactTile - 1) / kCompactTile;
    // groups of W consecutive tiles: their hit counts come from the raster's
    // hit bitmap (warp w pop-counts tile w's 32 words), so one atomic per
    // group reserves the list space (a single counter for every tile
    // serialised at L2)
    const int64_t ngroups = (ntiles + W - 1) / W;
    for (int64_t gi = blockIdx.x; gi < ngroups; gi += gridDim.x) {
      if (hitmap) {
          const int64_t tw = gi * W + warp;
          int c = 0;
          if (tw < ntiles) {
              const int64_t word = tw * (kCompactTile / 32) + lane;
              if (word * 32 < n_slots) c = __popc(__ldg(hitmap + word));
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
          if (lane == 0) s_gcnt[warp] = c;
          __syncthreads();
          if (tid == 0) {
              int run = 0;
              for (int w = 0; w < W; ++w) {
                  s_gat[w] = run;
                  run += s_gcnt[w];
              }
              s_gbase = run ? atomicAdd(nlist, (unsigned long long)run) : 0ULL;
          }
          __syncthreads();
      }
      for (int t8 = 0; t8 < W; ++t8) {
        const int64_t ti = gi * W + t8;
        if (ti >= ntiles) break;
        const int64_t tile = ti * kCompactTile;
        // slots are chunk-aligned per unit and kCompactTile == kChunk: one unit
        const int ui = chunk_unit ? __ldg(&chunk_unit[ti]) : find_unit(units, n_units, tile);
        const UnitDev U = units[ui];
        const bool alias_ok =
            cfg.allow_aliasing || !(grids[U.grid].spacing > cfg.spacing_limit);
        if (!alias_ok && tid == 0) atomicOr(cfg.error_flag, 1u);
        unsigned hitmask = 0;
        ulonglong2 hv[kCompactPer];
#pragma unroll
        for (int q = 0; q < kCompactPer; ++q) {
            const int64_t slot = tile + q * kCompactThreads + tid;
            bool hit = false;
            hv[q] = make_ulonglong2(kNoHitBits, kNoHitBits);
            // the raster's hit bitmap (one word per warp and q): only the
            // slots that were hit are read at all
            const bool marked =
                slot < n_slots &&
                (!hitmap || ((__ldg(hitmap + (slot >> 5)) >> (unsigned)(slot & 31)) & 1u));
            if (marked) {
                const int64_t r = U.ray_begin + (slot - U.slot_base);
                const bool real = r < U.ray_end && alias_ok;
                // streaming read: every hit slot is read once here
                hv[q] = __ldcs(reinterpret_cast<const ulonglong2 *>(slots) + slot);
                // with the bitmap a marked slot IS a hit (the group's list
                // space was reserved from the bitmap counts); an aliasing
                // violation is reported through the error flag instead
                hit = hitmap ? true : (real && hv[q].x != kNoHitBits);
                // the hit moves into the work list; its slot returns to the
                // raster's all-ones "no hit" (no memset before the next
                // pass).  Misses and padding keep their all-ones bits.
                if (hit)
                    __stcs(reinterpret_cast<ulonglong2 *>(slots) + slot,
                           make_ulonglong2(kNoHitBits, kNoHitBits));
            }
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            if (lane == 0) cnt[q][warp] = __popc(bal);
            hitmask |= (hit ? 1u : 0u) << q;
        }
        __syncthreads();
        static_assert(kCompactPer * W == 32, "one warp scans the (q, warp) counts");
        if (warp == 0) {   // exclusive scan in slot order + one atomic per tile
            const int v = (&cnt[0][0])[lane];
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            (&pos[0][0])[lane] = incl - v;
            if (lane == 31) {
                const int run = incl;
                s_at = hitmap ? s_gbase + (unsigned long long)s_gat[t8]
                              : (run ? atomicAdd(nlist, (unsigned long long)run) : 0ULL);
                // this chunk's hits: list[at, at + run), in slot order
                chunk_hits[ti] = make_uint2((unsigned int)s_at, (unsigned int)run);
            }
        }
        __syncthreads();
        const unsigned long long at = s_at;
#pragma unroll
        for (int q = 0; q < kCompactPer; ++q) {
            const bool hit = (hitmask >> q) & 1u;
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            if (hit) {
                // (t bits, id | offset in unit << 25 | unit << 44): the trace
                // refill needs nothing else
                const unsigned long long off = (unsigned long long)(tile - U.slot_base) +
                                               (unsigned long long)(q * kCompactThreads + tid);
                const unsigned long long pk = (hv[q].y >> 32) | (off << kWlOffShift) |
                                              ((unsigned long long)ui << kWlUnitShift);
                list[at + pos[q][warp] + __popc(bal & ((1u << lane) - 1u))] =
                    make_uint4((unsigned int)hv[q].x, (unsigned int)(hv[q].x >> 32),
                               (unsigned int)pk, (unsigned int)(pk >> 32));
            }
        }
        __syncthreads();
      }
    }
}

cudaError_t launch_prim_compact(const TraceCfg &cfg, const GridDev *d_grids,
                                const UnitDev *d_units, int n_units, int64_t n_slots,
                                SlotRec *d_slots, const unsigned int *d_hitmap,
                                const int *d_chunk_unit, uint4 *d_worklist,
                                unsigned long long *d_nwork, uint2 *d_chunk_hits,
                                cudaStream_t st, const LaunchStats &ls)
{
    cudaError_t e = cudaMemsetAsync(d_nwork, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    static_assert(kCompactTile == kChunk, "tiles must not straddle units");
    int64_t blocks = (n_slots + kCompactTile - 1) / kCompactTile;
    const int64_t cap = (int64_t)ls.num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    k_prim_compact<<<(unsigned)blocks, kCompactThreads, 0, st>>>(
        cfg, d_grids, d_units, n_units, n_slots, d_slots, d_hitmap, d_chunk_unit, d_worklist,
        d_nwork, d_chunk_hits);
    ++*ls.launches;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// deterministic pairwise trees
// ---------------------------------------------------------------------------
// Sequential adjacent-pair tree with odd-tail carry (po.py:59-80 shape),
// evaluated with a size-tagged stack: equal-size neighbours merge left+right,
// leftovers fold right-nested -- identical to the level-by-level algorithm.
__device__ double2 pairwise_seq(const double2 *p, int64_t n, int64_t stride)
{
    double2 st[48];
    int64_t sz[48];
    int top = 0;
    for (int64_t i = 0; i < n; ++i) {
        double2 v = p[i * stride];
        int64_t s = 1;
        while (top > 0 && sz[top - 1] == s) {
            v = make_double2(st[top - 1].x + v.x, st[top - 1].y + v.y);
            s <<= 1;
            --top;
        }
        st[top] = v;
        sz[top] = s;
        ++top;
    }
    if (top == 0) return make_double2(0.0, 0.0);
    double2 acc = st[top - 1];
    for (int j = top - 2; j >= 0; --j) acc = make_double2(st[j].x + acc.x, st[j].y + acc.y);
    return acc;
}

// One block per (unit, wavenumber): the unit's <= kSegChunks chunk partials
// are summed level by level in shared memory (adjacent pairs, odd tail
// carried -- the same tree as pairwise_seq / po.py:59-80).
constexpr int kSegThreads = 256;
__global__ void __launch_bounds__(kSegThreads)
k_seg_reduce(const double2 *__restrict__ chunk_part, const UnitDev *__restrict__ units,
             int n_units, int nk, double2 *__restrict__ seg_part)
{
    __shared__ double2 buf[2][kSegChunks];
    const int u = blockIdx.x, f = blockIdx.y;
    const UnitDev U = units[u];
    int n = (int)((U.ray_end - U.ray_begin + kChunk - 1) / kChunk);
    const int64_t c0 = U.slot_base / kChunk;
    for (int i = threadIdx.x; i < n; i += kSegThreads)
        buf[0][i] = chunk_part[(c0 + i) * nk + f];
    __syncthreads();
    int cur = 0;
    while (n > 1) {
        const int half = n >> 1;
        for (int i = threadIdx.x; i < half; i += kSegThreads) {
            const double2 a = buf[cur][2 * i], b = buf[cur][2 * i + 1];
            buf[cur ^ 1][i] = make_double2(a.x + b.x, a.y + b.y);
        }
        if ((n & 1) && threadIdx.x == 0) buf[cur ^ 1][half] = buf[cur][n - 1];
        n = half + (n & 1);
        cur ^= 1;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double2 v = n ? buf[cur][0] : make_double2(0.0, 0.0);
        v.x += 0.0;   // normalise -0.0 so a disjoint-support sum reduce is exact
        v.y += 0.0;
        seg_part[U.seg_out * nk + f] = v;
    }
}

__global__ void k_finalize(const double2 *__restrict__ seg_part,
                           const int64_t *__restrict__ seg_base, int ngrids, int nk,
                           const double *__restrict__ scale, double2 *__restrict__ amp)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)ngrids * nk) return;
    const int g = (int)(t / nk), f = (int)(t % nk);
    const int64_t s0 = seg_base[g], s1 = seg_base[g + 1];
    const double2 v = pairwise_seq(seg_part + s0 * nk + f, s1 - s0, nk);
    // sum carries (w sin, w cos); term = a (sin + j cos), a = k dA / 4pi
    const double a = scale[t];
    amp[t] = make_double2(a * v.x, a * v.y);
}

// ---------------------------------------------------------------------------
// packed reduce buffer (one SUM collective for partials AND diagnostics)
// ---------------------------------------------------------------------------
// tail = [diag (ng x stride) as doubles, column 2 zeroed][max bounce slots
// (ng x nranks), this rank's value in slot `rank`]: every entry is an
// integer < 2^53, so the SUM over ranks is exact, and the per-grid max bounce
// is the max over the slots after the sum.
__global__ void k_pack_diag(const int64_t *diag, int ng, int stride, int nranks, int rank,
                            double *tail)
{
    const int64_t n = (int64_t)ng * stride;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = i / stride, c = i - g * stride;
        tail[i] = c == 2 ? 0.0 : (double)diag[i];
        if (c == 2) {
            for (int r = 0; r < nranks; ++r)
                tail[n + g * nranks + r] = r == rank ? (double)diag[i] : 0.0;
        }
    }
}

__global__ void k_unpack_diag(const double *tail, int ng, int stride, int nranks, int64_t *diag)
{
    const int64_t n = (int64_t)ng * stride;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = i / stride, c = i - g * stride;
        if (c == 2) {
            double m = 0.0;
            for (int r = 0; r < nranks; ++r) m = fmax(m, tail[n + g * nranks + r]);
            diag[i] = (int64_t)m;
        } else {
            diag[i] = (int64_t)tail[i];
        }
    }
}

cudaError_t launch_pack_diag(const int64_t *d_diag, int ng, int stride, int nranks, int rank,
                             double *d_tail, cudaStream_t st, const LaunchStats &ls)
{
    k_pack_diag<<<64, 256, 0, st>>>(d_diag, ng, stride, nranks, rank, d_tail);
    ++*ls.launches;
    return cudaGetLastError();
}

cudaError_t launch_unpack_diag(const double *d_tail, int ng, int stride, int nranks,
                               int64_t *d_diag, cudaStream_t st, const LaunchStats &ls)
{
    k_unpack_diag<<<64, 256, 0, st>>>(d_tail, ng, stride, nranks, d_diag);
    ++*ls.launches;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// launch wrappers
// ---------------------------------------------------------------------------
template <class K>
static int persistent_blocks(K kernel, int threads, int num_sms)
{
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    return per_sm * num_sms;
}

template <int S, int M>
static void trace_dispatch(const TraceArgs &a, cudaStream_t st, int num_sms)
{
    // query 0 from the raster pass and a one-bounce budget: every traced
    // query is an escape probe (probe-only stack, see pop_next)
    const bool probes = M != kModeList && a.prim && a.cfg.max_bounces == 1;
    if (a.cfg.B.width == 8 && a.cfg.B.nodes8) {
        int nb = persistent_blocks(k_trace_persistent<S, M, 8>, kTraceThreads, num_sms);
        k_trace_persistent<S, M, 8><<<nb, kTraceThreads, 0, st>>>(a);
    } else if (probes) {
        int nb = persistent_blocks(k_trace_persistent<S, M, 4, true>, kTraceThreads, num_sms);
        k_trace_persistent<S, M, 4, true><<<nb, kTraceThreads, 0, st>>>(a);
    } else {
        int nb = persistent_blocks(k_trace_persistent<S, M, 4>, kTraceThreads, num_sms);
        k_trace_persistent<S, M, 4><<<nb, kTraceThreads, 0, st>>>(a);
    }
}

template <int M>
static void trace_storage_dispatch(const TraceArgs &a, cudaStream_t st, int num_sms)
{
    if (a.cfg.storage == kF64) trace_dispatch<kF64, M>(a, st, num_sms);
    else if (a.cfg.storage == kSingle) trace_dispatch<kSingle, M>(a, st, num_sms);
    else trace_dispatch<kF32Exact, M>(a, st, num_sms);
}

cudaError_t launch_trace_solve(const TraceCfg &cfg, const GridDev *d_grids,
                               const UnitDev *d_units, int n_units, int64_t n_slots,
                               SlotRec *d_slots, unsigned long long *d_counter,
                               bool prim_from_slots, uint4 *d_worklist,
                               const unsigned long long *d_nwork, cudaStream_t st,
                               const LaunchStats &ls)
{
    cudaError_t e = cudaMemsetAsync(d_counter, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    TraceArgs a = {};
    a.cfg = cfg;
    a.grids = d_grids;
    a.units = d_units;
    a.n_units = n_units;
    a.n_work = n_slots;
    a.counter = d_counter;
    a.slots = d_slots;
    a.prim = prim_from_slots ? reinterpret_cast<const PrimHit *>(d_slots) : nullptr;
    a.worklist = d_worklist;
    a.n_work_dev = d_nwork;
    trace_storage_dispatch<kModeSolve>(a, st, ls.num_sms);
    ++*ls.launches;
    return cudaGetLastError();
}

cudaError_t launch_trace_full(const TraceCfg &cfg, const GridDev *d_grid,
                              const double *d_orig, const double *d_dirs, int64_t n,
                              int64_t r_base, const FullOut &out, const PrimHit *d_prim,
                              unsigned long long *d_counter, cudaStream_t st,
                              const LaunchStats &ls)
{
    cudaError_t e = cudaMemsetAsync(d_counter, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    TraceArgs a = {};
    a.cfg = cfg;
    a.grids = d_grid;
    a.orig = d_orig;
    a.dirs = d_dirs;
    a.n_work = n;
    a.counter = d_counter;
    a.full = out;
    a.r_base = d_grid ? r_base : 0;
    a.prim = d_grid ? d_prim : nullptr;
    if (d_grid) trace_storage_dispatch<kModeGrid>(a, st, ls.num_sms);
    else trace_storage_dispatch<kModeList>(a, st, ls.num_sms);
    ++*ls.launches;
    return cudaGetLastError();
}

cudaError_t launch_closest(const BvhView &B, int storage, const double *d_orig,
                           const double *d_dirs, int64_t n, double t_min, double t_max,
                           int64_t *d_tri, double *d_t, int64_t *d_visits, cudaStream_t st,
                           const LaunchStats &ls)
{
    int64_t want = (n + kTraceThreads - 1) / kTraceThreads;
    int nb = (int)(want < 65535 ? (want > 0 ? want : 1) : 65535);
    if (storage == kF64)
        k_closest<kF64><<<nb, kTraceThreads, 0, st>>>(B, d_orig, d_dirs, n, t_min, t_max, d_tri,
                                                      d_t, d_visits);
    else if (storage == kSingle)
        k_closest<kSingle><<<nb, kTraceThreads, 0, st>>>(B, d_orig, d_dirs, n, t_min, t_max,
                                                         d_tri, d_t, d_visits);
    else
        k_closest<kF32Exact><<<nb, kTraceThreads, 0, st>>>(B, d_orig, d_dirs, n, t_min, t_max,
                                                           d_tri, d_t, d_visits);
    ++*ls.launches;
    return cudaGetLastError();
}

cudaError_t launch_records_to_slots(const uint8_t *valid, const double *n0,
                                    const double *path, const int32_t *bounces,
                                    const uint8_t *escaped, int64_t n, double kx,
                                    double ky, double kz, int count_trapped,
                                    int64_t n_slots, SlotRec *slots, cudaStream_t st,
                                    const LaunchStats &ls)
{
    int64_t want = (n_slots + 255) / 256;
    int nb = (int)(want < 65535 ? (want > 0 ? want : 1) : 65535);
    k_records_to_slots<<<nb, 256, 0, st>>>(valid, n0, path, bounces, escaped, n, kx, ky, kz,
                                           count_trapped, n_slots, slots);
    ++*ls.launches;
    return cudaGetLastError();
}

cudaError_t launch_po(SlotRec *d_slots, const UnitDev *d_units, int n_units,
                      const uint4 *d_list, const uint2 *d_chunk_hits,
                      int64_t n_chunks, const double *d_k2, int nk, double dkturn,
                      const double *d_gpow,
                      int max_bounces, double2 *d_chunk_part, int64_t *d_diag,
                      unsigned long long *d_bad, unsigned long long *d_counter,
                      const int *d_chunk_unit, cudaStream_t st, const LaunchStats &ls)
{
    if (n_chunks <= 0) return cudaSuccess;
    dim3 grid((unsigned)n_chunks);
    // uniform sweeps take the SFU rotation path (~1e-5 relative field);
    // SBR_PO_FP64=1 forces the FP64 per-wavenumber path for them too
    static const bool force64 = getenv("SBR_PO_FP64") && atoi(getenv("SBR_PO_FP64")) != 0;
    const bool rot = nk > 1 && dkturn != 0.0 && !force64;
#define SBR_PO(F, R)                                                                       \
    k_po<F, R><<<grid, kPoThreads, 0, st>>>(d_slots, d_units, n_units, d_list, d_chunk_hits, \
                                            d_k2, nk, dkturn, d_gpow, max_bounces,          \
                                            d_chunk_part, d_diag, d_bad)
    static const bool block_po = getenv("SBR_PO_BLOCK") != nullptr;   // A/B: one block per chunk
    if (d_list && nk == 1 && !block_po) {
        cudaError_t e = cudaMemsetAsync(d_counter, 0, sizeof(unsigned long long), st);
        if (e != cudaSuccess) return e;
        k_po_list<<<(unsigned)(ls.num_sms * 8), kPoListThreads, 0, st>>>(
            d_units, n_units, d_list, d_chunk_hits, n_chunks, d_k2, d_gpow, max_bounces,
            d_chunk_part, d_diag, d_bad, d_counter, d_chunk_unit);
    } else {
        if (nk >= 8) { if (rot) SBR_PO(8, true); else SBR_PO(8, false); }
        else if (nk >= 4) { if (rot) SBR_PO(4, true); else SBR_PO(4, false); }
        else if (nk >= 2) { if (rot) SBR_PO(2, true); else SBR_PO(2, false); }
        else SBR_PO(1, false);
    }
#undef SBR_PO
    ++*ls.launches;
    return cudaGetLastError();
}

cudaError_t launch_seg_reduce(const double2 *d_chunk_part, const UnitDev *d_units,
                              int n_units, int nk, double2 *d_seg_part, cudaStream_t st,
                              const LaunchStats &ls)
{
    if ((int64_t)n_units * nk == 0) return cudaSuccess;
    k_seg_reduce<<<dim3((unsigned)n_units, (unsigned)nk), kSegThreads, 0, st>>>(
        d_chunk_part, d_units, n_units, nk, d_seg_part);
    ++*ls.launches;
    return cudaGetLastError();
}

cudaError_t launch_finalize(const double2 *d_seg_part, const int64_t *d_seg_base,
                            int ngrids, int nk, const double *d_scale, double2 *d_amp,
                            cudaStream_t st, const LaunchStats &ls)
{
    int64_t n = (int64_t)ngrids * nk;
    if (n == 0) return cudaSuccess;
    k_finalize<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(d_seg_part, d_seg_base, ngrids, nk,
                                                             d_scale, d_amp);
    ++*ls.launches;
    return cudaGetLastError();
}

}  // namespace sbr

namespace sbr {

// ---------------------------------------------------------------------------
// scalar predicates over independent pairs (geometry.py:394-425)
// ---------------------------------------------------------------------------
__global__ void k_tri_pairs(const double *__restrict__ v0, const double *__restrict__ v1,
                            const double *__restrict__ v2, const double *__restrict__ o,
                            const double *__restrict__ d, int64_t n, double t_min,
                            double t_max, int single, double *__restrict__ t_out)
{
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        TriF64 T;
        T.ax = v0[3 * r]; T.ay = v0[3 * r + 1]; T.az = v0[3 * r + 2];
        if (single) {
            T.e1x = __fsub_rn((float)v1[3 * r], (float)T.ax);
            T.e1y = __fsub_rn((float)v1[3 * r + 1], (float)T.ay);
            T.e1z = __fsub_rn((float)v1[3 * r + 2], (float)T.az);
            T.e2x = __fsub_rn((float)v2[3 * r], (float)T.ax);
            T.e2y = __fsub_rn((float)v2[3 * r + 1], (float)T.ay);
            T.e2z = __fsub_rn((float)v2[3 * r + 2], (float)T.az);
        } else {
            T.e1x = DS(v1[3 * r], T.ax); T.e1y = DS(v1[3 * r + 1], T.ay);
            T.e1z = DS(v1[3 * r + 2], T.az);
            T.e2x = DS(v2[3 * r], T.ax); T.e2y = DS(v2[3 * r + 1], T.ay);
            T.e2z = DS(v2[3 * r + 2], T.az);
        }
        T.id = 0;
        t_out[r] = tri_hit_exact(T, o[3 * r], o[3 * r + 1], o[3 * r + 2], d[3 * r], d[3 * r + 1],
                                 d[3 * r + 2], t_min, t_max);
    }
}

// FP64 slab test exactly as geometry.py:358-391 (reciprocals given).
__global__ void k_box_pairs(const double *__restrict__ lo, const double *__restrict__ hi,
                            const double *__restrict__ o, const double *__restrict__ inv,
                            int64_t n, double t_max, uint8_t *__restrict__ hit,
                            double *__restrict__ entry)
{
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        double tn = 0.0, tf = t_max;
        bool h = true;
        for (int a = 0; a < 3 && h; ++a) {
            const double l = lo[3 * r + a], u = hi[3 * r + a], oo = o[3 * r + a],
                         iv = inv[3 * r + a];
            if (isinf(iv)) {
                if (oo < l || oo > u) h = false;
            } else {
                double t1 = DM(DS(l, oo), iv), t2 = DM(DS(u, oo), iv);
                if (t1 > t2) { double s = t1; t1 = t2; t2 = s; }
                if (t1 > tn) tn = t1;
                if (t2 < tf) tf = t2;
                if (tn > tf) h = false;
            }
        }
        hit[r] = h ? 1 : 0;
        entry[r] = h ? tn : 0.0;
    }
}

cudaError_t launch_tri_pairs(const double *v0, const double *v1, const double *v2,
                             const double *o, const double *d, int64_t n, double t_min,
                             double t_max, int single, double *t_out, cudaStream_t st,
                             const LaunchStats &ls)
{
    int64_t want = (n + 255) / 256;
    int nb = (int)(want < 65535 ? (want > 0 ? want : 1) : 65535);
    k_tri_pairs<<<nb, 256, 0, st>>>(v0, v1, v2, o, d, n, t_min, t_max, single, t_out);
    ++*ls.launches;
    return cudaGetLastError();
}

cudaError_t launch_box_pairs(const double *lo, const double *hi, const double *o,
                             const double *inv, int64_t n, double t_max, uint8_t *hit,
                             double *entry, cudaStream_t st, const LaunchStats &ls)
{
    int64_t want = (n + 255) / 256;
    int nb = (int)(want < 65535 ? (want > 0 ? want : 1) : 65535);
    k_box_pairs<<<nb, 256, 0, st>>>(lo, hi, o, inv, n, t_max, hit, entry);
    ++*ls.launches;
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// L2-resident read bandwidth probe (instrumentation for the roofline line)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_l2_read(const float4 *__restrict__ buf, int64_t n4,
                                                 int reps, float *__restrict__ sink)
{
    float acc = 0.f;
    for (int r = 0; r < reps; ++r)
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
             i += (int64_t)gridDim.x * blockDim.x) {
            const float4 v = __ldcg(buf + i);     // L2, not L1
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 12345.678f) sink[blockIdx.x] = acc;   // keep the loads
}

cudaError_t probe_l2_read(int64_t bytes, int reps, int num_sms, cudaStream_t st, double *gbs)
{
    const int64_t n4 = bytes / 16;
    float4 *buf = nullptr;
    float *sink = nullptr;
    cudaError_t e = cudaMalloc(&buf, n4 * 16);
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&sink, sizeof(float) * num_sms * 8);
    if (e == cudaSuccess) e = cudaMemsetAsync(buf, 0, n4 * 16, st);
    cudaEvent_t a = nullptr, b = nullptr;
    if (e == cudaSuccess) e = cudaEventCreate(&a);
    if (e == cudaSuccess) e = cudaEventCreate(&b);
    double best = 0.0;
    for (int t = 0; t < 5 && e == cudaSuccess; ++t) {
        k_l2_read<<<num_sms * 8, 256, 0, st>>>(buf, n4, 1, sink);     // warm L2
        cudaEventRecord(a, st);
        k_l2_read<<<num_sms * 8, 256, 0, st>>>(buf, n4, reps, sink);
        cudaEventRecord(b, st);
        e = cudaEventSynchronize(b);
        float ms = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
        if (e == cudaSuccess && ms > 0.f) best = fmax(best, (double)n4 * 16 * reps / (ms * 1e-3) / 1e9);
    }
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    cudaFree(buf);
    cudaFree(sink);
    *gbs = best;
    return e;
}

}  // namespace sbr
