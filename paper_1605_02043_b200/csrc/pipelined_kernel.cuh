// pipelined_kernel.cuh -- the B200 staged edge kernel (step a5): persistent CTAs, TMA
// bulk staging, double-buffered across partitions.
//
// The paper's transformed kernel has each thread block load its shared data
// into local_arrayA "coalesced into as few contiguous memory segments as possible" and
// then compute from it. On sm_100a every per-partition input is one contiguous segment
// after the remap:
//   plan blob  : halo ids, halo result positions, endpoint slots, incidence lists
//   state rows : the owned range O_p = [beginA[p], beginA[p+1]) of the cpack layout
//   payload    : the partition's edge range of the reorganised tasks
//   vertex const: the owned range again
// so one thread issues four 1-D TMA bulk copies (cp.async.bulk, completion on an
// mbarrier) per partition; only the halo rows H_p (the C = sum (p_v - 1) redundant
// loads of Eq. (1)) are gathered row by row with cp.async. A persistent CTA walks its
// partitions with two stage buffers: partition t+1's copies and gathers are in flight
// while partition t computes.
//
// Compute per partition (all from shared memory, no atomics):
//   derive  one float per local vertex (|u| + c for cfd)
//   edges   one thread per edge -> Phi[i] (the interaction)
//   reduce  one thread per local vertex sums its incidence list in a fixed order;
//           owned vertices write U + dt F (final if p_v = 1); halo vertices write their
//           partial sum to the vertex-grouped halo buffer; after a grid-wide barrier
//           the same CTAs add those to the owners' rows (fixed order: deterministic).
#pragma once

#include <stdint.h>

#include "functors.cuh"
#include "ptx.cuh"

namespace epg {

#ifdef EPG_TRACE
// development trace (build with -DEPG_TRACE): %globaltimer stamps per CTA and iteration
constexpr int kTraceIters = 16, kTracePts = 8;
__device__ unsigned long long g_trace[1024 * kTraceIters * kTracePts];
__device__ __forceinline__ void trace_point(int64_t t, int pt) {
    if (threadIdx.x == 0 && t < kTraceIters && blockIdx.x < 1024) {
        unsigned long long ns;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(ns));
        g_trace[(blockIdx.x * kTraceIters + t) * kTracePts + pt] = ns;
    }
}
#define EPG_TP(t, pt) trace_point(t, pt)
#else
#define EPG_TP(t, pt)
#endif

struct PartDesc {
    int32_t o0, nO, e0, s, h0, nH, blob16, blob_bytes, hid16, pad0, pad1, pad2;
};

struct PipeArgs {
    const PartDesc *desc;
    const unsigned char *blob;
    const int32_t *hid_blob;   // halo ids of every partition, each list 16-byte aligned
    const float *state_in;
    float *state_out;
    const float *payload;   // NULL when the functor runs without one (gather-scatter, w = 1)
    const float *vconst;    // cfd dt
    float *halo_buf;        // [C][ROW], grouped by vertex
    int64_t k;
    int nstage;             // 1 or 2
    int stage_bytes, off_rows, off_pay, off_vc;  // byte offsets inside a stage (blob at 0)
    int off_der, off_phi;                        // working arrays after the stages
    int off_hid, hid_slot_bytes;                 // 3-slot ring of halo-id lists
    int Lcap, Scap;                              // Phi has Scap + 1 columns (last = 0)
    // fused boundary finalise (after a grid-wide barrier)
    const int32_t *shared_ids;
    const int32_t *hv_off;
    int32_t S;
    int64_t touched, n;
    // partitions of CTA b: cta_list[cta_begin[b] .. cta_begin[b+1]) (balanced assignment)
    const int32_t *cta_begin;
    const int32_t *cta_list;
    // grid-wide barrier (normal launch, grid sized to be co-resident): counter + target
    unsigned long long *bar_ctr;
    unsigned long long bar_target;
};

// Generation-counted grid barrier: the counter only grows; launch g waits for g * grid
// arrivals. Requires all CTAs of the launch to be resident (grid <= SMs x occupancy).
__device__ __forceinline__ void grid_barrier(unsigned long long *ctr, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1ull);
        unsigned long long v;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
            if (v < target) __nanosleep(64);
        } while (v < target);
        __threadfence();
    }
    __syncthreads();
}

// Blob layout of one partition (16-byte aligned; W = padded incidence width, 0 = CSR):
//   [halo result positions nH x i32][slots s x u32] pad16
//   W > 0: [incidence W x L x u16]  entry (edge << 1 | side); unused entries (s << 1)
//   W = 0: [incidence 2s x u16][offsets L x u16]
// The halo ids live in a separate array (hid_blob) so they can be fetched one partition
// earlier than the rest: the halo gather of a partition depends on them.
__host__ __device__ __forceinline__ int blob_inc_offset(int nH, int s) { return (4 * nH + 4 * s + 15) & ~15; }
__host__ __device__ __forceinline__ int hid_bytes_for(int nH) { return (4 * nH + 15) & ~15; }
__host__ __device__ __forceinline__ int blob_bytes_for(int nH, int s, int L, int W) {
    const int inc = W > 0 ? 2 * W * L : 4 * s + 2 * L;
    return (blob_inc_offset(nH, s) + inc + 15) & ~15;
}

__device__ __forceinline__ uintptr_t up16(uintptr_t x) { return (x + 15) & ~uintptr_t(15); }
__device__ __forceinline__ uintptr_t down16(uintptr_t x) { return x & ~uintptr_t(15); }

// smem image of global range [g, g + bytes): byte x lives at sbase + (x - down16(g)).
// Returns the aligned body size (bulk-copied); ragged words are copied by gather_ragged.
__device__ __forceinline__ uint32_t region_body(const void *g, uint32_t bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(g);
    const uintptr_t lo = up16(a), hi = down16(a + bytes);
    return hi > lo ? (uint32_t)(hi - lo) : 0u;
}

__device__ __forceinline__ void region_bulk(unsigned char *sbase, const void *g, uint32_t bytes, uint64_t *bar) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(g);
    const uintptr_t lo = up16(a), hi = down16(a + bytes);
    if (hi > lo)
        ptx::bulk_g2s(sbase + (lo - down16(a)), reinterpret_cast<const void *>(lo), (uint32_t)(hi - lo), bar);
}

// lane `lane` of one warp copies the lane-th ragged word of the region (<= 7 words)
__device__ __forceinline__ void region_ragged(unsigned char *sbase, const void *g, uint32_t bytes, int lane) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(g);
    const uintptr_t end = a + bytes;
    const uintptr_t lo = up16(a), hi = down16(end);
    uintptr_t w;
    if (hi > lo) {
        const int head = (int)((lo - a) >> 2), tail = (int)((end - hi) >> 2);
        if (lane < head) w = a + 4 * lane;
        else if (lane < head + tail) w = hi + 4 * (lane - head);
        else return;
    } else {
        if (lane >= (int)(bytes >> 2)) return;
        w = a + 4 * lane;
    }
    ptx::cp_async4(sbase + (w - down16(a)), reinterpret_cast<const void *>(w));
}

template <class Fn>
struct Stage {
    const PartDesc d;
    unsigned char *base;
    const PipeArgs &a;
    __device__ Stage(const PartDesc &dd, unsigned char *b, const PipeArgs &aa) : d(dd), base(b), a(aa) {}
    __device__ const float *g_rows() const { return a.state_in + (int64_t)Fn::ROW * d.o0; }
    __device__ const float *g_pay() const { return a.payload + (int64_t)Fn::PAYW * d.e0; }
    __device__ const float *g_vc() const { return a.vconst + d.o0; }
    __device__ uint32_t rows_bytes() const { return 4u * Fn::ROW * d.nO; }
    __device__ uint32_t pay_bytes() const { return 4u * Fn::PAYW * d.s; }
    __device__ uint32_t vc_bytes() const { return 4u * d.nO; }
    __device__ unsigned char *s_rows_base() const { return base + a.off_rows; }
    __device__ unsigned char *s_pay_base() const { return base + a.off_pay; }
    __device__ unsigned char *s_vc_base() const { return base + a.off_vc; }
    __device__ float *rows() const {
        return reinterpret_cast<float *>(s_rows_base() + (reinterpret_cast<uintptr_t>(g_rows()) & 15));
    }
    __device__ const float *pay() const {
        return a.payload ? reinterpret_cast<const float *>(s_pay_base() + (reinterpret_cast<uintptr_t>(g_pay()) & 15))
                         : nullptr;
    }
    __device__ const float *vc() const {
        return reinterpret_cast<const float *>(s_vc_base() + (reinterpret_cast<uintptr_t>(g_vc()) & 15));
    }
    __device__ const int32_t *halo_pos() const { return reinterpret_cast<const int32_t *>(base); }
    __device__ const uint32_t *slots() const { return reinterpret_cast<const uint32_t *>(halo_pos() + d.nH); }
    __device__ const uint16_t *inc() const {
        return reinterpret_cast<const uint16_t *>(base + blob_inc_offset(d.nH, d.s));
    }
    __device__ const uint16_t *inc_off() const { return inc() + 2 * d.s; }

    // thread 0: arm the barrier with the bytes of all aligned bodies, then issue them
    __device__ void issue_bulk(uint64_t *bar) const {
        uint32_t tx = (uint32_t)d.blob_bytes + region_body(g_rows(), rows_bytes());
        if (a.payload) tx += region_body(g_pay(), pay_bytes());
        if (Fn::kUsesConst) tx += region_body(g_vc(), vc_bytes());
        ptx::mbar_arrive_expect_tx(bar, tx);
        if (d.blob_bytes) ptx::bulk_g2s(base, a.blob + 16 * (int64_t)d.blob16, (uint32_t)d.blob_bytes, bar);
        region_bulk(s_rows_base(), g_rows(), rows_bytes(), bar);
        if (a.payload) region_bulk(s_pay_base(), g_pay(), pay_bytes(), bar);
        if (Fn::kUsesConst) region_bulk(s_vc_base(), g_vc(), vc_bytes(), bar);
    }

    // thread 0: fetch the halo ids into a ring slot
    __device__ void issue_hid(int32_t *slot, uint64_t *bar) const {
        const uint32_t bytes = (uint32_t)hid_bytes_for(d.nH);
        ptx::mbar_arrive_expect_tx(bar, bytes);
        if (bytes) ptx::bulk_g2s(slot, a.hid_blob + 4 * (int64_t)d.hid16, bytes, bar);
    }

    // all threads, once the halo ids landed: ragged words + halo row gathers (the owned
    // rows may still be in flight: they occupy disjoint bytes of the rows region)
    template <int BLOCK>
    __device__ void issue_gather(const int32_t *hid) const {
        const int tid = threadIdx.x;
        if (tid < 32) {
            region_ragged(s_rows_base(), g_rows(), rows_bytes(), tid);
            if (a.payload) region_ragged(s_pay_base(), g_pay(), pay_bytes(), tid);
            if (Fn::kUsesConst) region_ragged(s_vc_base(), g_vc(), vc_bytes(), tid);
        }
        float *r = rows() + Fn::ROW * d.nO;
        for (int w = tid; w < Fn::ROW * d.nH; w += BLOCK) {
            const int j = w / Fn::ROW, c = w - j * Fn::ROW;
            ptx::cp_async4(r + w, a.state_in + (int64_t)Fn::ROW * hid[j] + c);
        }
    }
};

// phase A of a partition: per-vertex derived records, then one thread per edge -> Phi
// records (each thread takes edges i and i + BLOCK together, two independent chains)
template <class Fn, int BLOCK, int W>
__device__ __forceinline__ void compute_edges(const Stage<Fn> &S, const PipeArgs &a, unsigned char *sm) {
    const int tid = threadIdx.x;
    const PartDesc &d = S.d;
    const int L = d.nO + d.nH;
    const float *rows = S.rows();
    float *recs = reinterpret_cast<float *>(sm + a.off_der);
    float *phis = reinterpret_cast<float *>(sm + a.off_phi);
    for (int j = tid; j < L; j += BLOCK) Fn::derive_rec(rows + Fn::ROW * j, recs, j);
    __syncthreads();
    const uint32_t *slots = S.slots();
    const float *pay = S.pay();
    for (int i0 = tid; i0 < d.s; i0 += 2 * BLOCK) {
        const int i1 = i0 + BLOCK;
        const uint32_t s0 = slots[i0];
        if (i1 < d.s) {
            const uint32_t s1 = slots[i1];
            Fn::edge_rec(recs, (int)(s0 & 0xffffu), (int)(s0 >> 16), pay, i0, phis);
            Fn::edge_rec(recs, (int)(s1 & 0xffffu), (int)(s1 >> 16), pay, i1, phis);
        } else {
            Fn::edge_rec(recs, (int)(s0 & 0xffffu), (int)(s0 >> 16), pay, i0, phis);
        }
    }
    if constexpr (W > 0) {
        if (tid == 0) Fn::zero_phi(phis, d.s);                         // sentinel record
    }
}

// phase B: one thread per local vertex sums its incidence list (fixed order) and writes
template <class Fn, int BLOCK, int W>
__device__ __forceinline__ void reduce_write(const Stage<Fn> &S, const PipeArgs &a, unsigned char *sm) {
    const int tid = threadIdx.x;
    const PartDesc &d = S.d;
    const int L = d.nO + d.nH;
    const float *rows = S.rows();
    const float *phis = reinterpret_cast<const float *>(sm + a.off_phi);
    const uint16_t *inc = S.inc();
    const float *vc = S.vc();
    const int32_t *hpos = S.halo_pos();
    for (int j = tid; j < L; j += BLOCK) {
        float acc[Fn::ROW];
#pragma unroll
        for (int c = 0; c < Fn::ROW; c++) acc[c] = 0.0f;
        if constexpr (W > 0) {
            uint32_t w2[W / 2];   // W u16 entries, read as W/2 words (the list is 8-byte aligned)
            if constexpr (W == 4) {
                const uint2 v = *reinterpret_cast<const uint2 *>(inc + 4 * j);
                w2[0] = v.x; w2[1] = v.y;
            } else {
                const uint4 v = *reinterpret_cast<const uint4 *>(inc + 8 * j);
                w2[0] = v.x; w2[1] = v.y; w2[2] = v.z; w2[3] = v.w;
            }
#pragma unroll
            for (int r = 0; r < W; r++) {
                const uint32_t w = (w2[r >> 1] >> (16 * (r & 1))) & 0xffffu;
                Fn::gather_rec(phis, (int)(w >> 1), (int)(w & 1), acc);
            }
        } else {
            const uint16_t *ioff = S.inc_off();
            const int q0 = ioff[j], q1 = j + 1 < L ? ioff[j + 1] : 2 * d.s;
            for (int q = q0; q < q1; q++) {
                const int w = inc[q];
                Fn::gather_rec(phis, w >> 1, w & 1, acc);
            }
        }
        if (j < d.nO) {
            const float dt = Fn::kUsesConst ? vc[j] : 0.0f;
            Fn::finish_row(rows + Fn::ROW * j, acc, dt, a.state_out + (int64_t)Fn::ROW * (d.o0 + j));
        } else {
            float *hb = a.halo_buf + (int64_t)Fn::ROW * hpos[j - d.nO];
#pragma unroll
            for (int c = 0; c < Fn::ROW; c++) hb[c] = acc[c];
        }
    }
}

// Boundary finalise (a6), fused after the grid barrier: the owner rows of shared vertices
// already hold U + dt F_owner; add dt * (their halo partials, contiguous in halo_buf) in a
// fixed order. Threads past S copy (cfd) or clear (gather-scatter, SpMV) untouched rows.
template <class Fn>
__device__ __forceinline__ void finalise_item(const PipeArgs &a, int64_t t) {
    if (t < a.S) {
        const int64_t v = a.shared_ids[t];
        const int q0 = a.hv_off[t], q1 = a.hv_off[t + 1];
        float acc[Fn::ROW];
#pragma unroll
        for (int c = 0; c < Fn::ROW; c++) acc[c] = 0.0f;
        for (int q = q0; q < q1; q++) {
#pragma unroll
            for (int c = 0; c < Fn::ROW; c++) acc[c] += a.halo_buf[(int64_t)Fn::ROW * q + c];
        }
        const float dt = Fn::kUsesConst ? a.vconst[v] : 0.0f;
        Fn::finalise_add(a.state_out + Fn::ROW * v, acc, dt);
        return;
    }
    const int64_t v = a.touched + (t - a.S);
    if (v < a.n) Fn::untouched(a.state_in + Fn::ROW * v, a.state_out + Fn::ROW * v);
}

// Schedule of one CTA over its partitions q_0, q_1, ... (a balanced static list) with
// `ns` stage buffers (2, or 1 for large partitions) and a 3-slot ring of halo-id lists:
//   end of iteration t: bulk(q_{t+ns}) -> stage t % ns, hid(q_{t+ns+1}) -> ring,
//                       gather(q_{t+ns}) (its ids landed an iteration ago) -> stage t % ns
//   top of iteration t: wait bulk(q_t) and gather(q_t), then compute q_t
// so both the bulk copies and the row gathers have a whole iteration to land. All CTAs
// are co-resident (grid = SMs x occupancy); the finalise follows a grid-wide barrier.
template <class Fn, int BLOCK, int W>
__global__ void __launch_bounds__(BLOCK, 1) k_edge_tma(PipeArgs a) {
    extern __shared__ __align__(128) unsigned char pipe_smem[];
    unsigned char *sm = pipe_smem;
    __shared__ __align__(8) uint64_t bar[2], hbar[3];
    __shared__ PartDesc dsm[2];
    const int tid = threadIdx.x;
    const int64_t G = gridDim.x;
    const int ns = a.nstage;
    const int32_t lbeg = a.cta_begin[blockIdx.x], nmine = a.cta_begin[blockIdx.x + 1] - lbeg;
    const int32_t *mine = a.cta_list + lbeg;       // this CTA's partitions, in order
    if (nmine > 0) {
        if (tid == 0) {
            ptx::mbar_init(&bar[0], 1);
            ptx::mbar_init(&bar[1], 1);
            ptx::mbar_init(&hbar[0], 1);
            ptx::mbar_init(&hbar[1], 1);
            ptx::mbar_init(&hbar[2], 1);
            ptx::fence_mbar_init();
        }
        __syncthreads();
        uint32_t ph = 0;   // phase bits: stage barriers 0-1, ring barriers 2-4
        auto wait_bar = [&](uint64_t *b, int bit) {
            ptx::mbar_wait(b, (ph >> bit) & 1u);
            ph ^= 1u << bit;
        };
        auto stage_base = [&](int st) { return sm + (size_t)st * a.stage_bytes; };
        auto hid_slot = [&](int t) {
            return reinterpret_cast<int32_t *>(sm + a.off_hid + (size_t)(t % 3) * a.hid_slot_bytes);
        };
        // thread 0 keeps descriptors of q_{t+ns} and q_{t+ns+1} in registers
        PartDesc dnext, dnext2;
        if (tid == 0) {
            const PartDesc d0 = a.desc[mine[0]];
            const PartDesc d1 = nmine > 1 ? a.desc[mine[1]] : d0;
            const PartDesc d2 = nmine > 2 ? a.desc[mine[2]] : d0;
            Stage<Fn>(d0, nullptr, a).issue_hid(hid_slot(0), &hbar[0]);
            if (nmine > 1) Stage<Fn>(d1, nullptr, a).issue_hid(hid_slot(1), &hbar[1]);
            if (ns == 2 && nmine > 2) Stage<Fn>(d2, nullptr, a).issue_hid(hid_slot(2), &hbar[2]);
            dsm[0] = d0;
            Stage<Fn>(d0, stage_base(0), a).issue_bulk(&bar[0]);
            if (ns == 2 && nmine > 1) {
                dsm[1] = d1;
                Stage<Fn>(d1, stage_base(1), a).issue_bulk(&bar[1]);
            }
            dnext = ns == 2 ? d2 : d1;
        }
        __syncthreads();
        for (int j = 0; j < ns && j < nmine; j++) {
            wait_bar(&hbar[j], 2 + j);
            Stage<Fn>(dsm[j], stage_base(j), a).template issue_gather<BLOCK>(hid_slot(j));
            ptx::cp_async_commit();
        }
        for (int t = 0; t < nmine; t++) {
            const int st = ns == 2 ? (t & 1) : 0;
            const bool has_issue = t + ns < nmine, has_hid = t + ns + 1 < nmine;
            if (tid == 0 && has_hid) dnext2 = a.desc[mine[t + ns + 1]];   // consumed at the end
            EPG_TP(t, 0);
            wait_bar(&bar[st], st);                                       // bulk(q_t)
            EPG_TP(t, 2);
            if (ns == 2 && t + 1 < nmine) ptx::cp_async_wait<1>();        // gather(q_t)
            else ptx::cp_async_wait<0>();
            EPG_TP(t, 3);
            __syncthreads();
            EPG_TP(t, 1);
            const Stage<Fn> cur(dsm[st], stage_base(st), a);
            compute_edges<Fn, BLOCK, W>(cur, a, sm);
            __syncthreads();
            EPG_TP(t, 4);
            reduce_write<Fn, BLOCK, W>(cur, a, sm);
            __syncthreads();
            EPG_TP(t, 5);
            if (has_issue) {
                if (tid == 0) {
                    ptx::fence_proxy_async_smem();
                    dsm[st] = dnext;
                    Stage<Fn>(dnext, stage_base(st), a).issue_bulk(&bar[st]);
                    if (has_hid) Stage<Fn>(dnext2, nullptr, a).issue_hid(hid_slot(t + ns + 1), &hbar[(t + ns + 1) % 3]);
                    dnext = dnext2;
                }
                __syncthreads();
                EPG_TP(t, 6);
                wait_bar(&hbar[(t + ns) % 3], 2 + (t + ns) % 3);          // ids of q_{t+ns}
                Stage<Fn>(dsm[st], stage_base(st), a).template issue_gather<BLOCK>(hid_slot(t + ns));
                ptx::cp_async_commit();
                EPG_TP(t, 7);
            }
        }
    }
    grid_barrier(a.bar_ctr, a.bar_target);
    EPG_TP(15, 6);
    const int64_t fin = a.S + (a.n - a.touched);
    for (int64_t t = blockIdx.x * (int64_t)BLOCK + tid; t < fin; t += G * BLOCK) finalise_item<Fn>(a, t);
    EPG_TP(15, 7);
}

// blob of partition p (layout above)
__global__ void k_build_blob(const int32_t *__restrict__ peb, const int32_t *__restrict__ pvb,
                             const int32_t *__restrict__ hb, const int32_t *__restrict__ halo_ids,
                             const int32_t *__restrict__ halo_pos, const uint32_t *__restrict__ slots,
                             const uint16_t *__restrict__ inc, const uint16_t *__restrict__ inc_off,
                             const int32_t *__restrict__ blob16, const int32_t *__restrict__ hid16, int W,
                             unsigned char *blob, int32_t *hid_blob, PartDesc *desc) {
    const int p = blockIdx.x;
    const int o0 = pvb[p], nO = pvb[p + 1] - o0, h0 = hb[p], nH = hb[p + 1] - h0, e0 = peb[p], s = peb[p + 1] - e0;
    const int L = nO + nH;
    unsigned char *b = blob + 16 * (int64_t)blob16[p];
    int32_t *hid = hid_blob + 4 * (int64_t)hid16[p];
    int32_t *hpos = reinterpret_cast<int32_t *>(b);
    uint32_t *sl = reinterpret_cast<uint32_t *>(hpos + nH);
    uint16_t *ic = reinterpret_cast<uint16_t *>(b + blob_inc_offset(nH, s));
    for (int j = threadIdx.x; j < nH; j += blockDim.x) { hid[j] = halo_ids[h0 + j]; hpos[j] = halo_pos[h0 + j]; }
    for (int i = threadIdx.x; i < s; i += blockDim.x) sl[i] = slots[e0 + i];
    const int64_t lbase = (int64_t)o0 + h0;
    if (W > 0) {
        for (int j = threadIdx.x; j < L; j += blockDim.x) {
            const int q0 = inc_off[lbase + j], q1 = j + 1 < L ? inc_off[lbase + j + 1] : 2 * s;
            for (int r = 0; r < W; r++)
                ic[W * j + r] = q0 + r < q1 ? inc[2 * (int64_t)e0 + q0 + r] : (uint16_t)(s << 1);
        }
    } else {
        uint16_t *io = ic + 2 * s;
        for (int q = threadIdx.x; q < 2 * s; q += blockDim.x) ic[q] = inc[2 * (int64_t)e0 + q];
        for (int j = threadIdx.x; j < L; j += blockDim.x) io[j] = inc_off[lbase + j];
    }
    if (threadIdx.x == 0)
        desc[p] = PartDesc{o0, nO, e0, s, h0, nH, blob16[p], blob_bytes_for(nH, s, L, W), hid16[p], 0, 0, 0};
}

__global__ void k_blob_sizes(const int32_t *__restrict__ peb, const int32_t *__restrict__ pvb,
                             const int32_t *__restrict__ hb, int64_t k, int W, int32_t *units16,
                             int32_t *hid_units16) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p > k) return;
    if (p == k) { units16[p] = 0; hid_units16[p] = 0; return; }
    const int nO = pvb[p + 1] - pvb[p], nH = hb[p + 1] - hb[p], s = peb[p + 1] - peb[p];
    units16[p] = blob_bytes_for(nH, s, nO + nH, W) / 16;
    hid_units16[p] = hid_bytes_for(nH) / 16;
}

// largest number of incidences of one local vertex in its partition (all partitions)
__global__ void k_max_local_degree(const int32_t *__restrict__ peb, const int32_t *__restrict__ pvb,
                                   const int32_t *__restrict__ hb, const uint16_t *__restrict__ inc_off, int64_t k,
                                   int32_t *out) {
    const int p = blockIdx.x;
    const int o0 = pvb[p], L = pvb[p + 1] - o0 + hb[p + 1] - hb[p], s = peb[p + 1] - peb[p];
    const int64_t lbase = (int64_t)o0 + hb[p];
    int m = 0;
    for (int j = threadIdx.x; j < L; j += blockDim.x) {
        const int q1 = j + 1 < L ? inc_off[lbase + j + 1] : 2 * s;
        m = max(m, q1 - (int)inc_off[lbase + j]);
    }
    atomicMax(out, m);
}

// halo_pos[h] = position of halo entry h in the vertex-grouped order (inverse of hv_list)
__global__ void k_halo_pos(const int32_t *__restrict__ hv_list, int64_t C, int32_t *halo_pos) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < C) halo_pos[hv_list[r]] = (int32_t)r;
}

}  // namespace epg
