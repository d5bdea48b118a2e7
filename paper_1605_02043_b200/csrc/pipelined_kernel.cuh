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
//           partial sum to the vertex-grouped halo buffer; k_finalise2 adds those to
//           the owners' rows (fixed order: deterministic).
#pragma once

#include <stdint.h>

#include "functors.cuh"
#include "ptx.cuh"

namespace epg {

struct PartDesc {
    int32_t o0, nO, e0, s, h0, nH, blob16, blob_bytes;
};

struct PipeArgs {
    const PartDesc *desc;
    const unsigned char *blob;
    const float *state_in;
    float *state_out;
    const float *payload;   // NULL when the functor runs without one (gather-scatter, w = 1)
    const float *vconst;    // cfd dt
    float *halo_buf;        // [C][ROW], grouped by vertex
    int64_t k;
    int nstage;             // 1 or 2
    int stage_bytes, off_rows, off_pay, off_vc;  // byte offsets inside a stage (blob at 0)
    int off_spd, off_phi;                        // working arrays after the stages
    int Scap;
};

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
    __device__ const int32_t *halo_ids() const { return reinterpret_cast<const int32_t *>(base); }
    __device__ const int32_t *halo_pos() const { return halo_ids() + d.nH; }
    __device__ const uint32_t *slots() const { return reinterpret_cast<const uint32_t *>(halo_pos() + d.nH); }
    __device__ const uint16_t *inc() const { return reinterpret_cast<const uint16_t *>(slots() + d.s); }
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

    // all threads, after the bulk copies landed: ragged words + halo row gathers
    template <int BLOCK>
    __device__ void issue_gather() const {
        const int tid = threadIdx.x;
        if (tid < 32) {
            region_ragged(s_rows_base(), g_rows(), rows_bytes(), tid);
            if (a.payload) region_ragged(s_pay_base(), g_pay(), pay_bytes(), tid);
            if (Fn::kUsesConst) region_ragged(s_vc_base(), g_vc(), vc_bytes(), tid);
        }
        float *r = rows() + Fn::ROW * d.nO;
        const int32_t *hid = halo_ids();
        for (int w = tid; w < Fn::ROW * d.nH; w += BLOCK) {
            const int j = w / Fn::ROW, c = w - j * Fn::ROW;
            ptx::cp_async4(r + w, a.state_in + (int64_t)Fn::ROW * hid[j] + c);
        }
    }
};

template <class Fn, int BLOCK>
__device__ __forceinline__ void compute_partition(const Stage<Fn> &S, const PipeArgs &a, unsigned char *sm) {
    const int tid = threadIdx.x;
    const PartDesc &d = S.d;
    const int L = d.nO + d.nH;
    float *rows = S.rows();
    float *spd = reinterpret_cast<float *>(sm + a.off_spd);
    float *Phi = reinterpret_cast<float *>(sm + a.off_phi);
    if (Fn::kDerived) {
        for (int j = tid; j < L; j += BLOCK) spd[j] = Fn::derive(rows + Fn::ROW * j);
        __syncthreads();
    }
    const uint32_t *slots = S.slots();
    const float *pay = S.pay();
    for (int i = tid; i < d.s; i += BLOCK) {
        const uint32_t sl = slots[i];
        Fn::edge2(rows, spd, (int)(sl & 0xffffu), (int)(sl >> 16), pay, i, Phi, a.Scap);
    }
    __syncthreads();
    const uint16_t *inc = S.inc(), *ioff = S.inc_off();
    const float *vc = S.vc();
    const int32_t *hpos = S.halo_pos();
    for (int j = tid; j < L; j += BLOCK) {
        const int q0 = ioff[j], q1 = j + 1 < L ? ioff[j + 1] : 2 * d.s;
        float acc[Fn::ROW];
#pragma unroll
        for (int c = 0; c < Fn::ROW; c++) acc[c] = 0.0f;
        for (int q = q0; q < q1; q++) {
            const int w = inc[q];
            Fn::gather(Phi, a.Scap, w >> 1, w & 1, acc);
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

template <class Fn, int BLOCK>
__global__ void __launch_bounds__(BLOCK, 1) k_edge_tma(PipeArgs a) {
    extern __shared__ __align__(128) unsigned char pipe_smem[];
    unsigned char *sm = pipe_smem;
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ PartDesc dsm[2];
    const int tid = threadIdx.x;
    const int64_t G = gridDim.x;
    const int64_t q0 = blockIdx.x;
    if (q0 >= a.k) return;
    const int ns = a.nstage;
    if (tid == 0) {
        ptx::mbar_init(&bar[0], 1);
        ptx::mbar_init(&bar[1], 1);
        ptx::fence_mbar_init();
    }
    __syncthreads();
    uint32_t phase0 = 0, phase1 = 0;
    auto wait_stage = [&](int st) {
        if (st == 0) { ptx::mbar_wait(&bar[0], phase0); phase0 ^= 1u; }
        else { ptx::mbar_wait(&bar[1], phase1); phase1 ^= 1u; }
    };
    auto stage_base = [&](int st) { return sm + (size_t)st * a.stage_bytes; };
    // prologue: partitions q0 (stage 0) and, double-buffered, q0 + G (stage 1)
    if (tid == 0) {
        dsm[0] = a.desc[q0];
        Stage<Fn>(dsm[0], stage_base(0), a).issue_bulk(&bar[0]);
        if (ns == 2 && q0 + G < a.k) {
            dsm[1] = a.desc[q0 + G];
            Stage<Fn>(dsm[1], stage_base(1), a).issue_bulk(&bar[1]);
        }
    }
    __syncthreads();
    wait_stage(0);
    Stage<Fn>(dsm[0], stage_base(0), a).template issue_gather<BLOCK>();
    ptx::cp_async_commit();

    PartDesc dpre;
    for (int64_t t = 0;; t++) {
        const int64_t q = q0 + t * G;
        if (q >= a.k) break;
        const int st = ns == 2 ? (int)(t & 1) : 0;
        const int64_t qnext = q + G, qissue = q + ns * G;
        if (tid == 0 && qissue < a.k) dpre = a.desc[qissue];     // consumed after compute
        if (ns == 2 && qnext < a.k) {
            wait_stage(st ^ 1);
            Stage<Fn>(dsm[st ^ 1], stage_base(st ^ 1), a).template issue_gather<BLOCK>();
            ptx::cp_async_commit();
            ptx::cp_async_wait<1>();
        } else {
            ptx::cp_async_wait<0>();
        }
        __syncthreads();
        compute_partition<Fn, BLOCK>(Stage<Fn>(dsm[st], stage_base(st), a), a, sm);
        __syncthreads();
        if (qissue < a.k) {
            if (tid == 0) {
                ptx::fence_proxy_async_smem();
                dsm[st] = dpre;
                Stage<Fn>(dsm[st], stage_base(st), a).issue_bulk(st == 0 ? &bar[0] : &bar[1]);
            }
            if (ns == 1) {
                __syncthreads();
                wait_stage(0);
                Stage<Fn>(dsm[0], stage_base(0), a).template issue_gather<BLOCK>();
                ptx::cp_async_commit();
            }
        }
        __syncthreads();
    }
}

// blob of partition p: halo ids | halo result positions | slots | incidence | inc offsets
__global__ void k_build_blob(const int32_t *__restrict__ peb, const int32_t *__restrict__ pvb,
                             const int32_t *__restrict__ hb, const int32_t *__restrict__ halo_ids,
                             const int32_t *__restrict__ halo_pos, const uint32_t *__restrict__ slots,
                             const uint16_t *__restrict__ inc, const uint16_t *__restrict__ inc_off,
                             const int32_t *__restrict__ blob16, unsigned char *blob, PartDesc *desc) {
    const int p = blockIdx.x;
    const int o0 = pvb[p], nO = pvb[p + 1] - o0, h0 = hb[p], nH = hb[p + 1] - h0, e0 = peb[p], s = peb[p + 1] - e0;
    const int L = nO + nH;
    unsigned char *b = blob + 16 * (int64_t)blob16[p];
    int32_t *hid = reinterpret_cast<int32_t *>(b);
    int32_t *hpos = hid + nH;
    uint32_t *sl = reinterpret_cast<uint32_t *>(hpos + nH);
    uint16_t *ic = reinterpret_cast<uint16_t *>(sl + s);
    uint16_t *io = ic + 2 * s;
    for (int j = threadIdx.x; j < nH; j += blockDim.x) { hid[j] = halo_ids[h0 + j]; hpos[j] = halo_pos[h0 + j]; }
    for (int i = threadIdx.x; i < s; i += blockDim.x) sl[i] = slots[e0 + i];
    for (int q = threadIdx.x; q < 2 * s; q += blockDim.x) ic[q] = inc[2 * (int64_t)e0 + q];
    const int64_t lbase = (int64_t)o0 + h0;
    for (int j = threadIdx.x; j < L; j += blockDim.x) io[j] = inc_off[lbase + j];
    if (threadIdx.x == 0) {
        const int bytes = 8 * nH + 8 * s + 2 * L;
        desc[p] = PartDesc{o0, nO, e0, s, h0, nH, blob16[p], (bytes + 15) & ~15};
    }
}

__global__ void k_blob_sizes(const int32_t *__restrict__ peb, const int32_t *__restrict__ pvb,
                             const int32_t *__restrict__ hb, int64_t k, int32_t *units16) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p > k) return;
    if (p == k) { units16[p] = 0; return; }
    const int nO = pvb[p + 1] - pvb[p], nH = hb[p + 1] - hb[p], s = peb[p + 1] - peb[p];
    units16[p] = (8 * nH + 8 * s + 2 * (nO + nH) + 15) / 16;
}

// halo_pos[h] = position of halo entry h in the vertex-grouped order (inverse of hv_list)
__global__ void k_halo_pos(const int32_t *__restrict__ hv_list, int64_t C, int32_t *halo_pos) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < C) halo_pos[hv_list[r]] = (int32_t)r;
}

// boundary finalise for the pipelined kernel: owner rows already hold U + dt F_owner;
// add dt * (sum of the vertex's halo partials, contiguous in halo_buf), in order.
template <class Fn>
__global__ void k_finalise2(const int32_t *__restrict__ shared_ids, const int32_t *__restrict__ hv_off,
                            const float *__restrict__ halo_buf, const float *__restrict__ state_in,
                            float *__restrict__ state_out, const float *__restrict__ vconst, int32_t S,
                            int64_t touched, int64_t n) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < S) {
        const int64_t v = shared_ids[t];
        const int q0 = hv_off[t], q1 = hv_off[t + 1];
        float acc[Fn::ROW];
#pragma unroll
        for (int c = 0; c < Fn::ROW; c++) acc[c] = 0.0f;
        for (int q = q0; q < q1; q++) {
#pragma unroll
            for (int c = 0; c < Fn::ROW; c++) acc[c] += halo_buf[(int64_t)Fn::ROW * q + c];
        }
        const float dt = Fn::kUsesConst ? vconst[v] : 0.0f;
        Fn::finalise_add(state_out + Fn::ROW * v, acc, dt);
        return;
    }
    const int64_t v = touched + (t - S);
    if (v < n) Fn::untouched(state_in + Fn::ROW * v, state_out + Fn::ROW * v);
}

}  // namespace epg
