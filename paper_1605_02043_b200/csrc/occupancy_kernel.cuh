// occupancy_kernel.cuh -- the B200 staged edge kernel (step a5), one CTA per execution
// partition, several CTAs resident per SM.
//
// Per partition p (the paper's thread block; staging as in P:719-724):
//   0. before the PDL wait (plan data only): the descriptor, one thread's 1-D TMA bulk copies of
//      the plan blob (halo ids, incidence lists, record placement) and of the partition's slots,
//      edge payload and dt (into the Phi space, dead until the edge phase), the halo ids of a
//      halo-light partition and, in single-wave grids, L2 prefetches of its state rows;
//   1. after the wait: a bulk copy of its owned state rows O_p, a contiguous range of the cpack
//      layout, and the halo rows H_p (the C = sum_v (p_v - 1) redundant loads of Eq. (1)),
//      gathered with cp.async into the same shared array;
//   2. each staged row is turned in place into a derived record (two float4 halves in two
//      arrays, at the placed position of place_kernels.cuh);
//   3. one thread per edge evaluates the interaction from shared memory into a Phi record;
//   4. one thread per local vertex sums its incidence list in a fixed order (no atomics);
//   5. owned results U + dt F and the halo partial sums are packed in shared memory and
//      written back with two TMA bulk stores (contiguous: the owned range of state_out,
//      the partition's slice of the halo buffer).
// The boundary finalise (k_finalise_rec16) then adds the halo partials of shared vertices
// (p_v > 1) to their owners' rows in a fixed order. Latency is hidden by occupancy (3-4 CTAs per
// SM) and programmatic dependent launch rather than by an explicit pipeline; execution
// partitions are bounded so every buffer fits.
#pragma once

#include <stdint.h>

#include "functors.cuh"
#include "pipelined_kernel.cuh"
#include "ptx.cuh"

namespace epg {

// blob of the occupancy kernel: [halo ids nH x i32] ([hub index nH x i32] when the plan has
// hubs: hw = 2 words per halo row) pad16 [incidence] (W as in the pipelined blob: W x L u16
// padded lists, or W = 0: 2s u16 entries + L u16 offsets) pad16 [placement: L x u8, the
// in-group position of each local vertex's derived record, place_kernels.cuh]
__host__ __device__ __forceinline__ int blob3_inc_offset(int nH, int hw = 1) { return (4 * hw * nH + 15) & ~15; }
__host__ __device__ __forceinline__ int blob3_col_offset(int nH, int s, int L, int W, int hw = 1) {
    const int inc = W > 0 ? 2 * W * L : 4 * s + 2 * L;
    return (blob3_inc_offset(nH, hw) + inc + 15) & ~15;
}
// padded incidence entries point at Phi record `sentinel` (the plan's largest execution
// partition, >= every edge index), kept zero by the kernel
__host__ __device__ __forceinline__ int blob3_bytes_for(int nH, int s, int L, int W, int hw = 1) {
    return (blob3_col_offset(nH, s, L, W, hw) + L + 15) & ~15;
}

struct OccArgs {
    const PartDesc *desc;      // blob16 / blob_bytes refer to blob3
    const unsigned char *blob;
    const uint32_t *slots;     // [m] packed endpoint slots
    const float *state_in;
    float *state_out;
    const float *payload;      // NULL: gather-scatter with w = 1
    const float *vconst;
    float *halo_buf;           // [C][ROW] in halo (partition) order
    int off_recs, rows_land, off_phi;
    int64_t first;             // this launch runs execution partitions first .. first + grid
    int hw;                    // blob words per halo row (2: hub indices follow the halo ids)
    float *hub_acc;            // [hubs][ROW] or NULL: hub partials are added here as well
    int early_pdl;             // 1: trigger dependents at the start (single-wave grids)
    int sentinel;              // zero Phi record of padded incidence entries (plan Scap)
    int pstride;               // records of the split Phi layout (>= sentinel + 1, multiple of 4)
    int rstride;               // float4s from a derived record's first half to its second (REC = 8)
    int prewait_pf;            // single-wave grids: L2-prefetch the state rows before the PDL wait
    int64_t ahead;             // > 0 (multi-wave grids): L2-prefetch partition x + ahead's ranges
    int64_t count;             // execution partitions of this launch
    // the partition's endpoint slots, edge payload and dt are bulk-copied into the Phi space
    // (dead until the edge phase) at these byte offsets from off_phi
    int st_slots, st_pay, st_vc;
    const float *state_end;    // one past the last row of state_in (bound of the 32-byte halo reads)
    const int32_t *order;      // NULL, or the execution partitions of this launch are order[first + b]
                               // (multi-GPU: a shard's interior partitions, then its boundary ones)
    // multi-GPU peer push (EPG_EXCHANGE=p2p): the partial of a halo row owned by a lower rank p
    // is added straight into rank p's accumulator (peer memory over NVLink) by this kernel
    float *const *peer_acc;    // [G] accumulators of the ranks, or NULL
    const int32_t *vlo;        // [G + 1] first cpack row of each rank's shard
    int rank;                  // this rank
};

__device__ __forceinline__ int64_t occ_part(const OccArgs &a, int64_t x) { return a.order ? a.order[x] : x; }

// the 8 fields of a descriptor the occupancy kernel reads (o0 .. blob_bytes), as two 128-bit
// loads (descriptors are 48-byte records, 16-byte aligned) instead of one 32-bit load each
__device__ __forceinline__ PartDesc load_desc8(const PartDesc *p) {
    const int4 *q = reinterpret_cast<const int4 *>(p);
    const int4 x = __ldg(q), y = __ldg(q + 1);
    PartDesc d;
    d.o0 = x.x; d.nO = x.y; d.e0 = x.z; d.s = x.w;
    d.h0 = y.x; d.nH = y.y; d.blob16 = y.z; d.blob_bytes = y.w;
    return d;
}

// L2 prefetch of the aligned body of [g, g + bytes)
__device__ __forceinline__ void prefetch_region(const void *g, uint32_t bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(g);
    const uintptr_t lo = (a + 15) & ~uintptr_t(15), hi = (a + bytes) & ~uintptr_t(15);
    if (hi > lo) ptx::bulk_prefetch_l2(reinterpret_cast<const void *>(lo), (uint32_t)(hi - lo));
}

// EPG_OCC_MINB (experiments): minimum resident CTAs per SM the register allocation targets
#ifdef EPG_OCC_MINB
#define EPG_OCC_BOUNDS(b) __launch_bounds__(b, EPG_OCC_MINB)
#else
#define EPG_OCC_BOUNDS(b) __launch_bounds__(b)
#endif
template <class Fn, int BLOCK, int EPT, int VPT, int W>
__global__ void EPG_OCC_BOUNDS(BLOCK) k_edge_occ(OccArgs a) {
    extern __shared__ __align__(128) unsigned char occ_smem[];
    __shared__ __align__(8) uint64_t bar;
    constexpr int ROW = Fn::ROW, PW = Fn::PAYW;
    const int tid = threadIdx.x;
    EPG_TP(0, 0);
    const PartDesc d = load_desc8(a.desc + occ_part(a, a.first + blockIdx.x));
    const int L = d.nO + d.nH;
    unsigned char *sblob = occ_smem;
    const uint8_t *scol = sblob + blob3_col_offset(d.nH, d.s, L, W, a.hw);   // record placement
    float *recs = reinterpret_cast<float *>(occ_smem + a.off_recs);
    float *phis = reinterpret_cast<float *>(occ_smem + a.off_phi);
    float *recsB = recs + 4 * a.rstride;         // second halves of the derived records (REC = 8)
    float *phisB = phis + 4 * a.pstride;         // Phi_4 of the split Phi records
    const float *g_rows = a.state_in + (int64_t)ROW * d.o0;
    unsigned char *rows_base = occ_smem + a.off_recs + a.rows_land;   // upper part of the record array
    float *rows = reinterpret_cast<float *>(rows_base + (reinterpret_cast<uintptr_t>(g_rows) & 15));
    const uint32_t rows_bytes = 4u * ROW * d.nO;
    // Programmatic dependent launch: everything up to pdl_wait() reads only plan data and
    // may overlap the previous kernel in the stream (the finalise of the previous step).
    // static per-partition ranges (all contiguous after the remap), staged in the Phi space
    const uint32_t *g_sl = a.slots + d.e0;
    const float *g_pay = a.payload ? a.payload + (int64_t)PW * d.e0 : nullptr;
    const float *g_vc = Fn::kUsesConst ? a.vconst + d.o0 : nullptr;
    unsigned char *st_sl = occ_smem + a.off_phi + a.st_slots, *st_pay = occ_smem + a.off_phi + a.st_pay,
                  *st_vc = occ_smem + a.off_phi + a.st_vc;
    const uint32_t sl_bytes = 4u * d.s, pay_bytes = 4u * PW * d.s, vc_bytes = 4u * d.nO;
    if (tid == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_mbar_init();
        uint32_t tx = (uint32_t)d.blob_bytes + region_body(g_rows, rows_bytes) + region_body(g_sl, sl_bytes);
        if (g_pay) tx += region_body(g_pay, pay_bytes);
        if (g_vc) tx += region_body(g_vc, vc_bytes);
        ptx::mbar_arrive_expect_tx(&bar, tx);
        if (d.blob_bytes) ptx::bulk_g2s(sblob, a.blob + 16 * (int64_t)d.blob16, (uint32_t)d.blob_bytes, &bar);
        region_bulk(st_sl, g_sl, sl_bytes, &bar);
        if (g_pay) region_bulk(st_pay, g_pay, pay_bytes, &bar);
        if (g_vc) region_bulk(st_vc, g_vc, vc_bytes, &bar);
    }
    // multi-wave grids: the partition one resident wave ahead will need its contiguous ranges;
    // its descriptor is loaded now (in flight during this CTA's copies) and the ranges are
    // prefetched into L2 once this CTA's data has landed, so that CTA's first dependent DRAM
    // trips become L2 hits
    const bool ahead = a.ahead > 0 && tid == 32 && blockIdx.x + a.ahead < a.count;
    PartDesc f;                                    // read only by the `ahead` thread
    if (ahead) f = load_desc8(a.desc + occ_part(a, a.first + blockIdx.x + a.ahead));
    // halo rows H_p. With few halos (nH <= nO, the EP maps) they are gathered right after the
    // wait so they fly with the bulk copies -- the halo ids open the blob, so each thread reads
    // its ids from global memory, before the wait (plan data), instead of waiting for the copy.
    // Halo-heavy partitions (the default map) gather after the copies instead: their halo rows
    // are mostly other partitions' owned rows that those CTAs' bulk copies are bringing into L2
    // at the same time.
    const bool early_halo = d.nH <= d.nO;
    int32_t hid[VPT];                               // all ids first: one round trip, not VPT
    if (early_halo) {
        const int32_t *gh = reinterpret_cast<const int32_t *>(a.blob + 16 * (int64_t)d.blob16);
#pragma unroll
        for (int r = 0; r < VPT; r++) {
            const int j = tid + r * BLOCK;
            hid[r] = j < d.nH ? __ldg(gh + j) : 0;
        }
    }
    // single-wave grids start while the previous kernel (the last step's finalise) runs: the
    // owned rows and the early halo rows are prefetched into L2 now, so the copies after the
    // wait hit L2 (a prefetch never returns stale data -- L2 is the point of coherence -- and
    // the copies themselves still wait)
    if (a.early_pdl && a.prewait_pf) {
        if (tid == 64) prefetch_region(g_rows, rows_bytes);
        if (early_halo) {
#pragma unroll
            for (int r = 0; r < VPT; r++)
                if (tid + r * BLOCK < d.nH) ptx::prefetch_l2(a.state_in + (int64_t)ROW * hid[r]);
        }
    }
    ptx::pdl_wait();                               // state_in is final from here on
    // single-wave grids: every CTA of this grid is resident, so the finalise may launch now
    // and load its (static) records on SMs with room while the edge partitions run
    if (a.early_pdl) ptx::pdl_launch_dependents();
    if (tid == 0) region_bulk(rows_base, g_rows, rows_bytes, &bar);
    // 5-float rows: every halo row lands as the aligned 32 bytes that contain it (two 16-byte
    // cp.async, L1 bypassed) after the owned rows, the row at byte 4 (h mod 4) of the 32 (20 h
    // mod 16). The two 16-byte halves of halo row j go to halo_lo + 16 j and halo_hi + 16 j, so
    // a warp quarter's cp.async writes are 16-byte contiguous (a 32-byte slot per row made
    // lanes l and l + 4 collide on one bank group). One-float rows are gathered word by word.
    // (Per-thread 32-byte TMA bulk copies instead were measured slower: a bulk copy takes
    // uniform operands, so a divergent per-lane issue becomes a loop -- C3 8,469 -> 10,035
    // warp instructions per CTA, edge kernel 1.41 -> 1.61 ms.)
    constexpr bool kChunked = ROW == 5;
    unsigned char *halo_lo = reinterpret_cast<unsigned char *>(
        (reinterpret_cast<uintptr_t>(rows + ROW * d.nO) + 15) & ~uintptr_t(15));
    unsigned char *halo_hi = halo_lo + 16 * d.nH;
    // word p (0..7) of halo row j's 32-byte window
    auto halo_word = [&](int j, int p) -> float * {
        return reinterpret_cast<float *>((p < 4 ? halo_lo : halo_hi) + 16 * j) + (p & 3);
    };
    auto gather_halo = [&]() {
        float *hr = rows + ROW * d.nO;
#pragma unroll
        for (int r = 0; r < VPT; r++) {                 // one halo row per thread and r
            const int j = tid + r * BLOCK;
            if (j < d.nH) {
                const float *src = a.state_in + (int64_t)ROW * hid[r];
                if constexpr (kChunked) {
                    const float *base = reinterpret_cast<const float *>(reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15));
                    if (base + 8 <= a.state_end) {
                        ptx::cp_async16(halo_lo + 16 * j, base);
                        ptx::cp_async16(halo_hi + 16 * j, base + 4);
                    } else {                            // the array's last row: no read past its end
                        const int p0 = (int)(src - base);
#pragma unroll
                        for (int c = 0; c < ROW; c++) ptx::cp_async4(halo_word(j, p0 + c), src + c);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < ROW; c++) ptx::cp_async4(hr + ROW * j + c, src + c);
                }
            }
        }
    };
    if (early_halo) gather_halo();
    __syncthreads();                               // barrier initialisation visible
    EPG_TP(0, 1);
    ptx::mbar_wait(&bar, 0);
    EPG_TP(0, 2);
    if (ahead) {   // L2 is the point of coherence: a prefetch never returns stale data
        prefetch_region(a.blob + 16 * (int64_t)f.blob16, (uint32_t)f.blob_bytes);
        prefetch_region(a.slots + f.e0, 4u * f.s);
        if (a.payload) prefetch_region(a.payload + (int64_t)PW * f.e0, 4u * PW * f.s);
        if (Fn::kUsesConst) prefetch_region(a.vconst + f.o0, 4u * f.nO);
        prefetch_region(a.state_in + (int64_t)ROW * f.o0, 4u * ROW * f.nO);
    }
    if (tid < 32) region_ragged(rows_base, g_rows, rows_bytes, tid);   // ragged ends of the owned range
    else if (tid < 64) region_ragged(st_sl, g_sl, sl_bytes, tid - 32);   // ... and of the staged ranges
    else if (tid < 96) { if (g_pay) region_ragged(st_pay, g_pay, pay_bytes, tid - 64); }
    else if (tid < 128) { if (g_vc) region_ragged(st_vc, g_vc, vc_bytes, tid - 96); }
    if (!early_halo) {
        const int32_t *sh = reinterpret_cast<const int32_t *>(sblob);
#pragma unroll
        for (int r = 0; r < VPT; r++) {
            const int j = tid + r * BLOCK;
            hid[r] = j < d.nH ? sh[j] : 0;
        }
        gather_halo();
    }
    ptx::cp_async_commit();
    ptx::cp_async_wait<0>();
    __syncthreads();
    EPG_TP(0, 3);
    // staged slots / payload / dt -> registers (the Phi space is overwritten by the edge phase)
    // (unpredicated: the staging areas hold EPT x BLOCK edges and VPT x BLOCK rows, and the
    // values past s / nO are never used)
    uint32_t sl[EPT];
    float pw[EPT][PW];
    {
        const uint32_t *s_sl = reinterpret_cast<const uint32_t *>(st_sl + (reinterpret_cast<uintptr_t>(g_sl) & 15));
        const float *s_pay = reinterpret_cast<const float *>(st_pay + (reinterpret_cast<uintptr_t>(g_pay) & 15));
#pragma unroll
        for (int r = 0; r < EPT; r++) sl[r] = s_sl[tid + r * BLOCK];
        if (g_pay) {
#pragma unroll
            for (int r = 0; r < EPT; r++)
#pragma unroll
                for (int c = 0; c < PW; c++) pw[r][c] = s_pay[PW * (tid + r * BLOCK) + c];
        } else {
#pragma unroll
            for (int r = 0; r < EPT; r++)
#pragma unroll
                for (int c = 0; c < PW; c++) pw[r][c] = 1.0f;
        }
    }
    float dtv[VPT];
    {
        const float *s_vc = reinterpret_cast<const float *>(st_vc + (reinterpret_cast<uintptr_t>(g_vc) & 15));
#pragma unroll
        for (int r = 0; r < VPT; r++) dtv[r] = Fn::kUsesConst ? s_vc[tid + r * BLOCK] : 0.0f;
    }
    // rows -> registers -> derived records (in place: the rows sit in the upper part)
    float rv[VPT][ROW];
#pragma unroll
    for (int r = 0; r < VPT; r++) {
        const int j = tid + r * BLOCK;
        if (j < L) {
            const float *row = rows + ROW * j;
            if (kChunked && j >= d.nO) {
                const int jh = j - d.nO, p0 = reinterpret_cast<const int32_t *>(sblob)[jh] & 3;
#pragma unroll
                for (int c = 0; c < ROW; c++) rv[r][c] = *halo_word(jh, p0 + c);
            } else {
#pragma unroll
                for (int c = 0; c < ROW; c++) rv[r][c] = row[c];
            }
        }
    }
    __syncthreads();
    float ulast[VPT];                              // last state component of the owned rows, kept for the update
#pragma unroll
    for (int r = 0; r < VPT; r++) {
        const int j = tid + r * BLOCK;
        ulast[r] = rv[r][ROW - 1];
        if (j < L) Fn::derive_occ(rv[r], recs, (j & ~7) | scol[j], recsB);   // placed record (place_kernels.cuh)
    }
    __syncthreads();
    // edges
#pragma unroll
    for (int r = 0; r < EPT; r++) {
        const int i = tid + r * BLOCK;
        if (i < d.s)   // slots hold the placed record positions; bits 29-31 the Phi record's
            Fn::edge_split(recs, (int)(sl[r] & 0xffffu), (int)((sl[r] >> 16) & 0x1fffu), pw[r],
                           (i & ~7) | (int)(sl[r] >> 29), phis, phisB, recsB);
    }
    if constexpr (W > 0) {
        if (tid == 0) Fn::zero_split(phis, a.sentinel, phisB);
    }
    __syncthreads();
    EPG_TP(0, 4);
    // reduce per local vertex into registers
    const uint16_t *inc = reinterpret_cast<const uint16_t *>(sblob + blob3_inc_offset(d.nH, a.hw));
    // One-float rows with variable-length incidence lists (power-law graphs: a hub can hold most
    // of a partition's edges, and one thread summing its list stalls the whole CTA at the next
    // barrier): the 2s entries, in list order, are cut evenly over the threads and summed by a
    // block-wide segmented scan -- each thread sums its entries in order, the open segment
    // carries flow through a fixed shuffle tree, so the order is fixed (deterministic). The
    // vertex totals land in the record array (dead for these functors after the edge phase).
    constexpr bool kSegScan = (W == 0 && ROW == 1);
    float *tot = recs;
    if constexpr (kSegScan) {
        __shared__ float seg_wv[BLOCK / 32];
        __shared__ int seg_wf[BLOCK / 32];
        constexpr int IPT = 2 * EPT;
        const int ne = 2 * d.s;
        const uint16_t *ioff = inc + 2 * d.s;
        const int q0 = tid * IPT, q1 = min(q0 + IPT, ne);
        int j = 0;
        if (q0 < ne) {                                  // largest j with ioff[j] <= q0
            int lo = 0, hi = L - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if ((int)ioff[mid] <= q0) lo = mid;
                else hi = mid - 1;
            }
            j = lo;
        }
        const int j0 = j;
        const bool cont0 = q0 < ne && (int)ioff[j0] < q0;   // the first segment began before q0
        int bnd = j + 1 < L ? (int)ioff[j + 1] : ne;
        float part = 0.0f, first_part = 0.0f;
        bool first_closed = false;
        for (int q = q0; q < q1; q++) {
            if (q == bnd) {                             // segment j ended at q - 1
                if (j == j0) { first_part = part; first_closed = true; }
                else tot[j] = part;
                part = 0.0f;
                j++;
                bnd = j + 1 < L ? (int)ioff[j + 1] : ne;
            }
            const int w = inc[q];
            float v[1] = {0.0f};
            Fn::gather_split(phis, w >> 1, w & 1, v, phisB);
            part += v[0];
        }
        // carry of the open segment across threads: inclusive scan of (starts, value) with
        // (a, b) -> (a.f | b.f, b.f ? b.v : a.v + b.v); the exclusive value is the carry in
        const int starts = q0 < ne ? ((j != j0 || !cont0) ? 1 : 0) : 0;
        int f = starts;
        float sv = q0 < ne ? part : 0.0f;
        const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float ov = __shfl_up_sync(0xffffffffu, sv, o);
            const int of = __shfl_up_sync(0xffffffffu, f, o);
            if (lane >= o && !f) sv += ov;
            if (lane >= o) f |= of;
        }
        if (lane == 31) { seg_wv[wid] = sv; seg_wf[wid] = f; }
        __syncthreads();
        float pv = 0.0f;                                // prefix of the earlier warps
        for (int w = 0; w < wid; w++) pv = seg_wf[w] ? seg_wv[w] : pv + seg_wv[w];
        const float incl_prev = __shfl_up_sync(0xffffffffu, sv, 1);
        const int f_prev = __shfl_up_sync(0xffffffffu, f, 1);
        const float carry = lane == 0 ? pv : (f_prev ? incl_prev : pv + incl_prev);
        if (q0 < ne) {
            if (first_closed) tot[j0] = (cont0 ? carry : 0.0f) + first_part;
            if (bnd == q1 || q1 == ne) tot[j] = (j == j0 && cont0 ? carry : 0.0f) + part;
        }
        __syncthreads();
    }
    float out[VPT][ROW];
    bool pushed = false;                           // this thread added partials into peer memory
#pragma unroll
    for (int r = 0; r < VPT; r++) {
        const int j = tid + r * BLOCK;
        if (j >= L) continue;
        float acc[ROW];
#pragma unroll
        for (int c = 0; c < ROW; c++) acc[c] = 0.0f;
        if constexpr (W > 0) {
            uint32_t w2[W / 2];
            if constexpr (W == 4) {
                const uint2 v = *reinterpret_cast<const uint2 *>(inc + 4 * j);
                w2[0] = v.x; w2[1] = v.y;
            } else {
                const uint4 v = *reinterpret_cast<const uint4 *>(inc + 8 * j);
                w2[0] = v.x; w2[1] = v.y; w2[2] = v.z; w2[3] = v.w;
            }
#pragma unroll
            for (int q = 0; q < W; q++) {
                const uint32_t w = (w2[q >> 1] >> (16 * (q & 1))) & 0xffffu;
                Fn::gather_split(phis, (int)(w >> 1), (int)(w & 1), acc, phisB);
            }
        } else if constexpr (kSegScan) {
            acc[0] = tot[j];
        } else {
            const uint16_t *ioff = inc + 2 * d.s;
            const int q0 = ioff[j], q1 = j + 1 < L ? ioff[j + 1] : 2 * d.s;
            for (int q = q0; q < q1; q++) {
                const int w = inc[q];
                Fn::gather_split(phis, w >> 1, w & 1, acc, phisB);
            }
        }
        if (j < d.nO) {
            float U[ROW];
            Fn::rec_state_occ(recs, (j & ~7) | scol[j], U, ulast[r]);
            Fn::finish_occ(U, acc, dtv[r], out[r]);
        } else {
#pragma unroll
            for (int c = 0; c < ROW; c++) out[r][c] = acc[c];
            if (a.peer_acc) {  // fused push: a foreign vertex's partial goes to its owner's accumulator
                const int32_t h = reinterpret_cast<const int32_t *>(sblob)[j - d.nO];
                if (h < a.vlo[a.rank]) {
                    int p = 0;
                    while (p + 1 < a.rank && h >= a.vlo[p + 1]) p++;
                    float *dst = a.peer_acc[p] + (int64_t)ROW * h;
#pragma unroll
                    for (int c = 0; c < ROW; c++) ptx::red_add_f32(dst + c, acc[c]);
                    pushed = true;
                }
            }
            if (a.hub_acc) {   // hub split: this partition's partial of a hub, pre-summed above
                const int hx = reinterpret_cast<const int32_t *>(sblob)[d.nH + (j - d.nO)];
                if (hx >= 0) {
#pragma unroll
                    for (int c = 0; c < ROW; c++) ptx::red_add_f32(a.hub_acc + (int64_t)ROW * hx + c, acc[c]);
                }
            }
        }
    }
    // the pushed partials are performed in the peers' memory before this kernel ends (one fence
    // per pushing thread, after its last push; outside the loop, so the hub reductions stay REDs)
    if (pushed) __threadfence_system();
    __syncthreads();                               // records and Phi no longer read
    // pack: owned rows at the 16-byte phase of their destination, then the halo partials
    float *g_out = a.state_out + (int64_t)ROW * d.o0;
    float *g_halo = a.halo_buf + (int64_t)ROW * d.h0;
    unsigned char *outA_base = occ_smem + a.off_recs;
    unsigned char *outB_base = outA_base + ((4 * ROW * d.nO + 32 + 15) & ~15);
    float *outA = reinterpret_cast<float *>(outA_base + (reinterpret_cast<uintptr_t>(g_out) & 15));
    float *outB = reinterpret_cast<float *>(outB_base + (reinterpret_cast<uintptr_t>(g_halo) & 15));
#pragma unroll
    for (int r = 0; r < VPT; r++) {
        const int j = tid + r * BLOCK;
        if (j < d.nO) {
#pragma unroll
            for (int c = 0; c < ROW; c++) outA[ROW * j + c] = out[r][c];
        } else if (j < L) {
#pragma unroll
            for (int c = 0; c < ROW; c++) outB[ROW * (j - d.nO) + c] = out[r][c];
        }
    }
    __syncthreads();
    const uint32_t a_bytes = 4u * ROW * d.nO, b_bytes = 4u * ROW * d.nH;
    if (tid == 0) {
        ptx::fence_proxy_async_smem();
        const uintptr_t ga = reinterpret_cast<uintptr_t>(g_out), gb = reinterpret_cast<uintptr_t>(g_halo);
        const uintptr_t a_lo = up16(ga), a_hi = down16(ga + a_bytes), b_lo = up16(gb), b_hi = down16(gb + b_bytes);
        if (a_hi > a_lo)
            ptx::bulk_s2g(reinterpret_cast<void *>(a_lo), outA_base + (a_lo - down16(ga)), (uint32_t)(a_hi - a_lo));
        if (b_hi > b_lo)
            ptx::bulk_s2g(reinterpret_cast<void *>(b_lo), outB_base + (b_lo - down16(gb)), (uint32_t)(b_hi - b_lo));
        ptx::bulk_commit();
    }
    if (tid >= 32 && tid < 64) {                   // ragged words of both ranges, plain stores
        const int lane = tid - 32;
        const uintptr_t ga = reinterpret_cast<uintptr_t>(g_out), gb = reinterpret_cast<uintptr_t>(g_halo);
        auto ragged_store = [&](uintptr_t g, uint32_t bytes, const unsigned char *sbase) {
            const uintptr_t end = g + bytes, lo = up16(g), hi = down16(end);
            uintptr_t w;
            if (hi > lo) {
                const int head = (int)((lo - g) >> 2), tail = (int)((end - hi) >> 2);
                if (lane < head) w = g + 4 * lane;
                else if (lane < head + tail) w = hi + 4 * (lane - head);
                else return;
            } else {
                if (lane >= (int)(bytes >> 2)) return;
                w = g + 4 * lane;
            }
            *reinterpret_cast<float *>(w) = *reinterpret_cast<const float *>(sbase + (w - down16(g)));
        };
        ragged_store(ga, a_bytes, outA_base);
        ragged_store(gb, b_bytes, outB_base);
    }
    if (!a.early_pdl) ptx::pdl_launch_dependents();   // the finalise may start launching
    EPG_TP(0, 5);
    if (tid == 0) ptx::bulk_wait_read0();          // shared memory must outlive the stores' reads
    EPG_TP(0, 6);
}

// Boundary finalise (a6): U'_v = (U + dt F_owner)_v + dt * sum of v's halo partials, in
// the fixed order of hv_list; threads past S copy (cfd) or clear untouched rows. (A fused
// variant with per-vertex arrival counters in the edge kernel was measured slower on C2:
// each CTA then holds its SM slot through the extra global round trips.)
template <class Fn>
__global__ void k_finalise3(const int32_t *__restrict__ shared_ids, const int32_t *__restrict__ hv_off,
                            const int32_t *__restrict__ hv_list, const float *__restrict__ halo_buf,
                            const float *__restrict__ state_in, float *__restrict__ state_out,
                            const float *__restrict__ vconst, int32_t S, int64_t touched, int64_t n,
                            int32_t heavy) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    ptx::pdl_wait();                               // the edge kernel's outputs are visible
    ptx::pdl_launch_dependents();
    if (t < S) {
        if (hv_off[t + 1] - hv_off[t] > heavy) return;        // k_finalise_heavy's vertex
        const int64_t v = shared_ids[t];
        float acc[Fn::ROW];
#pragma unroll
        for (int c = 0; c < Fn::ROW; c++) acc[c] = 0.0f;
        for (int q = hv_off[t]; q < hv_off[t + 1]; q++) {
            const int64_t h = hv_list[q];
#pragma unroll
            for (int c = 0; c < Fn::ROW; c++) acc[c] += halo_buf[Fn::ROW * h + c];
        }
        const float dt = Fn::kUsesConst ? vconst[v] : 0.0f;
        Fn::finalise_add(state_out + Fn::ROW * v, acc, dt);
        EPG_TP(14, 2);
        return;
    }
    const int64_t v = touched + (t - S);
    if (v < n) Fn::untouched(state_in + Fn::ROW * v, state_out + Fn::ROW * v);
}

// Heavy shared vertices (more than `heavy` halo entries: the hubs of power-law graphs),
// one CTA each: thread t sums entries t, t + BLOCK, ... in order, then a fixed-shape tree
// reduction in shared memory -- deterministic, and a hub no longer serialises on one thread.
template <class Fn, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_finalise_heavy(const int32_t *__restrict__ heavy_list,
                                                          const int32_t *__restrict__ shared_ids,
                                                          const int32_t *__restrict__ hv_off,
                                                          const int32_t *__restrict__ hv_list,
                                                          const float *__restrict__ halo_buf,
                                                          float *__restrict__ state_out,
                                                          const float *__restrict__ vconst) {
    __shared__ float red[Fn::ROW][BLOCK];
    ptx::pdl_wait();
    const int s = heavy_list[blockIdx.x];
    const int q0 = hv_off[s], q1 = hv_off[s + 1];
    float acc[Fn::ROW];
#pragma unroll
    for (int c = 0; c < Fn::ROW; c++) acc[c] = 0.0f;
    for (int q = q0 + threadIdx.x; q < q1; q += BLOCK) {
        const int64_t h = hv_list[q];
#pragma unroll
        for (int c = 0; c < Fn::ROW; c++) acc[c] += halo_buf[Fn::ROW * h + c];
    }
#pragma unroll
    for (int c = 0; c < Fn::ROW; c++) red[c][threadIdx.x] = acc[c];
    __syncthreads();
    for (int w = BLOCK / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
#pragma unroll
            for (int c = 0; c < Fn::ROW; c++) red[c][threadIdx.x] += red[c][threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int64_t v = shared_ids[s];
        float tot[Fn::ROW];
#pragma unroll
        for (int c = 0; c < Fn::ROW; c++) tot[c] = red[c][0];
        Fn::finalise_add(state_out + Fn::ROW * v, tot, Fn::kUsesConst ? vconst[v] : 0.0f);
    }
}

// Medium shared vertices, one warp each (8 per CTA): lane l sums entries l, l + 32, ... in
// order, then a fixed xor-shuffle tree -- deterministic.
template <class Fn>
__global__ void __launch_bounds__(256) k_finalise_warp(const int32_t *__restrict__ list, int64_t count,
                                                       const int32_t *__restrict__ shared_ids,
                                                       const int32_t *__restrict__ hv_off,
                                                       const int32_t *__restrict__ hv_list,
                                                       const float *__restrict__ halo_buf,
                                                       float *__restrict__ state_out,
                                                       const float *__restrict__ vconst) {
    ptx::pdl_wait();
    const int64_t wi = blockIdx.x * 8ll + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (wi >= count) return;
    const int s = list[wi];
    const int q0 = hv_off[s], q1 = hv_off[s + 1];
    float acc[Fn::ROW];
#pragma unroll
    for (int c = 0; c < Fn::ROW; c++) acc[c] = 0.0f;
    for (int q = q0 + lane; q < q1; q += 32) {
        const int64_t h = hv_list[q];
#pragma unroll
        for (int c = 0; c < Fn::ROW; c++) acc[c] += halo_buf[Fn::ROW * h + c];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int c = 0; c < Fn::ROW; c++) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], off);
    }
    if (lane == 0) {
        const int64_t v = shared_ids[s];
        Fn::finalise_add(state_out + Fn::ROW * v, acc, Fn::kUsesConst ? vconst[v] : 0.0f);
    }
}

// Finalise of a vertex range (multi-GPU shards): for every shared vertex v
// in [v_lo, v_hi), add dt times (its halo partials at positions in [h_lo, h_hi), in
// ascending position, then acc[v] -- the partial sums pushed by other shards, already
// accumulated in ascending peer order) to the owner row; acc[v] is cleared. With the full
// ranges and acc = NULL this is exactly k_finalise3.
template <class Fn>
__global__ void k_finalise_range(const int32_t *__restrict__ shared_ids, const int32_t *__restrict__ hv_off,
                                 const int32_t *__restrict__ hv_list, const float *__restrict__ halo_buf,
                                 float *__restrict__ state_out, const float *__restrict__ vconst, int32_t s_lo,
                                 int32_t s_hi, int64_t h_lo, int64_t h_hi, float *__restrict__ acc) {
    const int64_t t = s_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    if (t >= s_hi) return;
    const int64_t v = shared_ids[t];
    float sum[Fn::ROW];
#pragma unroll
    for (int c = 0; c < Fn::ROW; c++) sum[c] = 0.0f;
    for (int q = hv_off[t]; q < hv_off[t + 1]; q++) {
        const int64_t h = hv_list[q];
        if (h < h_lo || h >= h_hi) continue;
#pragma unroll
        for (int c = 0; c < Fn::ROW; c++) sum[c] += halo_buf[Fn::ROW * h + c];
    }
    if (acc) {
#pragma unroll
        for (int c = 0; c < Fn::ROW; c++) {
            sum[c] += acc[Fn::ROW * v + c];
            acc[Fn::ROW * v + c] = 0.0f;
        }
    }
    const float dt = Fn::kUsesConst ? vconst[v] : 0.0f;
    Fn::finalise_add(state_out + Fn::ROW * v, sum, dt);
}

// untouched rows [touched, n): copied (cfd) or cleared
template <class Fn>
__global__ void k_untouched(const float *__restrict__ state_in, float *__restrict__ state_out, int64_t touched,
                            int64_t n) {
    const int64_t v = touched + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v < n) Fn::untouched(state_in + Fn::ROW * v, state_out + Fn::ROW * v);
}

// partial sums a shard pushes to an owner: out[i] = sum of the halo partials of vertex
// ids[i] at positions in [h_lo, h_hi), in ascending position
template <class Fn>
__global__ void k_shard_reduce(const int32_t *__restrict__ ids, int64_t count, const int32_t *__restrict__ sidx,
                               const int32_t *__restrict__ hv_off, const int32_t *__restrict__ hv_list,
                               const float *__restrict__ halo_buf, int64_t h_lo, int64_t h_hi,
                               float *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int32_t s = sidx[ids[i]];
    float sum[Fn::ROW];
#pragma unroll
    for (int c = 0; c < Fn::ROW; c++) sum[c] = 0.0f;
    if (s >= 0) {
        for (int q = hv_off[s]; q < hv_off[s + 1]; q++) {
            const int64_t h = hv_list[q];
            if (h < h_lo || h >= h_hi) continue;
#pragma unroll
            for (int c = 0; c < Fn::ROW; c++) sum[c] += halo_buf[Fn::ROW * h + c];
        }
    }
#pragma unroll
    for (int c = 0; c < Fn::ROW; c++) out[Fn::ROW * i + c] = sum[c];
}

// acc[ids[i]] += src[i] (rows of `w` floats; ids distinct within one call)
__global__ void k_accumulate_rows(const float *__restrict__ src, const int32_t *__restrict__ ids, int64_t count,
                                  int32_t w, float *__restrict__ acc) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= count * w) return;
    const int64_t i = t / w, c = t % w;
    acc[(int64_t)w * ids[i] + c] += src[t];
}

// Finalise from packed per-vertex records {v, count, h_0..h_5} (count <= 6 halo entries):
// one coalesced 32-byte record load, then the halo rows, dt and the owner row in
// parallel -- two dependent hops instead of three. Same summation order as k_finalise3.
template <class Fn>
__global__ void k_finalise_rec(const int4 *__restrict__ recs, const float *__restrict__ halo_buf,
                               const float *__restrict__ state_in, float *__restrict__ state_out,
                               const float *__restrict__ vconst, int32_t S, int64_t touched, int64_t n) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    EPG_TP(14, 0);
    // the records and dt are plan / constant data: loaded before the wait, i.e. while the
    // edge kernel still runs (it triggers this launch as soon as all of its CTAs started)
    int4 r0 = make_int4(0, -1, 0, 0), r1 = make_int4(0, 0, 0, 0);
    float dt = 0.0f;
    if (t < S) {
        r0 = recs[2 * t];
        r1 = recs[2 * t + 1];
        if (Fn::kUsesConst && r0.y >= 0) dt = vconst[r0.x];
    }
    ptx::pdl_wait();
    EPG_TP(14, 1);
    ptx::pdl_launch_dependents();
    if (t < S) {
        const int64_t v = r0.x;
        const int c = r0.y;
        if (c < 0) return;                         // a hub: k_finalise_hub's vertex
        const int h[6] = {r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
        float acc[Fn::ROW];
#pragma unroll
        for (int k = 0; k < Fn::ROW; k++) acc[k] = 0.0f;
#pragma unroll
        for (int i = 0; i < 6; i++) {
            if (i < c) {
#pragma unroll
                for (int k = 0; k < Fn::ROW; k++) acc[k] += halo_buf[Fn::ROW * (int64_t)h[i] + k];
            }
        }
        Fn::finalise_add(state_out + Fn::ROW * v, acc, dt);
        EPG_TP(14, 2);
        return;
    }
    const int64_t v = touched + (t - S);
    if (v < n) Fn::untouched(state_in + Fn::ROW * v, state_out + Fn::ROW * v);
}

// Finalise from 16-byte records {v, count, h0, x}: x = h1 when count <= 2, else the index of
// the vertex's entries h1..h5 in `over` (5 ints each). Same vertices, order and summation as
// k_finalise_rec, with half its record bytes (the C3 finalise is DRAM-bound and the 32-byte
// records were ~30 % of its traffic; most shared vertices of a mesh have one or two entries).
template <class Fn>
__global__ void k_finalise_rec16(const int4 *__restrict__ recs, const int32_t *__restrict__ over,
                                 const float *__restrict__ halo_buf, const float *__restrict__ state_in,
                                 float *__restrict__ state_out, const float *__restrict__ vconst, int32_t S,
                                 int64_t touched, int64_t n) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    EPG_TP(14, 0);
    // records, overflow entries and dt are plan / constant data: loaded before the wait
    int4 r = make_int4(0, -1, 0, 0);
    int h[6] = {0, 0, 0, 0, 0, 0};
    float dt = 0.0f;
    if (t < S) {
        r = recs[t];
        h[0] = r.z;
        if (r.y > 2) {
            const int32_t *o = over + 5 * (int64_t)r.w;
#pragma unroll
            for (int i = 1; i < 6; i++) h[i] = o[i - 1];
        } else {
            h[1] = r.w;
        }
        if (Fn::kUsesConst && r.y >= 0) dt = vconst[r.x];
    }
    ptx::pdl_wait();
    EPG_TP(14, 1);
    ptx::pdl_launch_dependents();
    if (t < S) {
        const int64_t v = r.x;
        const int c = r.y;
        if (c < 0) return;                         // a hub: k_finalise_hub's vertex
        float acc[Fn::ROW];
#pragma unroll
        for (int k = 0; k < Fn::ROW; k++) acc[k] = 0.0f;
#pragma unroll
        for (int i = 0; i < 6; i++) {
            if (i < c) {
#pragma unroll
                for (int k = 0; k < Fn::ROW; k++) acc[k] += halo_buf[Fn::ROW * (int64_t)h[i] + k];
            }
        }
        Fn::finalise_add(state_out + Fn::ROW * v, acc, dt);
        EPG_TP(14, 2);
        return;
    }
    const int64_t v = touched + (t - S);
    if (v < n) Fn::untouched(state_in + Fn::ROW * v, state_out + Fn::ROW * v);
}

// 16-byte records from the 32-byte ones: over_flag[t] = count > 2 (scanned into positions)
__global__ void k_rec16_flags(const int4 *__restrict__ recs, int32_t S, int32_t *flag) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < S) flag[t] = recs[2 * t].y > 2 ? 1 : 0;
}
__global__ void k_rec16_build(const int4 *__restrict__ recs, int32_t S, const int32_t *__restrict__ pos,
                              int4 *rec16, int32_t *over) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= S) return;
    const int4 r0 = recs[2 * t], r1 = recs[2 * t + 1];
    if (r0.y > 2) {
        const int32_t p = pos[t];
        rec16[t] = make_int4(r0.x, r0.y, r0.z, p);
        int32_t *o = over + 5 * (int64_t)p;
        o[0] = r0.w; o[1] = r1.x; o[2] = r1.y; o[3] = r1.z; o[4] = r1.w;
    } else {
        rec16[t] = make_int4(r0.x, r0.y, r0.z, r0.w);
    }
}

// records for k_finalise_rec; *hmax receives the largest halo count of a non-hub vertex
// (hubs: count >= hub_min > 0, recorded with count -1)
__global__ void k_finalise_records(const int32_t *__restrict__ shared_ids, const int32_t *__restrict__ hv_off,
                                   const int32_t *__restrict__ hv_list, int32_t S, int32_t hub_min, int4 *recs,
                                   int32_t *hmax) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= S) return;
    const int q0 = hv_off[t];
    int c = hv_off[t + 1] - q0;
    if (hub_min > 0 && c >= hub_min) {
        recs[2 * t] = make_int4(shared_ids[t], -1, 0, 0);
        recs[2 * t + 1] = make_int4(0, 0, 0, 0);
        atomicAdd(hmax + 1, 1);
        return;
    }
    int h[6];
    for (int i = 0; i < 6; i++) h[i] = i < c ? hv_list[q0 + i] : 0;
    recs[2 * t] = make_int4(shared_ids[t], c, h[0], h[1]);
    recs[2 * t + 1] = make_int4(h[2], h[3], h[4], h[5]);
    atomicMax(hmax, c);
}

// records for the finalise of one shard (multi-GPU): the shard's shared vertices with only
// their halo entries at positions in [h_lo, h_hi) (the shard's own partitions), in hv_list
// order; *hmax receives the largest local count
__global__ void k_shard_records(const int32_t *__restrict__ shared_ids, const int32_t *__restrict__ hv_off,
                                const int32_t *__restrict__ hv_list, int32_t count, int64_t h_lo, int64_t h_hi,
                                int4 *recs, int32_t *hmax) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= count) return;
    int h[6] = {0, 0, 0, 0, 0, 0};
    int c = 0;
    for (int q = hv_off[t]; q < hv_off[t + 1]; q++) {
        const int64_t x = hv_list[q];
        if (x < h_lo || x >= h_hi) continue;
        if (c < 6) h[c] = (int)x;
        c++;
    }
    recs[2 * t] = make_int4(shared_ids[t], c < 6 ? c : 6, h[0], h[1]);
    recs[2 * t + 1] = make_int4(h[2], h[3], h[4], h[5]);
    atomicMax(hmax, c);
}

// U'_v += dt_v * acc_v for the vertices other ranks pushed partial sums for; acc cleared
template <class Fn>
__global__ void k_acc_add(const int32_t *__restrict__ ids, int64_t count, float *__restrict__ acc,
                          float *__restrict__ state_out, const float *__restrict__ vconst) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    const int64_t v = ids[i];
    float sum[Fn::ROW];
#pragma unroll
    for (int c = 0; c < Fn::ROW; c++) {
        sum[c] = acc[Fn::ROW * v + c];
        acc[Fn::ROW * v + c] = 0.0f;
    }
    Fn::finalise_add(state_out + Fn::ROW * v, sum, Fn::kUsesConst ? vconst[v] : 0.0f);
}

// Hub finalise (hub split): U'_v += dt * hub_acc[i] for hub i of
// shared vertex hub_sid[i]; hub_acc is cleared for the next step. The hub's partials were
// added by the edge kernel with one red.global.add per (execution partition, hub) after
// the partition summed its edges in shared memory, so the sum order is not fixed.
template <class Fn>
__global__ void k_finalise_hub(const int32_t *__restrict__ hub_sid, int64_t nhub, const int32_t *__restrict__ shared_ids,
                               float *__restrict__ hub_acc, float *__restrict__ state_out,
                               const float *__restrict__ vconst) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    if (i >= nhub) return;
    const int64_t v = shared_ids[hub_sid[i]];
    float sum[Fn::ROW];
#pragma unroll
    for (int c = 0; c < Fn::ROW; c++) {
        sum[c] = hub_acc[Fn::ROW * i + c];
        hub_acc[Fn::ROW * i + c] = 0.0f;
    }
    Fn::finalise_add(state_out + Fn::ROW * v, sum, Fn::kUsesConst ? vconst[v] : 0.0f);
}

// hub_of_h[h] = hub index of halo entry h's vertex (entries of non-hubs keep -1)
__global__ void k_hub_mark(const int32_t *__restrict__ hub_of_s, int32_t S, const int32_t *__restrict__ hv_off,
                           const int32_t *__restrict__ hv_list, int32_t *__restrict__ hub_of_h) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= S) return;
    const int32_t hx = hub_of_s[t];
    if (hx < 0) return;
    for (int q = hv_off[t]; q < hv_off[t + 1]; q++) hub_of_h[hv_list[q]] = hx;
}

// blob3 of partition p
__global__ void k_build_blob3(const int32_t *__restrict__ peb, const int32_t *__restrict__ pvb,
                              const int32_t *__restrict__ hb, const int32_t *__restrict__ halo_ids,
                              const uint16_t *__restrict__ inc, const uint16_t *__restrict__ inc_off,
                              const int32_t *__restrict__ blob16, int W, const int32_t *__restrict__ hub_of_h,
                              int sentinel, unsigned char *blob, PartDesc *desc) {
    const int p = blockIdx.x;
    const int o0 = pvb[p], nO = pvb[p + 1] - o0, h0 = hb[p], nH = hb[p + 1] - h0, e0 = peb[p], s = peb[p + 1] - e0;
    const int L = nO + nH;
    unsigned char *b = blob + 16 * (int64_t)blob16[p];
    int32_t *hid = reinterpret_cast<int32_t *>(b);
    const int hw = hub_of_h ? 2 : 1;
    uint16_t *ic = reinterpret_cast<uint16_t *>(b + blob3_inc_offset(nH, hw));
    for (int j = threadIdx.x; j < nH; j += blockDim.x) hid[j] = halo_ids[h0 + j];
    if (hub_of_h)
        for (int j = threadIdx.x; j < nH; j += blockDim.x) hid[nH + j] = hub_of_h[h0 + j];
    const int64_t lbase = (int64_t)o0 + h0;
    if (W > 0) {
        for (int j = threadIdx.x; j < L; j += blockDim.x) {
            const int q0 = inc_off[lbase + j], q1 = j + 1 < L ? inc_off[lbase + j + 1] : 2 * s;
            for (int r = 0; r < W; r++)
                ic[W * j + r] = q0 + r < q1 ? inc[2 * (int64_t)e0 + q0 + r] : (uint16_t)(sentinel << 1);
        }
    } else {
        uint16_t *io = ic + 2 * s;
        for (int q = threadIdx.x; q < 2 * s; q += blockDim.x) ic[q] = inc[2 * (int64_t)e0 + q];
        for (int j = threadIdx.x; j < L; j += blockDim.x) io[j] = inc_off[lbase + j];
    }
    if (threadIdx.x == 0)
        desc[p] = PartDesc{o0, nO, e0, s, h0, nH, blob16[p], blob3_bytes_for(nH, s, L, W, hw), 0, 0, 0, 0};
}

// Apply the placement (place_kernels.cuh) to partition p of the plan: the occupancy kernel's slots
// (record positions of both endpoints, bits 29-31 the in-group position of the edge's Phi
// record), the blob's incidence entries (Phi positions) and its placement bytes.
__global__ void k_apply_place(const PartDesc *__restrict__ desc, const uint32_t *__restrict__ slots,
                              const uint8_t *__restrict__ vcol, const uint8_t *__restrict__ ecol, int W, int hw,
                              int sentinel, unsigned char *blob, uint32_t *slots_occ) {
    const PartDesc d = desc[blockIdx.x];
    const int L = d.nO + d.nH;
    const int64_t lb = (int64_t)d.o0 + d.h0;
    const uint8_t *vc = vcol + lb, *ec = ecol + d.e0;
    for (int i = threadIdx.x; i < d.s; i += blockDim.x) {
        const uint32_t sl = slots[d.e0 + i];
        const int a = (int)(sl & 0xffffu), b = (int)(sl >> 16);
        const uint32_t pa = (uint32_t)((a & ~7) | vc[a]), pb = (uint32_t)((b & ~7) | vc[b]);
        slots_occ[d.e0 + i] = pa | ((pb | ((uint32_t)ec[i] << 13)) << 16);
    }
    unsigned char *b0 = blob + 16 * (int64_t)d.blob16;
    uint16_t *ic = reinterpret_cast<uint16_t *>(b0 + blob3_inc_offset(d.nH, hw));
    const int ninc = W > 0 ? W * L : 2 * d.s;
    for (int q = threadIdx.x; q < ninc; q += blockDim.x) {
        const int e = ic[q], i = e >> 1;
        if (i != sentinel) ic[q] = (uint16_t)((((i & ~7) | ec[i]) << 1) | (e & 1));
    }
    uint8_t *cb = b0 + blob3_col_offset(d.nH, d.s, L, W, hw);
    for (int j = threadIdx.x; j < L; j += blockDim.x) cb[j] = vc[j];
}

__global__ void k_blob3_sizes(const int32_t *__restrict__ peb, const int32_t *__restrict__ pvb,
                              const int32_t *__restrict__ hb, int64_t k, int W, int hw, int32_t *units16) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p > k) return;
    if (p == k) { units16[p] = 0; return; }
    const int nO = pvb[p + 1] - pvb[p], nH = hb[p + 1] - hb[p], s = peb[p + 1] - peb[p];
    units16[p] = blob3_bytes_for(nH, s, nO + nH, W, hw) / 16;
}

// execution partitions: partition p of the EP map is cut into c_p contiguous edge ranges
// (by new edge index); exec id = base[p] + piece. Written per original task id.
__global__ void k_exec_map(const int32_t *__restrict__ peb, const int32_t *__restrict__ edge_perm,
                           const int32_t *__restrict__ cuts, const int32_t *__restrict__ base, int32_t *part_exec) {
    const int p = blockIdx.x;
    const int e0 = peb[p], s = peb[p + 1] - e0, c = cuts[p];
    for (int i = threadIdx.x; i < s; i += blockDim.x)
        part_exec[edge_perm[e0 + i]] = base[p] + (int)((int64_t)i * c / s);
}

}  // namespace epg
