// run_kernels.cuh -- the partition-scheduled edge kernel (step a5), boundary finalise
// (a6), row permutation (a7) and the default-schedule comparator.
//
// Staged kernel, one CTA per partition p (the paper's "thread block" = cluster):
//  (i)   stage V_p into shared memory: owned rows O_p = [beginA[p], beginA[p+1]) are a
//        contiguous range of the cpack layout (coalesced), halo rows H_p gathered by id
//        ("each thread block loads its shared parts ... coalesced");
//        per-vertex derived quantities are computed once while staging;
//  (ii)  one thread per edge computes the interaction from shared memory ("replace the
//        reference of the original input array with that of the local array")
//        and stores it in shared memory;
//  (iii) one thread per local vertex sums its incident edge results in the fixed order of
//        the incidence list (no atomics, deterministic);
//  (iv)  vertices touched only by p (p_v = 1) are final: U' = U + dt F is written
//        straight to state_out; shared vertices (p_v > 1) write their partial sum to the
//        plan's owner/halo buffers, which the finalise kernel adds in a fixed order.
#pragma once

#include <stdint.h>

#include "functors.cuh"

namespace epg {

struct RunArgs {
    const int32_t *peb, *pvb, *hb;   // [k+1]
    const int32_t *halo_ids;         // [C]
    const uint32_t *slots;           // [m] packed (slot_a | slot_b << 16)
    const uint16_t *inc;             // [2m]
    const uint16_t *inc_off;         // [touched + C]
    const int32_t *sidx;             // [n] shared index or -1
    const float *state_in;
    float *state_out;
    const float *payload;
    const float *vconst;
    float *owner_buf;                // [S][ROW]
    float *halo_buf;                 // [C][ROW]
    int Lcap, Scap;
};

template <class Fn, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_edge_staged(RunArgs a) {
    extern __shared__ __align__(16) float sm[];
    float *V = sm;                              // Fn::NV x Lcap
    float *Phi = sm + Fn::NV * a.Lcap;          // Fn::NPHI x Scap
    const int p = blockIdx.x;
    const int o0 = a.pvb[p], nO = a.pvb[p + 1] - o0;
    const int h0 = a.hb[p], nH = a.hb[p + 1] - h0;
    const int e0 = a.peb[p], s = a.peb[p + 1] - e0;
    const int L = nO + nH;
    // (i) stage
    for (int j = threadIdx.x; j < L; j += BLOCK) {
        const int64_t v = j < nO ? (int64_t)(o0 + j) : (int64_t)__ldg(a.halo_ids + h0 + (j - nO));
        Fn::stage(a.state_in + Fn::ROW * v, V, j, a.Lcap);
    }
    __syncthreads();
    // (ii) edges
    for (int i = threadIdx.x; i < s; i += BLOCK) {
        const uint32_t sl = __ldg(a.slots + e0 + i);
        Fn::edge(V, a.Lcap, (int)(sl & 0xffffu), (int)(sl >> 16), a.payload, (int64_t)e0 + i, Phi, a.Scap, i);
    }
    __syncthreads();
    // (iii) per-vertex reduction + (iv) write-back
    const int64_t lbase = (int64_t)o0 + h0;
    for (int j = threadIdx.x; j < L; j += BLOCK) {
        const int q0 = __ldg(a.inc_off + lbase + j);
        const int q1 = j + 1 < L ? __ldg(a.inc_off + lbase + j + 1) : 2 * s;
        float acc[Fn::ROW];
#pragma unroll
        for (int c = 0; c < Fn::ROW; c++) acc[c] = 0.0f;
        for (int q = q0; q < q1; q++) {
            const int w = __ldg(a.inc + 2 * (int64_t)e0 + q);
            Fn::gather(Phi, a.Scap, w >> 1, w & 1, acc);
        }
        if (j < nO) {
            const int64_t v = o0 + j;
            const int32_t si = __ldg(a.sidx + v);
            if (si < 0) {
                const float c = Fn::kUsesConst ? __ldg(a.vconst + v) : 0.0f;
                Fn::finish_smem(V, a.Lcap, j, acc, c, a.state_out + Fn::ROW * v);
            } else {
#pragma unroll
                for (int c = 0; c < Fn::ROW; c++) a.owner_buf[Fn::ROW * (int64_t)si + c] = acc[c];
            }
        } else {
            const int64_t h = (int64_t)h0 + (j - nO);
#pragma unroll
            for (int c = 0; c < Fn::ROW; c++) a.halo_buf[Fn::ROW * h + c] = acc[c];
        }
    }
}

// Boundary finalise (a6): shared vertex s = owner partial + its halo partials in halo order;
// threads beyond S copy/clear the untouched tail [touched, n).
template <class Fn>
__global__ void k_finalise(const int32_t *__restrict__ shared_ids, const int32_t *__restrict__ hv_off,
                           const int32_t *__restrict__ hv_list, const float *__restrict__ owner_buf,
                           const float *__restrict__ halo_buf, const float *__restrict__ state_in,
                           float *__restrict__ state_out, const float *__restrict__ vconst, int32_t S,
                           int64_t touched, int64_t n) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < S) {
        const int64_t v = shared_ids[t];
        float acc[Fn::ROW];
#pragma unroll
        for (int c = 0; c < Fn::ROW; c++) acc[c] = owner_buf[Fn::ROW * t + c];
        for (int q = hv_off[t]; q < hv_off[t + 1]; q++) {
            const int64_t h = hv_list[q];
#pragma unroll
            for (int c = 0; c < Fn::ROW; c++) acc[c] += halo_buf[Fn::ROW * h + c];
        }
        const float c = Fn::kUsesConst ? vconst[v] : 0.0f;
        Fn::finish_row(state_in + Fn::ROW * v, acc, c, state_out + Fn::ROW * v);
        return;
    }
    const int64_t v = touched + (t - S);
    if (v < n) Fn::untouched(state_in + Fn::ROW * v, state_out + Fn::ROW * v);
}

// ---- default-schedule comparator: thread per task, global gathers + atomics ------
template <class Fn>
__global__ void k_naive_edges(const int32_t *__restrict__ edges, int64_t m, const float *__restrict__ state,
                              const float *__restrict__ payload, float *__restrict__ F) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= m) return;
    Fn::naive_edge(state, edges[2 * e], edges[2 * e + 1], payload, e, F);
}

// per-vertex update; re-zeroes F for the next step. Untouched vertices have F = 0, so the
// cfd update leaves them unchanged and gather-scatter/SpMV write 0, as the oracle does.
template <class Fn>
__global__ void k_naive_update(int64_t n, const float *__restrict__ state_in, float *__restrict__ state_out,
                               const float *__restrict__ vconst, float *__restrict__ F) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    float acc[Fn::ROW];
#pragma unroll
    for (int c = 0; c < Fn::ROW; c++) { acc[c] = F[Fn::ROW * v + c]; F[Fn::ROW * v + c] = 0.0f; }
    const float c = Fn::kUsesConst ? vconst[v] : 0.0f;
    Fn::finish_row(state_in + Fn::ROW * v, acc, c, state_out + Fn::ROW * v);
}

// ---- row permutation (a7) ------------------------------------------------------------
__global__ void k_permute_rows(const uint32_t *__restrict__ src, uint32_t *__restrict__ dst, int64_t rows,
                               int32_t words, const int32_t *__restrict__ perm, int32_t scatter) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= rows * words) return;
    const int64_t i = t / words, w = t % words;
    const int64_t pi = perm[i];
    if (scatter) dst[pi * words + w] = src[i * words + w];
    else dst[i * words + w] = src[pi * words + w];
}

}  // namespace epg
