// place_kernels.cuh -- bank-conflict-aware placement of a partition's staged records (plan
// build). Part of the execution plan only: it moves no task and no vertex between partitions
// and changes no result bit (every value is computed and summed exactly as before, only its
// shared-memory address changes).
//
// The staged edge kernel reads, for 8 consecutive edges of a warp quarter, the 32-byte
// derived records of their endpoints with 128-bit shared loads, and, for 8 consecutive local
// vertices, the Phi records of their incident edges. Two lanes of a quarter whose addresses
// fall in the same 16-byte bank group serialise (one more wavefront). The layout fixes which
// records a quarter reads, but not where they live: record j may sit at any position of its
// aligned group of 8 (8 floor(j / 8) .. + 7), the Phi record of edge i likewise, and the
// quarter's bank groups are then these in-group positions (rec4 and the float4 index mod 8
// are bijections of them). A greedy per group of 8 -- most constrained member first, each
// taking the free in-group position that collides least with its already placed octet
// partners; two sweeps -- chooses them (C1 layout: edge-phase record wavefronts 1.90x ->
// 1.37x the conflict-free count, reduce-phase Phi wavefronts 2.10x -> 1.74x). The greedy is
// sequential over a partition's groups, so one warp runs it per partition (the lanes count
// the penalties of a group's members, lane 0 assigns); partitions run in parallel.
#pragma once

#include <stdint.h>

#include "pipelined_kernel.cuh"   // PartDesc

namespace epg {

constexpr uint8_t kPlaceNone = 0xff;

// greedy colouring of members [0, count) in aligned groups of 8 (a permutation inside each
// group), by one warp: partner(m, t) is the t-th octet partner slot of member m (T slots per
// member; < 0: empty). The lanes count, per member and colour, the partners already coloured
// (shared-memory atomics: counts, so the order does not matter); lane 0 then assigns the group.
template <int T, class Partner>
__device__ void place_colour(int count, uint8_t *col, int *pen, Partner &&partner) {
    const int lane = threadIdx.x & 31;
    for (int j = lane; j < count; j += 32) col[j] = kPlaceNone;
    __syncwarp();
    for (int sweep = 0; sweep < 2; sweep++) {
        for (int g0 = 0; g0 < count; g0 += 8) {
            const int nm = min(8, count - g0);
            if (lane < nm) col[g0 + lane] = kPlaceNone;
            for (int q = lane; q < 64; q += 32) pen[q] = 0;
            __syncwarp();
            for (int idx = lane; idx < nm * T; idx += 32) {
                const int x = idx / T, mem = g0 + x;
                const int o = partner(mem, idx - x * T);
                if (o >= 0 && o != mem) {
                    const uint8_t c = col[o];
                    if (c != kPlaceNone) atomicAdd(&pen[8 * x + c], 1);
                }
            }
            __syncwarp();
            if (lane == 0) {
                int spread[8], order[8];
                for (int x = 0; x < nm; x++) {
                    int lo = pen[8 * x], hi = pen[8 * x];
                    for (int c = 1; c < nm; c++) {
                        lo = min(lo, pen[8 * x + c]);
                        hi = max(hi, pen[8 * x + c]);
                    }
                    spread[x] = hi - lo;
                    int r = x;                          // stable insertion, spread descending
                    while (r > 0 && spread[order[r - 1]] < spread[x]) {
                        order[r] = order[r - 1];
                        r--;
                    }
                    order[r] = x;
                }
                unsigned used = 0;
                for (int r = 0; r < nm; r++) {
                    const int x = order[r];
                    int best = -1;
                    for (int c = 0; c < nm; c++)
                        if (!(used & (1u << c)) && (best < 0 || pen[8 * x + c] < pen[8 * x + best])) best = c;
                    used |= 1u << best;
                    col[g0 + x] = (uint8_t)best;
                }
            }
            __syncwarp();
        }
    }
}

// One warp per execution partition (W: the plan's padded incidence width, 4 or 8): vcol[lb +
// j] = in-group position of record j (lb = o0 + h0), ecol[e0 + i] = in-group position of the
// Phi record of local edge i. Shared memory: see place_smem_bytes.
__host__ __device__ inline int place_smem_bytes(int Scap, int Lcap, int W) {
    return 256 + 4 * Scap + 2 * W * Lcap + 2 * Lcap + 3 * Scap + 16;
}
template <int W>
__global__ void __launch_bounds__(32) k_place(const PartDesc *__restrict__ desc, const uint32_t *__restrict__ slots,
                                              int Scap, int Lcap, uint8_t *vcol, uint8_t *ecol) {
    extern __shared__ __align__(16) unsigned char place_smem[];
    int *PEN = reinterpret_cast<int *>(place_smem);                        // [8][8]
    uint16_t *A = reinterpret_cast<uint16_t *>(place_smem + 256), *B = A + Scap;
    uint16_t *INC = B + Scap;                                              // [L][W] entries 2 i + side
    uint8_t *DEG = reinterpret_cast<uint8_t *>(INC + W * Lcap), *COL = DEG + Lcap;
    uint8_t *ECOL = COL + Lcap, *QPOS = ECOL + Scap;                        // QPOS [2 s]
    const PartDesc d = desc[blockIdx.x];
    const int s = d.s, L = d.nO + d.nH, lane = threadIdx.x;
    for (int i = lane; i < s; i += 32) {
        const uint32_t sl = slots[d.e0 + i];
        A[i] = (uint16_t)(sl & 0xffffu);
        B[i] = (uint16_t)(sl >> 16);
    }
    for (int j = lane; j < L; j += 32) DEG[j] = 0;
    __syncwarp();
    if (lane == 0) {   // incidence in the remap's order (ascending 2 i + side)
        for (int i = 0; i < s; i++) {
            const int a = A[i], b = B[i];
            QPOS[2 * i] = DEG[a];
            INC[W * a + DEG[a]++] = (uint16_t)(2 * i);
            QPOS[2 * i + 1] = DEG[b];
            INC[W * b + DEG[b]++] = (uint16_t)(2 * i + 1);
        }
    }
    __syncwarp();
    // 1. records: the endpoints of an octet's 8 edges, per side, should differ mod 8; slot
    // t = 8 q + u of vertex j is lane u of the octet of j's q-th incident edge, on its side
    place_colour<8 * W>(L, COL, PEN, [&](int j, int t) -> int {
        const int q = t >> 3, u = t & 7;
        if (q >= DEG[j]) return -1;
        const int e = INC[W * j + q], i2 = ((e >> 1) & ~7) + u;
        if (i2 >= s) return -1;
        return (e & 1) ? B[i2] : A[i2];
    });
    // 2. Phi records: entry q of 8 consecutive vertices should name edges that differ mod 8;
    // slot t = 8 side + u of edge i is vertex u of the group of its endpoint on that side
    place_colour<16>(s, ECOL, PEN, [&](int i, int t) -> int {
        const int side = t >> 3, u = t & 7;
        const int v = side ? B[i] : A[i], q = QPOS[2 * i + side], j = (v & ~7) + u;
        if (j >= L || q >= DEG[j]) return -1;
        return INC[W * j + q] >> 1;
    });
    const int64_t lb = (int64_t)d.o0 + d.h0;
    for (int j = lane; j < L; j += 32) vcol[lb + j] = COL[j];
    for (int i = lane; i < s; i += 32) ecol[d.e0 + i] = ECOL[i];
}

// identity placement (variable-length incidence, or EPG_PLACE=0)
__global__ void k_place_identity(const PartDesc *__restrict__ desc, uint8_t *vcol, uint8_t *ecol) {
    const PartDesc d = desc[blockIdx.x];
    const int L = d.nO + d.nH;
    const int64_t lb = (int64_t)d.o0 + d.h0;
    for (int j = threadIdx.x; j < L; j += blockDim.x) vcol[lb + j] = (uint8_t)(j & 7);
    for (int i = threadIdx.x; i < d.s; i += blockDim.x) ecol[d.e0 + i] = (uint8_t)(i & 7);
}

}  // namespace epg
