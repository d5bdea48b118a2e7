// layout_kernels.cuh -- GPU cost function (step a3) and remap (step a4).
//
// Cost (Eq. (1); fig:mot P:68-74): one CTA per partition sorts the partition's
// <= 2P endpoint ids in shared memory (CUB block radix sort), flags heads
// (BlockDiscontinuity) and counts them: |V_p|. L = sum_p |V_p|, touched from a vertex
// flag array, C = L - touched.
//
// Remap (O6; task reorganisation + cpack): stable radix sort of
// tasks by partition, first-touch keys by atomicMin, vertex ranks by a scan over the 2m
// endpoint slots, beginA by reading the scan at 2*part_edge_begin[p], then one CTA per
// partition sorts (new id, endpoint index) pairs once and derives from that single sort:
// the halo list H_p (the prefix of V_p below beginA[p]), every endpoint's local slot,
// and the per-partition incidence lists (endpoints in slot order) the staged kernel uses
// to reduce shared-memory results without atomics.
#pragma once

#include <cub/cub.cuh>
#include <stdint.h>

namespace epg {

constexpr int kSentinel = 0x7fffffff;

__global__ void k_iota(int32_t *a, int64_t m) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) a[i] = (int32_t)i;
}

// first offending edge (endpoint outside [0,n)) and first edge with a bad partition id
__global__ void k_validate(const int32_t *__restrict__ edges, const int32_t *__restrict__ part, int64_t m, int32_t n,
                           int64_t k, unsigned long long *bad_edge, unsigned long long *bad_part) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= m) return;
    int32_t a = edges[2 * e], b = edges[2 * e + 1];
    if (a < 0 || a >= n || b < 0 || b >= n) atomicMin(bad_edge, (unsigned long long)e);
    if (part) {
        int32_t p = part[e];
        if (p < 0 || p >= k) atomicMin(bad_part, (unsigned long long)e);
    }
}

// part_edge_begin[p] = lower_bound(sorted_part, p), p in [0, k]
__global__ void k_part_begin(const int32_t *__restrict__ sorted_part, int64_t m, int64_t k, int32_t *peb) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p > k) return;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (sorted_part[mid] < p) lo = mid + 1; else hi = mid;
    }
    peb[p] = (int32_t)lo;
}

// default schedule (O3): task e -> chunk i of sizes s_i = floor(m/k) + [i < m mod k]
__global__ void k_default_partition(int64_t m, int64_t k, int32_t *part) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= m) return;
    const int64_t q = m / k, r = m % k;
    // the first r chunks have q+1 tasks
    int64_t i = (e < r * (q + 1)) ? e / (q + 1) : r + (e - r * (q + 1)) / q;
    part[e] = (int32_t)i;
}

__global__ void k_mark_touched(const int32_t *__restrict__ edges, int64_t m, int32_t *flag) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < 2 * m) flag[edges[j]] = 1;
}

// sum of an int32 array into an int64 (block reduce + one atomic per block)
__global__ void k_sum(const int32_t *__restrict__ a, int64_t len, unsigned long long *out) {
    using Red = cub::BlockReduce<long long, 256>;
    __shared__ typename Red::TempStorage ts;
    long long s = 0;
    for (int64_t i = blockIdx.x * 256ll + threadIdx.x; i < len; i += (int64_t)gridDim.x * 256) s += a[i];
    long long t = Red(ts).Sum(s);
    if (threadIdx.x == 0) atomicAdd(out, (unsigned long long)t);
}

// Per-partition distinct endpoint count, |V_p|, by block radix sort + head flags.
template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK) k_distinct(const int32_t *__restrict__ edges,
                                                    const int32_t *__restrict__ edge_perm,
                                                    const int32_t *__restrict__ peb, int32_t *per_part, int end_bit) {
    using Sort = cub::BlockRadixSort<int, BLOCK, ITEMS>;
    using Disc = cub::BlockDiscontinuity<int, BLOCK>;
    using Red = cub::BlockReduce<int, BLOCK>;
    union TS {
        typename Sort::TempStorage sort;
        typename Disc::TempStorage disc;
        typename Red::TempStorage red;
    };
    extern __shared__ __align__(16) unsigned char dsm[];
    TS &ts = *reinterpret_cast<TS *>(dsm);
    const int p = blockIdx.x;
    const int e0 = peb[p], nvalid = 2 * (peb[p + 1] - e0);
    int key[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; it++) {
        int j = threadIdx.x * ITEMS + it;  // blocked: endpoint j = 2*local_edge + side
        key[it] = j < nvalid ? edges[2 * (int64_t)edge_perm[e0 + (j >> 1)] + (j & 1)] : kSentinel;
    }
    Sort(ts.sort).Sort(key, 0, end_bit);
    __syncthreads();
    int head[ITEMS];
    Disc(ts.disc).FlagHeads(head, key, cub::Inequality());
    __syncthreads();
    int cnt = 0;
#pragma unroll
    for (int it = 0; it < ITEMS; it++) cnt += (head[it] && threadIdx.x * ITEMS + it < nvalid) ? 1 : 0;
    int total = Red(ts.red).Sum(cnt);
    if (threadIdx.x == 0) per_part[p] = total;
}

// Fallback for partitions larger than the block-sort capacity: (part, vertex) keys were
// sorted globally; count heads per partition.
__global__ void k_distinct_global(const unsigned long long *__restrict__ keys, int64_t len, int32_t *per_part) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= len) return;
    if (i == 0 || keys[i] != keys[i - 1]) atomicAdd(per_part + (keys[i] >> 32), 1);
}

__global__ void k_pv_keys(const int32_t *__restrict__ edges, const int32_t *__restrict__ part, int64_t m,
                          unsigned long long *keys) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < 2 * m) keys[j] = ((unsigned long long)(uint32_t)part[j >> 1] << 32) | (uint32_t)edges[j];
}

// key(v) = min over endpoint slots of (2 e' + s), e' = new edge index (O6 step 2)
__global__ void k_first_touch(const int32_t *__restrict__ edges, const int32_t *__restrict__ edge_perm, int64_t m,
                              int32_t *key) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    int64_t e = edge_perm[i];
    atomicMin(key + edges[2 * e], (int32_t)(2 * i));
    atomicMin(key + edges[2 * e + 1], (int32_t)(2 * i + 1));
}

// flag[j] = 1 iff endpoint slot j = 2e'+s is its vertex's first touch; flag[2m] = 0
__global__ void k_first_touch_flags(const int32_t *__restrict__ edges, const int32_t *__restrict__ edge_perm,
                                    int64_t m, const int32_t *__restrict__ key, int32_t *flag) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j > 2 * m) return;
    if (j == 2 * m) { flag[j] = 0; return; }
    int32_t v = edges[2 * (int64_t)edge_perm[j >> 1] + (j & 1)];
    flag[j] = key[v] == (int32_t)j ? 1 : 0;
}

// touched v: new id = rank of its first-touch slot; untouched flag for the second scan
__global__ void k_vperm_touched(const int32_t *__restrict__ key, const int32_t *__restrict__ rank, int32_t n,
                                int32_t *vertex_perm, int32_t *untouched) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v > n) return;
    if (v == n) { untouched[v] = 0; return; }
    int32_t kv = key[v];
    if (kv != kSentinel) { vertex_perm[v] = rank[kv]; untouched[v] = 0; }
    else untouched[v] = 1;
}

__global__ void k_vperm_untouched(const int32_t *__restrict__ key, const int32_t *__restrict__ urank, int32_t n,
                                  int32_t touched, int32_t *vertex_perm) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v < n && key[v] == kSentinel) vertex_perm[v] = touched + urank[v];
}

// beginA: pvb[p] = #{v : key(v) < 2 peb[p]} = rank[2 peb[p]]
__global__ void k_pvb(const int32_t *__restrict__ rank, const int32_t *__restrict__ peb, int64_t k, int32_t *pvb) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p <= k) pvb[p] = rank[2 * (int64_t)peb[p]];
}

// |H_p| = |V_p| - |O_p|
__global__ void k_halo_counts(const int32_t *__restrict__ distinct, const int32_t *__restrict__ pvb, int64_t k,
                              int32_t *nh) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p > k) return;
    nh[p] = p < k ? distinct[p] - (pvb[p + 1] - pvb[p]) : 0;
}

// One CTA per partition: sort (new id, endpoint index) and derive halo ids, slots and
// the incidence lists in slot order.
//   sorted by new id = [halo incidences (ids < pvb[p])..., owned incidences...]
//   slot order       = [owned slots 0..|O_p|-1, halo slots |O_p|..]  -> a rotation.
template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK) k_remap_part(const int32_t *__restrict__ edges,
                                                      const int32_t *__restrict__ edge_perm,
                                                      const int32_t *__restrict__ vertex_perm,
                                                      const int32_t *__restrict__ peb, const int32_t *__restrict__ pvb,
                                                      const int32_t *__restrict__ hb, int32_t *halo_ids,
                                                      uint16_t *slots, uint16_t *inc, uint16_t *inc_off, int end_bit) {
    using Sort = cub::BlockRadixSort<int, BLOCK, ITEMS, int>;
    using Disc = cub::BlockDiscontinuity<int, BLOCK>;
    using Scan = cub::BlockScan<int, BLOCK>;
    union TS {
        typename Sort::TempStorage sort;
        typename Disc::TempStorage disc;
        typename Scan::TempStorage scan;
    };
    extern __shared__ __align__(16) unsigned char dsm[];
    TS &ts = *reinterpret_cast<TS *>(dsm);
    const int p = blockIdx.x;
    const int e0 = peb[p], nvalid = 2 * (peb[p + 1] - e0);
    const int o0 = pvb[p], nO = pvb[p + 1] - o0;
    const int h0 = hb[p];
    const int lbase = o0 + h0;
    int key[ITEMS], val[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; it++) {
        int j = threadIdx.x * ITEMS + it;
        if (j < nvalid) {
            key[it] = vertex_perm[edges[2 * (int64_t)edge_perm[e0 + (j >> 1)] + (j & 1)]];
            val[it] = j;
        } else {
            key[it] = kSentinel;
            val[it] = j;
        }
    }
    Sort(ts.sort).Sort(key, val, 0, end_bit);
    __syncthreads();
    int head[ITEMS];
    Disc(ts.disc).FlagHeads(head, key, cub::Inequality());
    __syncthreads();
    int low[ITEMS], rank[ITEMS], lowpos[ITEMS];
#pragma unroll
    for (int it = 0; it < ITEMS; it++) {
        const bool valid = threadIdx.x * ITEMS + it < nvalid;
        head[it] = (head[it] && valid) ? 1 : 0;
        low[it] = (valid && key[it] < o0) ? 1 : 0;
    }
    int ndistinct;
    Scan(ts.scan).InclusiveSum(head, rank, ndistinct);  // rank among distinct ids = position in V_p
    __syncthreads();
#pragma unroll
    for (int it = 0; it < ITEMS; it++) rank[it] -= 1;     // (inclusive count of heads) - 1
    int nlow;
    Scan(ts.scan).ExclusiveSum(low, lowpos, nlow);      // nlow = #halo incidences
    (void)ndistinct;
#pragma unroll
    for (int it = 0; it < ITEMS; it++) {
        const int q = threadIdx.x * ITEMS + it;
        if (q >= nvalid) continue;
        const int v = key[it], j = val[it];
        const bool is_halo = v < o0;
        const int slot = is_halo ? nO + rank[it] : v - o0;
        if (head[it] && is_halo) halo_ids[h0 + rank[it]] = v;
        const int pos = is_halo ? q + (nvalid - nlow) : q - nlow;
        slots[2 * (int64_t)e0 + j] = (uint16_t)slot;
        inc[2 * (int64_t)e0 + pos] = (uint16_t)j;
        if (head[it]) inc_off[(int64_t)lbase + slot] = (uint16_t)pos;
    }
}

// vertices appearing in some halo list are shared (p_v > 1)
__global__ void k_mark_shared(const int32_t *__restrict__ halo_ids, int64_t C, int32_t *flag) {
    int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (h < C) flag[halo_ids[h]] = 1;
}

__global__ void k_shared_index(const int32_t *__restrict__ flag, const int32_t *__restrict__ scan, int32_t n,
                               int32_t *sidx, int32_t *shared_ids) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    if (flag[v]) { sidx[v] = scan[v]; shared_ids[scan[v]] = (int32_t)v; }
    else sidx[v] = -1;
}

// halo positions grouped by vertex (sorted keys = vertex ids): CSR offsets per shared index
__global__ void k_hv_off(const int32_t *__restrict__ sorted_ids, int64_t C, const int32_t *__restrict__ sidx,
                         int32_t S, int32_t *hv_off) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r > C) return;
    if (r == C) { hv_off[S] = (int32_t)C; return; }
    if (r == 0 || sorted_ids[r] != sorted_ids[r - 1]) hv_off[sidx[sorted_ids[r]]] = (int32_t)r;
}

// opt_indexA in global ids: new edge i -> (vertex_perm[u], vertex_perm[v]) of task edge_perm[i]
__global__ void k_remapped_edges(const int32_t *__restrict__ edges, const int32_t *__restrict__ edge_perm,
                                 const int32_t *__restrict__ vertex_perm, int64_t m, int32_t *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int64_t e = edge_perm[i];
    out[2 * i] = vertex_perm[edges[2 * e]];
    out[2 * i + 1] = vertex_perm[edges[2 * e + 1]];
}

}  // namespace epg
