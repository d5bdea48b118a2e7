// rb_kernels.cuh -- GPU levels of the EPG-RB partitioner (O5'', reading Z21; SURVEY §8(f)
// rank 2: a GPU-parallel EP partitioner, the role multilevel METIS plays in P:384-386 /
// P:418 and whose cost the paper weighs against the kernel time).
//
// Every node of a bisection level is an independent subproblem, so one level-synchronous
// BFS serves all nodes of the level at once: a frontier task t expands each of its endpoints
// v that is not a hub (more than 4P incident tasks), relaxing the tasks of v's incidence list
// that lie in t's node. Distances are BFS distances, so the result does not depend on the
// order in which threads claim tasks (atomicCAS on dist) or expand vertices (a vertex already
// expanded for the same node in this pass is skipped; one expanded for another node is
// expanded again, which only repeats work). The split sorts (node, dist, task) with a stable
// radix sort of task-ordered input and cuts each node after the task count of its first
// half of partitions.
#pragma once

#include <stdint.h>

namespace epg {

constexpr int32_t kRbInf = 0x7fffffff;
constexpr int kRbDistBits = 22;                  // sort key: node << 22 | min(dist, 2^22 - 1)
constexpr uint32_t kRbDistCap = (1u << kRbDistBits) - 1;

// endpoint slot j = 2t + s -> (vertex, task); the second slot of a self-loop gets vertex n
// (sorted past every real vertex and never read), so a task appears once per vertex
__global__ void k_rb_slot_keys(const int32_t *__restrict__ edges, int64_t m, int32_t n, int32_t *key, int32_t *val) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= 2 * m) return;
    const int32_t v = edges[j];
    key[j] = ((j & 1) && v == edges[j - 1]) ? n : v;
    val[j] = (int32_t)(j >> 1);
}

// ip[v] = first position of vertex v in the sorted slot keys, v in [0, n]
__global__ void k_rb_offsets(const int32_t *__restrict__ sorted, int64_t len, int32_t n, int32_t *ip) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v > n) return;
    int64_t lo = 0, hi = len;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (sorted[mid] < v) lo = mid + 1; else hi = mid;
    }
    ip[v] = (int32_t)lo;
}

__global__ void k_rb_init_dist(int32_t *dist, int64_t m) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < m) dist[t] = kRbInf;
}

// smallest task id of every node (BFS 1 sources). Per-block shared-memory minima first, then
// one global atomic per (block, node): the nodes of a level are few (<= 512), so direct
// global atomics would serialise m updates on a handful of addresses.
__global__ void k_rb_node_min(const int32_t *__restrict__ node, int64_t m, int32_t nodes, int32_t *node_min) {
    extern __shared__ int32_t smin[];
    for (int a = threadIdx.x; a < nodes; a += blockDim.x) smin[a] = INT32_MAX;
    __syncthreads();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x)
        atomicMin(smin + node[t], (int32_t)t);
    __syncthreads();
    for (int a = threadIdx.x; a < nodes; a += blockDim.x)
        if (smin[a] != INT32_MAX) atomicMin(node_min + a, smin[a]);
}

// farthest reached task of every node, ties by smallest id (BFS 2 sources); same two-stage
// reduction of the key (dist << 32) | (~task)
__global__ void k_rb_far_key(const int32_t *__restrict__ node, const int32_t *__restrict__ dist, int64_t m,
                             int32_t nodes, unsigned long long *far) {
    extern __shared__ unsigned long long sfar[];
    for (int a = threadIdx.x; a < nodes; a += blockDim.x) sfar[a] = 0ull;
    __syncthreads();
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m; t += (int64_t)gridDim.x * blockDim.x) {
        if (dist[t] == kRbInf) continue;
        atomicMax(sfar + node[t], ((unsigned long long)(uint32_t)dist[t] << 32) | (0xffffffffu - (uint32_t)t));
    }
    __syncthreads();
    for (int a = threadIdx.x; a < nodes; a += blockDim.x)
        if (sfar[a] != 0ull) atomicMax(far + a, sfar[a]);
}

// sources of a pass: dist = 0 and the frontier; mode 0 from node_min, mode 1 from far keys
__global__ void k_rb_sources(const int32_t *__restrict__ node_min, const unsigned long long *__restrict__ far,
                             int32_t nodes, int mode, int32_t *dist, int32_t *front) {
    const int32_t a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nodes) return;
    const int32_t t = mode == 0 ? node_min[a] : (int32_t)(0xffffffffu - (uint32_t)(far[a] & 0xffffffffull));
    dist[t] = 0;
    front[a] = t;
}

// One BFS level, launched in chunks without a host round trip: the level's frontier count
// is read from cnt[0] and the next level's count is accumulated into cnt[1] (a chunk of
// levels uses consecutive counter slots). Grid-stride over (frontier task, endpoint) items,
// warps kept converged (the loop bound is rounded to a multiple of 32). A vertex v is
// expanded at most once per (pass, node): bit v * nodes + a of the per-pass bitmap `vis`
// (bits == true), or, when the bitmap would not fit, the last (pass, node) key of v (then a
// vertex shared by several nodes may be expanded again -- repeated work, same distances).
// Relaxations are claimed with atomicCAS on dist; a warp reserves its appends with one
// atomicAdd.
__global__ void k_rb_expand(const int32_t *__restrict__ edges, const int32_t *__restrict__ ip,
                            const int32_t *__restrict__ inc, int32_t hub, const int32_t *__restrict__ node,
                            int32_t nodes, int32_t *dist, unsigned long long *vis, bool bits, unsigned long long pass,
                            const int32_t *__restrict__ front, const int32_t *cnt, int32_t *next, int32_t *nnext,
                            int32_t level) {
    const int64_t nf = *cnt;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t bound = (2 * nf + 31) & ~int64_t(31);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < bound; i += stride) {
        bool go = false;
        int32_t q0 = 0, q1 = 0, a = -1;
        if (i < 2 * nf) {
            const int64_t t = front[i >> 1];
            const int side = (int)(i & 1);
            const int32_t v = edges[2 * t + side];
            go = !(side == 1 && v == edges[2 * t]);
            a = node[t];
            if (go) {
                q0 = ip[v];
                q1 = ip[v + 1];
                go = q1 - q0 <= hub;
            }
            if (go) {
                if (bits) {
                    const uint64_t b = (uint64_t)v * (uint64_t)nodes + (uint64_t)a;
                    const unsigned long long bit = 1ull << (b & 63);
                    go = (atomicOr(vis + (b >> 6), bit) & bit) == 0;
                } else {
                    const unsigned long long key = (pass << 32) | (uint32_t)a;
                    go = atomicExch(vis + v, key) != key;
                }
            }
        }
        // relax in chunks of up to 8 claims per thread
        int32_t q = go ? q0 : q1;
        while (__any_sync(0xffffffffu, q < q1)) {
            int32_t buf[8];
            int c = 0;
            while (q < q1 && c < 8) {
                const int32_t u = inc[q++];
                if (node[u] != a || dist[u] != kRbInf) continue;
                if (atomicCAS(dist + u, kRbInf, level + 1) == kRbInf) buf[c++] = u;
            }
            int incl = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            int base = 0;
            if (lane == 31 && total > 0) base = atomicAdd(nnext, total);
            base = __shfl_sync(0xffffffffu, base, 31);
            for (int j = 0; j < c; j++) next[base + incl - c + j] = buf[j];
        }
    }
}

// sort keys of a level: node << 22 | min(dist, cap); values: task ids (ascending input)
__global__ void k_rb_sort_keys(const int32_t *__restrict__ node, const int32_t *__restrict__ dist, int64_t m,
                               uint32_t *key, int32_t *val) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= m) return;
    const uint32_t d = dist[t] == kRbInf ? kRbDistCap : (uint32_t)dist[t];
    key[t] = ((uint32_t)node[t] << kRbDistBits) | (d < kRbDistCap ? d : kRbDistCap);
    val[t] = (int32_t)t;
}

// the cut: position i of the sorted order belongs to node a = key >> 22; the first N0[a]
// tasks of the node (from node_begin[a]) go to child 2a, the rest to 2a + 1
__global__ void k_rb_split(const uint32_t *__restrict__ key, const int32_t *__restrict__ val, int64_t m,
                           const int64_t *__restrict__ node_begin, const int64_t *__restrict__ n0,
                           int32_t *next_node) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int32_t a = (int32_t)(key[i] >> kRbDistBits);
    next_node[val[i]] = 2 * a + (i - node_begin[a] >= n0[a] ? 1 : 0);
}

// ---- leaf grouping for the host EPG-2 stage ----------------------------------------------
// (leaf, vertex) key of endpoint slot j, value j
__global__ void k_rb_leaf_slot_keys(const int32_t *__restrict__ edges, int64_t m, const int32_t *__restrict__ leaf,
                                    unsigned long long *key, int32_t *val) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= 2 * m) return;
    key[j] = ((unsigned long long)(uint32_t)leaf[j >> 1] << 32) | (uint32_t)edges[j];
    val[j] = (int32_t)j;
}

__global__ void k_rb_heads(const unsigned long long *__restrict__ key, int64_t len, int32_t *flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < len) flag[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

// leaf-local vertex id of every endpoint slot: distinct (leaf, vertex) rank minus the rank at
// the leaf's first slot (slot_begin[leaf] = 2 x first task position of the leaf)
__global__ void k_rb_local_ids(const unsigned long long *__restrict__ key, const int32_t *__restrict__ val,
                               const int32_t *__restrict__ incl, int64_t len, const int64_t *__restrict__ slot_begin,
                               int32_t *local_of_slot) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= len) return;
    const int32_t j = (int32_t)(key[i] >> 32);
    local_of_slot[val[i]] = incl[i] - incl[slot_begin[j]];
}

__global__ void k_rb_nlocal(const int32_t *__restrict__ incl, const int64_t *__restrict__ slot_begin, int32_t leaves,
                            int32_t *n_local) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= leaves) return;
    const int64_t b = slot_begin[j], e = slot_begin[j + 1];
    n_local[j] = e > b ? incl[e - 1] - incl[b] + 1 : 0;
}

// tasks grouped by leaf (order[i] = task), endpoints as leaf-local ids
__global__ void k_rb_group_edges(const int32_t *__restrict__ order, int64_t m, const int32_t *__restrict__ local_of_slot,
                                 int32_t *grouped) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int64_t t = order[i];
    grouped[2 * i] = local_of_slot[2 * t];
    grouped[2 * i + 1] = local_of_slot[2 * t + 1];
}

__global__ void k_rb_scatter(const int32_t *__restrict__ order, const int32_t *__restrict__ part_local, int64_t m,
                             int32_t *part) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) part[order[i]] = part_local[i];
}

}  // namespace epg
