// partition.cpp -- host EP partitioner of libepg.so (step a2).
//
// The paper runs the optimisation "using a separate thread on the CPU while kernel is
// executed on the GPU": EP partitioning is sequential graph growing and
// belongs on the host. This is the library's own implementation (binary heap with lazy
// deletion, counting-sort chains); it shares no code with oracle/ and must agree with
// it bit for bit because EPG-1's order is fully fixed by its stamps (O5).
//
//  T (Def. 3, contracted; weight "very large" P:377; chain "in index order"
//  P:380): every vertex's endpoint slots in ascending (task, side) order form a chain;
//  each chain link between two different tasks adds weight 1 to the T-edge joining
//  them (a self-loop's own two slots contract away).
//
//  EPG-1 (replaces METIS, P:384 / P:418): for each partition i, seed at the unassigned
//  task with the earliest global stamp (else the smallest unassigned id); grow s_i
//  tasks, always taking the frontier task with the largest gain g (weight into the
//  partition), ties to the earliest local stamp; restart at the smallest unassigned
//  id when the frontier empties.
#include "epg_internal.h"

#include <algorithm>
#include <cstring>
#include <queue>
#include <string>
#include <vector>

namespace epg {

namespace {

constexpr int64_t kInf = INT64_MAX;

struct TaskGraph {
    std::vector<int64_t> ptr;   // [ntask + 1]
    std::vector<int32_t> adj;   // neighbours, ascending per task
    std::vector<int32_t> w;
};

// Contracted clone-and-connect graph from the edge list.
TaskGraph build_task_graph(const int32_t *edges, int64_t m, int32_t n) {
    // endpoint slots j = 2e + s grouped by vertex; iterating j upward keeps (e, s) order
    std::vector<int64_t> vbeg(static_cast<size_t>(n) + 1, 0);
    for (int64_t j = 0; j < 2 * m; j++) vbeg[edges[j] + 1]++;
    for (int32_t v = 0; v < n; v++) vbeg[v + 1] += vbeg[v];
    std::vector<int64_t> fill(vbeg.begin(), vbeg.end() - 1);
    std::vector<int64_t> chain(2 * m);
    for (int64_t j = 0; j < 2 * m; j++) chain[fill[edges[j]]++] = j;
    // each task has at most 4 chain neighbours (2 slots x predecessor/successor)
    std::vector<int32_t> nb(4 * m), cnt(m, 0);
    for (int32_t v = 0; v < n; v++) {
        for (int64_t q = vbeg[v]; q + 1 < vbeg[v + 1]; q++) {
            int64_t t0 = chain[q] >> 1, t1 = chain[q + 1] >> 1;
            if (t0 == t1) continue;
            nb[4 * t0 + cnt[t0]++] = static_cast<int32_t>(t1);
            nb[4 * t1 + cnt[t1]++] = static_cast<int32_t>(t0);
        }
    }
    TaskGraph T;
    T.ptr.assign(m + 1, 0);
    T.adj.reserve(4 * m);
    T.w.reserve(4 * m);
    for (int64_t t = 0; t < m; t++) {
        int32_t *b = &nb[4 * t];
        std::sort(b, b + cnt[t]);
        for (int c = 0; c < cnt[t]; c++) {
            if (c > 0 && b[c] == b[c - 1]) { T.w.back()++; continue; }
            T.adj.push_back(b[c]);
            T.w.push_back(1);
        }
        T.ptr[t + 1] = static_cast<int64_t>(T.adj.size());
    }
    return T;
}

struct HeapEntry {
    int64_t gain, stamp;
    int32_t task;
};
struct HeapLess {  // max-heap on gain, then min stamp
    bool operator()(const HeapEntry &a, const HeapEntry &b) const {
        if (a.gain != b.gain) return a.gain < b.gain;
        return a.stamp > b.stamp;
    }
};

void grow(const TaskGraph &T, const int64_t *sizes, int64_t nparts, int32_t *part) {
    const int64_t ntask = static_cast<int64_t>(T.ptr.size()) - 1;
    std::vector<int64_t> gst(ntask, kInf), lst(ntask, kInf), gain(ntask, 0);
    std::vector<int32_t> by_gst;
    by_gst.reserve(ntask);
    std::vector<int32_t> dirty;
    std::priority_queue<HeapEntry, std::vector<HeapEntry>, HeapLess> heap;
    std::fill(part, part + ntask, -1);
    size_t gnext = 0;
    int64_t lowest = 0, gclock = 0;
    auto next_unassigned = [&]() {
        while (lowest < ntask && part[lowest] != -1) lowest++;
        return lowest;
    };
    for (int64_t i = 0; i < nparts; i++) {
        while (gnext < by_gst.size() && part[by_gst[gnext]] != -1) gnext++;
        int64_t seed = gnext < by_gst.size() ? by_gst[gnext] : next_unassigned();
        for (int32_t t : dirty) { lst[t] = kInf; gain[t] = 0; }
        dirty.clear();
        heap = decltype(heap)();
        if (sizes[i] == 0) continue;
        int64_t clock = 0;
        lst[seed] = clock++;
        dirty.push_back(static_cast<int32_t>(seed));
        heap.push({0, lst[seed], static_cast<int32_t>(seed)});
        for (int64_t r = 0; r < sizes[i]; r++) {
            int32_t t = -1;
            while (!heap.empty()) {
                HeapEntry top = heap.top();
                heap.pop();
                if (part[top.task] == -1 && gain[top.task] == top.gain) { t = top.task; break; }
            }
            if (t < 0) {  // frontier exhausted: restart on the remainder
                t = static_cast<int32_t>(next_unassigned());
                lst[t] = clock++;
                dirty.push_back(t);
            }
            part[t] = static_cast<int32_t>(i);
            for (int64_t q = T.ptr[t]; q < T.ptr[t + 1]; q++) {
                int32_t u = T.adj[q];
                if (part[u] != -1) continue;
                if (lst[u] == kInf) { lst[u] = clock++; dirty.push_back(u); }
                gain[u] += T.w[q];
                if (gst[u] == kInf) { gst[u] = gclock++; by_gst.push_back(u); }
                heap.push({gain[u], lst[u], u});
            }
        }
    }
}

}  // namespace

epg_status host_partition(const int32_t *edges, int64_t m, int32_t n, int32_t part_size, int32_t shards,
                          int32_t *part, std::string *err) {
    if (m <= 0 || n <= 0 || edges == nullptr || part == nullptr) {
        *err = "partition: need m > 0, n > 0 and non-NULL arrays";
        return EPG_ERR_INPUT;
    }
    for (int64_t e = 0; e < m; e++) {
        int32_t a = edges[2 * e], b = edges[2 * e + 1];
        if (a < 0 || a >= n || b < 0 || b >= n) {
            *err = "partition: edge " + std::to_string(e) + " has an endpoint outside [0, n)";
            return EPG_ERR_INPUT;
        }
    }
    if (part_size < 1 || part_size > EPG_MAX_PART_SIZE) {
        *err = "partition: part_size must be in [1, 4096]";
        return EPG_ERR_INFEASIBLE;
    }
    const int64_t k = (m + part_size - 1) / part_size;
    if (!(shards == 1 || shards == 2 || shards == 4 || shards == 8) || shards > k) {
        *err = "partition: shards must be 1, 2, 4 or 8 and at most k";
        return EPG_ERR_INFEASIBLE;
    }
    std::vector<int64_t> s(k);
    for (int64_t i = 0; i < k; i++) s[i] = m / k + (i < m % k ? 1 : 0);
    TaskGraph T = build_task_graph(edges, m, n);
    if (shards == 1) {
        grow(T, s.data(), k, part);
        return EPG_OK;
    }
    // hierarchical: shard-level growing, then growing inside each shard
    std::vector<int64_t> ssize(shards, 0);
    for (int g = 0; g < shards; g++)
        for (int64_t i = g * k / shards; i < (g + 1) * k / shards; i++) ssize[g] += s[i];
    std::vector<int32_t> shard(m);
    grow(T, ssize.data(), shards, shard.data());
    std::vector<std::vector<int32_t>> members(shards);
    for (int64_t t = 0; t < m; t++) members[shard[t]].push_back(static_cast<int32_t>(t));
    std::vector<int32_t> local(m);
    for (int g = 0; g < shards; g++)
        for (size_t j = 0; j < members[g].size(); j++) local[members[g][j]] = static_cast<int32_t>(j);
    for (int g = 0; g < shards; g++) {
        const auto &mem = members[g];
        TaskGraph Tg;
        Tg.ptr.assign(mem.size() + 1, 0);
        for (size_t j = 0; j < mem.size(); j++) {
            int32_t t = mem[j];
            for (int64_t q = T.ptr[t]; q < T.ptr[t + 1]; q++) {
                if (shard[T.adj[q]] != g) continue;
                Tg.adj.push_back(local[T.adj[q]]);
                Tg.w.push_back(T.w[q]);
            }
            Tg.ptr[j + 1] = static_cast<int64_t>(Tg.adj.size());
        }
        const int64_t p0 = g * k / shards, p1 = (g + 1) * k / shards;
        std::vector<int32_t> sub(mem.size());
        grow(Tg, s.data() + p0, p1 - p0, sub.data());
        for (size_t j = 0; j < mem.size(); j++) part[mem[j]] = static_cast<int32_t>(sub[j] + p0);
    }
    return EPG_OK;
}

}  // namespace epg

extern "C" epg_status epg_partition_host(const int32_t *edges, int64_t m, int32_t n_vertices, int32_t part_size,
                                         int32_t shards, int32_t *part_of_edge, char *errbuf, int64_t errbuf_len) {
    std::string err;
    epg_status st = epg::host_partition(edges, m, n_vertices, part_size, shards, part_of_edge, &err);
    if (st != EPG_OK && errbuf && errbuf_len > 0) {
        std::strncpy(errbuf, err.c_str(), static_cast<size_t>(errbuf_len - 1));
        errbuf[errbuf_len - 1] = '\0';
    }
    return st;
}

extern "C" int64_t epg_num_parts(int64_t m, int32_t part_size) {
    if (m <= 0 || part_size <= 0) return 0;
    return (m + part_size - 1) / part_size;
}
