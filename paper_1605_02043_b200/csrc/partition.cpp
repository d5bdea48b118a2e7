// partition.cpp -- host EP partitioner of libepg.so (step a2).
//
// The paper runs the optimisation "using a separate thread on the CPU while kernel is
// executed on the GPU": EP partitioning is sequential graph growing and
// belongs on the host. This is the library's own implementation (fixed-width T, packed
// per-task state, one lazy-deletion min-heap per gain value, counting-sort chains); it
// shares no code with oracle/ and must agree with it bit for bit because EPG-1's order is
// fully fixed by its stamps (O5).
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
//
//  EPG-2 (reading Z20): the same schedule, but the gain
//  is Eq. (1)'s own objective -- a task's distinct endpoints already loaded by the
//  partition (one load per distinct vertex), so the pick adds the fewest new
//  loads. The frontier grows through the vertex incidence lists instead of T; vertices
//  with more than 4 x part_size tasks (hubs) attract none.
#include "epg_internal.h"

#include <sched.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <queue>
#include <string>
#include <thread>
#include <vector>

namespace epg {

namespace {

constexpr int64_t kInf = INT64_MAX;

// T with at most 4 chain links per task (2 endpoint slots x predecessor / successor in the
// vertex chains): fixed 4-slot rows, ascending, unused slots -1. A weight-w edge of T
// (w links to the same task) is kept as w repeated unit entries: visiting them one by one
// leaves the same gains, stamps and current heap entries as adding w at once (the
// intermediate entry goes stale under lazy deletion), so the gain never exceeds 4.
struct TaskGraph {
    int64_t ntask = 0;
    std::vector<int32_t> nb;   // [4 * ntask]
};

// Contracted clone-and-connect graph from the edge list.
TaskGraph build_task_graph(const int32_t *edges, int64_t m, int32_t n) {
    // endpoint slots j = 2e + s grouped by vertex; iterating j upward keeps (e, s) order
    std::vector<int64_t> vbeg(static_cast<size_t>(n) + 1, 0);
    for (int64_t j = 0; j < 2 * m; j++) vbeg[edges[j] + 1]++;
    for (int32_t v = 0; v < n; v++) vbeg[v + 1] += vbeg[v];
    std::vector<int64_t> fill(vbeg.begin(), vbeg.end() - 1);
    std::vector<uint32_t> chain(2 * m);   // m < 2^31 (checked by host_partition)
    for (int64_t j = 0; j < 2 * m; j++) chain[fill[edges[j]]++] = static_cast<uint32_t>(j);
    std::vector<int64_t>().swap(fill);
    TaskGraph T;
    T.ntask = m;
    T.nb.assign(4 * m, -1);
    std::vector<uint8_t> cnt(m, 0);
    for (int32_t v = 0; v < n; v++) {
        for (int64_t q = vbeg[v]; q + 1 < vbeg[v + 1]; q++) {
            int64_t t0 = chain[q] >> 1, t1 = chain[q + 1] >> 1;
            if (t0 == t1) continue;
            T.nb[4 * t0 + cnt[t0]++] = static_cast<int32_t>(t1);
            T.nb[4 * t1 + cnt[t1]++] = static_cast<int32_t>(t0);
        }
    }
    // per task: sort its <= 4 links ascending (slots past cnt stay -1)
    for (int64_t t = 0; t < m; t++) std::sort(&T.nb[4 * t], &T.nb[4 * t] + cnt[t]);
    return T;
}

// Per-task growing state in one 16-byte record (one cache line per neighbour visit).
struct TaskState {
    int32_t part;   // -1 unassigned
    int32_t lst;    // local stamp (kNoStamp = none since the last reset)
    int32_t gst;    // global stamp (kNoStamp = none)
    int32_t gain;   // weight into the current partition, 0..4
};
constexpr int32_t kNoStamp = INT32_MAX;

// Frontier: per gain value (0..4) the set of local stamps of the unassigned tasks whose gain
// currently equals it; the pick -- largest gain, then smallest local stamp -- is EPG-1's (O5).
// Gains only grow (0 for the seed, +1 per push), so a push moves the task's stamp from bucket
// g - 1 to g and every bucket holds exactly the current entries; stamps are unique within a
// partition. Each bucket is a hierarchical bitset over the stamps (64-way levels, find-first
// through the summaries): O(levels) per push and pop instead of a binary heap with lazy
// deletion -- the same picks, so the same maps.
class StampSet {
    std::vector<std::vector<uint64_t>> lv_;   // lv_[0]: one bit per stamp; lv_[l + 1]: word l non-zero
    size_t used_ = 0;                         // words of lv_[0] that may hold set bits
public:
    void reserve(size_t nbits) {
        size_t words = (nbits + 63) / 64;
        if (!lv_.empty() && lv_[0].size() >= words) return;
        words = std::max<size_t>(words, lv_.empty() ? 1 : 2 * lv_[0].size());
        std::vector<std::vector<uint64_t>> nl;
        for (size_t w = words;; w = (w + 63) / 64) {
            nl.emplace_back(w, 0);
            if (w == 1) break;
        }
        for (size_t l = 0; l < lv_.size() && l < nl.size(); l++)   // keep the set bits
            std::copy(lv_[l].begin(), lv_[l].end(), nl[l].begin());
        for (size_t l = std::max<size_t>(1, lv_.size()); l < nl.size(); l++)   // summaries of new levels
            for (size_t w = 0; w < nl[l - 1].size(); w++)
                if (nl[l - 1][w]) nl[l][w >> 6] |= 1ull << (w & 63);
        lv_.swap(nl);
    }
    void set(uint32_t s) {
        for (size_t l = 0; l < lv_.size(); l++) {
            uint64_t &w = lv_[l][s >> 6];
            const bool was = w != 0;
            w |= 1ull << (s & 63);
            if (l == 0) used_ = std::max<size_t>(used_, (s >> 6) + 1);
            if (was) return;
            s >>= 6;
        }
    }
    void reset(uint32_t s) {
        for (size_t l = 0; l < lv_.size(); l++) {
            uint64_t &w = lv_[l][s >> 6];
            w &= ~(1ull << (s & 63));
            if (w) return;
            s >>= 6;
        }
    }
    // smallest set stamp, or -1
    int64_t first() const {
        if (lv_.empty() || lv_.back()[0] == 0) return -1;
        uint64_t idx = 0;
        for (size_t l = lv_.size(); l-- > 0;) idx = (idx << 6) | static_cast<uint64_t>(__builtin_ctzll(lv_[l][idx]));
        return static_cast<int64_t>(idx);
    }
    void clear() {
        size_t words = used_;
        for (size_t l = 0; l < lv_.size() && words > 0; l++) {
            std::fill(lv_[l].begin(), lv_[l].begin() + std::min(words, lv_[l].size()), 0);
            words = (words + 63) / 64;
        }
        used_ = 0;
    }
};

struct BitFrontier {
    StampSet h[5];
    std::vector<int32_t> task_of;   // local stamp -> task
    void clear() { for (auto &b : h) b.clear(); }
    void push(int gain, int32_t stamp, int32_t task) {
        const uint32_t s = static_cast<uint32_t>(stamp);
        if (task_of.size() <= s) {
            task_of.resize(std::max<size_t>(2 * task_of.size(), s + 1));
            for (auto &b : h) b.reserve(task_of.size());
        }
        task_of[s] = task;
        if (gain > 0) h[gain - 1].reset(s);
        h[gain].set(s);
    }
    // pop the best current entry; -1 when empty
    int32_t pop(const std::vector<TaskState> &) {
        for (int g = 4; g >= 0; g--) {
            const int64_t s = h[g].first();
            if (s >= 0) {
                h[g].reset(static_cast<uint32_t>(s));
                return task_of[s];
            }
        }
        return -1;
    }
};

// The same frontier as binary min-heaps on (local stamp, task) per gain with lazy deletion (an
// entry is current iff the task is unassigned and its gain still equals the bucket): faster
// than the bitsets when a partition's stamps run into the millions (EPG-2 on power-law graphs,
// where loading one vertex stamps thousands of tasks); the picks are identical.
struct HeapFrontier {
    std::vector<uint64_t> h[5];   // (stamp << 32) | task, min-heaps
    void clear() { for (auto &v : h) v.clear(); }
    void push(int gain, int32_t stamp, int32_t task) {
        auto &v = h[gain];
        v.push_back((static_cast<uint64_t>(static_cast<uint32_t>(stamp)) << 32) | static_cast<uint32_t>(task));
        std::push_heap(v.begin(), v.end(), std::greater<uint64_t>());
    }
    int32_t pop(const std::vector<TaskState> &st) {
        for (int g = 4; g >= 0; g--) {
            auto &v = h[g];
            while (!v.empty()) {
                const uint64_t top = v.front();
                std::pop_heap(v.begin(), v.end(), std::greater<uint64_t>());
                v.pop_back();
                const int32_t t = static_cast<int32_t>(top & 0xffffffffu);
                if (st[t].part == -1 && st[t].gain == g) return t;
            }
        }
        return -1;
    }
};

// returns false if *cancel became non-zero (checked once per partition)
// rank (may be NULL): the step at which each task joined its partition (reading Z22)
bool grow(const TaskGraph &T, const int64_t *sizes, int64_t nparts, int32_t *part, const std::atomic<int> *cancel,
          int32_t *rank = nullptr) {
    const int64_t ntask = T.ntask;
    std::vector<TaskState> st(ntask, TaskState{-1, kNoStamp, kNoStamp, 0});
    std::vector<int32_t> by_gst;
    by_gst.reserve(ntask);
    std::vector<int32_t> dirty;
    BitFrontier fr;
    size_t gnext = 0;
    int64_t lowest = 0;
    int32_t gclock = 0;
    auto next_unassigned = [&]() {
        while (lowest < ntask && st[lowest].part != -1) lowest++;
        return lowest;
    };
    for (int64_t i = 0; i < nparts; i++) {
        if (cancel && cancel->load(std::memory_order_relaxed)) return false;
        while (gnext < by_gst.size() && st[by_gst[gnext]].part != -1) gnext++;
        const int64_t seed = gnext < by_gst.size() ? by_gst[gnext] : next_unassigned();
        for (int32_t t : dirty) { st[t].lst = kNoStamp; st[t].gain = 0; }
        dirty.clear();
        fr.clear();
        if (sizes[i] == 0) continue;
        int32_t clock = 0;
        st[seed].lst = clock++;
        dirty.push_back(static_cast<int32_t>(seed));
        fr.push(0, st[seed].lst, static_cast<int32_t>(seed));
        for (int64_t r = 0; r < sizes[i]; r++) {
            int32_t t = fr.pop(st);
            if (t < 0) {  // frontier exhausted: restart on the remainder
                t = static_cast<int32_t>(next_unassigned());
                st[t].lst = clock++;
                dirty.push_back(t);
            }
            st[t].part = static_cast<int32_t>(i);
            part[t] = static_cast<int32_t>(i);
            if (rank) rank[t] = static_cast<int32_t>(r);
            const int32_t *nb = &T.nb[4 * static_cast<int64_t>(t)];
            for (int c = 0; c < 4 && nb[c] >= 0; c++) __builtin_prefetch(&st[nb[c]]);
            for (int c = 0; c < 4 && nb[c] >= 0; c++) {
                TaskState &u = st[nb[c]];
                if (u.part != -1) continue;
                if (u.lst == kNoStamp) {
                    u.lst = clock++;
                    dirty.push_back(nb[c]);
                    __builtin_prefetch(&T.nb[4 * static_cast<int64_t>(nb[c])]);
                }
                u.gain += 1;
                if (u.gst == kNoStamp) { u.gst = gclock++; by_gst.push_back(nb[c]); }
                fr.push(u.gain, u.lst, nb[c]);
            }
        }
    }
    return true;
}

// ---- EPG-2 ----------------------------------------------------------------------
// Vertex -> incident tasks (ascending, each task once: a self-loop appears once).
struct Incidence {
    std::vector<int64_t> beg;   // [n + 1]
    std::vector<int32_t> task;
};

Incidence build_incidence(const int32_t *edges, int64_t m, int32_t n) {
    Incidence I;
    I.beg.assign(static_cast<size_t>(n) + 1, 0);
    for (int64_t t = 0; t < m; t++) {
        I.beg[edges[2 * t] + 1]++;
        if (edges[2 * t + 1] != edges[2 * t]) I.beg[edges[2 * t + 1] + 1]++;
    }
    for (int32_t v = 0; v < n; v++) I.beg[v + 1] += I.beg[v];
    std::vector<int64_t> at(I.beg.begin(), I.beg.end() - 1);
    I.task.resize(static_cast<size_t>(I.beg[n]));
    for (int64_t t = 0; t < m; t++) {   // ascending t: lists come out sorted
        I.task[at[edges[2 * t]]++] = static_cast<int32_t>(t);
        if (edges[2 * t + 1] != edges[2 * t]) I.task[at[edges[2 * t + 1]]++] = static_cast<int32_t>(t);
    }
    return I;
}

// EPG-2 growing: frontier heaps per gain 0..2 (distinct endpoints inside), lazy deletion
// as for EPG-1; a vertex joins V_i the first time one of its tasks is taken (mark[v] = i
// + 1, so the per-partition reset is free).
// A vertex with more than `hub` incident tasks (4 x part_size: it is cut into many clusters
// whatever happens) attracts no tasks -- the hub discussion of P:642-683, reading Z20.
template <class Frontier>
bool grow_direct_t(const int32_t *edges, int64_t ntask, int32_t n, const int64_t *sizes, int64_t nparts, int64_t hub,
                   int32_t *part, const std::atomic<int> *cancel, int32_t *rank, Incidence &I) {
    std::vector<int64_t> live_end(I.beg.begin() + 1, I.beg.end());   // end of v's live (unassigned) tasks
    std::vector<TaskState> st(ntask, TaskState{-1, kNoStamp, kNoStamp, 0});
    std::vector<int64_t> mark(static_cast<size_t>(n), 0);
    std::vector<int32_t> by_gst;
    by_gst.reserve(ntask);
    std::vector<int32_t> dirty;
    Frontier fr;
    size_t gnext = 0;
    int64_t lowest = 0;
    int32_t gclock = 0;
    auto next_unassigned = [&]() {
        while (lowest < ntask && st[lowest].part != -1) lowest++;
        return lowest;
    };
    for (int64_t i = 0; i < nparts; i++) {
        if (cancel && cancel->load(std::memory_order_relaxed)) return false;
        while (gnext < by_gst.size() && st[by_gst[gnext]].part != -1) gnext++;
        const int64_t seed = gnext < by_gst.size() ? by_gst[gnext] : next_unassigned();
        for (int32_t t : dirty) { st[t].lst = kNoStamp; st[t].gain = 0; }
        dirty.clear();
        fr.clear();
        if (sizes[i] == 0) continue;
        int32_t clock = 0;
        st[seed].lst = clock++;
        dirty.push_back(static_cast<int32_t>(seed));
        fr.push(0, st[seed].lst, static_cast<int32_t>(seed));
        for (int64_t r = 0; r < sizes[i]; r++) {
            int32_t t = fr.pop(st);
            if (t < 0) {  // frontier exhausted: restart on the remainder
                t = static_cast<int32_t>(next_unassigned());
                st[t].lst = clock++;
                dirty.push_back(t);
            }
            st[t].part = static_cast<int32_t>(i);
            part[t] = static_cast<int32_t>(i);
            if (rank) rank[t] = static_cast<int32_t>(r);
            const int32_t ends[2] = {edges[2 * static_cast<int64_t>(t)], edges[2 * static_cast<int64_t>(t) + 1]};
            for (int side = 0; side < 2; side++) {
                const int32_t v = ends[side];
                if (side == 1 && v == ends[0]) break;   // distinct endpoints only
                if (mark[v] == i + 1) continue;         // already loaded by this partition
                mark[v] = i + 1;
                if (I.beg[v + 1] - I.beg[v] > hub) continue;   // the hub rule uses the full degree
                // scan v's live tasks, dropping assigned ones from the list on the way (order
                // kept, so the visit order is still ascending id: same result, and a
                // high-degree vertex is not rescanned in full by every partition loading it)
                int64_t wr = I.beg[v];
                for (int64_t q = I.beg[v]; q < live_end[v]; q++) {
                    const int32_t w = I.task[q];
                    TaskState &u = st[w];
                    if (u.part != -1) continue;
                    I.task[wr++] = w;
                    if (u.lst == kNoStamp) {
                        u.lst = clock++;
                        dirty.push_back(w);
                    }
                    u.gain += 1;
                    if (u.gst == kNoStamp) { u.gst = gclock++; by_gst.push_back(w); }
                    fr.push(u.gain, u.lst, w);
                }
                live_end[v] = wr;
            }
        }
    }
    return true;
}

// EPG-2 with the frontier that suits the graph: the bitsets when every vertex has at most
// 64 incident tasks (meshes; a partition stamps a few thousand tasks), the heaps otherwise
bool grow_direct(const int32_t *edges, int64_t ntask, int32_t n, const int64_t *sizes, int64_t nparts, int64_t hub,
                 int32_t *part, const std::atomic<int> *cancel, int32_t *rank = nullptr) {
    Incidence I = build_incidence(edges, ntask, n);
    int64_t dmax = 0;
    for (int32_t v = 0; v < n; v++) dmax = std::max(dmax, I.beg[v + 1] - I.beg[v]);
    return dmax <= 64 ? grow_direct_t<BitFrontier>(edges, ntask, n, sizes, nparts, hub, part, cancel, rank, I)
                      : grow_direct_t<HeapFrontier>(edges, ntask, n, sizes, nparts, hub, part, cancel, rank, I);
}

}  // namespace

int host_cpus() {
    cpu_set_t set;
    if (sched_getaffinity(0, sizeof(set), &set) == 0) return std::max(1, CPU_COUNT(&set));
    return std::max(1u, std::thread::hardware_concurrency());
}

epg_status rb_leaves(const int32_t *local_edges, int64_t m, const int32_t *n_local, int32_t leaves,
                     int32_t part_size, int32_t *part_local, std::string *err, int threads,
                     const std::atomic<int32_t> *ready, int32_t *rank_local) {
    const int64_t k = (m + part_size - 1) / part_size;
    std::vector<int64_t> s(k), S(k + 1, 0);
    for (int64_t i = 0; i < k; i++) {
        s[i] = m / k + (i < m % k ? 1 : 0);
        S[i + 1] = S[i] + s[i];
    }
    const int64_t hub = 4 * static_cast<int64_t>(part_size);
    std::atomic<int32_t> next_leaf{0};
    auto worker = [&]() {
        for (;;) {
            const int32_t j = next_leaf.fetch_add(1);
            if (j >= leaves) return;
            const int64_t p0 = static_cast<int64_t>(j) * k / leaves, p1 = static_cast<int64_t>(j + 1) * k / leaves;
            const int64_t b = S[p0], nt = S[p1] - S[p0];   // the leaf's tasks, grouped and ascending
            if (nt == 0) continue;
            if (ready)   // the leaf's edges are still being copied in
                while (ready->load(std::memory_order_acquire) <= j) std::this_thread::yield();
            grow_direct(local_edges + 2 * b, nt, n_local[j], s.data() + p0, p1 - p0, hub, part_local + b, nullptr,
                        rank_local ? rank_local + b : nullptr);
            for (int64_t q = 0; q < nt; q++) part_local[b + q] += static_cast<int32_t>(p0);
        }
    };
    const int nth = std::max(1, std::min<int>(threads > 0 ? threads : host_cpus(), leaves));
    std::vector<std::thread> pool;
    for (int i = 1; i < nth; i++) pool.emplace_back(worker);
    worker();
    for (auto &th : pool) th.join();
    (void)err;
    return EPG_OK;
}

epg_status host_partition(const int32_t *edges, int64_t m, int32_t n, int32_t part_size, int32_t shards,
                          int32_t *part, std::string *err, const std::atomic<int> *cancel, int32_t method,
                          int32_t *rank) {
    if (method == EPG_PARTITION_RB) {
        *err = "partition: EPG-RB bisects on the GPU -- use epg_partition / epg_partition_rb";
        return EPG_ERR_INPUT;
    }
    if (method != EPG_PARTITION_EPG1 && method != EPG_PARTITION_EPG2) {
        *err = "partition: method must be 1 (EPG-1) or 2 (EPG-2)";
        return EPG_ERR_INPUT;
    }
    if (m <= 0 || n <= 0 || edges == nullptr || part == nullptr) {
        *err = "partition: need m > 0, n > 0 and non-NULL arrays";
        return EPG_ERR_INPUT;
    }
    if (m >= (int64_t(1) << 31)) {   // task ids and stamps are int32
        *err = "partition: m must be below 2^31";
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
    auto cancelled = [&]() {
        *err = "partition: cancelled";
        return EPG_ERR_STATE;
    };
    if (method == EPG_PARTITION_EPG2) {
        const int64_t hub = 4 * static_cast<int64_t>(part_size);
        if (shards == 1) return grow_direct(edges, m, n, s.data(), k, hub, part, cancel, rank) ? EPG_OK : cancelled();
        // hierarchical: shard-level growing, then growing on each shard's own edge list
        std::vector<int64_t> ssize(shards, 0);
        for (int g = 0; g < shards; g++)
            for (int64_t i = g * k / shards; i < (g + 1) * k / shards; i++) ssize[g] += s[i];
        std::vector<int32_t> shard(m);
        if (!grow_direct(edges, m, n, ssize.data(), shards, hub, shard.data(), cancel)) return cancelled();
        for (int g = 0; g < shards; g++) {
            std::vector<int32_t> mem, sub_edges;
            for (int64_t t = 0; t < m; t++)
                if (shard[t] == g) {
                    mem.push_back(static_cast<int32_t>(t));
                    sub_edges.push_back(edges[2 * t]);
                    sub_edges.push_back(edges[2 * t + 1]);
                }
            const int64_t p0 = g * k / shards, p1 = (g + 1) * k / shards;
            std::vector<int32_t> sub(mem.size()), subr(mem.size());
            if (!grow_direct(sub_edges.data(), static_cast<int64_t>(mem.size()), n, s.data() + p0, p1 - p0, hub,
                             sub.data(), cancel, subr.data()))
                return cancelled();
            for (size_t j = 0; j < mem.size(); j++) {
                part[mem[j]] = static_cast<int32_t>(sub[j] + p0);
                if (rank) rank[mem[j]] = subr[j];
            }
        }
        return EPG_OK;
    }
    TaskGraph T = build_task_graph(edges, m, n);
    if (shards == 1) return grow(T, s.data(), k, part, cancel, rank) ? EPG_OK : cancelled();
    // hierarchical: shard-level growing, then growing inside each shard
    std::vector<int64_t> ssize(shards, 0);
    for (int g = 0; g < shards; g++)
        for (int64_t i = g * k / shards; i < (g + 1) * k / shards; i++) ssize[g] += s[i];
    std::vector<int32_t> shard(m);
    if (!grow(T, ssize.data(), shards, shard.data(), cancel)) return cancelled();
    std::vector<std::vector<int32_t>> members(shards);
    for (int64_t t = 0; t < m; t++) members[shard[t]].push_back(static_cast<int32_t>(t));
    std::vector<int32_t> local(m);
    for (int g = 0; g < shards; g++)
        for (size_t j = 0; j < members[g].size(); j++) local[members[g][j]] = static_cast<int32_t>(j);
    for (int g = 0; g < shards; g++) {
        const auto &mem = members[g];
        TaskGraph Tg;
        Tg.ntask = static_cast<int64_t>(mem.size());
        Tg.nb.assign(4 * mem.size(), -1);
        for (size_t j = 0; j < mem.size(); j++) {
            const int64_t t = mem[j];
            int o = 0;   // ascending ids map to ascending local ids: order preserved
            for (int c = 0; c < 4 && T.nb[4 * t + c] >= 0; c++) {
                const int32_t u = T.nb[4 * t + c];
                if (shard[u] != g) continue;
                Tg.nb[4 * j + o] = local[u];
                o++;
            }
        }
        const int64_t p0 = g * k / shards, p1 = (g + 1) * k / shards;
        std::vector<int32_t> sub(mem.size()), subr(mem.size());
        if (!grow(Tg, s.data() + p0, p1 - p0, sub.data(), cancel, subr.data())) return cancelled();
        for (size_t j = 0; j < mem.size(); j++) {
            part[mem[j]] = static_cast<int32_t>(sub[j] + p0);
            if (rank) rank[mem[j]] = subr[j];
        }
    }
    return EPG_OK;
}

}  // namespace epg

extern "C" epg_status epg_partition_host(const int32_t *edges, int64_t m, int32_t n_vertices, int32_t part_size,
                                         int32_t shards, int32_t *part_of_edge, char *errbuf, int64_t errbuf_len) {
    return epg_partition_host_method(edges, m, n_vertices, part_size, shards, EPG_PARTITION_EPG1, part_of_edge, errbuf,
                                     errbuf_len);
}

extern "C" epg_status epg_partition_host_method(const int32_t *edges, int64_t m, int32_t n_vertices, int32_t part_size,
                                                int32_t shards, int32_t method, int32_t *part_of_edge, char *errbuf,
                                                int64_t errbuf_len) {
    return epg_partition_host_ranked(edges, m, n_vertices, part_size, shards, method, part_of_edge, nullptr, errbuf,
                                     errbuf_len);
}

extern "C" epg_status epg_partition_host_ranked(const int32_t *edges, int64_t m, int32_t n_vertices, int32_t part_size,
                                                int32_t shards, int32_t method, int32_t *part_of_edge,
                                                int32_t *rank_of_edge, char *errbuf, int64_t errbuf_len) {
    std::string err;
    epg_status st = epg::host_partition(edges, m, n_vertices, part_size, shards, part_of_edge, &err, nullptr, method,
                                        rank_of_edge);
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
