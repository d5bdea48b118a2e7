// baselines.cpp -- PowerGraph's two edge partitioners, the partition-quality
// comparators of SURVEY §8(f) rank 4, on the host (part of libepg.so).
//
// Both produce k = ceil(m / part_size) clusters like the EP partitioner (O1), so any of
// the three maps runs through the same remap and staged kernels. The definitions are the
// DESIGN.md readings Z18 (random: SplitMix64 order dealt round-robin, exact balance) and
// Z19 (greedy: one pass, highest endpoint-presence score among non-full clusters, ties
// by fewer edges then lower id). This file shares no code with oracle/; the GPU tests
// and tests/test_abi.py compare the two bit for bit.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "../../include/epg.h"

namespace epg {
namespace {

// SplitMix64 output number c of stream `seed` (the counter-based generator the inputs
// are drawn with; each side of the parity test implements it)
inline uint64_t splitmix64(uint64_t seed, uint64_t c) {
    uint64_t z = seed + (c + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void put_err(char *buf, int64_t len, const std::string &msg) {
    if (!buf || len <= 0) return;
    const size_t c = std::min<size_t>((size_t)len - 1, msg.size());
    std::memcpy(buf, msg.data(), c);
    buf[c] = '\0';
}

}  // namespace

epg_status host_partition_random(int64_t m, int32_t part_size, uint64_t seed, int32_t *part, std::string *err) {
    if (m <= 0 || !part) {
        *err = "partition_random: need m > 0 and a non-NULL output";
        return EPG_ERR_INPUT;
    }
    if (part_size < 1 || part_size > EPG_MAX_PART_SIZE) {
        *err = "partition_random: part_size must be in [1, 4096]";
        return EPG_ERR_INFEASIBLE;
    }
    const int64_t k = (m + part_size - 1) / part_size;
    std::vector<std::pair<uint64_t, int64_t>> order((size_t)m);
    for (int64_t e = 0; e < m; e++) order[(size_t)e] = {splitmix64(seed, (uint64_t)e), e};
    std::sort(order.begin(), order.end());
    for (int64_t i = 0; i < m; i++) part[order[(size_t)i].second] = (int32_t)(i % k);
    return EPG_OK;
}

epg_status host_partition_greedy(const int32_t *edges, int64_t m, int32_t n, int32_t part_size, int32_t *part,
                                 std::string *err) {
    if (m <= 0 || n <= 0 || !edges || !part) {
        *err = "partition_greedy: need m > 0, n > 0 and non-NULL arrays";
        return EPG_ERR_INPUT;
    }
    for (int64_t e = 0; e < m; e++) {
        const int32_t a = edges[2 * e], b = edges[2 * e + 1];
        if (a < 0 || a >= n || b < 0 || b >= n) {
            *err = "partition_greedy: edge " + std::to_string(e) + " has an endpoint outside [0, n)";
            return EPG_ERR_INPUT;
        }
    }
    if (part_size < 1 || part_size > EPG_MAX_PART_SIZE) {
        *err = "partition_greedy: part_size must be in [1, 4096]";
        return EPG_ERR_INFEASIBLE;
    }
    const int64_t k = (m + part_size - 1) / part_size;
    const int64_t cap = (m + k - 1) / k;
    // A(v): clusters already holding v, as singly linked lists in flat arrays
    std::vector<int64_t> head((size_t)n, -1), next;
    std::vector<int32_t> clus;
    next.reserve((size_t)(2 * m));
    clus.reserve((size_t)(2 * m));
    std::vector<int64_t> size((size_t)k, 0), seen_u((size_t)k, -1), seen_v((size_t)k, -1);
    std::set<std::pair<int64_t, int32_t>> open;   // (edges, id) of the non-full clusters
    for (int64_t c = 0; c < k; c++) open.insert({0, (int32_t)c});
    for (int64_t e = 0; e < m; e++) {
        const int32_t u = edges[2 * e], v = edges[2 * e + 1];
        for (int64_t q = head[u]; q >= 0; q = next[q]) seen_u[clus[q]] = e;
        for (int64_t q = head[v]; q >= 0; q = next[q]) seen_v[clus[q]] = e;
        // best non-full cluster holding an endpoint: (score desc, edges asc, id asc)
        int32_t best = -1;
        int best_score = 0;
        auto consider = [&](int32_t c) {
            if (size[c] >= cap) return;
            const int sc = (seen_u[c] == e ? 1 : 0) + (seen_v[c] == e ? 1 : 0);
            if (best < 0 || sc > best_score || (sc == best_score && (size[c] < size[best] ||
                                                                      (size[c] == size[best] && c < best)))) {
                best = c;
                best_score = sc;
            }
        };
        for (int64_t q = head[u]; q >= 0; q = next[q]) consider(clus[q]);
        for (int64_t q = head[v]; q >= 0; q = next[q]) consider(clus[q]);
        if (best < 0) best = open.begin()->second;   // no holder open: the fewest edges, lowest id
        part[e] = best;
        open.erase({size[best], best});
        if (++size[best] < cap) open.insert({size[best], best});
        if (seen_u[best] != e) {
            clus.push_back(best);
            next.push_back(head[u]);
            head[u] = (int64_t)clus.size() - 1;
            if (u == v) seen_v[best] = e;            // a self-loop adds its vertex once
        }
        if (seen_v[best] != e) {
            clus.push_back(best);
            next.push_back(head[v]);
            head[v] = (int64_t)clus.size() - 1;
        }
    }
    return EPG_OK;
}

}  // namespace epg

extern "C" {

epg_status epg_partition_random_host(int64_t m, int32_t part_size, uint64_t seed, int32_t *part_of_edge,
                                     char *errbuf, int64_t errbuf_len) {
    std::string err;
    const epg_status st = epg::host_partition_random(m, part_size, seed, part_of_edge, &err);
    if (st) epg::put_err(errbuf, errbuf_len, err);
    return st;
}

epg_status epg_partition_greedy_host(const int32_t *edges, int64_t m, int32_t n_vertices, int32_t part_size,
                                     int32_t *part_of_edge, char *errbuf, int64_t errbuf_len) {
    std::string err;
    const epg_status st = epg::host_partition_greedy(edges, m, n_vertices, part_size, part_of_edge, &err);
    if (st) epg::put_err(errbuf, errbuf_len, err);
    return st;
}

}  // extern "C"
