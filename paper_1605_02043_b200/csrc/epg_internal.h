// epg_internal.h -- private declarations of libepg.so (not installed, not part of the ABI).
#pragma once

#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/epg.h"

namespace epg {

// Host EPG-1 / EPG-2 (partition.cpp; method EPG_PARTITION_*). A non-zero *cancel (polled
// once per partition) stops it with EPG_ERR_STATE ("partition: cancelled").
// rank (may be NULL): each task's growth step within its partition (reading Z22).
epg_status host_partition(const int32_t *edges, int64_t m, int32_t n, int32_t part_size, int32_t shards,
                          int32_t *part, std::string *err, const std::atomic<int> *cancel = nullptr,
                          int32_t method = EPG_PARTITION_EPG1, int32_t *rank = nullptr);

// EPG-RB leaves (O5'', reading Z21): EPG-2 (hub = 4 x part_size) on every leaf's tasks.
// local_edges [m][2] HOST: the tasks grouped by leaf (leaf j holds the tasks of its
// partitions [floor(j k / L), floor((j+1) k / L)), so it starts at task position S_p0),
// ascending within a leaf, endpoints relabelled to leaf-local ids in [0, n_local[j]) --
// which leaves EPG-2 unchanged (it depends on vertex identity only). part_local [m] HOST out,
// in the same grouped order, global partition ids. Leaves run on `threads` host threads
// (0: every CPU this process may run on). ready (may be NULL): leaf j is processed once
// *ready > j (the caller streams local_edges in leaf order).
epg_status rb_leaves(const int32_t *local_edges, int64_t m, const int32_t *n_local, int32_t leaves,
                     int32_t part_size, int32_t *part_local, std::string *err, int threads = 0,
                     const std::atomic<int32_t> *ready = nullptr, int32_t *rank_local = nullptr);
// number of CPUs this process may run on (affinity mask)
int host_cpus();


// the CUDA stream a context enqueues on (api.cu)
void *ctx_stream(epg_ctx *ctx);
int ctx_device(epg_ctx *ctx);
int32_t ctx_partition_method(epg_ctx *ctx);
// records a failure on ctx (epg_last_error) and returns s
epg_status ctx_fail(epg_ctx *ctx, epg_status s, const std::string &msg);

}  // namespace epg
