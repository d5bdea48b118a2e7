// epg_internal.h -- private declarations of libepg.so (not installed, not part of the ABI).
#pragma once

#include <stdint.h>

#include <atomic>
#include <string>

#include "../../include/epg.h"

namespace epg {

// Host EPG-1 / EPG-2 (partition.cpp; method EPG_PARTITION_*). A non-zero *cancel (polled
// once per partition) stops it with EPG_ERR_STATE ("partition: cancelled").
epg_status host_partition(const int32_t *edges, int64_t m, int32_t n, int32_t part_size, int32_t shards,
                          int32_t *part, std::string *err, const std::atomic<int> *cancel = nullptr,
                          int32_t method = EPG_PARTITION_EPG1);

// the CUDA stream a context enqueues on (api.cu)
void *ctx_stream(epg_ctx *ctx);
int ctx_device(epg_ctx *ctx);
int32_t ctx_partition_method(epg_ctx *ctx);
// records a failure on ctx (epg_last_error) and returns s
epg_status ctx_fail(epg_ctx *ctx, epg_status s, const std::string &msg);

}  // namespace epg
