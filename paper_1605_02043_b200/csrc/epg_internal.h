// epg_internal.h -- private declarations of libepg.so (not installed, not part of the ABI).
#pragma once

#include <stdint.h>

#include <string>

#include "../../include/epg.h"

namespace epg {

epg_status host_partition(const int32_t *edges, int64_t m, int32_t n, int32_t part_size, int32_t shards,
                          int32_t *part, std::string *err);

}  // namespace epg
