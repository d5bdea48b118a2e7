// api.cu -- the C ABI of libepg.so (include/epg.h): context, plans, and the host-side
// orchestration of the cost, remap and run kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <type_traits>
#include <map>
#include <memory>
#include <queue>
#include <thread>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "epg_internal.h"
#include "layout_kernels.cuh"
#include "run_kernels.cuh"
#include "pipelined_kernel.cuh"
#include "occupancy_kernel.cuh"
#include "place_kernels.cuh"
#include "rb_kernels.cuh"

// epg_run_host's pipeline (ctx-owned): copy-in and copy-out streams beside the ctx stream,
// double-buffered staging so call i+1's H2D and call i's D2H overlap the compute.
struct HostRun {
    cudaStream_t s_in = nullptr, s_out = nullptr;
    size_t bytes = 0;                       // capacity of every buffer below
    void *stage_in[2] = {nullptr, nullptr}, *stage_out[2] = {nullptr, nullptr};
    void *buf[2] = {nullptr, nullptr};      // plan-layout ping-pong state
    cudaEvent_t ev_in[2] = {}, ev_consumed[2] = {}, ev_comp[2] = {}, ev_out[2] = {};
    bool used[2] = {false, false};
    int parity = 0;
};

struct epg_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t cap_stream = nullptr;   // private stream epg_run captures its CUDA graphs on
    HostRun *hr = nullptr;
    struct Comm *comm = nullptr;         // multi-GPU group (epg_comm_init / epg_comm_init_local)
    std::string err;
    float *naive_F = nullptr;
    size_t naive_F_bytes = 0;
    // profiling: event pairs around launches, per kernel class (0 edge, 1 finalise/update)
    bool profiling = false;
    int partition_method = EPG_PARTITION_EPG1;
    int variant = 0;  // 0 auto, 1 one CTA per partition, 2 pipelined TMA, 3 occupancy TMA
    int hub_min = -1; // hub split: shared vertices with >= hub_min halo entries (0 off, -1 default)
    int hub_l2 = 1;   // hub read side: persisting L2 access-policy window over the hubs' state rows
    int exec_rows = -1, exec_edges = -1;   // execution-split caps for later remaps (-1 default)
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_used;
    cudaEvent_t take_event() {
        if (ev_pool.empty()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            return e;
        }
        cudaEvent_t e = ev_pool.back();
        ev_pool.pop_back();
        return e;
    }
    // returns the start event (recorded) or nullptr when not profiling
    cudaEvent_t prof_begin() {
        if (!profiling) return nullptr;
        cudaEvent_t a = take_event();
        cudaEventRecord(a, stream);
        return a;
    }
    void prof_end(int cls, cudaEvent_t a) {
        if (!a) return;
        cudaEvent_t b = take_event();
        cudaEventRecord(b, stream);
        ev_used.push_back({cls, {a, b}});
    }
    epg_status fail(epg_status s, const std::string &msg) {
        err = msg;
        return s;
    }
};

struct epg_plan {
    epg_ctx *ctx = nullptr;
    int device = 0;
    int64_t m = 0, n = 0, k = 0, touched = 0, C = 0, S = 0;
    int Lcap = 0, Scap = 0;
    int32_t *peb = nullptr, *pvb = nullptr, *hb = nullptr, *halo_ids = nullptr, *sidx = nullptr;
    int32_t *shared_ids = nullptr, *hv_off = nullptr, *hv_list = nullptr;
    uint32_t *slots = nullptr;
    uint32_t *slots_occ = nullptr;   // occupancy kernel: placed record positions + Phi position (place_kernels.cuh)
    uint16_t *inc = nullptr, *inc_off = nullptr;
    float *owner_buf = nullptr, *halo_buf = nullptr;
    // pipelined kernel: per-partition descriptors and contiguous blobs
    epg::PartDesc *desc = nullptr;
    unsigned char *blob = nullptr;
    int32_t *hid_blob = nullptr;
    int Hcap = 0;
    int32_t *halo_pos = nullptr;
    int Ocap = 0, blob_max = 0, inc_width = 0;   // inc_width: padded incidence width (0 = CSR)
    std::vector<double> part_cost;                // modelled work per partition (ns)
    // occupancy kernel: descriptors + blobs (halo ids, incidence)
    epg::PartDesc *desc3 = nullptr;
    unsigned char *blob3 = nullptr;
    int blob3_max = 0;
    int4 *fin_recs = nullptr;   // packed finalise records (when every vertex has <= 6 halo entries)
    int4 *fin_rec16 = nullptr;  // ... as 16-byte records {v, count, h0, h1 or overflow index}
    int32_t *fin_over = nullptr;   // ... and the entries h1..h5 of the vertices with > 2
    int32_t *heavy = nullptr;   // shared vertices with more than kBlockHalo halo entries
    int64_t n_heavy = 0;
    int32_t *medium = nullptr;  // shared vertices with (kHeavyHalo, kBlockHalo] halo entries
    int64_t n_medium = 0;
    // hub split (occupancy kernel only): hubs = shared vertices with >= hub_min halo entries
    int32_t hub_min = 0;
    int64_t n_hub = 0;
    int32_t *hub_sid = nullptr;   // [n_hub] shared index of hub i
    float *hub_acc = nullptr;     // [n_hub][5] partial sums, zero between steps
    int64_t hub_rows = 0;         // 1 + largest hub id: hubs are first touched early, so cpack
                                  // gives them a prefix of the vertex order (the L2 window)
    int finalise_skip = 8;        // k_finalise3 leaves vertices with more halo entries
    int hub_words = 1;            // blob3 words per halo row (2 with hub indices)
    // the EP map the plan executes (k, C of the paper's partitions; the plan itself may
    // split oversized partitions into contiguous execution ranges)
    int64_t k_ep = 0, C_ep = 0;
    std::vector<int32_t> part_rows, part_edges;   // |V_p| and s_p of the plan's partitions
    std::vector<int32_t> exec_base;               // [k_ep + 1] first execution partition of each EP partition
    std::vector<int32_t> pvb_h, hb_h;             // host copies of the execution plan's beginA / halo_begin
    std::vector<int32_t> shared_h;                // host copy of shared_ids (lazy, for shard ranges)
    int assign_grid = 0;                          // grid size the assignment was built for
    unsigned long long *bar_ctr = nullptr;        // grid barrier counter (monotone)
    unsigned long long bar_sum = 0;               // CTAs that have arrived at the counter so far
                                                  // (cumulative over launches of any grid size)
    int32_t *cta_begin = nullptr, *cta_list = nullptr;
    std::map<const void *, int64_t> resident_ctas;   // per edge-kernel instance: SMs x occupancy
    // epg_run's CUDA graphs: one per (kernel, buffers, steps, variant)
    std::map<std::vector<uintptr_t>, cudaGraphExec_t> graphs;   // nullptr: key not capturable
    std::vector<void *> allocs;
    ~epg_plan() {
        for (auto &g : graphs)
            if (g.second) cudaGraphExecDestroy(g.second);
        for (void *p : allocs) cudaFree(p);
    }
};

namespace {

using namespace epg;

constexpr int kThreads = 256;
constexpr int kHeavyHalo = 8;      // halo entries above which a shared vertex leaves the thread path
constexpr int kBlockHalo = 1024;   // ... and above which a whole CTA (not a warp) finalises it
constexpr int kHubMinDefault = 7;  // hub split default: >= 7 halo entries (the rest fit k_finalise_rec)
constexpr int64_t kMaxEdges = int64_t(1) << 30;   // device layout: slot keys 2m + 1 fit int32

int hub_min_for(const epg_ctx *ctx) {
    if (ctx->hub_min >= 0) return ctx->hub_min;
    const char *e = std::getenv("EPG_HUB_MIN");
    return e ? std::max(0, std::atoi(e)) : kHubMinDefault;
}

inline unsigned grid_for(int64_t work, int threads = kThreads) {
    return (unsigned)std::max<int64_t>(1, (work + threads - 1) / threads);
}

inline int bits_for(int64_t maxval) {  // bits needed for values in [0, maxval]
    int b = 1;
    while (b < 31 && (int64_t(1) << b) <= maxval) b++;
    return b;
}

#define CU(call)                                                                                        \
    do {                                                                                                \
        cudaError_t _e = (call);                                                                        \
        if (_e != cudaSuccess) return ctx->fail(EPG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#define CHECK_LAUNCH() CU(cudaGetLastError())
#define CU_NOCTX(call)                                                                                  \
    do {                                                                                                \
        if ((call) != cudaSuccess) return EPG_ERR_CUDA;                                                 \
    } while (0)

// stream-ordered temporary device buffer
struct Tmp {
    epg_ctx *ctx;
    void *p = nullptr;
    explicit Tmp(epg_ctx *c) : ctx(c) {}
    ~Tmp() {
        if (p) cudaFreeAsync(p, ctx->stream);
    }
    cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, std::max<size_t>(bytes, 16), ctx->stream); }
    void release() {
        if (p) cudaFreeAsync(p, ctx->stream);
        p = nullptr;
    }
    template <class T> T *as() { return static_cast<T *>(p); }
};

bool is_device_ptr(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

template <class T>
__global__ void k_fill(T *a, int64_t len, T v) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < len) a[i] = v;
}

epg_status plan_alloc(epg_plan *pl, epg_ctx *ctx, void **out, size_t bytes) {
    *out = nullptr;
    cudaError_t e = cudaMalloc(out, std::max<size_t>(bytes, 16));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return ctx->fail(EPG_ERR_NOMEM, std::string("cudaMalloc(plan): ") + cudaGetErrorString(e));
    }
    pl->allocs.push_back(*out);
    return EPG_OK;
}

template <class T>
epg_status plan_alloc_t(epg_plan *pl, epg_ctx *ctx, T **out, int64_t count) {
    void *p;
    epg_status s = plan_alloc(pl, ctx, &p, sizeof(T) * (size_t)std::max<int64_t>(count, 1));
    *out = static_cast<T *>(p);
    return s;
}

// validate endpoints and (optionally) partition ids on the device
epg_status validate(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n, const int32_t *part, int64_t k) {
    Tmp bad(ctx);
    CU(bad.alloc(2 * sizeof(unsigned long long)));
    k_fill<unsigned long long><<<1, 2, 0, ctx->stream>>>(bad.as<unsigned long long>(), 2, ULLONG_MAX);
    k_validate<<<grid_for(m), kThreads, 0, ctx->stream>>>(edges, part, m, n, k, bad.as<unsigned long long>(),
                                                          bad.as<unsigned long long>() + 1);
    CHECK_LAUNCH();
    unsigned long long h[2];
    CU(cudaMemcpyAsync(h, bad.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (h[0] != ULLONG_MAX)
        return ctx->fail(EPG_ERR_INPUT, "edge " + std::to_string(h[0]) + " has an endpoint outside [0, n)");
    if (h[1] != ULLONG_MAX)
        return ctx->fail(EPG_ERR_INPUT, "edge " + std::to_string(h[1]) + " has a partition id outside [0, k)");
    return EPG_OK;
}

// stable sort of task ids by partition -> edge_perm (new -> old), part_edge_begin
// (partition, order key) of task e; order key in [0, 2^31)
__global__ void k_part_key(const int32_t *__restrict__ part, const int32_t *__restrict__ key, int64_t m,
                           unsigned long long *out) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < m) out[e] = ((unsigned long long)(uint32_t)part[e] << 32) | (uint32_t)key[e];
}
__global__ void k_key_part(const unsigned long long *__restrict__ in, int64_t m, int32_t *out) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < m) out[e] = (int32_t)(in[e] >> 32);
}

// stable sort of task ids by partition (then by `key`, if given: reading Z22) -> edge_perm
// (new -> old), part_edge_begin
epg_status group_by_part(epg_ctx *ctx, const int32_t *part, int64_t m, int64_t k, int32_t *edge_perm, int32_t *peb,
                         std::vector<int32_t> *peb_host, const int32_t *key = nullptr) {
    Tmp iota(ctx), keys_out(ctx), temp(ctx), k64(ctx), k64o(ctx);
    CU(iota.alloc(sizeof(int32_t) * m));
    CU(keys_out.alloc(sizeof(int32_t) * m));
    k_iota<<<grid_for(m), kThreads, 0, ctx->stream>>>(iota.as<int32_t>(), m);
    size_t tb = 0;
    const int kb = bits_for(k);
    if (key) {   // (part, key) composite, stable: ties keep the task id order
        CU(k64.alloc(sizeof(unsigned long long) * m));
        CU(k64o.alloc(sizeof(unsigned long long) * m));
        k_part_key<<<grid_for(m), kThreads, 0, ctx->stream>>>(part, key, m, k64.as<unsigned long long>());
        CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, k64.as<unsigned long long>(), k64o.as<unsigned long long>(),
                                           iota.as<int32_t>(), edge_perm, (int)m, 0, 32 + kb, ctx->stream));
        CU(temp.alloc(tb));
        CU(cub::DeviceRadixSort::SortPairs(temp.p, tb, k64.as<unsigned long long>(), k64o.as<unsigned long long>(),
                                           iota.as<int32_t>(), edge_perm, (int)m, 0, 32 + kb, ctx->stream));
        k_key_part<<<grid_for(m), kThreads, 0, ctx->stream>>>(k64o.as<unsigned long long>(), m, keys_out.as<int32_t>());
    } else {
        CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, part, keys_out.as<int32_t>(), iota.as<int32_t>(), edge_perm,
                                           (int)m, 0, kb, ctx->stream));
        CU(temp.alloc(tb));
        CU(cub::DeviceRadixSort::SortPairs(temp.p, tb, part, keys_out.as<int32_t>(), iota.as<int32_t>(), edge_perm,
                                           (int)m, 0, kb, ctx->stream));
    }
    k_part_begin<<<grid_for(k + 1), kThreads, 0, ctx->stream>>>(keys_out.as<int32_t>(), m, k, peb);
    CHECK_LAUNCH();
    peb_host->resize(k + 1);
    CU(cudaMemcpyAsync(peb_host->data(), peb, sizeof(int32_t) * (k + 1), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return EPG_OK;
}

template <int BLOCK, int ITEMS>
size_t distinct_smem() {
    using Sort = cub::BlockRadixSort<int, BLOCK, ITEMS>;
    using Disc = cub::BlockDiscontinuity<int, BLOCK>;
    using Red = cub::BlockReduce<int, BLOCK>;
    union TS {
        typename Sort::TempStorage sort;
        typename Disc::TempStorage disc;
        typename Red::TempStorage red;
    };
    return sizeof(TS);
}

template <int BLOCK, int ITEMS>
size_t remap_smem() {
    using Sort = cub::BlockRadixSort<int, BLOCK, ITEMS, int>;
    using Disc = cub::BlockDiscontinuity<int, BLOCK>;
    using Scan = cub::BlockScan<int, BLOCK>;
    union TS {
        typename Sort::TempStorage sort;
        typename Disc::TempStorage disc;
        typename Scan::TempStorage scan;
    };
    return sizeof(TS);
}

template <int BLOCK, int ITEMS>
epg_status launch_distinct(epg_ctx *ctx, const int32_t *edges, const int32_t *edge_perm, const int32_t *peb,
                           int64_t k, int32_t *per_part, int end_bit) {
    const size_t sm = distinct_smem<BLOCK, ITEMS>();
    CU(cudaFuncSetAttribute(k_distinct<BLOCK, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_distinct<BLOCK, ITEMS><<<(unsigned)k, BLOCK, sm, ctx->stream>>>(edges, edge_perm, peb, per_part, end_bit);
    CHECK_LAUNCH();
    return EPG_OK;
}

// |V_p| for every partition; edges grouped by edge_perm / peb
epg_status distinct_counts(epg_ctx *ctx, const int32_t *edges, const int32_t *part, int64_t m, int32_t n,
                           const int32_t *edge_perm, const int32_t *peb, int64_t k, int64_t smax, int32_t *per_part) {
    const int eb = bits_for(n);
    if (2 * smax <= 512) return launch_distinct<256, 2>(ctx, edges, edge_perm, peb, k, per_part, eb);
    if (2 * smax <= 2048) return launch_distinct<256, 8>(ctx, edges, edge_perm, peb, k, per_part, eb);
    if (2 * smax <= 8192) return launch_distinct<512, 16>(ctx, edges, edge_perm, peb, k, per_part, eb);
    // large partitions: global sort of (partition, vertex) keys
    Tmp keys(ctx), sorted(ctx), temp(ctx);
    CU(keys.alloc(sizeof(unsigned long long) * 2 * m));
    CU(sorted.alloc(sizeof(unsigned long long) * 2 * m));
    k_pv_keys<<<grid_for(2 * m), kThreads, 0, ctx->stream>>>(edges, part, m, keys.as<unsigned long long>());
    size_t tb = 0;
    CU(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.as<unsigned long long>(), sorted.as<unsigned long long>(),
                                      (int)(2 * m), 0, 32 + bits_for(k), ctx->stream));
    CU(temp.alloc(tb));
    CU(cub::DeviceRadixSort::SortKeys(temp.p, tb, keys.as<unsigned long long>(), sorted.as<unsigned long long>(),
                                      (int)(2 * m), 0, 32 + bits_for(k), ctx->stream));
    CU(cudaMemsetAsync(per_part, 0, sizeof(int32_t) * k, ctx->stream));
    k_distinct_global<<<grid_for(2 * m), kThreads, 0, ctx->stream>>>(sorted.as<unsigned long long>(), 2 * m, per_part);
    CHECK_LAUNCH();
    return EPG_OK;
}

epg_status sum_i32(epg_ctx *ctx, const int32_t *a, int64_t len, int64_t *out) {
    Tmp acc(ctx);
    CU(acc.alloc(sizeof(unsigned long long)));
    CU(cudaMemsetAsync(acc.p, 0, sizeof(unsigned long long), ctx->stream));
    k_sum<<<(unsigned)std::min<int64_t>(1184, std::max<int64_t>(1, (len + 255) / 256)), 256, 0, ctx->stream>>>(
        a, len, acc.as<unsigned long long>());
    CHECK_LAUNCH();
    unsigned long long h = 0;
    CU(cudaMemcpyAsync(&h, acc.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    *out = (int64_t)h;
    return EPG_OK;
}

epg_status exclusive_scan(epg_ctx *ctx, const int32_t *in, int32_t *out, int64_t len) {
    Tmp temp(ctx);
    size_t tb = 0;
    CU(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int)len, ctx->stream));
    CU(temp.alloc(tb));
    CU(cub::DeviceScan::ExclusiveSum(temp.p, tb, in, out, (int)len, ctx->stream));
    return EPG_OK;
}

epg_status read_i32(epg_ctx *ctx, const int32_t *dev, int32_t *host) {
    CU(cudaMemcpyAsync(host, dev, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return EPG_OK;
}

// cost function on device edges / part: report + optional per-partition counts
epg_status load_count_dev(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n, const int32_t *part, int64_t k,
                          int32_t *per_part_out, epg_report *rep) {
    if (m >= kMaxEdges)   // endpoint slots 2e + s and the scan / sort sizes are int32
        return ctx->fail(EPG_ERR_INPUT, "load_count: m must be below 2^30");
    epg_status st = validate(ctx, edges, m, n, part, k);
    if (st) return st;
    Tmp perm(ctx), peb(ctx), distinct(ctx), flag(ctx);
    CU(perm.alloc(sizeof(int32_t) * m));
    CU(peb.alloc(sizeof(int32_t) * (k + 1)));
    std::vector<int32_t> peb_h;
    st = group_by_part(ctx, part, m, k, perm.as<int32_t>(), peb.as<int32_t>(), &peb_h);
    if (st) return st;
    int64_t smax = 0, smin = INT64_MAX;
    for (int64_t p = 0; p < k; p++) {
        smax = std::max<int64_t>(smax, peb_h[p + 1] - peb_h[p]);
        smin = std::min<int64_t>(smin, peb_h[p + 1] - peb_h[p]);
    }
    int32_t *pp = per_part_out;
    if (!pp) {
        CU(distinct.alloc(sizeof(int32_t) * k));
        pp = distinct.as<int32_t>();
    }
    st = distinct_counts(ctx, edges, part, m, n, perm.as<int32_t>(), peb.as<int32_t>(), k, smax, pp);
    if (st) return st;
    CU(flag.alloc(sizeof(int32_t) * n));
    CU(cudaMemsetAsync(flag.p, 0, sizeof(int32_t) * n, ctx->stream));
    k_mark_touched<<<grid_for(2 * m), kThreads, 0, ctx->stream>>>(edges, m, flag.as<int32_t>());
    CHECK_LAUNCH();
    int64_t touched = 0, L = 0;
    if ((st = sum_i32(ctx, flag.as<int32_t>(), n, &touched))) return st;
    if ((st = sum_i32(ctx, pp, k, &L))) return st;
    rep->k = k;
    rep->load_count = L;
    rep->touched = touched;
    rep->cut_cost = L - touched;
    rep->max_size = smax;
    rep->min_size = smin;
    return EPG_OK;
}

template <int BLOCK, int ITEMS>
epg_status launch_remap_part(epg_ctx *ctx, const int32_t *edges, const int32_t *edge_perm,
                             const int32_t *vertex_perm, const int32_t *peb, const int32_t *pvb, const int32_t *hb,
                             int32_t *halo_ids, uint16_t *slots, uint16_t *inc, uint16_t *inc_off, int64_t k,
                             int end_bit) {
    const size_t sm = remap_smem<BLOCK, ITEMS>();
    CU(cudaFuncSetAttribute(k_remap_part<BLOCK, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_remap_part<BLOCK, ITEMS><<<(unsigned)k, BLOCK, sm, ctx->stream>>>(edges, edge_perm, vertex_perm, peb, pvb, hb,
                                                                        halo_ids, slots, inc, inc_off, end_bit);
    CHECK_LAUNCH();
    return EPG_OK;
}

template <class Fn>
epg_status run_one_cta_per_partition(epg_ctx *ctx, const epg_plan *pl, epg_state *state, int32_t steps);

// descriptors + contiguous per-partition blobs for the pipelined kernel
epg_status build_pipeline_blob(epg_ctx *ctx, epg_plan *pl) {
    const int64_t k = pl->k, C = pl->C;
    epg_status st;
    if ((st = plan_alloc_t(pl, ctx, &pl->halo_pos, C)) || (st = plan_alloc_t(pl, ctx, &pl->desc, k))) return st;
    if (C > 0) k_halo_pos<<<grid_for(C), kThreads, 0, ctx->stream>>>(pl->hv_list, C, pl->halo_pos);
    Tmp units(ctx), off(ctx), maxdeg(ctx), hunits(ctx), hoff(ctx);
    CU(maxdeg.alloc(sizeof(int32_t)));
    CU(cudaMemsetAsync(maxdeg.p, 0, sizeof(int32_t), ctx->stream));
    k_max_local_degree<<<(unsigned)k, 256, 0, ctx->stream>>>(pl->peb, pl->pvb, pl->hb, pl->inc_off, k,
                                                            maxdeg.as<int32_t>());
    int32_t md = 0;
    if ((st = read_i32(ctx, maxdeg.as<int32_t>(), &md))) return st;
    const int W = md <= 4 ? 4 : (md <= 8 ? 8 : 0);
    pl->inc_width = W;
    CU(units.alloc(sizeof(int32_t) * (k + 1)));
    CU(off.alloc(sizeof(int32_t) * (k + 1)));
    CU(hunits.alloc(sizeof(int32_t) * (k + 1)));
    CU(hoff.alloc(sizeof(int32_t) * (k + 1)));
    k_blob_sizes<<<grid_for(k + 1), kThreads, 0, ctx->stream>>>(pl->peb, pl->pvb, pl->hb, k, W, units.as<int32_t>(),
                                                               hunits.as<int32_t>());
    CHECK_LAUNCH();
    if ((st = exclusive_scan(ctx, units.as<int32_t>(), off.as<int32_t>(), k + 1))) return st;
    if ((st = exclusive_scan(ctx, hunits.as<int32_t>(), hoff.as<int32_t>(), k + 1))) return st;
    int32_t total16 = 0, htotal16 = 0;
    if ((st = read_i32(ctx, off.as<int32_t>() + k, &total16))) return st;
    if ((st = read_i32(ctx, hoff.as<int32_t>() + k, &htotal16))) return st;
    if ((st = plan_alloc_t(pl, ctx, &pl->blob, 16 * (int64_t)total16 + 16))) return st;
    if ((st = plan_alloc_t(pl, ctx, &pl->hid_blob, 4 * (int64_t)htotal16 + 4))) return st;
    k_build_blob<<<(unsigned)k, 256, 0, ctx->stream>>>(pl->peb, pl->pvb, pl->hb, pl->halo_ids, pl->halo_pos,
                                                      pl->slots, pl->inc, pl->inc_off, off.as<int32_t>(),
                                                      hoff.as<int32_t>(), W, pl->blob, pl->hid_blob, pl->desc);
    CHECK_LAUNCH();
    {   // occupancy-kernel blobs; hub split and finalise tiers first (the hubs shape the blob)
        Tmp hub_of_h(ctx);
        int hw = 1;
        if (pl->S > 0) {
            pl->hub_min = hub_min_for(ctx);
            Tmp hm(ctx);
            CU(hm.alloc(2 * sizeof(int32_t)));
            CU(cudaMemsetAsync(hm.p, 0, 2 * sizeof(int32_t), ctx->stream));
            if ((st = plan_alloc_t(pl, ctx, &pl->fin_recs, 2 * pl->S))) return st;
            k_finalise_records<<<grid_for(pl->S), kThreads, 0, ctx->stream>>>(
                pl->shared_ids, pl->hv_off, pl->hv_list, (int32_t)pl->S, pl->hub_min, pl->fin_recs, hm.as<int32_t>());
            int32_t hmax = 0, nhub = 0;
            if ((st = read_i32(ctx, hm.as<int32_t>(), &hmax)) || (st = read_i32(ctx, hm.as<int32_t>() + 1, &nhub)))
                return st;
            if (hmax > 6) pl->fin_recs = nullptr;   // (the allocation is released with the plan)
            const char *r16 = std::getenv("EPG_FIN_REC16");
            if (pl->fin_recs && !(r16 && std::atoi(r16) == 0)) {   // 16-byte records, same order
                Tmp flag(ctx), pos(ctx);
                CU(flag.alloc(sizeof(int32_t) * (pl->S + 1)));
                CU(pos.alloc(sizeof(int32_t) * (pl->S + 1)));
                CU(cudaMemsetAsync(flag.p, 0, sizeof(int32_t) * (pl->S + 1), ctx->stream));
                k_rec16_flags<<<grid_for(pl->S), kThreads, 0, ctx->stream>>>(pl->fin_recs, (int32_t)pl->S,
                                                                            flag.as<int32_t>());
                if ((st = exclusive_scan(ctx, flag.as<int32_t>(), pos.as<int32_t>(), pl->S + 1))) return st;
                int32_t nov = 0;
                if ((st = read_i32(ctx, pos.as<int32_t>() + pl->S, &nov))) return st;
                if ((st = plan_alloc_t(pl, ctx, &pl->fin_rec16, pl->S)) ||
                    (st = plan_alloc_t(pl, ctx, &pl->fin_over, 5 * std::max<int64_t>(nov, 1))))
                    return st;
                k_rec16_build<<<grid_for(pl->S), kThreads, 0, ctx->stream>>>(pl->fin_recs, (int32_t)pl->S,
                                                                            pos.as<int32_t>(), pl->fin_rec16,
                                                                            pl->fin_over);
                CHECK_LAUNCH();
                CU(cudaStreamSynchronize(ctx->stream));
            }
            pl->finalise_skip = nhub > 0 ? std::min(kHeavyHalo, pl->hub_min - 1) : kHeavyHalo;
            if (hmax > kHeavyHalo || nhub > 0) {    // list medium / heavy vertices and hubs on the host
                std::vector<int32_t> off(pl->S + 1), hv, md, hubs, hub_of_s;
                CU(cudaMemcpy(off.data(), pl->hv_off, sizeof(int32_t) * (pl->S + 1), cudaMemcpyDeviceToHost));
                if (nhub > 0) hub_of_s.assign(pl->S, -1);
                for (int64_t t = 0; t < pl->S; t++) {
                    const int c = off[t + 1] - off[t];
                    if (nhub > 0 && c >= pl->hub_min) {
                        hub_of_s[t] = (int32_t)hubs.size();
                        hubs.push_back((int32_t)t);
                    } else if (c > kBlockHalo) hv.push_back((int32_t)t);
                    else if (c > kHeavyHalo) md.push_back((int32_t)t);
                }
                pl->n_heavy = (int64_t)hv.size();
                pl->n_medium = (int64_t)md.size();
                pl->n_hub = (int64_t)hubs.size();
                if ((st = plan_alloc_t(pl, ctx, &pl->heavy, pl->n_heavy)) ||
                    (st = plan_alloc_t(pl, ctx, &pl->medium, pl->n_medium)) ||
                    (st = plan_alloc_t(pl, ctx, &pl->hub_sid, pl->n_hub)) ||
                    (st = plan_alloc_t(pl, ctx, &pl->hub_acc, 5 * pl->n_hub)))
                    return st;
                if (pl->n_heavy)
                    CU(cudaMemcpy(pl->heavy, hv.data(), sizeof(int32_t) * pl->n_heavy, cudaMemcpyHostToDevice));
                if (pl->n_medium)
                    CU(cudaMemcpy(pl->medium, md.data(), sizeof(int32_t) * pl->n_medium, cudaMemcpyHostToDevice));
                if (pl->n_hub) {
                    int32_t last = 0;
                    CU(cudaMemcpy(&last, pl->shared_ids + hubs.back(), sizeof(int32_t), cudaMemcpyDeviceToHost));
                    pl->hub_rows = (int64_t)last + 1;
                    CU(cudaMemcpy(pl->hub_sid, hubs.data(), sizeof(int32_t) * pl->n_hub, cudaMemcpyHostToDevice));
                    CU(cudaMemset(pl->hub_acc, 0, sizeof(float) * 5 * pl->n_hub));
                    Tmp hos(ctx);
                    CU(hos.alloc(sizeof(int32_t) * pl->S));
                    CU(cudaMemcpyAsync(hos.p, hub_of_s.data(), sizeof(int32_t) * pl->S, cudaMemcpyHostToDevice,
                                       ctx->stream));
                    CU(hub_of_h.alloc(sizeof(int32_t) * std::max<int64_t>(1, pl->C)));
                    CU(cudaMemsetAsync(hub_of_h.p, 0xff, sizeof(int32_t) * std::max<int64_t>(1, pl->C), ctx->stream));
                    k_hub_mark<<<grid_for(pl->S), kThreads, 0, ctx->stream>>>(hos.as<int32_t>(), (int32_t)pl->S,
                                                                             pl->hv_off, pl->hv_list,
                                                                             hub_of_h.as<int32_t>());
                    CHECK_LAUNCH();
                    CU(cudaStreamSynchronize(ctx->stream));   // hub_of_s is a host vector
                    hw = 2;
                }
            }
        }
        pl->hub_words = hw;
        Tmp u3(ctx), o3(ctx);
        CU(u3.alloc(sizeof(int32_t) * (k + 1)));
        CU(o3.alloc(sizeof(int32_t) * (k + 1)));
        k_blob3_sizes<<<grid_for(k + 1), kThreads, 0, ctx->stream>>>(pl->peb, pl->pvb, pl->hb, k, W, hw,
                                                                    u3.as<int32_t>());
        if ((st = exclusive_scan(ctx, u3.as<int32_t>(), o3.as<int32_t>(), k + 1))) return st;
        int32_t t3 = 0;
        if ((st = read_i32(ctx, o3.as<int32_t>() + k, &t3))) return st;
        if ((st = plan_alloc_t(pl, ctx, &pl->blob3, 16 * (int64_t)t3 + 16)) ||
            (st = plan_alloc_t(pl, ctx, &pl->desc3, k)))
            return st;
        k_build_blob3<<<(unsigned)k, 256, 0, ctx->stream>>>(pl->peb, pl->pvb, pl->hb, pl->halo_ids, pl->inc,
                                                           pl->inc_off, o3.as<int32_t>(), W,
                                                           hw == 2 ? hub_of_h.as<int32_t>() : nullptr, pl->Scap, pl->blob3,
                                                           pl->desc3);
        CHECK_LAUNCH();
        CU(cudaStreamSynchronize(ctx->stream));
    }
    std::vector<int32_t> peb(k + 1), pvb(k + 1), hb(k + 1);
    CU(cudaMemcpyAsync(peb.data(), pl->peb, sizeof(int32_t) * (k + 1), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(pvb.data(), pl->pvb, sizeof(int32_t) * (k + 1), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(hb.data(), pl->hb, sizeof(int32_t) * (k + 1), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    int ocap = 0, bmax = 0, hcap = 0;
    pl->part_cost.resize(k);
    pl->part_rows.resize(k);
    pl->part_edges.resize(k);
    for (int64_t p = 0; p < k; p++) {
        const int nO = pvb[p + 1] - pvb[p], nH = hb[p + 1] - hb[p], s = peb[p + 1] - peb[p];
        ocap = std::max(ocap, nO);
        hcap = std::max(hcap, nH);
        pl->part_rows[p] = nO + nH;
        pl->part_edges[p] = s;
        bmax = std::max(bmax, blob_bytes_for(nH, s, nO + nH, W));
        pl->blob3_max = std::max(pl->blob3_max, blob3_bytes_for(nH, s, nO + nH, W, pl->hub_words));
        // measured on B200 (cfd, P = 1024): ~1.4 ns per edge, ~1.6 per staged row, ~1 per halo row
        pl->part_cost[p] = 1.4 * s + 1.6 * (nO + nH) + 1.0 * nH;
    }
    pl->Ocap = ocap;
    pl->Hcap = hcap;
    pl->pvb_h = pvb;
    pl->hb_h = hb;
    pl->blob_max = bmax;
    {   // bank-conflict-aware placement of every partition's records (place_kernels.cuh, one
        // warp per partition); EPG_PLACE=0, or variable-length incidence, keeps the identity
        const int64_t m = peb[k], nl = (int64_t)pvb[k] + hb[k];
        if ((st = plan_alloc_t(pl, ctx, &pl->slots_occ, std::max<int64_t>(m, 1)))) return st;
        Tmp dv(ctx), de(ctx);
        CU(dv.alloc(std::max<int64_t>(nl, 1)));
        CU(de.alloc(std::max<int64_t>(m, 1)));
        const char *pe = std::getenv("EPG_PLACE");
        const bool place = !(pe && std::atoi(pe) == 0) && (W == 4 || W == 8);
        if (place) {
            const int sm = place_smem_bytes(pl->Scap, pl->Lcap, W);
            auto kp = W == 4 ? k_place<4> : k_place<8>;
            CU(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
            kp<<<(unsigned)k, 32, sm, ctx->stream>>>(pl->desc3, pl->slots, pl->Scap, pl->Lcap, dv.as<uint8_t>(),
                                                      de.as<uint8_t>());
        } else {
            k_place_identity<<<(unsigned)k, 256, 0, ctx->stream>>>(pl->desc3, dv.as<uint8_t>(), de.as<uint8_t>());
        }
        CHECK_LAUNCH();
        k_apply_place<<<(unsigned)k, 256, 0, ctx->stream>>>(pl->desc3, pl->slots, dv.as<uint8_t>(), de.as<uint8_t>(), W,
                                                            pl->hub_words, pl->Scap, pl->blob3, pl->slots_occ);
        CHECK_LAUNCH();
        CU(cudaStreamSynchronize(ctx->stream));   // the temporaries die here
    }
    return EPG_OK;
}

inline int up16i(int x) { return (x + 15) & ~15; }

// record array of the occupancy kernel: 8-float (cfd) records are two float4 arrays of
// up8(Lcap) entries each (placed positions stay inside their group of 8); the staged rows
// land inside it and are derived in place
template <class Fn>
int occ_recs_bytes(const epg_plan *pl) {
    return Fn::REC == 8 ? 32 * ((pl->Lcap + 7) & ~7) + 64 : up16i(4 * Fn::REC * pl->Lcap + 64);
}
template <class Fn>
int occ_rstride(const epg_plan *pl) { return Fn::REC == 8 ? ((pl->Lcap + 7) & ~7) : 0; }

// shared-memory layout of the pipelined kernel for `nstage` stage buffers
template <class Fn>
size_t pipe_layout(const epg_plan *pl, bool has_payload, int nstage, PipeArgs *a) {
    int off = up16i(pl->blob_max);
    a->off_rows = off;
    off += up16i(16 + 4 * Fn::ROW * pl->Lcap);
    a->off_pay = off;
    if (has_payload) off += up16i(16 + 4 * Fn::PAYW * pl->Scap);
    a->off_vc = off;
    if (Fn::kUsesConst) off += up16i(16 + 4 * pl->Ocap);
    a->stage_bytes = off;
    int w = nstage * off;
    a->off_der = w;
    w += up16i(4 * Fn::REC * pl->Lcap);
    a->off_phi = w;
    w += up16i(4 * Fn::PHIREC * (pl->Scap + 1));
    a->off_hid = w;
    a->hid_slot_bytes = up16i(4 * pl->Hcap + 16);
    w += 3 * a->hid_slot_bytes;
    a->nstage = nstage;
    a->Lcap = pl->Lcap;
    a->Scap = pl->Scap;
    return (size_t)w;
}

constexpr int kPipeThreads = 512;

// Longest-processing-time-first assignment of partitions to G persistent CTAs: partitions
// by decreasing modelled cost, each to the currently least-loaded CTA (ties: lower CTA).
epg_status assign_partitions(epg_ctx *ctx, epg_plan *pl, int G) {
    if (pl->assign_grid == G) return EPG_OK;
    const int64_t k = pl->k;
    std::vector<int32_t> order(k);
    for (int64_t p = 0; p < k; p++) order[p] = (int32_t)p;
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t x, int32_t y) { return pl->part_cost[x] > pl->part_cost[y]; });
    using Load = std::pair<double, int>;
    std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
    for (int b = 0; b < G; b++) heap.push({0.0, b});
    std::vector<std::vector<int32_t>> lists(G);
    for (int32_t p : order) {
        Load l = heap.top();
        heap.pop();
        lists[l.second].push_back(p);
        heap.push({l.first + pl->part_cost[p], l.second});
    }
    std::vector<int32_t> beg(G + 1, 0), flat;
    flat.reserve(k);
    for (int b = 0; b < G; b++) {
        // ascending ids: at any time the CTAs work on neighbouring partitions, whose halo
        // rows (owned by slightly lower partitions) are then likely resident in L2
        std::sort(lists[b].begin(), lists[b].end());
        beg[b + 1] = beg[b] + (int32_t)lists[b].size();
        flat.insert(flat.end(), lists[b].begin(), lists[b].end());
    }
    if (!pl->cta_begin || pl->assign_grid < G) {
        epg_status st;
        if ((st = plan_alloc_t(pl, ctx, &pl->cta_begin, G + 1)) || (st = plan_alloc_t(pl, ctx, &pl->cta_list, k)))
            return st;
    }
    CU(cudaMemcpy(pl->cta_begin, beg.data(), sizeof(int32_t) * (G + 1), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(pl->cta_list, flat.data(), sizeof(int32_t) * k, cudaMemcpyHostToDevice));
    pl->assign_grid = G;
    return EPG_OK;
}

template <class Fn, int W>
epg_status launch_pipelined(epg_ctx *ctx, epg_plan *pl, epg_state *state, int32_t steps, PipeArgs a,
                            size_t smem, int sms) {
    auto kern = k_edge_tma<Fn, kPipeThreads, W>;
    CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kPipeThreads, smem));
    if (occ < 1) return ctx->fail(EPG_ERR_INFEASIBLE, "run: pipelined kernel cannot be resident");
    // every CTA must be resident (the fused finalise follows a grid barrier): grid is at
    // most SMs x occupancy, and the plan's barrier counter is advanced once per launch
    const int64_t grid = std::min<int64_t>(std::max<int64_t>(pl->k, 1), (int64_t)sms * occ);
    epg_status st = assign_partitions(ctx, pl, (int)grid);
    if (st) return st;
    a.cta_begin = pl->cta_begin;
    a.cta_list = pl->cta_list;
    if (!pl->bar_ctr) {
        if ((st = plan_alloc_t(pl, ctx, &pl->bar_ctr, 1))) return st;
        CU(cudaMemset(pl->bar_ctr, 0, sizeof(unsigned long long)));
    }
    a.bar_ctr = pl->bar_ctr;
    float *bufs[2] = {static_cast<float *>(state->state_in), static_cast<float *>(state->state_out)};
    for (int32_t s = 0; s < steps; s++) {
        a.state_in = bufs[s & 1];
        a.state_out = bufs[(s + 1) & 1];
        // the counter is monotone across every launch on this plan, whatever its grid (the
        // grid depends on the functor and on the payload): the target is the running total
        pl->bar_sum += (unsigned long long)grid;
        a.bar_target = pl->bar_sum;
        cudaEvent_t t0 = ctx->prof_begin();
        kern<<<(unsigned)grid, kPipeThreads, smem, ctx->stream>>>(a);
        ctx->prof_end(0, t0);
    }
    return EPG_OK;
}

template <class Fn>
epg_status run_pipelined(epg_ctx *ctx, epg_plan *pl, epg_state *state, int32_t steps, bool *fits) {
    PipeArgs a{};
    const bool has_payload = state->edge_payload != nullptr;
    int dev_max = 0, sms = 0;
    CU(cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    const size_t reserve = 1024;  // static shared memory (barriers, descriptors)
    size_t smem = pipe_layout<Fn>(pl, has_payload, 2, &a);
    if (smem + reserve > (size_t)dev_max) smem = pipe_layout<Fn>(pl, has_payload, 1, &a);
    *fits = smem + reserve <= (size_t)dev_max;
    if (!*fits) return EPG_OK;
    a.desc = pl->desc;
    a.blob = pl->blob;
    a.hid_blob = pl->hid_blob;
    a.payload = static_cast<const float *>(state->edge_payload);
    a.vconst = static_cast<const float *>(state->vertex_const);
    a.halo_buf = pl->halo_buf;
    a.k = pl->k;
    a.shared_ids = pl->shared_ids;
    a.hv_off = pl->hv_off;
    a.S = (int32_t)pl->S;
    a.touched = pl->touched;
    a.n = pl->n;
    switch (pl->inc_width) {
        case 4: return launch_pipelined<Fn, 4>(ctx, pl, state, steps, a, smem, sms);
        case 8: return launch_pipelined<Fn, 8>(ctx, pl, state, steps, a, smem, sms);
        default: return launch_pipelined<Fn, 0>(ctx, pl, state, steps, a, smem, sms);
    }
}

// occupancy kernel limits: execution partitions of <= 1280 edges (EPT 5 x 256 threads) and
// <= 1280 staged rows (VPT 5), 2048 for one-float rows (VPT 8)
constexpr int kOccThreads = 256;
constexpr int kOccMaxEdges = 1280, kOccMaxRows = 1280, kOccMaxRowsScalar = 2048;
constexpr int kOccDefaultEdges = 1024;   // execution-split default (EPT 4 x 256 threads)
template <class Fn> constexpr int occ_max_rows() { return Fn::ROW == 1 ? kOccMaxRowsScalar : kOccMaxRows; }
// execution-split caps of a remap: epg_set_exec_limits, else EPG_EXEC_MAX_EDGES /
// EPG_EXEC_MAX_ROWS, else 1024 edges and 768 rows (768 rows keep a cfd CTA at ~53 KB of
// shared memory -- four CTAs per SM -- and at 3 rows per thread; C2 / C3 steps 1 % faster than
// at 704, 832 rows drop to three CTAs per SM)
int exec_max_edges(const epg_ctx *ctx) {
    if (ctx->exec_edges > 0) return ctx->exec_edges;
    const char *e = std::getenv("EPG_EXEC_MAX_EDGES");
    const int x = e ? std::atoi(e) : kOccDefaultEdges;
    return std::min(kOccMaxEdges, std::max(32, x));
}
int exec_max_rows(const epg_ctx *ctx) {
    if (ctx->exec_rows > 0) return ctx->exec_rows;
    const char *e = std::getenv("EPG_EXEC_MAX_ROWS");
    const int x = e ? std::atoi(e) : 768;
    return std::min(kOccMaxRowsScalar, std::max(64, x));
}

// launch with programmatic stream serialization (the kernel calls griddepcontrol.wait
// before touching what the previous kernel in the stream writes)
template <class K, class... Args>
cudaError_t launch_pdl_w(K kern, unsigned grid, unsigned block, size_t smem, cudaStream_t stream,
                         const cudaAccessPolicyWindow *window, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (window) {   // L2 access-policy window of this launch (the hub read side)
        attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[1].val.accessPolicyWindow = *window;
        cfg.numAttrs = 2;
    }
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <class K, class... Args>
cudaError_t launch_pdl(K kern, unsigned grid, unsigned block, size_t smem, cudaStream_t stream, Args... args) {
    return launch_pdl_w(kern, grid, block, smem, stream, nullptr, args...);
}

// Hub read side ("for the vertices with large degree ... we use
// hardware cache instead", the hub paragraph of P:642-683): the state rows of a plan's hubs
// (a prefix of the cpack order) are marked persisting in L2 for the edge kernel's launch, so
// the many partitions that gather a hub's row hit L2 while the edge records stream through.
// Sets the device's persisting-L2 carve-out once (cudaLimitPersistingL2CacheSize).
bool hub_window(epg_ctx *ctx, const epg_plan *pl, const void *state_in, int row_bytes, cudaAccessPolicyWindow *w) {
    if (!ctx->hub_l2 || pl->n_hub <= 0 || pl->hub_rows <= 0) return false;
    static int max_window = -1, max_persist = -1;
    if (max_window < 0) {
        if (cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device) != cudaSuccess ||
            cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, ctx->device) != cudaSuccess) {
            cudaGetLastError();
            max_window = max_persist = 0;
        }
    }
    if (max_window <= 0 || max_persist <= 0) return false;
    const size_t bytes = std::min<size_t>((size_t)pl->hub_rows * row_bytes, (size_t)max_window);
    size_t limit = 0;
    if (cudaDeviceGetLimit(&limit, cudaLimitPersistingL2CacheSize) == cudaSuccess && limit < (size_t)max_persist)
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)max_persist);
    cudaGetLastError();
    w->base_ptr = const_cast<void *>(state_in);
    w->num_bytes = bytes;
    w->hitRatio = std::min(1.0f, (float)max_persist / (float)std::max<size_t>(bytes, 1));
    w->hitProp = cudaAccessPropertyPersisting;
    w->missProp = cudaAccessPropertyStreaming;
    return true;
}

template <class Fn>
epg_status launch_occ(epg_ctx *ctx, epg_plan *pl, epg_state *state, int32_t steps, OccArgs a, size_t smem,
                      void (*kern)(OccArgs), int block) {
    CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    {   // early PDL trigger only when the whole grid is resident at once (one wave)
        auto it = pl->resident_ctas.find(reinterpret_cast<const void *>(kern));
        if (it == pl->resident_ctas.end()) {
            int occ = 0, sms = 0;
            CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem));
            CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
            it = pl->resident_ctas.emplace(reinterpret_cast<const void *>(kern), (int64_t)occ * sms).first;
        }
        a.early_pdl = pl->k <= it->second ? 1 : 0;
        // multi-wave grids: prefetch one resident wave ahead (EPG_PREFETCH_AHEAD=0 disables)
        const char *e = std::getenv("EPG_PREFETCH_AHEAD");
        const int64_t ahead = e ? std::atoll(e) : it->second;
        a.ahead = a.early_pdl ? 0 : ahead;
        a.count = pl->k;
    }
    float *bufs[2] = {static_cast<float *>(state->state_in), static_cast<float *>(state->state_out)};
    const int64_t fin_work = pl->S + (pl->n - pl->touched);
    const int prewait_pf = a.prewait_pf;
    for (int32_t s = 0; s < steps; s++) {
        a.state_in = bufs[s & 1];
        a.state_out = bufs[(s + 1) & 1];
        a.state_end = a.state_in + (int64_t)Fn::ROW * pl->n;
        // the pre-wait L2 prefetch helps a step whose rows were evicted since they were written;
        // the later steps of a call read rows the previous step has just written
        a.prewait_pf = s == 0 ? prewait_pf : 0;
        cudaAccessPolicyWindow win{};
        const bool use_win = hub_window(ctx, pl, a.state_in, 4 * Fn::ROW, &win);
        cudaEvent_t t0 = ctx->prof_begin();
        CU(launch_pdl_w(kern, (unsigned)pl->k, (unsigned)block, smem, ctx->stream, use_win ? &win : nullptr, a));
        ctx->prof_end(0, t0);
        if (fin_work > 0) {
            cudaEvent_t t1 = ctx->prof_begin();
            if (pl->fin_rec16)
                CU(launch_pdl(k_finalise_rec16<Fn>, grid_for(fin_work), kThreads, 0, ctx->stream,
                              (const int4 *)pl->fin_rec16, (const int32_t *)pl->fin_over,
                              (const float *)pl->halo_buf, (const float *)a.state_in, a.state_out, a.vconst,
                              (int32_t)pl->S, pl->touched, pl->n));
            else if (pl->fin_recs)
                CU(launch_pdl(k_finalise_rec<Fn>, grid_for(fin_work), kThreads, 0, ctx->stream,
                              (const int4 *)pl->fin_recs, (const float *)pl->halo_buf, (const float *)a.state_in,
                              a.state_out, a.vconst, (int32_t)pl->S, pl->touched, pl->n));
            else
                CU(launch_pdl(k_finalise3<Fn>, grid_for(fin_work), kThreads, 0, ctx->stream,
                              (const int32_t *)pl->shared_ids, (const int32_t *)pl->hv_off,
                              (const int32_t *)pl->hv_list, (const float *)pl->halo_buf, (const float *)a.state_in,
                              a.state_out, a.vconst, (int32_t)pl->S, pl->touched, pl->n, (int32_t)pl->finalise_skip));
            if (pl->n_medium > 0)
                CU(launch_pdl(k_finalise_warp<Fn>, (unsigned)((pl->n_medium + 7) / 8), 256u, 0, ctx->stream,
                              (const int32_t *)pl->medium, pl->n_medium, (const int32_t *)pl->shared_ids,
                              (const int32_t *)pl->hv_off, (const int32_t *)pl->hv_list,
                              (const float *)pl->halo_buf, a.state_out, a.vconst));
            if (pl->n_heavy > 0)
                CU(launch_pdl(k_finalise_heavy<Fn, 256>, (unsigned)pl->n_heavy, 256u, 0, ctx->stream,
                              (const int32_t *)pl->heavy, (const int32_t *)pl->shared_ids,
                              (const int32_t *)pl->hv_off, (const int32_t *)pl->hv_list,
                              (const float *)pl->halo_buf, a.state_out, a.vconst));
            if (pl->n_hub > 0)
                CU(launch_pdl(k_finalise_hub<Fn>, grid_for(pl->n_hub), kThreads, 0, ctx->stream,
                              (const int32_t *)pl->hub_sid, pl->n_hub, (const int32_t *)pl->shared_ids, pl->hub_acc,
                              a.state_out, a.vconst));
            ctx->prof_end(1, t1);
        }
    }
    CHECK_LAUNCH();
    return EPG_OK;
}

// CTA size of the occupancy kernel for a plan: 256 threads, or 288 (9 warps, EPT 4 / VPT 3-4:
// up to 1152 edges and 1152 rows) for cfd partitions of 1025..1152 edges -- the partition size
// that makes a one-wave grid a multiple of the SM count (C2: P = 1032, 444 = 3 x 148 CTAs, every
// SM three partitions) without the idle lanes and registers of the EPT 5 / VPT 5 instance
constexpr int kOccThreadsWide = 288;
template <class Fn>
int occ_block(const epg_plan *pl) {
    if (Fn::ROW == 5 && pl->inc_width > 0 && pl->Scap > 4 * kOccThreads && pl->Scap <= 4 * kOccThreadsWide &&
        pl->Lcap <= 4 * kOccThreadsWide)
        return kOccThreadsWide;
    return kOccThreads;
}
// EPT / VPT that occ_dispatch picks for a plan
template <class Fn>
int occ_ept(const epg_plan *pl) {
    if (occ_block<Fn>(pl) == kOccThreadsWide) return 4;
    if (pl->Scap <= 2 * kOccThreads && pl->Lcap <= 2 * kOccThreads) return 2;
    return pl->Scap > 4 * kOccThreads ? 5 : 4;
}
template <class Fn>
int occ_vpt(const epg_plan *pl) {
    const int L = pl->Lcap;
    if (occ_block<Fn>(pl) == kOccThreadsWide) return L > 3 * kOccThreadsWide ? 4 : 3;
    if (pl->Scap <= 2 * kOccThreads && L <= 2 * kOccThreads) return 2;
    if (Fn::ROW == 1 && L > 4 * kOccThreads) return 8;
    if (L > 4 * kOccThreads) return 5;
    return L > 3 * kOccThreads ? 4 : 3;
}

// Phi space of the occupancy kernel: the Phi records (Scap + 1, the last the zero sentinel),
// which before the edge phase hold the bulk-staged slots, payload (PAYW floats per edge, if
// any) and dt; returns its size and sets the staging offsets in *a.
template <class Fn>
int occ_phi_bytes(const epg_plan *pl, OccArgs *a) {
    // every thread reads EPT x BLOCK edge entries and VPT x BLOCK dt entries unpredicated
    const int B = occ_block<Fn>(pl);
    const int se = std::max(pl->Scap, occ_ept<Fn>(pl) * B), sv = std::max(pl->Ocap, occ_vpt<Fn>(pl) * B);
    a->st_slots = 0;
    a->st_pay = up16i(4 * se + 32);
    a->st_vc = a->st_pay + up16i(4 * Fn::PAYW * se + 32);
    const int stage = a->st_vc + (Fn::kUsesConst ? up16i(4 * sv + 32) : 0);
    a->pstride = (pl->Scap + 1 + 3) & ~3;
    return std::max(up16i(Fn::PHIBYTES * a->pstride), stage);
}

// Instance of the occupancy kernel for a plan: EPT edges and VPT staged rows per thread
// (256 or 288 threads, occ_block), W the padded incidence width. `go` is called with the
// chosen instance and its CTA size.
template <class Fn, class Go>
epg_status occ_dispatch(const epg_plan *pl, Go &&go) {
    const int S = pl->Scap, L = pl->Lcap;
    auto by_w = [&](auto ept, auto vpt) -> epg_status {
        constexpr int E = decltype(ept)::value, V = decltype(vpt)::value;
        switch (pl->inc_width) {
            case 4: return go(k_edge_occ<Fn, kOccThreads, E, V, 4>, kOccThreads);
            case 8: return go(k_edge_occ<Fn, kOccThreads, E, V, 8>, kOccThreads);
            default: return go(k_edge_occ<Fn, kOccThreads, E, V, 0>, kOccThreads);
        }
    };
    using I2 = std::integral_constant<int, 2>;
    using I3 = std::integral_constant<int, 3>;
    using I4 = std::integral_constant<int, 4>;
    using I5 = std::integral_constant<int, 5>;
    using I8 = std::integral_constant<int, 8>;
    if constexpr (Fn::ROW == 5) {
        if (occ_block<Fn>(pl) == kOccThreadsWide) {
            if (L > 3 * kOccThreadsWide)
                return pl->inc_width == 4 ? go(k_edge_occ<Fn, kOccThreadsWide, 4, 4, 4>, kOccThreadsWide)
                                          : go(k_edge_occ<Fn, kOccThreadsWide, 4, 4, 8>, kOccThreadsWide);
            return pl->inc_width == 4 ? go(k_edge_occ<Fn, kOccThreadsWide, 4, 3, 4>, kOccThreadsWide)
                                      : go(k_edge_occ<Fn, kOccThreadsWide, 4, 3, 8>, kOccThreadsWide);
        }
    }
    if (S <= 2 * kOccThreads && L <= 2 * kOccThreads) return by_w(I2{}, I2{});   // small partitions
    if constexpr (Fn::ROW == 1) {   // one-float rows: up to 2048 staged rows, 8 per thread
        if (L > 4 * kOccThreads) return S > 4 * kOccThreads ? by_w(I5{}, I8{}) : by_w(I4{}, I8{});
    }
    if (S > 4 * kOccThreads) {      // 1025..1280 edges (grids sized to the SM count)
        if (L > 4 * kOccThreads) return by_w(I5{}, I5{});
        return L > 3 * kOccThreads ? by_w(I5{}, I4{}) : by_w(I5{}, I3{});
    }
    if (L > 4 * kOccThreads) return by_w(I4{}, I5{});
    return L > 3 * kOccThreads ? by_w(I4{}, I4{}) : by_w(I4{}, I3{});
}

template <class Fn>
epg_status run_occ(epg_ctx *ctx, epg_plan *pl, epg_state *state, int32_t steps, bool *fits) {
    *fits = false;
    if (pl->Scap > kOccMaxEdges || pl->Lcap > occ_max_rows<Fn>()) return EPG_OK;
    int dev_max = 0;
    CU(cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    OccArgs a{};
    a.off_recs = up16i(pl->blob3_max);
    const int recs_bytes = occ_recs_bytes<Fn>(pl);
    a.rstride = occ_rstride<Fn>(pl);
    a.prewait_pf = std::getenv("EPG_PREWAIT_PF") ? std::atoi(std::getenv("EPG_PREWAIT_PF")) : 1;
    // landing area of the staged rows inside the record array (derived in place): owned rows
    // then, for 5-float rows, one 32-byte slot per halo row (<= 32 L + 48 bytes in all)
    a.rows_land = Fn::ROW == 5 ? 16 : up16i(recs_bytes - (4 * Fn::ROW * pl->Lcap + 16) - 16);
    a.off_phi = a.off_recs + recs_bytes;
    a.sentinel = pl->Scap;
    const size_t smem = (size_t)a.off_phi + occ_phi_bytes<Fn>(pl, &a);
    if (smem + 1024 > (size_t)dev_max) return EPG_OK;
    *fits = true;
    a.desc = pl->desc3;
    a.blob = pl->blob3;
    a.slots = pl->slots_occ;
    a.payload = static_cast<const float *>(state->edge_payload);
    a.vconst = static_cast<const float *>(state->vertex_const);
    a.halo_buf = pl->halo_buf;
    a.first = 0;
    a.state_end = nullptr;   // set per launch (the buffers alternate)
    a.hw = pl->hub_words;
    a.hub_acc = pl->n_hub > 0 ? pl->hub_acc : nullptr;
    return occ_dispatch<Fn>(pl, [&](auto kern, int block) {
        return launch_occ<Fn>(ctx, pl, state, steps, a, smem, kern, block);
    });
}

// edge kernel over execution partitions [first, first + count) only (no finalise)
template <class Fn>
epg_status run_edges_range(epg_ctx *ctx, epg_plan *pl, epg_state *state, int64_t first, int64_t count,
                           const int32_t *order = nullptr, float *const *peer_acc = nullptr,
                           const int32_t *vlo = nullptr, int rank = 0) {
    if (pl->Scap > kOccMaxEdges || pl->Lcap > occ_max_rows<Fn>())
        return ctx->fail(EPG_ERR_INFEASIBLE, "run_edges: plan exceeds the occupancy kernel limits");
    OccArgs a{};
    a.off_recs = up16i(pl->blob3_max);
    const int recs_bytes = occ_recs_bytes<Fn>(pl);
    a.rstride = occ_rstride<Fn>(pl);
    a.prewait_pf = std::getenv("EPG_PREWAIT_PF") ? std::atoi(std::getenv("EPG_PREWAIT_PF")) : 1;
    // landing area of the staged rows inside the record array (derived in place): owned rows
    // then, for 5-float rows, one 32-byte slot per halo row (<= 32 L + 48 bytes in all)
    a.rows_land = Fn::ROW == 5 ? 16 : up16i(recs_bytes - (4 * Fn::ROW * pl->Lcap + 16) - 16);
    a.off_phi = a.off_recs + recs_bytes;
    a.sentinel = pl->Scap;
    const size_t smem = (size_t)a.off_phi + occ_phi_bytes<Fn>(pl, &a);
    a.desc = pl->desc3;
    a.blob = pl->blob3;
    a.slots = pl->slots_occ;
    a.state_in = static_cast<const float *>(state->state_in);
    a.state_out = static_cast<float *>(state->state_out);
    a.state_end = a.state_in + (int64_t)Fn::ROW * pl->n;
    a.payload = static_cast<const float *>(state->edge_payload);
    a.vconst = static_cast<const float *>(state->vertex_const);
    a.halo_buf = pl->halo_buf;
    a.first = first;
    a.order = order;
    a.peer_acc = peer_acc;
    a.vlo = vlo;
    a.rank = rank;
    a.hw = pl->hub_words;
    a.hub_acc = nullptr;   // shard ranges sum every halo partial through hv_list
    if (count <= 0) return EPG_OK;
    return occ_dispatch<Fn>(pl, [&](auto kern, int block) -> epg_status {
        CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        {   // as launch_occ: multi-wave ranges prefetch the next wave's ranges into L2
            auto it = pl->resident_ctas.find(reinterpret_cast<const void *>(kern));
            if (it == pl->resident_ctas.end()) {
                int occ = 0, sms = 0;
                CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem));
                CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
                it = pl->resident_ctas.emplace(reinterpret_cast<const void *>(kern), (int64_t)occ * sms).first;
            }
            const char *e = std::getenv("EPG_PREFETCH_AHEAD");
            // one-wave ranges trigger their dependents at the start, as launch_occ does: the next
            // PDL launch's prologue (plan data only; it waits before reading state) overlaps this one
            a.early_pdl = count <= it->second ? 1 : 0;
            a.ahead = count > it->second ? (e ? std::atoll(e) : it->second) : 0;
            a.count = count;
        }
        cudaEvent_t t0 = ctx->prof_begin();
        CU(launch_pdl(kern, (unsigned)count, (unsigned)block, smem, ctx->stream, a));
        ctx->prof_end(0, t0);
        return EPG_OK;
    });
}

template <class Fn>
epg_status run_finalise_range(epg_ctx *ctx, epg_plan *pl, epg_state *state, int64_t s_first, int64_t s_count,
                              int64_t h_first, int64_t h_count, float *acc, int32_t untouched) {
    const float *vc = static_cast<const float *>(state->vertex_const);
    float *out = static_cast<float *>(state->state_out);
    if (s_count > 0) {
        cudaEvent_t t1 = ctx->prof_begin();
        CU(launch_pdl(k_finalise_range<Fn>, grid_for(s_count), kThreads, 0, ctx->stream, (const int32_t *)pl->shared_ids,
                      (const int32_t *)pl->hv_off, (const int32_t *)pl->hv_list, (const float *)pl->halo_buf, out, vc,
                      (int32_t)s_first, (int32_t)(s_first + s_count), h_first, h_first + h_count, acc));
        ctx->prof_end(1, t1);
    }
    if (untouched && pl->n > pl->touched)
        k_untouched<Fn><<<grid_for(pl->n - pl->touched), kThreads, 0, ctx->stream>>>(
            static_cast<const float *>(state->state_in), out, pl->touched, pl->n);
    CHECK_LAUNCH();
    return EPG_OK;
}

template <class Fn>
epg_status run_staged(epg_ctx *ctx, epg_plan *pl, epg_state *state, int32_t steps) {
    if (ctx->variant == 0 || ctx->variant == 3) {
        bool fits = false;
        epg_status st = run_occ<Fn>(ctx, pl, state, steps, &fits);
        if (st || fits) return st;
        if (ctx->variant == 3)
            return ctx->fail(EPG_ERR_INFEASIBLE, "run: occupancy kernel limits exceeded (plan Lcap/Scap)");
    }
    if (ctx->variant == 0 || ctx->variant == 2) {
        bool fits = false;
        epg_status st = run_pipelined<Fn>(ctx, pl, state, steps, &fits);
        if (st || fits) return st;
        if (ctx->variant == 2)
            return ctx->fail(EPG_ERR_INFEASIBLE, "run: pipelined kernel does not fit shared memory");
    }
    return run_one_cta_per_partition<Fn>(ctx, pl, state, steps);
}

template <class Fn>
epg_status run_one_cta_per_partition(epg_ctx *ctx, const epg_plan *pl, epg_state *state, int32_t steps) {
    const size_t smem = sizeof(float) * ((size_t)Fn::NV * pl->Lcap + (size_t)Fn::NPHI * pl->Scap);
    int dev_max = 0;
    CU(cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    if (smem > (size_t)dev_max)
        return ctx->fail(EPG_ERR_INFEASIBLE, "run: a partition stages " + std::to_string(pl->Lcap) +
                                                 " rows; shared memory needed " + std::to_string(smem) +
                                                 " B exceeds " + std::to_string(dev_max) + " B");
    CU(cudaFuncSetAttribute(k_edge_staged<Fn, kThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    RunArgs a;
    a.peb = pl->peb; a.pvb = pl->pvb; a.hb = pl->hb; a.halo_ids = pl->halo_ids; a.slots = pl->slots;
    a.inc = pl->inc; a.inc_off = pl->inc_off; a.sidx = pl->sidx;
    a.payload = static_cast<const float *>(state->edge_payload);
    a.vconst = static_cast<const float *>(state->vertex_const);
    a.owner_buf = pl->owner_buf; a.halo_buf = pl->halo_buf;
    a.Lcap = pl->Lcap; a.Scap = pl->Scap;
    float *bufs[2] = {static_cast<float *>(state->state_in), static_cast<float *>(state->state_out)};
    const int64_t fin_work = pl->S + (pl->n - pl->touched);
    for (int32_t s = 0; s < steps; s++) {
        a.state_in = bufs[s & 1];
        a.state_out = bufs[(s + 1) & 1];
        cudaEvent_t t0 = ctx->prof_begin();
        k_edge_staged<Fn, kThreads><<<(unsigned)pl->k, kThreads, smem, ctx->stream>>>(a);
        ctx->prof_end(0, t0);
        if (fin_work > 0) {
            cudaEvent_t t1 = ctx->prof_begin();
            k_finalise<Fn><<<grid_for(fin_work), kThreads, 0, ctx->stream>>>(
                pl->shared_ids, pl->hv_off, pl->hv_list, pl->owner_buf, pl->halo_buf, a.state_in, a.state_out,
                a.vconst, (int32_t)pl->S, pl->touched, pl->n);
            ctx->prof_end(1, t1);
        }
    }
    CHECK_LAUNCH();
    return EPG_OK;
}

template <class Fn>
epg_status run_naive(epg_ctx *ctx, const int32_t *edges, int64_t m, int64_t n, epg_state *state, int32_t steps) {
    const size_t need = sizeof(float) * Fn::ROW * (size_t)n;
    if (ctx->naive_F_bytes < need) {
        if (ctx->naive_F) cudaFree(ctx->naive_F);
        ctx->naive_F = nullptr;
        ctx->naive_F_bytes = 0;
        cudaError_t e = cudaMalloc(&ctx->naive_F, need);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return ctx->fail(EPG_ERR_NOMEM, std::string("cudaMalloc(naive workspace): ") + cudaGetErrorString(e));
        }
        ctx->naive_F_bytes = need;
        CU(cudaMemsetAsync(ctx->naive_F, 0, need, ctx->stream));
    }
    float *bufs[2] = {static_cast<float *>(state->state_in), static_cast<float *>(state->state_out)};
    const float *payload = static_cast<const float *>(state->edge_payload);
    const float *vc = static_cast<const float *>(state->vertex_const);
    for (int32_t s = 0; s < steps; s++) {
        cudaEvent_t t0 = ctx->prof_begin();
        k_naive_edges<Fn><<<grid_for(m), kThreads, 0, ctx->stream>>>(edges, m, bufs[s & 1], payload, ctx->naive_F);
        ctx->prof_end(0, t0);
        cudaEvent_t t1 = ctx->prof_begin();
        k_naive_update<Fn><<<grid_for(n), kThreads, 0, ctx->stream>>>(n, bufs[s & 1], bufs[(s + 1) & 1], vc,
                                                                        ctx->naive_F);
        ctx->prof_end(1, t1);
    }
    CHECK_LAUNCH();
    return EPG_OK;
}

epg_status check_state(epg_ctx *ctx, epg_kernel kernel, const epg_state *state) {
    if (!state || !state->state_in || !state->state_out)
        return ctx->fail(EPG_ERR_INPUT, "run: state_in and state_out are required");
    if (state->state_in == state->state_out) return ctx->fail(EPG_ERR_INPUT, "run: state_in and state_out alias");
    if (kernel == EPG_KERNEL_CFD_FLUX && (!state->edge_payload || !state->vertex_const))
        return ctx->fail(EPG_ERR_INPUT, "run: CFD_FLUX needs edge_payload (normals) and vertex_const (dt)");
    if (kernel == EPG_KERNEL_SPMV && !state->edge_payload)
        return ctx->fail(EPG_ERR_INPUT, "run: SPMV needs edge_payload (matrix values)");
    if (kernel < EPG_KERNEL_CFD_FLUX || kernel > EPG_KERNEL_SPMV)
        return ctx->fail(EPG_ERR_INPUT, "run: unknown kernel id");
    return EPG_OK;
}

// epg_run through a cached CUDA graph: the launches of one call (edge kernel + finalise per
// step, with their programmatic-dependent-launch edges) are captured once on a private stream
// and replayed into ctx's stream, which saves their per-launch overhead (C2: 21.5 -> 20.5 us per
// step in a scratch A/B). Only for the occupancy path (whose launches are capturable: no host
// synchronisation); not while profiling (the per-launch events would be baked in). Only for
// calls of two steps or more by default: a graph launch ends the PDL overlap at its boundary,
// and back-to-back one-step calls (a time loop driven by the caller, or the bench's
// round-robin over replicas) are faster launched directly (C2: 19.1 -> 12.7 us per step).
// EPG_GRAPHS=0 disables graphs, EPG_GRAPHS=2 captures one-step calls as well.
template <class Fn>
bool occ_applies(epg_ctx *ctx, const epg_plan *pl) {
    if (!(ctx->variant == 0 || ctx->variant == 3)) return false;
    if (pl->Scap > kOccMaxEdges || pl->Lcap > occ_max_rows<Fn>()) return false;
    int dev_max = 0;
    if (cudaDeviceGetAttribute(&dev_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device)) return false;
    OccArgs a{};
    const int off_phi = up16i(pl->blob3_max) + occ_recs_bytes<Fn>(pl);
    return (size_t)off_phi + occ_phi_bytes<Fn>(pl, &a) + 1024 <= (size_t)dev_max;
}

template <class Fn>
epg_status run_graphed(epg_ctx *ctx, epg_plan *pl, epg_kernel kernel, epg_state *state, int32_t steps) {
    const char *ge = std::getenv("EPG_GRAPHS");
    const int gmode = ge ? std::atoi(ge) : 1;
    if (steps == 0 || ctx->profiling || gmode == 0 || (steps == 1 && gmode != 2) || !occ_applies<Fn>(ctx, pl))
        return run_staged<Fn>(ctx, pl, state, steps);
    const std::vector<uintptr_t> key = {(uintptr_t)kernel, (uintptr_t)state->state_in, (uintptr_t)state->state_out,
                                        (uintptr_t)state->edge_payload, (uintptr_t)state->vertex_const,
                                        (uintptr_t)steps, (uintptr_t)ctx->variant};
    auto it = pl->graphs.find(key);
    if (it == pl->graphs.end()) {
        if (pl->graphs.size() >= 16) {   // bounded cache
            for (auto &g : pl->graphs)
                if (g.second) cudaGraphExecDestroy(g.second);
            pl->graphs.clear();
        }
        if (!ctx->cap_stream) CU(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
        // the capture starts after everything already on ctx's stream is ordered before it
        cudaStream_t user = ctx->stream;
        ctx->stream = ctx->cap_stream;
        cudaGraph_t g = nullptr;
        epg_status st = EPG_OK;
        cudaError_t e = cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal);
        if (e == cudaSuccess) {
            st = run_staged<Fn>(ctx, pl, state, steps);
            e = cudaStreamEndCapture(ctx->cap_stream, &g);
        }
        ctx->stream = user;
        cudaGraphExec_t ex = nullptr;
        if (e == cudaSuccess && st == EPG_OK && g) e = cudaGraphInstantiate(&ex, g, 0);
        if (g) cudaGraphDestroy(g);
        if (e != cudaSuccess || st != EPG_OK || !ex) {   // not capturable here: launch directly
            cudaGetLastError();
            if (ex) cudaGraphExecDestroy(ex);
            pl->graphs.emplace(key, nullptr);              // and do not try to capture this key again
            return run_staged<Fn>(ctx, pl, state, steps);
        }
        it = pl->graphs.emplace(key, ex).first;
    }
    if (!it->second) return run_staged<Fn>(ctx, pl, state, steps);
    CU(cudaGraphLaunch(it->second, ctx->stream));
    return EPG_OK;
}

// ---- EPG-RB (O5'', reading Z21): GPU bisection levels ------------------------------------
int rb_depth(int64_t k, int32_t shards, int32_t leaf_parts) {
    int d = 0;
    while ((1 << d) < shards) d++;
    while (d < 10 && (int64_t)leaf_parts * ((int64_t)1 << (d + 1)) <= k) d++;
    return d;
}

// One BFS pass over every node of a level at once (rb_kernels.cuh): levels are launched in
// chunks of kRbChunk with device-side frontier counts, one host round trip per chunk.
// front/next: [m] each; cnt: [kRbChunk + 1] device counters.
constexpr int kRbChunk = 32;
epg_status rb_bfs(epg_ctx *ctx, const int32_t *edges, const int32_t *ip, const int32_t *inc, int32_t hub,
                  const int32_t *node, int32_t nodes, int32_t *dist, unsigned long long *vis, bool bits,
                  unsigned long long pass, int32_t *front, int32_t *next, int32_t *cnt, int64_t nfront, int64_t m,
                  int grid) {
    int32_t level = 0;
    while (nfront > 0) {
        if ((uint32_t)level + kRbChunk + 2 >= kRbDistCap)
            return ctx->fail(EPG_ERR_INFEASIBLE, "partition (RB): BFS depth exceeds 2^22");
        const int32_t nf32 = (int32_t)nfront;
        CU(cudaMemsetAsync(cnt + 1, 0, sizeof(int32_t) * kRbChunk, ctx->stream));
        CU(cudaMemcpyAsync(cnt, &nf32, sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
        for (int c = 0; c < kRbChunk; c++) {
            k_rb_expand<<<grid, kThreads, 0, ctx->stream>>>(edges, ip, inc, hub, node, nodes, dist, vis, bits, pass,
                                                            front, cnt + c, next, cnt + c + 1, level + c);
            std::swap(front, next);
        }
        CHECK_LAUNCH();
        int32_t h = 0;
        CU(cudaMemcpyAsync(&h, cnt + kRbChunk, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));   // (also keeps nf32 alive for its copy)
        if (h < 0 || h > m) return ctx->fail(EPG_ERR_STATE, "partition (RB): frontier overflow");
        nfront = h;
        level += kRbChunk;
    }
    return EPG_OK;
}

double rb_now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

// Leaf of every task after the bisection levels (leaf_d [m], DEVICE); *depth_out = d.
epg_status rb_bisect(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n, int32_t P, int32_t shards,
                     int32_t leaf_parts, int32_t *leaf_d, int *depth_out) {
    const int64_t k = (m + P - 1) / P;
    const int d = rb_depth(k, shards, leaf_parts);
    *depth_out = d;
    if (d == 0) {
        CU(cudaMemsetAsync(leaf_d, 0, sizeof(int32_t) * m, ctx->stream));
        return EPG_OK;
    }
    std::vector<int64_t> S(k + 1, 0);
    for (int64_t i = 0; i < k; i++) S[i + 1] = S[i] + m / k + (i < m % k ? 1 : 0);
    const int32_t hub = 4 * P;
    // incidence: vertex -> tasks, ascending (stable sort of the task-ordered endpoint slots)
    Tmp key(ctx), val(ctx), skey(ctx), inc(ctx), ip(ctx), temp(ctx);
    CU(key.alloc(sizeof(int32_t) * 2 * m));
    CU(val.alloc(sizeof(int32_t) * 2 * m));
    CU(skey.alloc(sizeof(int32_t) * 2 * m));
    CU(inc.alloc(sizeof(int32_t) * 2 * m));
    CU(ip.alloc(sizeof(int32_t) * ((int64_t)n + 1)));
    k_rb_slot_keys<<<grid_for(2 * m), kThreads, 0, ctx->stream>>>(edges, m, n, key.as<int32_t>(), val.as<int32_t>());
    CHECK_LAUNCH();
    {
        size_t tb = 0;
        CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.as<int32_t>(), skey.as<int32_t>(), val.as<int32_t>(),
                                           inc.as<int32_t>(), (int)(2 * m), 0, bits_for(n), ctx->stream));
        CU(temp.alloc(tb));
        CU(cub::DeviceRadixSort::SortPairs(temp.p, tb, key.as<int32_t>(), skey.as<int32_t>(), val.as<int32_t>(),
                                           inc.as<int32_t>(), (int)(2 * m), 0, bits_for(n), ctx->stream));
    }
    k_rb_offsets<<<grid_for((int64_t)n + 1), kThreads, 0, ctx->stream>>>(skey.as<int32_t>(), 2 * m, n, ip.as<int32_t>());
    CHECK_LAUNCH();
    // per-task state; the slot buffers are reused for the level sorts
    Tmp node(ctx), nnode(ctx), dist(ctx), front(ctx), next(ctx), vis(ctx), cnt(ctx), nmin(ctx), far(ctx), nb(ctx),
        n0(ctx), stemp(ctx);
    CU(node.alloc(sizeof(int32_t) * m));
    CU(nnode.alloc(sizeof(int32_t) * m));
    CU(dist.alloc(sizeof(int32_t) * m));
    CU(front.alloc(sizeof(int32_t) * m));
    CU(next.alloc(sizeof(int32_t) * m));
    // per-(vertex, node) expansion bitmap of the deepest level, if it fits 16 GiB
    const uint64_t vis_words_max = ((uint64_t)n * (uint64_t)(1 << (d - 1)) + 63) / 64;
    const bool bits = vis_words_max * 8 <= (16ull << 30);
    CU(vis.alloc(sizeof(unsigned long long) * (bits ? vis_words_max : (uint64_t)n)));
    CU(cnt.alloc(sizeof(int32_t) * (kRbChunk + 1)));
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    const int grid = sms * 8;
    CU(nmin.alloc(sizeof(int32_t) << d));
    CU(far.alloc(sizeof(unsigned long long) << d));
    CU(nb.alloc(sizeof(int64_t) << d));
    CU(n0.alloc(sizeof(int64_t) << d));
    CU(cudaMemsetAsync(node.p, 0, sizeof(int32_t) * m, ctx->stream));
    if (!bits) CU(cudaMemsetAsync(vis.p, 0, sizeof(unsigned long long) * n, ctx->stream));
    Tmp vals2(ctx);
    CU(vals2.alloc(sizeof(int32_t) * m));
    uint32_t *skeys = reinterpret_cast<uint32_t *>(key.p), *skeys2 = reinterpret_cast<uint32_t *>(skey.p);
    int32_t *svals = val.as<int32_t>(), *svals2 = vals2.as<int32_t>();
    size_t stb = 0;
    CU(cub::DeviceRadixSort::SortPairs(nullptr, stb, skeys, skeys2, svals, svals2, (int)m, 0, 32, ctx->stream));
    CU(stemp.alloc(stb));
    unsigned long long pass = 0;
    epg_status st;
    for (int l = 0; l < d; l++) {
        const int32_t nodes = 1 << l;
        std::vector<int64_t> begin_h(nodes), n0_h(nodes);
        for (int64_t a = 0; a < nodes; a++) {
            const int64_t lo = a * k / nodes, mid = (2 * a + 1) * k / (2 * nodes);
            begin_h[a] = S[lo];
            n0_h[a] = S[mid] - S[lo];
        }
        // pass 1: from each node's smallest task id
        k_rb_init_dist<<<grid_for(m), kThreads, 0, ctx->stream>>>(dist.as<int32_t>(), m);
        k_fill<int32_t><<<grid_for(nodes), kThreads, 0, ctx->stream>>>(nmin.as<int32_t>(), nodes, INT32_MAX);
        k_rb_node_min<<<grid, kThreads, sizeof(int32_t) * nodes, ctx->stream>>>(node.as<int32_t>(), m, nodes,
                                                                                 nmin.as<int32_t>());
        k_rb_sources<<<grid_for(nodes), kThreads, 0, ctx->stream>>>(nmin.as<int32_t>(), far.as<unsigned long long>(),
                                                                    nodes, 0, dist.as<int32_t>(), front.as<int32_t>());
        CHECK_LAUNCH();
        if (bits)
            CU(cudaMemsetAsync(vis.p, 0, sizeof(unsigned long long) * (((uint64_t)n * nodes + 63) / 64), ctx->stream));
        if ((st = rb_bfs(ctx, edges, ip.as<int32_t>(), inc.as<int32_t>(), hub, node.as<int32_t>(), nodes,
                         dist.as<int32_t>(), vis.as<unsigned long long>(), bits, ++pass, front.as<int32_t>(),
                         next.as<int32_t>(), cnt.as<int32_t>(), nodes, m, grid)))
            return st;
        // pass 2: from each node's farthest reached task (ties: smallest id)
        CU(cudaMemsetAsync(far.p, 0, sizeof(unsigned long long) * nodes, ctx->stream));
        k_rb_far_key<<<grid, kThreads, sizeof(unsigned long long) * nodes, ctx->stream>>>(
            node.as<int32_t>(), dist.as<int32_t>(), m, nodes, far.as<unsigned long long>());
        k_rb_init_dist<<<grid_for(m), kThreads, 0, ctx->stream>>>(dist.as<int32_t>(), m);
        k_rb_sources<<<grid_for(nodes), kThreads, 0, ctx->stream>>>(nmin.as<int32_t>(), far.as<unsigned long long>(),
                                                                    nodes, 1, dist.as<int32_t>(), front.as<int32_t>());
        CHECK_LAUNCH();
        if (bits)
            CU(cudaMemsetAsync(vis.p, 0, sizeof(unsigned long long) * (((uint64_t)n * nodes + 63) / 64), ctx->stream));
        if ((st = rb_bfs(ctx, edges, ip.as<int32_t>(), inc.as<int32_t>(), hub, node.as<int32_t>(), nodes,
                         dist.as<int32_t>(), vis.as<unsigned long long>(), bits, ++pass, front.as<int32_t>(),
                         next.as<int32_t>(), cnt.as<int32_t>(), nodes, m, grid)))
            return st;
        // order (node, dist, id) and cut every node after its first half's task count
        k_rb_sort_keys<<<grid_for(m), kThreads, 0, ctx->stream>>>(node.as<int32_t>(), dist.as<int32_t>(), m, skeys,
                                                                  svals);
        CHECK_LAUNCH();
        CU(cub::DeviceRadixSort::SortPairs(stemp.p, stb, skeys, skeys2, svals, svals2, (int)m, 0,
                                           kRbDistBits + bits_for(nodes), ctx->stream));
        CU(cudaMemcpyAsync(nb.p, begin_h.data(), sizeof(int64_t) * nodes, cudaMemcpyHostToDevice, ctx->stream));
        CU(cudaMemcpyAsync(n0.p, n0_h.data(), sizeof(int64_t) * nodes, cudaMemcpyHostToDevice, ctx->stream));
        k_rb_split<<<grid_for(m), kThreads, 0, ctx->stream>>>(skeys2, svals2, m, nb.as<int64_t>(), n0.as<int64_t>(),
                                                              nnode.as<int32_t>());
        CHECK_LAUNCH();
        CU(cudaStreamSynchronize(ctx->stream));   // begin_h / n0_h are host vectors
        std::swap(node.p, nnode.p);
    }
    CU(cudaMemcpyAsync(leaf_d, node.p, sizeof(int32_t) * m, cudaMemcpyDeviceToDevice, ctx->stream));
    return EPG_OK;
}

// EPG-RB end to end on the device edges: bisection levels (GPU), leaf grouping and leaf-local
// vertex ids (GPU), EPG-2 per leaf (host threads), scatter of the map (GPU) into part_d.
epg_status rb_partition(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n, int32_t P, int32_t shards,
                        int32_t leaf_parts, int32_t *part_d, int32_t *rank_d, std::string *err) {
    const bool trace = std::getenv("EPG_RB_TRACE") != nullptr;
    double t0 = rb_now();
    auto mark = [&](const char *what) {
        if (!trace) return;
        cudaStreamSynchronize(ctx->stream);
        const double t = rb_now();
        std::fprintf(stderr, "[epg rb] %-28s %8.3f s\n", what, t - t0);
        t0 = t;
    };
    const int64_t k = (m + P - 1) / P;
    Tmp leaf(ctx);
    CU(leaf.alloc(sizeof(int32_t) * m));
    int d = 0;
    epg_status st = rb_bisect(ctx, edges, m, n, P, shards, leaf_parts, leaf.as<int32_t>(), &d);
    if (st) return st;
    mark("bisection levels (GPU)");
    const int32_t leaves = 1 << d;
    std::vector<int64_t> S(k + 1, 0), slot_begin(leaves + 1);
    for (int64_t i = 0; i < k; i++) S[i + 1] = S[i] + m / k + (i < m % k ? 1 : 0);
    for (int64_t j = 0; j <= leaves; j++) slot_begin[j] = 2 * S[j * k / leaves];
    Tmp key(ctx), skey(ctx), val(ctx), sval(ctx), flag(ctx), incl(ctx), local(ctx), sb(ctx), nloc(ctx), temp(ctx),
        order(ctx), iota(ctx), lkey(ctx), grouped(ctx), pl(ctx);
    const int64_t len = 2 * m;
    CU(key.alloc(sizeof(unsigned long long) * len));
    CU(skey.alloc(sizeof(unsigned long long) * len));
    CU(val.alloc(sizeof(int32_t) * len));
    CU(sval.alloc(sizeof(int32_t) * len));
    CU(sb.alloc(sizeof(int64_t) * (leaves + 1)));
    CU(nloc.alloc(sizeof(int32_t) * leaves));
    CU(cudaMemcpyAsync(sb.p, slot_begin.data(), sizeof(int64_t) * (leaves + 1), cudaMemcpyHostToDevice, ctx->stream));
    k_rb_leaf_slot_keys<<<grid_for(len), kThreads, 0, ctx->stream>>>(edges, m, leaf.as<int32_t>(),
                                                                     key.as<unsigned long long>(), val.as<int32_t>());
    CHECK_LAUNCH();
    {
        size_t tb = 0;
        const int eb = 32 + bits_for(leaves);
        CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.as<unsigned long long>(), skey.as<unsigned long long>(),
                                           val.as<int32_t>(), sval.as<int32_t>(), (int)len, 0, eb, ctx->stream));
        CU(temp.alloc(tb));
        CU(cub::DeviceRadixSort::SortPairs(temp.p, tb, key.as<unsigned long long>(), skey.as<unsigned long long>(),
                                           val.as<int32_t>(), sval.as<int32_t>(), (int)len, 0, eb, ctx->stream));
    }
    key.release();
    CU(flag.alloc(sizeof(int32_t) * len));
    CU(incl.alloc(sizeof(int32_t) * len));
    k_rb_heads<<<grid_for(len), kThreads, 0, ctx->stream>>>(skey.as<unsigned long long>(), len, flag.as<int32_t>());
    CHECK_LAUNCH();
    {
        Tmp t2(ctx);
        size_t tb = 0;
        CU(cub::DeviceScan::InclusiveSum(nullptr, tb, flag.as<int32_t>(), incl.as<int32_t>(), (int)len, ctx->stream));
        CU(t2.alloc(tb));
        CU(cub::DeviceScan::InclusiveSum(t2.p, tb, flag.as<int32_t>(), incl.as<int32_t>(), (int)len, ctx->stream));
    }
    CU(local.alloc(sizeof(int32_t) * len));
    k_rb_local_ids<<<grid_for(len), kThreads, 0, ctx->stream>>>(skey.as<unsigned long long>(), sval.as<int32_t>(),
                                                                incl.as<int32_t>(), len, sb.as<int64_t>(),
                                                                local.as<int32_t>());
    k_rb_nlocal<<<grid_for(leaves), kThreads, 0, ctx->stream>>>(incl.as<int32_t>(), sb.as<int64_t>(), leaves,
                                                                nloc.as<int32_t>());
    CHECK_LAUNCH();
    // tasks grouped by leaf, ascending inside (stable sort of the task-ordered leaf ids)
    CU(order.alloc(sizeof(int32_t) * m));
    CU(iota.alloc(sizeof(int32_t) * m));
    CU(lkey.alloc(sizeof(int32_t) * m));
    k_iota<<<grid_for(m), kThreads, 0, ctx->stream>>>(iota.as<int32_t>(), m);
    {
        Tmp t2(ctx);
        size_t tb = 0;
        CU(cub::DeviceRadixSort::SortPairs(nullptr, tb, leaf.as<int32_t>(), lkey.as<int32_t>(), iota.as<int32_t>(),
                                           order.as<int32_t>(), (int)m, 0, std::max(1, d), ctx->stream));
        CU(t2.alloc(tb));
        CU(cub::DeviceRadixSort::SortPairs(t2.p, tb, leaf.as<int32_t>(), lkey.as<int32_t>(), iota.as<int32_t>(),
                                           order.as<int32_t>(), (int)m, 0, std::max(1, d), ctx->stream));
    }
    CU(grouped.alloc(sizeof(int32_t) * len));
    k_rb_group_edges<<<grid_for(m), kThreads, 0, ctx->stream>>>(order.as<int32_t>(), m, local.as<int32_t>(),
                                                                grouped.as<int32_t>());
    CHECK_LAUNCH();
    std::vector<int32_t> nl(leaves);
    CU(cudaMemcpyAsync(nl.data(), nloc.p, sizeof(int32_t) * leaves, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    mark("leaf grouping + local ids");
    // the grouped edges stream to the host in leaf order (a copy thread, chunk by chunk)
    // while the leaf workers start on the chunks that have arrived
    std::unique_ptr<int32_t[]> ge(new int32_t[len]), part_local(new int32_t[m]),
        rank_local(rank_d ? new int32_t[m] : nullptr);
    std::atomic<int32_t> ready{0};
    cudaError_t copy_err = cudaSuccess;
    std::thread copier([&]() {
        cudaSetDevice(ctx->device);
        const int chunks = std::min<int32_t>(leaves, 16);
        for (int c = 0; c < chunks; c++) {
            const int32_t j0 = (int32_t)((int64_t)c * leaves / chunks), j1 = (int32_t)((int64_t)(c + 1) * leaves / chunks);
            const int64_t a = slot_begin[j0], b = slot_begin[j1];
            if (b > a && copy_err == cudaSuccess)
                copy_err = cudaMemcpy(ge.get() + a, grouped.as<int32_t>() + a, sizeof(int32_t) * (b - a),
                                      cudaMemcpyDeviceToHost);
            ready.store(copy_err == cudaSuccess ? j1 : leaves, std::memory_order_release);
        }
    });
    st = epg::rb_leaves(ge.get(), m, nl.data(), leaves, P, part_local.get(), err, 0, &ready, rank_local.get());
    copier.join();
    if (copy_err != cudaSuccess) return ctx->fail(EPG_ERR_CUDA, std::string("partition (RB): ") +
                                                                cudaGetErrorString(copy_err));
    if (st) return st;
    mark("copy-out + EPG-2 leaves (host)");
    CU(pl.alloc(sizeof(int32_t) * m));
    CU(cudaMemcpyAsync(pl.p, part_local.get(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, ctx->stream));
    k_rb_scatter<<<grid_for(m), kThreads, 0, ctx->stream>>>(order.as<int32_t>(), pl.as<int32_t>(), m, part_d);
    CHECK_LAUNCH();
    if (rank_d) {   // growth ranks, same grouped order
        CU(cudaStreamSynchronize(ctx->stream));
        CU(cudaMemcpyAsync(pl.p, rank_local.get(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, ctx->stream));
        k_rb_scatter<<<grid_for(m), kThreads, 0, ctx->stream>>>(order.as<int32_t>(), pl.as<int32_t>(), m, rank_d);
        CHECK_LAUNCH();
    }
    CU(cudaStreamSynchronize(ctx->stream));   // part_local is a host vector
    mark("scatter");
    return EPG_OK;
}

}  // namespace

void comm_release(epg_ctx *ctx);

// =====================================================================================
extern "C" {

epg_status epg_create(int device, void *cuda_stream, epg_ctx **out) {
    if (!out) return EPG_ERR_INPUT;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
        cudaGetLastError();
        return EPG_ERR_CUDA;
    }
    if (cudaSetDevice(device) != cudaSuccess) return EPG_ERR_CUDA;
    // the library's temporaries come from the device's default stream-ordered pool; keep up to
    // EPG_POOL_KEEP_GB (default 32) GiB of freed memory mapped instead of returning it at every
    // synchronisation, so partition / remap / plan builds reuse their multi-GB scratch instead of
    // mapping it afresh each time
    {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            const char *e = std::getenv("EPG_POOL_KEEP_GB");
            uint64_t keep = (uint64_t)(e ? std::max(0.0, std::atof(e)) : 32.0) << 30;
            uint64_t cur = 0;
            if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &cur) == cudaSuccess && cur < keep)
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    }
    epg_ctx *c = new epg_ctx();
    c->device = device;
    c->stream = static_cast<cudaStream_t>(cuda_stream);
    *out = c;
    return EPG_OK;
}

void epg_destroy(epg_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->naive_F) cudaFree(ctx->naive_F);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (HostRun *h = ctx->hr) {
        cudaStreamSynchronize(h->s_in);
        cudaStreamSynchronize(h->s_out);
        cudaStreamSynchronize(ctx->stream);
        for (int j = 0; j < 2; j++) {
            cudaFree(h->stage_in[j]); cudaFree(h->stage_out[j]); cudaFree(h->buf[j]);
            cudaEventDestroy(h->ev_in[j]); cudaEventDestroy(h->ev_consumed[j]);
            cudaEventDestroy(h->ev_comp[j]); cudaEventDestroy(h->ev_out[j]);
        }
        cudaStreamDestroy(h->s_in);
        cudaStreamDestroy(h->s_out);
        delete h;
    }
    comm_release(ctx);
    for (auto &u : ctx->ev_used) { cudaEventDestroy(u.second.first); cudaEventDestroy(u.second.second); }
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    delete ctx;
}

const char *epg_last_error(const epg_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

}  // extern "C"

namespace {
// epg_partition / epg_partition_rb: host partitioner (or, for EPG-RB, GPU bisection levels +
// host leaves), then the GPU cost function on the map
epg_status partition_impl(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n, int32_t part_size, int32_t shards,
                          int32_t method, int32_t leaf_parts, int32_t *part_of_edge, int32_t *rank_of_edge,
                          epg_report *out) {
    if (!edges || !part_of_edge || !out || m <= 0 || n <= 0)
        return ctx->fail(EPG_ERR_INPUT, "partition: need m > 0, n > 0 and non-NULL arrays");
    if (m >= kMaxEdges) return ctx->fail(EPG_ERR_INPUT, "partition: m must be below 2^30");
    CU(cudaSetDevice(ctx->device));
    const bool edges_dev = is_device_ptr(edges), part_dev = is_device_ptr(part_of_edge);
    Tmp ed(ctx), pd(ctx);
    const int32_t *edges_d = edges;
    if (!edges_dev) {
        CU(ed.alloc(sizeof(int32_t) * 2 * m));
        CU(cudaMemcpyAsync(ed.p, edges, sizeof(int32_t) * 2 * m, cudaMemcpyHostToDevice, ctx->stream));
        edges_d = ed.as<int32_t>();
    }
    int32_t *part_d = part_of_edge;
    if (!part_dev) {
        CU(pd.alloc(sizeof(int32_t) * m));
        part_d = pd.as<int32_t>();
    }
    const bool rank_dev = rank_of_edge && is_device_ptr(rank_of_edge);
    Tmp rd(ctx);
    int32_t *rank_d = rank_of_edge;
    if (rank_of_edge && !rank_dev) {
        CU(rd.alloc(sizeof(int32_t) * m));
        rank_d = rd.as<int32_t>();
    }
    std::string err;
    epg_status st;
    if (method == EPG_PARTITION_RB) {
        if (leaf_parts < 1) return ctx->fail(EPG_ERR_INPUT, "partition (RB): leaf_parts must be >= 1");
        if ((st = validate(ctx, edges_d, m, n, nullptr, 0))) return st;
        if (part_size < 1 || part_size > EPG_MAX_PART_SIZE)
            return ctx->fail(EPG_ERR_INFEASIBLE, "partition: part_size must be in [1, 4096]");
        const int64_t k = epg_num_parts(m, part_size);
        if (!(shards == 1 || shards == 2 || shards == 4 || shards == 8) || shards > k)
            return ctx->fail(EPG_ERR_INFEASIBLE, "partition: shards must be 1, 2, 4 or 8 and at most k");
        if ((st = rb_partition(ctx, edges_d, m, n, part_size, shards, leaf_parts, part_d, rank_d, &err)))
            return err.empty() ? st : ctx->fail(st, err);
        if (!part_dev) CU(cudaMemcpyAsync(part_of_edge, part_d, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, ctx->stream));
        if (rank_of_edge && !rank_dev)
            CU(cudaMemcpyAsync(rank_of_edge, rank_d, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    } else {
        std::vector<int32_t> eh, ph(m);
        const int32_t *edges_h = edges;
        if (edges_dev) {
            eh.resize(2 * m);
            CU(cudaMemcpyAsync(eh.data(), edges, sizeof(int32_t) * 2 * m, cudaMemcpyDeviceToHost, ctx->stream));
            CU(cudaStreamSynchronize(ctx->stream));
            edges_h = eh.data();
        }
        std::vector<int32_t> rh(rank_of_edge ? m : 0);
        st = epg::host_partition(edges_h, m, n, part_size, shards, ph.data(), &err, nullptr, method,
                                 rank_of_edge ? rh.data() : nullptr);
        if (st) return ctx->fail(st, err);
        if (!part_dev) std::memcpy(part_of_edge, ph.data(), sizeof(int32_t) * m);
        CU(cudaMemcpyAsync(part_d, ph.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, ctx->stream));
        if (rank_of_edge) {
            if (rank_dev)
                CU(cudaMemcpyAsync(rank_of_edge, rh.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, ctx->stream));
            else
                std::memcpy(rank_of_edge, rh.data(), sizeof(int32_t) * m);
        }
        CU(cudaStreamSynchronize(ctx->stream));   // ph / rh are host vectors
    }
    return load_count_dev(ctx, edges_d, m, n, part_d, epg_num_parts(m, part_size), nullptr, out);
}

int rb_leaf_parts_default() {
    const char *e = std::getenv("EPG_RB_LEAF_PARTS");
    return e ? std::max(1, std::atoi(e)) : 512;
}
}  // namespace

extern "C" {

epg_status epg_partition(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n, int32_t part_size,
                         int32_t shards, int32_t *part_of_edge, epg_report *out) {
    if (!ctx) return EPG_ERR_STATE;
    return partition_impl(ctx, edges, m, n, part_size, shards, ctx->partition_method, rb_leaf_parts_default(),
                          part_of_edge, nullptr, out);
}

epg_status epg_partition_ranked(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n, int32_t part_size,
                                int32_t shards, int32_t *part_of_edge, int32_t *rank_of_edge, epg_report *out) {
    if (!ctx) return EPG_ERR_STATE;
    return partition_impl(ctx, edges, m, n, part_size, shards, ctx->partition_method, rb_leaf_parts_default(),
                          part_of_edge, rank_of_edge, out);
}

epg_status epg_partition_rb(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n, int32_t part_size,
                            int32_t shards, int32_t leaf_parts, int32_t *part_of_edge, int32_t *rank_of_edge,
                            epg_report *out) {
    if (!ctx) return EPG_ERR_STATE;
    return partition_impl(ctx, edges, m, n, part_size, shards, EPG_PARTITION_RB, leaf_parts, part_of_edge,
                          rank_of_edge, out);
}

epg_status epg_default_partition(epg_ctx *ctx, int64_t m, int32_t part_size, int32_t *part_of_edge) {
    if (!ctx) return EPG_ERR_STATE;
    if (m <= 0 || !part_of_edge) return ctx->fail(EPG_ERR_INPUT, "default_partition: need m > 0 and an output");
    if (part_size < 1 || part_size > EPG_MAX_PART_SIZE)
        return ctx->fail(EPG_ERR_INFEASIBLE, "default_partition: part_size must be in [1, 4096]");
    CU(cudaSetDevice(ctx->device));
    k_default_partition<<<grid_for(m), kThreads, 0, ctx->stream>>>(m, epg_num_parts(m, part_size), part_of_edge);
    CHECK_LAUNCH();
    return EPG_OK;
}

epg_status epg_load_count(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n, const int32_t *part_of_edge,
                          int64_t k, int32_t *per_part_distinct, epg_report *out) {
    if (!ctx) return EPG_ERR_STATE;
    if (!edges || !part_of_edge || !out || m <= 0 || n <= 0 || k <= 0)
        return ctx->fail(EPG_ERR_INPUT, "load_count: need m > 0, n > 0, k > 0 and non-NULL arrays");
    CU(cudaSetDevice(ctx->device));
    return load_count_dev(ctx, edges, m, n, part_of_edge, k, per_part_distinct, out);
}

}  // extern "C"

namespace {
// Remap of one partition map (O6) + the execution plan built on it.
epg_status remap_impl(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n, const int32_t *part, int64_t k,
                      epg_layout *L, epg_plan **plan_out, const int32_t *order_key = nullptr) {
    if (!edges || !part || !L || !plan_out || m <= 0 || n <= 0 || k <= 0)
        return ctx->fail(EPG_ERR_INPUT, "remap: need m > 0, n > 0, k > 0 and non-NULL arrays");
    if (m >= kMaxEdges)   // first-touch keys 2e' + s and the scan / sort sizes are int32
        return ctx->fail(EPG_ERR_INPUT, "remap: m must be below 2^30");
    if (!L->edge_perm || !L->part_edge_begin || !L->vertex_perm || !L->part_vertex_begin || !L->halo_begin ||
        !L->slots || (!L->halo_ids && L->halo_cap > 0))
        return ctx->fail(EPG_ERR_INPUT, "remap: every layout array is required");
    *plan_out = nullptr;
    CU(cudaSetDevice(ctx->device));
    epg_status st = validate(ctx, edges, m, n, part, k);
    if (st) return st;
    // 1. task reorganisation: stable sort by partition
    std::vector<int32_t> peb_h;
    if ((st = group_by_part(ctx, part, m, k, L->edge_perm, L->part_edge_begin, &peb_h, order_key))) return st;
    int64_t smax = 0;
    for (int64_t p = 0; p < k; p++) smax = std::max<int64_t>(smax, peb_h[p + 1] - peb_h[p]);
    if (smax > EPG_MAX_PART_SIZE)
        return ctx->fail(EPG_ERR_INFEASIBLE, "remap: a partition has " + std::to_string(smax) +
                                                 " edges; at most 4096 fit the uint16 slots");
    Tmp distinct(ctx), key(ctx), flag(ctx), rank(ctx), uflag(ctx), urank(ctx), nh(ctx);
    CU(distinct.alloc(sizeof(int32_t) * k));
    if ((st = distinct_counts(ctx, edges, part, m, n, L->edge_perm, L->part_edge_begin, k, smax,
                              distinct.as<int32_t>())))
        return st;
    // 2. first-touch keys; 3. ranks -> vertex_perm
    CU(key.alloc(sizeof(int32_t) * n));
    k_fill<int32_t><<<grid_for(n), kThreads, 0, ctx->stream>>>(key.as<int32_t>(), n, kSentinel);
    k_first_touch<<<grid_for(m), kThreads, 0, ctx->stream>>>(edges, L->edge_perm, m, key.as<int32_t>());
    CU(flag.alloc(sizeof(int32_t) * (2 * m + 1)));
    CU(rank.alloc(sizeof(int32_t) * (2 * m + 1)));
    k_first_touch_flags<<<grid_for(2 * m + 1), kThreads, 0, ctx->stream>>>(edges, L->edge_perm, m,
                                                                          key.as<int32_t>(), flag.as<int32_t>());
    CHECK_LAUNCH();
    if ((st = exclusive_scan(ctx, flag.as<int32_t>(), rank.as<int32_t>(), 2 * m + 1))) return st;
    int32_t touched = 0;
    if ((st = read_i32(ctx, rank.as<int32_t>() + 2 * m, &touched))) return st;
    CU(uflag.alloc(sizeof(int32_t) * (n + 1)));
    CU(urank.alloc(sizeof(int32_t) * (n + 1)));
    k_vperm_touched<<<grid_for(n + 1), kThreads, 0, ctx->stream>>>(key.as<int32_t>(), rank.as<int32_t>(), n,
                                                                  L->vertex_perm, uflag.as<int32_t>());
    if ((st = exclusive_scan(ctx, uflag.as<int32_t>(), urank.as<int32_t>(), n + 1))) return st;
    k_vperm_untouched<<<grid_for(n), kThreads, 0, ctx->stream>>>(key.as<int32_t>(), urank.as<int32_t>(), n, touched,
                                                                L->vertex_perm);
    // 4. beginA
    k_pvb<<<grid_for(k + 1), kThreads, 0, ctx->stream>>>(rank.as<int32_t>(), L->part_edge_begin, k,
                                                        L->part_vertex_begin);
    // 5. halo sizes -> halo_begin
    CU(nh.alloc(sizeof(int32_t) * (k + 1)));
    k_halo_counts<<<grid_for(k + 1), kThreads, 0, ctx->stream>>>(distinct.as<int32_t>(), L->part_vertex_begin, k,
                                                                nh.as<int32_t>());
    CHECK_LAUNCH();
    if ((st = exclusive_scan(ctx, nh.as<int32_t>(), L->halo_begin, k + 1))) return st;
    int32_t C = 0;
    if ((st = read_i32(ctx, L->halo_begin + k, &C))) return st;
    if (C > L->halo_cap)
        return ctx->fail(EPG_ERR_INPUT, "remap: halo_cap " + std::to_string(L->halo_cap) + " < cut cost " +
                                            std::to_string(C));
    // plan
    epg_plan *pl = new epg_plan();
    pl->ctx = ctx; pl->device = ctx->device;
    pl->m = m; pl->n = n; pl->k = k; pl->touched = touched; pl->C = C;
    auto fail_plan = [&](epg_status s) { delete pl; return s; };
    if ((st = plan_alloc_t(pl, ctx, &pl->peb, k + 1)) || (st = plan_alloc_t(pl, ctx, &pl->pvb, k + 1)) ||
        (st = plan_alloc_t(pl, ctx, &pl->hb, k + 1)) || (st = plan_alloc_t(pl, ctx, &pl->halo_ids, C)) ||
        (st = plan_alloc_t(pl, ctx, &pl->slots, m)) || (st = plan_alloc_t(pl, ctx, &pl->inc, 2 * m)) ||
        (st = plan_alloc_t(pl, ctx, &pl->inc_off, (int64_t)touched + C)) ||
        (st = plan_alloc_t(pl, ctx, &pl->sidx, n + 1)))
        return fail_plan(st);
    // 6-7. per-partition sort: halo ids, slots, incidence lists
    {
        const int eb = bits_for(n);
        uint16_t *slots16 = L->slots;
        if (2 * smax <= 512)
            st = launch_remap_part<256, 2>(ctx, edges, L->edge_perm, L->vertex_perm, L->part_edge_begin,
                                           L->part_vertex_begin, L->halo_begin, L->halo_ids, slots16, pl->inc,
                                           pl->inc_off, k, eb);
        else if (2 * smax <= 2048)
            st = launch_remap_part<256, 8>(ctx, edges, L->edge_perm, L->vertex_perm, L->part_edge_begin,
                                           L->part_vertex_begin, L->halo_begin, L->halo_ids, slots16, pl->inc,
                                           pl->inc_off, k, eb);
        else
            st = launch_remap_part<512, 16>(ctx, edges, L->edge_perm, L->vertex_perm, L->part_edge_begin,
                                            L->part_vertex_begin, L->halo_begin, L->halo_ids, slots16, pl->inc,
                                            pl->inc_off, k, eb);
        if (st) return fail_plan(st);
    }
#define CPY(dst, src, bytes)                                                                          \
    do {                                                                                              \
        cudaError_t _e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream);     \
        if (_e != cudaSuccess) return fail_plan(ctx->fail(EPG_ERR_CUDA, cudaGetErrorString(_e)));      \
    } while (0)
    CPY(pl->peb, L->part_edge_begin, sizeof(int32_t) * (k + 1));
    CPY(pl->pvb, L->part_vertex_begin, sizeof(int32_t) * (k + 1));
    CPY(pl->hb, L->halo_begin, sizeof(int32_t) * (k + 1));
    if (C > 0) CPY(pl->halo_ids, L->halo_ids, sizeof(int32_t) * C);
    CPY(pl->slots, L->slots, sizeof(uint32_t) * m);
    // shared vertices (p_v > 1) and their halo positions
    {
        Tmp sflag(ctx), sscan(ctx), iota(ctx), skeys(ctx), temp(ctx);
        if (sflag.alloc(sizeof(int32_t) * (n + 1)) || sscan.alloc(sizeof(int32_t) * (n + 1)))
            return fail_plan(ctx->fail(EPG_ERR_NOMEM, "remap: temporaries"));
        cudaMemsetAsync(sflag.p, 0, sizeof(int32_t) * (n + 1), ctx->stream);
        if (C > 0) k_mark_shared<<<grid_for(C), kThreads, 0, ctx->stream>>>(pl->halo_ids, C, sflag.as<int32_t>());
        if ((st = exclusive_scan(ctx, sflag.as<int32_t>(), sscan.as<int32_t>(), n + 1))) return fail_plan(st);
        int32_t S = 0;
        if ((st = read_i32(ctx, sscan.as<int32_t>() + n, &S))) return fail_plan(st);
        pl->S = S;
        if ((st = plan_alloc_t(pl, ctx, &pl->shared_ids, S)) || (st = plan_alloc_t(pl, ctx, &pl->hv_off, S + 1)) ||
            (st = plan_alloc_t(pl, ctx, &pl->hv_list, C)) || (st = plan_alloc_t(pl, ctx, &pl->owner_buf, 5 * S)) ||
            (st = plan_alloc_t(pl, ctx, &pl->halo_buf, 5 * (int64_t)C)))
            return fail_plan(st);
        k_shared_index<<<grid_for(n), kThreads, 0, ctx->stream>>>(sflag.as<int32_t>(), sscan.as<int32_t>(), n,
                                                                 pl->sidx, pl->shared_ids);
        if (C > 0) {
            if (iota.alloc(sizeof(int32_t) * C) || skeys.alloc(sizeof(int32_t) * C))
                return fail_plan(ctx->fail(EPG_ERR_NOMEM, "remap: temporaries"));
            k_iota<<<grid_for(C), kThreads, 0, ctx->stream>>>(iota.as<int32_t>(), C);
            size_t tb = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tb, pl->halo_ids, skeys.as<int32_t>(), iota.as<int32_t>(),
                                            pl->hv_list, (int)C, 0, bits_for(n), ctx->stream);
            if (temp.alloc(tb)) return fail_plan(ctx->fail(EPG_ERR_NOMEM, "remap: temporaries"));
            cub::DeviceRadixSort::SortPairs(temp.p, tb, pl->halo_ids, skeys.as<int32_t>(), iota.as<int32_t>(),
                                            pl->hv_list, (int)C, 0, bits_for(n), ctx->stream);
        }
        k_hv_off<<<grid_for(C + 1), kThreads, 0, ctx->stream>>>(skeys.as<int32_t>(), C, pl->sidx, S, pl->hv_off);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return fail_plan(ctx->fail(EPG_ERR_CUDA, cudaGetErrorString(e)));
    }
#undef CPY
    // staging capacities
    {
        std::vector<int32_t> dh(k);
        cudaError_t e = cudaMemcpyAsync(dh.data(), distinct.p, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, ctx->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return fail_plan(ctx->fail(EPG_ERR_CUDA, cudaGetErrorString(e)));
        pl->Lcap = *std::max_element(dh.begin(), dh.end());
        pl->Scap = (int)smax;
    }
    if ((st = build_pipeline_blob(ctx, pl))) return fail_plan(st);
    pl->k_ep = k;
    pl->C_ep = C;
    pl->exec_base.resize(k + 1);
    for (int64_t p = 0; p <= k; p++) pl->exec_base[p] = (int32_t)p;
    *plan_out = pl;
    return EPG_OK;
}
}  // namespace

namespace epg {
void *ctx_stream(epg_ctx *ctx) { return ctx->stream; }
int32_t ctx_partition_method(epg_ctx *ctx) { return ctx->partition_method; }
int ctx_device(epg_ctx *ctx) { return ctx->device; }
epg_status ctx_fail(epg_ctx *ctx, epg_status s, const std::string &msg) { return ctx->fail(s, msg); }
}  // namespace epg

extern "C" {

// Task reorganisation + cpack layout of the EP map (the public layout), then the
// execution plan: EP partitions whose staged rows or edges exceed what one CTA holds are
// executed as contiguous ranges of their (reorganised) edges. Cutting a partition into
// contiguous edge ranges changes neither the edge order nor any first touch, so the
// execution plan shares the public edge_perm / vertex_perm exactly.
epg_status epg_remap(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n, const int32_t *part, int64_t k,
                     epg_layout *L, epg_plan **plan_out) {
    return epg_remap_keyed(ctx, edges, m, n, part, nullptr, k, L, plan_out);
}

epg_status epg_remap_keyed(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n, const int32_t *part,
                           const int32_t *order_key, int64_t k, epg_layout *L, epg_plan **plan_out) {
    if (!ctx) return EPG_ERR_STATE;
    if (!plan_out) return ctx->fail(EPG_ERR_INPUT, "remap: plan output is NULL");
    *plan_out = nullptr;
    epg_plan *ep = nullptr;
    epg_status st = remap_impl(ctx, edges, m, n, part, k, L, &ep, order_key);
    if (st) return st;
    const int kExecMaxEdges = exec_max_edges(ctx), kExecMaxRows = exec_max_rows(ctx);
    std::vector<int32_t> cuts(k, 1);
    bool split = false;
    for (int64_t p = 0; p < k; p++) {
        const int c = std::max((ep->part_edges[p] + kExecMaxEdges - 1) / kExecMaxEdges,
                               (ep->part_rows[p] + kExecMaxRows - 1) / kExecMaxRows);
        cuts[p] = std::max(c, 1);
        split |= cuts[p] > 1;
    }
    if (!split) {
        *plan_out = ep;
        return EPG_OK;
    }
    // temporary layout for the execution map
    Tmp pe(ctx), cu(ctx), ba(ctx), t_ep(ctx), t_peb(ctx), t_vp(ctx), t_pvb(ctx), t_hb(ctx), t_hid(ctx), t_sl(ctx);
    auto fail_ep = [&](epg_status s2) { delete ep; return s2; };
    if (pe.alloc(sizeof(int32_t) * m) || cu.alloc(sizeof(int32_t) * k) || ba.alloc(sizeof(int32_t) * k) ||
        t_ep.alloc(sizeof(int32_t) * m) || t_vp.alloc(sizeof(int32_t) * n) || t_hid.alloc(sizeof(int32_t) * 2 * m) ||
        t_sl.alloc(sizeof(uint16_t) * 2 * m))
        return fail_ep(ctx->fail(EPG_ERR_NOMEM, "remap: execution-plan temporaries"));
    for (int iter = 0; iter < 8; iter++) {
        std::vector<int32_t> base(k);
        int64_t kx = 0;
        for (int64_t p = 0; p < k; p++) { base[p] = (int32_t)kx; kx += cuts[p]; }
        Tmp peb_x(ctx), pvb_x(ctx), hb_x(ctx);
        if (peb_x.alloc(sizeof(int32_t) * (kx + 1)) || pvb_x.alloc(sizeof(int32_t) * (kx + 1)) ||
            hb_x.alloc(sizeof(int32_t) * (kx + 1)))
            return fail_ep(ctx->fail(EPG_ERR_NOMEM, "remap: execution-plan temporaries"));
        cudaMemcpyAsync(cu.p, cuts.data(), sizeof(int32_t) * k, cudaMemcpyHostToDevice, ctx->stream);
        cudaMemcpyAsync(ba.p, base.data(), sizeof(int32_t) * k, cudaMemcpyHostToDevice, ctx->stream);
        k_exec_map<<<(unsigned)k, 256, 0, ctx->stream>>>(ep->peb, L->edge_perm, cu.as<int32_t>(), ba.as<int32_t>(),
                                                         pe.as<int32_t>());
        epg_layout X{t_ep.as<int32_t>(), peb_x.as<int32_t>(), t_vp.as<int32_t>(), pvb_x.as<int32_t>(),
                     hb_x.as<int32_t>(), t_hid.as<int32_t>(), 2 * m, t_sl.as<uint16_t>()};
        epg_plan *xp = nullptr;
        // the pieces are contiguous ranges of the (partition, key, id) order, so sorting by
        // (piece, key, id) reproduces that order: same first touches, same vertex_perm
        if ((st = remap_impl(ctx, edges, m, n, pe.as<int32_t>(), kx, &X, &xp, order_key))) return fail_ep(st);
        bool again = false;
        for (int64_t p = 0, e = 0; p < k; p++)
            for (int c = 0; c < cuts[p]; c++, e++)
                if (xp->part_rows[e] > kExecMaxRows || xp->part_edges[e] > kExecMaxEdges) again = true;
        if (!again || iter == 7) {
            xp->k_ep = k;
            xp->C_ep = ep->C;
            xp->exec_base.assign(base.begin(), base.end());
            xp->exec_base.push_back((int32_t)kx);
            delete ep;
            *plan_out = xp;
            return EPG_OK;
        }
        for (int64_t p = 0, e = 0; p < k; p++) {
            bool bad = false;
            for (int c = 0; c < cuts[p]; c++, e++)
                bad |= xp->part_rows[e] > kExecMaxRows || xp->part_edges[e] > kExecMaxEdges;
            if (bad) cuts[p] += 1;
        }
        delete xp;
    }
    return fail_ep(ctx->fail(EPG_ERR_STATE, "remap: execution split did not converge"));
}

void epg_plan_destroy(epg_plan *plan) {
    if (!plan) return;
    cudaSetDevice(plan->device);
    delete plan;
}

epg_status epg_plan_info(const epg_plan *plan, int64_t *out8) {
    if (!plan || !out8) return EPG_ERR_INPUT;
    out8[0] = plan->m; out8[1] = plan->n; out8[2] = plan->k_ep;
    out8[3] = plan->touched; out8[4] = plan->C_ep; out8[5] = plan->S;
    out8[6] = plan->k; out8[7] = plan->C;
    return EPG_OK;
}

epg_status epg_permute_rows(epg_ctx *ctx, const void *src, void *dst, int64_t rows, int32_t row_bytes,
                            const int32_t *perm, int32_t mode) {
    if (!ctx) return EPG_ERR_STATE;
    if (rows == 0) return EPG_OK;
    if (!src || !dst || !perm || rows < 0 || row_bytes <= 0 || row_bytes % 4 || (mode != 0 && mode != 1))
        return ctx->fail(EPG_ERR_INPUT, "permute_rows: bad arguments");
    if (src == dst) return ctx->fail(EPG_ERR_INPUT, "permute_rows: src and dst alias");
    CU(cudaSetDevice(ctx->device));
    const int32_t words = row_bytes / 4;
    if (rows > 0)
        k_permute_rows<<<grid_for(rows * words), kThreads, 0, ctx->stream>>>(
            static_cast<const uint32_t *>(src), static_cast<uint32_t *>(dst), rows, words, perm, mode);
    CHECK_LAUNCH();
    return EPG_OK;
}

epg_status epg_run(epg_ctx *ctx, const epg_plan *plan, epg_kernel kernel, epg_state *state, int32_t steps) {
    if (!ctx) return EPG_ERR_STATE;
    if (!plan) return ctx->fail(EPG_ERR_INPUT, "run: plan is NULL");
    if (plan->ctx != ctx || plan->device != ctx->device)
        return ctx->fail(EPG_ERR_STATE, "run: plan belongs to another context");
    epg_status st = check_state(ctx, kernel, state);
    if (st) return st;
    if (steps < 0) return ctx->fail(EPG_ERR_INPUT, "run: steps < 0");
    CU(cudaSetDevice(ctx->device));
    epg_plan *pl = const_cast<epg_plan *>(plan);   // caches: CTA assignment, graphs (internal state)
    switch (kernel) {
        case EPG_KERNEL_CFD_FLUX: return run_graphed<CfdFlux>(ctx, pl, kernel, state, steps);
        case EPG_KERNEL_GATHER_SCATTER: return run_graphed<GatherScatter>(ctx, pl, kernel, state, steps);
        default: return run_graphed<Spmv>(ctx, pl, kernel, state, steps);
    }
}

epg_status epg_run_host(epg_ctx *ctx, const epg_plan *plan, epg_kernel kernel, const int32_t *vertex_perm,
                        const void *state_in_host, void *state_out_host, const void *edge_payload,
                        const void *vertex_const, int32_t steps) {
    if (!ctx) return EPG_ERR_STATE;
    if (!plan) return ctx->fail(EPG_ERR_INPUT, "run_host: plan is NULL");
    if (plan->ctx != ctx || plan->device != ctx->device)
        return ctx->fail(EPG_ERR_STATE, "run_host: plan belongs to another context");
    if (!vertex_perm || !state_in_host || !state_out_host || steps < 0)
        return ctx->fail(EPG_ERR_INPUT, "run_host: need vertex_perm, host state in/out and steps >= 0");
    if (kernel < EPG_KERNEL_CFD_FLUX || kernel > EPG_KERNEL_SPMV) return ctx->fail(EPG_ERR_INPUT, "run_host: unknown kernel id");
    CU(cudaSetDevice(ctx->device));
    const int row = kernel == EPG_KERNEL_CFD_FLUX ? 5 : 1;
    const size_t bytes = sizeof(float) * row * (size_t)plan->n;
    HostRun *h = ctx->hr;
    if (!h) {
        h = ctx->hr = new HostRun();
        CU(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
        CU(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
        for (int j = 0; j < 2; j++) {
            CU(cudaEventCreateWithFlags(&h->ev_in[j], cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&h->ev_consumed[j], cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&h->ev_comp[j], cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&h->ev_out[j], cudaEventDisableTiming));
        }
    }
    if (h->bytes < bytes) {   // (re)allocate: drain the pipeline first
        CU(cudaStreamSynchronize(h->s_in));
        CU(cudaStreamSynchronize(h->s_out));
        CU(cudaStreamSynchronize(ctx->stream));
        for (int j = 0; j < 2; j++) {
            cudaFree(h->stage_in[j]); cudaFree(h->stage_out[j]); cudaFree(h->buf[j]);
            h->stage_in[j] = h->stage_out[j] = h->buf[j] = nullptr;
            h->used[j] = false;
        }
        for (int j = 0; j < 2; j++) {
            if (cudaMalloc(&h->stage_in[j], bytes) || cudaMalloc(&h->stage_out[j], bytes) || cudaMalloc(&h->buf[j], bytes)) {
                cudaGetLastError();
                h->bytes = 0;
                return ctx->fail(EPG_ERR_NOMEM, "run_host: device buffers");
            }
        }
        h->bytes = bytes;
    }
    const int j = h->parity;
    h->parity ^= 1;
    // copy-in: stage_in[j] is free once call i-2's scatter consumed it
    if (h->used[j]) CU(cudaStreamWaitEvent(h->s_in, h->ev_consumed[j], 0));
    CU(cudaMemcpyAsync(h->stage_in[j], state_in_host, bytes, cudaMemcpyHostToDevice, h->s_in));
    CU(cudaEventRecord(h->ev_in[j], h->s_in));
    // compute on the ctx stream: original order -> plan layout, steps, back
    CU(cudaStreamWaitEvent(ctx->stream, h->ev_in[j], 0));
    epg_status st = epg_permute_rows(ctx, h->stage_in[j], h->buf[0], plan->n, 4 * row, vertex_perm, 1);
    if (st) return st;
    CU(cudaEventRecord(h->ev_consumed[j], ctx->stream));
    void *res = h->buf[0];
    if (steps > 0) {
        epg_state sst{h->buf[0], h->buf[1], edge_payload, vertex_const};
        if ((st = epg_run(ctx, plan, kernel, &sst, steps))) return st;
        res = h->buf[steps & 1];
    }
    if (h->used[j]) CU(cudaStreamWaitEvent(ctx->stream, h->ev_out[j], 0));   // call i-2's D2H read stage_out[j]
    if ((st = epg_permute_rows(ctx, res, h->stage_out[j], plan->n, 4 * row, vertex_perm, 0))) return st;
    CU(cudaEventRecord(h->ev_comp[j], ctx->stream));
    // copy-out
    CU(cudaStreamWaitEvent(h->s_out, h->ev_comp[j], 0));
    CU(cudaMemcpyAsync(state_out_host, h->stage_out[j], bytes, cudaMemcpyDeviceToHost, h->s_out));
    CU(cudaEventRecord(h->ev_out[j], h->s_out));
    h->used[j] = true;
    return EPG_OK;
}

epg_status epg_run_host_join(epg_ctx *ctx) {
    if (!ctx) return EPG_ERR_STATE;
    if (!ctx->hr) return EPG_OK;
    CU(cudaSetDevice(ctx->device));
    for (int j = 0; j < 2; j++)
        if (ctx->hr->used[j]) CU(cudaStreamWaitEvent(ctx->stream, ctx->hr->ev_out[j], 0));
    return EPG_OK;
}

epg_status epg_run_naive(epg_ctx *ctx, epg_kernel kernel, const int32_t *edges, int64_t m, int32_t n,
                         epg_state *state, int32_t steps) {
    if (!ctx) return EPG_ERR_STATE;
    if (!edges || m <= 0 || n <= 0) return ctx->fail(EPG_ERR_INPUT, "run_naive: need m > 0, n > 0, edges");
    epg_status st = check_state(ctx, kernel, state);
    if (st) return st;
    if (steps < 0) return ctx->fail(EPG_ERR_INPUT, "run_naive: steps < 0");
    CU(cudaSetDevice(ctx->device));
    switch (kernel) {
        case EPG_KERNEL_CFD_FLUX: return run_naive<CfdFlux>(ctx, edges, m, n, state, steps);
        case EPG_KERNEL_GATHER_SCATTER: return run_naive<GatherScatter>(ctx, edges, m, n, state, steps);
        default: return run_naive<Spmv>(ctx, edges, m, n, state, steps);
    }
}

// ---- multi-GPU shards ------------------------------------------------
epg_status epg_shard_ranges(const epg_plan *plan_c, int32_t G, int32_t g, int64_t *out8) {
    if (!plan_c || !out8 || G < 1 || g < 0 || g >= G || G > plan_c->k_ep) return EPG_ERR_INPUT;
    epg_plan *pl = const_cast<epg_plan *>(plan_c);
    const int64_t pb = (int64_t)g * pl->k_ep / G, pe = (int64_t)(g + 1) * pl->k_ep / G;
    const int64_t xb = pl->exec_base[pb], xe = pl->exec_base[pe];
    const int64_t vlo = pl->pvb_h[xb], vhi = pl->pvb_h[xe];
    if (pl->shared_h.size() != (size_t)pl->S) {
        pl->shared_h.resize(pl->S);
        if (pl->S > 0 && cudaMemcpy(pl->shared_h.data(), pl->shared_ids, sizeof(int32_t) * pl->S,
                                    cudaMemcpyDeviceToHost) != cudaSuccess)
            return EPG_ERR_CUDA;
    }
    const int64_t slo = std::lower_bound(pl->shared_h.begin(), pl->shared_h.end(), (int32_t)vlo) - pl->shared_h.begin();
    const int64_t shi = std::lower_bound(pl->shared_h.begin(), pl->shared_h.end(), (int32_t)vhi) - pl->shared_h.begin();
    out8[0] = xb; out8[1] = xe - xb;
    out8[2] = pl->hb_h[xb]; out8[3] = pl->hb_h[xe] - pl->hb_h[xb];
    out8[4] = vlo; out8[5] = vhi - vlo;
    out8[6] = slo; out8[7] = shi - slo;
    return EPG_OK;
}

epg_status epg_shard_halos_host(const int32_t *pvb, const int32_t *hb, const int32_t *halo_ids, int64_t k, int32_t G,
                                int32_t *begin_out, int32_t *ids_out, int64_t cap, int64_t *count_out) {
    if (!pvb || !hb || !begin_out || !count_out || k < 1 || G < 1 || G > k) return EPG_ERR_INPUT;
    std::vector<int64_t> own_lo(G + 1);
    for (int32_t g = 0; g <= G; g++) own_lo[g] = pvb[(int64_t)g * k / G];
    int64_t pos = 0;
    std::vector<int32_t> h;
    for (int32_t g = 0; g < G; g++) {
        const int64_t pb = (int64_t)g * k / G, pe = (int64_t)(g + 1) * k / G;
        h.assign(halo_ids + hb[pb], halo_ids + hb[pe]);
        std::sort(h.begin(), h.end());
        h.erase(std::unique(h.begin(), h.end()), h.end());
        // Halo^g = halo ids of g's partitions owned below g's range, by owner shard
        for (int32_t g2 = 0; g2 < G; g2++) {
            begin_out[g * G + g2] = (int32_t)pos;
            if (g2 >= g) continue;
            auto lo = std::lower_bound(h.begin(), h.end(), (int32_t)own_lo[g2]);
            auto hi = std::lower_bound(h.begin(), h.end(), (int32_t)own_lo[g2 + 1]);
            for (auto it = lo; it != hi; ++it) {
                if (ids_out) {
                    if (pos >= cap) return EPG_ERR_INPUT;
                    ids_out[pos] = *it;
                }
                pos++;
            }
        }
    }
    begin_out[G * G] = (int32_t)pos;
    *count_out = pos;
    return EPG_OK;
}

epg_status epg_run_edges(epg_ctx *ctx, const epg_plan *plan, epg_kernel kernel, epg_state *state, int64_t first,
                         int64_t count) {
    if (!ctx) return EPG_ERR_STATE;
    if (!plan || plan->ctx != ctx) return ctx->fail(EPG_ERR_STATE, "run_edges: plan belongs to another context");
    epg_status st = check_state(ctx, kernel, state);
    if (st) return st;
    if (first < 0 || count < 0 || first + count > plan->k) return ctx->fail(EPG_ERR_INPUT, "run_edges: bad range");
    CU(cudaSetDevice(ctx->device));
    epg_plan *pl = const_cast<epg_plan *>(plan);
    switch (kernel) {
        case EPG_KERNEL_CFD_FLUX: return run_edges_range<CfdFlux>(ctx, pl, state, first, count);
        case EPG_KERNEL_GATHER_SCATTER: return run_edges_range<GatherScatter>(ctx, pl, state, first, count);
        default: return run_edges_range<Spmv>(ctx, pl, state, first, count);
    }
}

epg_status epg_run_finalise(epg_ctx *ctx, const epg_plan *plan, epg_kernel kernel, epg_state *state,
                            int64_t shared_first, int64_t shared_count, int64_t halo_first, int64_t halo_count,
                            float *acc, int32_t untouched) {
    if (!ctx) return EPG_ERR_STATE;
    if (!plan || plan->ctx != ctx) return ctx->fail(EPG_ERR_STATE, "run_finalise: plan belongs to another context");
    epg_status st = check_state(ctx, kernel, state);
    if (st) return st;
    if (shared_first < 0 || shared_count < 0 || shared_first + shared_count > plan->S || halo_first < 0 ||
        halo_count < 0 || halo_first + halo_count > plan->C)
        return ctx->fail(EPG_ERR_INPUT, "run_finalise: bad range");
    CU(cudaSetDevice(ctx->device));
    epg_plan *pl = const_cast<epg_plan *>(plan);
    switch (kernel) {
        case EPG_KERNEL_CFD_FLUX:
            return run_finalise_range<CfdFlux>(ctx, pl, state, shared_first, shared_count, halo_first, halo_count, acc,
                                               untouched);
        case EPG_KERNEL_GATHER_SCATTER:
            return run_finalise_range<GatherScatter>(ctx, pl, state, shared_first, shared_count, halo_first,
                                                     halo_count, acc, untouched);
        default:
            return run_finalise_range<Spmv>(ctx, pl, state, shared_first, shared_count, halo_first, halo_count, acc,
                                            untouched);
    }
}

epg_status epg_shard_reduce(epg_ctx *ctx, const epg_plan *plan, epg_kernel kernel, const int32_t *ids, int64_t count,
                            int64_t halo_first, int64_t halo_count, float *out_rows) {
    if (!ctx) return EPG_ERR_STATE;
    if (!plan || plan->ctx != ctx) return ctx->fail(EPG_ERR_STATE, "shard_reduce: plan belongs to another context");
    if (count < 0 || (count > 0 && (!ids || !out_rows))) return ctx->fail(EPG_ERR_INPUT, "shard_reduce: arguments");
    if (count == 0) return EPG_OK;
    CU(cudaSetDevice(ctx->device));
    const int64_t hl = halo_first, hh = halo_first + halo_count;
    switch (kernel) {
        case EPG_KERNEL_CFD_FLUX:
            k_shard_reduce<CfdFlux><<<grid_for(count), kThreads, 0, ctx->stream>>>(
                ids, count, plan->sidx, plan->hv_off, plan->hv_list, plan->halo_buf, hl, hh, out_rows);
            break;
        case EPG_KERNEL_GATHER_SCATTER:
            k_shard_reduce<GatherScatter><<<grid_for(count), kThreads, 0, ctx->stream>>>(
                ids, count, plan->sidx, plan->hv_off, plan->hv_list, plan->halo_buf, hl, hh, out_rows);
            break;
        default:
            k_shard_reduce<Spmv><<<grid_for(count), kThreads, 0, ctx->stream>>>(
                ids, count, plan->sidx, plan->hv_off, plan->hv_list, plan->halo_buf, hl, hh, out_rows);
    }
    CHECK_LAUNCH();
    return EPG_OK;
}

epg_status epg_accumulate_rows(epg_ctx *ctx, const float *src, const int32_t *ids, int64_t count, int32_t row_floats,
                               float *acc) {
    if (!ctx) return EPG_ERR_STATE;
    if (count < 0 || row_floats <= 0 || (count > 0 && (!src || !ids || !acc)))
        return ctx->fail(EPG_ERR_INPUT, "accumulate_rows: arguments");
    if (count == 0) return EPG_OK;
    CU(cudaSetDevice(ctx->device));
    k_accumulate_rows<<<grid_for(count * row_floats), kThreads, 0, ctx->stream>>>(src, ids, count, row_floats, acc);
    CHECK_LAUNCH();
    return EPG_OK;
}

epg_status epg_remapped_edges(epg_ctx *ctx, const int32_t *edges, int64_t m, const int32_t *edge_perm,
                              const int32_t *vertex_perm, int32_t *out) {
    if (!ctx) return EPG_ERR_STATE;
    if (m <= 0 || !edges || !edge_perm || !vertex_perm || !out)
        return ctx->fail(EPG_ERR_INPUT, "remapped_edges: arguments");
    CU(cudaSetDevice(ctx->device));
    k_remapped_edges<<<grid_for(m), kThreads, 0, ctx->stream>>>(edges, edge_perm, vertex_perm, m, out);
    CHECK_LAUNCH();
    return EPG_OK;
}

epg_status epg_set_variant(epg_ctx *ctx, int32_t variant) {
    if (!ctx) return EPG_ERR_STATE;
    if (variant < 0 || variant > 3)
        return ctx->fail(EPG_ERR_INPUT, "set_variant: 0 auto, 1 per-partition, 2 pipelined, 3 occupancy");
    ctx->variant = variant;
    return EPG_OK;
}

epg_status epg_set_partition_method(epg_ctx *ctx, int32_t method) {
    if (!ctx) return EPG_ERR_STATE;
    if (method != EPG_PARTITION_EPG1 && method != EPG_PARTITION_EPG2 && method != EPG_PARTITION_RB)
        return ctx->fail(EPG_ERR_INPUT, "set_partition_method: 1 (EPG-1), 2 (EPG-2) or 3 (EPG-RB)");
    ctx->partition_method = method;
    return EPG_OK;
}

epg_status epg_set_exec_limits(epg_ctx *ctx, int32_t max_rows, int32_t max_edges) {
    if (!ctx) return EPG_ERR_STATE;
    if (!(max_rows == -1 || (max_rows >= 64 && max_rows <= kOccMaxRowsScalar)) ||
        !(max_edges == -1 || (max_edges >= 32 && max_edges <= kOccMaxEdges)))
        return ctx->fail(EPG_ERR_INPUT, "set_exec_limits: max_rows in [64, 2048], max_edges in [32, 1280], or -1");
    ctx->exec_rows = max_rows;
    ctx->exec_edges = max_edges;
    return EPG_OK;
}

epg_status epg_set_hub_l2(epg_ctx *ctx, int32_t enable) {
    if (!ctx) return EPG_ERR_STATE;
    ctx->hub_l2 = enable != 0;
    return EPG_OK;
}

epg_status epg_set_hub_split(epg_ctx *ctx, int32_t min_halo_entries) {
    if (!ctx) return EPG_ERR_STATE;
    if (min_halo_entries < -1)
        return ctx->fail(EPG_ERR_INPUT, "set_hub_split: min_halo_entries must be >= 0 (0 = off) or -1 (default)");
    ctx->hub_min = min_halo_entries;
    return EPG_OK;
}

int64_t epg_plan_hubs(const epg_plan *plan, int32_t *min_halo_entries) {
    if (!plan) return -1;
    if (min_halo_entries) *min_halo_entries = plan->hub_min;
    return plan->n_hub;
}

epg_status epg_set_profiling(epg_ctx *ctx, int32_t enable) {
    if (!ctx) return EPG_ERR_STATE;
    ctx->profiling = enable != 0;
    return EPG_OK;
}

epg_status epg_profile_read(epg_ctx *ctx, float *ms2, int64_t *launches2) {
    if (!ctx) return EPG_ERR_STATE;
    if (!ms2 || !launches2) return ctx->fail(EPG_ERR_INPUT, "profile_read: NULL output");
    CU(cudaSetDevice(ctx->device));
    CU(cudaStreamSynchronize(ctx->stream));
    ms2[0] = ms2[1] = 0.0f;
    launches2[0] = launches2[1] = 0;
    for (auto &u : ctx->ev_used) {
        float ms = 0.0f;
        CU(cudaEventElapsedTime(&ms, u.second.first, u.second.second));
        ms2[u.first] += ms;
        launches2[u.first] += 1;
        ctx->ev_pool.push_back(u.second.first);
        ctx->ev_pool.push_back(u.second.second);
    }
    ctx->ev_used.clear();
    return EPG_OK;
}

#ifdef EPG_TRACE
// development only (not in epg.h): copy the kernel trace buffer to the host
epg_status epg_debug_trace(unsigned long long *host, int64_t count) {
    cudaMemcpyFromSymbol(host, epg::g_trace, sizeof(unsigned long long) * count);
    return EPG_OK;
}
epg_status epg_debug_trace_clear() {
    void *p = nullptr;
    cudaGetSymbolAddress(&p, epg::g_trace);
    cudaMemset(p, 0, sizeof(epg::g_trace));
    return EPG_OK;
}
#endif

}  // extern "C"


// =====================================================================================
// Multi-GPU execution (SURVEY §8(b) epg_comm_init, §8(e); the paper is single-GPU).
//
// Rank g of G holds the same plan (a map partitioned with shards = G, so shard g owns the
// EP partitions [floor(gk/G), floor((g+1)k/G)) and, by cpack, a contiguous vertex range).
// Per time step (O7): (1) pull -- the owners g' < g send the rows of Halo^{g<-g'}: packed by
// a gather kernel, exchanged with grouped ncclSend/ncclRecv on the ctx stream, scattered into
// state_in; (2) the edge kernel over g's execution partitions; (3) push -- g reduces its halo
// partials of every vertex of Halo^{g<-g'} (fixed order) and sends them to the owner g',
// receiving the same from every g'' > g; the received rows are added to a per-vertex
// accumulator in ascending peer order; (4) the boundary finalise of g's shared vertices
// (local halo partials, then the accumulator) and g's untouched rows. Deterministic for a
// fixed G. The transport is NCCL (one process per GPU) or, for one-GPU tests, an in-process
// group whose "send" is a device copy between the group's contexts (epg_comm_init_local).
// =====================================================================================
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*errorString)(ncclResult_t) = nullptr;
};

// NCCL is resolved at run time (the torch-bundled libnccl.so.2 of this image), so libepg.so
// loads without it and only the multi-GPU calls need it
const NcclApi *nccl_api(std::string *err) {
    static NcclApi api;
    static bool tried = false;
    if (tried) {
        if (!api.h) *err = "NCCL (libnccl.so.2) could not be loaded";
        return api.h ? &api : nullptr;
    }
    tried = true;
    const char *cands[] = {"libnccl.so.2", "libnccl.so",
                           "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2"};
    for (const char *c : cands)
        if ((api.h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!api.h) {
        *err = "NCCL (libnccl.so.2) could not be loaded";
        return nullptr;
    }
#define NSYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(api.h, name))
    NSYM(getUniqueId, "ncclGetUniqueId");
    NSYM(commInitRank, "ncclCommInitRank");
    NSYM(commDestroy, "ncclCommDestroy");
    NSYM(groupStart, "ncclGroupStart");
    NSYM(groupEnd, "ncclGroupEnd");
    NSYM(send, "ncclSend");
    NSYM(recv, "ncclRecv");
    NSYM(allGather, "ncclAllGather");
    NSYM(errorString, "ncclGetErrorString");
#undef NSYM
    if (!api.getUniqueId || !api.commInitRank || !api.commDestroy || !api.groupStart || !api.groupEnd || !api.send ||
        !api.recv || !api.errorString) {
        *err = "NCCL: missing symbols in libnccl.so.2";
        api.h = nullptr;
        return nullptr;
    }
    return &api;
}

struct LocalGroup;   // in-process group (one-GPU tests)

struct Comm {
    int nranks = 1, rank = 0;
    ncclComm_t nccl = nullptr;
    LocalGroup *local = nullptr;
};

struct LocalGroup {
    std::vector<epg_ctx *> ctxs;
};

// exchange buffers and lists of one plan on one rank (built on the first sharded step)
struct ShardState {
    const epg_plan *plan = nullptr;
    int G = 1, g = 0, row = 0;
    int64_t xf = 0, xc = 0, hf = 0, hc = 0, sf = 0, sc = 0;
    // per peer: rows this rank receives in the pull (p < g) / sends (p > g), offsets into
    // the concatenated id lists; the same lists carry the push in the other direction
    std::vector<int64_t> recv_off, send_off;     // [G + 1]
    int32_t *recv_ids = nullptr, *send_ids = nullptr;
    float *pull_send = nullptr, *pull_recv = nullptr, *push_send = nullptr, *push_recv = nullptr, *acc = nullptr;
    int4 *recs = nullptr;     // finalise records of the shard's shared vertices (local halo entries only)
    int32_t *acc_ids = nullptr;   // distinct vertices other ranks push partial sums for
    int64_t acc_count = 0;
    // the shard's execution partitions, interior ones first (no halo row owned by a lower
    // rank: they need nothing from the pull and run while it is in flight), then the boundary
    int32_t *order = nullptr;
    int64_t n_interior = 0;
    // NCCL: the exchanges run on a stream of their own, ordered against the ctx stream by events
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // peer push (EPG_EXCHANGE=p2p): the boundary edge kernel adds the partials of foreign vertices
    // straight into their owners' accumulators (peer memory); a 1-float token per push pair then
    // orders the owner's accumulate-add after the pushers' kernels
    bool p2p = false;
    float **peer_acc = nullptr;   // DEVICE [G] accumulators of the ranks (peer-mapped)
    int32_t *vlo = nullptr;       // DEVICE [G + 1] first cpack row of each rank's shard
    float *tok = nullptr;         // [2 G] token send / receive slots
    std::vector<void *> ipc_opened;
    std::vector<void *> allocs;
    ~ShardState() {
        for (void *p : ipc_opened) cudaIpcCloseMemHandle(p);
        for (void *p : allocs) cudaFree(p);
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
        if (comm_stream) cudaStreamDestroy(comm_stream);
    }
};

namespace {

void *shard_alloc(ShardState *S, size_t bytes, cudaError_t *e) {
    void *p = nullptr;
    *e = cudaMalloc(&p, std::max<size_t>(bytes, 16));
    if (*e == cudaSuccess) S->allocs.push_back(p);
    return p;
}

std::map<std::pair<const epg_ctx *, const epg_plan *>, ShardState *> &shard_states() {
    static std::map<std::pair<const epg_ctx *, const epg_plan *>, ShardState *> m;
    return m;
}

// shard state of (ctx, plan) for the ctx's group; built once
epg_status shard_state(epg_ctx *ctx, epg_plan *pl, int row, ShardState **out) {
    auto key = std::make_pair((const epg_ctx *)ctx, (const epg_plan *)pl);
    auto it = shard_states().find(key);
    if (it != shard_states().end() && it->second->row == row) {
        *out = it->second;
        return EPG_OK;
    }
    if (it != shard_states().end()) {
        delete it->second;
        shard_states().erase(it);
    }
    const int G = ctx->comm ? ctx->comm->nranks : 1, g = ctx->comm ? ctx->comm->rank : 0;
    if (G > pl->k_ep) return ctx->fail(EPG_ERR_INFEASIBLE, "run_sharded: more ranks than EP partitions");
    std::unique_ptr<ShardState> S(new ShardState());
    S->plan = pl;
    S->G = G;
    S->g = g;
    S->row = row;
    int64_t r8[8];
    epg_status st = epg_shard_ranges(pl, G, g, r8);
    if (st) return ctx->fail(st, "run_sharded: shard ranges");
    S->xf = r8[0]; S->xc = r8[1]; S->hf = r8[2]; S->hc = r8[3]; S->sf = r8[6]; S->sc = r8[7];
    // O7 halo sets from the EP layout (the execution plan keeps the EP partitions' first
    // touches, so the shard ranges of the EP map and of the execution map agree)
    std::vector<int32_t> hid(pl->C);
    if (pl->C > 0) CU(cudaMemcpy(hid.data(), pl->halo_ids, sizeof(int32_t) * pl->C, cudaMemcpyDeviceToHost));
    std::vector<int32_t> pvb_ep(pl->k_ep + 1), hb_ep(pl->k_ep + 1);
    for (int64_t p = 0; p <= pl->k_ep; p++) {
        pvb_ep[p] = pl->pvb_h[pl->exec_base[p]];
        hb_ep[p] = pl->hb_h[pl->exec_base[p]];
    }
    std::vector<int32_t> begin(G * G + 1);
    int64_t cnt = 0;
    if ((st = epg_shard_halos_host(pvb_ep.data(), hb_ep.data(), hid.data(), pl->k_ep, G, begin.data(), nullptr, 0, &cnt)))
        return ctx->fail(st, "run_sharded: halo sets");
    std::vector<int32_t> ids(std::max<int64_t>(cnt, 1));
    if ((st = epg_shard_halos_host(pvb_ep.data(), hb_ep.data(), hid.data(), pl->k_ep, G, begin.data(), ids.data(),
                                   (int64_t)ids.size(), &cnt)))
        return ctx->fail(st, "run_sharded: halo sets");
    std::vector<int32_t> rl, sl;
    S->recv_off.assign(G + 1, 0);
    S->send_off.assign(G + 1, 0);
    for (int p = 0; p < G; p++) {
        S->recv_off[p] = (int64_t)rl.size();
        if (p < g) rl.insert(rl.end(), ids.begin() + begin[g * G + p], ids.begin() + begin[g * G + p + 1]);
        S->send_off[p] = (int64_t)sl.size();
        if (p > g) sl.insert(sl.end(), ids.begin() + begin[p * G + g], ids.begin() + begin[p * G + g + 1]);
    }
    S->recv_off[G] = (int64_t)rl.size();
    S->send_off[G] = (int64_t)sl.size();
    cudaError_t e;
    const size_t rb = sizeof(float) * row;
    S->recv_ids = (int32_t *)shard_alloc(S.get(), sizeof(int32_t) * rl.size(), &e);
    if (e == cudaSuccess) S->send_ids = (int32_t *)shard_alloc(S.get(), sizeof(int32_t) * sl.size(), &e);
    if (e == cudaSuccess) S->pull_send = (float *)shard_alloc(S.get(), rb * sl.size(), &e);
    if (e == cudaSuccess) S->pull_recv = (float *)shard_alloc(S.get(), rb * rl.size(), &e);
    if (e == cudaSuccess) S->push_send = (float *)shard_alloc(S.get(), rb * rl.size(), &e);
    if (e == cudaSuccess) S->push_recv = (float *)shard_alloc(S.get(), rb * sl.size(), &e);
    if (e == cudaSuccess) S->acc = (float *)shard_alloc(S.get(), rb * pl->n, &e);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return ctx->fail(EPG_ERR_NOMEM, "run_sharded: exchange buffers");
    }
    if (!rl.empty()) CU(cudaMemcpy(S->recv_ids, rl.data(), sizeof(int32_t) * rl.size(), cudaMemcpyHostToDevice));
    if (!sl.empty()) CU(cudaMemcpy(S->send_ids, sl.data(), sizeof(int32_t) * sl.size(), cudaMemcpyHostToDevice));
    {
        std::vector<int32_t> u(sl);
        std::sort(u.begin(), u.end());
        u.erase(std::unique(u.begin(), u.end()), u.end());
        S->acc_count = (int64_t)u.size();
        S->acc_ids = (int32_t *)shard_alloc(S.get(), sizeof(int32_t) * u.size(), &e);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return ctx->fail(EPG_ERR_NOMEM, "run_sharded: exchange buffers");
        }
        if (!u.empty()) CU(cudaMemcpy(S->acc_ids, u.data(), sizeof(int32_t) * u.size(), cudaMemcpyHostToDevice));
    }
    CU(cudaMemset(S->acc, 0, rb * pl->n));
    if (S->sc > 0) {   // packed records {v, count, h0..h5} when no shared vertex has > 6 local entries
        int4 *recs = (int4 *)shard_alloc(S.get(), sizeof(int4) * 2 * S->sc, &e);
        int32_t *hm = (int32_t *)shard_alloc(S.get(), 2 * sizeof(int32_t), &e);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return ctx->fail(EPG_ERR_NOMEM, "run_sharded: finalise records");
        }
        CU(cudaMemset(hm, 0, 2 * sizeof(int32_t)));
        k_shard_records<<<grid_for(S->sc), kThreads>>>(pl->shared_ids + S->sf, pl->hv_off + S->sf, pl->hv_list,
                                                       (int32_t)S->sc, S->hf, S->hf + S->hc, recs, hm);
        CU(cudaGetLastError());
        int32_t hmax = 0;
        CU(cudaMemcpy(&hmax, hm, sizeof(int32_t), cudaMemcpyDeviceToHost));
        if (hmax <= 6) S->recs = recs;
    }
    {   // interior / boundary split of the shard's execution partitions (ids in the plan's
        // halo lists are cpack ids; a lower rank owns exactly the ids below the shard's first row)
        std::vector<int32_t> xh;
        const int64_t h0 = pl->hb_h[S->xf], h1 = pl->hb_h[S->xf + S->xc];
        if (h1 > h0) {
            xh.resize(h1 - h0);
            CU(cudaMemcpy(xh.data(), pl->halo_ids + h0, sizeof(int32_t) * (h1 - h0), cudaMemcpyDeviceToHost));
        }
        const int32_t v_lo = pl->pvb_h[S->xf];
        std::vector<int32_t> inner, outer;
        for (int64_t x = S->xf; x < S->xf + S->xc; x++) {
            bool foreign = false;
            for (int64_t q = pl->hb_h[x]; q < pl->hb_h[x + 1] && !foreign; q++) foreign = xh[q - h0] < v_lo;
            (foreign ? outer : inner).push_back((int32_t)x);
        }
        S->n_interior = (int64_t)inner.size();
        inner.insert(inner.end(), outer.begin(), outer.end());
        S->order = (int32_t *)shard_alloc(S.get(), sizeof(int32_t) * inner.size(), &e);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return ctx->fail(EPG_ERR_NOMEM, "run_sharded: partition order");
        }
        if (!inner.empty())
            CU(cudaMemcpy(S->order, inner.data(), sizeof(int32_t) * inner.size(), cudaMemcpyHostToDevice));
    }
    if (ctx->comm && ctx->comm->nccl && G > 1) {
        CU(cudaStreamCreateWithFlags(&S->comm_stream, cudaStreamNonBlocking));
        for (cudaEvent_t &ev : S->ev) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    {
        const char *xe = std::getenv("EPG_EXCHANGE");
        S->p2p = G > 1 && xe && std::string(xe) == "p2p";
    }
    if (S->p2p) {
        std::vector<int32_t> vl(G + 1);
        for (int p = 0; p < G; p++) {
            int64_t q8[8];
            if ((st = epg_shard_ranges(pl, G, p, q8))) return ctx->fail(st, "run_sharded: shard ranges");
            vl[p] = (int32_t)q8[4];
            vl[p + 1] = (int32_t)(q8[4] + q8[5]);
        }
        S->vlo = (int32_t *)shard_alloc(S.get(), sizeof(int32_t) * (G + 1), &e);
        if (e == cudaSuccess) S->peer_acc = (float **)shard_alloc(S.get(), sizeof(float *) * G, &e);
        if (e == cudaSuccess) S->tok = (float *)shard_alloc(S.get(), sizeof(float) * 2 * G, &e);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return ctx->fail(EPG_ERR_NOMEM, "run_sharded: peer tables");
        }
        CU(cudaMemcpy(S->vlo, vl.data(), sizeof(int32_t) * (G + 1), cudaMemcpyHostToDevice));
        CU(cudaMemset(S->tok, 0, sizeof(float) * 2 * G));
        if (ctx->comm && ctx->comm->nccl) {   // exchange the accumulators' IPC handles
            std::string err;
            const NcclApi *n = nccl_api(&err);
            if (!n) return ctx->fail(EPG_ERR_NCCL, err);
            cudaIpcMemHandle_t mine;
            CU(cudaIpcGetMemHandle(&mine, S->acc));
            Tmp hd(ctx);
            CU(hd.alloc(sizeof(cudaIpcMemHandle_t) * G));
            CU(cudaMemcpy(static_cast<char *>(hd.p) + sizeof(cudaIpcMemHandle_t) * g, &mine, sizeof(mine),
                          cudaMemcpyHostToDevice));
            ncclResult_t r = n->allGather(static_cast<char *>(hd.p) + sizeof(cudaIpcMemHandle_t) * g, hd.p,
                                          sizeof(cudaIpcMemHandle_t), ncclChar, ctx->comm->nccl, ctx->stream);
            if (r != ncclSuccess) return ctx->fail(EPG_ERR_NCCL, std::string("run_sharded: ") + n->errorString(r));
            std::vector<cudaIpcMemHandle_t> hs(G);
            CU(cudaMemcpyAsync(hs.data(), hd.p, sizeof(cudaIpcMemHandle_t) * G, cudaMemcpyDeviceToHost, ctx->stream));
            CU(cudaStreamSynchronize(ctx->stream));
            std::vector<float *> tab(G, nullptr);
            for (int p = 0; p < G; p++) {
                if (p == g) {
                    tab[p] = S->acc;
                    continue;
                }
                void *q = nullptr;
                CU(cudaIpcOpenMemHandle(&q, hs[p], cudaIpcMemLazyEnablePeerAccess));
                S->ipc_opened.push_back(q);
                tab[p] = static_cast<float *>(q);
            }
            CU(cudaMemcpy(S->peer_acc, tab.data(), sizeof(float *) * G, cudaMemcpyHostToDevice));
        }   // in-process groups: run_group_t fills the table with the members' accumulators
    }
    *out = S.release();
    shard_states()[key] = *out;
    return EPG_OK;
}

// rows of `ids` (rows of `row` floats) gathered from / scattered into `state`
epg_status rows_move(epg_ctx *ctx, const float *src, float *dst, const int32_t *ids, int64_t count, int row,
                     int scatter) {
    if (count <= 0) return EPG_OK;
    k_permute_rows<<<grid_for(count * row), kThreads, 0, ctx->stream>>>(
        reinterpret_cast<const uint32_t *>(src), reinterpret_cast<uint32_t *>(dst), count, row, ids, scatter);
    CHECK_LAUNCH();
    return EPG_OK;
}

// the grouped point-to-point exchange of one phase: send[p] to every p in `to`, receive
// recv[p] from every p in `from` (rows of `row` floats)
epg_status exchange(epg_ctx *ctx, ShardState *S, const float *send, const std::vector<int64_t> &send_off,
                    float *recv, const std::vector<int64_t> &recv_off, cudaStream_t stream) {
    const int G = S->G, row = S->row;
    Comm *c = ctx->comm;
    if (G == 1) return EPG_OK;
    if (c->nccl) {
        std::string err;
        const NcclApi *n = nccl_api(&err);
        if (!n) return ctx->fail(EPG_ERR_NCCL, err);
        ncclResult_t r = n->groupStart();
        for (int p = 0; p < G && r == ncclSuccess; p++) {
            const int64_t sc = send_off[p + 1] - send_off[p], rc = recv_off[p + 1] - recv_off[p];
            if (sc > 0) r = n->send(send + row * send_off[p], (size_t)(row * sc), ncclFloat, p, c->nccl, stream);
            if (r == ncclSuccess && rc > 0)
                r = n->recv(recv + row * recv_off[p], (size_t)(row * rc), ncclFloat, p, c->nccl, stream);
        }
        ncclResult_t r2 = n->groupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess)
            return ctx->fail(EPG_ERR_NCCL, std::string("run_sharded: ") + n->errorString(r != ncclSuccess ? r : r2));
        return EPG_OK;
    }
    return EPG_OK;   // in-process groups exchange in run_sharded_group
}

// peer push: after this rank's boundary edge kernel, one float to every owner it pushed to
// (p < g) and one from every rank that pushed to it (p > g) -- stream-ordered, so a received
// token means the pusher's kernel (and its peer atomics) completed
epg_status exchange_token(epg_ctx *ctx, ShardState *S, cudaStream_t stream) {
    const int G = S->G, g = S->g;
    Comm *c = ctx->comm;
    if (G == 1 || !c || !c->nccl) return EPG_OK;
    std::string err;
    const NcclApi *n = nccl_api(&err);
    if (!n) return ctx->fail(EPG_ERR_NCCL, err);
    ncclResult_t r = n->groupStart();
    for (int p = 0; p < G && r == ncclSuccess; p++) {
        if (p < g && S->recv_off[p + 1] > S->recv_off[p]) r = n->send(S->tok + p, 1, ncclFloat, p, c->nccl, stream);
        if (r == ncclSuccess && p > g && S->send_off[p + 1] > S->send_off[p])
            r = n->recv(S->tok + G + p, 1, ncclFloat, p, c->nccl, stream);
    }
    ncclResult_t r2 = n->groupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
        return ctx->fail(EPG_ERR_NCCL, std::string("run_sharded: ") + n->errorString(r != ncclSuccess ? r : r2));
    return EPG_OK;
}

template <class Fn>
epg_status sharded_pull_pack(epg_ctx *ctx, ShardState *S, const float *state_in) {
    return rows_move(ctx, state_in, S->pull_send, S->send_ids, S->send_off[S->G], Fn::ROW, 0);
}
template <class Fn>
epg_status sharded_pull_unpack(epg_ctx *ctx, ShardState *S, float *state_in) {
    return rows_move(ctx, S->pull_recv, state_in, S->recv_ids, S->recv_off[S->G], Fn::ROW, 1);
}
template <class Fn>
epg_status sharded_push_pack(epg_ctx *ctx, epg_plan *pl, ShardState *S) {
    const int64_t cnt = S->recv_off[S->G];
    if (cnt <= 0) return EPG_OK;
    k_shard_reduce<Fn><<<grid_for(cnt), kThreads, 0, ctx->stream>>>(S->recv_ids, cnt, pl->sidx, pl->hv_off, pl->hv_list,
                                                                     pl->halo_buf, S->hf, S->hf + S->hc, S->push_send);
    CHECK_LAUNCH();
    return EPG_OK;
}
template <class Fn>
epg_status sharded_push_accumulate(epg_ctx *ctx, ShardState *S) {
    for (int p = S->g + 1; p < S->G; p++) {   // ascending peer order: a fixed summation order
        const int64_t c = S->send_off[p + 1] - S->send_off[p];
        if (c <= 0) continue;
        k_accumulate_rows<<<grid_for(c * Fn::ROW), kThreads, 0, ctx->stream>>>(
            S->push_recv + Fn::ROW * S->send_off[p], S->send_ids + S->send_off[p], c, Fn::ROW, S->acc);
        CHECK_LAUNCH();
    }
    return EPG_OK;
}

// finalise of the shard: its shared vertices from the packed local records (or the ranged
// kernel), then the pushed partial sums of the vertices other ranks share, then untouched rows
template <class Fn>
epg_status sharded_finalise_local(epg_ctx *ctx, epg_plan *pl, ShardState *S, epg_state *st) {
    const float *in = static_cast<const float *>(st->state_in);
    float *out = static_cast<float *>(st->state_out);
    const float *vc = static_cast<const float *>(st->vertex_const);
    const int64_t work = S->sc + (pl->n - pl->touched);
    if (work > 0)
        CU(launch_pdl(k_finalise_rec<Fn>, grid_for(work), kThreads, 0, ctx->stream, (const int4 *)S->recs,
                      (const float *)pl->halo_buf, in, out, vc, (int32_t)S->sc, pl->touched, pl->n));
    return EPG_OK;
}
template <class Fn>
epg_status sharded_acc_add(epg_ctx *ctx, ShardState *S, epg_state *st) {
    const int64_t cnt = S->acc_count;
    if (cnt > 0) {
        k_acc_add<Fn><<<grid_for(cnt), kThreads, 0, ctx->stream>>>(S->acc_ids, cnt, S->acc,
                                                                   static_cast<float *>(st->state_out),
                                                                   static_cast<const float *>(st->vertex_const));
        CHECK_LAUNCH();
    }
    return EPG_OK;
}
template <class Fn>
epg_status sharded_finalise(epg_ctx *ctx, epg_plan *pl, ShardState *S, epg_state *st) {
    if (!S->recs) return run_finalise_range<Fn>(ctx, pl, st, S->sf, S->sc, S->hf, S->hc, S->acc, 1);
    epg_status e = sharded_finalise_local<Fn>(ctx, pl, S, st);
    return e ? e : sharded_acc_add<Fn>(ctx, S, st);
}

template <class Fn>
epg_status run_sharded_t(epg_ctx *ctx, epg_plan *pl, epg_state *state, int32_t steps) {
    ShardState *S = nullptr;
    epg_status st = shard_state(ctx, pl, Fn::ROW, &S);
    if (st) return st;
    float *bufs[2] = {static_cast<float *>(state->state_in), static_cast<float *>(state->state_out)};
    // with a comm stream the exchanges overlap the ctx stream's work:
    //   ctx:  pack | interior edges .............. | unpack, boundary edges, push pack | local finalise ...... | accumulate
    //   comm:       (wait ev0) pull exchange (ev1) |                        (wait ev2) push exchange (ev3) |
    // the kernels and their order on the ctx stream are the sequential schedule's, so the result
    // is bit-identical to it (same partitions, same summation orders)
    cudaStream_t cs = S->comm_stream ? S->comm_stream : ctx->stream;
    auto fork = [&](int e) -> epg_status {
        if (!S->comm_stream) return EPG_OK;
        CU(cudaEventRecord(S->ev[e], ctx->stream));
        CU(cudaStreamWaitEvent(S->comm_stream, S->ev[e], 0));
        return EPG_OK;
    };
    auto join = [&](int e) -> epg_status {
        if (!S->comm_stream) return EPG_OK;
        CU(cudaEventRecord(S->ev[e], S->comm_stream));
        CU(cudaStreamWaitEvent(ctx->stream, S->ev[e], 0));
        return EPG_OK;
    };
    const int64_t nb = S->xc - S->n_interior;
    for (int32_t s = 0; s < steps; s++) {
        epg_state cur = *state;
        cur.state_in = bufs[s & 1];
        cur.state_out = bufs[(s + 1) & 1];
        float *in = static_cast<float *>(cur.state_in);
        if ((st = sharded_pull_pack<Fn>(ctx, S, in)) || (st = fork(0)) ||
            (st = exchange(ctx, S, S->pull_send, S->send_off, S->pull_recv, S->recv_off, cs)) ||
            (st = run_edges_range<Fn>(ctx, pl, &cur, 0, S->n_interior, S->order)) || (st = join(1)) ||
            (st = sharded_pull_unpack<Fn>(ctx, S, in)))
            return st;
        if (S->p2p) {   // the boundary kernel pushes foreign partials into the owners' accumulators
            if ((st = run_edges_range<Fn>(ctx, pl, &cur, S->n_interior, nb, S->order, S->peer_acc, S->vlo, S->g)) ||
                (st = fork(2)) || (st = exchange_token(ctx, S, cs)))
                return st;
            if (S->recs) {
                if ((st = sharded_finalise_local<Fn>(ctx, pl, S, &cur)) || (st = join(3)) ||
                    (st = sharded_acc_add<Fn>(ctx, S, &cur)))
                    return st;
            } else if ((st = join(3)) || (st = sharded_finalise<Fn>(ctx, pl, S, &cur))) {
                return st;
            }
            continue;
        }
        if ((st = run_edges_range<Fn>(ctx, pl, &cur, S->n_interior, nb, S->order)) ||
            (st = sharded_push_pack<Fn>(ctx, pl, S)) || (st = fork(2)) ||
            (st = exchange(ctx, S, S->push_send, S->recv_off, S->push_recv, S->send_off, cs)))
            return st;
        if (S->recs) {   // the local finalise needs nothing from the push: it runs while that is in flight
            if ((st = sharded_finalise_local<Fn>(ctx, pl, S, &cur)) || (st = join(3)) ||
                (st = sharded_push_accumulate<Fn>(ctx, S)) || (st = sharded_acc_add<Fn>(ctx, S, &cur)))
                return st;
        } else if ((st = join(3)) || (st = sharded_push_accumulate<Fn>(ctx, S)) ||
                   (st = sharded_finalise<Fn>(ctx, pl, S, &cur))) {
            return st;
        }
    }
    return EPG_OK;
}

// one step of every member of an in-process group, phase by phase; the "transfers" are
// device copies between the members' buffers ordered by events (one GPU, tests)
template <class Fn>
epg_status run_group_t(epg_ctx **ctxs, epg_plan **plans, epg_state *states, int G) {
    std::vector<ShardState *> S(G);
    for (int g = 0; g < G; g++) {
        epg_status st = shard_state(ctxs[g], plans[g], Fn::ROW, &S[g]);
        if (st) return st;
    }
    const bool p2p = S[0]->p2p;
    if (p2p) {   // the members' accumulators are the "peer" memory (one device)
        std::vector<float *> tab(G);
        for (int g = 0; g < G; g++) tab[g] = S[g]->acc;
        for (int g = 0; g < G; g++) CU_NOCTX(cudaMemcpy(S[g]->peer_acc, tab.data(), sizeof(float *) * G,
                                                         cudaMemcpyHostToDevice));
    }
    std::vector<cudaEvent_t> ev(G);
    for (int g = 0; g < G; g++) cudaEventCreateWithFlags(&ev[g], cudaEventDisableTiming);
    auto sync_all = [&]() {
        for (int g = 0; g < G; g++) cudaEventRecord(ev[g], ctxs[g]->stream);
        for (int g = 0; g < G; g++)
            for (int p = 0; p < G; p++) cudaStreamWaitEvent(ctxs[g]->stream, ev[p], 0);
    };
    // copies of one phase: member g receives from p the rows p sends to g
    auto copy_phase = [&](bool pull) {
        for (int g = 0; g < G; g++)
            for (int p = 0; p < G; p++) {
                ShardState *R = S[g], *T = S[p];
                // pull: p > ... p sends pull_send[p][g] to g (p < g); push: p sends push_send[p][g] to g (p > g)
                const int64_t rc = pull ? R->recv_off[p + 1] - R->recv_off[p] : R->send_off[p + 1] - R->send_off[p];
                if (rc <= 0) continue;
                const float *src = pull ? T->pull_send + Fn::ROW * T->send_off[g] : T->push_send + Fn::ROW * T->recv_off[g];
                float *dst = pull ? R->pull_recv + Fn::ROW * R->recv_off[p] : R->push_recv + Fn::ROW * R->send_off[p];
                cudaMemcpyAsync(dst, src, sizeof(float) * Fn::ROW * rc, cudaMemcpyDeviceToDevice, ctxs[g]->stream);
            }
    };
    epg_status st = EPG_OK;
    for (int g = 0; g < G && !st; g++) st = sharded_pull_pack<Fn>(ctxs[g], S[g], (const float *)states[g].state_in);
    sync_all();
    for (int g = 0; g < G && !st; g++)   // interior partitions: nothing from the pull
        st = run_edges_range<Fn>(ctxs[g], plans[g], &states[g], 0, S[g]->n_interior, S[g]->order);
    copy_phase(true);
    sync_all();
    for (int g = 0; g < G && !st; g++) {
        if ((st = sharded_pull_unpack<Fn>(ctxs[g], S[g], (float *)states[g].state_in))) break;
        if (p2p) {
            st = run_edges_range<Fn>(ctxs[g], plans[g], &states[g], S[g]->n_interior, S[g]->xc - S[g]->n_interior,
                                     S[g]->order, S[g]->peer_acc, S[g]->vlo, g);
            continue;
        }
        if ((st = run_edges_range<Fn>(ctxs[g], plans[g], &states[g], S[g]->n_interior, S[g]->xc - S[g]->n_interior,
                                      S[g]->order)))
            break;
        st = sharded_push_pack<Fn>(ctxs[g], plans[g], S[g]);
    }
    sync_all();
    if (!p2p) {
        copy_phase(false);
        sync_all();
    }
    for (int g = 0; g < G && !st; g++) {
        if (!p2p && (st = sharded_push_accumulate<Fn>(ctxs[g], S[g]))) break;
        st = sharded_finalise<Fn>(ctxs[g], plans[g], S[g], &states[g]);
    }
    sync_all();
    for (int g = 0; g < G; g++) cudaEventDestroy(ev[g]);
    return st;
}

}  // namespace

void comm_release(epg_ctx *ctx) {
    for (auto it = shard_states().begin(); it != shard_states().end();) {
        if (it->first.first == ctx) {
            delete it->second;
            it = shard_states().erase(it);
        } else {
            ++it;
        }
    }
    if (!ctx->comm) return;
    if (ctx->comm->nccl) {
        std::string err;
        if (const NcclApi *n = nccl_api(&err)) n->commDestroy(ctx->comm->nccl);
    }
    if (ctx->comm->local) {   // the group's members share it; the last one frees it
        auto &v = ctx->comm->local->ctxs;
        v.erase(std::remove(v.begin(), v.end(), ctx), v.end());
        if (v.empty()) delete ctx->comm->local;
    }
    delete ctx->comm;
    ctx->comm = nullptr;
}

extern "C" {

epg_status epg_comm_unique_id(void *id_out) {
    if (!id_out) return EPG_ERR_INPUT;
    std::string err;
    const NcclApi *n = nccl_api(&err);
    if (!n) return EPG_ERR_NCCL;
    ncclUniqueId id;
    if (n->getUniqueId(&id) != ncclSuccess) return EPG_ERR_NCCL;
    std::memcpy(id_out, &id, sizeof(id));
    return EPG_OK;
}

epg_status epg_comm_init(epg_ctx *ctx, const void *nccl_unique_id, int32_t nranks, int32_t rank) {
    if (!ctx) return EPG_ERR_STATE;
    if (!nccl_unique_id || nranks < 1 || rank < 0 || rank >= nranks)
        return ctx->fail(EPG_ERR_INPUT, "comm_init: need a unique id, nranks >= 1 and 0 <= rank < nranks");
    CU(cudaSetDevice(ctx->device));
    std::string err;
    const NcclApi *n = nccl_api(&err);
    if (!n) return ctx->fail(EPG_ERR_NCCL, err);
    comm_release(ctx);
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof(id));
    ncclComm_t c = nullptr;
    ncclResult_t r = n->commInitRank(&c, nranks, id, rank);
    if (r != ncclSuccess) return ctx->fail(EPG_ERR_NCCL, std::string("comm_init: ") + n->errorString(r));
    ctx->comm = new Comm();
    ctx->comm->nranks = nranks;
    ctx->comm->rank = rank;
    ctx->comm->nccl = c;
    return EPG_OK;
}

epg_status epg_comm_init_local(epg_ctx *const *ctxs, int32_t nranks) {
    if (!ctxs || nranks < 1) return EPG_ERR_INPUT;
    for (int g = 0; g < nranks; g++)
        if (!ctxs[g]) return EPG_ERR_INPUT;
    LocalGroup *grp = new LocalGroup();
    for (int g = 0; g < nranks; g++) {
        comm_release(ctxs[g]);
        ctxs[g]->comm = new Comm();
        ctxs[g]->comm->nranks = nranks;
        ctxs[g]->comm->rank = g;
        ctxs[g]->comm->local = grp;
        grp->ctxs.push_back(ctxs[g]);
    }
    return EPG_OK;
}

epg_status epg_run_sharded(epg_ctx *ctx, const epg_plan *plan, epg_kernel kernel, epg_state *state, int32_t steps) {
    if (!ctx) return EPG_ERR_STATE;
    if (!plan || plan->ctx != ctx) return ctx->fail(EPG_ERR_STATE, "run_sharded: plan belongs to another context");
    if (ctx->comm && ctx->comm->local && ctx->comm->nranks > 1)
        return ctx->fail(EPG_ERR_STATE, "run_sharded: an in-process group runs through epg_run_sharded_group");
    epg_status st = check_state(ctx, kernel, state);
    if (st) return st;
    if (steps < 0) return ctx->fail(EPG_ERR_INPUT, "run_sharded: steps < 0");
    CU(cudaSetDevice(ctx->device));
    epg_plan *pl = const_cast<epg_plan *>(plan);
    switch (kernel) {
        case EPG_KERNEL_CFD_FLUX: return run_sharded_t<CfdFlux>(ctx, pl, state, steps);
        case EPG_KERNEL_GATHER_SCATTER: return run_sharded_t<GatherScatter>(ctx, pl, state, steps);
        default: return run_sharded_t<Spmv>(ctx, pl, state, steps);
    }
}

epg_status epg_run_sharded_group(epg_ctx *const *ctxs, const epg_plan *const *plans, epg_kernel kernel,
                                 epg_state *states, int32_t nranks) {
    if (!ctxs || !plans || !states || nranks < 1) return EPG_ERR_INPUT;
    for (int g = 0; g < nranks; g++) {
        if (!ctxs[g] || !plans[g] || plans[g]->ctx != ctxs[g] || !ctxs[g]->comm || ctxs[g]->comm->rank != g ||
            ctxs[g]->comm->nranks != nranks || !ctxs[g]->comm->local)
            return EPG_ERR_STATE;
        epg_status st = check_state(ctxs[g], kernel, &states[g]);
        if (st) return st;
    }
    std::vector<epg_ctx *> c(ctxs, ctxs + nranks);
    std::vector<epg_plan *> p(nranks);
    for (int g = 0; g < nranks; g++) p[g] = const_cast<epg_plan *>(plans[g]);
    CU_NOCTX(cudaSetDevice(ctxs[0]->device));
    switch (kernel) {
        case EPG_KERNEL_CFD_FLUX: return run_group_t<CfdFlux>(c.data(), p.data(), states, nranks);
        case EPG_KERNEL_GATHER_SCATTER: return run_group_t<GatherScatter>(c.data(), p.data(), states, nranks);
        default: return run_group_t<Spmv>(c.data(), p.data(), states, nranks);
    }
}

}  // extern "C"
