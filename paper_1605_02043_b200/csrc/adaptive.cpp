// adaptive.cpp -- adaptive overhead control, the
// paper's runtime policy around the transformed kernel, built on the public ABI:
//
//   * "we perform data sharing optimization using a separate thread on the CPU while
//     kernel is executed on the GPU": epg_adaptive_create starts host EPG-1 on
//     a std::thread and the steps run the original kernel (epg_run_naive: original task
//     order, global-memory operands) meanwhile;
//   * "We check if the asynchronous optimization is completed before calling the kernel
//     and apply the optimization if so": before every step;
//   * "we record the transformed kernel runtime the first time it runs, and compare it
//     with the original kernel runtime. If the first run of the transformed kernel is
//     slower, then we fall back to the original kernel in the next iteration":
//     the first EP step is timed with CUDA events against the median timed original step;
//   * "If the optimization thread does not complete when the program finishes, we
//     terminate it to guarantee no slowdown": epg_adaptive_destroy cancels
//     the partition thread (polled once per partition) and joins it.
//
// The executor owns its state buffers; the state lives in the layout of the kernel in
// use (original order, or the EP plan's cpack order) and epg_adaptive_read_state returns
// it in original vertex order. Every step, in either phase, advances the same time
// step of the functor, so switching (or falling back) never changes the result beyond
// fp32 summation order (none for integer-valued data).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "epg_internal.h"

struct epg_adaptive {
    epg_ctx *ctx = nullptr;
    cudaStream_t stream = nullptr;
    epg_kernel kernel = EPG_KERNEL_CFD_FLUX;
    int64_t m = 0;
    int32_t n = 0, part_size = 0, row = 1, pw = 0;
    double fallback_ratio = 1.0;
    // inputs (owned copies)
    std::vector<int32_t> edges_h;
    int32_t *edges_d = nullptr;
    float *payload_o = nullptr, *vconst_o = nullptr;   // original orders (or NULL)
    float *state[2] = {nullptr, nullptr};
    int cur = 0;
    // the partition thread
    std::thread worker;
    std::atomic<int> done{0}, cancel{0};
    epg_status part_status = EPG_OK;
    std::string part_err;
    std::vector<int32_t> part_h;
    double part_seconds = 0.0;
    // EP phase
    epg_plan *plan = nullptr;
    int32_t *vertex_perm = nullptr;
    float *payload_ep = nullptr, *vconst_ep = nullptr;
    // policy
    int32_t phase = EPG_ADAPTIVE_ORIGINAL;
    int64_t steps_original = 0, steps_ep = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> orig_ev;   // ring of timed original steps
    int64_t orig_timed = 0;
    double original_ms = 0.0, ep_first_ms = 0.0;

    ~epg_adaptive() {
        cancel.store(1);
        if (worker.joinable()) worker.join();
        if (plan) epg_plan_destroy(plan);
        for (void *p : {(void *)edges_d, (void *)payload_o, (void *)vconst_o, (void *)state[0], (void *)state[1],
                        (void *)vertex_perm, (void *)payload_ep, (void *)vconst_ep})
            if (p) cudaFree(p);
        for (auto &e : orig_ev) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
    }
};

namespace {

constexpr int kTimedRing = 8;

#define ACU(call)                                                                                     \
    do {                                                                                              \
        cudaError_t _e = (call);                                                                      \
        if (_e != cudaSuccess)                                                                        \
            return epg::ctx_fail(ad->ctx, EPG_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

epg_state make_state(epg_adaptive *ad, bool ep) {
    epg_state st{};
    st.state_in = ad->state[ad->cur];
    st.state_out = ad->state[ad->cur ^ 1];
    st.edge_payload = ep ? ad->payload_ep : ad->payload_o;
    st.vertex_const = ep ? ad->vconst_ep : ad->vconst_o;
    return st;
}

// one original-kernel step, timed into the ring while the partition is pending
epg_status step_original(epg_adaptive *ad, bool timed) {
    epg_state st = make_state(ad, false);
    std::pair<cudaEvent_t, cudaEvent_t> *ev = nullptr;
    if (timed) {
        if ((int)ad->orig_ev.size() < kTimedRing) {
            std::pair<cudaEvent_t, cudaEvent_t> e;
            ACU(cudaEventCreate(&e.first));
            ACU(cudaEventCreate(&e.second));
            ad->orig_ev.push_back(e);
        }
        ev = &ad->orig_ev[ad->orig_timed % kTimedRing];
        ACU(cudaEventRecord(ev->first, ad->stream));
    }
    epg_status s = epg_run_naive(ad->ctx, ad->kernel, ad->edges_d, ad->m, ad->n, &st, 1);
    if (s) return s;
    if (timed) {
        ACU(cudaEventRecord(ev->second, ad->stream));
        ad->orig_timed++;
    }
    ad->cur ^= 1;
    ad->steps_original++;
    return EPG_OK;
}

// median of the timed original steps (synchronises on the last one)
epg_status original_time(epg_adaptive *ad) {
    const int64_t cnt = std::min<int64_t>(ad->orig_timed, kTimedRing);
    std::vector<float> t;
    for (int64_t i = 0; i < cnt; i++) {
        ACU(cudaEventSynchronize(ad->orig_ev[i].second));
        float ms = 0.0f;
        ACU(cudaEventElapsedTime(&ms, ad->orig_ev[i].first, ad->orig_ev[i].second));
        t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    ad->original_ms = t.empty() ? 0.0 : t[t.size() / 2];
    return EPG_OK;
}

void free_ep(epg_adaptive *ad) {
    if (ad->plan) epg_plan_destroy(ad->plan);
    ad->plan = nullptr;
    for (float **p : {&ad->payload_ep, &ad->vconst_ep}) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }
    if (ad->vertex_perm) cudaFree(ad->vertex_perm);
    ad->vertex_perm = nullptr;
}

// apply the finished partition: remap, move the state into the EP layout, run the first
// EP step timed, keep it or fall back
epg_status apply_ep(epg_adaptive *ad) {
    const int64_t m = ad->m, n = ad->n, k = epg_num_parts(m, ad->part_size);
    struct Dev {
        std::vector<void *> p;
        ~Dev() { for (void *x : p) cudaFree(x); }
        cudaError_t get(void **out, size_t bytes) {
            cudaError_t e = cudaMalloc(out, std::max<size_t>(bytes, 16));
            if (e == cudaSuccess) p.push_back(*out);
            return e;
        }
    } tmp;
    int32_t *part_d = nullptr;
    ACU(tmp.get((void **)&part_d, sizeof(int32_t) * m));
    ACU(cudaMemcpyAsync(part_d, ad->part_h.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, ad->stream));
    epg_report rep{};
    epg_status s = epg_load_count(ad->ctx, ad->edges_d, m, ad->n, part_d, k, nullptr, &rep);
    if (s) return s;
    epg_layout L{};
    ACU(tmp.get((void **)&L.edge_perm, sizeof(int32_t) * m));
    ACU(tmp.get((void **)&L.part_edge_begin, sizeof(int32_t) * (k + 1)));
    ACU(cudaMalloc((void **)&ad->vertex_perm, sizeof(int32_t) * n));
    L.vertex_perm = ad->vertex_perm;
    ACU(tmp.get((void **)&L.part_vertex_begin, sizeof(int32_t) * (k + 1)));
    ACU(tmp.get((void **)&L.halo_begin, sizeof(int32_t) * (k + 1)));
    L.halo_cap = std::max<int64_t>(rep.cut_cost, 1);
    ACU(tmp.get((void **)&L.halo_ids, sizeof(int32_t) * L.halo_cap));
    ACU(tmp.get((void **)&L.slots, sizeof(uint16_t) * 2 * m));
    if ((s = epg_remap(ad->ctx, ad->edges_d, m, ad->n, part_d, k, &L, &ad->plan))) {
        free_ep(ad);
        return s;
    }
    if (ad->payload_o) {
        ACU(cudaMalloc((void **)&ad->payload_ep, sizeof(float) * ad->pw * m));
        if ((s = epg_permute_rows(ad->ctx, ad->payload_o, ad->payload_ep, m, 4 * ad->pw, L.edge_perm, 0))) return s;
    }
    if (ad->vconst_o) {
        ACU(cudaMalloc((void **)&ad->vconst_ep, sizeof(float) * n));
        if ((s = epg_permute_rows(ad->ctx, ad->vconst_o, ad->vconst_ep, n, 4, ad->vertex_perm, 1))) return s;
    }
    if ((s = epg_permute_rows(ad->ctx, ad->state[ad->cur], ad->state[ad->cur ^ 1], n, 4 * ad->row,
                              ad->vertex_perm, 1)))
        return s;
    ad->cur ^= 1;
    // first run of the transformed kernel, timed. An untimed run of the same step comes
    // first (its output is overwritten by the timed one): it loads the kernel module and
    // captures epg_run's CUDA graph, one-off host work that the GPU would otherwise sit
    // idle through inside the timed window (and that the original kernel, already warm,
    // never pays) -- the comparison of P:778-779 is between kernel runtimes.
    epg_state st = make_state(ad, true);
    if ((s = epg_run(ad->ctx, ad->plan, ad->kernel, &st, 1))) return s;
    ACU(cudaStreamSynchronize(ad->stream));
    cudaEvent_t a, b;
    ACU(cudaEventCreate(&a));
    ACU(cudaEventCreate(&b));
    ACU(cudaEventRecord(a, ad->stream));
    s = epg_run(ad->ctx, ad->plan, ad->kernel, &st, 1);
    cudaEventRecord(b, ad->stream);
    float ms = 0.0f;
    if (!s && cudaEventSynchronize(b) == cudaSuccess) cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (s) return s;
    ad->cur ^= 1;
    ad->steps_ep++;
    ad->ep_first_ms = ms;
    if ((s = original_time(ad))) return s;
    if (ad->ep_first_ms > ad->fallback_ratio * ad->original_ms) {
        // slower: back to the original layout and kernel for the next iterations
        if ((s = epg_permute_rows(ad->ctx, ad->state[ad->cur], ad->state[ad->cur ^ 1], n, 4 * ad->row,
                                  ad->vertex_perm, 0)))
            return s;
        ad->cur ^= 1;
        free_ep(ad);
        ad->phase = EPG_ADAPTIVE_FELL_BACK;
    } else {
        ad->phase = EPG_ADAPTIVE_EP;
    }
    return EPG_OK;
}

}  // namespace

extern "C" {

epg_status epg_adaptive_create(epg_ctx *ctx, epg_kernel kernel, const int32_t *edges_host, int64_t m,
                               int32_t n_vertices, int32_t part_size, const void *edge_payload,
                               const void *vertex_const, const void *state, double fallback_ratio,
                               epg_adaptive **out) {
    if (!ctx) return EPG_ERR_STATE;
    if (!out) return epg::ctx_fail(ctx, EPG_ERR_INPUT, "adaptive_create: out is NULL");
    *out = nullptr;
    if (kernel < EPG_KERNEL_CFD_FLUX || kernel > EPG_KERNEL_SPMV)
        return epg::ctx_fail(ctx, EPG_ERR_INPUT, "adaptive_create: unknown kernel");
    if (m <= 0 || m >= (int64_t(1) << 31) || n_vertices <= 0 || !edges_host || !state)
        return epg::ctx_fail(ctx, EPG_ERR_INPUT, "adaptive_create: need 0 < m < 2^31, n > 0, edges and state");
    if (part_size < 1 || part_size > EPG_MAX_PART_SIZE)
        return epg::ctx_fail(ctx, EPG_ERR_INFEASIBLE, "adaptive_create: part_size must be in [1, 4096]");
    if ((kernel == EPG_KERNEL_CFD_FLUX && (!edge_payload || !vertex_const)) ||
        (kernel == EPG_KERNEL_SPMV && !edge_payload))
        return epg::ctx_fail(ctx, EPG_ERR_INPUT, "adaptive_create: the kernel needs its edge payload / vertex constants");
    if (!(fallback_ratio >= 0.0)) return epg::ctx_fail(ctx, EPG_ERR_INPUT, "adaptive_create: fallback_ratio < 0");
    for (int64_t e = 0; e < m; e++) {
        const int32_t u = edges_host[2 * e], v = edges_host[2 * e + 1];
        if (u < 0 || u >= n_vertices || v < 0 || v >= n_vertices)
            return epg::ctx_fail(ctx, EPG_ERR_INPUT,
                                 "adaptive_create: edge " + std::to_string(e) + " has an endpoint outside [0, n)");
    }
    auto *ad = new epg_adaptive();
    ad->ctx = ctx;
    ad->stream = static_cast<cudaStream_t>(epg::ctx_stream(ctx));
    ad->kernel = kernel;
    ad->m = m;
    ad->n = n_vertices;
    ad->part_size = part_size;
    ad->row = kernel == EPG_KERNEL_CFD_FLUX ? 5 : 1;
    ad->pw = kernel == EPG_KERNEL_CFD_FLUX ? 3 : 1;
    ad->fallback_ratio = fallback_ratio;
    auto fail = [&](const std::string &what, cudaError_t e) {
        delete ad;
        return epg::ctx_fail(ctx, EPG_ERR_CUDA, what + ": " + cudaGetErrorString(e));
    };
    cudaError_t e;
    ad->edges_h.assign(edges_host, edges_host + 2 * m);
    const size_t rb = sizeof(float) * ad->row * (size_t)n_vertices;
    if ((e = cudaMalloc((void **)&ad->edges_d, sizeof(int32_t) * 2 * m)) ||
        (e = cudaMemcpyAsync(ad->edges_d, edges_host, sizeof(int32_t) * 2 * m, cudaMemcpyHostToDevice, ad->stream)) ||
        (e = cudaMalloc((void **)&ad->state[0], rb)) || (e = cudaMalloc((void **)&ad->state[1], rb)) ||
        (e = cudaMemcpyAsync(ad->state[0], state, rb, cudaMemcpyDefault, ad->stream)))
        return fail("adaptive_create", e);
    if (edge_payload) {
        const size_t pb = sizeof(float) * ad->pw * (size_t)m;
        if ((e = cudaMalloc((void **)&ad->payload_o, pb)) ||
            (e = cudaMemcpyAsync(ad->payload_o, edge_payload, pb, cudaMemcpyDefault, ad->stream)))
            return fail("adaptive_create", e);
    }
    if (vertex_const) {
        const size_t vb = sizeof(float) * (size_t)n_vertices;
        if ((e = cudaMalloc((void **)&ad->vconst_o, vb)) ||
            (e = cudaMemcpyAsync(ad->vconst_o, vertex_const, vb, cudaMemcpyDefault, ad->stream)))
            return fail("adaptive_create", e);
    }
    if ((e = cudaStreamSynchronize(ad->stream))) return fail("adaptive_create", e);
    // the optimisation thread (host only; never touches the context or the device)
    ad->part_h.assign((size_t)m, 0);
    // (EPG-RB bisects on the device; this thread stays on the host and runs EPG-2 instead)
    const int32_t method = epg::ctx_partition_method(ctx) == EPG_PARTITION_RB ? EPG_PARTITION_EPG2
                                                                               : epg::ctx_partition_method(ctx);
    ad->worker = std::thread([ad, method] {
        const auto t0 = std::chrono::steady_clock::now();
        ad->part_status = epg::host_partition(ad->edges_h.data(), ad->m, ad->n, ad->part_size, 1, ad->part_h.data(),
                                              &ad->part_err, &ad->cancel, method);
        ad->part_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        ad->done.store(1, std::memory_order_release);
    });
    *out = ad;
    return EPG_OK;
}

epg_status epg_adaptive_step(epg_adaptive *ad, int32_t steps) {
    if (!ad) return EPG_ERR_STATE;
    if (steps < 0) return epg::ctx_fail(ad->ctx, EPG_ERR_INPUT, "adaptive_step: steps < 0");
    for (int32_t i = 0; i < steps; i++) {
        epg_status s;
        if (ad->phase == EPG_ADAPTIVE_ORIGINAL && ad->done.load(std::memory_order_acquire)) {
            if (ad->worker.joinable()) ad->worker.join();
            if (ad->part_status != EPG_OK) {
                ad->phase = EPG_ADAPTIVE_NO_PARTITION;
            } else if (ad->orig_timed > 0) {      // there is an original runtime to compare with
                if ((s = apply_ep(ad))) return s;
                continue;                         // the first EP step was this step
            }
        }
        if (ad->phase == EPG_ADAPTIVE_EP) {
            epg_state st = make_state(ad, true);
            if ((s = epg_run(ad->ctx, ad->plan, ad->kernel, &st, 1))) return s;
            ad->cur ^= 1;
            ad->steps_ep++;
        } else if ((s = step_original(ad, ad->phase == EPG_ADAPTIVE_ORIGINAL))) {
            return s;
        }
    }
    return EPG_OK;
}

epg_status epg_adaptive_wait(epg_adaptive *ad) {
    if (!ad) return EPG_ERR_STATE;
    while (ad->phase == EPG_ADAPTIVE_ORIGINAL && !ad->done.load(std::memory_order_acquire))
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    return EPG_OK;
}

epg_status epg_adaptive_read_state(epg_adaptive *ad, void *state_out) {
    if (!ad) return EPG_ERR_STATE;
    if (!state_out) return epg::ctx_fail(ad->ctx, EPG_ERR_INPUT, "adaptive_read_state: NULL output");
    if (ad->phase == EPG_ADAPTIVE_EP)
        return epg_permute_rows(ad->ctx, ad->state[ad->cur], state_out, ad->n, 4 * ad->row, ad->vertex_perm, 0);
    ACU(cudaMemcpyAsync(state_out, ad->state[ad->cur], sizeof(float) * ad->row * (size_t)ad->n, cudaMemcpyDefault,
                        ad->stream));
    return EPG_OK;
}

epg_status epg_adaptive_info(const epg_adaptive *ad, epg_adaptive_report *out) {
    if (!ad || !out) return EPG_ERR_INPUT;
    out->phase = ad->phase;
    out->steps_original = ad->steps_original;
    out->steps_ep = ad->steps_ep;
    out->partition_done = ad->done.load(std::memory_order_acquire);
    out->partition_seconds = out->partition_done ? ad->part_seconds : 0.0;
    out->original_ms = ad->original_ms;
    out->ep_first_ms = ad->ep_first_ms;
    return EPG_OK;
}

void epg_adaptive_destroy(epg_adaptive *ad) { delete ad; }

}  // extern "C"
