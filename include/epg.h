/*
 * epg.h -- C ABI of libepg.so: the edge-partition (EP) scheduled irregular kernel of
 * arXiv 1605.02043, "A Graph-based Model for GPU Caching Problems", on B200 (sm_100a).
 *
 * Citations: "P:n" = PAPER.md line n (section / equation named beside it);
 * "S:n" = SPEC.md line n; "O<k>"/"Z<k>" = SURVEY.md §8(c) items, restated in DESIGN.md.
 *
 * The calls follow the paper's problem statement: "partition all m edges
 * evenly into k clusters ... every edge (task) is assigned to exactly one cluster
 * (thread block)", then "reorganize tasks among thread blocks ... and data layout"
 * (P:751-757), then run the transformed kernel:
 *
 *   epg_partition  -> edge -> partition map + load count      (§3, Eq. (1), Def. 3-4)
 *   epg_load_count -> the cost function on any map            (Eq. (1); fig:mot P:68-74)
 *   epg_remap      -> reordered edges + cpack vertex layout   (opt_indexA,
 *                     + the run plan                            opt_arrayA, beginA)
 *   epg_run        -> one or more time steps of the staged edge kernel
 *
 * Conventions (all calls):
 *  - ids are int32, counts int64, little-endian. Vertex ids in [0, n). The input edge
 *    order is the task id. Self-loops and parallel edges are distinct tasks
 *    (S:78-79); isolated vertices cost nothing.
 *  - Ownership: the caller owns every array passed in or out and allocates outputs
 *    (sizes are m, n, k+1, or come from an earlier report). The library never frees
 *    caller memory. The ctx owns its stream handle reference, scratch workspace and
 *    error string; an epg_plan owns the device descriptors its kernels read.
 *  - Memory spaces are stated per argument: "device" = CUDA device memory of the
 *    ctx's device; "host" = host memory; "host or device" = either (detected with
 *    cudaPointerGetAttributes).
 *  - Streams: work is enqueued on the ctx stream. Calls that fill an epg_report
 *    (epg_partition, epg_load_count) synchronise that stream before returning; all
 *    others are asynchronous.
 *  - Threads: one ctx per host thread; a ctx is not thread-safe.
 *  - Errors: every call returns an epg_status; the message of the last failure is
 *    epg_last_error(ctx). On error no output is guaranteed to be written.
 *      EPG_ERR_INPUT      m <= 0 (m >= 2^30 for the device layout calls epg_load_count,
 *                         epg_remap and epg_partition), n <= 0, an endpoint outside [0, n) (the message
 *                         names the first offending edge id), a partition id outside
 *                         [0, k), a too-small output capacity, NULL required pointer.
 *      EPG_ERR_INFEASIBLE part_size outside [1, 4096]; shards not in {1,2,4,8} or
 *                         shards > k; a partition whose staged rows exceed shared memory.
 *      EPG_ERR_CUDA       a CUDA runtime error (message carries cudaGetErrorString).
 *      EPG_ERR_NOMEM      device allocation failed.
 *      EPG_ERR_STATE      ctx/plan mismatch (wrong device, plan from another ctx).
 */
#ifndef EPG_H
#define EPG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    EPG_OK = 0,
    EPG_ERR_INPUT = 2,
    EPG_ERR_INFEASIBLE = 3,
    EPG_ERR_CUDA = 4,
    EPG_ERR_NCCL = 5,
    EPG_ERR_NOMEM = 6,
    EPG_ERR_STATE = 7
} epg_status;

#define EPG_MAX_PART_SIZE 4096

typedef struct epg_ctx epg_ctx;
typedef struct epg_plan epg_plan;

/* Cost report, Eq. (1) with the load accounting of fig:mot:
 *   k          number of partitions (thread blocks);
 *   load_count L = sum_p |V_p|, V_p = distinct endpoints of partition p
 *              ("one load is for every distinct particle");
 *   touched    #vertices with degree >= 1;
 *   cut_cost   C = sum_v (p_v - 1) = L - touched (the redundant loads);
 *   max_size / min_size  largest / smallest partition, in edges (balance). */
typedef struct {
    int64_t k, load_count, touched, cut_cost, max_size, min_size;
} epg_report;

/* Remapped layout (O6). Every array is DEVICE memory,
 * caller-allocated with the stated sizes. The staged kernel does not read these
 * arrays (the plan keeps its own copies), so they may be freed after epg_remap.
 *   edge_perm         [m]   new edge index -> original task id (edges sorted by
 *                           (partition, task id); the paper's reorganised tasks)
 *   part_edge_begin   [k+1] first new edge index of each partition
 *   vertex_perm       [n]   original vertex id -> new id (cpack first-touch order;
 *                           untouched vertices appended by id)  -- opt_arrayA's map
 *   part_vertex_begin [k+1] first owned new vertex id of each partition ("beginA");
 *                           partition p owns O_p = [pvb[p], pvb[p+1])
 *   halo_begin        [k+1] offsets into halo_ids
 *   halo_ids          [halo_cap] concatenated H_p = V_p \ O_p, ascending; the total
 *                           is C, so halo_cap >= cut_cost from epg_load_count
 *   slots             [m][2] uint16 local slot of each endpoint within its partition:
 *                           v - pvb[p] if owned, else |O_p| + rank of v in H_p
 *                           ("opt_indexA") */
typedef struct {
    int32_t *edge_perm;
    int32_t *part_edge_begin;
    int32_t *vertex_perm;
    int32_t *part_vertex_begin;
    int32_t *halo_begin;
    int32_t *halo_ids;
    int64_t halo_cap;
    uint16_t *slots;
} epg_layout;

/* Edge functors (O9; reading Z9). Row layouts are AoS float32.
 *  EPG_KERNEL_CFD_FLUX       state rows (rho, m_x, m_y, m_z, E) [n][5]; edge payload
 *                            area-normal [m][3] oriented edges[e][0] -> edges[e][1];
 *                            vertex_const dt [n]. Output U' = U + dt F (untouched
 *                            vertices copied). Face flux of P:62-64's "interaction
 *                            between two adjacent particles" (Rodinia-style, Z9).
 *  EPG_KERNEL_GATHER_SCATTER state x [n]; payload weight w [m] or NULL (w = 1);
 *                            output y [n], y_a += w x_b, y_b += w x_a.
 *  EPG_KERNEL_SPMV           bipartite graph of P:859-861: edge e = (column vertex j,
 *                            row vertex i), payload A[i,j] [m]; output y [n],
 *                            y_i += A[i,j] x_j (y = 0 at column vertices).          */
typedef enum {
    EPG_KERNEL_CFD_FLUX = 1,
    EPG_KERNEL_GATHER_SCATTER = 2,
    EPG_KERNEL_SPMV = 3
} epg_kernel;

/* Arguments of a time step. All DEVICE pointers in the layout the call expects:
 * epg_run: rows in the plan's NEW vertex order and payload in NEW edge order
 * (use epg_permute_rows); epg_run_naive: original orders.
 * state_in and state_out must not alias. With steps > 1 the two buffers ping-pong:
 * step s (1-based) reads the buffer written by step s-1, so the final result is in
 * state_out when steps is odd and in state_in when steps is even (state_in is then
 * overwritten, so it must be writable). */
typedef struct {
    void *state_in;
    void *state_out;
    const void *edge_payload;
    const void *vertex_const;
} epg_state;

/* -- context ------------------------------------------------------------------ */
/* Create a context on CUDA device `device`, enqueuing on `cuda_stream` (a
 * cudaStream_t; NULL = the legacy default stream). The library's temporaries come from the
 * device's default stream-ordered memory pool; its release threshold is raised to
 * EPG_POOL_KEEP_GB GiB (default 32) so freed scratch stays mapped for the next call. */
epg_status epg_create(int device, void *cuda_stream, epg_ctx **out);
void epg_destroy(epg_ctx *ctx);
/* Message of the last failed call on ctx (ctx-owned, valid until the next call). */
const char *epg_last_error(const epg_ctx *ctx);
/* k = ceil(m / part_size) (O1); 0 if m <= 0 or part_size <= 0. */
int64_t epg_num_parts(int64_t m, int32_t part_size);

/* -- partition (step a2 + a3) ------------------------------------------------- */
/* Host-only EPG-1 partition (no device needed): the balanced growing partitioner on
 * the contracted clone-and-connect graph T (Def. 3, weight P:377, chain
 * order P:380; EPG-1 replaces METIS P:384/P:418, reading Z3). Partition sizes are
 * s_i = floor(m/k) + [i < m mod k] (Eq. (1) "L_i = m/k", exact +-1, Z2).
 * shards = G > 1 runs the hierarchical variant (shard-level EPG-1, then per shard).
 *   edges [m][2] HOST; part_of_edge [m] HOST out; 0 < m < 2^31.
 * Returns EPG_ERR_INPUT / EPG_ERR_INFEASIBLE as above; writes the message into
 * errbuf (errbuf_len bytes, may be NULL). */
epg_status epg_partition_host(const int32_t *edges, int64_t m, int32_t n_vertices, int32_t part_size,
                              int32_t shards, int32_t *part_of_edge, char *errbuf, int64_t errbuf_len);

/* Partitioner methods. EPG_PARTITION_EPG1 is epg_partition_host above. EPG_PARTITION_EPG2
 * (reading Z20) keeps EPG-1's seed and stamp schedule but
 * grows on Eq. (1)'s own objective: the gain of a frontier task is the number
 * of its distinct endpoints already loaded by the growing partition, so each step adds
 * the fewest new loads; the frontier grows through vertex incidence lists instead of T.
 * A vertex with more than 4 x part_size incident tasks (a hub, cut into many clusters
 * whatever happens) attracts no tasks. Same sizes, hierarchy (shards) and
 * determinism as EPG-1. */
#define EPG_PARTITION_EPG1 1
#define EPG_PARTITION_EPG2 2
/* EPG_PARTITION_RB (the GPU-parallel EP partitioner; DESIGN.md reading
 * Z21): recursive graph-growing bisection of the task set on the GPU, then EPG-2 in every
 * leaf on all host cores. Bisection depth d = log2(shards), raised while every leaf keeps at
 * least leaf_parts partitions (d <= 10). Node a of level l holds the partitions
 * [floor(a k/2^l), floor((a+1) k/2^l)) and exactly their tasks; it is split by a BFS over
 * tasks sharing a non-hub endpoint (hub: more than 4 x part_size tasks) from a
 * pseudo-peripheral task (the farthest from the node's smallest task id, ties to the smaller
 * id): in ascending (distance, id) the first tasks -- as many as its first half of
 * partitions holds -- form child 2a. Leaves run EPG-2 on their own tasks. With shards = G the
 * first log2(G) levels are the shards. Deterministic; needs a device (epg_partition /
 * epg_partition_rb), so epg_partition_host_method rejects it. */
#define EPG_PARTITION_RB 3
/* epg_partition_host with a method (EPG_ERR_INPUT for any other value). */
epg_status epg_partition_host_ranked(const int32_t *edges, int64_t m, int32_t n_vertices, int32_t part_size,
                                     int32_t shards, int32_t method, int32_t *part_of_edge, int32_t *rank_of_edge,
                                     char *errbuf, int64_t errbuf_len);
/* (the same, without ranks; rank_of_edge [m] HOST out of the one above: each task's growth step) */
epg_status epg_partition_host_method(const int32_t *edges, int64_t m, int32_t n_vertices, int32_t part_size,
                                     int32_t shards, int32_t method, int32_t *part_of_edge, char *errbuf,
                                     int64_t errbuf_len);

/* PowerGraph's edge partitioners, the quality baselines of SURVEY §8(f)
 * rank 4, with the same k = ceil(m / part_size) clusters (host only, no device needed).
 * epg_partition_random_host: "randomly assigns edges into partitions" with exact
 *   balance (reading Z18): the edges ordered by (SplitMix64(seed, e), e) are
 *   dealt round-robin, so cluster c gets floor(m/k) + [c < m mod k] edges.
 * epg_partition_greedy_host: one pass in task order; each edge goes to the cluster that
 *   "already possess[es] the endpoints": the highest [u in V_c] + [v in V_c]
 *   among clusters holding fewer than ceil(m/k) edges, ties by fewer edges, then lower
 *   id (with no holder open: "the partition with the fewest edges"; reading
 *   Z19). Time grows with the number of clusters holding each endpoint (slow on hubs).
 *   part_of_edge [m] HOST out. Status and errbuf as for epg_partition_host. */
epg_status epg_partition_random_host(int64_t m, int32_t part_size, uint64_t seed, int32_t *part_of_edge,
                                     char *errbuf, int64_t errbuf_len);
epg_status epg_partition_greedy_host(const int32_t *edges, int64_t m, int32_t n_vertices, int32_t part_size,
                                     int32_t *part_of_edge, char *errbuf, int64_t errbuf_len);

/* Partitioner used by epg_partition and the adaptive executor on ctx (default EPG1; the
 * adaptive executor's host thread runs EPG-2 in place of EPG-RB); EPG_ERR_INPUT for an
 * unknown method. */
epg_status epg_set_partition_method(epg_ctx *ctx, int32_t method);

/* epg_partition_host (with ctx's method), then the GPU cost function on the result (epg_load_count).
 *   edges [m][2] host or device; part_of_edge [m] host or device out; out report. */
epg_status epg_partition(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n_vertices, int32_t part_size,
                         int32_t shards, int32_t *part_of_edge, epg_report *out);

/* epg_partition with EPG_PARTITION_RB and an explicit leaf size (epg_partition uses 512, or
 * the EPG_RB_LEAF_PARTS environment variable). EPG_ERR_INPUT for leaf_parts < 1 or m >= 2^30;
 * EPG_ERR_INFEASIBLE as for epg_partition_host, or if a BFS is deeper than 2^22 - 2 levels.
 *   edges [m][2] host or device; part_of_edge [m] host or device out; rank_of_edge [m] host or
 *   device out, or NULL: the step at which each task joined its partition (EPG-2's growth in
 *   its leaf; reading Z22, for epg_remap_keyed); out report. */
epg_status epg_partition_rb(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n_vertices, int32_t part_size,
                            int32_t shards, int32_t leaf_parts, int32_t *part_of_edge, int32_t *rank_of_edge,
                            epg_report *out);
/* epg_partition that also returns the growth ranks (as epg_partition_rb; any method). */
epg_status epg_partition_ranked(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n_vertices, int32_t part_size,
                                int32_t shards, int32_t *part_of_edge, int32_t *rank_of_edge, epg_report *out);

/* Default task schedule (O3; "default task scheduling" P:75): task e goes to
 * the i-th contiguous chunk of sizes s_i.  part_of_edge [m] DEVICE out. */
epg_status epg_default_partition(epg_ctx *ctx, int64_t m, int32_t part_size, int32_t *part_of_edge);

/* GPU cost function (step a3; Eq. (1), fig:mot P:68-74). Any map with
 * part ids in [0, k).  edges [m][2] DEVICE; part_of_edge [m] DEVICE;
 * per_part_distinct [k] DEVICE out (|V_p|) or NULL; out report (host). Synchronises. */
epg_status epg_load_count(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n_vertices,
                          const int32_t *part_of_edge, int64_t k, int32_t *per_part_distinct, epg_report *out);

/* -- remap (step a4) ---------------------------------------------------------- */
/* Task reorganisation + cpack layout on the GPU (O6). Fills `layout` (device arrays,
 * see epg_layout) and creates *plan: the device descriptors of the staged kernel
 * (per-partition incidence lists, shared-vertex lists, accumulators). Requires every
 * partition to have at most EPG_MAX_PART_SIZE edges.
 * The plan also fixes where each partition's staged records live in shared memory: a
 * record (and an edge's Phi record) may take any position of its aligned group of 8, and a
 * greedy pass (one warp per partition) picks the positions so that the 128-bit shared loads
 * of a warp quarter hit distinct bank groups; EPG_PLACE=0 keeps the identity. The boundary
 * finalise reads 16-byte records {v, count, h0, h1 | overflow index} (EPG_FIN_REC16=0: the
 * 32-byte records). Neither changes a result bit (same values, same summation orders).
 *   edges [m][2] DEVICE (original task order); part_of_edge [m] DEVICE. */
epg_status epg_remap(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n_vertices,
                     const int32_t *part_of_edge, int64_t k, epg_layout *layout, epg_plan **plan);
/* epg_remap with the tasks of each partition ordered by (order_key, task id) instead of the
 * task id (reading Z22: the paper's reorganisation, leaves the order inside a
 * thread block open). With the growth ranks of epg_partition_ranked / epg_partition_rb,
 * consecutive tasks of a block share or neighbour their vertices, so the cpack numbering and
 * the local slots follow the growth and the staged kernel's threads read nearby records.
 * order_key [m] DEVICE, values in [0, 2^31), or NULL (= epg_remap). */
epg_status epg_remap_keyed(epg_ctx *ctx, const int32_t *edges, int64_t m, int32_t n_vertices, const int32_t *part_of_edge,
                           const int32_t *order_key, int64_t k, epg_layout *layout, epg_plan **plan);
void epg_plan_destroy(epg_plan *plan);
/* Sizes of a plan: out[0..7] = m, n, k, touched, cut_cost (= |halo_ids| of the layout),
 * shared vertex count of the execution plan, k_exec, cut cost of the execution plan.
 * Execution partitions: an EP partition whose staged rows or edges exceed what one CTA
 * of the staged kernel holds (768 rows, 1024 edges) is executed as contiguous ranges of
 * its reorganised edges; this changes neither edge_perm nor vertex_perm, only how many
 * thread blocks share the partition (k_exec >= k). */
epg_status epg_plan_info(const epg_plan *plan, int64_t *out8);

/* Row permutation (step a7 and the layout change of a4), DEVICE arrays:
 *   mode 0 (gather):  dst[i]       = src[perm[i]]   for i < rows
 *   mode 1 (scatter): dst[perm[i]] = src[i]         for i < rows
 * vertex rows into the new layout: scatter with vertex_perm; back to the original
 * layout: gather with vertex_perm; edge payload into the new order: gather with
 * edge_perm. row_bytes must be a multiple of 4. */
epg_status epg_permute_rows(epg_ctx *ctx, const void *src, void *dst, int64_t rows, int32_t row_bytes,
                            const int32_t *perm, int32_t mode);

/* The reorganised task list in the new vertex ids ("opt_indexA", P:755-757 / P:1343):
 * out[i] = (vertex_perm[edges[edge_perm[i]][0]], vertex_perm[edges[edge_perm[i]][1]]).
 * With epg_run_naive on these edges and the cpack-ordered state this is the paper's
 * hardware-cache variant: the EP order and layout, operands through the
 * read-only cache path instead of shared-memory staging.  All DEVICE, out [m][2]. */
epg_status epg_remapped_edges(epg_ctx *ctx, const int32_t *edges, int64_t m, const int32_t *edge_perm,
                              const int32_t *vertex_perm, int32_t *out);

/* -- run (steps a5 + a6) ------------------------------------------------------ */
/* `steps` time steps of the partition-scheduled kernel: one CTA per
 * partition stages V_p (owned rows O_p contiguous, halo rows H_p gathered) into
 * shared memory, evaluates the functor per edge from shared memory, reduces each
 * vertex's incident contributions in shared memory and writes interior vertices'
 * results directly; vertices shared by several partitions (p_v > 1) are completed
 * by a boundary-finalise pass. Deterministic: the summation order is fixed, except for
 * hub vertices under the hub split (epg_set_hub_split; never on cfd meshes).
 * On the occupancy-kernel path a call of steps >= 2 is captured once into a CUDA graph
 * per (plan, kernel, buffer pointers, steps, variant) -- at most 16 per plan, owned by
 * the plan -- and replayed into ctx's stream on later calls (not while profiling). A
 * one-step call launches its kernels directly, with programmatic-dependent-launch
 * attributes, so back-to-back calls overlap each kernel's prologue with the previous
 * kernel in the stream (a graph launch would end that overlap at every call boundary:
 * C2, 23 alternating plans, 19.1 -> 12.7 us per step). EPG_GRAPHS=0 in the environment
 * disables the graphs, EPG_GRAPHS=2 also captures one-step calls. Multi-wave grids
 * prefetch the next wave's ranges into L2 (EPG_PREFETCH_AHEAD=<CTAs>, 0 disables). */
epg_status epg_run(epg_ctx *ctx, const epg_plan *plan, epg_kernel kernel, epg_state *state, int32_t steps);

/* epg_run from and to HOST memory (the end-to-end call): one call copies the state
 * (state_in_host, [n][row] floats, ORIGINAL vertex order, row = 5 for CFD_FLUX, 1 otherwise)
 * to the device, moves it into the plan layout (vertex_perm: DEVICE, epg_remap's layout),
 * runs `steps` time steps as epg_run, moves the result back to the original order and
 * copies it to state_out_host (same shape). edge_payload / vertex_const: DEVICE, plan
 * layout, as for epg_run. Asynchronous: the H2D and D2H run on two ctx-owned streams and
 * the compute on ctx's stream, with double-buffered device staging, so consecutive calls
 * overlap one call's D2H with the next call's H2D and compute. Host buffers must stay
 * valid (and unchanged, for state_in_host) until the call's copies finish; pinned host
 * memory makes the copies truly asynchronous. The outputs of all calls so far are complete
 * once ctx's stream has executed a later epg_run_host_join(ctx) (which only enqueues a
 * wait). EPG_ERR_NOMEM if the ctx-owned buffers (5 x n x row floats) cannot be allocated. */
epg_status epg_run_host(epg_ctx *ctx, const epg_plan *plan, epg_kernel kernel, const int32_t *vertex_perm,
                        const void *state_in_host, void *state_out_host, const void *edge_payload,
                        const void *vertex_const, int32_t steps);
/* Makes ctx's stream wait for every D2H copy epg_run_host has enqueued so far. */
epg_status epg_run_host_join(epg_ctx *ctx);

/* The default (unscheduled) comparator: the same functor with one thread per task
 * in original order, operands read straight from global memory and results
 * accumulated with global atomics, then a per-vertex update (the original kernel of
 * P:75 / P:1009 that the paper's schedule replaces).  edges [m][2] DEVICE. */
epg_status epg_run_naive(epg_ctx *ctx, epg_kernel kernel, const int32_t *edges, int64_t m, int32_t n_vertices,
                         epg_state *state, int32_t steps);

/* -- multi-GPU shards (the paper is single-GPU) ------------------------ */
/* Shard g of G holds the EP partitions [floor(gk/G), floor((g+1)k/G)) (hierarchical EPG-1
 * with shards = G keeps them contiguous in the graph), owns the vertices their cpack ranges
 * cover, and per time step: pulls the halo rows owned by lower shards (Halo^{g<-g'}), runs
 * epg_run_edges on its execution partitions, pushes per-vertex partial sums
 * (epg_shard_reduce) to the owners, accumulates the ones it receives in ascending peer order
 * (epg_accumulate_rows) and finalises its shared vertices (epg_run_finalise). Every rank
 * holds the same plan and full-size state arrays; only owned rows are authoritative.
 *
 * out8 = execution partitions first, count; halo positions first, count; owned vertices
 * first, count; shared vertices (index into the plan's shared list) first, count. */
epg_status epg_shard_ranges(const epg_plan *plan, int32_t G, int32_t g, int64_t *out8);
/* Halo sets O7 from the layout of the EP map (HOST arrays pvb [k+1], halo_begin [k+1],
 * halo_ids): begin_out [G*G+1]; ids of Halo^{g<-g'} at begin_out[g*G+g'] .. [g*G+g'+1]
 * (ascending; non-empty only for g' < g). ids_out may be NULL to count (*count_out). */
epg_status epg_shard_halos_host(const int32_t *part_vertex_begin, const int32_t *halo_begin, const int32_t *halo_ids,
                                int64_t k, int32_t G, int32_t *begin_out, int32_t *ids_out, int64_t cap,
                                int64_t *count_out);
/* The staged edge kernel over execution partitions [first, first + count) (no finalise):
 * writes U + dt F_local into the owned rows of state_out and the halo partials into the
 * plan's halo buffer. Requires the default (occupancy) kernel's limits. */
epg_status epg_run_edges(epg_ctx *ctx, const epg_plan *plan, epg_kernel kernel, epg_state *state, int64_t first,
                         int64_t count);
/* Boundary finalise of the shared vertices [shared_first, +shared_count) of the plan's
 * shared list: state_out[v] += dt_v * (halo partials at positions in [halo_first,
 * +halo_count), ascending, then acc[v]); acc (DEVICE [n][row], or NULL) is cleared on
 * the way. untouched != 0 also copies (cfd) / clears untouched rows. */
epg_status epg_run_finalise(epg_ctx *ctx, const epg_plan *plan, epg_kernel kernel, epg_state *state,
                            int64_t shared_first, int64_t shared_count, int64_t halo_first, int64_t halo_count,
                            float *acc, int32_t untouched);
/* out_rows[i] = sum of the halo partials of vertex ids[i] at positions in [halo_first,
 * +halo_count), ascending (DEVICE arrays; ids [count], out_rows [count][row]). */
epg_status epg_shard_reduce(epg_ctx *ctx, const epg_plan *plan, epg_kernel kernel, const int32_t *ids, int64_t count,
                            int64_t halo_first, int64_t halo_count, float *out_rows);
/* acc[ids[i]] += src[i], rows of row_floats floats; ids distinct (DEVICE arrays). */
epg_status epg_accumulate_rows(epg_ctx *ctx, const float *src, const int32_t *ids, int64_t count, int32_t row_floats,
                               float *acc);

/* -- multi-GPU: the halo exchange inside the library ------------- */
/* One process per GPU. Rank g of G runs shard g of a plan built (identically on every rank)
 * from a map partitioned with shards = G (epg_partition / epg_partition_rb), so shard g owns
 * the EP partitions [floor(gk/G), floor((g+1)k/G)) and a contiguous cpack vertex range. A
 * sharded time step (O7): (1) pull: each owner g' < g sends the rows of Halo^{g<-g'} --
 * packed by a gather kernel, grouped ncclSend / ncclRecv on the ctx stream, scattered into
 * state_in (rows owned by other ranks are overwritten with their owners' values); (2) the
 * staged edge kernel over g's execution partitions; (3) push: g sends each owner the sum of
 * its halo partials of every vertex of Halo^{g<-g'} (fixed order) and adds what higher ranks
 * send into a per-vertex accumulator in ascending rank order; (4) the boundary finalise of
 * g's shared vertices and g's untouched rows. Only the rows g owns (epg_shard_ranges) are
 * authoritative in state_out. Deterministic for a fixed G. The interior partitions (no halo
 * row owned by a lower rank) run while the pull is in flight (NCCL on a stream of the ctx's
 * own), and the local finalise while the push is.
 * EPG_EXCHANGE=p2p (environment, read when a plan first steps sharded) fuses the push into the
 * boundary edge kernel: each partition adds its partial of a vertex owned by rank p straight
 * into p's accumulator in peer memory (atomics over NVLink; the accumulators' CUDA IPC handles
 * are exchanged once with ncclAllGather), and a one-float NCCL token per push pair orders the
 * owner's accumulate-add after the pushers' kernels; the summation order of those partials
 * is then not fixed (the rest of the step is unchanged).
 *
 * epg_comm_unique_id: ncclGetUniqueId into id_out (128 bytes, host) -- call on one rank and
 *   broadcast it (e.g. through torch.distributed).
 * epg_comm_init: ncclCommInitRank(nranks, id, rank) on ctx's device; the communicator is
 *   owned by ctx (destroyed with it, or by the next epg_comm_init*). NCCL is loaded at run
 *   time (libnccl.so.2); EPG_ERR_NCCL if it is missing or fails.
 * epg_comm_init_local: makes the nranks contexts (one process, e.g. one GPU) an in-process
 *   group with ranks 0..nranks-1 whose transfers are device copies -- the same exchange
 *   schedule without NCCL, for tests; its members step through epg_run_sharded_group.
 * epg_run_sharded: `steps` sharded time steps on this rank (all ranks must call it with the
 *   same plan shape, kernel and steps); state as for epg_run (DEVICE, full-size, plan layout).
 *   Without epg_comm_init it is the single-rank case (no transfers). EPG_ERR_INFEASIBLE if
 *   nranks > k or the plan exceeds the occupancy kernel's limits.
 * epg_run_sharded_group: one sharded step of every member of an in-process group
 *   (ctxs[g] has rank g; plans[g] is ctxs[g]'s plan; states[g] its state). */
epg_status epg_comm_unique_id(void *id_out);
epg_status epg_comm_init(epg_ctx *ctx, const void *nccl_unique_id, int32_t nranks, int32_t rank);
epg_status epg_comm_init_local(epg_ctx *const *ctxs, int32_t nranks);
epg_status epg_run_sharded(epg_ctx *ctx, const epg_plan *plan, epg_kernel kernel, epg_state *state, int32_t steps);
epg_status epg_run_sharded_group(epg_ctx *const *ctxs, const epg_plan *const *plans, epg_kernel kernel,
                                 epg_state *states, int32_t nranks);

/* Kernel variant used by epg_run: 0 = automatic (the first of 3, 2, 1 whose buffers fit),
 * 1 = one CTA per partition (plain loads), 2 = persistent pipelined TMA kernel, 3 = TMA
 * kernel with one CTA per execution partition and several CTAs per SM. 2 and 3 return
 * EPG_ERR_INFEASIBLE if the plan does not fit them. All compute the same result; they
 * differ in how partitions are staged and scheduled. */
epg_status epg_set_variant(epg_ctx *ctx, int32_t variant);

/* Execution-split caps for plans created by later epg_remap calls on ctx: an EP
 * partition with more than max_rows staged rows (|V_p|) or max_edges edges is executed
 * as contiguous ranges of its reorganised edges (the public layout is unchanged; see
 * epg_plan_info's k_exec). max_rows in [64, 2048] (above 1280 only one-float functors,
 * GATHER_SCATTER and SPMV, run the occupancy kernel), max_edges in [32, 1280]; -1 keeps
 * the default: EPG_EXEC_MAX_ROWS / EPG_EXEC_MAX_EDGES from the environment, else 768
 * rows (a cfd CTA at ~53 KB of shared memory, four per SM) and 1024 edges. Raising both
 * lets partitions of up to 1280 edges run unsplit, e.g. to size the grid to a multiple of
 * the SM count.
 * EPG_ERR_INPUT outside these ranges. */
epg_status epg_set_exec_limits(epg_ctx *ctx, int32_t max_rows, int32_t max_edges);

/* Hub split (power-law graphs, the hub discussion of P:642-683):
 * plans created by later epg_remap calls on ctx treat every shared vertex with at least
 * `min_halo_entries` halo entries as a hub. Variant 3 then sums each execution
 * partition's partial of a hub in shared memory, as for any vertex. It adds that partial
 * with one red.global.add into a per-hub accumulator, and a hub finalise applies the
 * accumulator. The finalise then no longer gathers the hub's scattered halo partials.
 * The sum order over partitions is then not fixed, so results are deterministic only up
 * to fp32 rounding for hubs (exact for integer-valued data). 0 turns it off. The default
 * (-1 = unset) is 7, overridable by the EPG_HUB_MIN environment variable. Meshes with
 * degree <= 4 (cfd) never have hubs at the default. -1 restores the default; values
 * below -1 return EPG_ERR_INPUT. */
epg_status epg_set_hub_split(epg_ctx *ctx, int32_t min_halo_entries);
/* Hub read side ("for the vertices with large degree ... we use hardware
 * cache instead", the hub paragraph of P:642-683): with enable != 0 (the default) the edge
 * kernel of a plan with hubs is launched with a persisting L2 access-policy window over the
 * prefix of state_in that holds the hubs' rows (cpack numbers vertices by first touch and
 * hubs are touched by the first partitions, so they sit at the front), so their rows stay
 * L2-resident while each partition gathers them; it raises the device's persisting-L2 limit
 * (cudaLimitPersistingL2CacheSize) to its maximum on first use. 0 launches without it. */
epg_status epg_set_hub_l2(epg_ctx *ctx, int32_t enable);
/* Hub count of a plan (-1 for NULL); *min_halo_entries (may be NULL) receives the
 * threshold it was built with (0 = off). */
int64_t epg_plan_hubs(const epg_plan *plan, int32_t *min_halo_entries);

/* -- adaptive overhead control --------------------- */
/* The paper's runtime policy around the transformed kernel, as a native executor:
 *   - "data sharing optimization using a separate thread on the CPU while kernel is
 *     executed on the GPU": create starts host EPG-1 (flat, part_size) on a
 *     std::thread; until it finishes, steps run the original kernel (epg_run_naive:
 *     original task order, global-memory operands), each timed with CUDA events;
 *   - "check if the asynchronous optimization is completed before calling the kernel
 *     and apply the optimization if so": before every step, a finished partition
 *     is remapped (epg_load_count + epg_remap on the ctx stream) and the state moved to
 *     the plan's layout. (If it finishes before any original step was timed, one original
 *     step runs first so there is a runtime to compare with.);
 *   - "record the transformed kernel runtime the first time it runs, and compare it with
 *     the original kernel runtime. If the first run ... is slower, then we fall back to the
 *     original kernel in the next iteration": the first EP step is timed and
 *     kept iff ep_first_ms <= fallback_ratio * (median timed original step); otherwise
 *     the state moves back and every later step runs the original kernel (1.0 = the
 *     paper's rule);
 *   - "If the optimization thread does not complete when the program finishes, we
 *     terminate it": epg_adaptive_destroy cancels (polled once per partition)
 *     and joins the thread.
 * Every step advances one time step of the functor (state_out = F(state_in), the two
 * state buffers alternating), whichever kernel runs it.
 *   create: edges_host [m][2] HOST (copied); edge_payload (original task order),
 *     vertex_const and state ([n][row] original vertex order) host or device, copied --
 *     the executor owns its buffers. Payload / constants as for epg_run (cfd needs both,
 *     SPMV the payload, GATHER_SCATTER optional weights). EPG_ERR_INPUT / INFEASIBLE as
 *     for epg_partition_host; EPG_ERR_CUDA on allocation failures.
 *   read_state: the current state in original vertex order into state_out (DEVICE,
 *     [n][row]; asynchronous on the ctx stream).
 *   wait: blocks until the partition thread has finished (the next step applies it).
 *   info: phase (epg_adaptive_phase), step counts and the timings the policy used. */
typedef struct epg_adaptive epg_adaptive;
typedef enum {
    EPG_ADAPTIVE_ORIGINAL = 0,     /* partition running; original kernel */
    EPG_ADAPTIVE_EP = 1,           /* EP plan applied and kept */
    EPG_ADAPTIVE_FELL_BACK = 2,    /* first EP step was slower; original kernel from then on */
    EPG_ADAPTIVE_NO_PARTITION = 3  /* the partition failed; original kernel */
} epg_adaptive_phase;
typedef struct {
    int32_t phase, partition_done;
    int64_t steps_original, steps_ep;
    double partition_seconds;      /* wall time of the host partition thread (0 while running) */
    double original_ms;            /* median of the timed original steps */
    double ep_first_ms;            /* the first EP step */
} epg_adaptive_report;
epg_status epg_adaptive_create(epg_ctx *ctx, epg_kernel kernel, const int32_t *edges_host, int64_t m,
                               int32_t n_vertices, int32_t part_size, const void *edge_payload,
                               const void *vertex_const, const void *state, double fallback_ratio,
                               epg_adaptive **out);
epg_status epg_adaptive_step(epg_adaptive *ad, int32_t steps);
epg_status epg_adaptive_wait(epg_adaptive *ad);
epg_status epg_adaptive_read_state(epg_adaptive *ad, void *state_out);
epg_status epg_adaptive_info(const epg_adaptive *ad, epg_adaptive_report *out);
void epg_adaptive_destroy(epg_adaptive *ad);

/* -- measurement -------------------------------------------------------------- */
/* Kernel timing for bench.py: while enabled, epg_run / epg_run_naive record a CUDA event
 * pair on the ctx stream around every kernel they launch. epg_profile_read synchronises
 * the stream, returns the summed device time (ms) per kernel class since the previous
 * read and resets the accumulators:
 *   ms[0] edge kernel (staged, or naive edge pass), ms[1] finalise / naive update;
 *   launches[0], launches[1] the matching launch counts. */
epg_status epg_set_profiling(epg_ctx *ctx, int32_t enable);
epg_status epg_profile_read(epg_ctx *ctx, float *ms2, int64_t *launches2);

#ifdef __cplusplus
}
#endif
#endif /* EPG_H */
