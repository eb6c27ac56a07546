/*
 * gimbal_gpu.h — C ABI of the B200 (sm_100a) expert-statistics + placement hot path.
 *
 * Drop-in boundary for the reference's operator API (/root/reference/proj):
 *   moe::RoutingStats / record_stats / comm_cost        include/gimbal/moe.hpp:86-111
 *   placement::eval_cost / build_affinity_set /
 *   greedy_place / maybe_relocate / static_placement     include/gimbal/placement.hpp:44-85
 * A C++ layer with the reference's exact signatures sits on top of this ABI
 * (paper_2602_21626_b200/shim/); the Python mirror binds it with ctypes.
 *
 * Conventions
 *  - Every entry point returns a gimbal_status; gimbal_last_error() returns the calling thread's
 *    last message (the reference's std::invalid_argument text where one exists).
 *  - Plain pointers + sizes only.  `mem` says whether a buffer is host (GIMBAL_MEM_HOST) or
 *    device (GIMBAL_MEM_DEVICE) memory.  Host buffers may be pageable; pinned ones overlap.
 *  - Matrices are row-major: A [L][n_e], E [(L-1)][n_e][n_e], W [n_e][n_e]  (the reference stores
 *    the same numbers column-major in Eigen).  Counts are uint64 (the reference keeps them as
 *    integer-valued doubles, exact below 2^53).
 *  - Traces are token-major [T][L][top_k] expert ids, the order of RoutedStream::choices
 *    (moe.hpp:75-83); id_bytes 1 (uint8, n_e <= 256, the native layout) or 4 (int32, the
 *    reference layout).  Ids outside [0, n_e) are an error (GIMBAL_OUT_OF_RANGE); the reference
 *    leaves them undefined (no range check at moe.cpp:176-187).
 *  - Handles own device memory and a CUDA stream on their device; no global mutable state, so
 *    independent handles may be driven from different host threads (the reference runs one
 *    MoeSubsystem per sweep thread, cli.cpp:145-162).
 *  - Work is enqueued asynchronously on the handle's stream; calls that return data to the
 *    host synchronise that stream.  Errors raised inside kernels (ids out of range) are sticky
 *    and reported by the next synchronising call.
 */
#ifndef GIMBAL_GPU_H_
#define GIMBAL_GPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GIMBAL_ABI_VERSION 4

typedef enum gimbal_status {
  GIMBAL_OK = 0,
  GIMBAL_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  GIMBAL_CUDA_ERROR = 2,
  GIMBAL_NCCL_ERROR = 3,
  GIMBAL_OVERFLOW = 4,         /* a count would leave the exactly representable range */
  GIMBAL_OUT_OF_RANGE = 5,     /* expert id outside [0, n_e) in a trace */
  GIMBAL_NOT_SUPPORTED = 6
} gimbal_status;

typedef enum gimbal_mem { GIMBAL_MEM_HOST = 0, GIMBAL_MEM_DEVICE = 1 } gimbal_mem;

/* moe::MoeTopology (moe.hpp:14-23); validated like MoeTopology::validate (moe.cpp:12-24). */
typedef struct gimbal_topology {
  int32_t n_layers;
  int32_t n_experts; /* per layer */
  int32_t top_k;
  int32_t n_gpus;    /* placement target g */
} gimbal_topology;

typedef struct gimbal_stats_s* gimbal_stats_t;

int gimbal_abi_version(void);
const char* gimbal_last_error(void);
/* Validates a topology (moe.cpp:12-24). */
int gimbal_topology_validate(const gimbal_topology* topo);

/* ---- routing statistics: replaces moe::RoutingStats (moe.hpp:86-105, moe.cpp:162-231) ---- */

/* RoutingStats(topo): zeroed A/E on `device`, with its own stream (moe.cpp:162-167). */
int gimbal_stats_create(const gimbal_topology* topo, int device, gimbal_stats_t* out);
int gimbal_stats_destroy(gimbal_stats_t h);
/* RoutingStats::reset (moe.cpp:193-197). */
int gimbal_stats_reset(gimbal_stats_t h);
/* Batch RoutingStats::add_token (moe.cpp:169-191) / record_stats (moe.cpp:233-239): counts
 * n_tokens tokens of a [T][L][k] trace, all k x k consecutive-layer pairings with multiplicity.
 * Asynchronous on the handle's stream; a host trace is staged through pinned buffers. */
int gimbal_stats_add_tokens(gimbal_stats_t h, const void* ids, int id_bytes, int64_t n_tokens,
                            int mem);
/* RoutingStats::tokens (moe.hpp:93). */
int gimbal_stats_tokens(gimbal_stats_t h, int64_t* tokens);
/* activation() / affinity() (moe.hpp:91-92, moe.cpp:199-205): copies A [L][n_e],
 * E [(L-1)][n_e][n_e] and W [n_e][n_e] (any may be NULL) into host or device buffers.
 * Synchronises and reports sticky kernel errors. */
int gimbal_stats_read(gimbal_stats_t h, uint64_t* A, uint64_t* E, uint64_t* W, int mem);
/* flat_activation() (moe.cpp:207-215) as doubles [L][L*n_e], and flat_pair_weights()
 * (moe.cpp:217-231) as doubles [m][m] (either may be NULL; m = L*n_e; host or device). */
int gimbal_stats_flat(gimbal_stats_t h, double* flat_activation, double* flat_pair_weights, int mem);
/* Device pointers of the handle's counters, for in-place collectives over the token shards of
 * several ranks (ncclAllReduce(ncclUint64, ncclSum) on E, then gimbal_stats_mark_reduced).
 * E has (L-1)*n_e*n_e uint64 (NULL when L == 1, then A is the counted buffer). */
int gimbal_stats_device_buffers(gimbal_stats_t h, uint64_t** E, uint64_t** A, void** stream);
/* After an external in-place reduction of E (or A when L == 1) over ranks: sets the token count
 * to the global total and re-derives A / W. */
int gimbal_stats_mark_reduced(gimbal_stats_t h, int64_t global_tokens);
/* Synchronises the handle's stream and returns sticky errors. */
int gimbal_stats_sync(gimbal_stats_t h);
/* Kernel timing of the trace-counting launches (CUDA events on the handle's stream around every
 * counting kernel).  enable = 1 starts recording (clears totals), 0 stops; when count_ms /
 * launches are non-NULL, synchronises and returns the summed device time and launch count. */
int gimbal_stats_count_timing(gimbal_stats_t h, int enable, double* count_ms, int64_t* launches);
/* Adds externally held counts into the handle: E [(L-1)][n_e][n_e] (or A [L][n_e] when L == 1)
 * and their token count (host or device).  Restores a snapshot taken with gimbal_stats_read
 * (checkpoint / resume of windowed statistics), copies a handle, or merges a peer's shard. */
int gimbal_stats_merge(gimbal_stats_t h, const uint64_t* counts, int64_t tokens, int mem);

/* ---- placement over the handle's statistics (placement.cpp:58-85, 186-331) ---- */

/* eval_cost for a batch of candidate placements [C][m] (uint8 GPU ids), m = L*n_e, on
 * A = flat_activation(), W = flat_pair_weights() without materialising W (placement.cpp:58-85).
 * Per candidate: deviation D, cut, objective = alpha*D + beta*cut (IEEE double, unfused).
 * argmin = lowest index among the minimal objectives (may be NULL).  Outputs host or device
 * (`out_mem`); candidates host or device (`cand_mem`).  A candidate that violates
 * check_feasible (placement.cpp:30-50) fails the call with GIMBAL_INVALID_ARGUMENT. */
int gimbal_eval_costs(gimbal_stats_t h, const uint8_t* candidates, int64_t n_candidates,
                      int cand_mem, double alpha, double beta, double* deviation, double* cut,
                      double* objective, int64_t* argmin, int out_mem);

/* Hotspot measure per candidate: the bottleneck excess sum_l max(0, peak_l * g / (T * k) - 1),
 * peak_l = the most loaded GPU's activation count in layer l under the candidate placement, T * k
 * = the activations per layer -- the simulator's per-iteration hotspot penalty (sim.cpp:132-144)
 * over the handle's counted trace, in the reference's double arithmetic.  Candidates [C][m]
 * uint8 (host or device), excess [C] doubles (host or device). */
int gimbal_eval_excess(gimbal_stats_t h, const uint8_t* candidates, int64_t n_candidates, int cand_mem,
                       double* excess, int out_mem);

/* build_affinity_set (placement.cpp:186-238) on the handle's E: pairs with count >= threshold
 * and > 0, ordered by count desc then flat ids asc, truncated to top_e (top_e < 0 keeps all),
 * then lightest pairs dropped until the endpoint union fits `capacity`.  Writes the sorted
 * member ids (at most min(2*top_e, capacity) when top_e >= 0, else capacity) to host `out`. */
int gimbal_affinity_set(gimbal_stats_t h, double threshold, int32_t top_e, int32_t capacity,
                        int32_t anchor_gpu, int32_t* out, int32_t* n_out);

/* greedy_place (placement.cpp:240-299) on the handle's flat activation with affinity set M
 * (sorted unique flat ids, host) anchored on anchor_gpu.  Writes m int32 GPU ids to `out`
 * (host or device per out_mem).  Also writes them as uint8 to `out_u8` if non-NULL (device),
 * e.g. row 0 of a candidate batch. */
int gimbal_greedy_place(gimbal_stats_t h, const int32_t* M, int32_t n_M, int32_t anchor_gpu,
                        int32_t* out, int out_mem, uint8_t* out_u8_device);

/* One tumbling window of streaming re-placement (MoeSubsystem::on_forward_step, sim.cpp:149-165,
 * with the strong-pair set fixed after calibration, sim.cpp:94-104), queued on the handle's stream
 * with no host synchronisation (one exception: when tokens * top_k^2 >= 2^27 the evaluator first reads
 * the largest E cell back to pick 32- or 64-bit partial sums): greedy_place (placement.cpp:240-299) with M anchored on
 * anchor_gpu -> `placement` (m int32, device) and row 0 of `candidates` (uint8 [C][m], device),
 * then eval_cost of all C candidates (placement.cpp:58-85) -> `scores` (device f64 [3][C]: D, cut,
 * objective) and `argmin` (device int64, lowest index on ties).  M is validated (reference
 * messages) and uploaded only when it differs from the previous call's.  Device-side errors
 * (infeasible candidate, overflow) are deferred: the next gimbal_stats_sync reports them.  With
 * two handles a caller pipelines window w+1's counting behind window w's placement. */
int gimbal_window_place_async(gimbal_stats_t h, const int32_t* M, int32_t n_M, int32_t anchor_gpu,
                              uint8_t* candidates_device, int64_t n_candidates, double alpha, double beta,
                              double* scores_device, int64_t* argmin_device, int32_t* placement_device);

/* The whole placement half of the north-star pass queued on the handle's stream with no host
 * synchronisation (same max-cell exception as gimbal_window_place_async): build_affinity_set (placement.cpp:186-238; members -> `members` [m] and
 * `n_members` [1], device int32) -> greedy_place with that set on anchor_gpu (placement.cpp:240-299;
 * -> `placement` [m] int32 and row 0 of `candidates`) -> eval_cost of all C candidates ->
 * `scores` [3][C] f64 and `argmin` [1] int64 (device).  capacity must be <= m/g (the reference's
 * greedy_place would reject a larger set).  Device-side errors are reported by the next
 * gimbal_stats_sync; when `flags_device` (2 x u32, may be NULL) is given, the handle's error words
 * are copied there at the end of the pass, so a caller reading its results back can skip that sync
 * when both are zero. */
int gimbal_pass_async(gimbal_stats_t h, double threshold, int32_t top_e, int32_t capacity, int32_t anchor_gpu,
                      uint8_t* candidates_device, int64_t n_candidates, double alpha, double beta,
                      double* scores_device, int64_t* argmin_device, int32_t* placement_device,
                      int32_t* members_device, int32_t* n_members_device, uint32_t* flags_device);

/* One whole pass on a device trace as a CUDA graph: reset + add_tokens (device ids) +
 * gimbal_pass_async with the same arguments.  The first call runs eagerly (validation, scratch
 * sizing), the second records the step on the handle's stream as a graph, and every later call
 * with identical arguments (pointers, sizes, parameters; the data behind them may change)
 * replays it with one launch -- for launch-bound small shapes (Mixtral class: ~10 kernels a
 * pass).  Counting-kernel timing (gimbal_stats_count_timing) covers replays through event-record
 * nodes.  Not for concurrent use of the handle from another thread while recording. */
int gimbal_pass_graph(gimbal_stats_t h, const void* ids_device, int id_bytes, int64_t n_tokens, double threshold,
                      int32_t top_e, int32_t capacity, int32_t anchor_gpu, uint8_t* candidates_device,
                      int64_t n_candidates, double alpha, double beta, double* scores_device, int64_t* argmin_device,
                      int32_t* placement_device, int32_t* members_device, int32_t* n_members_device,
                      uint32_t* flags_device);

/* gimbal_pass_graph as one queued unit for back-to-back passes from a host that owns another
 * stream (a framework's current stream): the handle's stream first waits for caller_stream (the
 * inputs may still be being written there), the pass replays, its packed results
 *   [argmin (int64) | |M| (int32) | pad | error words 0-1 (uint32) | M (m x int32) | greedy (m x int32)]
 * (6 + 2m int32 words; the pass writes them into packed_device) reach host memory, and
 * caller_stream then waits for all of it (so memory the caller frees afterwards is reused only
 * behind the pass).  *results_host says where they will be: packed_host (pinned or registered,
 * same size) after a device-to-host copy queued behind the pass, or -- for the fused small-shape
 * pass, which writes them into mapped host memory itself -- a slot of the handle's 64-slot ring,
 * valid until 64 more passes are queued on the handle.  No host synchronisation: the caller
 * records an event on caller_stream after this returns and reads *results_host once that event has
 * completed; nonzero error words mean gimbal_stats_sync reports the deferred error.  caller_stream
 * may be 0 (the legacy default stream) or the handle's own stream (no joins). */
int gimbal_pass_enqueue(gimbal_stats_t h, const void* ids_device, int id_bytes, int64_t n_tokens, double threshold,
                        int32_t top_e, int32_t capacity, int32_t anchor_gpu, uint8_t* candidates_device,
                        int64_t n_candidates, double alpha, double beta, double* scores_device,
                        int32_t* packed_device, int32_t* packed_host, void* caller_stream, int32_t** results_host);

/* Counting kernels of this handle run on n_sms SMs (default: all).  Leaving SMs free lets a
 * latency-bound kernel on another stream (the previous window's greedy walk) run alongside. */
int gimbal_stats_set_count_sms(gimbal_stats_t h, int n_sms);

/* ---- multi-GPU: token shards over ranks, NCCL over NVLink ----
 * A, E and W are sums over tokens (moe.cpp:169-191), so ranks count contiguous token shards and
 * one in-place SUM all-reduce of the u64 counts gives every rank the counts of the whole trace;
 * the strong-pair set and greedy (placement.cpp:186-299) are then recomputed identically per
 * rank, candidates are split into contiguous slices, and a MIN all-reduce of the per-candidate
 * objectives yields the global argmin (lowest index on ties, as the single-GPU argmin).  NCCL is
 * resolved at run time from the process's libnccl.so.2 (no link dependency). */
#define GIMBAL_DIST_UNIQUE_ID_BYTES 128
typedef void* gimbal_comm_t; /* an ncclComm_t: from gimbal_dist_comm_init, or the caller's own */
/* ncclGetUniqueId: rank 0 calls it and shares the bytes with the other ranks out of band. */
int gimbal_dist_unique_id(void* unique_id);
/* ncclCommInitRank on `device` (one rank per GPU). */
int gimbal_dist_comm_init(int32_t n_ranks, int32_t rank, const void* unique_id, int device, gimbal_comm_t* out);
int gimbal_dist_comm_destroy(gimbal_comm_t comm);
int gimbal_dist_comm_size(gimbal_comm_t comm, int32_t* n_ranks, int32_t* rank);
/* In-place SUM all-reduce of the handle's counts (E, or A when L == 1) over `comm`, queued on the
 * handle's stream behind its counting (no host synchronisation).  global_tokens >= 0 sets the
 * token count; < 0 leaves it on the device (gimbal_stats_tokens reads it back as sum_j A(0,j)/k). */
int gimbal_stats_allreduce(gimbal_stats_t h, gimbal_comm_t comm, int64_t global_tokens);
/* Global argmin over the ranks' candidate slices, queued on the handle's stream: this rank's
 * objectives [n_local] (device) land at [offset, offset + n_local) of `global_objectives` [n_total]
 * (device scratch, +inf elsewhere), a MIN all-reduce merges the ranks, and the lowest index of the
 * minimum goes to argmin_device. */
int gimbal_dist_merge_argmin(gimbal_stats_t h, gimbal_comm_t comm, const double* objectives_device,
                             int64_t n_local, int64_t offset, int64_t n_total, double* global_objectives_device,
                             int64_t* argmin_device);
/* One rank's whole distributed pass, queued on the handle's stream with no host synchronisation:
 * gimbal_stats_allreduce (token count left on the device) -> gimbal_pass_async on this rank's
 * candidate slice -> gimbal_dist_merge_argmin.  Global candidate 0 is the greedy placement.  The
 * rank holding global candidates [cand_offset, cand_offset + n_local) passes them in
 * `candidates_device` with one extra leading scratch row (which receives the greedy placement)
 * unless cand_offset == 0 and n_local > 0 (its row 0 is global candidate 0 itself): rows =
 * n_local + lead, lead = (cand_offset == 0 && n_local > 0) ? 0 : 1.  scores_device: [3][rows];
 * global_objectives_device: [n_total] scratch; argmin_device: the global argmin. */
int gimbal_pass_distributed_async(gimbal_stats_t h, gimbal_comm_t comm, double threshold, int32_t top_e,
                                  int32_t capacity, int32_t anchor_gpu, uint8_t* candidates_device, int64_t n_local,
                                  int64_t cand_offset, int64_t n_total, double alpha, double beta,
                                  double* scores_device, double* global_objectives_device, int64_t* argmin_device,
                                  int32_t* placement_device, int32_t* members_device, int32_t* n_members_device,
                                  uint32_t* flags_device);

/* ---- the online expert-layer hook: MoeHook::iteration_cost (sim.cpp:113-147) on the GPU ----
 * Replaces the per-token host loop of MoeSubsystem (engine.hpp:56-68, called once per engine
 * iteration from Engine::try_start_iteration, engine.cpp:149-152).  The routed ids of one batch
 * are counted into a window statistics handle (RoutingStats::add_token semantics), and the
 * layer x GPU load histogram under the current placement, the cross-GPU transitions
 * (token_crossings, sim.cpp:183-198) and the bottleneck excess sum_l max(0, peak_l * g / (n * k) - 1)
 * (sim.cpp:132-144, the reference's double arithmetic in layer order) come back per call; the
 * per-GPU activation totals (gpu_activation_total_, report.expert_load) accumulate on the device.
 * One CUDA graph per call (H2D ids, two kernels, 16-byte D2H). */
typedef struct gimbal_online_s* gimbal_online_t;
/* Per-iteration state counting into `window` (its device, stream and topology; n_e <= 256). */
int gimbal_online_create(gimbal_stats_t window, gimbal_online_t* out);
int gimbal_online_destroy(gimbal_online_t o);
/* The placement the loads are measured under (m int32 GPU ids, host). */
int gimbal_online_set_placement(gimbal_online_t o, const int32_t* assign, int64_t m);
/* One iteration: n tokens of [n][L][k] ids (host; id_bytes 1 or 4).  Synchronises (the engine's
 * iteration time depends on the result). */
int gimbal_online_iteration(gimbal_online_t o, const void* ids, int id_bytes, int64_t n, double* excess_sum,
                            int64_t* crossings);
/* Activations per GPU over every iteration so far (g int64, host). */
int gimbal_online_gpu_totals(gimbal_online_t o, int64_t* out);

/* ---- the reference's general dense forms (PlacementProblem with arbitrary A / W) ---- */

/* eval_cost (placement.cpp:58-85) on dense A [rows][m] and W [m][m] doubles (host). */
int gimbal_eval_cost_dense(int32_t rows, int32_t m, const double* A, const double* W, int32_t g,
                           double alpha, double beta, const int32_t* assign, double* deviation,
                           double* cut, double* objective);
/* exact_solve (placement.cpp:87-184, placement.hpp:49-51): the objective-minimal balanced placement
 * of m <= 16 experts on g <= 4 GPUs, the lexicographically least (labels in first-use order) among
 * ties, as the reference's branch and bound returns it; every placement is scored on the GPU.  The
 * assignment (m int32) and eval_cost of it go to host memory.  A / W must be non-negative,
 * integer-valued doubles below 2^40 (else GIMBAL_NOT_SUPPORTED); too large an instance returns
 * GIMBAL_INVALID_ARGUMENT with the reference's message.  Replaces: placement::exact_solve. */
int gimbal_exact_solve_dense(int32_t rows, int32_t m, const double* A, const double* W, int32_t g,
                             double alpha, double beta, int32_t* assign_out, double* deviation,
                             double* cut, double* objective);
/* build_affinity_set from an explicit double tensor E [(n_blocks)][n_e][n_e] (host). */
int gimbal_affinity_set_dense(const gimbal_topology* topo, const double* E, int32_t n_blocks,
                              double threshold, int32_t top_e, int32_t capacity,
                              int32_t anchor_gpu, int32_t* out, int32_t* n_out);
/* greedy_place on a dense double activation [rows][m] (host). */
int gimbal_greedy_place_dense(int32_t rows, int32_t m, const double* activation,
                              const int32_t* M, int32_t n_M, int32_t anchor_gpu, int32_t g,
                              int32_t* out);
/* static_placement (placement.cpp:320-331): m int32 to host `out`. */
int gimbal_static_placement(const gimbal_topology* topo, int32_t* out);

/* ---- comm_cost (moe.cpp:241-267) ---- */
/* Cross-GPU transition count of a [T][L][k] trace under expert_to_gpu (m int32, host). */
int gimbal_comm_cost(const gimbal_topology* topo, const void* ids, int id_bytes, int64_t n_tokens,
                     int mem, const int32_t* expert_to_gpu, int32_t n_assign, int device,
                     int64_t* out);

/* ---- synthetic routing traces (RoutingModel semantics, moe.cpp:43-160; distributional) ---- */
/* Zipf(zipf_s) base weights over a per-layer permutation seeded like the reference
 * (Rng(mix_seed(model_seed, 0x5a1f)).shuffle, moe.cpp:61-71), mixed with the successor kernel
 * (lambda, affinity_peak) conditioned on the previous layer's choices; top_k distinct draws.
 * `drift` in [0,1]: fraction of each layer's rank permutation re-drawn (config 5 streaming
 * windows; 0 = the reference model).  Writes n_tokens x L x k uint8 ids to device `out`,
 * tokens numbered from first_token (a counter-based stream: any token range is reproducible). */
int gimbal_generate_trace(const gimbal_topology* topo, double zipf_s, double lambda,
                          double affinity_peak, uint64_t model_seed, uint64_t stream_seed,
                          double drift, uint64_t drift_epoch, int64_t first_token,
                          int64_t n_tokens, uint8_t* out_device, int device);
/* Host tables the generator uses (for the bit-exact CPU twin in oracle/): cdf [L][n_e] u32
 * (inclusive cumulative base weights scaled to 2^32), component thresholds thr[2] in [0, 2^32]
 * (u < thr[0]: base draw, u < thr[1]: uniform draw, else successor of a previous-layer slot). */
int gimbal_generator_tables(const gimbal_topology* topo, double zipf_s, double lambda,
                            double affinity_peak, uint64_t model_seed, double drift,
                            uint64_t drift_epoch, uint32_t* cdf, uint64_t* thr);

/* Balanced random candidates by the reference recipe (acceptance_main.cpp:344-351):
 * assign[e] = e % g, then Rng(seed + c).shuffle (mt19937_64, rng.hpp:64-71), for c in
 * [0, n); writes [n][m] uint8 to host `out`. */
int gimbal_shuffled_candidates(int32_t m, int32_t g, uint64_t seed, int64_t n, uint8_t* out);

#ifdef __cplusplus
}
#endif

#endif /* GIMBAL_GPU_H_ */
