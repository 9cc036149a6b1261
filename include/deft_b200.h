/*
 * deft_b200.h -- C-ABI of the B200-native DeFT hot path (libdeft_b200.so).
 *
 * The reference (deftsim, pure Python) has no FFI; its drop-in boundary is the
 * Python API.  Every entry point below replaces one piece of that API, cited as
 * reference file:line (paths relative to /root/reference/pkg/src/deftsim):
 *
 *   subset-sum solver ...... naive_knapsack         knapsack.py:55-94
 *                            recursive_knapsack     knapsack.py:97-127 (batched levels)
 *   bucket communication ... the simulated link transfer  simulator.py:136-147, 184-196
 *   delayed SGD update ..... the implicit update event    scheduler.py:56-61, 223-241;
 *                                                         simulator.py:238-243
 *
 * Conventions: plain pointers and sizes, no torch types.  Every function
 * returns 0 (DEFT_OK) or a negative deft_status_t; deft_last_error() gives the
 * thread-local message.  The Python wrapper (paper_2503_16815_b200/_native.py)
 * re-raises them as the matching DeftError subclass (errors.py:7-60).
 * Pointers named d_* are device pointers; `stream` is a cudaStream_t passed as
 * void* so this header needs no CUDA include.
 */
#ifndef DEFT_B200_H_
#define DEFT_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t deft_status_t;
#define DEFT_OK 0
#define DEFT_ERR_INVALID_ARGUMENT (-1) /* -> DeftError            */
#define DEFT_ERR_CUDA (-2)             /* -> DeviceError          */
#define DEFT_ERR_WORKSPACE (-3)        /* -> DeviceError          */
#define DEFT_ERR_UNSUPPORTED (-4)      /* -> DeviceError          */
#define DEFT_ERR_PEER (-5)             /* -> DeviceError          */

/* knapsack.py:16 */
#define DEFT_MAX_EXACT_CAPACITY 10000000LL

int32_t deft_abi_version(void);
const char* deft_last_error(void);
/* Number of kernels this library has launched in this process (all devices). */
uint64_t deft_launch_count(void);

/* ------------------------------------------------------------------------
 * K1  batched subset-sum (weight == value) with include-earliest reconstruction.
 *
 * Problem p owns items [item_off[p], item_off[p+1]) of `weights`, ordered by
 * ASCENDING bucket id, with ORIGINAL integer-us weights (> 0) and an original
 * capacity cap[p] >= 1.  The kernel applies the reference's scaling
 * (knapsack.py:47-52: q = ceil(cap/1e7), w' = ceil(w/q), cap' = cap // q, in
 * IEEE double exactly as CPython evaluates it), builds the suffix bitsets
 * (knapsack.py:72-78), takes the highest reachable sum (:79) and reconstructs
 * the include-earliest optimum (:80-88).  take[i] = 1 for chosen items;
 * best[p] = the optimum in SCALED units.
 * ------------------------------------------------------------------------ */

/* Workspace (bytes) for a batch, given host copies of item counts and caps. */
size_t deft_subset_sum_workspace_bytes(int32_t batch, const int32_t* n_items,
                                       const int64_t* caps);

/* Stream-ordered solve on device buffers. d_item_off has batch+1 entries.
 * d_ws must be at least deft_subset_sum_workspace_bytes() bytes; the host
 * arrays n_items/caps are needed to lay the workspace out. */
deft_status_t deft_subset_sum_batched(const int64_t* d_weights, const int32_t* d_item_off,
                                      const int64_t* d_caps, int32_t batch,
                                      const int32_t* n_items, const int64_t* caps,
                                      uint8_t* d_take, int64_t* d_best, void* d_ws,
                                      size_t ws_bytes, void* stream);

/* Synchronous host convenience used by the Python scheduler: a solver owns a
 * high-priority stream, pinned staging and a growing device workspace. */
typedef struct deft_solver deft_solver;
deft_status_t deft_solver_create(int32_t device, deft_solver** out);
deft_status_t deft_solver_destroy(deft_solver* s);
/* Host arrays in, host arrays out; one H2D copy, <= 2 launches, one D2H copy. */
deft_status_t deft_solver_solve(deft_solver* s, int32_t batch, const int32_t* n_items,
                                const int64_t* weights, const int64_t* caps,
                                uint8_t* take_out, int64_t* best_out);
/* K5: the DeFT delayed-update state machine (scheduler.py:159-342) for
 * `instances` independent schedulers over one partitioned profile (n buckets,
 * ids 1..n; comm / backward times in us) and n_links links, each instance with
 * its own per-link forward / backward stage capacities (the host computes them
 * with the reference's float rounding, scheduler.py:121-125), `iterations`
 * iterations, ONE persistent launch (one CTA per instance).  Writes compact
 * decision records (layout: csrc/scheduler_kernel.cu) into out[i*out_stride..],
 * used[i] ints each, and status[i] (0, or -4 = unsupported: scaled-mode
 * capacities above 1e7 us; -3 = out_stride too small; -6 = invariant). */
deft_status_t deft_solver_schedule(deft_solver* s, int32_t instances, int32_t n,
                                   int32_t n_links, int32_t iterations, const int64_t* comm,
                                   const int64_t* bwd, const int64_t* fwd_caps,
                                   const int64_t* bwd_caps, int32_t* out, int64_t out_stride,
                                   int64_t* used, int32_t* status);
/* The same in chunks, for unbounded runs: iterations [t0, t0+iterations), each
 * instance starting from carry_in[i] (NULL = fresh scheduler) and leaving its
 * state in carry_out[i] (NULL = not needed); carry records are
 * deft_sched_carry_bytes() each, opaque to the caller. */
size_t deft_sched_carry_bytes(void);
deft_status_t deft_solver_schedule_chunk(deft_solver* s, int32_t instances, int32_t n,
                                         int32_t n_links, int32_t t0, int32_t iterations,
                                         const int64_t* comm, const int64_t* bwd,
                                         const int64_t* fwd_caps, const int64_t* bwd_caps,
                                         const void* carry_in, void* carry_out, int32_t* out,
                                         int64_t out_stride, int64_t* used, int32_t* status);
/* Device time (ms) of the kernels of the last solve, measured with CUDA events. */
float deft_solver_last_kernel_ms(const deft_solver* s);

/* ------------------------------------------------------------------------
 * Symmetric device memory for the NVLink/NVSwitch P2P channels.
 * deft_mem_alloc returns a cudaMalloc'ed region plus its 64-byte CUDA IPC
 * handle; peers map it with deft_mem_open (lazy peer access enabled).
 * ------------------------------------------------------------------------ */
#define DEFT_IPC_HANDLE_BYTES 64
deft_status_t deft_mem_alloc(size_t bytes, void** d_ptr, uint8_t* ipc_handle_out);
deft_status_t deft_mem_free(void* d_ptr);
deft_status_t deft_mem_open(const uint8_t* ipc_handle, void** d_peer_ptr);
deft_status_t deft_mem_close(void* d_peer_ptr);

/* ------------------------------------------------------------------------
 * Communicator: one per rank over W <= 8 ranks of one NVSwitch node.
 *   grads[r]  : rank r's gradient arena (n_slots group buffers of `slot_elems`
 *               elements each) -- what autograd writes, what peers read;
 *   params[r] : rank r's flat parameter buffer, output-side bucket first, in the
 *               gradient dtype (fp32, or bf16 for bf16-gradient models);
 *   flags[r]  : rank r's barrier flag area (deft_comm_flag_bytes());
 *   d_master  : this rank's fp32 master parameters (required for bf16, else NULL):
 *               the update reads/writes it and stores bf16 copies to params[*].
 * Pointer arrays are HOST arrays of already-mapped device pointers (own
 * pointer at index `rank`).
 * ------------------------------------------------------------------------ */
typedef struct deft_comm deft_comm;
size_t deft_comm_flag_bytes(int32_t world);
deft_status_t deft_comm_create(int32_t rank, int32_t world, void* const* grads,
                               void* const* params, void* const* flags, float* d_master,
                               int64_t slot_elems, int32_t n_slots, int32_t grad_dtype,
                               deft_comm** out);
deft_status_t deft_comm_destroy(deft_comm* c);
/* CTA budget of the update kernels (0 = default); must be equal on every rank. */
deft_status_t deft_comm_set_update_blocks(deft_comm* c, int32_t blocks);
/* grid_cap (>= 0; 0 = none): CTA cap of every kernel that meets its peers in a
 * barrier -- a loopback world (W ranks in one process on ONE GPU, peer
 * pointers local) sets about 148/(2W) so that all ranks' blocks are
 * co-resident.  spin_timeout_ms (>= 0; 0 = unbounded; default
 * DEFT_SPIN_TIMEOUT_MS or 120000): a barrier spin longer than this traps
 * instead of hanging the GPU.  A negative argument keeps the current value.
 * Both must be equal on every rank. */
deft_status_t deft_comm_configure(deft_comm* c, int32_t grid_cap, int64_t spin_timeout_ms);
/* Diagnostics (no reference counterpart): dev_stamps (device, >= 256 x 8
 * uint64, or NULL to stop) receives globaltimer ns stamps of every block of the
 * TMA reduce-scatter, TMA update + all-gather and one-shot kernels at their
 * phase boundaries [block * 8 + k]: 0 start, 1 epoch read, 2 entry barrier
 * passed, 3 first stage landed, 4 body done, 5 stores drained, 6 end.  Phases a
 * kernel does not have stay untouched.  tools/comm_bench.py --phases. */
deft_status_t deft_comm_set_phase_trace(deft_comm* c, uint64_t* dev_stamps);

/* grad_dtype codes */
#define DEFT_DTYPE_F32 0
#define DEFT_DTYPE_BF16 1

/* Channel ids: the paper's fast / slow links become two NVLink channels. */
#define DEFT_CHANNEL_SM 0 /* SM-driven P2P loads (ratio 1.0, "fast link")     */
#define DEFT_CHANNEL_CE 1 /* copy engines + local SM reduce ("slow link", mu) */

/* Reduce-scatter of bucket [offset, offset+numel) of group slot `slot`:
 * rank r sums shard r over all ranks (fp32 accumulation) and writes it in
 * place into its own slot.  Stream-ordered on `stream`; the cross-rank
 * entry barrier is inside the kernel. Replaces the simulated transfer of one
 * planned bucket (simulator.py:136-147). With world == 1 it is a no-op. */
deft_status_t deft_bucket_reduce_scatter(deft_comm* c, int32_t channel, int32_t slot,
                                         int64_t offset, int64_t numel, void* stream);

/* The transfers one release point puts on one link (simulator.py:184-196: a
 * forward/backward-stage plan, or the fresh buckets that become ready at the
 * same backward moment) in ONE launch with one cross-rank barrier: the same
 * result as `count` deft_bucket_reduce_scatter calls in list order. */
deft_status_t deft_bucket_reduce_scatter_multi(deft_comm* c, int32_t channel, int32_t slot,
                                               int32_t count, const int64_t* offsets,
                                               const int64_t* numels, void* stream);

/* Fused delayed SGD/momentum update of the owned shard + all-gather of the
 * updated parameters to every rank (the update event, scheduler.py:56-61):
 *   g = shard(slot) * grad_scale          (grad_scale = 1 / (W * merge_count))
 *   v = momentum * v + g  ;  p -= lr * v  (torch.optim.SGD, dampening 0)
 * and p is stored to every rank's params (P2P stores over NVLink).  `mom` is
 * this rank's momentum buffer, indexed like params. Entry and exit barriers
 * are inside the kernel. */
deft_status_t deft_bucket_update(deft_comm* c, int32_t slot, int64_t offset, int64_t numel,
                                 float lr, float momentum, float grad_scale, float* d_mom,
                                 void* stream);

/* Every bucket of one update event ([offsets[k], offsets[k]+numels[k]) of slot
 * `slot`, host arrays) in ONE launch with one entry/exit barrier pair per CTA;
 * same arithmetic as deft_bucket_update. */
deft_status_t deft_bucket_update_multi(deft_comm* c, int32_t slot, int32_t count,
                                       const int64_t* offsets, const int64_t* numels, float lr,
                                       float momentum, float grad_scale, float* d_mom,
                                       void* stream);

/* One-shot bucket sync (small buckets): the all-reduce AND the update of
 * every bucket of one update event in ONE launch -- each rank reads the whole
 * of [offsets[k], +numels[k]) from every rank's slot `slot` (own + W-1 peers
 * over NVLink), sums in rank order in fp32, rounds to the gradient dtype and
 * applies g*grad_scale, v = m*v + g, p -= lr*v to the FULL bucket locally
 * (momentum / fp32 master of such buckets are replicated on every rank,
 * bit-identical).  No deft_bucket_reduce_scatter may run for these buckets;
 * entry and exit barriers inside.  Same results as reduce-scatter +
 * deft_bucket_update_multi.  Replaces the simulated transfer + update event
 * of a bucket whose startup cost dominates (simulator.py:136-147). */
deft_status_t deft_bucket_sync_update_multi(deft_comm* c, int32_t slot, int32_t count,
                                            const int64_t* offsets, const int64_t* numels,
                                            float lr, float momentum, float grad_scale,
                                            float* d_mom, void* stream);

/* Local (W == 1 or rank-private) fused update over device arrays:
 * v = m*v + s*g ; p -= lr*v. grad_dtype as above; d_param has the grad dtype;
 * for bf16 the fp32 master d_master is updated and rounded into d_param. */
deft_status_t deft_sgd_momentum_update(const void* d_grad, int32_t grad_dtype, void* d_param,
                                       float* d_master, float* d_mom, int64_t numel, float lr,
                                       float momentum, float grad_scale, void* stream);

/* Multi-bucket variant: one launch updates `count` (offset, numel, scale)
 * segments of the same arrays (the buckets of one update event). Host arrays. */
deft_status_t deft_sgd_momentum_update_multi(const void* d_grad, int32_t grad_dtype,
                                             void* d_param, float* d_master, float* d_mom,
                                             int32_t count,
                                             const int64_t* offsets, const int64_t* numels,
                                             const float* grad_scales, float lr,
                                             float momentum, void* stream);

/* Gather `count` device byte ranges (d_srcs[i], byte_lens[i]) into
 * d_dst + dst_offsets[i]: the per-parameter gradients autograd just produced
 * land in their bucket's contiguous slot range in one launch (the store half
 * of scheduler.py:223-233's store-or-merge; merges accumulate in place).
 * d_srcs / dst_offsets / byte_lens are HOST arrays (copied into the kernel
 * parameters, so CUDA-graph captures keep them).  Ranges of at least
 * ce_min_bytes go through the copy engines instead (no SMs: for a gather that
 * runs beside the backward); 0 = kernel only, < 0 = DEFT_GATHER_CE_MIN
 * (default 4 MiB). */
deft_status_t deft_gather_segments(void* d_dst, const void* const* d_srcs,
                                   const int64_t* dst_offsets, const int64_t* byte_lens,
                                   int32_t count, int64_t ce_min_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Loopback collectives: ONE launch carries every rank of a loopback world
 * (comms[r] = rank r's communicator; all ranks' buffers on the same device;
 * gridDim.y = world).  The peer barriers meet inside one co-resident grid, so
 * these complete even when kernels are serialized (a kernel profiler), where
 * W separate per-rank launches never meet.  Same kernels, arithmetic and
 * results as each rank's deft_bucket_reduce_scatter_multi /
 * deft_bucket_update_multi; synchronous.  d_moms: rank r's momentum buffer.
 * ------------------------------------------------------------------------ */
deft_status_t deft_loopback_reduce_scatter(deft_comm* const* comms, int32_t world,
                                           int32_t channel, int32_t slot, int32_t count,
                                           const int64_t* offsets, const int64_t* numels,
                                           void* stream);
deft_status_t deft_loopback_update(deft_comm* const* comms, int32_t world, int32_t slot,
                                   int32_t count, const int64_t* offsets, const int64_t* numels,
                                   float lr, float momentum, float grad_scale,
                                   float* const* d_moms, void* stream);

/* ------------------------------------------------------------------------
 * Streams and hardware work queues (loopback worlds, loopback.py).
 * deft_stream_create: a non-blocking stream of the given priority.
 * deft_stream_alias_probe: *aliased = 1 if work on stream_b issued after a
 * blocked entry of stream_a waits for it (the two share a hardware queue),
 * measured with a bounded spin of timeout_us; the blocked entry is a kernel
 * (mode 0) or a device-to-device copy (mode 1); synchronizes both streams.
 * ------------------------------------------------------------------------ */
deft_status_t deft_stream_create(int32_t priority, void** out);
deft_status_t deft_stream_destroy(void* stream);
deft_status_t deft_stream_alias_probe(void* stream_a, void* stream_b, int32_t timeout_us,
                                      int32_t mode, int32_t* aliased);

#ifdef __cplusplus
}
#endif
#endif /* DEFT_B200_H_ */
