// Shared declarations of the libdeft_b200 translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define DEFT_MAX_EXACT_CAPACITY_DEV 10000000LL  // knapsack.py:16

namespace deft {

// ---- launch accounting (deft_launch_count) --------------------------------
void count_launch(uint64_t n = 1);

// ---- K1 subset-sum --------------------------------------------------------
struct SubsetSumLaunch {
  const int64_t* weights;
  const int32_t* item_off;
  const int64_t* caps;
  const int64_t* row_off;
  const int64_t* meta_off;
  uint32_t* rows;
  int32_t* meta;
  uint8_t* take;
  int64_t* best;
  const int32_t* pids_small;  // problems whose row fits in shared memory
  int32_t n_small;
  int64_t max_small_words;
  const int32_t* pids_large;  // problems on the global-memory row path
  int32_t n_large;
};
cudaError_t launch_subset_sum(const SubsetSumLaunch& L, cudaStream_t stream);
int64_t host_scaled_cap(int64_t cap0);
int64_t host_row_words(int64_t cap0);
int64_t smem_words_limit();

// ---- bucket communication + fused update ----------------------------------
constexpr int kMaxWorld = 8;
constexpr int kMaxCommBlocks = 256;
// flag area layout (uint32): [kNumBarrierSets][kMaxCommBlocks][kMaxWorld] peer-written
// epoch words, then [kNumBarrierSets][kMaxCommBlocks] rank-private epoch counters
enum BarrierSet : int { kBarrierRS = 0, kBarrierCE = 1, kBarrierUpdate = 2, kNumBarrierSets = 3 };

struct PeerPtrs {
  char* grads[kMaxWorld];
  void* params[kMaxWorld];   // same dtype as the gradients (fp32 or bf16)
  uint32_t* flags[kMaxWorld];
  float* master;             // this rank's fp32 master copy when params are bf16, else null
  // CTA cap of every kernel that meets its peers in a barrier (0 = none).  A
  // loopback world (W ranks on ONE GPU) sets it so that all ranks' blocks of a
  // barrier kernel are co-resident.  Equal on every rank (grids must match).
  int32_t grid_cap;
  // a barrier spin longer than this traps (0 = unbounded): a peer that never
  // arrives becomes a loud kernel fault instead of a hung GPU
  uint64_t spin_timeout_ns;
  // PROFILING ONLY (DEFT_PROFILE_NO_PEER_BARRIER=1): peer barriers return at once,
  // so a kernel profiler can replay one rank's launch without its peers (the
  // results are then racy -- never set outside an ncu capture)
  int32_t no_peer_barrier;
  // DEFT_BARRIER_FENCE=all: every thread executes membar.sys before a peer barrier
  int32_t barrier_fence_all;
  // DIAGNOSTICS (deft_comm_set_phase_trace): when set, thread 0 of every block of
  // the TMA reduce-scatter / TMA update / one-shot kernels stores globaltimer
  // stamps at phase boundaries: phase_ts[block * kPhases + k]
  uint64_t* phase_ts;
};
constexpr int kPhases = 8;  // start | epoch | entry barrier | first data | body | drain | exit

// grid of a peer-barrier kernel after the communicator's cap
__host__ inline int cap_grid(const PeerPtrs& P, int grid) {
  return (P.grid_cap > 0 && grid > P.grid_cap) ? P.grid_cap : grid;
}

struct ShardRange {
  int64_t lo, hi;  // absolute element range [lo, hi) of this rank's shard
};

// Absolute element shard [lo, hi) of rank `r` for bucket [offset, offset+numel):
// interior boundaries are 16-byte aligned so the body can use 128-bit accesses.
__host__ __device__ inline ShardRange shard_of(int64_t offset, int64_t numel, int r, int world,
                                               int align_elems) {
  const int64_t per = (numel + world - 1) / world;
  auto bound = [&](int k) -> int64_t {
    if (k <= 0) return offset;
    if (k >= world) return offset + numel;
    int64_t b = offset + (int64_t)k * per;
    b = (b + align_elems - 1) / align_elems * align_elems;
    return b < offset + numel ? b : offset + numel;
  };
  return ShardRange{bound(r), bound(r + 1)};
}

int comm_grid_for(int64_t elems_per_rank);

// one-shot bucket sync: all-reduce of the full buckets (every rank reads every
// peer) fused with the update, parameters written locally (bucket_comm.cu)
cudaError_t launch_oneshot_update(const PeerPtrs& P, int rank, int world, int dtype,
                                  int64_t slot_base, int32_t count, const int64_t* offsets,
                                  const int64_t* numels, float lr, float momentum,
                                  float grad_scale, float* mom, int max_blocks,
                                  cudaStream_t stream);

// loopback collectives (one launch, gridDim.y = world; synchronous)
cudaError_t launch_barrier_loopback(const PeerPtrs& P, int world, int set, cudaStream_t stream);
cudaError_t launch_rs_tma_loopback(const PeerPtrs& P, int world, int dtype, int64_t slot_base,
                                   int32_t count, const int64_t* offsets, const int64_t* numels,
                                   cudaStream_t stream);
cudaError_t launch_update_tma_loopback(const PeerPtrs& P, int world, int dtype,
                                       int64_t slot_base, int32_t count,
                                       const int64_t* offsets, const int64_t* numels,
                                       float lr, float momentum, float grad_scale,
                                       float* const* moms, float* const* masters,
                                       int max_blocks, cudaStream_t stream);

cudaError_t launch_reduce_scatter_sm(const PeerPtrs& P, int rank, int world, int dtype,
                                     int64_t slot_base, int64_t offset, int64_t numel,
                                     cudaStream_t stream);
cudaError_t launch_reduce_scatter_sm_multi(const PeerPtrs& P, int rank, int world, int dtype,
                                           int64_t slot_base, int32_t count,
                                           const int64_t* offsets, const int64_t* numels,
                                           cudaStream_t stream);
cudaError_t launch_barrier(const PeerPtrs& P, int rank, int world, int set,
                           cudaStream_t stream);
cudaError_t launch_ce_reduce(char* own_grad_slot, const char* staging, int dtype, int world,
                             int rank, int64_t shard_lo, int64_t shard_len,
                             int64_t staging_stride_elems, cudaStream_t stream);
cudaError_t launch_update_allgather(const PeerPtrs& P, int rank, int world, int dtype,
                                    int64_t slot_base, int64_t offset, int64_t numel, float lr,
                                    float momentum, float grad_scale, float* mom,
                                    int max_blocks, cudaStream_t stream);
cudaError_t launch_sgd_local(const void* grad, int dtype, void* param, float* master,
                             float* mom, int32_t count, const int64_t* offsets, const int64_t* numels,
                             const float* scales, float lr, float momentum,
                             cudaStream_t stream);

cudaError_t launch_update_allgather_multi(const PeerPtrs& P, int rank, int world, int dtype,
                                          int64_t slot_base, int32_t count,
                                          const int64_t* offsets, const int64_t* numels,
                                          float lr, float momentum, float grad_scale,
                                          float* mom, int max_blocks, cudaStream_t stream);
// State a scheduler instance carries from one chunk of iterations to the next
// (pending updates are always flushed at the end of a backward stage).
struct SchedCarry {
  int32_t cur_uid, cur_first, cur_k, cur_count;
  int64_t cur_backlog;
  int32_t fut_uid, fut_first, fut_k, next_uid;
  uint8_t in_cur[1032];  // by bucket id, n <= 1024
};

struct SchedArgs {
  int32_t n, L, T;
  const int64_t* comm;     // [n+1], by bucket id (index 0 unused)
  const int64_t* bwd;      // [n+1] backward_us (level caps; exact mode never needs them)
  const int64_t* fcaps;    // [instances][L] forward-stage link capacities
  const int64_t* bcaps;    // [instances][L] backward-stage link capacities
  uint32_t* rows;          // [instances][(n+1) * words]
  int64_t words;           // row words for the largest dual capacity of the batch
  int32_t* reach;          // [instances][n+1]
  int32_t* out;            // [instances][out_stride] decision records
  int64_t out_stride;
  int32_t* status;         // [instances]
  int64_t* used;           // [instances] ints written to `out`
  int64_t smem_row_words;  // row words the launch's dynamic shared memory can hold
  int32_t t0;              // iteration index of the first iteration of this chunk
  const SchedCarry* carry_in;  // [instances] or null (fresh schedulers)
  SchedCarry* carry_out;       // [instances] or null
};
int64_t sched_smem_bytes(int64_t words);
cudaError_t launch_scheduler(const SchedArgs& a, int32_t instances, int64_t smem,
                             cudaStream_t stream);
cudaError_t launch_gather(char* dst, const void* const* srcs, const int64_t* dst_off,
                          const int64_t* lens, int32_t count, int64_t ce_min,
                          cudaStream_t stream);

}  // namespace deft
