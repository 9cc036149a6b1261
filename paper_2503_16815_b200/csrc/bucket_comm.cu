// K2/K3/K4: gradient-bucket communication over NVLink / NVSwitch, fused with
// the delayed SGD/momentum update, sm_100a.
//
// The reference only SIMULATES this step: a planned bucket occupies a link for
// comm_fast_us * ratio (simulator.py:136-147, profiles.py:155-157) and a group
// update is bookkeeping once its last bucket is sent (scheduler.py:56-61,
// simulator.py:238-243).  Here it is real, split the way the delayed update
// allows:
//
//  * at the DeFT-planned window (link stream)      -> reduce-scatter:
//      rank r sums shard r of the bucket over all ranks, reading the peers'
//      gradient slots directly over NVLink (SM channel, 128-bit loads, fp32
//      accumulation) or pulling them with the copy engines first (CE channel),
//      and writes the sum in place into its own slot;
//  * at the update's visibility point (update stream) -> fused update + all-gather:
//      v = m*v + g/(W*k); p -= lr*v on the owned shard, and the updated
//      parameters are STORED into every rank's parameter buffer over NVLink.
//    One pass over the shard, no separate elementwise kernel, momentum touched
//    only for the owned 1/W shard.
//
// Cross-rank ordering: per-block barriers on system-scope flags.  Block b of
// rank r only waits for block b of the peers (each block owns the same
// sub-range on every rank), so no kernel ever waits for a whole peer grid.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "common.cuh"

namespace deft {

constexpr int kCommThreads = 512;
constexpr int kLocalThreads = 256;

// CTAs per comm kernel: enough bytes in flight for NVLink, few enough to leave
// the SMs to the concurrent forward/backward.  DEFT_COMM_BLOCKS overrides.
static int comm_max_blocks() {
  static int v = [] {
    const char* e = getenv("DEFT_COMM_BLOCKS");
    int x = e ? atoi(e) : 128;
    if (x < 1) x = 1;
    if (x > kMaxCommBlocks) x = kMaxCommBlocks;
    return x;
  }();
  return v;
}

int comm_grid_for(int64_t elems_per_rank) {
  const int64_t per_block = 16384;  // ~64 KB of fp32 per rank per CTA
  int64_t g = (elems_per_rank + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > comm_max_blocks()) g = comm_max_blocks();
  return (int)g;
}

// ---- system-scope flag primitives -----------------------------------------
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Rank-private epoch counters live right after the peer-written flag words:
// counters[set][block].  Block b of every kernel in barrier set `set` runs in
// the same order on every rank (one stream per set), so the counters advance in
// lock-step without any host involvement -- which keeps the kernels replayable
// inside CUDA graphs.
__device__ __forceinline__ uint32_t* epoch_counter(const PeerPtrs& P, int rank, int set,
                                                   int block) {
  return P.flags[rank] + (int64_t)kNumBarrierSets * kMaxCommBlocks * kMaxWorld +
         (int64_t)set * kMaxCommBlocks + block;
}

// Advance this block's epoch by `step`; returns the previous value (all threads).
__device__ __forceinline__ uint32_t take_epochs(const PeerPtrs& P, int rank, int set,
                                                uint32_t step) {
  __shared__ uint32_t s_epoch;
  if (threadIdx.x == 0) {
    uint32_t* c = epoch_counter(P, rank, set, blockIdx.x);
    const uint32_t e = *c;
    *c = e + step;
    s_epoch = e;
  }
  __syncthreads();
  return s_epoch;
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Diagnostics: globaltimer stamp of phase k of this block (deft_comm_set_phase_trace)
__device__ __forceinline__ void phase_stamp(const PeerPtrs& P, int k) {
  if (P.phase_ts != nullptr && threadIdx.x == 0 && blockIdx.y == 0)
    P.phase_ts[(int64_t)blockIdx.x * kPhases + k] = global_ns();
}

// Block-level barrier with the same-index block on every rank.  The spin is
// bounded by P.spin_timeout_ns: a peer block that never arrives (a launch whose
// blocks cannot all be resident, a rank that died) traps with a message.
//
// Ordering: the flag store is st.release.sys (fence.acq_rel.sys + store) by the
// signalling thread after bar.sync, so every write of the CTA that precedes the
// bar.sync is ordered before it (release cumulativity through the CTA-scope
// barrier -- the cooperative-groups grid-sync pattern); the acquire spin + the
// closing bar.sync order the peers' writes before every thread's later reads.
// DEFT_BARRIER_FENCE=all restores a per-thread membar.sys before the bar.sync
// (round-1 behaviour, kept for A/B).
__device__ __forceinline__ void peer_block_barrier(const PeerPtrs& P, int rank, int world,
                                                   int set, int block, uint32_t value) {
  if (P.barrier_fence_all) __threadfence_system();
  __syncthreads();
  if (P.no_peer_barrier) return;   // profiling only (common.cuh)
  if ((int)threadIdx.x < world) {
    const int peer = threadIdx.x;
    const int64_t base = ((int64_t)set * kMaxCommBlocks + block) * kMaxWorld;
    st_release_sys(P.flags[peer] + base + rank, value);
    const uint32_t* mine = P.flags[rank] + base + peer;
    const uint64_t limit = P.spin_timeout_ns;
    const uint64_t t0 = limit ? global_ns() : 0;
    // wrap-safe "mine >= value"
    uint32_t seen;
    while ((int32_t)((seen = ld_acquire_sys(mine)) - value) < 0) {
      if (limit && global_ns() - t0 > limit) {
        printf("deft: peer barrier timeout: rank %d waits for rank %d (set %d block %d, "
               "epoch %u, seen %u)\n", rank, peer, set, block, value, seen);
        __trap();
      }
    }
  }
  __syncthreads();
}

// ---- element access helpers -----------------------------------------------
template <typename T>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int N = 4;
  using Raw = float4;
  __device__ static void to_f32(const Raw& r, float* o) {
    o[0] = r.x; o[1] = r.y; o[2] = r.z; o[3] = r.w;
  }
  __device__ static Raw from_f32(const float* o) { return make_float4(o[0], o[1], o[2], o[3]); }
  __device__ static float scalar(const float* p) { return *p; }
  __device__ static void put(float* p, float v) { *p = v; }
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  using Raw = uint4;
  __device__ static void to_f32(const Raw& r, float* o) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(h[k]);
      o[2 * k] = f.x;
      o[2 * k + 1] = f.y;
    }
  }
  __device__ static Raw from_f32(const float* o) {
    Raw r;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(o[2 * k], o[2 * k + 1]);
    return r;
  }
  __device__ static float scalar(const __nv_bfloat16* p) { return __bfloat162float(*p); }
  __device__ static void put(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
};

// 4 consecutive elements <-> float4, for fp32 or bf16 storage
__device__ __forceinline__ float4 load4(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ float4 load4(const __nv_bfloat16* p) {
  const uint2 r = *reinterpret_cast<const uint2*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
  const float2 a = __bfloat1622float2(h[0]), b = __bfloat1622float2(h[1]);
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void store4(float* p, const float4& v) {
  *reinterpret_cast<float4*>(p) = v;
}
__device__ __forceinline__ void store4(__nv_bfloat16* p, const float4& v) {
  uint2 r;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
  h[0] = __floats2bfloat162_rn(v.x, v.y);
  h[1] = __floats2bfloat162_rn(v.z, v.w);
  *reinterpret_cast<uint2*>(p) = r;
}
__device__ __forceinline__ void store1(float* p, float v) { *p = v; }
__device__ __forceinline__ void store1(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

template <typename Raw>
__device__ __forceinline__ Raw ld_nc(const Raw* p) {
  return __ldg(p);
}

// Split [lo, hi) into an unaligned scalar head, an aligned vector body and a
// scalar tail; block `blk` of `nblk` gets a contiguous share of the body.
struct Span {
  int64_t head_lo, head_hi, body_lo, body_hi, tail_lo, tail_hi;  // elements
};
template <int N>
__device__ __forceinline__ Span split_span(int64_t lo, int64_t hi) {
  Span s;
  int64_t a = (lo + N - 1) / N * N;
  if (a > hi) a = hi;
  int64_t b = hi / N * N;
  if (b < a) b = a;
  s.head_lo = lo; s.head_hi = a; s.body_lo = a; s.body_hi = b; s.tail_lo = b; s.tail_hi = hi;
  return s;
}

// ============================================================================
// Reduce-scatter, SM channel: shard r = sum over ranks, written in place.
// W is a template parameter so the peer pointers live in registers and every
// loop unrolls; U = 16/W vectors per thread keep 16 independent 128-bit loads
// in flight (the peer-load latency is ~2 us on NVLink).
// ============================================================================
template <typename T, int W>
__global__ void __launch_bounds__(kCommThreads) reduce_scatter_kernel(
    PeerPtrs P, int rank, int64_t slot_base, int64_t lo, int64_t hi) {
  using V = Vec<T>;
  using Raw = typename V::Raw;
  constexpr int U = 16 / W > 0 ? 16 / W : 1;
  const uint32_t epoch = take_epochs(P, rank, kBarrierRS, 1u) + 1u;
  peer_block_barrier(P, rank, W, kBarrierRS, blockIdx.x, epoch);
  const T* src[W];
#pragma unroll
  for (int k = 0; k < W; ++k) src[k] = reinterpret_cast<const T*>(P.grads[k]) + slot_base;
  T* dst = reinterpret_cast<T*>(P.grads[rank]) + slot_base;

  const Span s = split_span<V::N>(lo, hi);
  if (blockIdx.x == 0) {  // unaligned edges
    for (int64_t e = s.head_lo + threadIdx.x; e < s.head_hi; e += blockDim.x) {
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < W; ++k) acc += V::scalar(src[k] + e);
      V::put(dst + e, acc);
    }
    for (int64_t e = s.tail_lo + threadIdx.x; e < s.tail_hi; e += blockDim.x) {
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < W; ++k) acc += V::scalar(src[k] + e);
      V::put(dst + e, acc);
    }
  }
  const int64_t nv = (s.body_hi - s.body_lo) / V::N;
  const int64_t v0 = s.body_lo / V::N;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride * U) {
    Raw raw[U][W];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vi = i + u * stride;
      if (vi < nv) {
#pragma unroll
        for (int k = 0; k < W; ++k) raw[u][k] = ld_nc(reinterpret_cast<const Raw*>(src[k]) + v0 + vi);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vi = i + u * stride;
      if (vi < nv) {
        float acc[V::N], tmp[V::N];
        V::to_f32(raw[u][0], acc);
#pragma unroll
        for (int k = 1; k < W; ++k) {
          V::to_f32(raw[u][k], tmp);
#pragma unroll
          for (int c = 0; c < V::N; ++c) acc[c] += tmp[c];
        }
        reinterpret_cast<Raw*>(dst)[v0 + vi] = V::from_f32(acc);
      }
    }
  }
}

template <typename T>
static void rs_dispatch(int world, int grid, cudaStream_t stream, const PeerPtrs& P, int rank,
                        int64_t slot_base, int64_t lo, int64_t hi) {
#define DEFT_RS_CASE(WW) \
  case WW:               \
    reduce_scatter_kernel<T, WW><<<grid, kCommThreads, 0, stream>>>(P, rank, slot_base, lo, hi); \
    break;
  switch (world) {
    DEFT_RS_CASE(2) DEFT_RS_CASE(3) DEFT_RS_CASE(4) DEFT_RS_CASE(5)
    DEFT_RS_CASE(6) DEFT_RS_CASE(7) DEFT_RS_CASE(8)
    default: break;
  }
#undef DEFT_RS_CASE
}

bool launch_reduce_scatter_tma(const PeerPtrs& P, int rank, int world, int dtype,
                               int64_t slot_base, int64_t offset, int64_t numel,
                               cudaStream_t stream);

bool launch_reduce_scatter_tma_multi(const PeerPtrs& P, int rank, int world, int dtype,
                                     int64_t slot_base, int32_t count, const int64_t* offsets,
                                     const int64_t* numels, cudaStream_t stream);

cudaError_t launch_reduce_scatter_sm_multi(const PeerPtrs& P, int rank, int world, int dtype,
                                           int64_t slot_base, int32_t count,
                                           const int64_t* offsets, const int64_t* numels,
                                           cudaStream_t stream) {
  if (launch_reduce_scatter_tma_multi(P, rank, world, dtype, slot_base, count, offsets, numels,
                                      stream))
    return cudaGetLastError();
  for (int32_t k = 0; k < count; ++k) {   // LDG kernel: one launch per bucket
    cudaError_t e = launch_reduce_scatter_sm(P, rank, world, dtype, slot_base, offsets[k],
                                             numels[k], stream);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_reduce_scatter_sm(const PeerPtrs& P, int rank, int world, int dtype,
                                     int64_t slot_base, int64_t offset, int64_t numel,
                                     cudaStream_t stream) {
  if (launch_reduce_scatter_tma(P, rank, world, dtype, slot_base, offset, numel, stream))
    return cudaGetLastError();
  const int align = dtype == 0 ? 4 : 8;
  const ShardRange sh = shard_of(offset, numel, rank, world, align);
  const int grid = cap_grid(P, comm_grid_for((numel + world - 1) / world));
  if (dtype == 0)
    rs_dispatch<float>(world, grid, stream, P, rank, slot_base, sh.lo, sh.hi);
  else
    rs_dispatch<__nv_bfloat16>(world, grid, stream, P, rank, slot_base, sh.lo, sh.hi);
  count_launch();
  return cudaGetLastError();
}

// ============================================================================
// Barrier-only kernel (CE channel: the copy engines cannot wait on a flag).
// ============================================================================
// loopback: one launch with gridDim.y = world carries every rank (rank = blockIdx.y)
__global__ void barrier_kernel(PeerPtrs P, int rank, int world, int set, int loopback) {
  if (loopback) rank = blockIdx.y;
  const uint32_t epoch = take_epochs(P, rank, set, 1u) + 1u;
  peer_block_barrier(P, rank, world, set, 0, epoch);
}

cudaError_t launch_barrier(const PeerPtrs& P, int rank, int world, int set,
                           cudaStream_t stream) {
  barrier_kernel<<<1, 32, 0, stream>>>(P, rank, world, set, 0);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_barrier_loopback(const PeerPtrs& P, int world, int set, cudaStream_t stream) {
  barrier_kernel<<<dim3(1, world), 32, 0, stream>>>(P, 0, world, set, 1);
  count_launch();
  return cudaGetLastError();
}

// CE channel local reduce: own shard += staged peer shards (128-bit accesses;
// the staged copies and the own shard share their alignment).
template <typename T>
__global__ void __launch_bounds__(kLocalThreads) ce_reduce_kernel(
    T* own, const T* staging, int world, int rank, int64_t len, int64_t stride_elems) {
  using V = Vec<T>;
  using Raw = typename V::Raw;
  const int64_t nv = ((reinterpret_cast<uintptr_t>(own) % 16) == 0 &&
                      (reinterpret_cast<uintptr_t>(staging) % 16) == 0 &&
                      (stride_elems % V::N) == 0) ? len / V::N : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) {
    float acc[V::N], tmp[V::N];
    V::to_f32(reinterpret_cast<const Raw*>(own)[v], acc);
    int slot = 0;
    for (int k = 0; k < world; ++k) {
      if (k == rank) continue;
      V::to_f32(__ldg(reinterpret_cast<const Raw*>(staging + (int64_t)slot * stride_elems) + v),
                tmp);
#pragma unroll
      for (int c = 0; c < V::N; ++c) acc[c] += tmp[c];
      ++slot;
    }
    reinterpret_cast<Raw*>(own)[v] = V::from_f32(acc);
  }
  for (int64_t e = nv * V::N + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < len;
       e += stride) {  // scalar remainder
    float acc = V::scalar(own + e);
    int slot = 0;
    for (int k = 0; k < world; ++k) {
      if (k == rank) continue;
      acc += V::scalar(staging + (int64_t)slot * stride_elems + e);
      ++slot;
    }
    V::put(own + e, acc);
  }
}

cudaError_t launch_ce_reduce(char* own_grad_slot, const char* staging, int dtype, int world,
                             int rank, int64_t shard_lo, int64_t shard_len,
                             int64_t staging_stride_elems, cudaStream_t stream) {
  if (shard_len <= 0) return cudaSuccess;
  int grid = (int)((shard_len + kLocalThreads * 4 - 1) / (kLocalThreads * 4));
  if (grid > 148 * 4) grid = 148 * 4;
  if (dtype == 0)
    ce_reduce_kernel<float><<<grid, kLocalThreads, 0, stream>>>(
        reinterpret_cast<float*>(own_grad_slot) + shard_lo,
        reinterpret_cast<const float*>(staging), world, rank, shard_len, staging_stride_elems);
  else
    ce_reduce_kernel<__nv_bfloat16><<<grid, kLocalThreads, 0, stream>>>(
        reinterpret_cast<__nv_bfloat16*>(own_grad_slot) + shard_lo,
        reinterpret_cast<const __nv_bfloat16*>(staging), world, rank, shard_len,
        staging_stride_elems);
  count_launch();
  return cudaGetLastError();
}

// ============================================================================
// Fused delayed SGD/momentum update of the owned shard + parameter all-gather.
// ============================================================================
template <typename T, int W>
__global__ void __launch_bounds__(kCommThreads) update_allgather_kernel(
    PeerPtrs P, int rank, int64_t slot_base, int64_t lo, int64_t hi, float lr, float momentum,
    float scale, float* __restrict__ mom) {
  using V = Vec<T>;
  constexpr int U = 2;
  constexpr bool kMaster = sizeof(T) == 2;  // bf16 params: fp32 master is authoritative
  // entry: every rank's no-read window for this bucket is open
  const uint32_t epoch = take_epochs(P, rank, kBarrierUpdate, 2u);
  peer_block_barrier(P, rank, W, kBarrierUpdate, blockIdx.x, epoch + 1u);
  const T* g = reinterpret_cast<const T*>(P.grads[rank]) + slot_base;
  float* ref = kMaster ? P.master : reinterpret_cast<float*>(P.params[rank]);
  T* dst[W];
#pragma unroll
  for (int k = 0; k < W; ++k) dst[k] = reinterpret_cast<T*>(P.params[k]);

  const Span s = split_span<4>(lo, hi);
  if (blockIdx.x == 0) {
    auto step = [&](int64_t e) {
      const float v = fmaf(momentum, mom[e], V::scalar(g + e) * scale);
      mom[e] = v;
      const float p = fmaf(-lr, v, ref[e]);
      if (kMaster) ref[e] = p;
#pragma unroll
      for (int k = 0; k < W; ++k) store1(dst[k] + e, p);
    };
    for (int64_t e = s.head_lo + threadIdx.x; e < s.head_hi; e += blockDim.x) step(e);
    for (int64_t e = s.tail_lo + threadIdx.x; e < s.tail_hi; e += blockDim.x) step(e);
  }
  const int64_t nv = (s.body_hi - s.body_lo) / 4;
  const int64_t v0 = s.body_lo / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride * U) {
    float4 g4[U], m4[U], p4[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vi = i + u * stride;
      if (vi < nv) {
        const int64_t e = (v0 + vi) * 4;
        g4[u] = load4(g + e);
        m4[u] = load4(mom + e);
        p4[u] = load4(ref + e);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t vi = i + u * stride;
      if (vi < nv) {
        const int64_t e = (v0 + vi) * 4;
        float4 v4, q4;
        v4.x = fmaf(momentum, m4[u].x, g4[u].x * scale);
        v4.y = fmaf(momentum, m4[u].y, g4[u].y * scale);
        v4.z = fmaf(momentum, m4[u].z, g4[u].z * scale);
        v4.w = fmaf(momentum, m4[u].w, g4[u].w * scale);
        q4.x = fmaf(-lr, v4.x, p4[u].x);
        q4.y = fmaf(-lr, v4.y, p4[u].y);
        q4.z = fmaf(-lr, v4.z, p4[u].z);
        q4.w = fmaf(-lr, v4.w, p4[u].w);
        store4(mom + e, v4);
        if (kMaster) store4(ref + e, q4);
#pragma unroll
        for (int k = 0; k < W; ++k) store4(dst[k] + e, q4);
      }
    }
  }
  // exit: every rank's stores into every parameter buffer have landed
  peer_block_barrier(P, rank, W, kBarrierUpdate, blockIdx.x, epoch + 2u);
}

template <typename T>
static void upd_dispatch(int world, int grid, cudaStream_t stream, const PeerPtrs& P, int rank,
                         int64_t slot_base, int64_t lo, int64_t hi, float lr, float momentum,
                         float scale, float* mom) {
#define DEFT_UP_CASE(WW)                                                               \
  case WW:                                                                             \
    update_allgather_kernel<T, WW><<<grid, kCommThreads, 0, stream>>>(P, rank, slot_base, lo, \
                                                                      hi, lr, momentum, scale, \
                                                                      mom);            \
    break;
  switch (world) {
    DEFT_UP_CASE(2) DEFT_UP_CASE(3) DEFT_UP_CASE(4) DEFT_UP_CASE(5)
    DEFT_UP_CASE(6) DEFT_UP_CASE(7) DEFT_UP_CASE(8)
    default: break;
  }
#undef DEFT_UP_CASE
}

cudaError_t launch_update_allgather(const PeerPtrs& P, int rank, int world, int dtype,
                                    int64_t slot_base, int64_t offset, int64_t numel, float lr,
                                    float momentum, float grad_scale, float* mom,
                                    int max_blocks, cudaStream_t stream) {
  const ShardRange sh = shard_of(offset, numel, rank, world, dtype == 0 ? 4 : 8);
  int grid = comm_grid_for((numel + world - 1) / world);
  if (max_blocks > 0 && grid > max_blocks) grid = max_blocks;
  grid = cap_grid(P, grid);
  if (dtype == 0)
    upd_dispatch<float>(world, grid, stream, P, rank, slot_base, sh.lo, sh.hi, lr, momentum,
                        grad_scale, mom);
  else
    upd_dispatch<__nv_bfloat16>(world, grid, stream, P, rank, slot_base, sh.lo, sh.hi, lr,
                                momentum, grad_scale, mom);
  count_launch();
  return cudaGetLastError();
}

// ============================================================================
// Local fused update (W == 1): one launch covers up to kMaxSeg buckets.
// ============================================================================
constexpr int kMaxSeg = 32;
struct SegTable {
  int64_t off[kMaxSeg];
  int64_t len[kMaxSeg];
  int64_t first_vec[kMaxSeg + 1];  // prefix of per-segment work units
  float scale[kMaxSeg];
  int32_t count;
};

template <typename T, int U>
__global__ void __launch_bounds__(kLocalThreads) sgd_local_kernel(
    const T* __restrict__ grad, T* __restrict__ param, float* __restrict__ master,
    float* __restrict__ mom, const __grid_constant__ SegTable t, float lr, float momentum) {
  using V = Vec<T>;
  constexpr bool kMaster = sizeof(T) == 2;  // bf16 params: fp32 master is authoritative
  float* ref = kMaster ? master : reinterpret_cast<float*>(param);
  const int64_t total = t.first_vec[t.count];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int seg = 0;
  auto one = [&](int64_t e, float s) {
    const float v = fmaf(momentum, mom[e], V::scalar(grad + e) * s);
    mom[e] = v;
    const float p = fmaf(-lr, v, ref[e]);
    if (kMaster) ref[e] = p;
    store1(param + e, p);
  };
  // U units per thread per pass (unit u covers 4 consecutive elements of its
  // segment from the segment's aligned start): all 3U 16-byte loads are issued
  // before the first use, so each thread keeps U x 48 B of HBM reads in flight
  for (int64_t u0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u0 < total;
       u0 += stride * U) {
    float4 g4[U], m4[U], p4[U];
    int64_t el[U];
    float sc[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int64_t u = u0 + q * stride;
      el[q] = -1;
      if (u >= total) continue;
      while (u >= t.first_vec[seg + 1]) ++seg;   // u grows: seg only moves forward
      const int64_t base = t.off[seg];
      const int64_t end = base + t.len[seg];
      const int64_t aligned = (base + 3) / 4 * 4;
      const int64_t k = u - t.first_vec[seg];
      sc[q] = t.scale[seg];
      if (k == 0 && aligned > base) {  // unit 0 also owns the unaligned head
        for (int64_t e = base; e < aligned && e < end; ++e) one(e, sc[q]);
      }
      const int64_t e = aligned + k * 4;
      if (e + 4 <= end) {
        el[q] = e;
        g4[q] = load4(grad + e);
        m4[q] = load4(mom + e);
        p4[q] = load4(ref + e);
      } else {
        for (int64_t x = e; x < end; ++x) one(x, sc[q]);  // tail
      }
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      if (el[q] < 0) continue;
      const float s = sc[q];
      float4 m = m4[q], pp = p4[q];
      m.x = fmaf(momentum, m.x, g4[q].x * s);
      m.y = fmaf(momentum, m.y, g4[q].y * s);
      m.z = fmaf(momentum, m.z, g4[q].z * s);
      m.w = fmaf(momentum, m.w, g4[q].w * s);
      pp.x = fmaf(-lr, m.x, pp.x);
      pp.y = fmaf(-lr, m.y, pp.y);
      pp.z = fmaf(-lr, m.z, pp.z);
      pp.w = fmaf(-lr, m.w, pp.w);
      store4(mom + el[q], m);
      if (kMaster) store4(ref + el[q], pp);
      store4(param + el[q], pp);
    }
  }
}

// DEFT_SGD_UNROLL (1, 2 or 4): units per thread per pass of sgd_local_kernel
static int sgd_unroll() {
  static int v = [] {
    const char* e = getenv("DEFT_SGD_UNROLL");
    const int x = e ? atoi(e) : 2;
    return x == 1 || x == 4 ? x : 2;
  }();
  return v;
}
// DEFT_SGD_CTAS_PER_SM: grid cap of sgd_local_kernel = 148 x this (default 32:
// four waves of 8 resident CTAs per SM, each CTA a short grid-stride loop;
// tools/update_bench.py on ResNet-101's 44.5 M parameters, unroll 2: 32 -> 0.998
// of the HBM peak, 16 -> 0.968-0.974, 8 -> 0.945; unroll 1 x 8 (round 1) -> 0.946;
// profiles/r02_update_w1*.jsonl)
static int sgd_ctas_per_sm() {
  static int v = [] {
    const char* e = getenv("DEFT_SGD_CTAS_PER_SM");
    const int x = e ? atoi(e) : 32;
    return x < 1 ? 1 : (x > 64 ? 64 : x);
  }();
  return v;
}

cudaError_t launch_sgd_local(const void* grad, int dtype, void* param, float* master,
                             float* mom, int32_t count, const int64_t* offsets, const int64_t* numels,
                             const float* scales, float lr, float momentum,
                             cudaStream_t stream) {
  for (int32_t s0 = 0; s0 < count; s0 += kMaxSeg) {
    SegTable t{};
    t.count = count - s0 < kMaxSeg ? count - s0 : kMaxSeg;
    t.first_vec[0] = 0;
    for (int k = 0; k < t.count; ++k) {
      t.off[k] = offsets[s0 + k];
      t.len[k] = numels[s0 + k];
      t.scale[k] = scales[s0 + k];
      const int64_t aligned = (t.off[k] + 3) / 4 * 4;
      const int64_t end = t.off[k] + t.len[k];
      int64_t units = end > aligned ? (end - aligned + 3) / 4 : 0;
      if (units == 0 && t.len[k] > 0) units = 1;  // head-only segment
      t.first_vec[k + 1] = t.first_vec[k] + units;
    }
    const int64_t total = t.first_vec[t.count];
    if (total == 0) continue;
    const int U = sgd_unroll();
    int64_t grid = (total + (int64_t)kLocalThreads * U - 1) / ((int64_t)kLocalThreads * U);
    if (grid > 148 * sgd_ctas_per_sm()) grid = 148 * sgd_ctas_per_sm();
#define DEFT_SGD_LAUNCH(UU)                                                                      \
  if (dtype == 0)                                                                              \
    sgd_local_kernel<float, UU><<<(int)grid, kLocalThreads, 0, stream>>>(                      \
        reinterpret_cast<const float*>(grad), reinterpret_cast<float*>(param), nullptr, mom, t, \
        lr, momentum);                                                                         \
  else                                                                                         \
    sgd_local_kernel<__nv_bfloat16, UU><<<(int)grid, kLocalThreads, 0, stream>>>(              \
        reinterpret_cast<const __nv_bfloat16*>(grad), reinterpret_cast<__nv_bfloat16*>(param), \
        master, mom, t, lr, momentum);
    if (U == 1) { DEFT_SGD_LAUNCH(1) } else if (U == 4) { DEFT_SGD_LAUNCH(4) } else { DEFT_SGD_LAUNCH(2) }
#undef DEFT_SGD_LAUNCH
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace deft

namespace deft {

// ============================================================================
// Bucket gather: copy the freshly produced per-parameter gradient tensors of
// one bucket into its contiguous range of the group slot (one launch per
// bucket instead of one accumulate kernel per parameter).  The segment table
// travels in the kernel parameters, so a captured CUDA graph keeps it.
// ============================================================================
constexpr int kMaxGatherSeg = 256;
struct GatherTable {
  const char* src[kMaxGatherSeg];
  int64_t dst_off[kMaxGatherSeg];  // bytes from the destination base
  int64_t first[kMaxGatherSeg + 1];  // prefix of 16-byte units per segment
  int64_t len[kMaxGatherSeg];      // bytes
  int32_t count;
};

__global__ void __launch_bounds__(kLocalThreads) gather_kernel(char* __restrict__ dst,
                                                              GatherTable t, int64_t total_units) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int seg = 0;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < total_units; u += stride) {
    while (u >= t.first[seg + 1]) ++seg;
    const int64_t k = u - t.first[seg];
    const char* s = t.src[seg] + k * 16;
    char* d = dst + t.dst_off[seg] + k * 16;
    const int64_t left = t.len[seg] - k * 16;
    if (left >= 16 && ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d)) & 15) == 0) {
      *reinterpret_cast<uint4*>(d) = __ldg(reinterpret_cast<const uint4*>(s));
    } else {
      const int64_t n = left < 16 ? left : 16;
      for (int64_t b = 0; b < n; ++b) d[b] = s[b];
    }
  }
}

}  // namespace deft

namespace deft {
// Default copy-engine threshold of launch_gather (ce_min < 0): segments of at
// least this many bytes are copied by the copy engines (cudaMemcpyAsync D2D: no
// SMs, so a concurrent backward keeps all of them); the rest by gather_kernel.
// DEFT_GATHER_CE_MIN (bytes; 0 = kernel only).
static int64_t gather_ce_min() {
  static int64_t v = [] {
    const char* e = getenv("DEFT_GATHER_CE_MIN");
    return e ? (int64_t)atoll(e) : (int64_t)(4 << 20);
  }();
  return v;
}

cudaError_t launch_gather(char* dst, const void* const* srcs, const int64_t* dst_off,
                          const int64_t* lens, int32_t count, int64_t ce_min,
                          cudaStream_t stream) {
  if (ce_min < 0) ce_min = gather_ce_min();
  std::vector<int32_t> small;
  small.reserve(count);
  for (int32_t k = 0; k < count; ++k) {
    if (ce_min > 0 && lens[k] >= ce_min) {
      cudaError_t e = cudaMemcpyAsync(dst + dst_off[k], srcs[k], (size_t)lens[k],
                                      cudaMemcpyDeviceToDevice, stream);
      if (e != cudaSuccess) return e;
    } else if (lens[k] > 0) {
      small.push_back(k);
    }
  }
  const int32_t n_small = (int32_t)small.size();
  for (int32_t s0 = 0; s0 < n_small; s0 += kMaxGatherSeg) {
    GatherTable t;
    t.count = n_small - s0 < kMaxGatherSeg ? n_small - s0 : kMaxGatherSeg;
    t.first[0] = 0;
    for (int k = 0; k < t.count; ++k) {
      const int32_t i = small[s0 + k];
      t.src[k] = reinterpret_cast<const char*>(srcs[i]);
      t.dst_off[k] = dst_off[i];
      t.len[k] = lens[i];
      t.first[k + 1] = t.first[k] + (lens[i] + 15) / 16;
    }
    const int64_t total = t.first[t.count];
    if (total == 0) continue;
    int64_t grid = (total + kLocalThreads - 1) / kLocalThreads;
    if (grid > 148 * 8) grid = 148 * 8;
    gather_kernel<<<(int)grid, kLocalThreads, 0, stream>>>(dst, t, total);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}
}  // namespace deft

namespace deft {

// ============================================================================
// Multi-bucket fused update + all-gather (W > 1): every bucket of one update
// event in ONE launch with ONE entry/exit barrier pair per CTA.  The table
// holds this rank's owned shard of each bucket (segments over the same flat
// index space on every rank); the grid is a function of the bucket sizes only,
// so block b meets block b of every peer.
// ============================================================================
template <typename T, int W>
__global__ void __launch_bounds__(kLocalThreads) update_allgather_multi_kernel(
    PeerPtrs P, int rank, int64_t slot_base, SegTable t, float lr, float momentum,
    float* __restrict__ mom) {
  using V = Vec<T>;
  constexpr bool kMaster = sizeof(T) == 2;
  const uint32_t epoch = take_epochs(P, rank, kBarrierUpdate, 2u);
  peer_block_barrier(P, rank, W, kBarrierUpdate, blockIdx.x, epoch + 1u);
  const T* g = reinterpret_cast<const T*>(P.grads[rank]) + slot_base;
  float* ref = kMaster ? P.master : reinterpret_cast<float*>(P.params[rank]);
  T* dst[W];
#pragma unroll
  for (int k = 0; k < W; ++k) dst[k] = reinterpret_cast<T*>(P.params[k]);
  auto one = [&](int64_t e, float s) {
    const float v = fmaf(momentum, mom[e], V::scalar(g + e) * s);
    mom[e] = v;
    const float p = fmaf(-lr, v, ref[e]);
    if (kMaster) ref[e] = p;
#pragma unroll
    for (int k = 0; k < W; ++k) store1(dst[k] + e, p);
  };
  const int64_t total = t.first_vec[t.count];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int seg = 0;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < total; u += stride) {
    while (u >= t.first_vec[seg + 1]) ++seg;
    const int64_t base = t.off[seg];
    const int64_t end = base + t.len[seg];
    const int64_t aligned = (base + 3) / 4 * 4;
    const int64_t k = u - t.first_vec[seg];
    const float s = t.scale[seg];
    if (k == 0 && aligned > base) {
      for (int64_t e = base; e < aligned && e < end; ++e) one(e, s);
    }
    const int64_t e = aligned + k * 4;
    if (e + 4 <= end) {
      const float4 g4 = load4(g + e);
      float4 m4 = load4(mom + e);
      float4 p4 = load4(ref + e);
      m4.x = fmaf(momentum, m4.x, g4.x * s);
      m4.y = fmaf(momentum, m4.y, g4.y * s);
      m4.z = fmaf(momentum, m4.z, g4.z * s);
      m4.w = fmaf(momentum, m4.w, g4.w * s);
      p4.x = fmaf(-lr, m4.x, p4.x);
      p4.y = fmaf(-lr, m4.y, p4.y);
      p4.z = fmaf(-lr, m4.z, p4.z);
      p4.w = fmaf(-lr, m4.w, p4.w);
      store4(mom + e, m4);
      if (kMaster) store4(ref + e, p4);
#pragma unroll
      for (int kk = 0; kk < W; ++kk) store4(dst[kk] + e, p4);
    } else {
      for (int64_t x = e; x < end; ++x) one(x, s);
    }
  }
  peer_block_barrier(P, rank, W, kBarrierUpdate, blockIdx.x, epoch + 2u);
}

bool launch_update_allgather_tma(const PeerPtrs& P, int rank, int world, int dtype,
                                 int64_t slot_base, int32_t count, const int64_t* offsets,
                                 const int64_t* numels, float lr, float momentum,
                                 float grad_scale, float* mom, int max_blocks,
                                 cudaStream_t stream);

cudaError_t launch_update_allgather_multi(const PeerPtrs& P, int rank, int world, int dtype,
                                          int64_t slot_base, int32_t count,
                                          const int64_t* offsets, const int64_t* numels,
                                          float lr, float momentum, float grad_scale,
                                          float* mom, int max_blocks, cudaStream_t stream) {
  if (launch_update_allgather_tma(P, rank, world, dtype, slot_base, count, offsets, numels, lr,
                                  momentum, grad_scale, mom, max_blocks, stream))
    return cudaGetLastError();
  const int align = dtype == 0 ? 4 : 8;
  for (int32_t s0 = 0; s0 < count; s0 += kMaxSeg) {
    SegTable t{};
    t.count = count - s0 < kMaxSeg ? count - s0 : kMaxSeg;
    t.first_vec[0] = 0;
    int64_t total_elems = 0;
    for (int k = 0; k < t.count; ++k) {
      const ShardRange sh = shard_of(offsets[s0 + k], numels[s0 + k], rank, world, align);
      t.off[k] = sh.lo;
      t.len[k] = sh.hi - sh.lo;
      t.scale[k] = grad_scale;
      const int64_t aligned = (sh.lo + 3) / 4 * 4;
      int64_t units = sh.hi > aligned ? (sh.hi - aligned + 3) / 4 : 0;
      if (units == 0 && t.len[k] > 0) units = 1;
      t.first_vec[k + 1] = t.first_vec[k] + units;
      total_elems += numels[s0 + k];
    }
    // identical on every rank: depends on the bucket sizes, not on this rank's shards
    int grid = comm_grid_for((total_elems + world - 1) / world);
    if (max_blocks > 0 && grid > max_blocks) grid = max_blocks;
    grid = cap_grid(P, grid);
#define DEFT_UPM_CASE(WW)                                                                   \
  case WW:                                                                                  \
    if (dtype == 0)                                                                         \
      update_allgather_multi_kernel<float, WW><<<grid, kLocalThreads, 0, stream>>>(         \
          P, rank, slot_base, t, lr, momentum, mom);                                        \
    else                                                                                    \
      update_allgather_multi_kernel<__nv_bfloat16, WW><<<grid, kLocalThreads, 0, stream>>>( \
          P, rank, slot_base, t, lr, momentum, mom);                                        \
    break;
    switch (world) {
      DEFT_UPM_CASE(2) DEFT_UPM_CASE(3) DEFT_UPM_CASE(4) DEFT_UPM_CASE(5)
      DEFT_UPM_CASE(6) DEFT_UPM_CASE(7) DEFT_UPM_CASE(8)
      default: break;
    }
#undef DEFT_UPM_CASE
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace deft

namespace deft {

// ============================================================================
// Reduce-scatter, SM channel, TMA-staged: per CTA a ring of kTmaStages shared-
// memory stages; one elected thread issues one cp.async.bulk (global -> shared,
// completing on the stage's mbarrier) per rank for the next chunk while all
// threads sum the current chunk's W copies in fp32 and store the result.  The
// bytes in flight are held by the copy engine of the SM (TMA), not by thread
// registers, so a few CTAs saturate NVLink and the rest of the SMs stay with
// the concurrent backward.
// ============================================================================
constexpr int kTmaThreads = 256;
constexpr int kTmaStagesDefault = 4;   // DEFT_RS_TMA_STAGES: 4 or 6
constexpr int kTmaStageBytes = 32 * 1024;  // W peer chunks per stage

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst_smem)), "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct ChunkTable {           // this rank's owned shards, cut into TMA chunks
  int64_t off[kMaxSeg];       // aligned body start of each segment
  int64_t len[kMaxSeg];       // aligned body length (multiple of 8 elements)
  int64_t first[kMaxSeg + 1]; // prefix of chunks per segment
  int64_t head_lo[kMaxSeg], head_hi[kMaxSeg], tail_lo[kMaxSeg], tail_hi[kMaxSeg];
  int32_t count;
};

// Loopback collective launches (gridDim.y = world, rank = blockIdx.y): every
// rank's table and private buffers, in device memory.
struct RankSlice {
  ChunkTable t;
  float* mom;
  float* master;
};

template <bool kLoop>
__device__ __forceinline__ const ChunkTable& pick_table(const ChunkTable& own,
                                                        const RankSlice* slices) {
  if constexpr (kLoop) return slices[blockIdx.y].t;
  else return own;
}

// Segments [s0, s0 + t.count) of a bucket list -> this rank's shard of each
// (shard_of: the same ownership every comm kernel uses), 8-element-aligned
// bodies cut into `chunk`-element pieces, unaligned heads/tails apart.
// Returns the number of owned elements.
static int64_t build_chunk_table(ChunkTable& t, int32_t s0, int32_t count,
                                 const int64_t* offsets, const int64_t* numels, int rank,
                                 int world, int align, int64_t chunk) {
  t.count = count - s0 < kMaxSeg ? count - s0 : kMaxSeg;
  t.first[0] = 0;
  int64_t owned = 0;
  for (int k = 0; k < t.count; ++k) {
    const ShardRange sh = shard_of(offsets[s0 + k], numels[s0 + k], rank, world, align);
    int64_t a = (sh.lo + 7) / 8 * 8;
    if (a > sh.hi) a = sh.hi;
    int64_t b = sh.hi / 8 * 8;
    if (b < a) b = a;
    t.head_lo[k] = sh.lo; t.head_hi[k] = a;
    t.tail_lo[k] = b; t.tail_hi[k] = sh.hi;
    t.off[k] = a;
    t.len[k] = b - a;
    t.first[k + 1] = t.first[k] + (t.len[k] + chunk - 1) / chunk;
    owned += sh.hi - sh.lo;
  }
  return owned;
}

__device__ __forceinline__ void table_chunk(const ChunkTable& t, int64_t chunk, int64_t c,
                                            int64_t* e0, int64_t* len) {
  int sgi = 0;
  while (c >= t.first[sgi + 1]) ++sgi;
  *e0 = t.off[sgi] + (c - t.first[sgi]) * chunk;
  const int64_t rem = t.off[sgi] + t.len[sgi] - *e0;
  *len = rem < chunk ? rem : chunk;
}

// Elements per peer chunk: a stage holds the W-1 PEER chunks only (the own chunk
// is read from global memory by the consumer threads, prefetched into registers
// while the stage is in flight), so the whole stage carries NVLink bytes.
template <typename T, int W>
__host__ __device__ constexpr int64_t rs_tma_chunk() {
  return (kTmaStageBytes / (W - 1) / (int)sizeof(T)) / 8 * 8;
}

// One launch reduces every segment of the table (all buckets released together
// on this link): one entry barrier instead of one per bucket.
template <typename T, int W, int kTmaStages, bool kLoop = false>
__global__ void __launch_bounds__(kTmaThreads) reduce_scatter_tma_kernel(
    PeerPtrs P, int rank_arg, int64_t slot_base, const __grid_constant__ ChunkTable t_arg,
    const RankSlice* __restrict__ slices) {
  const int rank = kLoop ? (int)blockIdx.y : rank_arg;
  const ChunkTable& t = pick_table<kLoop>(t_arg, slices);
  using V = Vec<T>;
  extern __shared__ __align__(128) unsigned char tma_smem[];
  __shared__ __align__(8) uint64_t full[kTmaStages];
  // elements per peer chunk: a stage holds the W-1 peer chunks, 16-byte granular
  constexpr int64_t kChunk = rs_tma_chunk<T, W>();
  phase_stamp(P, 0);
  const uint32_t epoch = take_epochs(P, rank, kBarrierRS, 1u) + 1u;
  phase_stamp(P, 1);
  peer_block_barrier(P, rank, W, kBarrierRS, blockIdx.x, epoch);
  phase_stamp(P, 2);
  // the barrier's acquire is a generic-proxy operation; the peers' gradient
  // bytes are read by the async proxy (cp.async.bulk): order the two
  if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
  const T* src[W];
#pragma unroll
  for (int k = 0; k < W; ++k) src[k] = reinterpret_cast<const T*>(P.grads[k]) + slot_base;
  T* dst = reinterpret_cast<T*>(P.grads[rank]) + slot_base;
  if (blockIdx.x == 0) {  // unaligned edges of every segment
    for (int sgi = 0; sgi < t.count; ++sgi) {
      for (int part = 0; part < 2; ++part) {
        const int64_t a = part ? t.tail_lo[sgi] : t.head_lo[sgi];
        const int64_t b = part ? t.tail_hi[sgi] : t.head_hi[sgi];
        for (int64_t e = a + threadIdx.x; e < b; e += blockDim.x) {
          float acc = 0.f;
#pragma unroll
          for (int k = 0; k < W; ++k) acc += V::scalar(src[k] + e);
          V::put(dst + e, acc);
        }
      }
    }
  }
  // this CTA's contiguous share of the table's chunks
  const int64_t n_chunks = t.first[t.count];
  const int64_t c_begin = n_chunks * blockIdx.x / gridDim.x;
  const int64_t c_end = n_chunks * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kTmaStages; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // stage slot of peer k (the own rank has none)
  auto stage_ptr = [&](int st, int k) -> T* {
    const int slot = k < rank ? k : k - 1;
    return reinterpret_cast<T*>(tma_smem + (size_t)st * kTmaStageBytes) + (int64_t)slot * kChunk;
  };
  auto issue = [&](int64_t c) {  // one elected thread: W-1 bulk copies of chunk c
    const int st = (int)((c - c_begin) % kTmaStages);
    int64_t e0, len;
    table_chunk(t, kChunk, c, &e0, &len);
    const uint32_t bytes = (uint32_t)(len * sizeof(T));
    // the stage was last read through the generic proxy; order that before the
    // async-proxy (TMA) writes that refill it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&full[st], bytes * (W - 1));
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k != rank) tma_load_1d(stage_ptr(st, k), src[k] + e0, bytes, &full[st]);
  };
  if (threadIdx.x == 0)
    for (int64_t c = c_begin; c < min(c_end, c_begin + kTmaStages - 1); ++c) issue(c);
  using Raw = typename V::Raw;
  // vectors of one chunk per thread (the own values are prefetched in registers)
  constexpr int kPer = (int)((kChunk / V::N + kTmaThreads - 1) / kTmaThreads);
  for (int64_t c = c_begin; c < c_end; ++c) {
    const int st = (int)((c - c_begin) % kTmaStages);
    const uint32_t parity = (uint32_t)(((c - c_begin) / kTmaStages) & 1);
    // keep the ring full: chunk c + S - 1 goes into the stage freed at the end of c - 1
    if (threadIdx.x == 0 && c + kTmaStages - 1 < c_end) issue(c + kTmaStages - 1);
    int64_t e0, len;
    table_chunk(t, kChunk, c, &e0, &len);
    const int64_t nv = len / V::N;
    // own chunk: plain loads (this kernel writes these same elements below, each
    // thread only its own) issued before the wait so they overlap the stage's flight
    Raw own[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int64_t v = threadIdx.x + (int64_t)j * kTmaThreads;
      if (v < nv) own[j] = reinterpret_cast<const Raw*>(dst + e0)[v];
    }
    mbar_wait(&full[st], parity);
    if (c == c_begin) phase_stamp(P, 3);
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int64_t v = threadIdx.x + (int64_t)j * kTmaThreads;
      if (v >= nv) break;
      // rank order, exactly as before: acc = x_0 + x_1 + ... + x_{W-1}
      float acc[V::N], tmp[V::N];
      if (rank == 0) V::to_f32(own[j], acc);
      else V::to_f32(reinterpret_cast<const Raw*>(stage_ptr(st, 0))[v], acc);
#pragma unroll
      for (int k = 1; k < W; ++k) {
        if (k == rank) V::to_f32(own[j], tmp);
        else V::to_f32(reinterpret_cast<const Raw*>(stage_ptr(st, k))[v], tmp);
#pragma unroll
        for (int q = 0; q < V::N; ++q) acc[q] += tmp[q];
      }
      reinterpret_cast<Raw*>(dst + e0)[v] = V::from_f32(acc);
    }
    __syncthreads();  // stage st fully consumed before it is refilled
  }
  phase_stamp(P, 6);
}

template <typename T, int S>
static void rs_tma_dispatch_s(int world, int grid, cudaStream_t stream, const PeerPtrs& P,
                              int rank, int64_t slot_base, const ChunkTable& t) {
  const size_t smem = (size_t)S * kTmaStageBytes;
#define DEFT_RST_CASE(WW)                                                                      \
  case WW: {                                                                                   \
    static bool attr = false;                                                                  \
    if (!attr) {                                                                               \
      cudaFuncSetAttribute(reduce_scatter_tma_kernel<T, WW, S>,                                \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);            \
      attr = true;                                                                             \
    }                                                                                          \
    reduce_scatter_tma_kernel<T, WW, S><<<grid, kTmaThreads, smem, stream>>>(P, rank,         \
                                                                            slot_base, t,      \
                                                                            nullptr);          \
    break;                                                                                     \
  }
  switch (world) {
    DEFT_RST_CASE(2) DEFT_RST_CASE(3) DEFT_RST_CASE(4) DEFT_RST_CASE(5)
    DEFT_RST_CASE(6) DEFT_RST_CASE(7) DEFT_RST_CASE(8)
    default: break;
  }
#undef DEFT_RST_CASE
}

static int rs_tma_stages() {
  static int v = [] {
    const char* e = getenv("DEFT_RS_TMA_STAGES");
    return e && atoi(e) == 6 ? 6 : kTmaStagesDefault;
  }();
  return v;
}

template <typename T>
static void rs_tma_dispatch(int world, int grid, cudaStream_t stream, const PeerPtrs& P,
                            int rank, int64_t slot_base, const ChunkTable& t) {
  if (rs_tma_stages() == 6)
    rs_tma_dispatch_s<T, 6>(world, grid, stream, P, rank, slot_base, t);
  else
    rs_tma_dispatch_s<T, 4>(world, grid, stream, P, rank, slot_base, t);
}

// DEFT_RS_IMPL=tma|ldg selects the SM-channel reduce-scatter (default tma: the
// same NVLink bandwidth from 24 CTAs as the LDG kernel from 128, K2b);
// DEFT_RS_TMA_BLOCKS its CTA count (default 24).
static int rs_impl_tma() {
  static int v = [] {
    const char* e = getenv("DEFT_RS_IMPL");
    return e && e[0] == 'l' ? 0 : 1;
  }();
  return v;
}
static int rs_tma_blocks() {
  static int v = [] {
    const char* e = getenv("DEFT_RS_TMA_BLOCKS");
    int x = e ? atoi(e) : 24;
    return x < 1 ? 1 : (x > kMaxCommBlocks ? kMaxCommBlocks : x);
  }();
  return v;
}

static int64_t rs_chunk_for(int world, int dtype) {
  const int esz = dtype == 0 ? 4 : 2;
  return (kTmaStageBytes / (world - 1) / esz) / 8 * 8;   // == rs_tma_chunk<T, W>()
}

bool launch_reduce_scatter_tma_multi(const PeerPtrs& P, int rank, int world, int dtype,
                                     int64_t slot_base, int32_t count, const int64_t* offsets,
                                     const int64_t* numels, cudaStream_t stream) {
  if (!rs_impl_tma() || world < 2 || world > 8) return false;
  const int align = dtype == 0 ? 4 : 8;
  for (int32_t s0 = 0; s0 < count; s0 += kMaxSeg) {
    ChunkTable t{};
    build_chunk_table(t, s0, count, offsets, numels, rank, world, align,
                      rs_chunk_for(world, dtype));
    // the grid must be the same on every rank (block b meets block b of each
    // peer): a function of the bucket sizes only, not of this rank's shards
    int64_t per = 0;
    for (int k = 0; k < t.count; ++k) per += (numels[s0 + k] + world - 1) / world;
    int grid = (int)((per + 32767) / 32768);
    if (grid < 1) grid = 1;
    if (grid > rs_tma_blocks()) grid = rs_tma_blocks();
    grid = cap_grid(P, grid);
    if (dtype == 0)
      rs_tma_dispatch<float>(world, grid, stream, P, rank, slot_base, t);
    else
      rs_tma_dispatch<__nv_bfloat16>(world, grid, stream, P, rank, slot_base, t);
    count_launch();
  }
  return true;
}

bool launch_reduce_scatter_tma(const PeerPtrs& P, int rank, int world, int dtype,
                               int64_t slot_base, int64_t offset, int64_t numel,
                               cudaStream_t stream) {
  return launch_reduce_scatter_tma_multi(P, rank, world, dtype, slot_base, 1, &offset, &numel,
                                         stream);
}

}  // namespace deft

namespace deft {

// ============================================================================
// Multi-bucket fused update + all-gather, TMA-pipelined (W > 1).  Same math and
// barriers as update_allgather_multi_kernel; per CTA a ring of shared-memory
// stages: one elected thread bulk-loads a chunk of g / v / p (cp.async.bulk,
// mbarrier complete_tx), all threads update it in place, and the elected
// thread bulk-STORES the new momentum (and fp32 master) locally and the new
// parameters to every rank (cp.async.bulk.global.shared::cta, peer addresses).
// The bytes in flight live in the TMA unit, so the small CTA budget the
// "start" placement uses still streams at NVLink rate.
// ============================================================================
constexpr int kUpdTmaThreads = 256;
// ring of S shared-memory stages of which up to P hold chunks whose bulk stores
// are still reading them (DEFT_UPDATE_TMA_PIPE=S:P, 3:0 | 4:1 | 6:2): loads run
// S - 1 - P chunks ahead, and refilling a stage waits only for the stores of
// the chunk P + 1 back -- never for the chunk just stored (whose remote stores
// drain at NVLink latency)
constexpr int kUpdTmaStagesDefault = 4;
constexpr int kUpdTmaPendingDefault = 1;
constexpr int kUpdChunk = 2048;  // elements per chunk (multiple of 8); 4096 at W = 2 (upd_chunk)

__device__ __forceinline__ void tma_store_1d(void* dst_gmem, const void* src_smem,
                                             uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem),
               "r"(smem_u32(src_smem)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_store_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void tma_store_wait_read() {   // all but the newest N groups
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void tma_store_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


template <typename T, int W, int kUpdTmaStages, int kPending, bool kLoop = false,
          int kChunkE = kUpdChunk>
__global__ void __launch_bounds__(kUpdTmaThreads) update_allgather_tma_kernel(
    PeerPtrs P, int rank_arg, int64_t slot_base, const __grid_constant__ ChunkTable t_arg,
    float lr, float momentum, float scale, float* __restrict__ mom_arg,
    const RankSlice* __restrict__ slices) {
  const int rank = kLoop ? (int)blockIdx.y : rank_arg;
  const ChunkTable& t = pick_table<kLoop>(t_arg, slices);
  float* __restrict__ mom = kLoop ? slices[blockIdx.y].mom : mom_arg;
  using V = Vec<T>;
  constexpr bool kMaster = sizeof(T) == 2;
  // stage layout: g (T) | v (f32) | p (f32) | p_out (T, bf16 only)
  constexpr int64_t kG = (int64_t)kChunkE * sizeof(T);
  constexpr int64_t kF = (int64_t)kChunkE * 4;
  constexpr int64_t kStage = kG + 2 * kF + (kMaster ? kG : 0);
  extern __shared__ __align__(128) unsigned char usmem[];
  __shared__ __align__(8) uint64_t full[kUpdTmaStages];

  phase_stamp(P, 0);
  const T* g = reinterpret_cast<const T*>(P.grads[rank]) + slot_base;
  float* ref = kMaster ? (kLoop ? slices[blockIdx.y].master : P.master)
                       : reinterpret_cast<float*>(P.params[rank]);
  T* dst[W];
#pragma unroll
  for (int k = 0; k < W; ++k) dst[k] = reinterpret_cast<T*>(P.params[k]);

  const int64_t n_chunks = t.first[t.count];
  const int64_t c_begin = n_chunks * blockIdx.x / gridDim.x;
  const int64_t c_end = n_chunks * (blockIdx.x + 1) / gridDim.x;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kUpdTmaStages; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  auto chunk_range = [&](int64_t c, int64_t* e0, int64_t* len) {
    table_chunk(t, kChunkE, c, e0, len);
  };
  auto base = [&](int st) { return usmem + (size_t)st * kStage; };
  static_assert(kPending >= 0 && kPending <= kUpdTmaStages - 2, "ring too small");
  constexpr int kAhead = kUpdTmaStages - 1 - kPending;   // loads in flight
  auto issue_load = [&](int64_t c) {
    const int st = (int)((c - c_begin) % kUpdTmaStages);
    int64_t e0, len;
    chunk_range(c, &e0, &len);
    // the stage's previous chunk (c - S) was stored kPending + 1 chunks ago:
    // only its bulk stores must have finished reading it
    tma_store_wait_read<kPending>();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t bg = (uint32_t)(len * sizeof(T)), bf = (uint32_t)(len * 4);
    mbar_expect_tx(&full[st], bg + 2 * bf);
    tma_load_1d(base(st), g + e0, bg, &full[st]);
    tma_load_1d(base(st) + kG, mom + e0, bf, &full[st]);
    tma_load_1d(base(st) + kG + kF, ref + e0, bf, &full[st]);
  };
  // The first stages read only this rank's own gradient shard, momentum and
  // parameter shard (stream-ordered, never written by a peer): they are issued
  // BEFORE the entry barrier so its NVLink round trip overlaps their HBM latency.
  // Only the stores into the peers' parameter buffers must wait for it.
  if (threadIdx.x == 0)
    for (int64_t c = c_begin; c < min(c_end, c_begin + kAhead); ++c) issue_load(c);
  const uint32_t epoch = take_epochs(P, rank, kBarrierUpdate, 2u);  // + bar.sync: mbarriers init'd
  phase_stamp(P, 1);
  peer_block_barrier(P, rank, W, kBarrierUpdate, blockIdx.x, epoch + 1u);
  phase_stamp(P, 2);
  // generic acquire -> async-proxy (bulk copy) accesses of global memory
  if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");

  // unaligned edges of every segment: block 0, scalar
  if (blockIdx.x == 0) {
    for (int sgi = 0; sgi < t.count; ++sgi) {
      for (int part = 0; part < 2; ++part) {
        const int64_t a = part ? t.tail_lo[sgi] : t.head_lo[sgi];
        const int64_t b = part ? t.tail_hi[sgi] : t.head_hi[sgi];
        for (int64_t e = a + threadIdx.x; e < b; e += blockDim.x) {
          const float v = fmaf(momentum, mom[e], V::scalar(g + e) * scale);
          mom[e] = v;
          const float p = fmaf(-lr, v, ref[e]);
          if (kMaster) ref[e] = p;
#pragma unroll
          for (int k = 0; k < W; ++k) store1(dst[k] + e, p);
        }
      }
    }
  }
  for (int64_t c = c_begin; c < c_end; ++c) {
    const int st = (int)((c - c_begin) % kUpdTmaStages);
    const uint32_t parity = (uint32_t)(((c - c_begin) / kUpdTmaStages) & 1);
    if (threadIdx.x == 0 && c + kAhead < c_end) issue_load(c + kAhead);
    mbar_wait(&full[st], parity);
    if (c == c_begin) phase_stamp(P, 3);
    int64_t e0, len;
    chunk_range(c, &e0, &len);
    const T* sg = reinterpret_cast<const T*>(base(st));
    float* sv = reinterpret_cast<float*>(base(st) + kG);
    float* sp = reinterpret_cast<float*>(base(st) + kG + kF);
    T* so = reinterpret_cast<T*>(base(st) + kG + 2 * kF);
    for (int64_t i = threadIdx.x * 4; i < len; i += (int64_t)blockDim.x * 4) {
      const float4 g4 = load4(sg + i);
      float4 m4 = *reinterpret_cast<float4*>(sv + i);
      float4 p4 = *reinterpret_cast<float4*>(sp + i);
      m4.x = fmaf(momentum, m4.x, g4.x * scale);
      m4.y = fmaf(momentum, m4.y, g4.y * scale);
      m4.z = fmaf(momentum, m4.z, g4.z * scale);
      m4.w = fmaf(momentum, m4.w, g4.w * scale);
      p4.x = fmaf(-lr, m4.x, p4.x);
      p4.y = fmaf(-lr, m4.y, p4.y);
      p4.z = fmaf(-lr, m4.z, p4.z);
      p4.w = fmaf(-lr, m4.w, p4.w);
      *reinterpret_cast<float4*>(sv + i) = m4;
      *reinterpret_cast<float4*>(sp + i) = p4;
      if (kMaster) store4(so + i, p4);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> TMA reads
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t bf = (uint32_t)(len * 4), bo = (uint32_t)(len * sizeof(T));
      tma_store_1d(mom + e0, sv, bf);
      if (kMaster) {
        tma_store_1d(ref + e0, sp, bf);
#pragma unroll
        for (int k = 0; k < W; ++k) tma_store_1d(dst[k] + e0, so, bo);
      } else {
#pragma unroll
        for (int k = 0; k < W; ++k) tma_store_1d(dst[k] + e0, sp, bo);
      }
      tma_store_commit();
    }
  }
  phase_stamp(P, 4);
  if (threadIdx.x == 0) {
    tma_store_wait_all();  // every bulk store of this CTA performed (incl. peers)
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  phase_stamp(P, 5);
  // exit: every rank's stores into every parameter buffer have landed
  peer_block_barrier(P, rank, W, kBarrierUpdate, blockIdx.x, epoch + 2u);
  phase_stamp(P, 6);
}

// DEFT_UPDATE_TMA_PIPE=S:P -> 30 (3:0), 41 (4:1, default) or 62 (6:2)
static int upd_tma_pipe() {
  static int v = [] {
    const char* e = getenv("DEFT_UPDATE_TMA_PIPE");
    if (!e) return kUpdTmaStagesDefault * 10 + kUpdTmaPendingDefault;
    const int x = atoi(e) * 10 + (strchr(e, ':') ? atoi(strchr(e, ':') + 1) : 0);
    return x == 30 || x == 41 || x == 62 ? x : kUpdTmaStagesDefault * 10 + kUpdTmaPendingDefault;
  }();
  return v;
}

// Elements per ring chunk of the update kernel (4:1 ring): 4096 at W = 2 (4 x 48
// KB of shared memory for fp32), else 2048.  Measured at the step's 32-CTA update
// budget: W = 2, 64 MB 358 -> 431 GB/s, ResNet-101's two start-group launches
// 272 -> 425 GB/s with the step time unchanged; W = 4 ResNet-101 516 -> 531 GB/s
// but VGG-19 bs8 in-step 7267 -> 7191 samples/s (profiles/r02h_*, r02i_*).
// DEFT_UPDATE_TMA_CHUNK=2048|4096 overrides.
static int upd_chunk(int world) {
  static int env = [] {
    const char* e = getenv("DEFT_UPDATE_TMA_CHUNK");
    return e ? (atoi(e) == 4096 ? 4096 : kUpdChunk) : 0;
  }();
  if (env) return env;
  return world == 2 ? 4096 : kUpdChunk;
}

static size_t upd_stage_bytes(int chunk, int dtype) {
  const size_t esz = dtype == 0 ? 4 : 2;
  return (size_t)chunk * esz + 2 * (size_t)chunk * 4 + (dtype == 0 ? 0 : (size_t)chunk * esz);
}

bool launch_update_allgather_tma(const PeerPtrs& P, int rank, int world, int dtype,
                                 int64_t slot_base, int32_t count, const int64_t* offsets,
                                 const int64_t* numels, float lr, float momentum,
                                 float grad_scale, float* mom, int max_blocks,
                                 cudaStream_t stream) {
  static int enabled = [] {
    const char* e = getenv("DEFT_UPDATE_IMPL");
    return e && e[0] == 'l' ? 0 : 1;   // default: TMA
  }();
  if (!enabled || world < 2) return false;
  const int align = dtype == 0 ? 4 : 8;
  for (int32_t s0 = 0; s0 < count; s0 += kMaxSeg) {
    const int pipe = upd_tma_pipe();
    const int chunk = pipe == 41 ? upd_chunk(world) : kUpdChunk;
    ChunkTable t{};
    build_chunk_table(t, s0, count, offsets, numels, rank, world, align, chunk);
    int64_t total_elems = 0;
    for (int k = 0; k < t.count; ++k) total_elems += numels[s0 + k];
    int grid = comm_grid_for((total_elems + world - 1) / world);
    if (max_blocks > 0 && grid > max_blocks) grid = max_blocks;
    grid = cap_grid(P, grid);
    const size_t smem = (size_t)(pipe / 10) * upd_stage_bytes(chunk, dtype);
#define DEFT_UPT_LAUNCH(TT, WW, SS, PP, CC)                                                    \
  {                                                                                            \
    cudaFuncSetAttribute(update_allgather_tma_kernel<TT, WW, SS, PP, false, CC>,               \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);              \
    update_allgather_tma_kernel<TT, WW, SS, PP, false, CC>                                     \
        <<<grid, kUpdTmaThreads, smem, stream>>>(P, rank, slot_base, t, lr, momentum,          \
                                                 grad_scale, mom, nullptr);                    \
  }
#define DEFT_UPT_PIPE(TT, WW)                                                                  \
  if (pipe == 30) DEFT_UPT_LAUNCH(TT, WW, 3, 0, kUpdChunk)                                     \
  else if (pipe == 62) DEFT_UPT_LAUNCH(TT, WW, 6, 2, kUpdChunk)                                \
  else if (chunk == 4096) DEFT_UPT_LAUNCH(TT, WW, 4, 1, 4096)                                  \
  else DEFT_UPT_LAUNCH(TT, WW, 4, 1, kUpdChunk)
#define DEFT_UPT_CASE(WW)                                                                      \
  case WW:                                                                                     \
    if (dtype == 0) { DEFT_UPT_PIPE(float, WW) } else { DEFT_UPT_PIPE(__nv_bfloat16, WW) }     \
    break;
    switch (world) {
      DEFT_UPT_CASE(2) DEFT_UPT_CASE(3) DEFT_UPT_CASE(4) DEFT_UPT_CASE(5)
      DEFT_UPT_CASE(6) DEFT_UPT_CASE(7) DEFT_UPT_CASE(8)
      default: break;
    }
#undef DEFT_UPT_CASE
#undef DEFT_UPT_PIPE
#undef DEFT_UPT_LAUNCH
    count_launch();
  }
  return true;
}

}  // namespace deft

namespace deft {

// ============================================================================
// Loopback collectives: ONE launch carries every rank of a loopback world
// (gridDim.y = world, rank = blockIdx.y, each rank's table / momentum / master
// in a device RankSlice array).  The rendezvous of the peer barriers happens
// inside one grid whose blocks are all co-resident (grid capped by
// P.grid_cap), so it completes even when kernels are serialized -- the
// situation of a kernel profiler, where W separate launches never meet.
// ============================================================================
static cudaError_t upload_slices(const std::vector<RankSlice>& h, RankSlice** d) {
  cudaError_t e = cudaMalloc(d, h.size() * sizeof(RankSlice));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*d, h.data(), h.size() * sizeof(RankSlice), cudaMemcpyHostToDevice);
}

cudaError_t launch_rs_tma_loopback(const PeerPtrs& P, int world, int dtype, int64_t slot_base,
                                   int32_t count, const int64_t* offsets, const int64_t* numels,
                                   cudaStream_t stream) {
  if (world < 2 || world > 8) return cudaErrorInvalidValue;
  const int align = dtype == 0 ? 4 : 8;
  for (int32_t s0 = 0; s0 < count; s0 += kMaxSeg) {
    std::vector<RankSlice> h(world);
    for (int r = 0; r < world; ++r)
      build_chunk_table(h[r].t, s0, count, offsets, numels, r, world, align,
                        rs_chunk_for(world, dtype));
    int64_t per = 0;
    for (int k = 0; k < h[0].t.count; ++k) per += (numels[s0 + k] + world - 1) / world;
    int grid = (int)((per + 32767) / 32768);
    if (grid < 1) grid = 1;
    if (grid > rs_tma_blocks()) grid = rs_tma_blocks();
    grid = cap_grid(P, grid);
    RankSlice* d = nullptr;
    cudaError_t e = upload_slices(h, &d);
    if (e != cudaSuccess) return e;
    const size_t smem = (size_t)kTmaStagesDefault * kTmaStageBytes;
#define DEFT_RSL_CASE(WW)                                                                 \
  case WW:                                                                                \
    if (dtype == 0) {                                                                     \
      cudaFuncSetAttribute(reduce_scatter_tma_kernel<float, WW, kTmaStagesDefault, true>, \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);       \
      reduce_scatter_tma_kernel<float, WW, kTmaStagesDefault, true>                       \
          <<<dim3(grid, world), kTmaThreads, smem, stream>>>(P, 0, slot_base, h[0].t, d); \
    } else {                                                                              \
      cudaFuncSetAttribute(                                                               \
          reduce_scatter_tma_kernel<__nv_bfloat16, WW, kTmaStagesDefault, true>,          \
          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                        \
      reduce_scatter_tma_kernel<__nv_bfloat16, WW, kTmaStagesDefault, true>               \
          <<<dim3(grid, world), kTmaThreads, smem, stream>>>(P, 0, slot_base, h[0].t, d); \
    }                                                                                     \
    break;
    switch (world) {
      DEFT_RSL_CASE(2) DEFT_RSL_CASE(3) DEFT_RSL_CASE(4) DEFT_RSL_CASE(5)
      DEFT_RSL_CASE(6) DEFT_RSL_CASE(7) DEFT_RSL_CASE(8)
      default: break;
    }
#undef DEFT_RSL_CASE
    count_launch();
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    cudaFree(d);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_update_tma_loopback(const PeerPtrs& P, int world, int dtype,
                                       int64_t slot_base, int32_t count,
                                       const int64_t* offsets, const int64_t* numels,
                                       float lr, float momentum, float grad_scale,
                                       float* const* moms, float* const* masters,
                                       int max_blocks, cudaStream_t stream) {
  if (world < 2 || world > 8) return cudaErrorInvalidValue;
  const int align = dtype == 0 ? 4 : 8;
  for (int32_t s0 = 0; s0 < count; s0 += kMaxSeg) {
    std::vector<RankSlice> h(world);
    int64_t total_elems = 0;
    const int chunk = upd_chunk(world);   // the production ring (4:1) and chunk
    for (int r = 0; r < world; ++r) {
      build_chunk_table(h[r].t, s0, count, offsets, numels, r, world, align, chunk);
      h[r].mom = moms[r];
      h[r].master = masters[r];
    }
    for (int k = 0; k < h[0].t.count; ++k) total_elems += numels[s0 + k];
    int grid = comm_grid_for((total_elems + world - 1) / world);
    if (max_blocks > 0 && grid > max_blocks) grid = max_blocks;
    grid = cap_grid(P, grid);
    RankSlice* d = nullptr;
    cudaError_t e = upload_slices(h, &d);
    if (e != cudaSuccess) return e;
    const size_t smem = (size_t)kUpdTmaStagesDefault * upd_stage_bytes(chunk, dtype);
#define DEFT_UPL_LAUNCH(TT, WW, CC)                                                           \
  {                                                                                           \
    cudaFuncSetAttribute(update_allgather_tma_kernel<TT, WW, kUpdTmaStagesDefault,            \
                                                     kUpdTmaPendingDefault, true, CC>,        \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);             \
    update_allgather_tma_kernel<TT, WW, kUpdTmaStagesDefault, kUpdTmaPendingDefault, true, CC> \
        <<<dim3(grid, world), kUpdTmaThreads, smem, stream>>>(P, 0, slot_base, h[0].t, lr,    \
                                                              momentum, grad_scale, nullptr,  \
                                                              d);                             \
  }
#define DEFT_UPL_CASE(WW)                                           \
  case WW:                                                          \
    if (chunk == 4096) {                                            \
      if (dtype == 0) DEFT_UPL_LAUNCH(float, WW, 4096)              \
      else DEFT_UPL_LAUNCH(__nv_bfloat16, WW, 4096)                 \
    } else {                                                        \
      if (dtype == 0) DEFT_UPL_LAUNCH(float, WW, kUpdChunk)         \
      else DEFT_UPL_LAUNCH(__nv_bfloat16, WW, kUpdChunk)            \
    }                                                               \
    break;
    switch (world) {
      DEFT_UPL_CASE(2) DEFT_UPL_CASE(3) DEFT_UPL_CASE(4) DEFT_UPL_CASE(5)
      DEFT_UPL_CASE(6) DEFT_UPL_CASE(7) DEFT_UPL_CASE(8)
      default: break;
    }
#undef DEFT_UPL_CASE
#undef DEFT_UPL_LAUNCH
    count_launch();
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    cudaFree(d);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace deft

namespace deft {

// ============================================================================
// One-shot bucket sync for small buckets: ONE launch per update event does the
// all-reduce and the update.  Every rank reads the WHOLE bucket from every
// rank's gradient slot (own + W-1 peers over NVLink, 128-bit loads), sums in
// rank order in fp32, rounds to the slot dtype (exactly what the two-shot
// reduce-scatter stores), and applies the fused SGD/momentum update to the
// full bucket locally -- momentum and (bf16) master of one-shot buckets are
// replicated, bit-identical on every rank because every rank sums in the same
// order.  No reduce-scatter launch at the transfer point, no parameter
// all-gather: the per-bucket fixed cost (two launches, three barrier rounds)
// becomes one launch and one barrier pair.  Reads (W-1) x bucket bytes per rank
// over NVLink instead of 2 (W-1)/W x: the small-bucket trade.
// ============================================================================
constexpr int kOneShotThreads = 256;
constexpr int kOneShotUnroll = 2;

template <typename T, int W>
__global__ void __launch_bounds__(kOneShotThreads) oneshot_update_kernel(
    PeerPtrs P, int rank, int64_t slot_base, const __grid_constant__ SegTable t, float lr,
    float momentum, float* __restrict__ mom) {
  using V = Vec<T>;
  using Raw = typename V::Raw;
  constexpr int N = V::N;
  constexpr bool kMaster = sizeof(T) == 2;
  phase_stamp(P, 0);
  const uint32_t epoch = take_epochs(P, rank, kBarrierUpdate, 2u);
  phase_stamp(P, 1);
  // entry: every rank's slot holds this group's complete gradient
  peer_block_barrier(P, rank, W, kBarrierUpdate, blockIdx.x, epoch + 1u);
  phase_stamp(P, 2);
  const T* src[W];
#pragma unroll
  for (int k = 0; k < W; ++k) src[k] = reinterpret_cast<const T*>(P.grads[k]) + slot_base;
  float* ref = kMaster ? P.master : reinterpret_cast<float*>(P.params[rank]);
  T* dst = reinterpret_cast<T*>(P.params[rank]);
  auto one = [&](int64_t e, float s) {   // scalar element (unaligned heads / tails)
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < W; ++k) acc += V::scalar(src[k] + e);
    T r;
    V::put(&r, acc);
    const float g = V::scalar(&r);
    const float v = fmaf(momentum, mom[e], g * s);
    mom[e] = v;
    const float p = fmaf(-lr, v, ref[e]);
    if (kMaster) ref[e] = p;
    store1(dst + e, p);
  };
  const int64_t total = t.first_vec[t.count];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t u0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u0 < total;
       u0 += stride * kOneShotUnroll) {
    Raw raw[kOneShotUnroll][W];
    float4 m4s[kOneShotUnroll][N / 4], p4s[kOneShotUnroll][N / 4];
    int64_t el[kOneShotUnroll];
    float sc[kOneShotUnroll];
    bool vec[kOneShotUnroll];
#pragma unroll
    for (int q = 0; q < kOneShotUnroll; ++q) {
      const int64_t u = u0 + q * stride;
      vec[q] = false;
      el[q] = -1;
      if (u >= total) continue;
      int sg = 0;
      while (u >= t.first_vec[sg + 1]) ++sg;
      const int64_t base = t.off[sg], end = base + t.len[sg];
      const int64_t aligned = (base + N - 1) / N * N;
      const int64_t k = u - t.first_vec[sg];
      sc[q] = t.scale[sg];
      if (k == 0)
        for (int64_t e = base; e < aligned && e < end; ++e) one(e, sc[q]);  // head
      const int64_t e = aligned + k * N;
      el[q] = e;
      if (e + N <= end) {
        vec[q] = true;
#pragma unroll
        for (int r = 0; r < W; ++r) raw[q][r] = ld_nc(reinterpret_cast<const Raw*>(src[r] + e));
        // the local momentum / fp32 parameters ride along with the peer loads
#pragma unroll
        for (int c = 0; c < N / 4; ++c) {
          m4s[q][c] = load4(mom + e + 4 * c);
          p4s[q][c] = load4(ref + e + 4 * c);
        }
      } else {
        for (int64_t x = e; x < end; ++x) one(x, sc[q]);                     // tail
      }
    }
#pragma unroll
    for (int q = 0; q < kOneShotUnroll; ++q) {
      if (!vec[q]) continue;
      float acc[N], tmp[N];
      V::to_f32(raw[q][0], acc);
#pragma unroll
      for (int r = 1; r < W; ++r) {
        V::to_f32(raw[q][r], tmp);
#pragma unroll
        for (int c = 0; c < N; ++c) acc[c] += tmp[c];
      }
      V::to_f32(V::from_f32(acc), acc);        // the slot dtype's rounding
      const int64_t e = el[q];
      float vv[N], pp[N];
#pragma unroll
      for (int c = 0; c < N; c += 4) {
        const float4 m4 = m4s[q][c / 4];
        const float4 p4 = p4s[q][c / 4];
        vv[c + 0] = fmaf(momentum, m4.x, acc[c + 0] * sc[q]);
        vv[c + 1] = fmaf(momentum, m4.y, acc[c + 1] * sc[q]);
        vv[c + 2] = fmaf(momentum, m4.z, acc[c + 2] * sc[q]);
        vv[c + 3] = fmaf(momentum, m4.w, acc[c + 3] * sc[q]);
        pp[c + 0] = fmaf(-lr, vv[c + 0], p4.x);
        pp[c + 1] = fmaf(-lr, vv[c + 1], p4.y);
        pp[c + 2] = fmaf(-lr, vv[c + 2], p4.z);
        pp[c + 3] = fmaf(-lr, vv[c + 3], p4.w);
        store4(mom + e + c, make_float4(vv[c], vv[c + 1], vv[c + 2], vv[c + 3]));
        if (kMaster) store4(ref + e + c, make_float4(pp[c], pp[c + 1], pp[c + 2], pp[c + 3]));
      }
      reinterpret_cast<Raw*>(dst + e)[0] = V::from_f32(pp);
    }
  }
  phase_stamp(P, 4);
  // exit: no peer reads this rank's slot any more (it may be recycled)
  peer_block_barrier(P, rank, W, kBarrierUpdate, blockIdx.x, epoch + 2u);
  phase_stamp(P, 6);
}

// DEFT_ONESHOT_BLOCKS: CTA cap of the one-shot kernel (default 128)
static int oneshot_max_blocks() {
  static int v = [] {
    const char* e = getenv("DEFT_ONESHOT_BLOCKS");
    int x = e ? atoi(e) : 128;
    return x < 1 ? 1 : (x > kMaxCommBlocks ? kMaxCommBlocks : x);
  }();
  return v;
}

cudaError_t launch_oneshot_update(const PeerPtrs& P, int rank, int world, int dtype,
                                  int64_t slot_base, int32_t count, const int64_t* offsets,
                                  const int64_t* numels, float lr, float momentum,
                                  float grad_scale, float* mom, int max_blocks,
                                  cudaStream_t stream) {
  if (world < 2 || world > 8) return cudaErrorInvalidValue;
  const int N = dtype == 0 ? 4 : 8;
  for (int32_t s0 = 0; s0 < count; s0 += kMaxSeg) {
    SegTable t{};
    t.count = count - s0 < kMaxSeg ? count - s0 : kMaxSeg;
    t.first_vec[0] = 0;
    for (int k = 0; k < t.count; ++k) {
      t.off[k] = offsets[s0 + k];
      t.len[k] = numels[s0 + k];
      t.scale[k] = grad_scale;
      const int64_t aligned = (t.off[k] + N - 1) / N * N;
      const int64_t end = t.off[k] + t.len[k];
      int64_t units = end > aligned ? (end - aligned + N - 1) / N : 0;
      if (units == 0 && t.len[k] > 0) units = 1;
      t.first_vec[k + 1] = t.first_vec[k] + units;
    }
    const int64_t total = t.first_vec[t.count];
    if (total == 0) continue;
    // identical on every rank: a function of the bucket sizes only
    int64_t g = (total + (int64_t)kOneShotThreads * kOneShotUnroll - 1) /
                ((int64_t)kOneShotThreads * kOneShotUnroll);
    int grid = (int)(g < 1 ? 1 : (g > oneshot_max_blocks() ? oneshot_max_blocks() : g));
    if (max_blocks > 0 && grid > max_blocks) grid = max_blocks;
    grid = cap_grid(P, grid);
#define DEFT_OS_CASE(WW)                                                                  \
  case WW:                                                                                \
    if (dtype == 0)                                                                       \
      oneshot_update_kernel<float, WW><<<grid, kOneShotThreads, 0, stream>>>(             \
          P, rank, slot_base, t, lr, momentum, mom);                                      \
    else                                                                                  \
      oneshot_update_kernel<__nv_bfloat16, WW><<<grid, kOneShotThreads, 0, stream>>>(     \
          P, rank, slot_base, t, lr, momentum, mom);                                      \
    break;
    switch (world) {
      DEFT_OS_CASE(2) DEFT_OS_CASE(3) DEFT_OS_CASE(4) DEFT_OS_CASE(5)
      DEFT_OS_CASE(6) DEFT_OS_CASE(7) DEFT_OS_CASE(8)
      default: break;
    }
#undef DEFT_OS_CASE
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace deft
