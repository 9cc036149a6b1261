// K1: batched exact subset-sum (weight == value) for the DeFT solver, sm_100a.
//
// Replaces naive_knapsack (reference knapsack.py:55-94) -- and, batched over
// recursion levels, recursive_knapsack (knapsack.py:97-127).  One CTA owns one
// problem.  Items are in ascending bucket id; the suffix bitsets
//     S[n] = {0},  S[i] = S[i+1] | (S[i+1] << w_i)   masked to cap'+1 bits
// are built from the highest id down (knapsack.py:72-78).  The working row
// lives in shared memory when it fits (<= kSmemWords words, i.e. capacities
// up to ~1.8M us -- every fixture configuration) and is updated IN PLACE,
// top-down in chunks of 4 words per thread: word j of the new row reads only
// words <= j of the old row, so after the chunk's loads a single
// __syncthreads() makes the stores safe, and lower chunks never read the
// stored words.  Every changed row is also streamed to global memory because
// the include-earliest reconstruction (knapsack.py:80-88) walks the rows
// again in the opposite order.  Larger (scaled-mode) rows take the global
// path: row i is computed from the stored row i+1.
//
// Only words up to the reachable bound reach_i = min(cap', sum_{k>=i} w'_k)
// are ever touched (bits above it are provably zero), which makes the common
// "everything fits" case O(n * reach/32) instead of O(n * cap/32).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"

namespace deft {

constexpr int kSubsetThreads = 1024;
constexpr int kWordsPerThread = 4;  // words per thread per in-place chunk
constexpr int64_t kSmemWords = 56 * 1024;  // 224 KiB working row

struct SubsetSumArgs {
  const int64_t* weights;   // concatenated, ascending id, original us
  const int32_t* item_off;  // batch + 1
  const int64_t* caps;      // original capacities (>= 1)
  const int32_t* pids;      // CTA -> problem id
  const int64_t* row_off;   // per problem: offset (uint32 words) of its (n+1) rows
  const int64_t* meta_off;  // per problem: offset (int32) of reach[n+1], slot[n+1]
  uint32_t* rows;
  int32_t* meta;
  uint8_t* take;
  int64_t* best;
};

__device__ __forceinline__ void scale_params(int64_t cap0, int64_t* q, int64_t* cap) {
  // knapsack.py:49-52 -- evaluated in IEEE double like CPython's int/int true division.
  if (cap0 <= DEFT_MAX_EXACT_CAPACITY_DEV) {
    *q = 1;
    *cap = cap0;
  } else {
    *q = (int64_t)ceil((double)cap0 / (double)DEFT_MAX_EXACT_CAPACITY_DEV);
    *cap = cap0 / *q;
  }
}

__device__ __forceinline__ int64_t scaled_w(int64_t w, int64_t q) {
  return q == 1 ? w : (int64_t)ceil((double)w / (double)q);
}

template <bool kSmem>
__global__ void __launch_bounds__(kSubsetThreads, 1) subset_sum_kernel(SubsetSumArgs a) {
  extern __shared__ uint32_t smem_row[];
  __shared__ int64_t s_best[kSubsetThreads / 32];

  const int p = a.pids[blockIdx.x];
  const int tid = threadIdx.x;
  const int32_t i0 = a.item_off[p];
  const int n = a.item_off[p + 1] - i0;
  const int64_t* w_in = a.weights + i0;
  int64_t q, cap;
  scale_params(a.caps[p], &q, &cap);
  const int64_t words = (cap + 1 + 31) >> 5;
  const uint32_t last_mask =
      ((cap & 31) == 31) ? 0xFFFFFFFFu : ((1u << ((cap & 31) + 1)) - 1u);
  uint32_t* rows = a.rows + a.row_off[p];
  int32_t* reach_of = a.meta + a.meta_off[p];  // reach bound of S[k], k = 0..n
  int32_t* slot_of = reach_of + (n + 1);       // which stored row holds S[k]

  // S[n] = {0}: stored explicitly in slot n (one word), reach 0.
  uint32_t* row_n = rows + (int64_t)n * words;
  if (tid == 0) {
    row_n[0] = 1u;
    reach_of[n] = 0;
    slot_of[n] = n;
  }
  if (kSmem && tid == 0) smem_row[0] = 1u;
  __syncthreads();

  int64_t reach = 0;
  int cur_slot = n;  // slot holding the current row (global path source)
  for (int i = n - 1; i >= 0; --i) {
    const int64_t w = scaled_w(w_in[i], q);
    if (w > cap) {  // cannot be placed: S[i] == S[i+1], alias the stored row
      if (tid == 0) {
        reach_of[i] = (int32_t)reach;
        slot_of[i] = cur_slot;
      }
      continue;
    }
    const int64_t reach_new = min(cap, reach + w);
    const int64_t hi_old = reach >> 5, hi_new = reach_new >> 5;
    const int64_t qw = w >> 5;
    const uint32_t r = (uint32_t)(w & 31);
    const uint32_t* src = kSmem ? smem_row : rows + (int64_t)cur_slot * words;
    uint32_t* gdst = rows + (int64_t)i * words;
    const bool store_global = kSmem ? (i >= 1) : true;  // S[0] is only scanned for best
    // chunks of kWordsPerThread * 1024 words, top-down; thread t owns words
    // top - t - k*1024 (k < kWordsPerThread) so every pass stays coalesced
    for (int64_t top = hi_new; top >= 0; top -= kSubsetThreads * kWordsPerThread) {
      uint32_t v[kWordsPerThread];
#pragma unroll
      for (int k = 0; k < kWordsPerThread; ++k) {
        const int64_t j = top - tid - (int64_t)k * kSubsetThreads;
        v[k] = 0;
        if (j >= 0) {
          const uint32_t cur = (j <= hi_old) ? src[j] : 0u;
          const int64_t js = j - qw;
          const uint32_t hi = (js >= 0 && js <= hi_old) ? src[js] : 0u;
          const uint32_t lo = (js >= 1 && js - 1 <= hi_old) ? src[js - 1] : 0u;
          v[k] = cur | __funnelshift_l(lo, hi, r);
          if (j == words - 1) v[k] &= last_mask;
        }
      }
      if (kSmem) __syncthreads();  // all loads of this chunk precede its in-place stores
#pragma unroll
      for (int k = 0; k < kWordsPerThread; ++k) {
        const int64_t j = top - tid - (int64_t)k * kSubsetThreads;
        if (j >= 0) {
          if (kSmem) smem_row[j] = v[k];
          if (store_global) gdst[j] = v[k];
        }
      }
    }
    __syncthreads();
    reach = reach_new;
    cur_slot = i;
    if (tid == 0) {
      reach_of[i] = (int32_t)reach;
      slot_of[i] = i;
    }
  }

  // best = highest set bit of S[0] (knapsack.py:79); bit 0 is always set.
  const uint32_t* row0 = kSmem ? smem_row : rows + (int64_t)cur_slot * words;
  const int64_t hi0 = reach >> 5;
  int64_t best = -1;
  for (int64_t top = hi0; top >= 0 && best < 0; top -= kSubsetThreads) {
    const int64_t j = top - tid;
    int64_t cand = -1;
    if (j >= 0) {
      const uint32_t x = row0[j];
      if (x) cand = j * 32 + 31 - __clz(x);
    }
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t other = __shfl_xor_sync(0xffffffffu, cand, o);
      cand = other > cand ? other : cand;
    }
    if ((tid & 31) == 0) s_best[tid >> 5] = cand;
    __syncthreads();
    int64_t m = -1;
    for (int k = 0; k < kSubsetThreads / 32; ++k) m = s_best[k] > m ? s_best[k] : m;
    best = m;
    __syncthreads();
  }

  // Include-earliest reconstruction (knapsack.py:80-88): item i (ascending id)
  // is taken iff w'_i <= target and bit (target - w'_i) of S[i+1] is set.
  // One warp speculates 5 decisions per round: lane l assumes decision bits
  // l[0..4] for items i..i+4, loads the 5 bits its path needs (independent
  // loads, one memory latency), and the unique self-consistent lane wins.
  if (tid < 32) {
    const int lane = tid;
    int64_t target = best;
    uint8_t* take = a.take + i0;
    for (int i = 0; i < n; i += 5) {
      const int steps = min(5, n - i);
      int64_t t = target;
      bool consistent = true;
      uint32_t path_bits = 0;
      for (int s = 0; s < steps; ++s) {
        const int k = i + s;
        const int64_t w = scaled_w(w_in[k], q);
        bool bit = false;
        if (w <= t) {
          const int64_t pos = t - w;
          if (pos <= reach_of[k + 1]) {
            const uint32_t* rw = rows + (int64_t)slot_of[k + 1] * words;
            bit = (rw[pos >> 5] >> (pos & 31)) & 1u;
          }
        }
        const bool assumed = (lane >> s) & 1;
        if (assumed != bit) consistent = false;
        if (assumed) t -= w;
        path_bits |= (uint32_t)assumed << s;
      }
      if (lane >= (1 << steps)) consistent = false;
      const uint32_t ballot = __ballot_sync(0xffffffffu, consistent);
      const int winner = __ffs(ballot) - 1;  // exactly one lane is consistent
      target = __shfl_sync(0xffffffffu, t, winner);
      const uint32_t bits = __shfl_sync(0xffffffffu, path_bits, winner);
      if (lane < steps) take[i + lane] = (bits >> lane) & 1u;
    }
    if (lane == 0) a.best[p] = best;
  }
}

int64_t host_scaled_cap(int64_t cap0) {
  if (cap0 <= DEFT_MAX_EXACT_CAPACITY_DEV) return cap0;
  const int64_t q = (int64_t)ceil((double)cap0 / (double)DEFT_MAX_EXACT_CAPACITY_DEV);
  return cap0 / q;
}

int64_t host_row_words(int64_t cap0) { return (host_scaled_cap(cap0) + 1 + 31) >> 5; }

cudaError_t launch_subset_sum(const SubsetSumLaunch& L, cudaStream_t stream) {
  SubsetSumArgs a{L.weights, L.item_off, L.caps, nullptr, L.row_off, L.meta_off,
                  L.rows,    L.meta,     L.take, L.best};
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(subset_sum_kernel<true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kSmemWords * 4));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (L.n_small > 0) {
    a.pids = L.pids_small;
    const size_t smem = (size_t)L.max_small_words * 4;
    subset_sum_kernel<true><<<L.n_small, kSubsetThreads, smem, stream>>>(a);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (L.n_large > 0) {
    a.pids = L.pids_large;
    subset_sum_kernel<false><<<L.n_large, kSubsetThreads, 0, stream>>>(a);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int64_t smem_words_limit() { return kSmemWords; }

}  // namespace deft
