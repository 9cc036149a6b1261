// K5: the whole DeFT delayed-update state machine as ONE persistent kernel,
// one CTA per scheduler instance (e.g. every retry multiplier of the
// feedback loop, preserver.py:195-234, in parallel).  Replaces
// DeftScheduler.run (scheduler.py:159-342) for exact-mode profiles; the host
// only decodes the compact decision records.
//
// Why it is cheap: _select_from_future (scheduler.py:312-335) always solves
// the subset-sum over ALL n buckets with the same weights -- only the capacity
// changes from stage to stage.  The suffix bitsets built once for the largest
// capacity any stage can ask for (the dual backward window, sum of the link
// capacities) restricted to bits <= c ARE the rows naive_knapsack builds for
// capacity c (knapsack.py:72-78 masks to cap+1 bits; reachability below c does
// not depend on the mask).  So after one O(n * C/32) precompute every stage is
// "highest set bit <= remain" plus the include-earliest reconstruction
// (knapsack.py:79-88).  In exact mode (every capacity <= 1e7) level 0 of the
// recursion always wins (knapsack.py:97-127), so no other level
// is solved.  Scaled-mode instances report DEFT_SCHED_UNSUPPORTED.
//
// Bookkeeping mirrors scheduler.py (greedy multi-knapsack knapsack.py:130-159,
// forced / within placement :187-208, store-or-merge :223-233, drain and flush
// :210-241); it runs on one warp -- it is O(links * n) per stage because the
// (-comm, id) ranking of the buckets never changes and is computed once.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace deft {

constexpr int kSchedThreads = 1024;
constexpr int kSchedMaxN = 1024;
constexpr int kSchedMaxLinks = 4;


// Record layout, per stage: header of 7 ints -- stage (0 fwd / 1 bwd), case
// (1..4), n_transfers, n_events, merged (0/1), grad_group, grad_merge (0/1) --
// then n_transfers x (link, id, group, fresh) and n_events x (uid,
// first_origin, merge_count).  Decoded by gpu_scheduler.py.

struct SchedState {
  uint8_t in_cur[kSchedMaxN + 1];
  uint8_t placed[kSchedMaxN + 1];
  int16_t rank_all[kSchedMaxN];        // bucket ids ordered by (-comm, id)
  int16_t plan_ids[kSchedMaxLinks][kSchedMaxN];
  int32_t plan_len[kSchedMaxLinks];
  int32_t tr_link[2 * kSchedMaxN];     // transfers of the current stage, emit order
  int16_t tr_id[2 * kSchedMaxN];
  int32_t tr_group[2 * kSchedMaxN];
  uint8_t tr_fresh[2 * kSchedMaxN];
  int32_t n_tr;
  int64_t loads[kSchedMaxLinks];
  uint8_t pick[kSchedMaxN + 1];        // reconstruction result, by id
};

__device__ __forceinline__ int roomiest(const int64_t* caps, const int64_t* loads, int L,
                                        int64_t need, bool require_fit) {
  int best = -1;
  int64_t best_room = 0;
  for (int j = 0; j < L; ++j) {
    const int64_t room = caps[j] - loads[j];
    if (require_fit && room < need) continue;
    if (best < 0 || room > best_room) {  // ties keep the lower index: max(room, -j)
      best = j;
      best_room = room;
    }
  }
  return best;
}

__global__ void __launch_bounds__(kSchedThreads, 1) deft_scheduler_kernel(SchedArgs a) {
  extern __shared__ uint32_t smem_row[];
  const int inst = blockIdx.x;
  const int tid = threadIdx.x;
  const int n = a.n, L = a.L;
  const int64_t* fcap = a.fcaps + (int64_t)inst * L;
  const int64_t* bcap = a.bcaps + (int64_t)inst * L;
  int64_t dual = 0;
  for (int j = 0; j < L; ++j) dual += bcap[j];
  if (dual > DEFT_MAX_EXACT_CAPACITY_DEV || n > kSchedMaxN || L > kSchedMaxLinks || n < 1) {
    if (tid == 0) a.status[inst] = -4;  // DEFT_ERR_UNSUPPORTED: host keeps the stage loop
    return;
  }
  const int64_t C = dual;
  const int64_t words = (C + 1 + 31) >> 5;
  uint32_t* rows = a.rows + (int64_t)inst * (n + 1) * a.words;
  int32_t* reach_of = a.reach + (int64_t)inst * (n + 1);

  // ---- phase 1: suffix rows over ascending ids 1..n for capacity C -------------
  // (the in-place top-down chunked update of subset_sum_kernel while the row
  // fits in shared memory; above that, row i is built from the stored row i+1)
  const bool in_smem = words <= a.smem_row_words;
  if (C > 0) {
    if (tid == 0) {
      if (in_smem) smem_row[0] = 1u;
      rows[(int64_t)n * a.words] = 1u;
      reach_of[n] = 0;
    }
    __syncthreads();
    const uint32_t last_mask = ((C & 31) == 31) ? 0xFFFFFFFFu : ((1u << ((C & 31) + 1)) - 1u);
    int64_t reach = 0;
    for (int i = n - 1; i >= 0; --i) {  // item i = bucket id i+1
      const int64_t w = a.comm[i + 1];
      uint32_t* gdst = rows + (int64_t)i * a.words;
      const uint32_t* gsrc = rows + (int64_t)(i + 1) * a.words;
      if (w > C) {  // unplaceable: S[i] == S[i+1]; copy the reachable prefix
        const int64_t hi = reach >> 5;
        for (int64_t j = tid; j <= hi; j += kSchedThreads) gdst[j] = gsrc[j];
        if (tid == 0) reach_of[i] = (int32_t)reach;
        __syncthreads();
        continue;
      }
      const int64_t reach_new = min(C, reach + w);
      const int64_t hi_old = reach >> 5, hi_new = reach_new >> 5;
      const int64_t qw = w >> 5;
      const uint32_t r = (uint32_t)(w & 31);
      const uint32_t* src = in_smem ? smem_row : gsrc;
      for (int64_t top = hi_new; top >= 0; top -= kSchedThreads * 4) {
        uint32_t v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t j = top - tid - (int64_t)k * kSchedThreads;
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
        if (in_smem) __syncthreads();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t j = top - tid - (int64_t)k * kSchedThreads;
          if (j >= 0) {
            if (in_smem) smem_row[j] = v[k];
            gdst[j] = v[k];
          }
        }
      }
      __syncthreads();
      reach = reach_new;
      if (tid == 0) reach_of[i] = (int32_t)reach;
    }
  }
  __syncthreads();

  // (-comm, id) ranking of all buckets, computed in parallel, into shared memory
  // that the row no longer needs.
  SchedState* st = reinterpret_cast<SchedState*>(smem_row);
  for (int i = tid; i < n; i += kSchedThreads) {
    const int64_t wi = a.comm[i + 1];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const int64_t wj = a.comm[j + 1];
      rank += (wj > wi) || (wj == wi && j < i);
    }
    st->rank_all[rank] = (int16_t)(i + 1);
  }
  for (int i = tid; i <= n; i += kSchedThreads)
    st->in_cur[i] = a.carry_in ? a.carry_in[inst].in_cur[i] : 0;
  __syncthreads();
  if (tid >= 32) return;

  // ---- phase 2: the state machine on warp 0 ------------------------------------
  const int lane = tid;
  int32_t* out = a.out + (int64_t)inst * a.out_stride;
  int64_t pos = 0;
  bool overflow = false;
  const SchedCarry* cin = a.carry_in ? a.carry_in + inst : nullptr;
  int next_uid = cin ? cin->next_uid : 0;
  // current group (leftovers being sent): exists iff some in_cur flag is set
  int cur_uid = cin ? cin->cur_uid : -1, cur_first = cin ? cin->cur_first : 0;
  int cur_k = cin ? cin->cur_k : 0, cur_count = cin ? cin->cur_count : 0;
  int64_t cur_backlog = cin ? cin->cur_backlog : 0;
  // future group (all buckets, stored / merged, not yet started)
  int fut_uid = cin ? cin->fut_uid : -1, fut_first = cin ? cin->fut_first : 0;
  int fut_k = cin ? cin->fut_k : 0;
  // pending update events (drained groups) -- at most two per stage
  int pend_n = 0, pend_uid[4], pend_first[4], pend_k[4];

  // link visiting order by (cap, index) for the greedy, per stage kind
  int ford[kSchedMaxLinks], bord[kSchedMaxLinks];
  for (int j = 0; j < L; ++j) ford[j] = bord[j] = j;
  for (int x = 1; x < L; ++x)
    for (int y = x; y > 0; --y) {
      if (fcap[ford[y]] < fcap[ford[y - 1]] ||
          (fcap[ford[y]] == fcap[ford[y - 1]] && ford[y] < ford[y - 1])) {
        const int t = ford[y]; ford[y] = ford[y - 1]; ford[y - 1] = t;
      }
      if (bcap[bord[y]] < bcap[bord[y - 1]] ||
          (bcap[bord[y]] == bcap[bord[y - 1]] && bord[y] < bord[y - 1])) {
        const int t = bord[y]; bord[y] = bord[y - 1]; bord[y - 1] = t;
      }
    }

  auto put = [&](int32_t v) {
    if (pos < a.out_stride) out[pos] = v;
    else overflow = true;
    ++pos;
  };
  auto add_tr = [&](int link, int id, int group, int fresh) {
    const int k = st->n_tr++;
    st->tr_link[k] = link;
    st->tr_id[k] = (int16_t)id;
    st->tr_group[k] = group;
    st->tr_fresh[k] = (uint8_t)fresh;
  };
  // drop ids from the current queue; a drained current group becomes pending
  auto drop_current = [&](int id) {
    if (st->in_cur[id]) {
      st->in_cur[id] = 0;
      --cur_count;
      cur_backlog -= a.comm[id];
    }
  };
  auto check_drained = [&]() {
    if (cur_uid >= 0 && cur_count == 0) {
      pend_uid[pend_n] = cur_uid;
      pend_first[pend_n] = cur_first;
      pend_k[pend_n] = cur_k;
      ++pend_n;
      cur_uid = -1;
    }
  };
  // greedy multi-knapsack over the current queue (knapsack.py:130-159):
  // knapsacks by (cap, index), items by (-weight, id), first fit; transfers are
  // emitted grouped by link index in placement order (like enumerate(selections)).
  auto greedy_current = [&](const int64_t* caps, const int* order) {
    for (int j = 0; j < L; ++j) st->plan_len[j] = 0;
    for (int i = 1; i <= n; ++i) st->placed[i] = 0;
    for (int oi = 0; oi < L; ++oi) {
      const int k = order[oi];
      int64_t room = caps[k];
      for (int r = 0; r < n; ++r) {
        const int id = st->rank_all[r];
        if (!st->in_cur[id] || st->placed[id] || a.comm[id] > room) continue;
        st->placed[id] = 1;
        st->plan_ids[k][st->plan_len[k]++] = (int16_t)id;
        room -= a.comm[id];
      }
    }
    for (int k = 0; k < L; ++k) {
      st->loads[k] = 0;
      for (int x = 0; x < st->plan_len[k]; ++x) {
        const int id = st->plan_ids[k][x];
        add_tr(k, id, cur_uid, 0);
        st->loads[k] += a.comm[id];
      }
    }
    for (int k = 0; k < L; ++k)
      for (int x = 0; x < st->plan_len[k]; ++x) drop_current(st->plan_ids[k][x]);
    check_drained();
  };
  // store-or-merge the new gradients (scheduler.py:223-233); returns merged flag
  auto store_or_merge = [&](int t) -> int {
    if (fut_uid >= 0) {
      ++fut_k;
      return 1;
    }
    fut_uid = next_uid++;
    fut_first = t;
    fut_k = 1;
    return 0;
  };

  for (int t = a.t0; t < a.t0 + a.T && !overflow; ++t) {
    // ------------------------------ forward stage: Case 1
    if (lane == 0) {
      st->n_tr = 0;
      greedy_current(fcap, ford);
      put(0); put(1); put(st->n_tr); put(0); put(0); put(-1); put(0);
      for (int x = 0; x < st->n_tr; ++x) {
        put(st->tr_link[x]); put(st->tr_id[x]); put(st->tr_group[x]); put(st->tr_fresh[x]);
      }
    }
    __syncwarp();
    // ------------------------------ backward stage
    int cas = 0, merged = 0, grad_uid = -1;
    int64_t remain = -1;
    if (lane == 0) {
      st->n_tr = 0;
      for (int k = 0; k < L; ++k) st->loads[k] = 0;
      if (cur_count > 0 && cur_backlog > dual) {           // Case 2
        cas = 2;
        const int uid = cur_uid;
        greedy_current(bcap, bord);
        if (cur_uid < 0 || uid != cur_uid) {
          a.status[inst] = -6;  // "insufficient capacity yet queue drained" (scheduler.py:285-286)
        }
        merged = store_or_merge(t);
        grad_uid = fut_uid;
      } else if (cur_count > 0) {                          // Case 3
        cas = 3;
        const int64_t backlog = cur_backlog;
        for (int r = 0; r < n; ++r) {                      // forced: (-comm, id) order
          const int id = st->rank_all[r];
          if (!st->in_cur[id]) continue;
          const int k = roomiest(bcap, st->loads, L, 0, false);
          add_tr(k, id, cur_uid, 0);
          st->loads[k] += a.comm[id];
        }
        for (int id = 1; id <= n; ++id) drop_current(id);
        check_drained();
        merged = store_or_merge(t);
        grad_uid = fut_uid;
        remain = dual - backlog > 0 ? dual - backlog : 0;
      } else {                                             // Case 4
        cas = 4;
        merged = store_or_merge(t);
        grad_uid = fut_uid;
        remain = dual;
      }
    }
    remain = __shfl_sync(0xffffffffu, remain, 0);
    // select_from_future: level-0 knapsack at capacity `remain` over all buckets
    if (remain >= 0) {  // a future group always exists here (just stored / merged)
      int64_t best = 0;
      const int64_t c = remain < C ? remain : C;
      if (c > 0) {
        // highest reachable sum <= c in S[0] (knapsack.py:79)
        const int64_t top = min((int64_t)reach_of[0], c);
        const uint32_t* s0 = rows;
        int64_t found = -1;
        for (int64_t base = top >> 5; base >= 0 && found < 0; base -= 32) {
          const int64_t j = base - lane;
          int64_t cand = -1;
          if (j >= 0) {
            uint32_t x = s0[j];
            if (j == (top >> 5)) {
              const int b = (int)(top & 31);
              x &= (b == 31) ? 0xFFFFFFFFu : ((1u << (b + 1)) - 1u);
            }
            if (x) cand = j * 32 + 31 - __clz(x);
          }
          for (int o = 16; o > 0; o >>= 1) {
            const int64_t other = __shfl_xor_sync(0xffffffffu, cand, o);
            cand = other > cand ? other : cand;
          }
          found = cand;
        }
        best = found < 0 ? 0 : found;
      }
      // include-earliest reconstruction (knapsack.py:80-88), 5 speculative steps per round
      int64_t target = best;
      for (int i = 0; i < n; i += 5) {
        const int steps = min(5, n - i);
        int64_t tt = target;
        bool consistent = true;
        uint32_t bits = 0;
        for (int s = 0; s < steps; ++s) {
          const int k = i + s;
          const int64_t w = a.comm[k + 1];
          bool bit = false;
          if (w <= tt) {
            const int64_t p = tt - w;
            if (p <= reach_of[k + 1]) bit = (rows[(int64_t)(k + 1) * a.words + (p >> 5)] >> (p & 31)) & 1u;
          }
          const bool assumed = (lane >> s) & 1;
          if (assumed != bit) consistent = false;
          if (assumed) tt -= w;
          bits |= (uint32_t)assumed << s;
        }
        if (lane >= (1 << steps)) consistent = false;
        const uint32_t ballot = __ballot_sync(0xffffffffu, consistent);
        const int winner = __ffs(ballot) - 1;
        target = __shfl_sync(0xffffffffu, tt, winner);
        const uint32_t wb = __shfl_sync(0xffffffffu, bits, winner);
        if (lane < steps) st->pick[i + lane + 1] = (wb >> lane) & 1u;
      }
      __syncwarp();
      if (lane == 0) {
        // place the picks in items order (descending id) on the roomiest fitting link
        int left = 0;
        for (int id = n; id >= 1; --id) {
          if (!st->pick[id]) { ++left; continue; }
          const int64_t w = a.comm[id];
          int k = roomiest(bcap, st->loads, L, w, true);
          if (k < 0) k = roomiest(bcap, st->loads, L, 0, false);
          add_tr(k, id, fut_uid, 1);
          st->loads[k] += w;
        }
        if (left > 0) {  // leftovers become the current group
          cur_uid = fut_uid;
          cur_first = fut_first;
          cur_k = fut_k;
          cur_count = left;
          cur_backlog = 0;
          for (int id = 1; id <= n; ++id)
            if (!st->pick[id]) {
              st->in_cur[id] = 1;
              cur_backlog += a.comm[id];
            }
        } else {
          pend_uid[pend_n] = fut_uid;
          pend_first[pend_n] = fut_first;
          pend_k[pend_n] = fut_k;
          ++pend_n;
        }
        fut_uid = -1;
      }
    }
    if (lane == 0) {
      put(1); put(cas); put(st->n_tr); put(pend_n); put(merged); put(grad_uid); put(merged);
      for (int x = 0; x < st->n_tr; ++x) {
        put(st->tr_link[x]); put(st->tr_id[x]); put(st->tr_group[x]); put(st->tr_fresh[x]);
      }
      for (int e = 0; e < pend_n; ++e) {
        put(pend_uid[e]); put(pend_first[e]); put(pend_k[e]);
      }
      pend_n = 0;
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (a.status[inst] == 0 && overflow) a.status[inst] = -3;
    a.used[inst] = pos;
    if (a.carry_out) {
      SchedCarry* c = a.carry_out + inst;
      c->cur_uid = cur_uid; c->cur_first = cur_first; c->cur_k = cur_k;
      c->cur_count = cur_count; c->cur_backlog = cur_backlog;
      c->fut_uid = fut_uid; c->fut_first = fut_first; c->fut_k = fut_k;
      c->next_uid = next_uid;
      for (int i = 0; i <= n; ++i) c->in_cur[i] = st->in_cur[i];
    }
  }
}

// dynamic shared memory of a launch: the largest row that fits (instances with
// longer rows use the global-row path) or the bookkeeping state, whichever is larger
int64_t sched_smem_bytes(int64_t words) {
  const int64_t row = (words < smem_words_limit() ? words : smem_words_limit()) * 4;
  const int64_t state = (int64_t)sizeof(SchedState);
  return row > state ? row : state;
}

cudaError_t launch_scheduler(const SchedArgs& a, int32_t instances, int64_t smem,
                             cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(deft_scheduler_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(smem_words_limit() * 4));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  deft_scheduler_kernel<<<instances, kSchedThreads, smem, stream>>>(a);
  count_launch();
  return cudaGetLastError();
}

}  // namespace deft
