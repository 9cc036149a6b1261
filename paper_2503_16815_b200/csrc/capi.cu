// C-ABI of libdeft_b200.so (declared in include/deft_b200.h).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <vector>

#include "../../include/deft_b200.h"
#include "common.cuh"

namespace deft {
static std::atomic<uint64_t> g_launches{0};
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace deft

using namespace deft;

static thread_local std::string g_err;

static deft_status_t fail(deft_status_t code, const std::string& msg) {
  g_err = msg;
  return code;
}
static deft_status_t cuda_fail(cudaError_t e, const char* where) {
  return fail(DEFT_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
// for the other translation units (streams.cu)
deft_status_t deft_fail_cuda(cudaError_t e, const char* where) { return cuda_fail(e, where); }
#define DEFT_CUDA(call)                                  \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

extern "C" int32_t deft_abi_version(void) { return 1; }
extern "C" const char* deft_last_error(void) { return g_err.c_str(); }
extern "C" uint64_t deft_launch_count(void) { return g_launches.load(); }

// ============================================================================
// K1 subset-sum
// ============================================================================
namespace {
struct Layout {
  std::vector<int64_t> row_off, meta_off;
  std::vector<int32_t> small, large;
  int64_t max_small_words = 0;
  size_t rows_words = 0, meta_ints = 0;
};

deft_status_t plan_layout(int32_t batch, const int32_t* n_items, const int64_t* caps, Layout* L) {
  L->row_off.assign(batch + 1, 0);
  L->meta_off.assign(batch + 1, 0);
  for (int32_t p = 0; p < batch; ++p) {
    if (n_items[p] < 1) return fail(DEFT_ERR_INVALID_ARGUMENT, "subset-sum: empty problem");
    if (caps[p] < 1) return fail(DEFT_ERR_INVALID_ARGUMENT, "subset-sum: capacity must be >= 1");
    const int64_t words = host_row_words(caps[p]);
    L->row_off[p + 1] = L->row_off[p] + (int64_t)(n_items[p] + 1) * words;
    L->meta_off[p + 1] = L->meta_off[p] + 2 * (int64_t)(n_items[p] + 1);
    if (words <= smem_words_limit()) {
      L->small.push_back(p);
      L->max_small_words = std::max(L->max_small_words, words);
    } else {
      L->large.push_back(p);
    }
  }
  L->rows_words = (size_t)L->row_off[batch];
  L->meta_ints = (size_t)L->meta_off[batch];
  return DEFT_OK;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// workspace: rows | meta | row_off | meta_off | pids
size_t ws_bytes_for(const Layout& L, int32_t batch) {
  size_t b = align_up(L.rows_words * 4, 256);
  b += align_up(L.meta_ints * 4, 256);
  b += 2 * align_up((size_t)(batch + 1) * 8, 256);
  b += align_up((size_t)batch * 4, 256);
  return b;
}
}  // namespace

extern "C" size_t deft_subset_sum_workspace_bytes(int32_t batch, const int32_t* n_items,
                                                  const int64_t* caps) {
  Layout L;
  if (batch <= 0 || plan_layout(batch, n_items, caps, &L) != DEFT_OK) return 0;
  return ws_bytes_for(L, batch);
}

static deft_status_t launch_with_layout(const Layout& L, const int64_t* d_weights,
                                        const int32_t* d_item_off, const int64_t* d_caps,
                                        int32_t batch, uint8_t* d_take, int64_t* d_best,
                                        char* ws, cudaStream_t stream, bool upload_tables) {
  char* cur = ws;
  uint32_t* rows = reinterpret_cast<uint32_t*>(cur);
  cur += align_up(L.rows_words * 4, 256);
  int32_t* meta = reinterpret_cast<int32_t*>(cur);
  cur += align_up(L.meta_ints * 4, 256);
  int64_t* d_row_off = reinterpret_cast<int64_t*>(cur);
  cur += align_up((size_t)(batch + 1) * 8, 256);
  int64_t* d_meta_off = reinterpret_cast<int64_t*>(cur);
  cur += align_up((size_t)(batch + 1) * 8, 256);
  int32_t* d_pids = reinterpret_cast<int32_t*>(cur);
  if (upload_tables) {
    DEFT_CUDA(cudaMemcpyAsync(d_row_off, L.row_off.data(), (batch + 1) * 8,
                              cudaMemcpyHostToDevice, stream));
    DEFT_CUDA(cudaMemcpyAsync(d_meta_off, L.meta_off.data(), (batch + 1) * 8,
                              cudaMemcpyHostToDevice, stream));
    std::vector<int32_t> pids(L.small);
    pids.insert(pids.end(), L.large.begin(), L.large.end());
    DEFT_CUDA(cudaMemcpyAsync(d_pids, pids.data(), pids.size() * 4, cudaMemcpyHostToDevice,
                              stream));
    // the host vectors must outlive the copies
    DEFT_CUDA(cudaStreamSynchronize(stream));
  }
  SubsetSumLaunch S{};
  S.weights = d_weights;
  S.item_off = d_item_off;
  S.caps = d_caps;
  S.row_off = d_row_off;
  S.meta_off = d_meta_off;
  S.rows = rows;
  S.meta = meta;
  S.take = d_take;
  S.best = d_best;
  S.pids_small = d_pids;
  S.n_small = (int32_t)L.small.size();
  S.max_small_words = L.max_small_words;
  S.pids_large = d_pids + L.small.size();
  S.n_large = (int32_t)L.large.size();
  cudaError_t e = launch_subset_sum(S, stream);
  if (e != cudaSuccess) return cuda_fail(e, "subset_sum_kernel");
  return DEFT_OK;
}

extern "C" deft_status_t deft_subset_sum_batched(const int64_t* d_weights,
                                                 const int32_t* d_item_off,
                                                 const int64_t* d_caps, int32_t batch,
                                                 const int32_t* n_items, const int64_t* caps,
                                                 uint8_t* d_take, int64_t* d_best, void* d_ws,
                                                 size_t ws_bytes, void* stream) {
  if (batch <= 0) return DEFT_OK;
  Layout L;
  deft_status_t st = plan_layout(batch, n_items, caps, &L);
  if (st != DEFT_OK) return st;
  if (ws_bytes < ws_bytes_for(L, batch))
    return fail(DEFT_ERR_WORKSPACE, "subset-sum: workspace too small");
  return launch_with_layout(L, d_weights, d_item_off, d_caps, batch, d_take, d_best,
                            reinterpret_cast<char*>(d_ws), (cudaStream_t)stream, true);
}

struct deft_solver {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  char* pinned = nullptr;
  size_t pinned_bytes = 0;
  char* dev = nullptr;  // inputs + outputs + workspace
  size_t dev_bytes = 0;
  float last_ms = 0.f;
};

static deft_status_t grow(deft_solver* s, size_t pinned_need, size_t dev_need) {
  if (pinned_need > s->pinned_bytes) {
    if (s->pinned) cudaFreeHost(s->pinned);
    size_t nb = std::max(pinned_need, s->pinned_bytes * 2);
    DEFT_CUDA(cudaMallocHost(&s->pinned, nb));
    s->pinned_bytes = nb;
  }
  if (dev_need > s->dev_bytes) {
    if (s->dev) cudaFree(s->dev);
    size_t nb = std::max(dev_need, s->dev_bytes * 2);
    DEFT_CUDA(cudaMalloc(&s->dev, nb));
    s->dev_bytes = nb;
  }
  return DEFT_OK;
}

extern "C" deft_status_t deft_solver_create(int32_t device, deft_solver** out) {
  if (!out) return fail(DEFT_ERR_INVALID_ARGUMENT, "null out");
  deft_solver* s = new deft_solver();
  s->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete s;
    return cuda_fail(e, "cudaSetDevice");
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  e = cudaStreamCreateWithPriority(&s->stream, cudaStreamNonBlocking, hi);
  if (e == cudaSuccess) e = cudaEventCreate(&s->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&s->ev1);
  if (e != cudaSuccess) {
    delete s;
    return cuda_fail(e, "deft_solver_create");
  }
  *out = s;
  return DEFT_OK;
}

extern "C" deft_status_t deft_solver_destroy(deft_solver* s) {
  if (!s) return DEFT_OK;
  if (s->stream) cudaStreamSynchronize(s->stream);
  if (s->pinned) cudaFreeHost(s->pinned);
  if (s->dev) cudaFree(s->dev);
  if (s->ev0) cudaEventDestroy(s->ev0);
  if (s->ev1) cudaEventDestroy(s->ev1);
  if (s->stream) cudaStreamDestroy(s->stream);
  delete s;
  return DEFT_OK;
}

extern "C" float deft_solver_last_kernel_ms(const deft_solver* s) { return s ? s->last_ms : 0.f; }

extern "C" deft_status_t deft_solver_solve(deft_solver* s, int32_t batch, const int32_t* n_items,
                                           const int64_t* weights, const int64_t* caps,
                                           uint8_t* take_out, int64_t* best_out) {
  if (!s) return fail(DEFT_ERR_INVALID_ARGUMENT, "null solver");
  if (batch <= 0) return DEFT_OK;
  Layout L;
  deft_status_t st = plan_layout(batch, n_items, caps, &L);
  if (st != DEFT_OK) return st;
  int64_t total_items = 0;
  for (int32_t p = 0; p < batch; ++p) total_items += n_items[p];
  // pinned staging: weights | item_off | caps | row_off | meta_off | pids  ||  take | best
  const size_t b_w = align_up(total_items * 8, 256), b_io = align_up((batch + 1) * 4, 256);
  const size_t b_caps = align_up(batch * 8, 256), b_tab = align_up((batch + 1) * 8, 256);
  const size_t b_pids = align_up(batch * 4, 256);
  const size_t in_bytes = b_w + b_io + b_caps + 2 * b_tab + b_pids;
  const size_t b_take = align_up(total_items, 256), b_best = align_up(batch * 8, 256);
  const size_t out_bytes = b_take + b_best;
  const size_t ws = align_up(L.rows_words * 4, 256) + align_up(L.meta_ints * 4, 256);
  if (cudaSetDevice(s->device) != cudaSuccess) return fail(DEFT_ERR_CUDA, "cudaSetDevice");
  st = grow(s, in_bytes + out_bytes, in_bytes + out_bytes + ws);
  if (st != DEFT_OK) return st;

  char* h = s->pinned;
  memcpy(h, weights, total_items * 8);
  int32_t* io = reinterpret_cast<int32_t*>(h + b_w);
  io[0] = 0;
  for (int32_t p = 0; p < batch; ++p) io[p + 1] = io[p] + n_items[p];
  memcpy(h + b_w + b_io, caps, batch * 8);
  memcpy(h + b_w + b_io + b_caps, L.row_off.data(), (batch + 1) * 8);
  memcpy(h + b_w + b_io + b_caps + b_tab, L.meta_off.data(), (batch + 1) * 8);
  int32_t* pids = reinterpret_cast<int32_t*>(h + b_w + b_io + b_caps + 2 * b_tab);
  size_t k = 0;
  for (int32_t p : L.small) pids[k++] = p;
  for (int32_t p : L.large) pids[k++] = p;

  char* d = s->dev;
  DEFT_CUDA(cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, s->stream));
  SubsetSumLaunch S{};
  S.weights = reinterpret_cast<const int64_t*>(d);
  S.item_off = reinterpret_cast<const int32_t*>(d + b_w);
  S.caps = reinterpret_cast<const int64_t*>(d + b_w + b_io);
  S.row_off = reinterpret_cast<const int64_t*>(d + b_w + b_io + b_caps);
  S.meta_off = reinterpret_cast<const int64_t*>(d + b_w + b_io + b_caps + b_tab);
  const int32_t* d_pids = reinterpret_cast<const int32_t*>(d + b_w + b_io + b_caps + 2 * b_tab);
  S.pids_small = d_pids;
  S.n_small = (int32_t)L.small.size();
  S.max_small_words = L.max_small_words;
  S.pids_large = d_pids + L.small.size();
  S.n_large = (int32_t)L.large.size();
  char* d_out = d + in_bytes;
  S.take = reinterpret_cast<uint8_t*>(d_out);
  S.best = reinterpret_cast<int64_t*>(d_out + b_take);
  char* wsp = d_out + out_bytes;
  S.rows = reinterpret_cast<uint32_t*>(wsp);
  S.meta = reinterpret_cast<int32_t*>(wsp + align_up(L.rows_words * 4, 256));
  DEFT_CUDA(cudaEventRecord(s->ev0, s->stream));
  cudaError_t e = launch_subset_sum(S, s->stream);
  if (e != cudaSuccess) return cuda_fail(e, "subset_sum_kernel");
  DEFT_CUDA(cudaEventRecord(s->ev1, s->stream));
  char* h_out = h + in_bytes;
  DEFT_CUDA(cudaMemcpyAsync(h_out, d_out, out_bytes, cudaMemcpyDeviceToHost, s->stream));
  DEFT_CUDA(cudaStreamSynchronize(s->stream));
  cudaEventElapsedTime(&s->last_ms, s->ev0, s->ev1);
  memcpy(take_out, h_out, total_items);
  memcpy(best_out, h_out + b_take, batch * 8);
  return DEFT_OK;
}

// ============================================================================
// Symmetric memory (CUDA IPC)
// ============================================================================
extern "C" deft_status_t deft_mem_alloc(size_t bytes, void** d_ptr, uint8_t* ipc_handle_out) {
  if (!d_ptr || bytes == 0) return fail(DEFT_ERR_INVALID_ARGUMENT, "deft_mem_alloc");
  DEFT_CUDA(cudaMalloc(d_ptr, bytes));
  DEFT_CUDA(cudaMemset(*d_ptr, 0, bytes));
  if (ipc_handle_out) {
    cudaIpcMemHandle_t h;
    DEFT_CUDA(cudaIpcGetMemHandle(&h, *d_ptr));
    memcpy(ipc_handle_out, &h, sizeof(h));
  }
  return DEFT_OK;
}
extern "C" deft_status_t deft_mem_free(void* d_ptr) {
  DEFT_CUDA(cudaFree(d_ptr));
  return DEFT_OK;
}
extern "C" deft_status_t deft_mem_open(const uint8_t* ipc_handle, void** d_peer_ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  DEFT_CUDA(cudaIpcOpenMemHandle(d_peer_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return DEFT_OK;
}
extern "C" deft_status_t deft_mem_close(void* d_peer_ptr) {
  DEFT_CUDA(cudaIpcCloseMemHandle(d_peer_ptr));
  return DEFT_OK;
}

// ============================================================================
// Communicator
// ============================================================================
struct deft_comm {
  int rank = 0, world = 1, dtype = 0, n_slots = 0;
  int64_t slot_elems = 0;
  PeerPtrs P{};
  char* staging = nullptr;  // CE channel: (W-1) peer shards
  size_t staging_bytes = 0;
  int update_blocks = 0;    // CTA budget of the update kernels (0 = comm default)
};

extern "C" size_t deft_comm_flag_bytes(int32_t world) {
  (void)world;
  return (size_t)kNumBarrierSets * kMaxCommBlocks * (kMaxWorld + 1) * sizeof(uint32_t);
}

// DEFT_SPIN_TIMEOUT_MS (default 120 s; 0 = unbounded): longest wait of a peer
// barrier before the kernel traps
static uint64_t default_spin_timeout_ns() {
  const char* e = getenv("DEFT_SPIN_TIMEOUT_MS");
  const long long ms = e ? atoll(e) : 120000LL;
  return ms > 0 ? (uint64_t)ms * 1000000ull : 0ull;
}

extern "C" deft_status_t deft_comm_create(int32_t rank, int32_t world, void* const* grads,
                                          void* const* params, void* const* flags,
                                          float* d_master, int64_t slot_elems, int32_t n_slots,
                                          int32_t grad_dtype, deft_comm** out) {
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world || !out)
    return fail(DEFT_ERR_INVALID_ARGUMENT, "deft_comm_create: bad rank/world");
  if (grad_dtype != DEFT_DTYPE_F32 && grad_dtype != DEFT_DTYPE_BF16)
    return fail(DEFT_ERR_INVALID_ARGUMENT, "deft_comm_create: bad dtype");
  if (grad_dtype == DEFT_DTYPE_BF16 && !d_master)
    return fail(DEFT_ERR_INVALID_ARGUMENT, "deft_comm_create: bf16 parameters need an fp32 master");
  deft_comm* c = new deft_comm();
  c->P.master = grad_dtype == DEFT_DTYPE_BF16 ? d_master : nullptr;
  c->P.grid_cap = 0;
  c->P.spin_timeout_ns = default_spin_timeout_ns();
  c->P.phase_ts = nullptr;
  {
    const char* e = getenv("DEFT_BARRIER_FENCE");
    c->P.barrier_fence_all = e && strcmp(e, "all") == 0;
  }
  {
    const char* e = getenv("DEFT_PROFILE_NO_PEER_BARRIER");
    c->P.no_peer_barrier = e && atoi(e) == 1;
    if (c->P.no_peer_barrier)
      fprintf(stderr, "deft: DEFT_PROFILE_NO_PEER_BARRIER=1 -- peer barriers disabled, "
                      "results are racy (profiling only)\n");
  }
  c->rank = rank;
  c->world = world;
  c->dtype = grad_dtype;
  c->slot_elems = slot_elems;
  c->n_slots = n_slots;
  for (int r = 0; r < world; ++r) {
    c->P.grads[r] = reinterpret_cast<char*>(grads[r]);
    c->P.params[r] = params[r];
    c->P.flags[r] = flags ? reinterpret_cast<uint32_t*>(flags[r]) : nullptr;
    if (world > 1 && !c->P.flags[r]) {
      delete c;
      return fail(DEFT_ERR_INVALID_ARGUMENT, "deft_comm_create: flags required for world > 1");
    }
  }
  if (world > 1) {
    // copy-engine staging sized up front for any transfer list over one slot (the
    // (W-1) peer shards of every bucket + 16-byte stride padding for up to 4096
    // buckets): growing it later would synchronise, which a CUDA-graph capture
    // cannot do
    const size_t esz = grad_dtype == DEFT_DTYPE_F32 ? 4 : 2;
    const size_t need = (size_t)(world - 1) *
                        ((size_t)(slot_elems + world - 1) / world + (size_t)24 * 4096) * esz;
    cudaError_t e = cudaMalloc(&c->staging, need);
    if (e != cudaSuccess) {
      delete c;
      return cuda_fail(e, "deft_comm_create: staging");
    }
    c->staging_bytes = need;
  }
  *out = c;
  return DEFT_OK;
}

extern "C" deft_status_t deft_comm_set_update_blocks(deft_comm* c, int32_t blocks) {
  if (!c || blocks < 0 || blocks > kMaxCommBlocks)
    return fail(DEFT_ERR_INVALID_ARGUMENT, "deft_comm_set_update_blocks");
  c->update_blocks = blocks;
  return DEFT_OK;
}

extern "C" deft_status_t deft_comm_configure(deft_comm* c, int32_t grid_cap,
                                             int64_t spin_timeout_ms) {
  if (!c || grid_cap > kMaxCommBlocks)
    return fail(DEFT_ERR_INVALID_ARGUMENT, "deft_comm_configure");
  if (grid_cap >= 0) c->P.grid_cap = grid_cap;
  if (spin_timeout_ms >= 0) c->P.spin_timeout_ns = (uint64_t)spin_timeout_ms * 1000000ull;
  return DEFT_OK;
}

extern "C" deft_status_t deft_comm_set_phase_trace(deft_comm* c, uint64_t* dev_stamps) {
  if (!c) return fail(DEFT_ERR_INVALID_ARGUMENT, "deft_comm_set_phase_trace");
  c->P.phase_ts = dev_stamps;
  return DEFT_OK;
}

extern "C" deft_status_t deft_comm_destroy(deft_comm* c) {
  if (!c) return DEFT_OK;
  if (c->staging) cudaFree(c->staging);
  delete c;
  return DEFT_OK;
}

static deft_status_t check_range(const deft_comm* c, int32_t slot, int64_t offset, int64_t numel) {
  if (slot < 0 || slot >= c->n_slots) return fail(DEFT_ERR_INVALID_ARGUMENT, "bad slot");
  if (offset < 0 || numel < 0 || offset + numel > c->slot_elems)
    return fail(DEFT_ERR_INVALID_ARGUMENT, "bucket range outside the gradient slot");
  return DEFT_OK;
}

extern "C" deft_status_t deft_bucket_reduce_scatter(deft_comm* c, int32_t channel, int32_t slot,
                                                    int64_t offset, int64_t numel,
                                                    void* stream) {
  if (!c) return fail(DEFT_ERR_INVALID_ARGUMENT, "null comm");
  deft_status_t st = check_range(c, slot, offset, numel);
  if (st != DEFT_OK) return st;
  if (c->world == 1 || numel == 0) return DEFT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t slot_base = (int64_t)slot * c->slot_elems;
  if (channel == DEFT_CHANNEL_SM) {
    cudaError_t e = launch_reduce_scatter_sm(c->P, c->rank, c->world, c->dtype, slot_base, offset,
                                             numel, s);
    if (e != cudaSuccess) return cuda_fail(e, "reduce_scatter_kernel");
    return DEFT_OK;
  }
  if (channel != DEFT_CHANNEL_CE) return fail(DEFT_ERR_INVALID_ARGUMENT, "bad channel");
  // copy-engine channel: barrier, (W-1) peer->local DMA copies, local SM reduce
  const int esz = c->dtype == DEFT_DTYPE_F32 ? 4 : 2;
  const ShardRange sh = shard_of(offset, numel, c->rank, c->world, c->dtype == 0 ? 4 : 8);
  const int64_t len = sh.hi - sh.lo;
  const int64_t per = ((numel + c->world - 1) / c->world + 16 + 7) / 8 * 8;  // 16-B strides
  const size_t need = (size_t)(c->world - 1) * per * esz;
  if (need > c->staging_bytes) {
    if (c->staging) {
      DEFT_CUDA(cudaStreamSynchronize(s));
      cudaFree(c->staging);
    }
    DEFT_CUDA(cudaMalloc(&c->staging, need));
    c->staging_bytes = need;
  }
  cudaError_t e = launch_barrier(c->P, c->rank, c->world, kBarrierCE, s);
  if (e != cudaSuccess) return cuda_fail(e, "barrier_kernel");
  if (len > 0) {
    int k = 0;
    for (int r = 0; r < c->world; ++r) {
      if (r == c->rank) continue;
      const char* src = c->P.grads[r] + (slot_base + sh.lo) * esz;
      DEFT_CUDA(cudaMemcpyAsync(c->staging + (size_t)k * per * esz, src, (size_t)len * esz,
                                cudaMemcpyDeviceToDevice, s));
      ++k;
    }
  }
  e = launch_ce_reduce(c->P.grads[c->rank] + slot_base * esz, c->staging, c->dtype, c->world,
                       c->rank, sh.lo, len, per, s);
  if (e != cudaSuccess) return cuda_fail(e, "ce_reduce_kernel");
  // peers must be done pulling from us before our slot can change again: the
  // update kernel's entry barrier orders that (see bucket_comm.cu).
  return DEFT_OK;
}

extern "C" deft_status_t deft_bucket_reduce_scatter_multi(deft_comm* c, int32_t channel,
                                                          int32_t slot, int32_t count,
                                                          const int64_t* offsets,
                                                          const int64_t* numels, void* stream) {
  if (!c) return fail(DEFT_ERR_INVALID_ARGUMENT, "null comm");
  if (count < 0 || (count > 0 && (!offsets || !numels)))
    return fail(DEFT_ERR_INVALID_ARGUMENT, "bad bucket list");
  for (int32_t k = 0; k < count; ++k) {
    deft_status_t st = check_range(c, slot, offsets[k], numels[k]);
    if (st != DEFT_OK) return st;
  }
  if (c->world == 1 || count == 0) return DEFT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t slot_base = (int64_t)slot * c->slot_elems;
  if (channel == DEFT_CHANNEL_SM) {
    cudaError_t e = launch_reduce_scatter_sm_multi(c->P, c->rank, c->world, c->dtype, slot_base,
                                                   count, offsets, numels, s);
    if (e != cudaSuccess) return cuda_fail(e, "reduce_scatter_tma_kernel");
    return DEFT_OK;
  }
  if (channel != DEFT_CHANNEL_CE) return fail(DEFT_ERR_INVALID_ARGUMENT, "bad channel");
  // copy-engine channel: ONE barrier, then per bucket (W-1) DMA copies + local reduce
  const int esz = c->dtype == DEFT_DTYPE_F32 ? 4 : 2;
  size_t need = 0;
  for (int32_t k = 0; k < count; ++k) {
    const int64_t per = ((numels[k] + c->world - 1) / c->world + 16 + 7) / 8 * 8;
    need += (size_t)(c->world - 1) * per * esz;
  }
  if (need > c->staging_bytes) {
    if (c->staging) {
      DEFT_CUDA(cudaStreamSynchronize(s));
      cudaFree(c->staging);
    }
    DEFT_CUDA(cudaMalloc(&c->staging, need));
    c->staging_bytes = need;
  }
  cudaError_t e = launch_barrier(c->P, c->rank, c->world, kBarrierCE, s);
  if (e != cudaSuccess) return cuda_fail(e, "barrier_kernel");
  size_t base = 0;
  for (int32_t k = 0; k < count; ++k) {
    const ShardRange sh = shard_of(offsets[k], numels[k], c->rank, c->world,
                                   c->dtype == 0 ? 4 : 8);
    const int64_t len = sh.hi - sh.lo;
    const int64_t per = ((numels[k] + c->world - 1) / c->world + 16 + 7) / 8 * 8;
    char* stage = c->staging + base;
    if (len > 0) {
      int j = 0;
      for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) continue;
        const char* src = c->P.grads[r] + (slot_base + sh.lo) * esz;
        DEFT_CUDA(cudaMemcpyAsync(stage + (size_t)j * per * esz, src, (size_t)len * esz,
                                  cudaMemcpyDeviceToDevice, s));
        ++j;
      }
      e = launch_ce_reduce(c->P.grads[c->rank] + slot_base * esz, stage, c->dtype, c->world,
                           c->rank, sh.lo, len, per, s);
      if (e != cudaSuccess) return cuda_fail(e, "ce_reduce_kernel");
    }
    base += (size_t)(c->world - 1) * per * esz;
  }
  return DEFT_OK;
}

extern "C" deft_status_t deft_bucket_update(deft_comm* c, int32_t slot, int64_t offset,
                                           int64_t numel, float lr, float momentum,
                                           float grad_scale, float* d_mom, void* stream) {
  if (!c) return fail(DEFT_ERR_INVALID_ARGUMENT, "null comm");
  deft_status_t st = check_range(c, slot, offset, numel);
  if (st != DEFT_OK) return st;
  if (numel == 0) return DEFT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t slot_base = (int64_t)slot * c->slot_elems;
  if (c->world == 1) {
    const int esz = c->dtype == DEFT_DTYPE_F32 ? 4 : 2;
    const char* g = c->P.grads[0] + slot_base * esz;
    cudaError_t e = launch_sgd_local(g, c->dtype, c->P.params[0], c->P.master, d_mom, 1,
                                     &offset, &numel, &grad_scale, lr, momentum, s);
    if (e != cudaSuccess) return cuda_fail(e, "sgd_local_kernel");
    return DEFT_OK;
  }
  cudaError_t e = launch_update_allgather(c->P, c->rank, c->world, c->dtype, slot_base, offset,
                                          numel, lr, momentum, grad_scale, d_mom,
                                          c->update_blocks, s);
  if (e != cudaSuccess) return cuda_fail(e, "update_allgather_kernel");
  return DEFT_OK;
}

extern "C" deft_status_t deft_sgd_momentum_update(const void* d_grad, int32_t grad_dtype,
                                                  void* d_param, float* d_master, float* d_mom,
                                                  int64_t numel, float lr, float momentum,
                                                  float grad_scale, void* stream) {
  if (numel == 0) return DEFT_OK;
  if (grad_dtype == DEFT_DTYPE_BF16 && !d_master)
    return fail(DEFT_ERR_INVALID_ARGUMENT, "bf16 parameters need an fp32 master");
  int64_t off = 0;
  cudaError_t e = launch_sgd_local(d_grad, grad_dtype, d_param, d_master, d_mom, 1, &off, &numel,
                                   &grad_scale, lr, momentum, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "sgd_local_kernel");
  return DEFT_OK;
}

extern "C" deft_status_t deft_sgd_momentum_update_multi(const void* d_grad, int32_t grad_dtype,
                                                        void* d_param, float* d_master,
                                                        float* d_mom, int32_t count,
                                                        const int64_t* offsets,
                                                        const int64_t* numels,
                                                        const float* grad_scales, float lr,
                                                        float momentum, void* stream) {
  if (count <= 0) return DEFT_OK;
  if (grad_dtype == DEFT_DTYPE_BF16 && !d_master)
    return fail(DEFT_ERR_INVALID_ARGUMENT, "bf16 parameters need an fp32 master");
  cudaError_t e = launch_sgd_local(d_grad, grad_dtype, d_param, d_master, d_mom, count, offsets,
                                   numels, grad_scales, lr, momentum, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "sgd_local_kernel");
  return DEFT_OK;
}

extern "C" deft_status_t deft_gather_segments(void* d_dst, const void* const* d_srcs,
                                              const int64_t* dst_offsets,
                                              const int64_t* byte_lens, int32_t count,
                                              int64_t ce_min_bytes, void* stream) {
  if (count <= 0) return DEFT_OK;
  if (!d_dst || !d_srcs || !dst_offsets || !byte_lens)
    return fail(DEFT_ERR_INVALID_ARGUMENT, "deft_gather_segments: null argument");
  cudaError_t e = launch_gather(reinterpret_cast<char*>(d_dst), d_srcs, dst_offsets, byte_lens,
                                count, ce_min_bytes, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "gather_kernel");
  return DEFT_OK;
}

extern "C" deft_status_t deft_bucket_update_multi(deft_comm* c, int32_t slot, int32_t count,
                                                 const int64_t* offsets, const int64_t* numels,
                                                 float lr, float momentum, float grad_scale,
                                                 float* d_mom, void* stream) {
  if (!c) return fail(DEFT_ERR_INVALID_ARGUMENT, "null comm");
  if (count <= 0) return DEFT_OK;
  for (int32_t k = 0; k < count; ++k) {
    deft_status_t st = check_range(c, slot, offsets[k], numels[k]);
    if (st != DEFT_OK) return st;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t slot_base = (int64_t)slot * c->slot_elems;
  if (c->world == 1) {
    const int esz = c->dtype == DEFT_DTYPE_F32 ? 4 : 2;
    std::vector<float> scales(count, grad_scale);
    cudaError_t e = launch_sgd_local(c->P.grads[0] + slot_base * esz, c->dtype, c->P.params[0],
                                     c->P.master, d_mom, count, offsets, numels, scales.data(),
                                     lr, momentum, s);
    if (e != cudaSuccess) return cuda_fail(e, "sgd_local_kernel");
    return DEFT_OK;
  }
  cudaError_t e = launch_update_allgather_multi(c->P, c->rank, c->world, c->dtype, slot_base,
                                                count, offsets, numels, lr, momentum, grad_scale,
                                                d_mom, c->update_blocks, s);
  if (e != cudaSuccess) return cuda_fail(e, "update_allgather_multi_kernel");
  return DEFT_OK;
}

extern "C" deft_status_t deft_bucket_sync_update_multi(deft_comm* c, int32_t slot,
                                                      int32_t count, const int64_t* offsets,
                                                      const int64_t* numels, float lr,
                                                      float momentum, float grad_scale,
                                                      float* d_mom, void* stream) {
  if (!c) return fail(DEFT_ERR_INVALID_ARGUMENT, "null comm");
  if (count <= 0) return DEFT_OK;
  if (!d_mom) return fail(DEFT_ERR_INVALID_ARGUMENT, "momentum buffer required");
  for (int32_t k = 0; k < count; ++k) {
    deft_status_t st = check_range(c, slot, offsets[k], numels[k]);
    if (st != DEFT_OK) return st;
  }
  if (c->world == 1)   // nothing to reduce: the local fused update
    return deft_bucket_update_multi(c, slot, count, offsets, numels, lr, momentum, grad_scale,
                                    d_mom, stream);
  cudaError_t e = launch_oneshot_update(c->P, c->rank, c->world, c->dtype,
                                        (int64_t)slot * c->slot_elems, count, offsets, numels,
                                        lr, momentum, grad_scale, d_mom, c->update_blocks,
                                        (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "oneshot_update_kernel");
  return DEFT_OK;
}

// ============================================================================
// Loopback collectives (one launch for all ranks of a loopback world)
// ============================================================================
static deft_status_t check_loopback(deft_comm* const* comms, int32_t world) {
  if (!comms || world < 2 || world > kMaxWorld)
    return fail(DEFT_ERR_INVALID_ARGUMENT, "loopback: bad world");
  for (int32_t r = 0; r < world; ++r) {
    if (!comms[r] || comms[r]->rank != r || comms[r]->world != world ||
        comms[r]->dtype != comms[0]->dtype || comms[r]->slot_elems != comms[0]->slot_elems)
      return fail(DEFT_ERR_INVALID_ARGUMENT, "loopback: comms must be ranks 0..W-1 of one world");
    for (int k = 0; k < world; ++k)
      if (comms[r]->P.grads[k] != comms[0]->P.grads[k] ||
          comms[r]->P.flags[k] != comms[0]->P.flags[k])
        return fail(DEFT_ERR_INVALID_ARGUMENT, "loopback: comms of different worlds");
  }
  return DEFT_OK;
}

extern "C" deft_status_t deft_loopback_reduce_scatter(deft_comm* const* comms, int32_t world,
                                                      int32_t channel, int32_t slot,
                                                      int32_t count, const int64_t* offsets,
                                                      const int64_t* numels, void* stream) {
  deft_status_t st = check_loopback(comms, world);
  if (st != DEFT_OK) return st;
  const deft_comm* c0 = comms[0];
  for (int32_t k = 0; k < count; ++k) {
    st = check_range(c0, slot, offsets[k], numels[k]);
    if (st != DEFT_OK) return st;
  }
  if (count <= 0) return DEFT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t slot_base = (int64_t)slot * c0->slot_elems;
  if (channel == DEFT_CHANNEL_SM) {
    cudaError_t e = launch_rs_tma_loopback(c0->P, world, c0->dtype, slot_base, count, offsets,
                                           numels, s);
    if (e != cudaSuccess) return cuda_fail(e, "reduce_scatter_tma_kernel (loopback)");
    return DEFT_OK;
  }
  if (channel != DEFT_CHANNEL_CE) return fail(DEFT_ERR_INVALID_ARGUMENT, "bad channel");
  // one barrier launch for all ranks, then every rank's copies + local reduce
  cudaError_t e = launch_barrier_loopback(c0->P, world, kBarrierCE, s);
  if (e != cudaSuccess) return cuda_fail(e, "barrier_kernel (loopback)");
  const int esz = c0->dtype == DEFT_DTYPE_F32 ? 4 : 2;
  for (int32_t r = 0; r < world; ++r) {
    deft_comm* c = comms[r];
    size_t base = 0;
    for (int32_t k = 0; k < count; ++k) {
      const ShardRange sh = shard_of(offsets[k], numels[k], r, world, c0->dtype == 0 ? 4 : 8);
      const int64_t len = sh.hi - sh.lo;
      const int64_t per = ((numels[k] + world - 1) / world + 16 + 7) / 8 * 8;
      if (base + (size_t)(world - 1) * per * esz > c->staging_bytes)
        return fail(DEFT_ERR_WORKSPACE, "loopback: copy-engine staging too small");
      char* stage = c->staging + base;
      if (len > 0) {
        int j = 0;
        for (int q = 0; q < world; ++q) {
          if (q == r) continue;
          DEFT_CUDA(cudaMemcpyAsync(stage + (size_t)j * per * esz,
                                    c->P.grads[q] + (slot_base + sh.lo) * esz, (size_t)len * esz,
                                    cudaMemcpyDeviceToDevice, s));
          ++j;
        }
        e = launch_ce_reduce(c->P.grads[r] + slot_base * esz, stage, c0->dtype, world, r, sh.lo,
                             len, per, s);
        if (e != cudaSuccess) return cuda_fail(e, "ce_reduce_kernel (loopback)");
      }
      base += (size_t)(world - 1) * per * esz;
    }
  }
  DEFT_CUDA(cudaStreamSynchronize(s));
  return DEFT_OK;
}

extern "C" deft_status_t deft_loopback_update(deft_comm* const* comms, int32_t world,
                                              int32_t slot, int32_t count,
                                              const int64_t* offsets, const int64_t* numels,
                                              float lr, float momentum, float grad_scale,
                                              float* const* d_moms, void* stream) {
  deft_status_t st = check_loopback(comms, world);
  if (st != DEFT_OK) return st;
  if (!d_moms) return fail(DEFT_ERR_INVALID_ARGUMENT, "loopback: momentum buffers required");
  const deft_comm* c0 = comms[0];
  for (int32_t k = 0; k < count; ++k) {
    st = check_range(c0, slot, offsets[k], numels[k]);
    if (st != DEFT_OK) return st;
  }
  if (count <= 0) return DEFT_OK;
  std::vector<float*> masters(world);
  for (int32_t r = 0; r < world; ++r) masters[r] = comms[r]->P.master;
  cudaError_t e = launch_update_tma_loopback(
      c0->P, world, c0->dtype, (int64_t)slot * c0->slot_elems, count, offsets, numels, lr,
      momentum, grad_scale, d_moms, masters.data(), c0->update_blocks, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "update_allgather_tma_kernel (loopback)");
  return DEFT_OK;
}

// ============================================================================
// K5: persistent DeFT state machine (scheduler_kernel.cu)
// ============================================================================
extern "C" size_t deft_sched_carry_bytes(void) { return sizeof(SchedCarry); }

extern "C" deft_status_t deft_solver_schedule_chunk(
    deft_solver* s, int32_t instances, int32_t n, int32_t n_links, int32_t t0,
    int32_t iterations, const int64_t* comm, const int64_t* bwd, const int64_t* fwd_caps,
    const int64_t* bwd_caps, const void* carry_in, void* carry_out, int32_t* out,
    int64_t out_stride, int64_t* used, int32_t* status) {
  if (!s || instances <= 0 || n <= 0 || n_links <= 0 || iterations < 0)
    return fail(DEFT_ERR_INVALID_ARGUMENT, "deft_solver_schedule: bad arguments");
  if (cudaSetDevice(s->device) != cudaSuccess) return fail(DEFT_ERR_CUDA, "cudaSetDevice");
  int64_t words = 1, smem_words = 0;
  for (int32_t i = 0; i < instances; ++i) {
    int64_t dual = 0;
    for (int32_t j = 0; j < n_links; ++j) dual += bwd_caps[(int64_t)i * n_links + j];
    if (dual > DEFT_MAX_EXACT_CAPACITY) continue;
    const int64_t w = (dual + 1 + 31) >> 5;
    words = std::max(words, w);
    if (w <= smem_words_limit()) smem_words = std::max(smem_words, w);
  }
  const size_t b_vec = align_up((size_t)(n + 1) * 8, 256);
  const size_t b_caps = align_up((size_t)instances * n_links * 8, 256);
  const size_t b_stat = align_up((size_t)instances * 4, 256);
  const size_t b_used = align_up((size_t)instances * 8, 256);
  const size_t b_out = align_up((size_t)instances * out_stride * 4, 256);
  const size_t b_rows = align_up((size_t)instances * (n + 1) * words * 4, 256);
  const size_t b_reach = align_up((size_t)instances * (n + 1) * 4, 256);
  const size_t b_carry = align_up((size_t)instances * sizeof(SchedCarry), 256);
  const size_t in_bytes = 2 * b_vec + 2 * b_caps + b_stat + b_carry;
  const size_t dev_bytes = in_bytes + b_used + b_out + b_rows + b_reach + b_carry;
  deft_status_t st = grow(s, in_bytes + b_used + b_out + b_carry, dev_bytes);
  if (st != DEFT_OK) return st;
  char* h = s->pinned;
  int64_t* hc = reinterpret_cast<int64_t*>(h);
  int64_t* hb = reinterpret_cast<int64_t*>(h + b_vec);
  hc[0] = hb[0] = 0;
  memcpy(hc + 1, comm, (size_t)n * 8);
  memcpy(hb + 1, bwd, (size_t)n * 8);
  memcpy(h + 2 * b_vec, fwd_caps, (size_t)instances * n_links * 8);
  memcpy(h + 2 * b_vec + b_caps, bwd_caps, (size_t)instances * n_links * 8);
  memset(h + 2 * b_vec + 2 * b_caps, 0, (size_t)instances * 4);
  if (carry_in)
    memcpy(h + 2 * b_vec + 2 * b_caps + b_stat, carry_in, (size_t)instances * sizeof(SchedCarry));
  char* d = s->dev;
  DEFT_CUDA(cudaMemcpyAsync(d, h, in_bytes, cudaMemcpyHostToDevice, s->stream));
  SchedArgs A{};
  A.n = n;
  A.L = n_links;
  A.T = iterations;
  A.comm = reinterpret_cast<const int64_t*>(d);
  A.bwd = reinterpret_cast<const int64_t*>(d + b_vec);
  A.fcaps = reinterpret_cast<const int64_t*>(d + 2 * b_vec);
  A.bcaps = reinterpret_cast<const int64_t*>(d + 2 * b_vec + b_caps);
  A.status = reinterpret_cast<int32_t*>(d + 2 * b_vec + 2 * b_caps);
  A.used = reinterpret_cast<int64_t*>(d + in_bytes);
  A.out = reinterpret_cast<int32_t*>(d + in_bytes + b_used);
  A.out_stride = out_stride;
  A.rows = reinterpret_cast<uint32_t*>(d + in_bytes + b_used + b_out);
  A.words = words;
  A.reach = reinterpret_cast<int32_t*>(d + in_bytes + b_used + b_out + b_rows);
  A.smem_row_words = smem_words;
  A.t0 = t0;
  A.carry_in = carry_in ? reinterpret_cast<const SchedCarry*>(d + 2 * b_vec + 2 * b_caps + b_stat)
                        : nullptr;
  SchedCarry* d_carry_out =
      reinterpret_cast<SchedCarry*>(d + in_bytes + b_used + b_out + b_rows + b_reach);
  A.carry_out = carry_out ? d_carry_out : nullptr;
  DEFT_CUDA(cudaEventRecord(s->ev0, s->stream));
  cudaError_t e = launch_scheduler(A, instances, sched_smem_bytes(smem_words), s->stream);
  if (e != cudaSuccess) return cuda_fail(e, "deft_scheduler_kernel");
  DEFT_CUDA(cudaEventRecord(s->ev1, s->stream));
  // status + used + records back in one copy (they are contiguous)
  char* h_out = h + in_bytes;
  DEFT_CUDA(cudaMemcpyAsync(h + 2 * b_vec + 2 * b_caps, A.status, (size_t)instances * 4,
                            cudaMemcpyDeviceToHost, s->stream));
  DEFT_CUDA(cudaMemcpyAsync(h_out, A.used, b_used + b_out, cudaMemcpyDeviceToHost, s->stream));
  char* h_carry = h_out + b_used + b_out;
  if (carry_out)
    DEFT_CUDA(cudaMemcpyAsync(h_carry, d_carry_out, (size_t)instances * sizeof(SchedCarry),
                              cudaMemcpyDeviceToHost, s->stream));
  DEFT_CUDA(cudaStreamSynchronize(s->stream));
  if (carry_out) memcpy(carry_out, h_carry, (size_t)instances * sizeof(SchedCarry));
  cudaEventElapsedTime(&s->last_ms, s->ev0, s->ev1);
  memcpy(status, h + 2 * b_vec + 2 * b_caps, (size_t)instances * 4);
  memcpy(used, h_out, (size_t)instances * 8);
  for (int32_t i = 0; i < instances; ++i) {
    const int64_t u = std::min<int64_t>(used[i], out_stride);
    memcpy(out + (int64_t)i * out_stride, h_out + b_used + (size_t)i * out_stride * 4,
           (size_t)u * 4);
  }
  return DEFT_OK;
}

extern "C" deft_status_t deft_solver_schedule(deft_solver* s, int32_t instances, int32_t n,
                                              int32_t n_links, int32_t iterations,
                                              const int64_t* comm, const int64_t* bwd,
                                              const int64_t* fwd_caps,
                                              const int64_t* bwd_caps, int32_t* out,
                                              int64_t out_stride, int64_t* used,
                                              int32_t* status) {
  return deft_solver_schedule_chunk(s, instances, n, n_links, 0, iterations, comm, bwd, fwd_caps,
                                    bwd_caps, nullptr, nullptr, out, out_stride, used, status);
}
