// Streams and hardware work queues (loopback worlds).
//
// Streams are multiplexed onto a small number of hardware work queues
// (CUDA_DEVICE_MAX_CONNECTIONS).  Two streams that share a queue are not
// independent: work of stream B issued after a blocked entry of stream A waits
// for it.  A loopback world (W ranks on one GPU, loopback.py) must give every
// rank its own queue, because rank r's barrier kernels wait for kernels of the
// other ranks that the host issues LATER.  The mapping of streams to queues is
// not specified, so it is measured: deft_stream_alias_probe() launches on A a
// kernel that spins on a flag (bounded), then a no-op kernel (mode 0) or a
// device-to-device copy (mode 1, the copy-engine channel's operation) on A --
// it depends on the spin: same stream --, then on B the kernel that sets the
// flag.  If B's work sits behind A's blocked entry the spin times out.
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/deft_b200.h"
#include "common.cuh"

namespace {
__device__ __forceinline__ uint64_t probe_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void probe_spin(volatile uint32_t* flag, uint32_t* timed_out, uint64_t limit_ns) {
  const uint64_t t0 = probe_ns();
  while (*flag == 0u) {
    if (probe_ns() - t0 > limit_ns) {
      *timed_out = 1u;
      return;
    }
  }
  *timed_out = 0u;
}
__global__ void probe_nop() {}
__global__ void probe_set(volatile uint32_t* flag) { *flag = 1u; }
}  // namespace

deft_status_t deft_fail_cuda(cudaError_t e, const char* where);

extern "C" deft_status_t deft_stream_create(int32_t priority, void** out) {
  if (!out) return deft_fail_cuda(cudaErrorInvalidValue, "deft_stream_create: null out");
  cudaStream_t s = nullptr;
  cudaError_t e = cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority);
  if (e != cudaSuccess) return deft_fail_cuda(e, "cudaStreamCreateWithPriority");
  *out = s;
  return DEFT_OK;
}

extern "C" deft_status_t deft_stream_destroy(void* stream) {
  cudaError_t e = cudaStreamDestroy((cudaStream_t)stream);
  if (e != cudaSuccess) return deft_fail_cuda(e, "cudaStreamDestroy");
  return DEFT_OK;
}

extern "C" deft_status_t deft_stream_alias_probe(void* stream_a, void* stream_b,
                                                 int32_t timeout_us, int32_t mode,
                                                 int32_t* aliased) {
  static thread_local uint32_t* scratch = nullptr;  // [flag, timed_out, copy src/dst ...]
  cudaError_t e = cudaSuccess;
  if (!scratch) {
    e = cudaMalloc(&scratch, 1 << 20);
    if (e != cudaSuccess) return deft_fail_cuda(e, "deft_stream_alias_probe: cudaMalloc");
  }
  cudaStream_t a = (cudaStream_t)stream_a, b = (cudaStream_t)stream_b;
  if ((e = cudaStreamSynchronize(a)) != cudaSuccess ||
      (e = cudaStreamSynchronize(b)) != cudaSuccess ||
      (e = cudaMemset(scratch, 0, 2 * sizeof(uint32_t))) != cudaSuccess ||
      (e = cudaDeviceSynchronize()) != cudaSuccess)
    return deft_fail_cuda(e, "deft_stream_alias_probe: setup");
  probe_spin<<<1, 1, 0, a>>>(scratch, scratch + 1, (uint64_t)timeout_us * 1000ull);
  if (mode == 0) {
    probe_nop<<<1, 1, 0, a>>>();
  } else {  // a copy-engine copy queued behind the spin
    char* base = reinterpret_cast<char*>(scratch);
    e = cudaMemcpyAsync(base + (512 << 10), base + 4096, 64 << 10, cudaMemcpyDeviceToDevice, a);
    if (e != cudaSuccess) return deft_fail_cuda(e, "deft_stream_alias_probe: copy");
  }
  probe_set<<<1, 1, 0, b>>>(scratch);
  if ((e = cudaGetLastError()) != cudaSuccess ||
      (e = cudaStreamSynchronize(a)) != cudaSuccess ||
      (e = cudaStreamSynchronize(b)) != cudaSuccess)
    return deft_fail_cuda(e, "deft_stream_alias_probe: run");
  uint32_t h = 0;
  if ((e = cudaMemcpy(&h, scratch + 1, sizeof(h), cudaMemcpyDeviceToHost)) != cudaSuccess)
    return deft_fail_cuda(e, "deft_stream_alias_probe: read");
  *aliased = h ? 1 : 0;
  return DEFT_OK;
}
