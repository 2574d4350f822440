// device_once.cuh — kernel attributes (e.g. the dynamic shared-memory
// opt-in) belong to a device's context, so one process driving several GPUs
// (the C++ API's DREAMSCHED_GPUS) must set them once per DEVICE, not once
// per process.
#pragma once

#include <cuda_runtime.h>

#include <atomic>

namespace dsx {

template <typename F>
void once_per_device(std::atomic<unsigned long long>& done, F&& f) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  f();  // idempotent: two threads on the same device may both run it
  done.fetch_or(bit, std::memory_order_acq_rel);
}

}  // namespace dsx
