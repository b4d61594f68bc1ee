// ad2_launch.cuh — host-side helpers shared by the kernel launchers.
#pragma once
#include <cuda_runtime.h>

#include <atomic>

namespace ad2k {

// One-time per-device set-up (cudaFuncSetAttribute is a per-device setting): first() is true on a
// device until done() has been called there.  Setting an attribute twice is harmless, so two
// threads racing on first() only repeat idempotent work.
struct PerDevice {
  std::atomic<unsigned long long> mask{0};
  static unsigned long long bit() {
    int dev = 0;
    cudaGetDevice(&dev);
    return 1ull << (dev & 63);
  }
  bool first() const { return (mask.load(std::memory_order_acquire) & bit()) == 0; }
  void done() { mask.fetch_or(bit(), std::memory_order_release); }
};

// A per-device cached integer (0 = not yet computed), e.g. a resident-grid size.
struct PerDeviceInt {
  std::atomic<int> v[64] = {};
  static int dev() {
    int d = 0;
    cudaGetDevice(&d);
    return d & 63;
  }
  int get() const { return v[dev()].load(std::memory_order_relaxed); }
  void set(int x) { v[dev()].store(x, std::memory_order_relaxed); }
};

}  // namespace ad2k
