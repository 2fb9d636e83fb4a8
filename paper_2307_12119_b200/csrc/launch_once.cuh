// launch_once.cuh — one-time kernel setup (dynamic shared-memory attributes, occupancy),
// per device and thread-safe. cudaFuncSetAttribute acts on the current device's context,
// so a process that drives several devices runs the setup once on each; a concurrent first
// call on the same device waits for the thread doing it. The occupancy numbers it records
// are the same on every device of a node (one sm_100a part).
#pragma once
#include <cuda_runtime.h>

#include <mutex>

namespace gtb {

class DeviceOnce {
  public:
    template <typename F>
    void operator()(F&& setup) {
        int d = 0;
        cudaGetDevice(&d);
        const unsigned long long bit = 1ull << (d & 63);
        std::lock_guard<std::mutex> lk(mu_);
        if (done_ & bit) return;
        setup();
        done_ |= bit;
    }

  private:
    std::mutex mu_;
    unsigned long long done_ = 0;
};

}  // namespace gtb
