// Maps gimbal_gpu.h status codes back to the exceptions the reference API throws.
#pragma once

#include <stdexcept>
#include <string>

#include "gimbal_gpu.h"

namespace gimbal::gpu_shim {

inline void check(int status, const char* what) {
  if (status == GIMBAL_OK) return;
  const std::string msg = gimbal_last_error();
  switch (status) {
    case GIMBAL_INVALID_ARGUMENT:
      throw std::invalid_argument(msg.empty() ? std::string(what) : msg);
    case GIMBAL_OUT_OF_RANGE:
      throw std::out_of_range(msg.empty() ? std::string(what) : msg);
    case GIMBAL_OVERFLOW:
      throw std::overflow_error(msg.empty() ? std::string(what) : msg);
    default:
      throw std::runtime_error(std::string(what) + ": " + msg);
  }
}

// Device the shim's handles live on (GIMBAL_DEVICE, default 0).
int shim_device();

}  // namespace gimbal::gpu_shim
