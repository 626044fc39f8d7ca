// Shared between the host C-ABI (capi.cpp) and the device C-ABI
// (device/capi_device.cu): the opaque handle behind nx_engine*.
#pragma once

#include <string>

#include "engine.hpp"

struct nx_engine {
  explicit nx_engine(const nx_sim_config& cfg) : e(cfg) {}
  nxb::Engine e;
  std::string err;
};

namespace nxb {
// Thread-local last-error string shared by both ABI halves.
std::string& last_error();
}  // namespace nxb
