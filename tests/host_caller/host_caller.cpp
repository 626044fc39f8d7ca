// A plain C++ host of libnexus_b200.so: the INTEGRATION.md §2 caller, compiled
// and run by tests/test_abi.py (CPU, virtual clock) and tests/test_gpu_host_caller.py
// (B200, device clock). No Python, no ctypes: this is what a reference-side
// C++ program (the nexussim CLI's run_engines, tools/main.cpp:217) links.
//
//   host_caller <calib file> <preset> <rate> <count> <seed> [--device]
//
// Prints the event log (reference serialize_event_log bytes) to stdout, then
// "# tokens <id> <n>" lines when a device is bound.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "nexus_b200.h"

static void fail(const char* what, const char* msg) {
  std::fprintf(stderr, "host_caller: %s: %s\n", what, msg ? msg : "");
  std::exit(2);
}

int main(int argc, char** argv) {
  if (argc < 6) fail("usage", "host_caller <calib> <preset> <rate> <count> <seed> [--device]");
  const bool use_device = argc > 6 && std::strcmp(argv[6], "--device") == 0;
  std::ifstream f(argv[1]);
  if (!f) fail("open", argv[1]);
  std::stringstream ss;
  ss << f.rdbuf();

  nx_sim_config cfg{};
  cfg.model = nx_model_derive(256, 1024, 2, 4, 2);  // BASELINE configs[0] (C1)
  cfg.gpu.total_sm = 64;                             // presets.cpp "desk"
  cfg.gpu.peak_compute = 2.0e12;
  cfg.gpu.peak_bandwidth = 1.0e11;
  cfg.gpu.kv_capacity_bytes = int64_t{4} << 30;
  cfg.ctrl = nx_controller_config_default();
  char warn[1024];
  if (nx_kernel_profile_from_text(ss.str().c_str(), &cfg.profile, warn, sizeof(warn)) != NX_OK)
    fail("calibration", nx_last_error());
  cfg.engine = nx_engine_config_default();
  cfg.engine.clock_mode = use_device ? NX_CLOCK_DEVICE : NX_CLOCK_VIRTUAL;

  std::vector<nx_request> trace(static_cast<size_t>(std::atoll(argv[4])));
  size_t n = 0;
  if (nx_workload_preset_trace(argv[2], std::atof(argv[3]), static_cast<int64_t>(trace.size()),
                               std::strtoull(argv[5], nullptr, 10), trace.data(), trace.size(), &n) != NX_OK)
    fail("trace", nx_last_error());
  trace.resize(n);

  nx_device* dev = nullptr;
  if (use_device) {
    for (auto& r : trace) {  // keep the tiny model's run short
      if (r.prompt_len > 300) r.prompt_len = 300;
      if (r.output_len > 8) r.output_len = 8;
    }
    nx_device_config dc{};
    dc.arch = {256, 2, 2, 2, 128, 1024, 1024, 0, 10000.f, 1e-5f};  // device.py "tiny"
    dc.page_tokens = 16;
    dc.num_pages = 512;
    dc.max_prefill_tokens = 2048 + 64;
    dc.max_decode_batch = 64;
    dc.green_contexts = 1;
    dc.weight_seed = 3;
    dc.weight_gain = 1.f;
    dc.lm_head_gain = 4.f;
    dc.tp_size = 1;
    if (nx_device_create(&dc, &dev) != NX_OK) fail("device", nx_last_error());
  }

  nx_engine* eng = nullptr;
  if (nx_engine_create(&cfg, &eng) != NX_OK) fail("engine", nx_last_error());
  if (dev && nx_engine_bind_device(eng, dev) != NX_OK) fail("bind", nx_engine_last_error(eng));
  if (nx_submit_trace(eng, trace.data(), trace.size()) != NX_OK) fail("submit", nx_engine_last_error(eng));
  if (nx_run(eng) != NX_OK) fail("run", nx_engine_last_error(eng));

  size_t len = 0;
  nx_engine_event_log(eng, nullptr, 0, &len);
  std::string log(len + 1, '\0');
  nx_engine_event_log(eng, log.data(), log.size(), &len);
  log.resize(len);
  std::fwrite(log.data(), 1, log.size(), stdout);
  if (dev) {
    for (const auto& r : trace) {
      size_t nt = 0;
      nx_engine_tokens(eng, r.id, nullptr, 0, &nt);
      std::printf("# tokens %llu %zu\n", static_cast<unsigned long long>(r.id), nt);
    }
  }
  nx_engine_destroy(eng);
  if (dev) nx_device_destroy(dev);
  return 0;
}
