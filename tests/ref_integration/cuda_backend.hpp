// cuda_backend.hpp -- the reference-side binding of libmmx (INTEGRATION.md section 2 lists this file verbatim).
//
// A maintainer of the reference adds this as include/acctune/cuda_backend.hpp and links with -lmmx.  It is compiled
// here (oracle/Makefile: `make ref`) against the UNMODIFIED reference headers and libacctune_core.a, so that the
// reference's own Evaluator (src/evaluator.cpp:144-292) and run_ga (src/ga.cpp:247-295) drive the CUDA path in
// tests/test_ref_dropin.py.  Test infrastructure: nothing in the product includes it.
#pragma once

#include <condition_variable>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "acctune/errors.hpp"
#include "acctune/evaluator.hpp"
#include "mmx.h"

namespace acctune {

struct CudaConfig {  // config block "cuda": { "n": 4096, "dtype": "f64", "devices": [0,1,...], ... }
  int n = 256;
  int dtype = MMX_F64;
  int numerics = MMX_NUMERICS_FAST;
  double timeout_s = 120.0;
  int repetitions = 1;
  int matmul_variant = 0;
  std::vector<int> devices = {0};  // one device slot per entry; `jobs` = devices.size()
};

class CudaBackend : public EvalBackend {
 public:
  explicit CudaBackend(const CudaConfig& cfg) {
    mmx_config c;
    mmx_default_config(&c);
    c.n = cfg.n;
    c.dtype = cfg.dtype;
    c.numerics = cfg.numerics;
    c.timeout_s = cfg.timeout_s;
    c.repetitions = cfg.repetitions;
    c.matmul_variant = cfg.matmul_variant;
    c.num_slots = static_cast<int>(cfg.devices.size());
    c.devices = cfg.devices.data();
    if (int rc = mmx_create(&c, &ctx_); rc != MMX_OK) raise(rc, mmx_last_error(nullptr));
    free_slots_.resize(cfg.devices.size());
    std::iota(free_slots_.begin(), free_slots_.end(), 0);
  }
  ~CudaBackend() override { mmx_destroy(ctx_); }
  CudaBackend(const CudaBackend&) = delete;
  CudaBackend& operator=(const CudaBackend&) = delete;

  std::size_t gene_length() const override { return mmx_gene_length(ctx_); }

  // called concurrently from up to `jobs` threads (evaluator.cpp:196-205): each call borrows a device slot
  EvaluationOutcome measure(const Genome& genome) override {
    const int slot = take_slot();
    mmx_outcome o{};
    const int rc = mmx_measure(ctx_, slot, genome.bits().data(), genome.size(), &o);
    const std::string why = rc != MMX_OK ? mmx_last_error(ctx_) : "";
    give_slot(slot);
    if (rc != MMX_OK) raise(rc, why.c_str());
    return EvaluationOutcome{static_cast<EvalStatus>(o.status), o.time_s, o.wall_cost_s};
  }

 private:
  [[noreturn]] static void raise(int rc, const char* msg) {
    switch (rc) {
      case MMX_E_LENGTH: throw GenomeLengthMismatch(msg);
      case MMX_E_NODEVICE: throw ToolchainMissing(msg);
      case MMX_E_INVALID: throw ConfigError(msg);
      case MMX_E_NOMEM: throw WorkdirUnwritable(msg);
      default: throw Error(msg);
    }
  }
  int take_slot() {
    std::unique_lock<std::mutex> lock(mu_);
    cv_.wait(lock, [&] { return !free_slots_.empty(); });
    const int slot = free_slots_.back();
    free_slots_.pop_back();
    return slot;
  }
  void give_slot(int slot) {
    {
      std::lock_guard<std::mutex> lock(mu_);
      free_slots_.push_back(slot);
    }
    cv_.notify_one();
  }

  mmx_ctx* ctx_ = nullptr;
  std::vector<int> free_slots_;
  std::mutex mu_;
  std::condition_variable cv_;
};

}  // namespace acctune
