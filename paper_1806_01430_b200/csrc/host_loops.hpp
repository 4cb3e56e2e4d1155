// host_loops.hpp -- the CPU side of a genome: loops whose gene bit is 0 run here, on the
// slot's pinned host arrays, exactly as the program writes them
// (/root/reference/proj/fixtures/matmul.c:8-32; same loop order, k ascending, separate
// multiply and add -- this translation unit is built with -ffp-contract=off).
#pragma once

#include <chrono>
#include <cstddef>

namespace mmx {

using Clock = std::chrono::steady_clock;

// Budget shared by every step of one benchmark run (ToolchainConfig::timeout_s).
struct Deadline {
  Clock::time_point at;
  bool early = false;  // mmx_config.early_timeout: give up as soon as measured progress shows the budget cannot be met
  bool expired() const { return Clock::now() >= at; }
  // `done` of `total` equal units of work took the time since `start`: is what remains hopeless -- at least twice the time left until
  // the deadline (plus 10 ms), judged only once 20 ms and 8 units have been measured?  The outcome of a run that is given up is the
  // one the full wait would produce (Timeout, time = the budget, evaluator.cpp:103-108); only its wall cost is smaller.
  bool hopeless(Clock::time_point start, long long done, long long total) const {
    if (!early || done < 8 || done >= total) return false;
    const Clock::time_point now = Clock::now();
    const double elapsed = std::chrono::duration<double>(now - start).count();
    if (elapsed < 0.020) return false;
    const double remaining = elapsed * static_cast<double>(total - done) / static_cast<double>(done);
    const double left = std::chrono::duration<double>(at - now).count();
    return remaining > 2.0 * (left > 0.0 ? left : 0.0) + 0.010;
  }
};

// The threads a CPU-mapped nest runs on: `threads` > 1 splits the outer loop into contiguous row blocks (per-element arithmetic is
// unchanged, so results do not depend on it); with `cpus` set, thread t pins itself to cpus[t % ncpus] -- the slot's own CPUs, so
// that concurrent measurements on other slots do not share cores with it.
struct HostTeam {
  int threads = 1;
  const int* cpus = nullptr;
  int ncpus = 0;
};

// Iterations [row0, row1) of the nest's outer loop (the whole nest is [0, n)): the executor runs a nest block by block when the
// array it writes is needed on the device next, so that finished rows cross the bus while the later ones are still being computed.
// Each returns false when the deadline passed before the block finished (rows are the unit of the check).
template <typename T> bool host_init_a(T* a, int n, int row0, int row1, const HostTeam& team, const Deadline& dl);
template <typename T> bool host_init_b(T* b, int n, int row0, int row1, const HostTeam& team, const Deadline& dl);
template <typename T> bool host_zero_c(T* c, int n, int row0, int row1, const HostTeam& team, const Deadline& dl);
template <typename T> bool host_transpose(T* bt, const T* b, int n, int row0, int row1, const HostTeam& team, const Deadline& dl);
template <typename T> bool host_matmul(T* c, const T* a, const T* bt, int n, int row0, int row1, const HostTeam& team, const Deadline& dl);
// matmul.c:30-32; the accumulator has the array's type, the result is widened for printf.
template <typename T> double host_trace(const T* c, int n);

// Pieces used when the host only drives an outer loop and the device runs the inner one
// are not needed here: in those modes the host loop body is just a kernel launch.

}  // namespace mmx
