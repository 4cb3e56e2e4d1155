#include "host_loops.hpp"

#include <pthread.h>
#include <sched.h>

#include <atomic>
#include <thread>
#include <vector>

namespace mmx {

namespace {

// Run body(i) for i in [0, n) on `threads` workers over contiguous blocks; stop early once
// the deadline passes.  The deadline is polled once per row (every 16 rows for cheap nests
// would be enough, but a row is never shorter than the clock read by much at the sizes
// where it matters).
void pin_self(int cpu) {
  cpu_set_t set;
  CPU_ZERO(&set);
  CPU_SET(cpu, &set);
  pthread_setaffinity_np(pthread_self(), sizeof(set), &set);  // best effort: an unpinned thread is slower, not wrong
}

template <typename Body>
bool for_rows(int row0, int row1, const HostTeam& team, const Deadline& dl, int poll_every, Body body) {
  const int n = row1 - row0;
  if (n <= 0) return !dl.expired();
  int threads = team.threads;
  if (threads < 1) threads = 1;
  if (threads > n) threads = n;
  std::atomic<bool> expired{false};
  auto block = [&](int r0, int r1) {
    const Clock::time_point started = Clock::now();
    for (int i = r0; i < r1; ++i) {
      // every thread projects its own block (the rows of a nest cost the same): one hopeless block makes the nest hopeless
      if ((i - r0) % poll_every == 0 &&
          (expired.load(std::memory_order_relaxed) || dl.expired() || dl.hopeless(started, i - r0, r1 - r0))) {
        expired.store(true, std::memory_order_relaxed);
        return;
      }
      body(i);
    }
  };
  if (threads == 1) {
    block(row0, row1);
  } else {
    std::vector<std::thread> pool;
    pool.reserve(threads);
    for (int t = 0; t < threads; ++t) {
      const int r0 = row0 + static_cast<int>(static_cast<long long>(n) * t / threads);
      const int r1 = row0 + static_cast<int>(static_cast<long long>(n) * (t + 1) / threads);
      pool.emplace_back([&, t, r0, r1] {
        if (team.cpus != nullptr && team.ncpus > 0) pin_self(team.cpus[t % team.ncpus]);
        block(r0, r1);
      });
    }
    for (auto& th : pool) th.join();
  }
  return !expired.load();
}

}  // namespace

template <typename T>
bool host_init_a(T* a, int n, int row0, int row1, const HostTeam& team, const Deadline& dl) {
  return for_rows(row0, row1, team, dl, 64, [=](int i) {
    T* row = a + static_cast<std::size_t>(i) * n;
    for (int j = 0; j < n; ++j) row[j] = static_cast<T>(i + j) / n;  // matmul.c:10
  });
}

template <typename T>
bool host_init_b(T* b, int n, int row0, int row1, const HostTeam& team, const Deadline& dl) {
  return for_rows(row0, row1, team, dl, 64, [=](int i) {
    T* row = b + static_cast<std::size_t>(i) * n;
    for (int j = 0; j < n; ++j) row[j] = static_cast<T>(i - j) / n;  // matmul.c:14
  });
}

template <typename T>
bool host_zero_c(T* c, int n, int row0, int row1, const HostTeam& team, const Deadline& dl) {
  return for_rows(row0, row1, team, dl, 64, [=](int i) {
    T* row = c + static_cast<std::size_t>(i) * n;
    for (int j = 0; j < n; ++j) row[j] = static_cast<T>(0.0);  // matmul.c:18
  });
}

template <typename T>
bool host_transpose(T* bt, const T* b, int n, int row0, int row1, const HostTeam& team, const Deadline& dl) {
  return for_rows(row0, row1, team, dl, 16, [=](int i) {
    T* row = bt + static_cast<std::size_t>(i) * n;
    for (int j = 0; j < n; ++j) row[j] = b[static_cast<std::size_t>(j) * n + i];  // matmul.c:23
  });
}

template <typename T>
bool host_matmul(T* c, const T* a, const T* bt, int n, int row0, int row1, const HostTeam& team, const Deadline& dl) {
  return for_rows(row0, row1, team, dl, 1, [=](int i) {
    T* crow = c + static_cast<std::size_t>(i) * n;
    const T* arow = a + static_cast<std::size_t>(i) * n;
    for (int j = 0; j < n; ++j) {
      const T* brow = bt + static_cast<std::size_t>(j) * n;
      for (int k = 0; k < n; ++k) crow[j] += arow[k] * brow[k];  // matmul.c:28
    }
  });
}

template <typename T>
double host_trace(const T* c, int n) {
  T sum = static_cast<T>(0.0);
  for (int i = 0; i < n; ++i) sum += c[static_cast<std::size_t>(i) * n + i];  // matmul.c:32
  return static_cast<double>(sum);
}

#define MMX_INSTANTIATE(T)                                                           \
  template bool host_init_a<T>(T*, int, int, int, const HostTeam&, const Deadline&);                      \
  template bool host_init_b<T>(T*, int, int, int, const HostTeam&, const Deadline&);                      \
  template bool host_zero_c<T>(T*, int, int, int, const HostTeam&, const Deadline&);                      \
  template bool host_transpose<T>(T*, const T*, int, int, int, const HostTeam&, const Deadline&);         \
  template bool host_matmul<T>(T*, const T*, const T*, int, int, int, const HostTeam&, const Deadline&);  \
  template double host_trace<T>(const T*, int);
MMX_INSTANTIATE(double)
MMX_INSTANTIATE(float)

}  // namespace mmx
