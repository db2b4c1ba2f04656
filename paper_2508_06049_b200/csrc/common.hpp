// Shared host-side definitions of the klref-b200 library.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <exception>
#include <thread>
#include <vector>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace kb {

// Status codes of the C-ABI (include/klref_b200.h).  They mirror the
// exception hierarchy of the reference, proj/include/klref/errors.hpp:10-53.
enum Status : int {
  KB_OK = 0,
  KB_STRUCTURAL = 1,  // StructuralError
  KB_DOMAIN = 2,      // DomainError
  KB_SOLVER = 3,      // SolverError (carries last residual)
  KB_IO = 4,          // IoError
  KB_INTERNAL = 5,    // InternalError
  KB_RESOURCE = 6,    // ResourceError (carries level)
  KB_CUDA = 7,        // CUDA runtime failure (no reference counterpart)
};

struct Error : std::runtime_error {
  int code;
  double residual = 0.0;
  int level = -1;
  Error(int c, const std::string& what) : std::runtime_error(what), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& what) { throw Error(code, what); }

// Lattice helpers of the 2-d macro triangle, row-major in j
// (proj/include/klref/hhg.hpp:13-14).
inline int lattice_index(int n, int i, int j) { return j * (n + 1) - (j * (j - 1)) / 2 + i; }
inline int lattice_size(int n) { return (n + 1) * (n + 2) / 2; }

// fn(l) for l = lo..hi, one host thread per level (the levels' tables are
// independent); the first exception is rethrown on the caller's thread.
// KB_HOST_THREADS=0 runs them in order on the caller's thread.
template <typename F>
inline void parallel_levels(int lo, int hi, F fn) {
  static const bool serial = [] {
    const char* e = getenv("KB_HOST_THREADS");
    return e && e[0] == '0';
  }();
  if (serial || hi <= lo) {
    for (int l = lo; l <= hi; ++l) fn(l);
    return;
  }
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(static_cast<std::size_t>(hi - lo + 1));
  for (int l = hi; l >= lo; --l)  // largest level first
    th.emplace_back([&, l] {
      try {
        fn(l);
      } catch (...) {
        err[static_cast<std::size_t>(l - lo)] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

// fn(i) for i = 0..count-1 on up to 16 host threads (contiguous chunks); the
// first exception is rethrown on the caller's thread.  KB_HOST_THREADS=0 runs
// the loop on the caller's thread, as does worth_threads = false (small loops:
// spawning the threads costs more than they save).
template <typename F>
inline void parallel_for(int count, F fn, bool worth_threads = true) {
  static const int nthreads = [] {
    const char* e = getenv("KB_HOST_THREADS");
    if (e) return std::max(1, atoi(e));
    const unsigned hw = std::thread::hardware_concurrency();
    return static_cast<int>(std::min(16u, std::max(1u, hw)));
  }();
  const int T = worth_threads ? std::min(nthreads, count) : 1;
  if (T <= 1) {
    for (int i = 0; i < count; ++i) fn(i);
    return;
  }
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(static_cast<std::size_t>(T));
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      try {
        const int lo = static_cast<int>(static_cast<long long>(count) * t / T);
        const int hi = static_cast<int>(static_cast<long long>(count) * (t + 1) / T);
        for (int i = lo; i < hi; ++i) fn(i);
      } catch (...) {
        err[static_cast<std::size_t>(t)] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

}  // namespace kb

#define KB_CUDA_CHECK(expr)                                                              \
  do {                                                                                   \
    cudaError_t kb_err__ = (expr);                                                       \
    if (kb_err__ != cudaSuccess)                                                         \
      ::kb::fail(::kb::KB_CUDA, std::string(#expr) + ": " + cudaGetErrorString(kb_err__)); \
  } while (0)
