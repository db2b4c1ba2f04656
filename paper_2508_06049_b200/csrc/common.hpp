// Shared host-side definitions of the klref-b200 library.
#pragma once

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

}  // namespace kb

#define KB_CUDA_CHECK(expr)                                                              \
  do {                                                                                   \
    cudaError_t kb_err__ = (expr);                                                       \
    if (kb_err__ != cudaSuccess)                                                         \
      ::kb::fail(::kb::KB_CUDA, std::string(#expr) + ": " + cudaGetErrorString(kb_err__)); \
  } while (0)
