// Status -> exception mapping for the C++ drop-in (the reference throws
// std::invalid_argument / std::runtime_error / std::bad_alloc).
#pragma once

#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "curvalign/geometry.hpp"
#include "curvalign_cuda.h"

namespace curvalign::detail {

inline void check(int status, const char* (*msg)() = cva_last_error) {
  if (status == CVA_OK) return;
  const std::string m = msg ? msg() : "";
  switch (status) {
    case CVA_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case CVA_BAD_ALLOC: throw std::bad_alloc();
    case CVA_RUNTIME_ERROR: throw std::runtime_error(m);
    default: throw std::runtime_error("curvalign (CUDA): " + m);
  }
}

inline void check_dropin(int status) { check(status, cva_dropin_last_error); }

inline const double* raw(const Point2* p) { return reinterpret_cast<const double*>(p); }
inline double* raw(Point2* p) { return reinterpret_cast<double*>(p); }

}  // namespace curvalign::detail
