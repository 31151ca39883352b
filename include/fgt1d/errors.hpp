#pragma once
// Error taxonomy of the fgt1d API (same classes as the reference,
// proj/include/fgt1d/errors.hpp:8-15): std::domain_error for bad arguments
// (delta, non-finite coordinates), std::invalid_argument for structural
// problems (sizes, SOE, plan kind), fgt::numerical_error for algorithmic
// failures.  Device failures surface as fgt::device_error.
#include <stdexcept>
#include <string>

namespace fgt {

class numerical_error : public std::runtime_error {
 public:
  explicit numerical_error(const std::string& what) : std::runtime_error(what) {}
};

// No usable CUDA device or a CUDA failure (there is no CPU fallback).
class device_error : public std::runtime_error {
 public:
  explicit device_error(const std::string& what) : std::runtime_error(what) {}
};

}  // namespace fgt
