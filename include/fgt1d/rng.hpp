#pragma once
// Counter-based RNG of the reference (proj/include/fgt1d/rng.hpp:6-39).
#include <cstdint>
#include <vector>

namespace fgt::rng {

std::uint64_t mix64(std::uint64_t z);
std::uint64_t counter_rand(std::uint64_t seed, std::uint64_t stream, std::uint64_t i);
double uniform01(std::uint64_t seed, std::uint64_t stream, std::uint64_t i);

inline constexpr std::uint64_t kStreamSources = 0;
inline constexpr std::uint64_t kStreamStrengths = 1;
inline constexpr std::uint64_t kStreamEvalIndices = 2;
inline constexpr std::uint64_t kStreamTargets = 3;

std::vector<double> uniform_points(std::size_t count, std::uint64_t seed, std::uint64_t stream);
std::vector<double> chebyshev_points(std::size_t count);

}  // namespace fgt::rng
