// Host-side types shared by host.cpp and engine.cu.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/slablu_gpu.h"

namespace slb {

struct HostError : std::runtime_error {
  int code;
  int64_t index;
  double residual = 0.0;  // CompressionError::residual_estimate (common.hpp:55-60)
  HostError(int c, const std::string& m, int64_t i = -1) : std::runtime_error(m), code(c), index(i) {}
};

// splitmix64 step (common.hpp:64-69): per-task seeds from the one user seed.
inline uint64_t mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// CompressionError (residual estimate) or, for invalid options, ConfigError.
inline HostError HbsError(const std::string& m, double residual, bool config, int64_t block = -1) {
  HostError e(config ? SLABLU_ERR_CONFIG : SLABLU_ERR_COMPRESSION, m, block);
  e.residual = residual;
  return e;
}

struct GridStrip {
  int64_t first_col, width;
};
struct Partition {
  int64_t n1 = 0, n2 = 0, b = 0;
  std::vector<GridStrip> interfaces, interiors;
};

slablu_gpu_status make_status(int code, const std::string& msg, int64_t index, double residual = 0.0);
int64_t choose_b(int64_t n1, int64_t n2, int64_t b, double c);
Partition partition(int64_t n1, int64_t n2, int64_t b);
double bessel_j0(double t);

}  // namespace slb
