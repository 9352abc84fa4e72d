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
  HostError(int c, const std::string& m, int64_t i = -1) : std::runtime_error(m), code(c), index(i) {}
};

struct GridStrip {
  int64_t first_col, width;
};
struct Partition {
  int64_t n1 = 0, n2 = 0, b = 0;
  std::vector<GridStrip> interfaces, interiors;
};

slablu_gpu_status make_status(int code, const std::string& msg, int64_t index);
int64_t choose_b(int64_t n1, int64_t n2, int64_t b, double c);
Partition partition(int64_t n1, int64_t n2, int64_t b);
double bessel_j0(double t);

}  // namespace slb
