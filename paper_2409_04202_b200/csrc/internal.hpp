// Shared internals of the C-ABI library (not part of the public header).
#pragma once

#include <atomic>
#include <cstdint>
#include <string>
#include <vector>

#include "planner.hpp"

struct gt_plan {
  gtar::Plan plan;
  std::vector<gtar::SwitchReport> reports;
  gtar::Topology topo;
  bool topo_params = true;     // built with per-link parameters from the document
  int dtype = 0;
  int esize = 4;
  std::string json;            // canonical plan JSON
  std::string report;          // GenTree report JSON
  uint64_t uid = 0;            // unique id (lowering cache key)
  bool is_allreduce = true;    // passed symbolic verification (gt_plan_from_json may load other plans)
};

struct ar_nvls;

namespace gtar {
void set_error(const std::string &msg);
// nvls.cu: in-switch AllReduce of `count` elements of the rank's NVLS buffer (throws)
void nvls_launch(ar_nvls *n, const void *dptr, uint64_t count, int32_t dtype, void *stream, int avg_n = 0);
uint64_t next_plan_uid();
inline int esize_of(int dtype) { return dtype == 0 ? 4 : 2; }
inline const char *dtype_name(int dtype) { return dtype == 0 ? "f32" : "bf16"; }
}  // namespace gtar
