// Error reporting and the growable device workspace shared by the ABI files.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/ltsgpu.h"

namespace ltsg {

void set_error(const char* fmt, ...);

struct Status {
  int code = LTSG_OK;
};

#define LTSG_CUDA(expr)                                                                     \
  do {                                                                                      \
    cudaError_t err_ = (expr);                                                              \
    if (err_ != cudaSuccess) {                                                              \
      ::ltsg::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(err_)); \
      return LTSG_ECUDA;                                                                    \
    }                                                                                       \
  } while (0)

#define LTSG_CHECK_LAUNCH() LTSG_CUDA(cudaGetLastError())

#define LTSG_TRY(expr)          \
  do {                          \
    int rc_ = (expr);           \
    if (rc_ != LTSG_OK) return rc_; \
  } while (0)

inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 2147483647LL) g = 2147483647LL;
  return (int)g;
}

}  // namespace ltsg

// Named growable buffers.  Growing frees the old buffer (cudaFree
// synchronises), so callers only grow between kernels whose inputs they do
// not need to keep.
struct ltsg_workspace {
  struct Buf {
    void* ptr = nullptr;
    size_t bytes = 0;
  };
  std::unordered_map<std::string, Buf> bufs;
  size_t total = 0;
  size_t budget = 0;
  int device = 0;
  // sizes seen by earlier calls: the async traversal preallocates from them
  size_t hint_front = 0, hint_rest = 0, hint_entries = 0, hint_cross = 0, hint_seed = 0;
  size_t hint_mrows = 0;  // moving path: most surviving rows of one generation
  size_t hint_bp_cand = 0;  // broad phase: most Check-1 candidates seen
  int hint_gens = 0;  // deepest traversal seen: async mode launches one generation more

  int get(const char* name, size_t bytes, void** out, bool keep = false);
  // CUDA events for per-kernel timing, created on first use and reused
  std::vector<cudaEvent_t> events;
  cudaEvent_t event(size_t i) {
    while (events.size() <= i) {
      cudaEvent_t e = nullptr;
      cudaEventCreate(&e);
      events.push_back(e);
    }
    return events[i];
  }
  ~ltsg_workspace();
};
