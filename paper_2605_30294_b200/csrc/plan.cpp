// plan.cpp -- host-side exchange planning from the count matrix (pure host
// code, usable without a GPU).  PAPER:124-128: send_offset/send_count per
// destination, recv_count via the all-to-all, recv_offset via prefix sums.
#include <cstdint>

#include "rafi.h"

extern "C" int rafi_plan(int R, const uint64_t* C, uint64_t capacity, int d, uint64_t* recv_count,
                         uint64_t* recv_off, uint64_t* src_off, uint64_t* total, uint64_t* G, int* overflow) {
  if (R < 1 || !C || d < 0 || d >= R) return RAFI_ERR_INVALID_ARG;
  uint64_t tot = 0;
  for (int s = 0; s < R; ++s) {
    const uint64_t c = C[(uint64_t)s * R + d];
    if (recv_count) recv_count[s] = c;
    if (recv_off) recv_off[s] = tot;  // exclusive prefix over sources
    tot += c;
    if (src_off) {                    // exclusive prefix over destinations of row s
      uint64_t o = 0;
      for (int e = 0; e < d; ++e) o += C[(uint64_t)s * R + e];
      src_off[s] = o;
    }
  }
  if (total) *total = tot;
  uint64_t g = 0;
  int ovf = 0;
  for (int e = 0; e < R; ++e) {
    uint64_t col = 0;
    for (int s = 0; s < R; ++s) col += C[(uint64_t)s * R + e];
    g += col;
    if (col > capacity) ovf = 1;
  }
  if (G) *G = g;
  if (overflow) *overflow = ovf;
  return RAFI_OK;
}
