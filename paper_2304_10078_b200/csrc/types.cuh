// Device-side descriptors shared by the level-synchronous scheduler and its
// kernels.  One "node" is one call of the reference's _SortRun.node /
// _AggRun.node (core.py:447-498, aggregate.py:133-170) that is large enough
// to bucket; one "work item" is one subarray (row of the counting matrix).
#pragma once

#include <cstdint>

namespace ss {

struct Params {              // mirrors TuningParams (params.py:38-47)
  uint64_t input_size;
  uint32_t light_buckets;
  uint32_t light_bits;
  uint64_t subarray_len;
  uint64_t base_case_cutoff;
  uint32_t max_heavy;
  uint32_t sample_factor;
  uint64_t seed;
  uint64_t sample_count;
  uint64_t heavy_threshold_int;  // ceil(heavy_threshold): count >= float(log2 n)
  double heavy_threshold;
};

struct Node {
  uint64_t lo;          // start in the level's source buffer
  uint64_t size;
  uint64_t path;        // per-node sample-stream path (core.py:466, 498)
  uint64_t out_base;    // where the node's buckets start in the destination
  uint64_t row_base;    // first counting-matrix row
  uint64_t parent_size; // for telemetry / valve bookkeeping
  uint32_t n_rows;
  uint32_t depth;       // effective depth after the safety valve
  uint32_t stalled;
  uint32_t n_heavy;     // written by the sampling kernel
  uint32_t grp_base;    // first row group (scan kernels)
  uint32_t n_grps;
};

struct Work {            // one subarray of one node
  uint64_t begin;        // absolute index in the source buffer
  uint32_t len;
  uint32_t node;
  uint64_t row;          // counting-matrix row
};

struct Leaf {
  uint64_t lo;
  uint64_t size;
};

constexpr int kRowGroup = 8;   // rows per scan group

}  // namespace ss
