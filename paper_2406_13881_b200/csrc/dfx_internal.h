// dfx_internal.h -- shared declarations between the C-ABI layer and kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/dfx.h"

namespace dfx {

struct ReplayDev {
  const dfx_fn_desc* fns;
  const int32_t* ops;
  const int32_t* var_flags;
  const int32_t* stmt_span;
  const int32_t* sites;
  const int32_t* arms;
  const int32_t* item_fn;
  const int32_t* item_chunk;
  int n_items;
  int max_slots;
  dfx_event* events;
  int64_t event_cap;
  unsigned long long* event_count;
  uint8_t* var_out;
};

int replay_launch(const ReplayDev& r, cudaStream_t stream);

}  // namespace dfx
