// Shared C-ABI plumbing: exception -> status mapping with the thread-local
// last error (ss_last_error), stream and telemetry helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <exception>
#include <string>

#include "engine.cuh"

namespace ss {

extern thread_local std::string g_last_error;   // defined in capi.cu

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return SS_OK;
  } catch (const Fail& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SS_ERR_RESOURCE;
  } catch (...) {
    g_last_error = "unknown error";
    return SS_ERR_RESOURCE;
  }
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

inline void reset_tel(ss_telemetry* t) {
  if (!t) return;
  int32_t timing = t->timing;
  std::memset(t, 0, sizeof(*t));
  t->timing = timing;
}

}  // namespace ss
