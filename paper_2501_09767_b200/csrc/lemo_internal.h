// Internal helpers shared by the liblemo translation units.
#pragma once

#include <cuda_runtime.h>

#define LEMO_ABI_VERSION 1

namespace lemo {
void set_error(const char* where, int code);
void set_error_msg(const char* msg);
const char* last_error();
}  // namespace lemo

// Every C-ABI entry point returns 0 on success and a nonzero code (with a
// message retrievable through lemo_last_error()) on failure.
#define LEMO_CHECK_LAUNCH(where)                 \
  do {                                           \
    cudaError_t _e = cudaGetLastError();         \
    if (_e != cudaSuccess) {                     \
      lemo::set_error(where, (int)_e);           \
      return (int)_e;                            \
    }                                            \
  } while (0)

// Code returned by helpers that already recorded a message.
#define LEMO_ERR_REPORTED 1000

#define LEMO_RETURN_RC(where, rc)                                      \
  do {                                                                 \
    int _rc = (rc);                                                    \
    if (_rc) {                                                         \
      if (_rc != LEMO_ERR_REPORTED) lemo::set_error(where, _rc);       \
      return _rc;                                                      \
    }                                                                  \
    return 0;                                                          \
  } while (0)

#define LEMO_ARG_CHECK(cond, msg)      \
  do {                                 \
    if (!(cond)) {                     \
      lemo::set_error_msg(msg);        \
      return LEMO_ERR_REPORTED;         \
    }                                  \
  } while (0)
