// Thread-local error state shared by every translation unit of libhm_page.
#pragma once
#include <cstdint>

#include "../../include/hm_page.h"

int hm_set_error(int code, const char* fmt, ...);
void hm_set_alloc_bytes(int64_t requested, int64_t available);

// Null device/descriptor pointer with work to do: HM_ERR_INVALID instead of a
// kernel fault (which would poison the CUDA context).
#define HM_REQUIRE_PTRS(who, ...)                                                   \
  do {                                                                              \
    const void* hm_ptrs_[] = {__VA_ARGS__};                                         \
    for (const void* hm_p_ : hm_ptrs_)                                              \
      if (!hm_p_) return hm_set_error(HM_ERR_INVALID, "%s: null pointer argument", who); \
  } while (0)
