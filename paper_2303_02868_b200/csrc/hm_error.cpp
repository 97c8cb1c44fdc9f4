#include "hm_error.h"

#include <cstdarg>
#include <cstdio>

#include "../../include/hm_page.h"

namespace {
thread_local char g_msg[1024] = "";
thread_local int64_t g_requested = 0;
thread_local int64_t g_available = 0;
}  // namespace

int hm_set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_msg, sizeof(g_msg), fmt, ap);
  va_end(ap);
  return code;
}

void hm_set_alloc_bytes(int64_t requested, int64_t available) {
  g_requested = requested;
  g_available = available;
}

extern "C" {

const char* hm_last_error(void) { return g_msg; }

void hm_last_error_bytes(int64_t* requested, int64_t* available) {
  if (requested) *requested = g_requested;
  if (available) *available = g_available;
}

int hm_abi_version(void) { return 2; }

int hm_device_chunk_elems(void) { return HM_ADAM_CHUNK; }

}  // extern "C"
