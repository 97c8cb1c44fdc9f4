// Thread-local error state shared by every translation unit of libhm_page.
#pragma once
#include <cstdint>

int hm_set_error(int code, const char* fmt, ...);
void hm_set_alloc_bytes(int64_t requested, int64_t available);
