// Launcher of the TMA bulk-copy variant of the page-Adam main kernel
// (page_adam_tma.cu), selected with hm_set_adam_variant(1).
#pragma once
#include <atomic>
#include <cuda_runtime.h>

#include "../../include/hm_page.h"

namespace hm {

// 0 = LDG/STG streaming kernel (adam_main), 1 = persistent TMA bulk-copy pipeline.
extern std::atomic<int> g_adam_variant;

// Returns an HM_* status; supports g in {f16, bf16, f32} and p16 in {none, f16, bf16}.
int launch_adam_tma(const hm_adam_chunk* chunks, int64_t n_chunks, const hm_group_launch* groups,
                    const hm_group_rt* rt, const void* g, int g_dtype, float* p32, float* m32,
                    float* v32, void* p16, int p16_dtype, const hm_adam_hyper& hyper,
                    cudaStream_t stream);

}  // namespace hm
