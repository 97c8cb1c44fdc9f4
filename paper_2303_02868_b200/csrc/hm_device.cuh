// Device helpers shared by the page kernels (sm_100a).
//
// Every page kernel is a streaming, HBM-bound pass: each byte is touched once,
// so loads bypass L1 (L1::no_allocate) and 256-bit f32 traffic carries the
// L2 evict-first hint (sm_100a accepts .L2::evict_* only on 256-bit access).
// A unit of 8 consecutive elements is the vector granule: 16 B for the
// 16-bit types, 32 B (one LDG.E.256 / STG.E.256) for f32.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hm_page.h"

namespace hm {

constexpr int kThreads = 256;
constexpr int kChunk = HM_ADAM_CHUNK;             // elements per CTA unit
constexpr int kVec = 8;                           // elements per vector granule
constexpr int kVecPerThread = kChunk / (kThreads * kVec);  // 2
static_assert(kChunk == kThreads * kVec * kVecPerThread, "chunk geometry");

struct F8 {
  float v[8];
};

// ---- raw vector memory ops ------------------------------------------------
__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream_u4(void* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
// 256-bit f32 load of data this kernel later overwrites (no .nc).
__device__ __forceinline__ void ld_stream_f8(const float* p, F8& r) {
  uint32_t u[8];
  asm volatile(
      "ld.global.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
        "=r"(u[7])
      : "l"(p));
#pragma unroll
  for (int i = 0; i < 8; ++i) r.v[i] = __uint_as_float(u[i]);
}
// 256-bit f32 load of read-only data (.nc path).
__device__ __forceinline__ void ld_ro_f8(const float* p, F8& r) {
  uint32_t u[8];
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
        "=r"(u[7])
      : "l"(p));
#pragma unroll
  for (int i = 0; i < 8; ++i) r.v[i] = __uint_as_float(u[i]);
}
__device__ __forceinline__ void st_stream_f8(float* p, const F8& r) {
  asm volatile(
      "st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
      "r"(__float_as_uint(r.v[0])), "r"(__float_as_uint(r.v[1])), "r"(__float_as_uint(r.v[2])),
      "r"(__float_as_uint(r.v[3])), "r"(__float_as_uint(r.v[4])), "r"(__float_as_uint(r.v[5])),
      "r"(__float_as_uint(r.v[6])), "r"(__float_as_uint(r.v[7]))
      : "memory");
}

// 256-bit access of 16 sixteen-bit elements (read-only source, evict-first).
__device__ __forceinline__ void ld_ro_u8(const void* p, uint32_t (&u)[8]) {
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
      : "l"(p));
}
__device__ __forceinline__ void st_u8(void* p, const uint32_t (&u)[8]) {
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(u[0]),
               "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7])
               : "memory");
}

// ---- typed element access (widen exactly / narrow with RNE) ---------------
template <int DT>
struct Elem;

template <>
struct Elem<HM_DT_F16> {
  using T = __half;
  static __device__ __forceinline__ float widen(T x) { return __half2float(x); }
  static __device__ __forceinline__ T narrow(float x) { return __float2half_rn(x); }
};
template <>
struct Elem<HM_DT_BF16> {
  using T = __nv_bfloat16;
  static __device__ __forceinline__ float widen(T x) { return __bfloat162float(x); }
  static __device__ __forceinline__ T narrow(float x) { return __float2bfloat16_rn(x); }
};
template <>
struct Elem<HM_DT_F32> {
  using T = float;
  static __device__ __forceinline__ float widen(T x) { return x; }
  static __device__ __forceinline__ T narrow(float x) { return x; }
};

// 16-bit element <-> its bit pattern (16-bit DT only).
template <int DT>
__device__ __forceinline__ float widen_bits(uint16_t b) {
  using T = typename Elem<DT>::T;
  return Elem<DT>::widen(*reinterpret_cast<const T*>(&b));
}
template <int DT>
__device__ __forceinline__ uint32_t narrow_bits(float x) {
  using T = typename Elem<DT>::T;
  const T h = Elem<DT>::narrow(x);
  return (uint32_t)(*reinterpret_cast<const uint16_t*>(&h));
}

template <int DT>
__device__ __forceinline__ float load1(const void* base, uint64_t off) {
  using T = typename Elem<DT>::T;
  return Elem<DT>::widen(static_cast<const T*>(base)[off]);
}
template <int DT>
__device__ __forceinline__ void store1(void* base, uint64_t off, float x) {
  using T = typename Elem<DT>::T;
  static_cast<T*>(base)[off] = Elem<DT>::narrow(x);
}

// Read-only streaming load of 8 elements at an 8-aligned offset.
template <int DT>
__device__ __forceinline__ void load8_ro(const void* base, uint64_t off, F8& r) {
  if constexpr (DT == HM_DT_F32) {
    ld_ro_f8(static_cast<const float*>(base) + off, r);
  } else {
    using T = typename Elem<DT>::T;
    uint4 u = ld_stream_u4(static_cast<const T*>(base) + off);
    const T* h = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int i = 0; i < 8; ++i) r.v[i] = Elem<DT>::widen(h[i]);
  }
}
// Load of 8 elements that this kernel overwrites afterwards.
template <int DT>
__device__ __forceinline__ void load8_rw(const void* base, uint64_t off, F8& r) {
  if constexpr (DT == HM_DT_F32) {
    ld_stream_f8(static_cast<const float*>(base) + off, r);
  } else {
    using T = typename Elem<DT>::T;
    uint4 u = *reinterpret_cast<const uint4*>(static_cast<const T*>(base) + off);
    const T* h = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int i = 0; i < 8; ++i) r.v[i] = Elem<DT>::widen(h[i]);
  }
}
template <int DT>
__device__ __forceinline__ void store8(void* base, uint64_t off, const F8& r) {
  if constexpr (DT == HM_DT_F32) {
    st_stream_f8(static_cast<float*>(base) + off, r);
  } else {
    using T = typename Elem<DT>::T;
    uint4 u;
    T* h = reinterpret_cast<T*>(&u);
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = Elem<DT>::narrow(r.v[i]);
    st_stream_u4(static_cast<T*>(base) + off, u);
  }
}

// Raw (undecoded) 8-element granules: issue every load of a thread first and
// decode afterwards, so no use sits between two loads (the compiler otherwise
// serialises load -> convert -> next load when a load is conditional).
template <int DT>
struct Raw8 {
  uint4 u;
};
template <>
struct Raw8<HM_DT_F32> {
  F8 f;
};

template <int DT>
__device__ __forceinline__ void ld_raw_ro(const void* base, uint64_t off, Raw8<DT>& r) {
  if constexpr (DT == HM_DT_F32) ld_ro_f8(static_cast<const float*>(base) + off, r.f);
  else r.u = ld_stream_u4(static_cast<const typename Elem<DT>::T*>(base) + off);
}
template <int DT>
__device__ __forceinline__ void ld_raw_rw(const void* base, uint64_t off, Raw8<DT>& r) {
  if constexpr (DT == HM_DT_F32) ld_stream_f8(static_cast<const float*>(base) + off, r.f);
  else r.u = *reinterpret_cast<const uint4*>(static_cast<const typename Elem<DT>::T*>(base) + off);
}
template <int DT>
__device__ __forceinline__ void decode(const Raw8<DT>& r, F8& out) {
  if constexpr (DT == HM_DT_F32) {
    out = r.f;
  } else {
    using T = typename Elem<DT>::T;
    const T* h = reinterpret_cast<const T*>(&r.u);
#pragma unroll
    for (int i = 0; i < 8; ++i) out.v[i] = Elem<DT>::widen(h[i]);
  }
}

__device__ __forceinline__ bool is_finite(float x) { return isfinite(x); }

// A buffer base the 8-element vector path may use: 16 B aligned for the
// 16-bit types (128-bit accesses), 32 B for f32 (256-bit accesses).  With an
// element offset that is a multiple of 8 the access is then aligned.  The
// kernels fall back to scalar element access otherwise, so any base works.
template <int DT>
__device__ __forceinline__ bool vec_base(const void* p) {
  return ((uintptr_t)p & (DT == HM_DT_F32 ? 31u : 15u)) == 0;
}

// Deterministic block reduction of a double (fixed tree order).
template <int NT>
__device__ __forceinline__ double block_sum(double x, double* smem) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) smem[warp] = x;
  __syncthreads();
  double r = 0.0;
  if (warp == 0) {
    r = lane < NT / 32 ? smem[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  return r;  // valid in thread 0
}

// ---- programmatic dependent launch -----------------------------------------
// A kernel launched by launch_pdl may become resident while the previous
// kernel of the stream drains.  pdl_enter, its first statement, lets its own
// successor do the same and then waits for the previous grid to complete
// with its memory visible — before any data is touched, so stream order is
// unchanged and only the launch latency between the two kernels is hidden
// (the three-call path issues ~2 small launches per layer).  Both
// instructions are no-ops in a normal launch.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, cudaStream_t stream,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace hm

#define HM_CUDA_CHECK_LAUNCH()                                                          \
  do {                                                                                  \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess)                                                              \
      return hm_set_error(HM_ERR_CUDA, "%s: %s", __func__, cudaGetErrorString(e_));     \
  } while (0)
