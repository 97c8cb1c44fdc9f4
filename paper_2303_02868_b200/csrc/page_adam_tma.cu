// Page-Adam main pass as a persistent TMA bulk-copy pipeline (sm_100a).
//
// Same arithmetic and bytes as adam_main (page_adam.cu, 28 B/param, bit-exact
// to hiermem/lockfree.py:127-142 + the publish cast :168-171), different
// data movement: one CTA per SM, warp-specialised.
//
//   producer warp   : for each of the CTA's chunks, wait until stage s is
//                     free, then cp.async.bulk (TMA) the chunk's g, p, m, v
//                     runs into stage s, completing on an mbarrier (tx bytes);
//   8 consumer warps: wait for the stage, run the Adam chain from shared
//                     memory, write p/m/v (+ the 16-bit publish) back into the
//                     stage, and one thread bulk-stores them to HBM and frees
//                     the stage once the TMA has read it.
//
// With 3 stages of 64 KB the SM keeps two chunks (112 KB) of loads in flight
// while the third is computed and stored, with no register pressure from the
// loads themselves.  Chunks whose runs are not 16-byte aligned (segment heads
// and tails) are processed straight from global memory by the consumers.
#include "hm_adam.cuh"
#include "hm_error.h"
#include "hm_tma.h"

namespace hm {

std::atomic<int> g_adam_variant{0};

namespace {

constexpr int kMaxStages = 4;
constexpr int kConsumerWarps = 16;  // the Adam chain is latency-bound per warp: 16 warps hide it
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kTmaThreads = kConsumers + 32;

// One stage = one 4096-element chunk: g | p | m | v, and the 16-bit publish.
// With a 16-bit gradient each thread writes its published granule over the
// g granule it has just consumed (same 16 B), so a stage is 56 KB and four
// stages (224 KB) fit: two chunks loading while one computes and one drains.
template <int GDT>
struct StageLayout {
  static constexpr bool kF32G = GDT == HM_DT_F32;
  static constexpr int kGBytes = kChunk * (kF32G ? 4 : 2);
  static constexpr int kOffP = kGBytes;
  static constexpr int kOffM = kOffP + kChunk * 4;
  static constexpr int kOffV = kOffM + kChunk * 4;
  static constexpr int kOffP16 = kF32G ? kOffV + kChunk * 4 : 0;
  static constexpr int kBytes = kOffV + kChunk * 4 + (kF32G ? kChunk * 2 : 0);
  static constexpr int kStages = kF32G ? 3 : 4;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "HM_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra HM_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Every byte is touched once per sweep: both directions carry an L2
// evict-first policy so the stream does not displace reusable lines (the
// LDG kernel's .L2::evict_first on its 256-bit accesses, as a TMA hint).
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
               ::"l"(dst), "r"(smem_u32(src)), "r"(bytes), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

template <int DT>
__device__ __forceinline__ void smem_load8(const unsigned char* base, int e, F8& out) {
  if constexpr (DT == HM_DT_F32) {
    const float4* q = reinterpret_cast<const float4*>(base + e * 4);
    const float4 a = q[0], b = q[1];
    out.v[0] = a.x; out.v[1] = a.y; out.v[2] = a.z; out.v[3] = a.w;
    out.v[4] = b.x; out.v[5] = b.y; out.v[6] = b.z; out.v[7] = b.w;
  } else {
    Raw8<DT> r;
    r.u = *reinterpret_cast<const uint4*>(base + e * 2);
    decode<DT>(r, out);
  }
}
__device__ __forceinline__ void smem_store8f(unsigned char* base, int e, const F8& v) {
  float4* q = reinterpret_cast<float4*>(base + e * 4);
  q[0] = make_float4(v.v[0], v.v[1], v.v[2], v.v[3]);
  q[1] = make_float4(v.v[4], v.v[5], v.v[6], v.v[7]);
}
template <int PDT>
__device__ __forceinline__ void smem_store8h(unsigned char* base, int e, const F8& v) {
  using T = typename Elem<PDT>::T;
  uint4 u;
  T* h = reinterpret_cast<T*>(&u);
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] = Elem<PDT>::narrow(v.v[i]);
  *reinterpret_cast<uint4*>(base + e * 2) = u;
}

template <int GDT, int PDT>
__global__ void __launch_bounds__(kTmaThreads, 1)
adam_tma(const hm_adam_chunk* __restrict__ chunks, int n_chunks,
         const hm_group_launch* __restrict__ groups, const hm_group_rt* __restrict__ rt,
         const void* __restrict__ g, float* __restrict__ p32, float* __restrict__ m32,
         float* __restrict__ v32, void* __restrict__ p16, hm_adam_hyper hyper) {
  using L = StageLayout<GDT>;
  constexpr int kGE = GDT == HM_DT_F32 ? 4 : 2;
  constexpr bool kPub = PDT != 0;
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int kStages = L::kStages;
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ int vecflag[kMaxStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t pol = evict_first_policy();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int iters = blockIdx.x < n_chunks ? (n_chunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (warp == kConsumerWarps) {  // ---- producer ----
    if (lane == 0) {
      for (int it = 0; it < iters; ++it) {
        const int s = it % kStages;
        mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
        const hm_adam_chunk c = chunks[blockIdx.x + it * gridDim.x];
        const hm_group_launch gl = groups[c.slot];
        const uint64_t go = c.g_off + gl.g_shift, so = c.s_off, po = c.p_off + gl.p_shift;
        // bulk copies need 16 B aligned global addresses and sizes
        const bool vec = ((go | so | po | (uint64_t)c.n) & (kVec - 1)) == 0 && vec_base<GDT>(g) &&
                         vec_base<HM_DT_F32>(p32) && vec_base<HM_DT_F32>(m32) && vec_base<HM_DT_F32>(v32) &&
                         (PDT == 0 || vec_base<PDT>(p16));
        vecflag[s] = vec ? 1 : 0;
        unsigned char* st = smem + s * L::kBytes;
        if (vec) {
          const uint32_t gb = c.n * kGE, fb = c.n * 4;
          mbar_expect_tx(&full[s], gb + 3 * fb);
          bulk_g2s(st, static_cast<const char*>(g) + go * kGE, gb, &full[s], pol);
          bulk_g2s(st + L::kOffP, p32 + so, fb, &full[s], pol);
          bulk_g2s(st + L::kOffM, m32 + so, fb, &full[s], pol);
          bulk_g2s(st + L::kOffV, v32 + so, fb, &full[s], pol);
        } else {
          mbar_arrive(&full[s]);  // consumers take this chunk straight from global memory
        }
      }
    }
    return;
  }

  // ---- consumers ----
  const int tid = threadIdx.x;
  int pending = -1;  // stage whose bulk stores may still be reading shared memory (thread 0)
  for (int it = 0; it < iters; ++it) {
    const int s = it % kStages;
    mbar_wait(&full[s], (it / kStages) & 1);
    const hm_adam_chunk c = chunks[blockIdx.x + it * gridDim.x];
    const hm_group_launch gl = groups[c.slot];
    const hm_group_rt r = rt[c.slot];
    const uint64_t go = c.g_off + gl.g_shift, so = c.s_off, po = c.p_off + gl.p_shift;
    const uint32_t n = c.n;
    const AdamScalars sc = make_scalars(hyper, r);
    unsigned char* st = smem + s * L::kBytes;
    if (vecflag[s]) {
#pragma unroll
      for (int k = 0; k < kChunk / (kConsumers * kVec); ++k) {
        const int e = (k * kConsumers + tid) * kVec;
        if ((uint32_t)e >= n) continue;
        F8 gv, pv, mv, vv;
        smem_load8<HM_DT_F32>(st + L::kOffP, e, pv);
        if (r.apply) {
          smem_load8<GDT>(st, e, gv);
          smem_load8<HM_DT_F32>(st + L::kOffM, e, mv);
          smem_load8<HM_DT_F32>(st + L::kOffV, e, vv);
#pragma unroll
          for (int j = 0; j < kVec; ++j) adam_elem(sc, gv.v[j], pv.v[j], mv.v[j], vv.v[j]);
          smem_store8f(st + L::kOffP, e, pv);
          smem_store8f(st + L::kOffM, e, mv);
          smem_store8f(st + L::kOffV, e, vv);
        }
        if constexpr (kPub) smem_store8h<PDT>(st + L::kOffP16, e, pv);
      }
      // Every writing thread orders its generic-proxy shared-memory stores
      // before the async-proxy bulk reads of them, then the barrier.
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      consumers_sync();  // the stage holds the results
      if (tid == 0) {
        if (r.apply) {
          bulk_s2g(p32 + so, st + L::kOffP, n * 4, pol);
          bulk_s2g(m32 + so, st + L::kOffM, n * 4, pol);
          bulk_s2g(v32 + so, st + L::kOffV, n * 4, pol);
        }
        if constexpr (kPub)
          bulk_s2g(static_cast<typename Elem<PDT>::T*>(p16) + po, st + L::kOffP16, n * 2, pol);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // Release the PREVIOUS stage once its stores have read shared memory
        // (at most this stage's group still reading): the store of chunk i
        // drains while chunk i+1 is computed.
        if (pending >= 0) {
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          mbar_arrive(&empty[pending]);
        }
        pending = s;
      }
    } else {
      for (uint32_t i = tid; i < n; i += kConsumers) {
        float p = p32[so + i];
        if (r.apply) {
          float gg = load1<GDT>(g, go + i), m = m32[so + i], v = v32[so + i];
          adam_elem(sc, gg, p, m, v);
          p32[so + i] = p;
          m32[so + i] = m;
          v32[so + i] = v;
        }
        if constexpr (kPub) store1<PDT>(p16, po + i, p);
      }
      consumers_sync();
      if (tid == 0) {
        if (pending >= 0) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          mbar_arrive(&empty[pending]);
          pending = -1;
        }
        mbar_arrive(&empty[s]);
      }
    }
  }
  if (tid == 0) {
    if (pending >= 0) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      mbar_arrive(&empty[pending]);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

using TmaFn = void (*)(const hm_adam_chunk*, int, const hm_group_launch*, const hm_group_rt*,
                       const void*, float*, float*, float*, void*, hm_adam_hyper);

template <int GDT>
TmaFn pick_p(int pdt) {
  switch (pdt) {
    case 0: return adam_tma<GDT, 0>;
    case HM_DT_F16: return adam_tma<GDT, HM_DT_F16>;
    case HM_DT_BF16: return adam_tma<GDT, HM_DT_BF16>;
  }
  return nullptr;
}

TmaFn pick(int gdt, int pdt) {
  switch (gdt) {
    case HM_DT_F16: return pick_p<HM_DT_F16>(pdt);
    case HM_DT_BF16: return pick_p<HM_DT_BF16>(pdt);
    case HM_DT_F32: return pick_p<HM_DT_F32>(pdt);
  }
  return nullptr;
}

int stage_bytes(int gdt) {
  return gdt == HM_DT_F32 ? StageLayout<HM_DT_F32>::kStages * StageLayout<HM_DT_F32>::kBytes
                          : StageLayout<HM_DT_BF16>::kStages * StageLayout<HM_DT_BF16>::kBytes;
}

}  // namespace

int launch_adam_tma(const hm_adam_chunk* chunks, int64_t n_chunks, const hm_group_launch* groups,
                    const hm_group_rt* rt, const void* g, int g_dtype, float* p32, float* m32,
                    float* v32, void* p16, int p16_dtype, const hm_adam_hyper& hyper,
                    cudaStream_t stream) {
  const int pdt = p16 ? p16_dtype : 0;
  TmaFn fn = pick(g_dtype, pdt);
  if (!fn) return hm_set_error(HM_ERR_INVALID, "adam_tma: unsupported dtypes g=%d p16=%d", g_dtype, pdt);
  if (n_chunks == 0) return HM_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = stage_bytes(g_dtype);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return hm_set_error(HM_ERR_CUDA, "adam_tma: %s", cudaGetErrorString(e));
  const int grid = (int)(n_chunks < sms ? n_chunks : sms);
  fn<<<grid, kTmaThreads, smem, stream>>>(chunks, (int)n_chunks, groups, rt, g, p32, m32, v32, p16,
                                          hyper);
  e = cudaGetLastError();
  if (e != cudaSuccess) return hm_set_error(HM_ERR_CUDA, "adam_tma: %s", cudaGetErrorString(e));
  return HM_OK;
}

}  // namespace hm

extern "C" int hm_set_adam_variant(int variant) {
  if (variant != 0 && variant != 1)
    return hm_set_error(HM_ERR_INVALID, "hm_set_adam_variant: 0 (LDG) or 1 (TMA), got %d", variant);
  hm::g_adam_variant = variant;
  return HM_OK;
}
