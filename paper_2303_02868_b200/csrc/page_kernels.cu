// Segment kernels around the fused update:
//   hm_accumulate   ParamBuffer.accumulate (hiermem/lockfree.py:210-224) with the
//                   layer's reject flag and grad-norm term fused into the pass (K3)
//   hm_cast         publish cast (lockfree.py:169) / take widen (lockfree.py:234)
//   hm_reduce_stats isfinite + f64 sums (lockfree.py:133, 218-237) as a read-only pass
//   hm_copy_runs    page pack / unpack / relocation (pagemem.py:303-407 data motion, K1)
//   hm_memcpy_runs  pinned-host <-> HBM page swap on copy engines (K8)
#include "hm_device.cuh"
#include "hm_error.h"

#include <cstring>

namespace hm {
namespace {

// The segment kernels below stream 2-6 B/param with little math, so they
// need many bytes in flight per thread: 128 threads x 4 granules per
// 4096-element chunk (vs 256 x 2 for the register-heavy page-Adam).
constexpr int kSegThreads = 128;
constexpr int kSegVecPer = kChunk / (kSegThreads * kVec);
static_assert(kSegVecPer * kSegThreads * kVec == kChunk, "segment chunk geometry");

// Flush of the fused statistics: warp shuffles, ONE block barrier, then one
// atomic per CTA and statistic (per-warp f64 atomics on a few hundred layer
// addresses serialise in L2 and cost 3x in measurement).  sumsq feeds the
// grad norm / clip only, so its f64 atomic order is free to vary.  The
// ledger sum (LEDGER) is the f64 sum of (new - old) over the chunk: it goes
// to the slot's running sum (the buffer's total, read at take) and to the
// message's delta row (ConservationLedger.record_accumulate,
// hiermem/lockfree.py:218-222).  REUSE: a second barrier so the CTA can
// flush again (multi-chunk CTAs).
template <bool LEDGER, bool REUSE>
__device__ __forceinline__ void flush_stats(bool bad, float sq, double ls, uint32_t* nonfinite,
                                            double* sumsq, double* lsum, double* ldelta,
                                            uint32_t slot) {
  __shared__ float s_sq[kSegThreads / 32];
  __shared__ int s_bad[kSegThreads / 32];
  __shared__ double s_ls[LEDGER ? kSegThreads / 32 : 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if constexpr (LEDGER) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
  }
  const int any = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    s_sq[warp] = sq;
    s_bad[warp] = any;
    if constexpr (LEDGER) s_ls[warp] = ls;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    double l = 0.0;
    int b = 0;
#pragma unroll
    for (int w = 0; w < kSegThreads / 32; ++w) {
      t += s_sq[w];
      b |= s_bad[w];
      if constexpr (LEDGER) l += s_ls[w];
    }
    if (nonfinite && b) atomicOr(&nonfinite[slot], 1u);
    if (sumsq && t != 0.f) atomicAdd(&sumsq[slot], (double)t);
    if constexpr (LEDGER) {
      if (l != 0.0 || l != l) {   // NaN must propagate (a poisoned ledger is unbalanced)
        atomicAdd(&lsum[slot], l);
        if (ldelta) atomicAdd(&ldelta[slot], l);
      }
    }
  }
  if constexpr (REUSE) __syncthreads();
}

// Per-thread ledger accumulator.  LM 1: f64 adds per element (every
// widening conversion on the FP64 path); LM 2: compensated f32 (Neumaier:
// running sum + f32 error term, both widened to f64 once per flush).  For
// 16-bit inputs of a realistic range both are exact, so the device sums
// equal the reference's np.sum(g16, dtype=float64) (tests/test_gpu_toy_sync.py).
template <int LM>
struct LedgerAcc;
template <>
struct LedgerAcc<0> {
  __device__ __forceinline__ void add(float) {}
  __device__ __forceinline__ void add_delta(float, float) {}
  __device__ __forceinline__ double total() const { return 0.0; }
  __device__ __forceinline__ void reset() {}
};
template <>
struct LedgerAcc<1> {
  double s = 0.0;
  __device__ __forceinline__ void add(float x) { s += (double)x; }
  __device__ __forceinline__ void add_delta(float r, float b) { s += (double)r - (double)b; }
  __device__ __forceinline__ double total() const { return s; }
  __device__ __forceinline__ void reset() { s = 0.0; }
};
template <>
struct LedgerAcc<2> {
  float s = 0.f, c = 0.f;
  __device__ __forceinline__ void add(float x) {
    const float t = __fadd_rn(s, x);
    c = __fadd_rn(c, fabsf(s) >= fabsf(x) ? __fadd_rn(__fsub_rn(s, t), x) : __fadd_rn(__fsub_rn(x, t), s));
    s = t;
  }
  __device__ __forceinline__ void add_delta(float r, float b) {
    add(r);
    add(-b);
  }
  __device__ __forceinline__ double total() const { return (double)s + (double)c; }
  __device__ __forceinline__ void reset() { s = c = 0.f; }
};


// dst = rn(f32(dst) + f32(src)) (add) or rn(0.0f + f32(src)) (first message).
// sumsq accumulates sum(new^2 - old^2) so that it telescopes to the squared
// norm of the final buffer over any number of messages; the ledger sum
// likewise accumulates sum(new - old).
//
// One 4096-element chunk per CTA, every raw load of the thread issued before
// any decode.  KIND: 0 = every chunk is a first message (the common case:
// one message per step; only the source is read — ncu on C2: round 1's
// 48-register kernel was register-limited to 40 warps per SM and latency-
// bound at 60% of DRAM peak; this form runs 12 CTAs of 40 registers with
// 32 B accesses); 1 = every chunk adds; 2 = per-slot mode from slot_modes.  More
// chunks per CTA with the same bytes in flight measured 50% slower (fewer
// resident CTAs to overlap the store and epilogue phases).
// The 32 B first-message path (HM_K3_WIDE=0 at build time restores the
// 16 B-access form for measurement: tools/build_variants.sh).
#ifndef HM_K3_WIDE
#define HM_K3_WIDE 1
#endif
constexpr bool kWideK3 = HM_K3_WIDE != 0;

// First-message form between 16-bit buffers: 12 resident CTAs (40 registers,
// no spill) measured best — 16 CTAs force 32 registers and spill the
// compensated ledger sum (C2, ledger on: 0.840-0.846 ms vs 0.861-0.913; the
// 16 B-access form at 16 CTAs: 0.852).
#ifndef HM_K3_MINB
#define HM_K3_MINB 12
#endif
template <int SDT, int DDT>
constexpr int acc_min_blocks(int kind) {
  // f32 granules are 32 B (twice the registers of a 16-bit granule)
  return SDT == HM_DT_F32 || DDT == HM_DT_F32 ? (kind == 0 ? 8 : 4) : (kind == 0 ? HM_K3_MINB : 8);
}

template <int SDT, int DDT, int KIND, int LM>
__global__ void __launch_bounds__(kSegThreads, acc_min_blocks<SDT, DDT>(KIND))
accumulate_kernel(const hm_seg_chunk* __restrict__ chunks, const void* __restrict__ src,
                  void* __restrict__ dst, const uint8_t* __restrict__ slot_modes,
                  uint32_t* __restrict__ nonfinite, double* __restrict__ sumsq,
                  double* __restrict__ lsum, double* __restrict__ ldelta) {
  constexpr bool LEDGER = LM != 0;
  const hm_seg_chunk c = chunks[blockIdx.x];
  const bool add = KIND == 1 || (KIND == 2 && slot_modes[c.slot] != 0);
  const int tid = threadIdx.x;
  bool bad = false;
  float sq = 0.f;
  LedgerAcc<LM> ls;
  const bool vec = ((c.src_off | c.dst_off | (uint64_t)c.n) & (kVec - 1)) == 0 &&
                   vec_base<SDT>(src) && vec_base<DDT>(dst);
  // First messages between 16-bit buffers: 32 B accesses (16 elements) —
  // half the load/store instructions of the 16 B path, and the source read
  // carries the L2 evict-first hint (256-bit accesses only, sm_100a).  Chunks
  // whose offsets / count / bases do not allow it (segment heads and tails)
  // take the element path: keeping the 16 B path in the same kernel would
  // cost registers, i.e. resident CTAs, for every chunk.
  constexpr bool k16 = SDT != HM_DT_F32 && DDT != HM_DT_F32;
  if constexpr (KIND == 0 && k16 && kWideK3) {
    const bool wide = ((c.src_off | c.dst_off | (uint64_t)c.n) & 15) == 0 &&
                      (((uintptr_t)src | (uintptr_t)dst) & 31u) == 0;
    if (wide) {
      using TS = typename Elem<SDT>::T;
      using TD = typename Elem<DDT>::T;
      constexpr int kW = kChunk / (kSegThreads * 16);   // 2 wide granules per thread
      uint32_t ra[kW][8];
#pragma unroll
      for (int k = 0; k < kW; ++k) {
        const uint32_t e = (uint32_t)(k * kSegThreads + tid) * 16;
        if (e < c.n) ld_ro_u8(static_cast<const TS*>(src) + c.src_off + e, ra[k]);
      }
#pragma unroll
      for (int k = 0; k < kW; ++k) {
        const uint32_t e = (uint32_t)(k * kSegThreads + tid) * 16;
        if (e >= c.n) continue;
        // converted in place: element j of the output overwrites element j
        // of the input once it has been read (both types are 16-bit)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          uint32_t& w = ra[k][j >> 1];
          const uint16_t bits = (j & 1) ? (uint16_t)(w >> 16) : (uint16_t)(w & 0xffffu);
          const TD nv = Elem<DDT>::narrow(__fadd_rn(0.0f, widen_bits<SDT>(bits)));   // stored as is
          const float r = Elem<DDT>::widen(nv);
          bad |= !is_finite(r);
          sq = __fmaf_rn(r, r, sq);   // the norm only feeds clipping: one rounding per term is fine
          if constexpr (LEDGER) ls.add(r);
          const uint32_t ob = (uint32_t)(*reinterpret_cast<const uint16_t*>(&nv));
          w = (j & 1) ? ((w & 0xffffu) | (ob << 16)) : ((w & 0xffff0000u) | ob);
        }
        st_u8(static_cast<TD*>(dst) + c.dst_off + e, ra[k]);
      }
    } else {
      for (uint32_t i = tid; i < c.n; i += kSegThreads) {
        const float r = Elem<DDT>::widen(Elem<DDT>::narrow(__fadd_rn(0.0f, load1<SDT>(src, c.src_off + i))));
        bad |= !is_finite(r);
        sq += __fmul_rn(r, r);
        if constexpr (LEDGER) ls.add(r);
        store1<DDT>(dst, c.dst_off + i, r);
      }
    }
    flush_stats<LEDGER, false>(bad, sq, ls.total(), nonfinite, sumsq, lsum, ldelta, c.slot);
    return;
  }
  if (vec) {
    Raw8<SDT> ra[kSegVecPer];
    Raw8<DDT> rb[KIND == 0 ? 1 : kSegVecPer];
#pragma unroll
    for (int k = 0; k < kSegVecPer; ++k) {
      const uint32_t e = (uint32_t)(k * kSegThreads + tid) * kVec;
      if (e < c.n) {
        ld_raw_ro<SDT>(src, c.src_off + e, ra[k]);
        if constexpr (KIND != 0) {
          if (add) ld_raw_rw<DDT>(dst, c.dst_off + e, rb[k]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kSegVecPer; ++k) {
      const uint32_t e = (uint32_t)(k * kSegThreads + tid) * kVec;
      if (e >= c.n) continue;
      F8 a, o;
      decode<SDT>(ra[k], a);
      if (KIND != 0 && add) {
        F8 b;
        decode<DDT>(rb[KIND == 0 ? 0 : k], b);
#pragma unroll
        for (int j = 0; j < kVec; ++j) {
          const float r = Elem<DDT>::widen(Elem<DDT>::narrow(__fadd_rn(b.v[j], a.v[j])));
          bad |= !is_finite(r);
          sq += __fsub_rn(__fmul_rn(r, r), __fmul_rn(b.v[j], b.v[j]));
          if constexpr (LEDGER) ls.add_delta(r, b.v[j]);
          o.v[j] = r;
        }
      } else {   // first message after a take: the buffer holds zeros, r = 0 + a
#pragma unroll
        for (int j = 0; j < kVec; ++j) {
          // 0 + a keeps the reference's -0 -> +0; r*r - 0*0 == r*r exactly
          const float r = Elem<DDT>::widen(Elem<DDT>::narrow(__fadd_rn(0.0f, a.v[j])));
          bad |= !is_finite(r);
          sq += __fmul_rn(r, r);
          if constexpr (LEDGER) ls.add(r);
          o.v[j] = r;
        }
      }
      store8<DDT>(dst, c.dst_off + e, o);
    }
  } else {
    for (uint32_t i = tid; i < c.n; i += kSegThreads) {
      const float a1 = load1<SDT>(src, c.src_off + i);
      const float b1 = add ? load1<DDT>(dst, c.dst_off + i) : 0.0f;
      const float r = Elem<DDT>::widen(Elem<DDT>::narrow(__fadd_rn(b1, a1)));
      bad |= !is_finite(r);
      sq += __fsub_rn(__fmul_rn(r, r), __fmul_rn(b1, b1));
      if constexpr (LEDGER) ls.add_delta(r, b1);
      store1<DDT>(dst, c.dst_off + i, r);
    }
  }
  flush_stats<LEDGER, false>(bad, sq, ls.total(), nonfinite, sumsq, lsum, ldelta, c.slot);
}

// Snapshot-and-clear of a gradient buffer's fused statistics at a take
// (hiermem/lockfree.py:226-241 hand-over): out[2i] = running ledger sum,
// out[2i+1] = non-finite flag of slot slots[i]; then the slot's flag, norm
// and ledger sum are reset for the buffer's next first message.  Any
// pointer may be NULL (out NULL: reset only).
__global__ void stats_take_kernel(const uint32_t* __restrict__ slots, int n,
                                  uint32_t* __restrict__ nonfinite, double* __restrict__ sumsq,
                                  double* __restrict__ lsum, double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t s = slots[i];
    if (out) {
      out[2 * i] = lsum ? lsum[s] : 0.0;
      out[2 * i + 1] = nonfinite ? (double)nonfinite[s] : 0.0;
    }
    if (nonfinite) nonfinite[s] = 0u;
    if (sumsq) sumsq[s] = 0.0;
    if (lsum) lsum[s] = 0.0;
  }
}

template <int SDT, int DDT>
__global__ void __launch_bounds__(kSegThreads)
cast_kernel(const hm_seg_chunk* __restrict__ chunks, const void* __restrict__ src,
            void* __restrict__ dst) {
  pdl_enter();
  const hm_seg_chunk c = chunks[blockIdx.x];
  const int tid = threadIdx.x;
  const bool vec = ((c.src_off | c.dst_off | (uint64_t)c.n) & (kVec - 1)) == 0 &&
                   vec_base<SDT>(src) && vec_base<DDT>(dst);
  if (vec) {
    Raw8<SDT> ra[kSegVecPer];
#pragma unroll
    for (int k = 0; k < kSegVecPer; ++k) {
      const uint32_t e = (uint32_t)(k * kSegThreads + tid) * kVec;
      if (e < c.n) ld_raw_ro<SDT>(src, c.src_off + e, ra[k]);
    }
#pragma unroll
    for (int k = 0; k < kSegVecPer; ++k) {
      const uint32_t e = (uint32_t)(k * kSegThreads + tid) * kVec;
      if (e >= c.n) continue;
      F8 a;
      decode<SDT>(ra[k], a);
      store8<DDT>(dst, c.dst_off + e, a);
    }
  } else {
    for (uint32_t i = tid; i < c.n; i += kSegThreads)
      store1<DDT>(dst, c.dst_off + i, load1<SDT>(src, c.src_off + i));
  }
}

template <int SDT>
__global__ void __launch_bounds__(kSegThreads)
reduce_kernel(const hm_seg_chunk* __restrict__ chunks, const void* __restrict__ src,
              uint32_t* __restrict__ nonfinite, double* __restrict__ sums,
              double* __restrict__ sumsq) {
  __shared__ double red[kSegThreads / 32];
  const hm_seg_chunk c = chunks[blockIdx.x];
  const int tid = threadIdx.x;
  bool bad = false;
  double s = 0.0, sq = 0.0;
  const bool vec = ((c.src_off | (uint64_t)c.n) & (kVec - 1)) == 0 && vec_base<SDT>(src);
  if (vec) {
    Raw8<SDT> ra[kSegVecPer];
#pragma unroll
    for (int k = 0; k < kSegVecPer; ++k) {
      const uint32_t e = (uint32_t)(k * kSegThreads + tid) * kVec;
      if (e < c.n) ld_raw_ro<SDT>(src, c.src_off + e, ra[k]);
    }
#pragma unroll
    for (int k = 0; k < kSegVecPer; ++k) {
      const uint32_t e = (uint32_t)(k * kSegThreads + tid) * kVec;
      if (e >= c.n) continue;
      F8 a;
      decode<SDT>(ra[k], a);
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        const float x = a.v[j];
        bad |= !is_finite(x);
        s += (double)x;
        sq += (double)x * (double)x;
      }
    }
  } else {
    for (uint32_t i = tid; i < c.n; i += kSegThreads) {
      const float x = load1<SDT>(src, c.src_off + i);
      bad |= !is_finite(x);
      s += (double)x;
      sq += (double)x * (double)x;
    }
  }
  if (sums) {
    const double tot = block_sum<kSegThreads>(s, red);
    if (threadIdx.x == 0) atomicAdd(&sums[c.slot], tot);
  }
  flush_stats<false, false>(bad, (float)sq, 0.0, nonfinite, sumsq, nullptr, nullptr, c.slot);
}

// Occupies one warp of the stream for `ns` nanoseconds of %globaltimer: the
// stand-in for a compute slot of modelled duration when an Algorithm-1
// schedule is executed (executor.py); it moves no bytes.
__global__ void spin_kernel(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

// Byte-run copy: one CTA per descriptor; 16-byte vectors once source and
// destination are co-aligned, 4/2/1-byte granules otherwise.
__global__ void __launch_bounds__(kThreads)
copy_runs_kernel(const char* __restrict__ src, char* __restrict__ dst,
                 const hm_copy_desc* __restrict__ descs) {
  const hm_copy_desc d = descs[blockIdx.x];
  const char* s = src + d.src_off;
  char* t = dst + d.dst_off;
  uint64_t n = d.bytes;
  const int tid = threadIdx.x;
  const uint64_t mis = ((uint64_t)s ^ (uint64_t)t);
  if ((mis & 15) == 0) {
    const uint64_t head = (16 - ((uint64_t)s & 15)) & 15;
    const uint64_t h = head < n ? head : n;
    if ((uint64_t)tid < h) t[tid] = s[tid];
    s += h;
    t += h;
    n -= h;
    const uint64_t nv = n >> 4;
    const uint4* sv = reinterpret_cast<const uint4*>(s);
    uint4* tv = reinterpret_cast<uint4*>(t);
    uint64_t i = tid;
    for (; i + 3 * kThreads < nv; i += 4 * kThreads) {
      uint4 a0 = ld_stream_u4(sv + i), a1 = ld_stream_u4(sv + i + kThreads);
      uint4 a2 = ld_stream_u4(sv + i + 2 * kThreads), a3 = ld_stream_u4(sv + i + 3 * kThreads);
      st_stream_u4(tv + i, a0);
      st_stream_u4(tv + i + kThreads, a1);
      st_stream_u4(tv + i + 2 * kThreads, a2);
      st_stream_u4(tv + i + 3 * kThreads, a3);
    }
    for (; i < nv; i += kThreads) st_stream_u4(tv + i, ld_stream_u4(sv + i));
    for (uint64_t j = (nv << 4) + tid; j < n; j += kThreads) t[j] = s[j];
  } else if ((mis & 3) == 0) {
    const uint64_t head = (4 - ((uint64_t)s & 3)) & 3;
    const uint64_t h = head < n ? head : n;
    if ((uint64_t)tid < h) t[tid] = s[tid];
    s += h;
    t += h;
    n -= h;
    const uint64_t nw = n >> 2;
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(s);
    uint32_t* tw = reinterpret_cast<uint32_t*>(t);
    for (uint64_t i = tid; i < nw; i += kThreads) tw[i] = sw[i];
    for (uint64_t j = (nw << 2) + tid; j < n; j += kThreads) t[j] = s[j];
  } else if ((mis & 1) == 0) {
    const uint64_t h = ((uint64_t)s & 1) && n ? 1 : 0;
    if ((uint64_t)tid < h) t[0] = s[0];
    s += h;
    t += h;
    n -= h;
    const uint64_t nh = n >> 1;
    const uint16_t* sh = reinterpret_cast<const uint16_t*>(s);
    uint16_t* th = reinterpret_cast<uint16_t*>(t);
    for (uint64_t i = tid; i < nh; i += kThreads) th[i] = sh[i];
    if ((n & 1) && tid == 0) t[n - 1] = s[n - 1];
  } else {
    for (uint64_t j = tid; j < n; j += kThreads) t[j] = s[j];
  }
}


using AccFn = void (*)(const hm_seg_chunk*, const void*, void*, const uint8_t*, uint32_t*, double*,
                       double*, double*);
using CastFn = void (*)(const hm_seg_chunk*, const void*, void*);
using RedFn = void (*)(const hm_seg_chunk*, const void*, uint32_t*, double*, double*);

// Ledger accumulator per kernel form (measured on C2, bf16): first messages
// with the compensated f32 sum run at 0.86-0.88 ms (f64 per element: 1.03
// ms — the widening conversions, not the memory, become the limit); adds
// (two terms per element) with f64 at 1.20 ms (compensated f32: 1.49 ms).
template <int S, int D, int K>
AccFn acc_k(bool ledger) {
  if (!ledger) return accumulate_kernel<S, D, K, 0>;
  return accumulate_kernel<S, D, K, K == 0 ? 2 : 1>;
}
template <int S, int D>
AccFn acc_sd(int kind, bool ledger) {
  switch (kind) {
    case 0: return acc_k<S, D, 0>(ledger);
    case 1: return acc_k<S, D, 1>(ledger);
    default: return acc_k<S, D, 2>(ledger);
  }
}
template <int S>
AccFn acc_d(int d, int kind, bool ledger) {
  switch (d) {
    case HM_DT_F16: return acc_sd<S, HM_DT_F16>(kind, ledger);
    case HM_DT_BF16: return acc_sd<S, HM_DT_BF16>(kind, ledger);
    case HM_DT_F32: return acc_sd<S, HM_DT_F32>(kind, ledger);
  }
  return nullptr;
}
AccFn pick_acc(int s, int d, int kind, bool ledger) {
  switch (s) {
    case HM_DT_F16: return acc_d<HM_DT_F16>(d, kind, ledger);
    case HM_DT_BF16: return acc_d<HM_DT_BF16>(d, kind, ledger);
    case HM_DT_F32: return acc_d<HM_DT_F32>(d, kind, ledger);
  }
  return nullptr;
}
template <int S>
CastFn cast_d(int d) {
  switch (d) {
    case HM_DT_F16: return cast_kernel<S, HM_DT_F16>;
    case HM_DT_BF16: return cast_kernel<S, HM_DT_BF16>;
    case HM_DT_F32: return cast_kernel<S, HM_DT_F32>;
  }
  return nullptr;
}
CastFn pick_cast(int s, int d) {
  switch (s) {
    case HM_DT_F16: return cast_d<HM_DT_F16>(d);
    case HM_DT_BF16: return cast_d<HM_DT_BF16>(d);
    case HM_DT_F32: return cast_d<HM_DT_F32>(d);
  }
  return nullptr;
}
RedFn pick_red(int s) {
  switch (s) {
    case HM_DT_F16: return reduce_kernel<HM_DT_F16>;
    case HM_DT_BF16: return reduce_kernel<HM_DT_BF16>;
    case HM_DT_F32: return reduce_kernel<HM_DT_F32>;
  }
  return nullptr;
}

int check_grid(int64_t n, const char* who) {
  if (n < 0 || n > 0x7fffffffLL)
    return hm_set_error(HM_ERR_INVALID, "%s: bad chunk count %lld", who, (long long)n);
  return HM_OK;
}

}  // namespace
}  // namespace hm

extern "C" {

int hm_accumulate(const void* src, int src_dtype, void* dst, int dst_dtype,
                  const hm_seg_chunk* chunks, int64_t n_chunks, int mode,
                  const uint8_t* slot_modes, uint32_t* nonfinite, double* sumsq,
                  double* lsum, double* ldelta, const hm_launch_opts* opts, void* stream) {
  (void)opts;   // one launch shape (see accumulate_kernel)
  if (int rc = hm::check_grid(n_chunks, "hm_accumulate")) return rc;
  if (ldelta && !lsum)
    return hm_set_error(HM_ERR_INVALID, "hm_accumulate: a ledger delta row needs the running sums");
  const int kind = slot_modes ? 2 : mode ? 1 : 0;
  hm::AccFn fn = hm::pick_acc(src_dtype, dst_dtype, kind, lsum != nullptr);
  if (!fn) return hm_set_error(HM_ERR_INVALID, "hm_accumulate: unsupported dtypes %d -> %d", src_dtype, dst_dtype);
  if (n_chunks == 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_accumulate", src, dst, chunks);
  fn<<<(unsigned)n_chunks, hm::kSegThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      chunks, src, dst, slot_modes, nonfinite, sumsq, lsum, ldelta);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

int hm_stats_take(const uint32_t* slots, int32_t n_slots, uint32_t* nonfinite, double* sumsq,
                  double* lsum, double* out, void* stream) {
  if (n_slots < 0) return hm_set_error(HM_ERR_INVALID, "hm_stats_take: negative slot count");
  if (n_slots == 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_stats_take", slots);
  const int blocks = (n_slots + 255) / 256;
  hm::stats_take_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(slots, n_slots, nonfinite,
                                                                               sumsq, lsum, out);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

int hm_cast(const void* src, int src_dtype, void* dst, int dst_dtype, const hm_seg_chunk* chunks,
            int64_t n_chunks, void* stream) {
  if (int rc = hm::check_grid(n_chunks, "hm_cast")) return rc;
  hm::CastFn fn = hm::pick_cast(src_dtype, dst_dtype);
  if (!fn) return hm_set_error(HM_ERR_INVALID, "hm_cast: unsupported dtypes %d -> %d", src_dtype, dst_dtype);
  if (n_chunks == 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_cast", src, dst, chunks);
  const cudaError_t e = hm::launch_pdl(fn, (unsigned)n_chunks, hm::kSegThreads, static_cast<cudaStream_t>(stream),
                                       chunks, src, dst);
  if (e != cudaSuccess) return hm_set_error(HM_ERR_CUDA, "hm_cast: %s", cudaGetErrorString(e));
  return HM_OK;
}

int hm_reduce_stats(const void* src, int src_dtype, const hm_seg_chunk* chunks, int64_t n_chunks,
                    uint32_t* nonfinite, double* sums, double* sumsq, void* stream) {
  if (int rc = hm::check_grid(n_chunks, "hm_reduce_stats")) return rc;
  hm::RedFn fn = hm::pick_red(src_dtype);
  if (!fn) return hm_set_error(HM_ERR_INVALID, "hm_reduce_stats: unsupported dtype %d", src_dtype);
  if (n_chunks == 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_reduce_stats", src, chunks);
  fn<<<(unsigned)n_chunks, hm::kSegThreads, 0, static_cast<cudaStream_t>(stream)>>>(chunks, src, nonfinite,
                                                                                 sums, sumsq);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

int hm_copy_runs(const void* src, void* dst, const hm_copy_desc* descs, int64_t n_descs,
                 void* stream) {
  if (int rc = hm::check_grid(n_descs, "hm_copy_runs")) return rc;
  if (n_descs == 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_copy_runs", src, dst, descs);
  hm::copy_runs_kernel<<<(unsigned)n_descs, hm::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const char*>(src), static_cast<char*>(dst), descs);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

int hm_spin(int64_t ns, void* stream) {
  if (ns < 0) return hm_set_error(HM_ERR_INVALID, "hm_spin: negative duration");
  if (ns == 0) return HM_OK;
  hm::spin_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>((uint64_t)ns);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

int hm_host_alloc(int64_t bytes, void** out) {
  if (bytes <= 0 || !out) return hm_set_error(HM_ERR_INVALID, "hm_host_alloc: bad size %lld", (long long)bytes);
  *out = nullptr;
  cudaError_t e = cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    hm_set_alloc_bytes(bytes, 0);
    return hm_set_error(HM_ERR_ALLOCATION, "hm_host_alloc(%lld bytes): %s", (long long)bytes,
                        cudaGetErrorString(e));
  }
  std::memset(*out, 0, (size_t)bytes);
  return HM_OK;
}

int hm_host_free(void* ptr) {
  if (!ptr) return HM_OK;
  cudaError_t e = cudaFreeHost(ptr);
  if (e != cudaSuccess) return hm_set_error(HM_ERR_CUDA, "hm_host_free: %s", cudaGetErrorString(e));
  return HM_OK;
}

int hm_memcpy_runs(const void* src, void* dst, const hm_copy_desc* descs, int64_t n_descs,
                   int kind, void* stream) {
  if (n_descs < 0 || (n_descs > 0 && !descs))
    return hm_set_error(HM_ERR_INVALID, "hm_memcpy_runs: bad descriptors");
  cudaMemcpyKind k;
  switch (kind) {
    case 1: k = cudaMemcpyHostToDevice; break;
    case 2: k = cudaMemcpyDeviceToHost; break;
    case 3: k = cudaMemcpyDeviceToDevice; break;
    default: return hm_set_error(HM_ERR_INVALID, "hm_memcpy_runs: bad kind %d", kind);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int64_t i = 0; i < n_descs; ++i) {
    const hm_copy_desc& d = descs[i];
    cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + d.dst_off,
                                    static_cast<const char*>(src) + d.src_off, d.bytes, k, st);
    if (e != cudaSuccess)
      return hm_set_error(HM_ERR_CUDA, "hm_memcpy_runs: %s", cudaGetErrorString(e));
  }
  return HM_OK;
}

}  // extern "C"
