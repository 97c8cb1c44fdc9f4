// Fused page-Adam (K2 with the take/publish fusions K4/K5 of SURVEY §2.4).
//
// One HBM pass per element: read g (2 B bf16/fp16, or 4 B f32) and p32/m32/v32
// (12 B), write p32/m32/v32 (12 B) and the 16-bit published copy (2 B) —
// 28 B/param, the algorithmic minimum for the reference chain
//   take (hiermem/lockfree.py:226-241) -> update_layer (:155-165) ->
//   apply_update (:127-142) -> publish cast (:168-171, :243-263).
// The arithmetic is the reference's numpy chain restated op for op with
// correctly rounded binary32 operations and no contraction (numpy issues one
// ufunc per operator, so there is no FMA): bit-identical results.
//   m  = b1*m + (1-b1)*g                 lockfree.py:135
//   v  = b2*v + (1-b2)*(g*g)             lockfree.py:136
//   mh = m / f32(1-b1**step)             lockfree.py:137,139
//   vh = v / f32(1-b2**step)             lockfree.py:138,140
//   p  = p - (lr*mh) / (sqrt(vh) + eps)  lockfree.py:141
// The whole-layer reject of lockfree.py:133-134 (+ step rollback :163-164) is
// decided once per layer by the prologue from the flag that the gradient's
// producer (hm_accumulate / hm_reduce_stats) fused into its own pass.
#include <atomic>

#include "hm_adam.cuh"
#include "hm_device.cuh"
#include "hm_dp.cuh"
#include "hm_error.h"
#include "hm_tma.h"

namespace hm {
namespace {

constexpr int kPrologueThreads = 1024;

// Global-norm clip coefficient folded into the gradient scale (f64 norm of
// the unscaled gradient, one f32 rounding), shared by both prologue forms.
__device__ __forceinline__ float clip_gscale(const hm_adam_hyper& hyper, double total) {
  const double norm = sqrt(total) * (double)hyper.inv_scale;
  const double coef = norm > (double)hyper.max_norm ? (double)hyper.max_norm / (norm + 1e-6) : 1.0;
  return __fmul_rn(hyper.inv_scale, (float)coef);
}

// Per-layer decision: reject flag, step advance, bias-correction lookup,
// optional global grad-norm clip.  One CTA; deterministic reduction order.
__global__ void __launch_bounds__(kPrologueThreads)
adam_prologue(const hm_group_launch* __restrict__ groups, int n_groups,
              hm_group_rt* __restrict__ rt, hm_adam_hyper hyper,
              const float* __restrict__ bc_table, int64_t bc_len, int64_t explicit_step,
              int32_t* __restrict__ steps, uint32_t* __restrict__ applied,
              uint32_t* __restrict__ nonfinite, double* __restrict__ sumsq, int consume,
              double* __restrict__ lsum, double* __restrict__ ledger_out) {
  __shared__ double red[kPrologueThreads / 32];
  __shared__ float s_gscale;
  const bool clip = hyper.max_norm > 0.f && sumsq != nullptr;
  if (clip) {
    double local = 0.0;
    for (int i = threadIdx.x; i < n_groups; i += blockDim.x) {
      const uint32_t f = groups[i].flag;
      if (nonfinite == nullptr || nonfinite[f] == 0) local += sumsq[f];
    }
    const double total = block_sum<kPrologueThreads>(local, red);
    if (threadIdx.x == 0) s_gscale = clip_gscale(hyper, total);   // norm of the unscaled gradient
  } else if (threadIdx.x == 0) {
    s_gscale = hyper.inv_scale;
  }
  __syncthreads();
  const float gscale = s_gscale;
  for (int i = threadIdx.x; i < n_groups; i += blockDim.x) {
    const hm_group_launch gl = groups[i];
    const bool finite = nonfinite == nullptr || nonfinite[gl.flag] == 0;
    int64_t s;
    if (explicit_step > 0) {
      s = 0;  // bc_table[0] holds the caller's step
    } else {
      s = (int64_t)steps[gl.group] + 1;
      if (finite) steps[gl.group] = (int32_t)s;
      if (s >= bc_len) s = bc_len - 1;  // table is extended until it saturates at 1.0f
    }
    hm_group_rt r;
    r.bc1 = bc_table[2 * s];
    r.bc2 = bc_table[2 * s + 1];
    r.gscale = gscale;
    r.apply = finite ? 1u : 0u;
    rt[i] = r;
    if (applied) applied[gl.group] = r.apply;
    if (ledger_out) {   // ConservationLedger take/apply record (lockfree.py:237, :300)
      ledger_out[2 * i] = lsum ? lsum[gl.flag] : 0.0;
      ledger_out[2 * i + 1] = finite ? 1.0 : 0.0;
    }
    if (consume) {
      if (nonfinite) nonfinite[gl.flag] = 0u;
      if (sumsq) sumsq[gl.flag] = 0.0;
      if (lsum) lsum[gl.flag] = 0.0;
    }
  }
}


// Publish modes of the 16-bit epilogue: local pool, every peer's pool (P2P
// stores over NVLink = a fused all-gather), or one NVLS multicast store.
// kPubPeersBulk: the CTA stages its published chunk in shared memory and one
// thread pushes it to every peer with cp.async.bulk (one 8 KB bulk copy per
// peer instead of 512 per-thread 16 B stores; the stores no longer occupy the
// warps that stream the HBM state).
// The bulk mode waits for the remote writes before the CTA retires
// (hm_launch_opts.ag_publish 1 and 2 both select it).
constexpr int kPubLocal = 0, kPubPeers = 1, kPubMulticast = 2, kPubPeersBulk = 3;
template <int PUB>
constexpr bool is_bulk() { return PUB == kPubPeersBulk; }
// Process-wide DEFAULTS of the tuning knobs (hm_set_*).  A launch takes its
// settings from its own hm_launch_opts argument; a field < 0 (or a NULL
// opts) falls back to these, read once per launch.
std::atomic<int> g_ag_publish{0};   // hm_set_ag_publish: 0 per-thread stores; 1 bulk; 2 bulk + full wait
std::atomic<int> g_update_ctas{0};  // hm_set_dp_update_ctas: 0 one CTA per chunk; >0 persistent grid

template <int PDT, int PUB>
__device__ __forceinline__ void publish8(void* p16, const PeerPtrs& peers, char* mc, uint64_t po,
                                         const F8& v) {
  if constexpr (PUB == kPubLocal) {
    store8<PDT>(p16, po, v);
  } else {
    using T = typename Elem<PDT>::T;
    uint4 u;
    T* h = reinterpret_cast<T*>(&u);
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = Elem<PDT>::narrow(v.v[i]);
    if constexpr (PUB == kPubPeers || is_bulk<PUB>()) {
#pragma unroll
      for (int r = 0; r < kMaxPeers; ++r)
        if (r < peers.n) st_stream_u4(reinterpret_cast<T*>(peers.p[r]) + po, u);
    } else {
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(
                       mc + po * sizeof(T)),
                   "r"(u.x), "r"(u.y), "r"(u.z), "r"(u.w)
                   : "memory");
    }
  }
}

template <int PDT, int PUB>
__device__ __forceinline__ void publish1(void* p16, const PeerPtrs& peers, uint64_t po, float x) {
  if constexpr (PUB == kPubLocal) {
    store1<PDT>(p16, po, x);
  } else {
    // constant indices only: a runtime-indexed peers.p[r] would copy the
    // peer table to local memory and push ptxas into spilling the hot path
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r)
      if (r < peers.n) store1<PDT>(reinterpret_cast<void*>(peers.p[r]), po, x);
  }
}

// NT threads per 4096-element chunk: 256 (2 granules/thread, all 7 loads of
// both issued up front) or 512 (1 granule/thread, more warps to hide latency).
// OUT: the new masters are also stored to a contiguous tensor (pout, at the
// chunk's tensor offset oo) — MasterState.p32[l] without an unpack pass.
template <int GDT, int PDT, int PUB, int NT, bool OUT = false>
__device__ __forceinline__ void adam_chunk(const hm_adam_chunk& c,
                                           const hm_group_launch* __restrict__ groups,
                                           const hm_group_rt* __restrict__ rt,
                                           const void* __restrict__ g, float* __restrict__ p32,
                                           float* __restrict__ m32, float* __restrict__ v32,
                                           void* __restrict__ p16, const hm_adam_hyper& hyper,
                                           const PeerPtrs& peers, char* mc,
                                           float* __restrict__ pout = nullptr, uint64_t oo = 0) {
  const hm_group_launch gl = groups[c.slot];
  const hm_group_rt r = rt[c.slot];
  const uint64_t go = c.g_off + gl.g_shift;
  const uint64_t so = c.s_off;
  const uint64_t po = c.p_off + gl.p_shift;
  const uint32_t n = c.n;
  const int tid = threadIdx.x;
  constexpr bool kPub = PDT != 0;
  __shared__ __align__(128) uint4 s_pub[is_bulk<PUB>() ? kChunk / kVec : 1];

  if (!r.apply) {
    // Rejected layer: state untouched; still publish the unchanged masters.
    if constexpr (kPub || OUT) {
      for (uint32_t i = tid; i < n; i += NT) {
        const float x = p32[so + i];
        if constexpr (kPub) publish1<PDT, PUB>(p16, peers, po + i, x);
        if constexpr (OUT) pout[oo + i] = x;
      }
    }
    return;
  }
  AdamScalars s;
  s.lr = hyper.lr;
  s.b1 = hyper.beta1;
  s.ob1 = hyper.one_minus_beta1;
  s.b2 = hyper.beta2;
  s.ob2 = hyper.one_minus_beta2;
  s.eps = hyper.eps;
  s.bc1 = r.bc1;
  s.bc2 = r.bc2;
  s.gscale = r.gscale;

  const bool vec = ((go | so | po | (uint64_t)n) & (kVec - 1)) == 0 && vec_base<GDT>(g) &&
                   vec_base<HM_DT_F32>(p32) && vec_base<HM_DT_F32>(m32) && vec_base<HM_DT_F32>(v32) &&
                   (PDT == 0 || PUB != kPubLocal || vec_base<PDT>(p16));
  if (vec) {
    // Issue every load of the thread's 2 granules before any math: 2 x
    // (16 B g + 3 x 32 B state) in flight per thread.
    constexpr int VPT = kChunk / (NT * kVec);
    // Raw loads of every granule first (4 per granule: g 128-bit, p/m/v
    // 256-bit), decode afterwards: no use between two loads, so all of a
    // thread's loads are in flight together.
    Raw8<GDT> graw[VPT];
    F8 pv[VPT], mv[VPT], vv[VPT];
    bool live[VPT];
    const bool ovec = OUT && (oo & (kVec - 1)) == 0 && vec_base<HM_DT_F32>(pout);
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const uint32_t e = (uint32_t)(k * NT + tid) * kVec;
      live[k] = e < n;
      if (live[k]) {
        ld_raw_ro<GDT>(g, go + e, graw[k]);
        load8_rw<HM_DT_F32>(p32, so + e, pv[k]);
        load8_rw<HM_DT_F32>(m32, so + e, mv[k]);
        load8_rw<HM_DT_F32>(v32, so + e, vv[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      if (!live[k]) continue;
      const uint32_t e = (uint32_t)(k * NT + tid) * kVec;
      F8 gk;
      decode<GDT>(graw[k], gk);
#pragma unroll
      for (int j = 0; j < kVec; ++j) adam_elem(s, gk.v[j], pv[k].v[j], mv[k].v[j], vv[k].v[j]);
      store8<HM_DT_F32>(p32, so + e, pv[k]);
      store8<HM_DT_F32>(m32, so + e, mv[k]);
      store8<HM_DT_F32>(v32, so + e, vv[k]);
      if constexpr (OUT) {
        if (ovec) {
          store8<HM_DT_F32>(pout, oo + e, pv[k]);
        } else {
#pragma unroll
          for (int j = 0; j < kVec; ++j) pout[oo + e + j] = pv[k].v[j];
        }
      }
      if constexpr (is_bulk<PUB>()) {
        using T = typename Elem<PDT>::T;
        uint4 u;
        T* h = reinterpret_cast<T*>(&u);
#pragma unroll
        for (int i = 0; i < 8; ++i) h[i] = Elem<PDT>::narrow(pv[k].v[i]);
        s_pub[e / kVec] = u;
      } else if constexpr (kPub) {
        publish8<PDT, PUB>(p16, peers, mc, po + e, pv[k]);
      }
    }
    if constexpr (is_bulk<PUB>()) {
      // every writer fences its shared stores toward the async proxy, then the barrier
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        using T = typename Elem<PDT>::T;
        const uint32_t src = (uint32_t)__cvta_generic_to_shared(s_pub);
#pragma unroll
        for (int r = 0; r < kMaxPeers; ++r) {
          if (r >= peers.n) break;
          T* dst = reinterpret_cast<T*>(peers.p[r]) + po;
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                       ::"l"(dst), "r"(src), "r"(n * (uint32_t)sizeof(T)) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // Remote writes must be complete (not just read out of shared
        // memory) before the CTA retires: the step's closing symmetric
        // barrier is what tells the peers their pages have landed.
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      }
    }
  } else {
    for (uint32_t i = tid; i < n; i += NT) {
      float gg = load1<GDT>(g, go + i);
      float p = p32[so + i], m = m32[so + i], v = v32[so + i];
      adam_elem(s, gg, p, m, v);
      p32[so + i] = p;
      m32[so + i] = m;
      v32[so + i] = v;
      if constexpr (kPub) publish1<PDT, PUB>(p16, peers, po + i, p);
      if constexpr (OUT) pout[oo + i] = p;
    }
  }
}

// update_layer of ONE layer from its 16-bit pages in ONE launch (the three-
// call path, hiermem/lockfree.py:155-165): each CTA derives the layer's
// runtime record itself — reject flag, step + 1, bias pair, clip scale, as
// adam_prologue does for a multi-layer launch — and the last CTA to retire
// commits the step (applied layers only) and the applied word.  Every CTA
// reads steps[] before its arrival on `done`, so the commit never races a
// read; the last CTA re-arms `done` for the stream's next launch.
template <int GDT, int PDT, bool OUT>
__global__ void __launch_bounds__(kThreads)
adam_layer(const hm_adam_chunk* __restrict__ chunks, const hm_group_launch* __restrict__ group,
           const void* __restrict__ g, float* __restrict__ p32, float* __restrict__ m32,
           float* __restrict__ v32, void* __restrict__ p16, hm_adam_hyper hyper,
           const float* __restrict__ bc_table, int64_t bc_len, int32_t* __restrict__ steps,
           uint32_t* __restrict__ applied, const uint32_t* __restrict__ nonfinite,
           const double* __restrict__ sumsq, uint32_t* __restrict__ done, float* __restrict__ pout,
           const uint64_t* __restrict__ out_off) {
  __shared__ hm_group_rt s_rt;
  __shared__ int32_t s_step;
  pdl_enter();
  if (threadIdx.x == 0) {
    const hm_group_launch gl = group[0];
    const bool finite = nonfinite == nullptr || nonfinite[gl.flag] == 0;
    int64_t st = (int64_t)steps[gl.group] + 1;
    s_step = (int32_t)st;
    if (st >= bc_len) st = bc_len - 1;   // the table saturates at 1.0f
    hm_group_rt r;
    r.bc1 = bc_table[2 * st];
    r.bc2 = bc_table[2 * st + 1];
    r.gscale = hyper.max_norm > 0.f && sumsq != nullptr ? clip_gscale(hyper, finite ? sumsq[gl.flag] : 0.0)
                                                         : hyper.inv_scale;
    r.apply = finite ? 1u : 0u;
    s_rt = r;
  }
  __syncthreads();
  adam_chunk<GDT, PDT, kPubLocal, kThreads, OUT>(chunks[blockIdx.x], group, &s_rt, g, p32, m32, v32, p16,
                                                 hyper, PeerPtrs{}, nullptr, pout,
                                                 OUT ? out_off[blockIdx.x] : 0);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(done, 1u) == gridDim.x - 1) {
      if (s_rt.apply) steps[group[0].group] = s_step;
      *applied = s_rt.apply;
      *done = 0u;
    }
  }
}

using AdamLayerFn = void (*)(const hm_adam_chunk*, const hm_group_launch*, const void*, float*, float*,
                             float*, void*, hm_adam_hyper, const float*, int64_t, int32_t*, uint32_t*,
                             const uint32_t*, const double*, uint32_t*, float*, const uint64_t*);

template <int DT>
AdamLayerFn pick_adam_layer_dt(bool out) {
  return out ? adam_layer<DT, DT, true> : adam_layer<DT, DT, false>;
}

template <int GDT, int PDT, int PUB = kPubLocal, int NT = kThreads>
__global__ void __launch_bounds__(NT)
adam_main(const hm_adam_chunk* __restrict__ chunks, const hm_group_launch* __restrict__ groups,
          const hm_group_rt* __restrict__ rt, const void* __restrict__ g,
          float* __restrict__ p32, float* __restrict__ m32, float* __restrict__ v32,
          void* __restrict__ p16, hm_adam_hyper hyper, PeerPtrs peers, char* mc) {
  adam_chunk<GDT, PDT, PUB, NT>(chunks[blockIdx.x], groups, rt, g, p32, m32, v32, p16, hyper,
                                peers, mc);
}

// Persistent form for the layer-group pipelined DP step: a grid of
// hm_set_dp_update_ctas CTAs strides over the chunks, so the update of group
// k occupies a fixed share of the SMs next to the persistent reduce of
// group k+1 instead of competing for every free slot.
template <int GDT, int PDT, int PUB>
__global__ void __launch_bounds__(kThreads)
adam_main_loop(const hm_adam_chunk* __restrict__ chunks, int n_chunks,
               const hm_group_launch* __restrict__ groups, const hm_group_rt* __restrict__ rt,
               const void* __restrict__ g, float* __restrict__ p32, float* __restrict__ m32,
               float* __restrict__ v32, hm_adam_hyper hyper, PeerPtrs peers, char* mc) {
  static_assert(!is_bulk<PUB>(), "the staged bulk epilogue reuses shared memory per chunk");
  for (int i = blockIdx.x; i < n_chunks; i += gridDim.x)
    adam_chunk<GDT, PDT, PUB, kThreads>(chunks[i], groups, rt, g, p32, m32, v32, nullptr, hyper,
                                        peers, mc);
}

using AdamFn = void (*)(const hm_adam_chunk*, const hm_group_launch*, const hm_group_rt*,
                        const void*, float*, float*, float*, void*, hm_adam_hyper, PeerPtrs, char*);

template <int DT>
AdamFn pick_adam_ag_dt(int pub) {
  switch (pub) {
    case kPubPeers: return adam_main<DT, DT, kPubPeers>;
    case kPubMulticast: return adam_main<DT, DT, kPubMulticast>;
    case kPubPeersBulk: return adam_main<DT, DT, kPubPeersBulk>;
  }
  return nullptr;
}

using AdamLoopFn = void (*)(const hm_adam_chunk*, int, const hm_group_launch*, const hm_group_rt*,
                           const void*, float*, float*, float*, hm_adam_hyper, PeerPtrs, char*);

AdamLoopFn pick_adam_ag_loop(int dt, int pub) {
  if (dt == HM_DT_BF16)
    return pub == kPubPeers ? adam_main_loop<HM_DT_BF16, HM_DT_BF16, kPubPeers>
                            : adam_main_loop<HM_DT_BF16, HM_DT_BF16, kPubMulticast>;
  return pub == kPubPeers ? adam_main_loop<HM_DT_F16, HM_DT_F16, kPubPeers>
                          : adam_main_loop<HM_DT_F16, HM_DT_F16, kPubMulticast>;
}

AdamFn pick_adam_ag(int gdt, int pdt, int pub) {
  if (pdt != gdt) return nullptr;
  if (gdt == HM_DT_BF16) return pick_adam_ag_dt<HM_DT_BF16>(pub);
  if (gdt == HM_DT_F16) return pick_adam_ag_dt<HM_DT_F16>(pub);
  return nullptr;
}

std::atomic<int> g_adam_threads{kThreads};  // tuning knob: hm_set_adam_threads

template <int GDT, int NT>
AdamFn pick_p(int pdt) {
  switch (pdt) {
    case 0: return adam_main<GDT, 0, kPubLocal, NT>;
    case HM_DT_F16: return adam_main<GDT, HM_DT_F16, kPubLocal, NT>;
    case HM_DT_BF16: return adam_main<GDT, HM_DT_BF16, kPubLocal, NT>;
  }
  return nullptr;
}

template <int NT>
AdamFn pick_adam_nt(int gdt, int pdt) {
  switch (gdt) {
    case HM_DT_F16: return pick_p<HM_DT_F16, NT>(pdt);
    case HM_DT_BF16: return pick_p<HM_DT_BF16, NT>(pdt);
    case HM_DT_F32: return pick_p<HM_DT_F32, NT>(pdt);
  }
  return nullptr;
}

AdamFn pick_adam(int gdt, int pdt, int threads) {
  return threads == 512 ? pick_adam_nt<512>(gdt, pdt) : pick_adam_nt<kThreads>(gdt, pdt);
}

}  // namespace
}  // namespace hm

namespace {
int prologue_args_ok(const hm_adam_hyper* hyper, const float* bc_table, int64_t bc_len,
                     const hm_group_rt* rt, int32_t n_groups, int64_t explicit_step,
                     const int32_t* steps) {
  if (!hyper || !bc_table || bc_len < 1 || !rt)
    return hm_set_error(HM_ERR_INVALID, "adam prologue: missing hyper/bc_table/rt scratch");
  if (n_groups <= 0)
    return hm_set_error(HM_ERR_INVALID, "adam prologue: bad group count %d", (int)n_groups);
  if (explicit_step <= 0 && !steps)
    return hm_set_error(HM_ERR_INVALID, "adam prologue: steps[] required without explicit_step");
  return HM_OK;
}

// Per-launch setting: the opts field when given (>= 0), else the process default.
int opt_or(const hm_launch_opts* o, int32_t hm_launch_opts::*field, int dflt) {
  return o && o->*field >= 0 ? o->*field : dflt;
}
}  // namespace

extern "C" int hm_adam_prologue(const hm_group_launch* groups, int32_t n_groups,
                                hm_group_rt* rt_scratch, const hm_adam_hyper* hyper,
                                const float* bc_table, int64_t bc_len, int64_t explicit_step,
                                int32_t* steps, uint32_t* applied, uint32_t* nonfinite,
                                double* sumsq, int consume_flags, double* lsum,
                                double* ledger_out, void* stream) {
  if (int rc = prologue_args_ok(hyper, bc_table, bc_len, rt_scratch, n_groups, explicit_step, steps))
    return rc;
  HM_REQUIRE_PTRS("hm_adam_prologue", groups);
  hm::adam_prologue<<<1, hm::kPrologueThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      groups, n_groups, rt_scratch, *hyper, bc_table, bc_len, explicit_step, steps, applied,
      nonfinite, sumsq, consume_flags, lsum, ledger_out);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

extern "C" int hm_adam_main(const hm_adam_chunk* chunks, int64_t n_chunks,
                            const hm_group_launch* groups, const hm_group_rt* rt, const void* g,
                            int g_dtype, float* p32, float* m32, float* v32, void* p16,
                            int p16_dtype, const hm_adam_hyper* hyper, const hm_launch_opts* opts,
                            void* stream) {
  if (!hyper || !rt) return hm_set_error(HM_ERR_INVALID, "hm_adam_main: missing hyper/rt");
  if (n_chunks < 0 || n_chunks > 0x7fffffffLL)
    return hm_set_error(HM_ERR_INVALID, "hm_adam_main: bad chunk count %lld", (long long)n_chunks);
  const int pdt = p16 ? p16_dtype : 0;
  const int threads = opt_or(opts, &hm_launch_opts::adam_threads,
                             hm::g_adam_threads.load(std::memory_order_relaxed));
  const int variant = opt_or(opts, &hm_launch_opts::adam_variant,
                             hm::g_adam_variant.load(std::memory_order_relaxed));
  if (threads != 256 && threads != 512)
    return hm_set_error(HM_ERR_INVALID, "hm_adam_main: 256 or 512 threads, got %d", threads);
  if (variant != 0 && variant != 1)
    return hm_set_error(HM_ERR_INVALID, "hm_adam_main: variant 0 or 1, got %d", variant);
  hm::AdamFn fn = hm::pick_adam(g_dtype, pdt, threads);
  if (!fn) return hm_set_error(HM_ERR_INVALID, "hm_adam_main: unsupported dtypes g=%d p16=%d", g_dtype, pdt);
  if (n_chunks == 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_adam_main", chunks, groups, g, p32, m32, v32);
  if (variant == 1)
    return hm::launch_adam_tma(chunks, n_chunks, groups, rt, g, g_dtype, p32, m32, v32, p16, p16_dtype,
                               *hyper, static_cast<cudaStream_t>(stream));
  hm::PeerPtrs none{};
  fn<<<(unsigned)n_chunks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
      chunks, groups, rt, g, p32, m32, v32, p16, *hyper, none, nullptr);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

extern "C" int hm_adam_layer(const hm_adam_chunk* chunks, int64_t n_chunks, const hm_group_launch* group,
                             const void* g16, int dtype, float* p32, float* m32, float* v32, void* p16,
                             const hm_adam_hyper* hyper, const float* bc_table, int64_t bc_len,
                             int32_t* steps, uint32_t* applied, const uint32_t* nonfinite,
                             const double* sumsq, uint32_t* done, float* p_out, const uint64_t* out_off,
                             void* stream) {
  if (!hyper || !bc_table || bc_len < 1)
    return hm_set_error(HM_ERR_INVALID, "hm_adam_layer: missing hyper/bc_table");
  if (n_chunks <= 0 || n_chunks > 0x7fffffffLL)
    return hm_set_error(HM_ERR_INVALID, "hm_adam_layer: bad chunk count %lld (a layer without "
                        "pages here takes hm_adam_step)", (long long)n_chunks);
  if (dtype != HM_DT_BF16 && dtype != HM_DT_F16)
    return hm_set_error(HM_ERR_INVALID, "hm_adam_layer: 16-bit pages only, got dtype %d", dtype);
  if ((p_out == nullptr) != (out_off == nullptr))
    return hm_set_error(HM_ERR_INVALID, "hm_adam_layer: p_out and out_off go together");
  HM_REQUIRE_PTRS("hm_adam_layer", chunks, group, g16, p32, m32, v32, p16, steps, applied, done);
  hm::AdamLayerFn fn = dtype == HM_DT_BF16 ? hm::pick_adam_layer_dt<HM_DT_BF16>(p_out != nullptr)
                                           : hm::pick_adam_layer_dt<HM_DT_F16>(p_out != nullptr);
  const cudaError_t e = hm::launch_pdl(fn, (unsigned)n_chunks, hm::kThreads, static_cast<cudaStream_t>(stream),
                                       chunks, group, g16, p32, m32, v32, p16, *hyper, bc_table, bc_len, steps,
                                       applied, nonfinite, sumsq, done, p_out, out_off);
  if (e != cudaSuccess) return hm_set_error(HM_ERR_CUDA, "hm_adam_layer: %s", cudaGetErrorString(e));
  return HM_OK;
}

extern "C" int hm_set_adam_threads(int threads) {
  if (threads != 256 && threads != 512)
    return hm_set_error(HM_ERR_INVALID, "hm_set_adam_threads: 256 or 512, got %d", threads);
  hm::g_adam_threads = threads;
  return HM_OK;
}

extern "C" int hm_set_dp_update_ctas(int ctas) {
  if (ctas < 0) return hm_set_error(HM_ERR_INVALID, "hm_set_dp_update_ctas: negative grid %d", ctas);
  hm::g_update_ctas = ctas;
  return HM_OK;
}

extern "C" int hm_set_ag_publish(int mode) {
  if (mode < 0 || mode > 2)
    return hm_set_error(HM_ERR_INVALID, "hm_set_ag_publish: 0, 1 or 2, got %d", mode);
  hm::g_ag_publish = mode;
  return HM_OK;
}

extern "C" int hm_adam_main_ag(const hm_adam_chunk* chunks, int64_t n_chunks,
                               const hm_group_launch* groups, const hm_group_rt* rt, const void* g,
                               int g_dtype, float* p32, float* m32, float* v32,
                               const uint64_t* peer_p16, int n_peers, void* mc_p16, int p16_dtype,
                               const hm_adam_hyper* hyper, const hm_launch_opts* opts, void* stream) {
  if (!hyper || !rt) return hm_set_error(HM_ERR_INVALID, "hm_adam_main_ag: missing hyper/rt");
  hm::PeerPtrs peers;
  if (int rc = hm::make_peers(peer_p16, n_peers, &peers)) return rc;
  const int agp = opt_or(opts, &hm_launch_opts::ag_publish, hm::g_ag_publish.load(std::memory_order_relaxed));
  if (agp < 0 || agp > 2)
    return hm_set_error(HM_ERR_INVALID, "hm_adam_main_ag: publish mode 0, 1 or 2, got %d", agp);
  const int pub = mc_p16 ? hm::kPubMulticast
                 : agp >= 1 ? hm::kPubPeersBulk : hm::kPubPeers;
  hm::AdamFn fn = hm::pick_adam_ag(g_dtype, p16_dtype, pub);
  if (!fn) return hm_set_error(HM_ERR_INVALID, "hm_adam_main_ag: unsupported dtypes g=%d p16=%d", g_dtype, p16_dtype);
  if (n_chunks < 0 || n_chunks > 0x7fffffffLL)
    return hm_set_error(HM_ERR_INVALID, "hm_adam_main_ag: bad chunk count");
  if (n_chunks == 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_adam_main_ag", chunks, groups, g, p32, m32, v32);
  const int uctas = opt_or(opts, &hm_launch_opts::grid_ctas, hm::g_update_ctas.load(std::memory_order_relaxed));
  if (uctas > 0 && (pub == hm::kPubPeers || pub == hm::kPubMulticast)) {
    hm::AdamLoopFn lf = hm::pick_adam_ag_loop(g_dtype, pub);
    const int64_t grid = uctas < n_chunks ? uctas : n_chunks;
    lf<<<(unsigned)grid, hm::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        chunks, (int)n_chunks, groups, rt, g, p32, m32, v32, *hyper, peers,
        static_cast<char*>(mc_p16));
    HM_CUDA_CHECK_LAUNCH();
    return HM_OK;
  }
  fn<<<(unsigned)n_chunks, hm::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      chunks, groups, rt, g, p32, m32, v32, nullptr, *hyper, peers, static_cast<char*>(mc_p16));
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

extern "C" int hm_adam_step(const hm_adam_chunk* chunks, int64_t n_chunks,
                            const hm_group_launch* groups, int32_t n_groups,
                            hm_group_rt* rt_scratch, const void* g, int g_dtype, float* p32,
                            float* m32, float* v32, void* p16, int p16_dtype,
                            const hm_adam_hyper* hyper, const float* bc_table, int64_t bc_len,
                            int64_t explicit_step, int32_t* steps, uint32_t* applied,
                            uint32_t* nonfinite, double* sumsq, int consume_flags,
                            double* lsum, double* ledger_out, const hm_launch_opts* opts,
                            void* stream) {
  const int pdt = p16 ? p16_dtype : 0;
  if (!hm::pick_adam(g_dtype, pdt, hm::kThreads))   // dtype check only
    return hm_set_error(HM_ERR_INVALID, "hm_adam_step: unsupported dtypes g=%d p16=%d", g_dtype, pdt);
  if (int rc = hm_adam_prologue(groups, n_groups, rt_scratch, hyper, bc_table, bc_len,
                                explicit_step, steps, applied, nonfinite, sumsq, consume_flags,
                                lsum, ledger_out, stream))
    return rc;
  return hm_adam_main(chunks, n_chunks, groups, rt_scratch, g, g_dtype, p32, m32, v32, p16,
                      p16_dtype, hyper, opts, stream);
}
