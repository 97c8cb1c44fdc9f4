// The data-parallel page step as ONE pass over the owned pages (round 2):
//
//   hm_dp_onepass_update   per owned chunk: pull the chunk's 16-bit gradient
//                          from every rank's pool (P2P loads over NVLink, the
//                          owner's own included), sum in f32 in rank order and
//                          round once (the same bits as hm_dp_reduce_check),
//                          run the page-Adam chain, and store the new p32/m32/
//                          v32 into the layer's OTHER state buffer and the new
//                          16-bit page into every rank's publish pool (the
//                          all-gather epilogue of hm_adam_main_ag);
//   hm_dp_onepass_finalize after a cross-rank barrier: OR of the per-layer
//                          non-finite flags over the ranks; an applied layer
//                          commits its step and flips its state buffer, a
//                          rejected one keeps both (hiermem/lockfree.py:133-
//                          134, 163-164: state untouched, step rolled back);
//   hm_dp_republish_rejected  the rare rejected layer's pages get the
//                          unchanged parameters published again.
//
// Why: the two-phase step (reduce-scatter kernel, flag merge, update) has
// to finish every layer's reduce before its update may commit — the whole-
// layer reject.  Double-buffering the fp32 state makes the update
// speculative (the old state survives in the other buffer), so the reduce
// need not be written back and re-read, and the gradient transfer overlaps
// the update inside one kernel instead of two overlapping streams.  The
// reference models the exchange only (hiermem/simengine.py:255-257);
// ownership is hiermem/scheduler.py:72-76 (page % N).
#include "hm_adam.cuh"
#include "hm_device.cuh"
#include "hm_dp.cuh"
#include "hm_error.h"

namespace hm {
namespace {

// 512 threads x one granule per thread, two resident CTAs (64 registers) up
// to 4 peers: the remote loads need warps in flight more than granules per
// thread (N=2, C2: 4.04 ms vs 4.70 with 256 threads x 2).  Eight peers'
// gradient granules do not fit 64 registers: one CTA of 94.
template <int DT, int NP, int NT>
__global__ void __launch_bounds__(NT, NP <= 4 ? 2 : 1)
onepass_kernel(const hm_adam_chunk* __restrict__ chunks, const hm_group_launch* __restrict__ groups,
               const hm_group_rt* __restrict__ rt, const uint32_t* __restrict__ state_sel, uint64_t es,
               PeerPtrs gpeers, PeerPtrs ppeers, float* __restrict__ p32, float* __restrict__ m32,
               float* __restrict__ v32, uint32_t* __restrict__ nonfinite, hm_adam_hyper hyper) {
  using T = typename Elem<DT>::T;
  const hm_adam_chunk c = chunks[blockIdx.x];
  const hm_group_launch gl = groups[c.slot];
  const hm_group_rt r = rt[c.slot];
  const uint32_t sel = state_sel[gl.group];
  const uint64_t go = c.g_off + gl.g_shift, po = c.p_off + gl.p_shift;
  const uint64_t sr = c.s_off + (uint64_t)sel * es, sw = c.s_off + (uint64_t)(sel ^ 1u) * es;
  const uint32_t n = c.n;
  const int tid = threadIdx.x;
  const AdamScalars s = make_scalars(hyper, r);
  bool bad = false;
  const bool vec = ((go | sr | sw | po | (uint64_t)n) & (kVec - 1)) == 0 && vec_base<HM_DT_F32>(p32) &&
                   vec_base<HM_DT_F32>(m32) && vec_base<HM_DT_F32>(v32);
  if (vec) {
    constexpr int VPT = kChunk / (NT * kVec);
    uint4 graw[VPT][NP];
    F8 pv[VPT], mv[VPT], vv[VPT];
    // every load of the thread first: the peers' gradient granules (NVLink)
    // and the state granules (HBM)
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const uint32_t e = (uint32_t)(k * NT + tid) * kVec;
      if (e >= n) continue;
#pragma unroll
      for (int q = 0; q < NP; ++q)
        if (q < gpeers.n) graw[k][q] = ld_stream_u4(reinterpret_cast<const T*>(gpeers.p[q]) + go + e);
      load8_rw<HM_DT_F32>(p32, sr + e, pv[k]);
      load8_rw<HM_DT_F32>(m32, sr + e, mv[k]);
      load8_rw<HM_DT_F32>(v32, sr + e, vv[k]);
    }
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const uint32_t e = (uint32_t)(k * NT + tid) * kVec;
      if (e >= n) continue;
      float acc[kVec];
#pragma unroll
      for (int j = 0; j < kVec; ++j) acc[j] = 0.f;
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        if (q >= gpeers.n) break;
        const T* h = reinterpret_cast<const T*>(&graw[k][q]);
#pragma unroll
        for (int j = 0; j < kVec; ++j) acc[j] = __fadd_rn(acc[j], Elem<DT>::widen(h[j]));
      }
      uint4 u;
      T* hp = reinterpret_cast<T*>(&u);
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        const float g = Elem<DT>::widen(Elem<DT>::narrow(acc[j]));   // the reduced 16-bit gradient
        bad |= !is_finite(g);
        adam_elem(s, g, pv[k].v[j], mv[k].v[j], vv[k].v[j]);
        hp[j] = Elem<DT>::narrow(pv[k].v[j]);
      }
      store8<HM_DT_F32>(p32, sw + e, pv[k]);
      store8<HM_DT_F32>(m32, sw + e, mv[k]);
      store8<HM_DT_F32>(v32, sw + e, vv[k]);
#pragma unroll
      for (int q = 0; q < kMaxPeers; ++q)
        if (q < ppeers.n) st_stream_u4(reinterpret_cast<T*>(ppeers.p[q]) + po + e, u);
    }
  } else {
    for (uint32_t i = tid; i < n; i += NT) {
      float a = 0.f;
#pragma unroll
      for (int q = 0; q < NP; ++q)
        if (q < gpeers.n) a = __fadd_rn(a, Elem<DT>::widen(reinterpret_cast<const T*>(gpeers.p[q])[go + i]));
      const float g = Elem<DT>::widen(Elem<DT>::narrow(a));
      bad |= !is_finite(g);
      float p = p32[sr + i], m = m32[sr + i], v = v32[sr + i];
      adam_elem(s, g, p, m, v);
      p32[sw + i] = p;
      m32[sw + i] = m;
      v32[sw + i] = v;
#pragma unroll
      for (int q = 0; q < kMaxPeers; ++q)
        if (q < ppeers.n) store1<DT>(reinterpret_cast<void*>(ppeers.p[q]), po + i, p);
    }
  }
  if (__syncthreads_or(bad) && tid == 0) atomicOr(&nonfinite[gl.flag], 1u);
}

// ---- push form (N >= 4) ---------------------------------------------------
// hm_dp_push_grad: every rank STORES the gradient of the pages it does not
// own into the owner's receive pool (NVLink writes: no read requests on the
// reverse link, which the pull form pays on every 16 B it loads);
// hm_dp_onepass_recv_update, after a barrier, is onepass_kernel with every
// other rank's share read from the local receive pool.  Same rank-order f32
// sum, same bits.
constexpr int kPushThreads = 512;

constexpr int kPushPer = 4;   // chunks per CTA: their loads are all in flight before the remote stores

__global__ void __launch_bounds__(kPushThreads)
push_grad_kernel(const hm_seg_chunk* __restrict__ chunks, int n_chunks, const uint16_t* __restrict__ g16,
                 const uint64_t* __restrict__ recv_ptrs, uint64_t dst_base) {
  uint4 u[kPushPer];
  bool live[kPushPer];
  const uint32_t e = threadIdx.x * kVec;
#pragma unroll
  for (int k = 0; k < kPushPer; ++k) {
    const int i = blockIdx.x * kPushPer + k;
    live[k] = false;
    if (i >= n_chunks) continue;
    const hm_seg_chunk c = chunks[i];
    const uint16_t* src = g16 + c.src_off;
    const uint16_t* dst = reinterpret_cast<const uint16_t*>(recv_ptrs[c.slot]) + dst_base + c.dst_off;
    const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0 &&
                     (c.n & (kVec - 1)) == 0;
    if (vec) {
      live[k] = e < c.n;
      if (live[k]) u[k] = ld_stream_u4(src + e);
    } else {   // segment head / tail: element copies
      uint16_t* d = const_cast<uint16_t*>(dst);
      for (uint32_t j = threadIdx.x; j < c.n; j += kPushThreads) d[j] = src[j];
    }
  }
#pragma unroll
  for (int k = 0; k < kPushPer; ++k) {
    if (!live[k]) continue;
    const hm_seg_chunk c = chunks[blockIdx.x * kPushPer + k];
    st_stream_u4(reinterpret_cast<uint16_t*>(recv_ptrs[c.slot]) + dst_base + c.dst_off + e, u[k]);
  }
}

template <int DT, int NP, int NT>
__global__ void __launch_bounds__(NT, (NP <= 2 || (NP <= 4 && DT == HM_DT_BF16)) ? 2 : 1)
onepass_recv_kernel(const hm_adam_chunk* __restrict__ chunks, const hm_group_launch* __restrict__ groups,
                    const hm_group_rt* __restrict__ rt, const uint32_t* __restrict__ state_sel, uint64_t es,
                    const void* __restrict__ gself, const void* __restrict__ recv, uint64_t slot_elems, int self_q,
                    int n_ranks, PeerPtrs ppeers, float* __restrict__ p32, float* __restrict__ m32,
                    float* __restrict__ v32, uint32_t* __restrict__ nonfinite, hm_adam_hyper hyper) {
  using T = typename Elem<DT>::T;
  const hm_adam_chunk c = chunks[blockIdx.x];
  const hm_group_launch gl = groups[c.slot];
  const hm_group_rt r = rt[c.slot];
  const uint32_t sel = state_sel[gl.group];
  const uint64_t go = c.g_off + gl.g_shift, po = c.p_off + gl.p_shift;
  const uint64_t sr = c.s_off + (uint64_t)sel * es, sw = c.s_off + (uint64_t)(sel ^ 1u) * es;
  const uint32_t n = c.n;
  const int tid = threadIdx.x;
  const AdamScalars s = make_scalars(hyper, r);
  // rank q's share: this rank's own gradient page, or q's slot of the receive pool
  const T* own = static_cast<const T*>(gself) + go;
  const T* rb = static_cast<const T*>(recv) + c.s_off;
  bool bad = false;
  const bool vec = ((go | sr | sw | po | c.s_off | slot_elems | (uint64_t)n) & (kVec - 1)) == 0 &&
                   vec_base<HM_DT_F32>(p32) && vec_base<HM_DT_F32>(m32) && vec_base<HM_DT_F32>(v32) &&
                   vec_base<DT>(gself) && vec_base<DT>(recv);
  if (vec) {
    constexpr int VPT = kChunk / (NT * kVec);
    uint4 graw[VPT][NP];
    F8 pv[VPT], mv[VPT], vv[VPT];
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const uint32_t e = (uint32_t)(k * NT + tid) * kVec;
      if (e >= n) continue;
      const T* sp = rb + e;
#pragma unroll
      for (int q = 0; q < NP; ++q, sp += slot_elems)
        if (q < n_ranks) graw[k][q] = ld_stream_u4(q == self_q ? own + e : sp);
      load8_rw<HM_DT_F32>(p32, sr + e, pv[k]);
      load8_rw<HM_DT_F32>(m32, sr + e, mv[k]);
      load8_rw<HM_DT_F32>(v32, sr + e, vv[k]);
    }
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const uint32_t e = (uint32_t)(k * NT + tid) * kVec;
      if (e >= n) continue;
      float acc[kVec];
#pragma unroll
      for (int j = 0; j < kVec; ++j) acc[j] = 0.f;
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        if (q >= n_ranks) break;
        const T* h = reinterpret_cast<const T*>(&graw[k][q]);
#pragma unroll
        for (int j = 0; j < kVec; ++j) acc[j] = __fadd_rn(acc[j], Elem<DT>::widen(h[j]));
      }
      uint4 u;
      T* hp = reinterpret_cast<T*>(&u);
#pragma unroll
      for (int j = 0; j < kVec; ++j) {
        const float g = Elem<DT>::widen(Elem<DT>::narrow(acc[j]));
        bad |= !is_finite(g);
        adam_elem(s, g, pv[k].v[j], mv[k].v[j], vv[k].v[j]);
        hp[j] = Elem<DT>::narrow(pv[k].v[j]);
      }
      store8<HM_DT_F32>(p32, sw + e, pv[k]);
      store8<HM_DT_F32>(m32, sw + e, mv[k]);
      store8<HM_DT_F32>(v32, sw + e, vv[k]);
#pragma unroll
      for (int q = 0; q < kMaxPeers; ++q)
        if (q < ppeers.n) st_stream_u4(reinterpret_cast<T*>(ppeers.p[q]) + po + e, u);
    }
  } else {
    for (uint32_t i = tid; i < n; i += NT) {
      float a = 0.f;
      const T* sp = rb + i;
#pragma unroll
      for (int q = 0; q < NP; ++q, sp += slot_elems)
        if (q < n_ranks) a = __fadd_rn(a, Elem<DT>::widen(q == self_q ? own[i] : *sp));
      const float g = Elem<DT>::widen(Elem<DT>::narrow(a));
      bad |= !is_finite(g);
      float p = p32[sr + i], m = m32[sr + i], v = v32[sr + i];
      adam_elem(s, g, p, m, v);
      p32[sw + i] = p;
      m32[sw + i] = m;
      v32[sw + i] = v;
#pragma unroll
      for (int q = 0; q < kMaxPeers; ++q)
        if (q < ppeers.n) store1<DT>(reinterpret_cast<void*>(ppeers.p[q]), po + i, p);
    }
  }
  if (__syncthreads_or(bad) && tid == 0) atomicOr(&nonfinite[gl.flag], 1u);
}

using OnepassRecvFn = void (*)(const hm_adam_chunk*, const hm_group_launch*, const hm_group_rt*, const uint32_t*,
                               uint64_t, const void*, const void*, uint64_t, int, int, PeerPtrs, float*, float*,
                               float*, uint32_t*, hm_adam_hyper);

template <int DT>
OnepassRecvFn pick_onepass_recv_dt(int n) {
  return n <= 2 ? onepass_recv_kernel<DT, 2, 512> : n <= 4 ? onepass_recv_kernel<DT, 4, 512>
                                                            : onepass_recv_kernel<DT, 8, 512>;
}

__global__ void onepass_finalize_kernel(PeerPtrs flag_peers, int n_layers, int32_t* __restrict__ steps,
                                        const int32_t* __restrict__ steps_spec,
                                        uint32_t* __restrict__ state_sel, uint32_t* __restrict__ applied,
                                        double* __restrict__ ledger_out) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < n_layers; l += gridDim.x * blockDim.x) {
    uint32_t f = 0;
#pragma unroll
    for (int q = 0; q < kMaxPeers; ++q)   // constant indices: no local-memory copy of the peer table
      if (q < flag_peers.n) f |= reinterpret_cast<const volatile uint32_t*>(flag_peers.p[q])[l];
    const bool finite = f == 0;
    if (finite) {
      steps[l] = steps_spec[l];
      state_sel[l] ^= 1u;
    }
    if (applied) applied[l] = finite ? 1u : 0u;
    if (ledger_out) ledger_out[2 * l + 1] = finite ? 1.0 : 0.0;
  }
}

template <int DT>
__global__ void __launch_bounds__(kThreads)
republish_kernel(const hm_adam_chunk* __restrict__ chunks, int n_chunks,
                 const hm_group_launch* __restrict__ groups, const uint32_t* __restrict__ applied,
                 const uint32_t* __restrict__ state_sel, uint64_t es, const float* __restrict__ p32,
                 PeerPtrs ppeers) {
  // a persistent grid striding over the chunks: the common case (nothing
  // rejected) is one descriptor + one flag read per chunk, not one CTA each
  for (int k = blockIdx.x; k < n_chunks; k += gridDim.x) {
    const hm_adam_chunk c = chunks[k];
    const hm_group_launch gl = groups[c.slot];
    if (applied[gl.group]) continue;   // uniform per chunk
    const uint64_t sr = c.s_off + (uint64_t)state_sel[gl.group] * es, po = c.p_off + gl.p_shift;
    for (uint32_t i = threadIdx.x; i < c.n; i += kThreads) {
      const float p = p32[sr + i];
#pragma unroll
      for (int q = 0; q < kMaxPeers; ++q)
        if (q < ppeers.n) store1<DT>(reinterpret_cast<void*>(ppeers.p[q]), po + i, p);
    }
  }
}

using OnepassFn = void (*)(const hm_adam_chunk*, const hm_group_launch*, const hm_group_rt*, const uint32_t*,
                           uint64_t, PeerPtrs, PeerPtrs, float*, float*, float*, uint32_t*, hm_adam_hyper);

template <int DT>
OnepassFn pick_onepass_dt(int n, int* threads) {
  *threads = 512;
  return n <= 2 ? onepass_kernel<DT, 2, 512> : n <= 4 ? onepass_kernel<DT, 4, 512> : onepass_kernel<DT, 8, 512>;
}

}  // namespace
}  // namespace hm

extern "C" {

int hm_dp_onepass_update(const hm_adam_chunk* chunks, int64_t n_chunks, const hm_group_launch* groups,
                         const hm_group_rt* rt, const uint32_t* state_sel, int64_t state_elems,
                         const uint64_t* peer_g16, const uint64_t* peer_p16, int n_peers, int dtype,
                         float* p32, float* m32, float* v32, uint32_t* nonfinite,
                         const hm_adam_hyper* hyper, const hm_launch_opts* opts, void* stream) {
  if (!hyper || !rt) return hm_set_error(HM_ERR_INVALID, "hm_dp_onepass_update: missing hyper/rt");
  hm::PeerPtrs gp, pp;
  if (int rc = hm::make_peers(peer_g16, n_peers, &gp)) return rc;
  if (int rc = hm::make_peers(peer_p16, n_peers, &pp)) return rc;
  if (n_chunks < 0 || n_chunks > 0x7fffffffLL || state_elems < 0)
    return hm_set_error(HM_ERR_INVALID, "hm_dp_onepass_update: bad chunk count / state size");
  int threads = 256;
  // opts.reduce_width: minimum peer-array width (8 runs the N=8 instantiation on a smaller box)
  const int width = opts && opts->reduce_width > n_peers ? opts->reduce_width : n_peers;
  if (width > hm::kMaxPeers)
    return hm_set_error(HM_ERR_INVALID, "hm_dp_onepass_update: width %d > %d", width, hm::kMaxPeers);
  hm::OnepassFn fn = dtype == HM_DT_BF16 ? hm::pick_onepass_dt<HM_DT_BF16>(width, &threads)
                   : dtype == HM_DT_F16 ? hm::pick_onepass_dt<HM_DT_F16>(width, &threads) : nullptr;
  if (!fn) return hm_set_error(HM_ERR_INVALID, "hm_dp_onepass_update: unsupported dtype %d", dtype);
  if (n_chunks == 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_dp_onepass_update", chunks, groups, state_sel, p32, m32, v32, nonfinite);
  fn<<<(unsigned)n_chunks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
      chunks, groups, rt, state_sel, (uint64_t)state_elems, gp, pp, p32, m32, v32, nonfinite, *hyper);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

int hm_dp_push_grad(const hm_seg_chunk* chunks, int64_t n_chunks, const void* g16_local,
                    const uint64_t* recv_ptrs, int64_t dst_base, void* stream) {
  if (n_chunks < 0 || n_chunks > 0x7fffffffLL || dst_base < 0)
    return hm_set_error(HM_ERR_INVALID, "hm_dp_push_grad: bad chunk count / base");
  if (n_chunks == 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_dp_push_grad", chunks, g16_local, recv_ptrs);
  const unsigned grid = (unsigned)((n_chunks + hm::kPushPer - 1) / hm::kPushPer);
  hm::push_grad_kernel<<<grid, hm::kPushThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      chunks, (int)n_chunks, static_cast<const uint16_t*>(g16_local), recv_ptrs, (uint64_t)dst_base);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

int hm_dp_onepass_recv_update(const hm_adam_chunk* chunks, int64_t n_chunks, const hm_group_launch* groups,
                              const hm_group_rt* rt, const uint32_t* state_sel, int64_t state_elems,
                              const void* g16_local, const void* recv_local, int64_t slot_elems, int self_rank,
                              int n_ranks, const uint64_t* peer_p16, int n_peers, int dtype, float* p32,
                              float* m32, float* v32, uint32_t* nonfinite, const hm_adam_hyper* hyper,
                              void* stream) {
  if (!hyper || !rt) return hm_set_error(HM_ERR_INVALID, "hm_dp_onepass_recv_update: missing hyper/rt");
  hm::PeerPtrs pp;
  if (int rc = hm::make_peers(peer_p16, n_peers, &pp)) return rc;
  if (n_chunks < 0 || n_chunks > 0x7fffffffLL || state_elems < 0 || slot_elems < 0)
    return hm_set_error(HM_ERR_INVALID, "hm_dp_onepass_recv_update: bad chunk count / sizes");
  if (n_ranks < 1 || n_ranks > hm::kMaxPeers || self_rank < 0 || self_rank >= n_ranks)
    return hm_set_error(HM_ERR_INVALID, "hm_dp_onepass_recv_update: rank %d of %d", self_rank, n_ranks);
  hm::OnepassRecvFn fn = dtype == HM_DT_BF16 ? hm::pick_onepass_recv_dt<HM_DT_BF16>(n_ranks)
                       : dtype == HM_DT_F16 ? hm::pick_onepass_recv_dt<HM_DT_F16>(n_ranks) : nullptr;
  if (!fn) return hm_set_error(HM_ERR_INVALID, "hm_dp_onepass_recv_update: unsupported dtype %d", dtype);
  if (n_chunks == 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_dp_onepass_recv_update", chunks, groups, state_sel, g16_local, recv_local, p32, m32, v32,
                  nonfinite);
  fn<<<(unsigned)n_chunks, 512, 0, static_cast<cudaStream_t>(stream)>>>(
      chunks, groups, rt, state_sel, (uint64_t)state_elems, g16_local, recv_local, (uint64_t)slot_elems, self_rank,
      n_ranks, pp, p32, m32, v32, nonfinite, *hyper);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

int hm_dp_onepass_finalize(const uint64_t* peer_flags, int n_peers, int n_layers, int32_t* steps,
                           const int32_t* steps_spec, uint32_t* state_sel, uint32_t* applied,
                           double* ledger_out, void* stream) {
  hm::PeerPtrs f;
  if (int rc = hm::make_peers(peer_flags, n_peers, &f, 4)) return rc;
  if (n_layers <= 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_dp_onepass_finalize", steps, steps_spec, state_sel);
  const int blocks = (n_layers + 255) / 256;
  hm::onepass_finalize_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      f, n_layers, steps, steps_spec, state_sel, applied, ledger_out);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

int hm_dp_republish_rejected(const hm_adam_chunk* chunks, int64_t n_chunks, const hm_group_launch* groups,
                             const uint32_t* applied, const uint32_t* state_sel, int64_t state_elems,
                             const float* p32, const uint64_t* peer_p16, int n_peers, int dtype,
                             void* stream) {
  hm::PeerPtrs pp;
  if (int rc = hm::make_peers(peer_p16, n_peers, &pp)) return rc;
  if (n_chunks < 0 || n_chunks > 0x7fffffffLL)
    return hm_set_error(HM_ERR_INVALID, "hm_dp_republish_rejected: bad chunk count");
  if (dtype != HM_DT_BF16 && dtype != HM_DT_F16)
    return hm_set_error(HM_ERR_INVALID, "hm_dp_republish_rejected: unsupported dtype %d", dtype);
  if (n_chunks == 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_dp_republish_rejected", chunks, groups, applied, state_sel, p32);
  auto fn = dtype == HM_DT_BF16 ? hm::republish_kernel<HM_DT_BF16> : hm::republish_kernel<HM_DT_F16>;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = n_chunks < 8 * sms ? n_chunks : 8 * sms;   // 8 resident CTAs per SM
  fn<<<(unsigned)grid, hm::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      chunks, (int)n_chunks, groups, applied, state_sel, (uint64_t)state_elems, p32, pp);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

}  // extern "C"
