// Data-parallel page collectives fused with their compute, over NVLink /
// NVSwitch peer memory (symmetric buffers mapped into every rank).
//
//   hm_dp_reduce_check   gradient reduce-scatter of the owned pages fused with
//                        the layer's finite flag and squared norm (K6 + K3):
//                        each owner reads its pages from every peer (P2P
//                        loads, summed in f32 in rank order 0..N-1 and rounded
//                        once — deterministic), or asks the switch for the sum
//                        (NVLS multimem.ld_reduce, inbound S/N bytes per rank).
//   hm_dp_flags_merge    OR of the per-layer flags / sum of the norms over
//                        peers (replaces an all-reduce of a few hundred words).
//   hm_adam_main_ag      (page_adam.cu) page-Adam whose publish epilogue writes
//                        the 16-bit pages into every peer's pool (P2P stores or
//                        one NVLS multimem.st): the all-gather (K7) fused into
//                        the update, tile by tile.
//
// The reference only models these transfers (hiermem/simengine.py:255-257,
// all_gather = lat + page*(N-1)/N / bw) and has no reduce-scatter
// (SPEC.md:348); ownership is hiermem/scheduler.py:72-76 (page % N).
#include <atomic>

#include "hm_device.cuh"
#include "hm_dp.cuh"
#include "hm_error.h"

namespace hm {
namespace {

__device__ __forceinline__ uint4 ld_peer_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

template <int DT>
__device__ __forceinline__ uint4 ld_reduce_mc(const void* p);

template <>
__device__ __forceinline__ uint4 ld_reduce_mc<HM_DT_BF16>(const void* p) {
  uint4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
template <>
__device__ __forceinline__ uint4 ld_reduce_mc<HM_DT_F16>(const void* p) {
  uint4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.f16x2 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}

__device__ __forceinline__ void flush(bool bad, float sq, uint32_t* nonfinite, double* sumsq,
                                      uint32_t slot) {
  __shared__ float s_sq[kThreads / 32];
  __shared__ int s_bad[kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  const int any = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    s_sq[warp] = sq;
    s_bad[warp] = any;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    int b = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      t += s_sq[w];
      b |= s_bad[w];
    }
    if (nonfinite && b) atomicOr(&nonfinite[slot], 1u);
    if (sumsq && t != 0.f) atomicAdd(&sumsq[slot], (double)t);
  }
  __syncthreads();   // s_sq / s_bad are reused by the CTA's next chunk
}

// M owned chunks per CTA pass; chunk offsets are pool element offsets.
// NP = peer count rounded up to 2/4/8, so the in-flight load array is sized
// to the world.  Every remote load of the pass (chunks x granules x peers) is
// issued before any of them is consumed: NVLink latency (~2 us) needs the
// depth, and M > 1 deepens it for a small persistent grid.
template <int DT, bool MC, int NP, int M>
__device__ __forceinline__ void reduce_chunks(const hm_seg_chunk* __restrict__ chunks, int first,
                                              int n_chunks, const PeerPtrs& peers, const char* mc,
                                              void* __restrict__ local,
                                              uint32_t* __restrict__ nonfinite,
                                              double* __restrict__ sumsq) {
  using T = typename Elem<DT>::T;
  const int tid = threadIdx.x;
  hm_seg_chunk c[M];
  bool vec[M];
  uint4 u[M][kVecPerThread][MC ? 1 : NP];
#pragma unroll
  for (int m = 0; m < M; ++m) {
    if (first + m < n_chunks) {
      c[m] = chunks[first + m];
    } else {
      c[m].src_off = 0;
      c[m].n = 0;
      c[m].slot = 0;
    }
    vec[m] = ((c[m].src_off | (uint64_t)c[m].n) & (kVec - 1)) == 0 && vec_base<DT>(local) &&
             (MC ? vec_base<DT>(mc) : true);   // peer bases: checked by make_peers
  }
#pragma unroll
  for (int m = 0; m < M; ++m) {
    if (!vec[m]) continue;
#pragma unroll
    for (int k = 0; k < kVecPerThread; ++k) {
      const uint32_t e = (uint32_t)(k * kThreads + tid) * kVec;
      if (e >= c[m].n) continue;
      if constexpr (MC) {
        u[m][k][0] = ld_reduce_mc<DT>(mc + (c[m].src_off + e) * sizeof(T));
      } else {
#pragma unroll
        for (int r = 0; r < NP; ++r)
          if (r < peers.n)
            u[m][k][r] = ld_peer_u4(reinterpret_cast<const T*>(peers.p[r]) + c[m].src_off + e);
      }
    }
  }
#pragma unroll
  for (int m = 0; m < M; ++m) {
    if (c[m].n == 0) continue;   // uniform over the CTA
    const uint64_t off = c[m].src_off;
    bool bad = false;
    float sq = 0.f;
    if (vec[m]) {
#pragma unroll
      for (int k = 0; k < kVecPerThread; ++k) {
        const uint32_t e = (uint32_t)(k * kThreads + tid) * kVec;
        if (e >= c[m].n) continue;
        F8 acc;
        if constexpr (MC) {
          const T* h = reinterpret_cast<const T*>(&u[m][k][0]);
#pragma unroll
          for (int j = 0; j < kVec; ++j) acc.v[j] = Elem<DT>::widen(h[j]);
        } else {
#pragma unroll
          for (int j = 0; j < kVec; ++j) acc.v[j] = 0.f;
#pragma unroll
          for (int r = 0; r < NP; ++r) {
            if (r >= peers.n) break;
            const T* h = reinterpret_cast<const T*>(&u[m][k][r]);
#pragma unroll
            for (int j = 0; j < kVec; ++j) acc.v[j] = __fadd_rn(acc.v[j], Elem<DT>::widen(h[j]));
          }
        }
        F8 o;
#pragma unroll
        for (int j = 0; j < kVec; ++j) {
          const float r = Elem<DT>::widen(Elem<DT>::narrow(acc.v[j]));
          bad |= !is_finite(r);
          sq += __fmul_rn(r, r);
          o.v[j] = r;
        }
        store8<DT>(local, off + e, o);
      }
    } else {
      for (uint32_t i = tid; i < c[m].n; i += kThreads) {
        float a = 0.f;
#pragma unroll
        for (int r = 0; r < NP; ++r)
          if (r < peers.n)
            a = __fadd_rn(a, Elem<DT>::widen(reinterpret_cast<const T*>(peers.p[r])[off + i]));
        const float r = Elem<DT>::widen(Elem<DT>::narrow(a));
        bad |= !is_finite(r);
        sq += __fmul_rn(r, r);
        store1<DT>(local, off + i, r);
      }
    }
    flush(bad, sq, nonfinite, sumsq, c[m].slot);
  }
}

// One CTA per chunk (M = 1, grid = n_chunks), or a persistent grid striding
// over the chunks M at a time: a small resident grid (hm_set_dp_reduce_ctas)
// keeps the NVLink pipe full from a few SMs and leaves the rest to the
// page-Adam kernel of the previous layer group running concurrently
// (FusedShardedPageStep.step_pipelined).
template <int DT, bool MC, int NP, int M>
__global__ void __launch_bounds__(kThreads)
reduce_check_kernel(const hm_seg_chunk* __restrict__ chunks, int n_chunks, PeerPtrs peers,
                    const char* mc, void* __restrict__ local, uint32_t* __restrict__ nonfinite,
                    double* __restrict__ sumsq) {
  for (int i = blockIdx.x * M; i < n_chunks; i += gridDim.x * M)
    reduce_chunks<DT, MC, NP, M>(chunks, i, n_chunks, peers, mc, local, nonfinite, sumsq);
}

// 256-bit peer loads: each thread pulls 16 contiguous elements (32 B) from
// every peer in one access instead of two 16 B ones (hm_set_dp_reduce_wide,
// on by default).  Same rank-order f32 sum, so the same bits; chunks not
// 32 B aligned fall back to the 16 B path.  The payload on the link is the
// same, but the read requests going the other way shrink by a quarter (ncu:
// 494 -> 370 MB per GPU for C2 at N=4), and in the full step both directions
// are busy: the reduce gets 4-5% faster (profiles/r1_nvlink_ncu.md).
__device__ __forceinline__ void ld_peer_u8(const void* p, uint32_t (&u)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]),
                 "=r"(u[6]), "=r"(u[7])
               : "l"(p));
}

template <int DT, int NP>
__global__ void __launch_bounds__(kThreads)
reduce_check_wide_kernel(const hm_seg_chunk* __restrict__ chunks, int n_chunks, PeerPtrs peers,
                         const char* mc, void* __restrict__ local, uint32_t* __restrict__ nonfinite,
                         double* __restrict__ sumsq) {
  using T = typename Elem<DT>::T;
  static_assert(kChunk == kThreads * 16, "16 elements per thread");
  const hm_seg_chunk c = chunks[blockIdx.x];
  const uint64_t off = c.src_off;
  bool wide_ok = ((uintptr_t)local & 31u) == 0;
#pragma unroll
  for (int r = 0; r < NP; ++r)
    if (r < peers.n) wide_ok &= (peers.p[r] & 31u) == 0;
  if (((off | (uint64_t)c.n) & 15) != 0 || !wide_ok) {
    reduce_chunks<DT, false, NP, 1>(chunks, blockIdx.x, n_chunks, peers, mc, local, nonfinite, sumsq);
    return;
  }
  const uint32_t e = (uint32_t)threadIdx.x * 16;
  bool bad = false;
  float sq = 0.f;
  if (e < c.n) {
    uint32_t u[NP][8];
#pragma unroll
    for (int r = 0; r < NP; ++r)
      if (r < peers.n) ld_peer_u8(reinterpret_cast<const T*>(peers.p[r]) + off + e, u[r]);
    float acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.f;
#pragma unroll
    for (int r = 0; r < NP; ++r) {
      if (r >= peers.n) break;
      const T* h = reinterpret_cast<const T*>(u[r]);
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = __fadd_rn(acc[j], Elem<DT>::widen(h[j]));
    }
    F8 o0, o1;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float x = Elem<DT>::widen(Elem<DT>::narrow(acc[j]));
      bad |= !is_finite(x);
      sq += __fmul_rn(x, x);
      if (j < 8) o0.v[j] = x; else o1.v[j - 8] = x;
    }
    store8<DT>(local, off + e, o0);
    store8<DT>(local, off + e + 8, o1);
  }
  flush(bad, sq, nonfinite, sumsq, c.slot);
}

__global__ void flags_merge_kernel(PeerPtrs flag_peers, PeerPtrs sumsq_peers, int n,
                                   uint32_t* __restrict__ flags_out, double* __restrict__ sumsq_out) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < n; l += gridDim.x * blockDim.x) {
    uint32_t f = 0;
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < kMaxPeers; ++r) {   // constant indices: no local-memory copy of the peer table
      if (r >= flag_peers.n) break;
      f |= reinterpret_cast<const volatile uint32_t*>(flag_peers.p[r])[l];
      if (sumsq_out) s += reinterpret_cast<const volatile double*>(sumsq_peers.p[r])[l];
    }
    flags_out[l] = f;
    if (sumsq_out) sumsq_out[l] = s;
  }
}

using RcFn = void (*)(const hm_seg_chunk*, int, PeerPtrs, const char*, void*, uint32_t*, double*);

// Process-wide defaults; each launch's hm_launch_opts overrides them.
std::atomic<int> g_reduce_ctas{0};   // 0: one CTA per chunk; >0: persistent grid (hm_set_dp_reduce_ctas)
std::atomic<int> g_reduce_width{0};  // minimum peer-array width of the reduce kernel (test hook)
std::atomic<int> g_reduce_wide{1};   // 1: 256-bit peer loads (hm_set_dp_reduce_wide), the default

RcFn pick_rc_wide(int dt, int n) {
  if (dt == HM_DT_BF16)
    return n <= 2 ? reduce_check_wide_kernel<HM_DT_BF16, 2>
                  : n <= 4 ? reduce_check_wide_kernel<HM_DT_BF16, 4> : reduce_check_wide_kernel<HM_DT_BF16, 8>;
  if (dt == HM_DT_F16)
    return n <= 2 ? reduce_check_wide_kernel<HM_DT_F16, 2>
                  : n <= 4 ? reduce_check_wide_kernel<HM_DT_F16, 4> : reduce_check_wide_kernel<HM_DT_F16, 8>;
  return nullptr;
}

// Chunks per pass of the persistent grid: as deep as the registers allow.
template <int NP>
constexpr int persistent_depth() { return NP <= 2 ? 4 : NP <= 4 ? 2 : 1; }

template <int DT, int NP>
RcFn pick_rc_np(bool persistent) {
  return persistent ? reduce_check_kernel<DT, false, NP, persistent_depth<NP>()>
                    : reduce_check_kernel<DT, false, NP, 1>;
}

// Multicast reduce as a persistent grid: one in-switch load per granule and
// chunk, so a CTA can keep more chunks in flight than the P2P form at the
// same register cost (the layer-group pipeline gives it a few SMs only).
constexpr int kMcDepth = 4;

template <int DT>
RcFn pick_rc_dt(bool mc, int n, bool persistent) {
  // multicast: one in-switch load per granule; NP still bounds the P2P loads of
  // the unaligned head/tail chunks, which are summed peer by peer
  if (mc) return persistent ? reduce_check_kernel<DT, true, kMaxPeers, kMcDepth>
                            : reduce_check_kernel<DT, true, kMaxPeers, 1>;
  if (n <= 2) return pick_rc_np<DT, 2>(persistent);
  if (n <= 4) return pick_rc_np<DT, 4>(persistent);
  return pick_rc_np<DT, 8>(persistent);
}

RcFn pick_rc(int dt, bool mc, int n, bool persistent, int* depth) {
  *depth = !persistent ? 1 : mc ? kMcDepth : n <= 2 ? persistent_depth<2>() : n <= 4 ? persistent_depth<4>()
                                                                                      : persistent_depth<8>();
  if (dt == HM_DT_BF16) return pick_rc_dt<HM_DT_BF16>(mc, n, persistent);
  if (dt == HM_DT_F16) return pick_rc_dt<HM_DT_F16>(mc, n, persistent);
  return nullptr;
}

}  // namespace

int make_peers(const uint64_t* ptrs, int n, PeerPtrs* out, unsigned align) {
  if (n < 1 || n > kMaxPeers || !ptrs)
    return hm_set_error(HM_ERR_INVALID, "peer count %d outside 1..%d", n, kMaxPeers);
  out->n = n;
  for (int i = 0; i < kMaxPeers; ++i) {
    out->p[i] = i < n ? ptrs[i] : 0;
    // peer pools are symmetric allocations (page aligned); the 16 B vector
    // loads/stores to them assume at least that (flag / norm arrays: their
    // element size)
    if (i < n && (ptrs[i] & (align - 1)) != 0)
      return hm_set_error(HM_ERR_INVALID, "peer buffer %d at %#llx is not %u-byte aligned", i,
                          (unsigned long long)ptrs[i], align);
  }
  return HM_OK;
}

}  // namespace hm

extern "C" {

int hm_dp_reduce_check(const uint64_t* peer_pools, int n_peers, const void* mc_pool,
                       void* local_pool, int dtype, const hm_seg_chunk* chunks, int64_t n_chunks,
                       uint32_t* nonfinite, double* sumsq, const hm_launch_opts* opts, void* stream) {
  hm::PeerPtrs peers;
  if (int rc = hm::make_peers(peer_pools, n_peers, &peers)) return rc;
  if (n_chunks < 0 || n_chunks > 0x7fffffffLL)
    return hm_set_error(HM_ERR_INVALID, "hm_dp_reduce_check: bad chunk count");
  if (n_chunks == 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_dp_reduce_check", local_pool, chunks);
  // per-launch settings (opts field >= 0), else the process defaults
  const int rctas = opts && opts->grid_ctas >= 0 ? opts->grid_ctas
                                                 : hm::g_reduce_ctas.load(std::memory_order_relaxed);
  const int minw = opts && opts->reduce_width >= 0 ? opts->reduce_width
                                                   : hm::g_reduce_width.load(std::memory_order_relaxed);
  const int wide = opts && opts->reduce_wide >= 0 ? opts->reduce_wide
                                                  : hm::g_reduce_wide.load(std::memory_order_relaxed);
  if (minw > hm::kMaxPeers)
    return hm_set_error(HM_ERR_INVALID, "hm_dp_reduce_check: width %d > %d", minw, hm::kMaxPeers);
  const bool persistent = rctas > 0;
  int depth = 1;
  // template width: the peer count rounded up to 2/4/8, or wider if forced
  // (reduce_width: runs the 8-wide kernel on a 2- or 4-GPU box)
  const int width = n_peers > minw ? n_peers : minw;
  hm::RcFn fn = hm::pick_rc(dtype, mc_pool != nullptr, width, persistent, &depth);
  if (fn && !persistent && mc_pool == nullptr && wide) fn = hm::pick_rc_wide(dtype, width);
  if (!fn) return hm_set_error(HM_ERR_INVALID, "hm_dp_reduce_check: unsupported dtype %d", dtype);
  const int64_t passes = (n_chunks + depth - 1) / depth;
  const int64_t grid = persistent && rctas < passes ? rctas : passes;
  fn<<<(unsigned)grid, hm::kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      chunks, (int)n_chunks, peers, static_cast<const char*>(mc_pool), local_pool, nonfinite, sumsq);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

int hm_set_dp_reduce_width(int width) {
  if (width < 0 || width > hm::kMaxPeers)
    return hm_set_error(HM_ERR_INVALID, "hm_set_dp_reduce_width: 0..%d, got %d", hm::kMaxPeers, width);
  hm::g_reduce_width = width;
  return HM_OK;
}

int hm_set_dp_reduce_wide(int wide) {
  hm::g_reduce_wide = wide ? 1 : 0;
  return HM_OK;
}

int hm_set_dp_reduce_ctas(int ctas) {
  if (ctas < 0) return hm_set_error(HM_ERR_INVALID, "hm_set_dp_reduce_ctas: negative grid %d", ctas);
  hm::g_reduce_ctas = ctas;
  return HM_OK;
}

int hm_dp_flags_merge(const uint64_t* peer_flags, const uint64_t* peer_sumsq, int n_peers,
                      int n_layers, uint32_t* flags_out, double* sumsq_out, void* stream) {
  hm::PeerPtrs f, s;
  if (int rc = hm::make_peers(peer_flags, n_peers, &f, 4)) return rc;
  if (peer_sumsq) {
    if (int rc = hm::make_peers(peer_sumsq, n_peers, &s, 8)) return rc;
  } else {
    s = f;
    sumsq_out = nullptr;
  }
  if (n_layers <= 0) return HM_OK;
  HM_REQUIRE_PTRS("hm_dp_flags_merge", flags_out);
  const int blocks = (n_layers + 255) / 256;
  hm::flags_merge_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(f, s, n_layers,
                                                                                flags_out, sumsq_out);
  HM_CUDA_CHECK_LAUNCH();
  return HM_OK;
}

}  // extern "C"
