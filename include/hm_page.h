/*
 * hm_page.h — C-ABI of the B200-native page-granular update path
 * (Angel-PTM, arxiv 2303.02868; reference package `hiermem` 0.1.0).
 *
 * The reference is pure Python/numpy and has no FFI of its own: its
 * boundary is the Python API re-exported by hiermem/__init__.py:8-74.
 * Every entry point below replaces one reference operation (cited as
 * hiermem/<file>.py:<line>, i.e. /root/reference/pkg/src/hiermem/...).
 * The Python host package (paper_2303_02868_b200) binds these with ctypes;
 * INTEGRATION.md shows the binding a maintainer would add to `hiermem`.
 *
 * Conventions
 *  - extern "C", plain pointers and sizes, no torch/C++ types.
 *  - Every function returns an int status: HM_OK (0) or one of HM_ERR_*.
 *    The thread-local message is read with hm_last_error(); allocation
 *    failures also carry (requested_bytes, available_bytes) through
 *    hm_last_error_bytes(), mirroring hiermem/errors.py:8-14.
 *  - Device entry points are asynchronous on the caller's cudaStream_t
 *    (passed as void*), never allocate or free device memory, and never
 *    synchronise the device.  No CPU fallback exists.
 *  - Element offsets are in elements of the named buffer, byte offsets
 *    in bytes.  Kernels handle any alignment; 16/32-byte aligned runs
 *    take the 128/256-bit vector path.
 */
#ifndef HM_PAGE_H
#define HM_PAGE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map to hiermem/errors.py:4-39) ---------------------- */
#define HM_OK              0
#define HM_ERR_CONFIG      1   /* ConfigError      hiermem/errors.py:4     */
#define HM_ERR_ALLOCATION  2   /* AllocationError  hiermem/errors.py:8-14  */
#define HM_ERR_MOVE        3   /* MoveError        hiermem/errors.py:17    */
#define HM_ERR_PROTOCOL    4   /* ProtocolError    hiermem/errors.py:38    */
#define HM_ERR_KEY         5   /* KeyError (unknown page / tensor id)      */
#define HM_ERR_CUDA        6   /* CUDA runtime error (message has details) */
#define HM_ERR_INVALID     7   /* bad argument to the C-ABI itself         */

/* ---- element types ------------------------------------------------------ */
#define HM_DT_F16   1   /* IEEE binary16 (the reference's np.float16)        */
#define HM_DT_BF16  2   /* bfloat16 (north-star parameter/gradient type)     */
#define HM_DT_F32   3   /* binary32 master/moment type                       */

/* ---- tiers (hiermem/pagemem.py:29-32) and tensor kinds (footprint.py:22) */
#define HM_TIER_GPU 0
#define HM_TIER_CPU 1
#define HM_TIER_SSD 2
#define HM_KIND_PARAM16 0
#define HM_KIND_GRAD16  1
#define HM_KIND_OPTIM32 2
#define HM_KIND_ACT16   3

const char* hm_last_error(void);
void        hm_last_error_bytes(int64_t* requested_bytes, int64_t* available_bytes);
int         hm_abi_version(void);   /* bumped on any layout change below (2) */
int         hm_device_chunk_elems(void);  /* HM_ADAM_CHUNK, the kernel unit */

/* ======================================================================== *
 *  Host page table (replaces hiermem/pagemem.py:111-446, metadata only).   *
 *  One handle = one PageManager (hiermem/pagemem.py:188-229).  Reentrant   *
 *  per handle, not thread-safe per handle: callers serialise mutations,    *
 *  exactly the single-owner contract of hiermem/pagemem.py:11-12.          *
 * ======================================================================== */
typedef struct hm_pagetable hm_pagetable;

int hm_pt_create(hm_pagetable** out);
int hm_pt_destroy(hm_pagetable* pt);
/* TierPool.__init__ + PageManager.__init__ pool loop (pagemem.py:114-134,
 * 195-203).  first_page_id < 0 means "next free global id" (manager order). */
int hm_pt_add_pool(hm_pagetable* pt, int tier, int64_t capacity_bytes,
                   int64_t page_bytes, int64_t first_page_id);
/* PageManager.allocate (pagemem.py:233-283). */
int hm_pt_allocate(hm_pagetable* pt, int tier, int kind, int64_t bytes, int64_t* tensor_id);
/* PageManager.release (pagemem.py:285-299). */
int hm_pt_release(hm_pagetable* pt, int64_t tensor_id, int64_t* freed_bytes);
/* PageManager.page_move (pagemem.py:303-334); out = TransferDescriptor
 * {bytes, src_tier, dst_tier, page_id, new_page_id} (pagemem.py:102-108). */
int hm_pt_page_move(hm_pagetable* pt, int64_t page_id, int target_tier, int64_t out[5]);
/* PageManager.tensor_merge (pagemem.py:338-407).  out = {moved_chunks, first_page}. */
int hm_pt_tensor_merge(hm_pagetable* pt, int64_t tensor_id, int64_t out[2]);

/* Introspection (Page/ManagedTensor/TierPool/state_dict, pagemem.py:46-99,
 * 136-165, 411-446).  Array outputs return the element count; pass cap=0
 * to query the size. */
int     hm_pt_num_pools(const hm_pagetable* pt);
/* out = {tier, capacity_bytes, page_bytes, first_page_id, num_pages,
 *        free_pages, allocations, releases, moves_in, moves_out,
 *        peak_allocated_pages, occupied_bytes_of_allocated_pages} */
int     hm_pt_pool_info(const hm_pagetable* pt, int pool_index, int64_t out[12]);
int64_t hm_pt_allocated_pages(const hm_pagetable* pt, int tier, int64_t* out, int64_t cap);
int64_t hm_pt_free_pages(const hm_pagetable* pt, int tier, int64_t* out, int64_t cap);
/* out = {tier, total_bytes, n_occupants, then per occupant
 *        (tensor_id, bytes, shareable, byte_offset)}  (max 2 occupants) */
int     hm_pt_page_info(const hm_pagetable* pt, int64_t page_id, int64_t out[11]);
int64_t hm_pt_tensor_ids(const hm_pagetable* pt, int64_t* out, int64_t cap);
/* out = {kind, bytes, tier_or_-1 (NOT_READY), n_pages} */
int     hm_pt_tensor_info(const hm_pagetable* pt, int64_t tensor_id, int64_t out[4]);
int64_t hm_pt_tensor_pages(const hm_pagetable* pt, int64_t tensor_id, int64_t* out, int64_t cap);
/* The physical placement the reference leaves implicit: one triple
 * (page_id, byte_offset_in_page, bytes) per page of the tensor, in
 * tensor order.  Occupant slot 0 sits at offset 0, a second occupant is
 * end-aligned, so any legal pair never overlaps. */
int64_t hm_pt_tensor_segments(const hm_pagetable* pt, int64_t tensor_id, int64_t* out3, int64_t cap);

/* ======================================================================== *
 *  Device kernels (sm_100a).                                               *
 * ======================================================================== */
#define HM_ADAM_CHUNK 4096   /* elements per CTA work unit */

/* One unit of the fused page-Adam kernel: a run of <= HM_ADAM_CHUNK
 * elements of one segment (a tensor's share of one page). */
typedef struct hm_adam_chunk {
  uint64_t g_off;   /* element offset into the gradient source               */
  uint64_t s_off;   /* element offset into p32 / m32 / v32                   */
  uint64_t p_off;   /* element offset into the 16-bit parameter output       */
  uint32_t n;       /* element count                                         */
  uint32_t slot;    /* index into the launch's group table                   */
} hm_adam_chunk;

/* Per-launch, per-group record built by the host (one per MasterState
 * layer touched by the launch). */
typedef struct hm_group_launch {
  uint64_t g_shift;   /* added to g_off: selects the taken gradient buffer   */
  uint64_t p_shift;   /* added to p_off: selects the p16 publish buffer      */
  uint32_t group;     /* index into steps[] / applied[]                      */
  uint32_t flag;      /* index into nonfinite[] / sumsq[] of the gradient    */
} hm_group_launch;

/* Written by the prologue for the main kernel (device scratch, one per slot). */
typedef struct hm_group_rt {
  float    bc1;       /* f32(1 - beta1**step), host-double exact table       */
  float    bc2;       /* f32(1 - beta2**step)                                */
  float    gscale;    /* unscale x clip coefficient (1.0f: exact identity)   */
  uint32_t apply;     /* 0: layer rejected (hiermem/lockfree.py:133-134)     */
} hm_group_rt;

/* Scalars of AdamHyper (hiermem/lockfree.py:37-42) rounded to f32 exactly as
 * numpy's weak-scalar promotion does (lockfree.py:135-141). */
typedef struct hm_adam_hyper {
  float lr, beta1, one_minus_beta1, beta2, one_minus_beta2, eps;
  float inv_scale;    /* loss-scale unscale; 1.0f for reference parity       */
  float max_norm;     /* global grad-norm clip; <= 0 disables               */
} hm_adam_hyper;

/* Per-launch tuning (nullable; any field < 0 = the process default set by
 * the matching hm_set_* call).  Launch settings travel with the launch, so
 * two threads or streams with different settings never see each other's.
 *   adam_threads  256 | 512 threads per 4096-element chunk (page-Adam)
 *   adam_variant  0 LDG/STG streaming | 1 TMA bulk-copy pipeline
 *   grid_ctas     hm_adam_main_ag / hm_dp_reduce_check: persistent grid size
 *                 (0 = one CTA per chunk)
 *   ag_publish    0 per-thread peer stores | 1 (or 2) staged bulk copies
 *   reduce_width  minimum peer-array width of the reduce kernel (0, 2, 4, 8)
 *   reduce_wide   1 = 256-bit peer loads | 0 = 128-bit                      */
typedef struct hm_launch_opts {
  int32_t adam_threads, adam_variant, grid_ctas, ag_publish, reduce_width, reduce_wide;
} hm_launch_opts;

/* Fused take -> update -> publish over page segments: one HBM pass reading
 * g (16-bit or f32) + p32/m32/v32 and writing p32/m32/v32 + p16.
 *   hiermem/lockfree.py:127-142 (apply_update), :155-165 (update_layer with
 *   step rollback), :168-171 + :243-263 (publish cast), :226-241 (take).
 * The prologue consumes nonfinite[flag] (computed when the gradient was
 * produced: hm_accumulate / hm_reduce_stats), advances steps[group] only
 * for applied groups, writes applied[group], clears the consumed flag and
 * sumsq (and the ledger sum lsum[flag]) when consume_flags != 0, and
 * looks up bc1/bc2 in bc_table
 * (pairs, index = step; must cover every reachable step).
 * explicit_step > 0 selects the functional apply_update form: the step is
 * given, steps[] is neither read nor written, and bc_table[0] holds its
 * (bc1, bc2).  p16 == NULL skips the publish cast.
 * On a rejected group nothing is written to p32/m32/v32; if p16 != NULL
 * the unchanged p32 is still cast (the reference publishes after a reject,
 * hiermem/lockfree.py:631-638).
 * Ledger (nullable): ledger_out[2i] = lsum[flag of group i] (the taken
 * gradient's f64 sum, ConservationLedger.record_take, lockfree.py:237) and
 * ledger_out[2i+1] = 1.0 if group i was applied else 0.0 (record_apply,
 * lockfree.py:300), read before the consume resets lsum. */
int hm_adam_step(const hm_adam_chunk* chunks, int64_t n_chunks,
                 const hm_group_launch* groups, int32_t n_groups,
                 hm_group_rt* rt_scratch,
                 const void* g, int g_dtype,
                 float* p32, float* m32, float* v32,
                 void* p16, int p16_dtype,
                 const hm_adam_hyper* hyper,
                 const float* bc_table, int64_t bc_len, int64_t explicit_step,
                 int32_t* steps, uint32_t* applied,
                 uint32_t* nonfinite, double* sumsq, int consume_flags,
                 double* lsum, double* ledger_out, const hm_launch_opts* opts,
                 void* stream);

/* Process-wide DEFAULT of the page-Adam main kernel's threads per chunk: 256
 * (default) or 512 (2 or 1 granule of 8 elements per thread). */
int hm_set_adam_threads(int threads);
/* Process-wide DEFAULT data-movement variant of the page-Adam main pass (same
 * arithmetic, bytes and results): 0 = LDG/STG streaming kernel (default),
 * 1 = persistent TMA bulk-copy pipeline (cp.async.bulk + mbarrier). */
int hm_set_adam_variant(int variant);

/* The two halves of hm_adam_step, for callers that pipeline the main pass
 * (e.g. per all-gather bucket) after ONE prologue over every group: the
 * prologue must run exactly once per update or steps[] would advance twice. */
int hm_adam_prologue(const hm_group_launch* groups, int32_t n_groups, hm_group_rt* rt_scratch,
                     const hm_adam_hyper* hyper, const float* bc_table, int64_t bc_len,
                     int64_t explicit_step, int32_t* steps, uint32_t* applied,
                     uint32_t* nonfinite, double* sumsq, int consume_flags,
                     double* lsum, double* ledger_out, void* stream);
int hm_adam_main(const hm_adam_chunk* chunks, int64_t n_chunks, const hm_group_launch* groups,
                 const hm_group_rt* rt, const void* g, int g_dtype,
                 float* p32, float* m32, float* v32, void* p16, int p16_dtype,
                 const hm_adam_hyper* hyper, const hm_launch_opts* opts, void* stream);

/* MasterState.update_layer of ONE layer whose gradient is its taken 16-bit
 * page buffer (the three-call path, hiermem/lockfree.py:155-165 after
 * ParamBuffer.take :226-241), prologue fused: one launch.  group: ONE
 * hm_group_launch row (device).  Each CTA derives the layer's reject flag
 * (nonfinite[flag], nullable), step = steps[group] + 1, bias pair and clip
 * scale (sumsq[flag], nullable) itself; the last CTA to retire writes
 * steps[group] (applied only) and *applied.  done: a device word that is 0
 * between launches (the kernel re-arms it; one per stream).  p_out/out_off
 * (nullable, together): the new p32 of every chunk is also stored to
 * p_out[out_off[chunk] + i] — the layer as a contiguous tensor, so
 * MasterState.p32[layer] needs no unpack.  Requires n_chunks >= 1 and
 * 16-bit g16/p16 of the same dtype. */
int hm_adam_layer(const hm_adam_chunk* chunks, int64_t n_chunks, const hm_group_launch* group,
                  const void* g16, int dtype, float* p32, float* m32, float* v32, void* p16,
                  const hm_adam_hyper* hyper, const float* bc_table, int64_t bc_len,
                  int32_t* steps, uint32_t* applied, const uint32_t* nonfinite,
                  const double* sumsq, uint32_t* done, float* p_out, const uint64_t* out_off,
                  void* stream);

/* ---- data-parallel page collectives fused with compute (NVLink/NVSwitch) ---
 * Pools are symmetric buffers mapped into every rank (peer virtual addresses,
 * optionally one NVLS multicast address).  Ownership: page % N
 * (hiermem/scheduler.py:72-76); the reference models these transfers only
 * (hiermem/simengine.py:255-257) and has no reduce-scatter.
 * peer arrays are HOST arrays of n_peers (<= 8) device addresses in rank order. */
typedef struct hm_seg_chunk hm_seg_chunk;

/* Gradient reduce-scatter of the owned pages fused with the layer's finite
 * flag and squared norm: local[off] = rn16(sum_r peer_r[off]) in f32, rank
 * order 0..N-1 (P2P loads), or the switch's sum (mc_pool != NULL: NVLS
 * multimem.ld_reduce).  chunks: owned pool segments, slot = layer.
 * opts: grid_ctas (0 = one CTA per chunk; > 0 = a persistent grid striding
 * over the chunks, so the reduce of one layer group can share the SMs with
 * the page-Adam of the previous group), reduce_width, reduce_wide. */
int hm_dp_reduce_check(const uint64_t* peer_pools, int n_peers, const void* mc_pool,
                       void* local_pool, int dtype, const hm_seg_chunk* chunks, int64_t n_chunks,
                       uint32_t* nonfinite, double* sumsq, const hm_launch_opts* opts, void* stream);
/* Process-wide DEFAULTS of hm_launch_opts.grid_ctas / reduce_width /
 * reduce_wide for hm_dp_reduce_check: persistent grid (0 = one CTA per
 * chunk); minimum peer-array width (0 = the peer count rounded up to
 * 2/4/8; 8 exercises the N=8 instantiation on a 2- or 4-GPU box, same
 * results at every width); 1 (default) = 32 B per thread and peer (256-bit
 * loads; fewer read requests on the reverse link), 0 = 16 B loads. */
int hm_set_dp_reduce_ctas(int ctas);
int hm_set_dp_reduce_width(int width);
int hm_set_dp_reduce_wide(int wide);
/* flags_out[l] = OR_r peer_flags_r[l]; sumsq_out[l] = sum_r peer_sumsq_r[l]
 * (rank order).  Replaces an all-reduce of the per-layer reject flags. */
int hm_dp_flags_merge(const uint64_t* peer_flags, const uint64_t* peer_sumsq, int n_peers,
                      int n_layers, uint32_t* flags_out, double* sumsq_out, void* stream);
/* hm_adam_main whose publish epilogue writes each 16-bit page into every
 * peer's p16 pool (P2P stores) or once through the NVLS multicast address
 * (mc_p16 != NULL): the parameter all-gather fused into the update. */
int hm_adam_main_ag(const hm_adam_chunk* chunks, int64_t n_chunks, const hm_group_launch* groups,
                    const hm_group_rt* rt, const void* g, int g_dtype,
                    float* p32, float* m32, float* v32,
                    const uint64_t* peer_p16, int n_peers, void* mc_p16, int p16_dtype,
                    const hm_adam_hyper* hyper, const hm_launch_opts* opts, void* stream);
/* The DP page step as ONE pass (round 2; state double-buffered per layer):
 * per owned chunk, pull the chunk's 16-bit gradient from every rank's pool
 * (peer_g16: every rank's gradient pool base in rank order, the caller's
 * own included; offsets = chunk g_off + group g_shift), sum in f32 in rank
 * order and round once (the bits of hm_dp_reduce_check), run the page-Adam
 * chain (hiermem/lockfree.py:135-141) on the layer's current state buffer
 * (state_sel[group] selects buffer 0 or 1 of each [2 x state_elems] pool)
 * and write the OTHER buffer, publish the new 16-bit page into every rank's
 * pool (peer_p16), and OR the layer's non-finite flag into nonfinite[flag].
 * Speculative: the prologue must have run on a copy of steps[], and
 * hm_dp_onepass_finalize commits after a cross-rank barrier.
 * opts.reduce_width: minimum peer-array width of the kernel (nullable). */
int hm_dp_onepass_update(const hm_adam_chunk* chunks, int64_t n_chunks, const hm_group_launch* groups,
                         const hm_group_rt* rt, const uint32_t* state_sel, int64_t state_elems,
                         const uint64_t* peer_g16, const uint64_t* peer_p16, int n_peers, int dtype,
                         float* p32, float* m32, float* v32, uint32_t* nonfinite,
                         const hm_adam_hyper* hyper, const hm_launch_opts* opts, void* stream);
/* Push form of the one-pass step's gradient exchange (N >= 4): every rank
 * stores the gradient of the pages it does NOT own into the owner's receive
 * pool (NVLink writes, no read requests).  chunks: src_off = element offset
 * in g16_local (this rank's active gradient buffer), dst_off = the page's
 * state-slot offset on its owner, slot = owner rank; recv_ptrs: DEVICE array
 * of every rank's receive-pool address; element dst_base (= rank x
 * slot_elems) selects this rank's slot there. */
int hm_dp_push_grad(const hm_seg_chunk* chunks, int64_t n_chunks, const void* g16_local,
                    const uint64_t* recv_ptrs, int64_t dst_base, void* stream);
/* hm_dp_onepass_update reading rank q's share of an owned chunk from
 * g16_local (q == self_rank, at the chunk's gradient offset) or from
 * recv_local + q x slot_elems + the chunk's state offset (after
 * hm_dp_push_grad and a barrier): same rank-order f32 sum, same bits. */
int hm_dp_onepass_recv_update(const hm_adam_chunk* chunks, int64_t n_chunks, const hm_group_launch* groups,
                              const hm_group_rt* rt, const uint32_t* state_sel, int64_t state_elems,
                              const void* g16_local, const void* recv_local, int64_t slot_elems, int self_rank,
                              int n_ranks, const uint64_t* peer_p16, int n_peers, int dtype, float* p32,
                              float* m32, float* v32, uint32_t* nonfinite, const hm_adam_hyper* hyper,
                              void* stream);
/* Commit of a one-pass step: per layer, flag = OR over the ranks' flags
 * (peer_flags); applied: steps[l] = steps_spec[l] and state_sel[l] flips;
 * rejected: both stay (hiermem/lockfree.py:133-134, 163-164).  applied[]
 * and the ledger row's applied column (ledger_out[2l+1]) are nullable. */
int hm_dp_onepass_finalize(const uint64_t* peer_flags, int n_peers, int n_layers, int32_t* steps,
                           const int32_t* steps_spec, uint32_t* state_sel, uint32_t* applied,
                           double* ledger_out, void* stream);
/* Publish the unchanged parameters of the owned pages of every REJECTED
 * layer again (the one-pass update published speculatively). */
int hm_dp_republish_rejected(const hm_adam_chunk* chunks, int64_t n_chunks, const hm_group_launch* groups,
                             const uint32_t* applied, const uint32_t* state_sel, int64_t state_elems,
                             const float* p32, const uint64_t* peer_p16, int n_peers, int dtype,
                             void* stream);
/* Process-wide DEFAULTS of hm_launch_opts.ag_publish / grid_ctas for
 * hm_adam_main_ag.  Publish epilogue over P2P: 0 = every thread stores its
 * 16 B granules into every peer (default); 1 (or 2) = the CTA stages its
 * 16-bit chunk in shared memory, one thread pushes it to every peer with
 * cp.async.bulk and waits for the remote writes before the CTA retires.
 * Grid (per-thread stores or multicast): 0 = one CTA per chunk; > 0 = a
 * persistent grid striding over the chunks. */
int hm_set_ag_publish(int mode);
int hm_set_dp_update_ctas(int ctas);

/* Elementwise segment chunk used by accumulate / cast / reduce. */
typedef struct hm_seg_chunk {
  uint64_t src_off;   /* element offset into src */
  uint64_t dst_off;   /* element offset into dst */
  uint32_t n;         /* element count (<= HM_ADAM_CHUNK) */
  uint32_t slot;      /* index into nonfinite[] / sumsq[] / sums[] */
} hm_seg_chunk;

/* ParamBuffer.accumulate (hiermem/lockfree.py:210-224):
 *   dst = rn_dst(f32(dst) + f32(src))   (mode 1: add)
 *   dst = rn_dst(0.0f + f32(src))       (mode 0: first message into a taken
 *                                        buffer; == add onto zeros, bitwise)
 * and, fused into the same pass, nonfinite[slot] |= any(!isfinite(dst)) and
 * sumsq[slot] += sum(dst^2) (f64) — the layer's reject flag
 * (lockfree.py:133) and grad-norm term, so the update never re-reads g.
 * slot_modes (nullable): per-slot mode overriding `mode`, so one launch can
 * accumulate a whole flat gradient into many layers' pages.
 * Ledger (nullable, ConservationLedger, lockfree.py:218-222, 275-326):
 * lsum[slot] += f64 sum(new - old) — the buffer's running f64 sum, read and
 * reset at the take — and, if ldelta != NULL, ldelta[slot] += the same
 * value: this message's produced delta (ldelta is a zeroed row per launch).
 * opts: reserved (one launch shape; pass NULL). */
int hm_accumulate(const void* src, int src_dtype, void* dst, int dst_dtype,
                  const hm_seg_chunk* chunks, int64_t n_chunks, int mode,
                  const uint8_t* slot_modes, uint32_t* nonfinite, double* sumsq,
                  double* lsum, double* ldelta, const hm_launch_opts* opts, void* stream);

/* The take of a gradient buffer's fused statistics (ParamBuffer.take /
 * publish(clear=True) hand-over, lockfree.py:226-241, 251-256): for each
 * slots[i] (device array), out[2i] = lsum[slot] (ledger record_take sum)
 * and out[2i+1] = nonfinite[slot] as a double; then nonfinite, sumsq and
 * lsum of the slot are reset to zero.  Any of nonfinite / sumsq / lsum /
 * out may be NULL. */
int hm_stats_take(const uint32_t* slots, int32_t n_slots, uint32_t* nonfinite, double* sumsq,
                  double* lsum, double* out, void* stream);

/* RNE dtype conversion over segments: publish cast (lockfree.py:169), take
 * widen (lockfree.py:234), pack/unpack of typed tensors. */
int hm_cast(const void* src, int src_dtype, void* dst, int dst_dtype,
            const hm_seg_chunk* chunks, int64_t n_chunks, void* stream);

/* Read-only statistics over segments: nonfinite flag, f64 sum and f64 sum of
 * squares per slot (any output may be NULL).  Used for the functional
 * apply_update check (lockfree.py:133), the post-reduce-scatter check, and
 * the optional ConservationLedger sums (lockfree.py:218-237, 275-326). */
int hm_reduce_stats(const void* src, int src_dtype, const hm_seg_chunk* chunks,
                    int64_t n_chunks, uint32_t* nonfinite, double* sums,
                    double* sumsq, void* stream);

/* Byte-copy descriptors: page pack/unpack (tensor <-> page pool), page
 * relocation (page_move / tensor_merge data motion, pagemem.py:303-407). */
typedef struct hm_copy_desc {
  uint64_t src_off;   /* bytes */
  uint64_t dst_off;   /* bytes */
  uint64_t bytes;
} hm_copy_desc;

/* Device-side gather/scatter copy of many runs in one launch (16-byte
 * vector path when src/dst/len are co-aligned). */
int hm_copy_runs(const void* src, void* dst, const hm_copy_desc* descs,
                 int64_t n_descs, void* stream);

/* Pinned-host <-> device page swap (the CPU tier of hiermem/simengine.py:
 * 250-274 and DelayModel state fetch/store, lockfree.py:96-103): one
 * cudaMemcpyAsync per run on the caller's copy stream (copy engines, no SMs).
 * kind: 1 = host->device, 2 = device->host, 3 = device->device. */
int hm_memcpy_runs(const void* src, void* dst, const hm_copy_desc* descs,
                   int64_t n_descs, int kind, void* stream);

/* Page-locked host memory of exactly `bytes` (cudaHostAlloc, portable):
 * the pinned-host state tier's page pools (the CPU tier of
 * hiermem/pagemem.py:29-32 holding MasterState, hiermem/lockfree.py:148).
 * torch's pinned allocator rounds blocks up to powers of two, which does
 * not fit a 154 GB state in a 196 GB host.  Zero-filled. */
int hm_host_alloc(int64_t bytes, void** out);
int hm_host_free(void* ptr);

/* A compute slot of modelled duration when executing an Algorithm-1 schedule
 * (hiermem/scheduler.py:264-403 tasks, durations from hiermem/simengine.py's
 * timing model): one warp spins on %globaltimer for `ns` nanoseconds. */
int hm_spin(int64_t ns, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HM_PAGE_H */
