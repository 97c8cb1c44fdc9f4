// Host page table: the page-granular allocator of Angel-PTM §4.1 (PAPER.md
// Fig. 5/6) with the exact packing policy of the reference simulator
// hiermem/pagemem.py (cited per function).  The reference keeps pages in a
// Python dict, finds a tail to share by scanning every allocated page in id
// order (pagemem.py:245-249, O(pages) per call) and rebuilds a sorted
// allocated-page list on every query (pagemem.py:163-165).  Here:
//   * free pages live in an ordered set (claim = smallest id, O(log P));
//   * tail sharing is a leftmost-fit query on a max segment tree keyed by
//     page index whose leaf is the page's free bytes when the page is a
//     single shareable tail, else -1 (O(log P));
//   * tensor_merge finds the smallest run with one sliding window (O(P)).
// The observable state (page ids, occupants and their order, stats,
// fragmentation) is identical to the reference for every operation
// sequence; tests/test_pagetable.py pins that against reference dumps.
//
// The reference is metadata-only (pagemem.py:7-9).  This table additionally
// records where each occupant sits inside its page, so device pools can be
// addressed: the first occupant of an empty page sits at byte 0, a second
// occupant is end-aligned; a moved page keeps its layout and a merged chunk
// keeps its in-page offset.  Any two legal occupants therefore never overlap.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdarg>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "../../include/hm_page.h"
#include "hm_error.h"

namespace {

constexpr int64_t kMinPageBytes = 64 * 1024;  // MIN_PAGE_BYTES, pagemem.py:24

const char* tier_name(int t) {
  switch (t) {
    case HM_TIER_GPU: return "GPU";
    case HM_TIER_CPU: return "CPU";
    case HM_TIER_SSD: return "SSD";
  }
  return "?";
}

struct Occ {
  int64_t tid;
  int64_t bytes;
  int64_t offset;
  bool shareable;
};

struct PageRec {
  Occ occ[2];
  int n = 0;
  bool allocated = false;
  int64_t occupied() const {
    int64_t s = 0;
    for (int i = 0; i < n; ++i) s += occ[i].bytes;
    return s;
  }
};

// Max segment tree over page indices answering "leftmost index whose value
// is >= x" — the first-fit tail scan of pagemem.py:245-249.
class ShareIndex {
 public:
  void init(int64_t n) {
    size_ = 1;
    while (size_ < n) size_ <<= 1;
    tree_.assign(2 * size_, -1);
  }
  void set(int64_t i, int64_t v) {
    int64_t k = i + size_;
    tree_[k] = v;
    for (k >>= 1; k >= 1; k >>= 1) tree_[k] = std::max(tree_[2 * k], tree_[2 * k + 1]);
  }
  int64_t leftmost_at_least(int64_t x) const {
    if (tree_.empty() || tree_[1] < x) return -1;
    int64_t k = 1;
    while (k < size_) k = (tree_[2 * k] >= x) ? 2 * k : 2 * k + 1;
    return k - size_;
  }

 private:
  int64_t size_ = 1;
  std::vector<int64_t> tree_;
};

struct Pool {
  int tier;
  int64_t capacity, page_bytes, first, num;
  std::vector<PageRec> pages;
  std::set<int64_t> free_ids;  // global page ids
  ShareIndex share;
  int64_t allocations = 0, releases = 0, moves_in = 0, moves_out = 0, peak = 0;

  int64_t allocated_count() const { return num - (int64_t)free_ids.size(); }
  bool contains(int64_t pid) const { return pid >= first && pid < first + num; }
  PageRec& page(int64_t pid) { return pages[pid - first]; }
  const PageRec& page(int64_t pid) const { return pages[pid - first]; }

  void refresh_share(int64_t pid) {
    const PageRec& p = page(pid);
    int64_t v = -1;
    if (p.n == 1 && p.occ[0].shareable) v = page_bytes - p.occupied();
    share.set(pid - first, v);
  }
  // TierPool.claim, pagemem.py:148-157 (error raised by callers that pre-check).
  int64_t claim() {
    int64_t pid = *free_ids.begin();
    free_ids.erase(free_ids.begin());
    page(pid).allocated = true;
    peak = std::max(peak, allocated_count());
    return pid;
  }
  // TierPool.free, pagemem.py:159-161.
  void release_page(int64_t pid) {
    PageRec& p = page(pid);
    p.n = 0;
    p.allocated = false;
    free_ids.insert(pid);
    refresh_share(pid);
  }
};

struct Tensor {
  int kind;
  int64_t bytes;
  std::vector<int64_t> pages;
};

}  // namespace

struct hm_pagetable {
  std::vector<Pool> pools;        // in PageManager construction order
  std::map<int64_t, Tensor> tensors;
  int64_t next_tid = 0;
  int64_t next_page_id = 0;

  Pool* pool_of_tier(int tier) {
    for (auto& p : pools)
      if (p.tier == tier) return &p;
    return nullptr;
  }
  // PageManager._pool_of_page, pagemem.py:225-229 (first pool in order).
  Pool* pool_of_page(int64_t pid) {
    for (auto& p : pools)
      if (p.contains(pid)) return &p;
    return nullptr;
  }
  const Pool* pool_of_page(int64_t pid) const {
    for (auto& p : pools)
      if (p.contains(pid)) return &p;
    return nullptr;
  }
  // ManagedTensor.tier, pagemem.py:84-90: tier or -1 (NOT_READY).
  int tensor_tier(const Tensor& t) const {
    int tier = -2;
    for (int64_t pid : t.pages) {
      const Pool* p = pool_of_page(pid);
      int pt = p ? p->tier : -1;
      if (tier == -2) tier = pt;
      else if (tier != pt) return -1;
    }
    return tier;
  }
};

namespace {

bool valid_tier(int t) { return t == HM_TIER_GPU || t == HM_TIER_CPU || t == HM_TIER_SSD; }

int no_pool(int tier) {
  return hm_set_error(HM_ERR_CONFIG, "no pool configured for tier %s", tier_name(tier));
}

}  // namespace

extern "C" {

int hm_pt_create(hm_pagetable** out) {
  if (!out) return hm_set_error(HM_ERR_INVALID, "null output pointer");
  *out = new hm_pagetable();
  return HM_OK;
}

int hm_pt_destroy(hm_pagetable* pt) {
  delete pt;
  return HM_OK;
}

// TierPool.__init__ (pagemem.py:114-134) inside PageManager.__init__
// (pagemem.py:191-203).
int hm_pt_add_pool(hm_pagetable* pt, int tier, int64_t capacity, int64_t page_bytes,
                   int64_t first_page_id) {
  if (!pt) return hm_set_error(HM_ERR_INVALID, "null page table");
  if (!valid_tier(tier)) return hm_set_error(HM_ERR_CONFIG, "unknown tier %d", tier);
  if (pt->pool_of_tier(tier))
    return hm_set_error(HM_ERR_CONFIG, "duplicate pool for tier %s", tier_name(tier));
  if (page_bytes < kMinPageBytes || (page_bytes & (page_bytes - 1)))
    return hm_set_error(HM_ERR_CONFIG, "page_bytes must be a power of two >= %lld, got %lld",
                        (long long)kMinPageBytes, (long long)page_bytes);
  if (capacity <= 0 || capacity % page_bytes)
    return hm_set_error(HM_ERR_CONFIG,
                        "capacity_bytes (%lld) must be a positive multiple of page_bytes (%lld)",
                        (long long)capacity, (long long)page_bytes);
  Pool p;
  p.tier = tier;
  p.capacity = capacity;
  p.page_bytes = page_bytes;
  p.first = first_page_id >= 0 ? first_page_id : pt->next_page_id;
  p.num = capacity / page_bytes;
  p.pages.assign((size_t)p.num, PageRec());
  for (int64_t i = 0; i < p.num; ++i) p.free_ids.insert(p.free_ids.end(), p.first + i);
  p.share.init(p.num);
  pt->next_page_id = std::max(pt->next_page_id, p.first + p.num);
  pt->pools.push_back(std::move(p));
  return HM_OK;
}

// PageManager.allocate, pagemem.py:233-283.
int hm_pt_allocate(hm_pagetable* pt, int tier, int kind, int64_t bytes, int64_t* tensor_id) {
  if (!pt || !tensor_id) return hm_set_error(HM_ERR_INVALID, "null argument");
  if (bytes <= 0) return hm_set_error(HM_ERR_CONFIG, "tensor has non-positive size %lld", (long long)bytes);
  if (kind < HM_KIND_PARAM16 || kind > HM_KIND_ACT16)
    return hm_set_error(HM_ERR_CONFIG, "unknown tensor kind %d", kind);
  Pool* pool = pt->pool_of_tier(tier);
  if (!pool) return no_pool(tier);
  if (pool->tier == HM_TIER_SSD && kind != HM_KIND_OPTIM32) {
    static const char* kinds[] = {"param16", "grad16", "optim32", "activation16"};
    hm_set_alloc_bytes(bytes, (int64_t)pool->free_ids.size() * pool->page_bytes);
    return hm_set_error(HM_ERR_ALLOCATION,
                        "tier policy: SSD holds only fp32 optimizer tensors, not %s", kinds[kind]);
  }
  const int64_t page = pool->page_bytes;
  const int64_t full = bytes / page, tail = bytes % page;
  int64_t shared = -1;
  if (tail) {
    int64_t idx = pool->share.leftmost_at_least(tail);  // first-fit, id order
    if (idx >= 0) shared = pool->first + idx;
  }
  const int64_t fresh = full + ((tail && shared < 0) ? 1 : 0);
  const int64_t nfree = (int64_t)pool->free_ids.size();
  if (nfree < fresh) {
    hm_set_alloc_bytes(bytes, nfree * page);
    return hm_set_error(HM_ERR_ALLOCATION,
                        "%s pool cannot fit %lld bytes (%lld fresh pages needed, %lld free)",
                        tier_name(pool->tier), (long long)bytes, (long long)fresh, (long long)nfree);
  }
  const int64_t tid = pt->next_tid++;
  Tensor t;
  t.kind = kind;
  t.bytes = bytes;
  for (int64_t i = 0; i < full; ++i) {
    int64_t pid = pool->claim();
    PageRec& pr = pool->page(pid);
    pr.occ[0] = Occ{tid, page, 0, false};
    pr.n = 1;
    pool->refresh_share(pid);
    t.pages.push_back(pid);
  }
  if (tail) {
    const bool large_tail = full > 0;
    if (shared >= 0) {
      PageRec& pr = pool->page(shared);
      const int64_t off = pr.occ[0].offset == 0 ? page - tail : 0;
      pr.occ[pr.n++] = Occ{tid, tail, off, large_tail};
      pool->refresh_share(shared);
      t.pages.push_back(shared);
    } else {
      int64_t pid = pool->claim();
      PageRec& pr = pool->page(pid);
      pr.occ[0] = Occ{tid, tail, 0, large_tail};
      pr.n = 1;
      pool->refresh_share(pid);
      t.pages.push_back(pid);
    }
  }
  pt->tensors.emplace(tid, std::move(t));
  pool->allocations += 1;
  pool->peak = std::max(pool->peak, pool->allocated_count());
  *tensor_id = tid;
  return HM_OK;
}

// PageManager.release, pagemem.py:285-299.
int hm_pt_release(hm_pagetable* pt, int64_t tid, int64_t* freed_bytes) {
  if (!pt) return hm_set_error(HM_ERR_INVALID, "null page table");
  auto it = pt->tensors.find(tid);
  if (it == pt->tensors.end())
    return hm_set_error(HM_ERR_KEY, "unknown or already released tensor %lld", (long long)tid);
  Tensor t = std::move(it->second);
  pt->tensors.erase(it);
  int64_t freed = 0;
  for (int64_t pid : t.pages) {
    Pool* pool = pt->pool_of_page(pid);
    PageRec& pr = pool->page(pid);
    int k = 0;
    for (int i = 0; i < pr.n; ++i) {
      if (pr.occ[i].tid == tid) freed += pr.occ[i].bytes;
      else pr.occ[k++] = pr.occ[i];
    }
    pr.n = k;
    if (k == 0) pool->release_page(pid);
    else pool->refresh_share(pid);
    pool->releases += 1;
  }
  if (freed_bytes) *freed_bytes = freed;
  return HM_OK;
}

// PageManager.page_move, pagemem.py:303-334.
int hm_pt_page_move(hm_pagetable* pt, int64_t pid, int target_tier, int64_t out[5]) {
  if (!pt || !out) return hm_set_error(HM_ERR_INVALID, "null argument");
  Pool* src = pt->pool_of_page(pid);
  if (!src) return hm_set_error(HM_ERR_KEY, "unknown page id %lld", (long long)pid);
  PageRec& pr = src->page(pid);
  if (pr.n == 0) return hm_set_error(HM_ERR_KEY, "page %lld is free; nothing to move", (long long)pid);
  Pool* dst = pt->pool_of_tier(target_tier);
  if (!dst) return no_pool(target_tier);
  if (dst->tier == src->tier)
    return hm_set_error(HM_ERR_MOVE, "page %lld already resides on %s", (long long)pid,
                        tier_name(src->tier));
  if (dst->tier == HM_TIER_SSD) {
    for (int i = 0; i < pr.n; ++i) {
      const Tensor& t = pt->tensors.at(pr.occ[i].tid);
      if (t.kind != HM_KIND_OPTIM32)
        return hm_set_error(HM_ERR_MOVE,
                            "tier policy: SSD holds only fp32 optimizer tensors (tensor %lld is fp16)",
                            (long long)pr.occ[i].tid);
    }
  }
  if (dst->free_ids.empty())
    return hm_set_error(HM_ERR_MOVE, "destination %s pool is full", tier_name(dst->tier));
  if (dst->page_bytes != src->page_bytes)
    return hm_set_error(HM_ERR_MOVE, "pools use different page sizes; cannot carry the page over");
  const int64_t npid = dst->claim();
  PageRec& np = dst->page(npid);
  np.n = pr.n;
  for (int i = 0; i < pr.n; ++i) np.occ[i] = pr.occ[i];
  dst->refresh_share(npid);
  src->release_page(pid);
  src->moves_out += 1;
  dst->moves_in += 1;
  for (int i = 0; i < np.n; ++i) {
    Tensor& t = pt->tensors.at(np.occ[i].tid);
    auto pos = std::find(t.pages.begin(), t.pages.end(), pid);
    if (pos != t.pages.end()) *pos = npid;
  }
  out[0] = src->page_bytes;
  out[1] = src->tier;
  out[2] = dst->tier;
  out[3] = pid;
  out[4] = npid;
  return HM_OK;
}

// PageManager.tensor_merge, pagemem.py:338-407.  A page of the run is usable
// iff it is free, or it is one of the tensor's own pages and holds no other
// tensor's chunk (pagemem.py:366-376); the smallest start of n consecutive
// usable ids wins.
int hm_pt_tensor_merge(hm_pagetable* pt, int64_t tid, int64_t out[2]) {
  if (!pt || !out) return hm_set_error(HM_ERR_INVALID, "null argument");
  auto it = pt->tensors.find(tid);
  if (it == pt->tensors.end()) return hm_set_error(HM_ERR_KEY, "unknown tensor %lld", (long long)tid);
  Tensor& t = it->second;
  const int tier = pt->tensor_tier(t);
  if (tier < 0)
    return hm_set_error(HM_ERR_MOVE, "tensor %lld is not ready (pages span tiers or mid-move)",
                        (long long)tid);
  Pool* pool = pt->pool_of_tier(tier);
  if (!pool) return no_pool(tier);
  const int64_t n = (int64_t)t.pages.size();
  bool contiguous = true;
  for (int64_t i = 1; i < n; ++i)
    if (t.pages[i] != t.pages[0] + i) contiguous = false;
  if (contiguous) {
    out[0] = 0;
    out[1] = t.pages[0];
    return HM_OK;
  }
  std::set<int64_t> own(t.pages.begin(), t.pages.end());
  auto usable = [&](int64_t pid) {
    const PageRec& pr = pool->page(pid);
    if (!pr.allocated) return true;
    if (!own.count(pid)) return false;
    for (int i = 0; i < pr.n; ++i)
      if (pr.occ[i].tid != tid) return false;
    return true;
  };
  int64_t start = -1, run = 0;
  for (int64_t i = 0; i < pool->num; ++i) {
    run = usable(pool->first + i) ? run + 1 : 0;
    if (run == n) {
      start = pool->first + i - n + 1;
      break;
    }
  }
  if (start < 0) {
    hm_set_alloc_bytes(t.bytes, (int64_t)pool->free_ids.size() * pool->page_bytes);
    return hm_set_error(HM_ERR_ALLOCATION, "no contiguous run of %lld pages available in %s for merge",
                        (long long)n, tier_name(pool->tier));
  }
  // The chunk of this tensor on each of its pages (pagemem.py:352-355).
  std::vector<Occ> chunks;
  chunks.reserve((size_t)n);
  for (int64_t pid : t.pages) {
    const PageRec& pr = pool->page(pid);
    for (int i = 0; i < pr.n; ++i)
      if (pr.occ[i].tid == tid) { chunks.push_back(pr.occ[i]); break; }
  }
  int64_t moved = 0;
  // Phase 1: detach chunks that are not already in their target slot.
  for (int64_t pos = 0; pos < n; ++pos) {
    const int64_t pid = t.pages[pos];
    if (pid == start + pos) continue;
    PageRec& pr = pool->page(pid);
    int k = 0;
    for (int i = 0; i < pr.n; ++i)
      if (pr.occ[i].tid != tid) pr.occ[k++] = pr.occ[i];
    pr.n = k;
    if (k == 0) pool->release_page(pid);
    else pool->refresh_share(pid);
    moved += 1;
  }
  // Phase 2: attach each moved chunk to its (now empty) target page; the
  // target leaves the free list without a stats update (pagemem.py:401-403).
  for (int64_t pos = 0; pos < n; ++pos) {
    const int64_t pid = t.pages[pos], target = start + pos;
    if (pid == target) continue;
    PageRec& pr = pool->page(target);
    if (pr.n == 0 && !pr.allocated) {
      pool->free_ids.erase(target);
      pr.allocated = true;
    }
    pr.occ[pr.n++] = chunks[(size_t)pos];
    pool->refresh_share(target);
  }
  for (int64_t pos = 0; pos < n; ++pos) t.pages[pos] = start + pos;
  out[0] = moved;
  out[1] = start;
  return HM_OK;
}

int hm_pt_num_pools(const hm_pagetable* pt) { return pt ? (int)pt->pools.size() : 0; }

int hm_pt_pool_info(const hm_pagetable* pt, int index, int64_t out[12]) {
  if (!pt || !out || index < 0 || index >= (int)pt->pools.size())
    return hm_set_error(HM_ERR_INVALID, "bad pool index %d", index);
  const Pool& p = pt->pools[(size_t)index];
  int64_t occupied = 0;
  for (const auto& pr : p.pages)
    if (pr.allocated) occupied += pr.occupied();
  const int64_t v[12] = {p.tier, p.capacity, p.page_bytes, p.first, p.num,
                         (int64_t)p.free_ids.size(), p.allocations, p.releases,
                         p.moves_in, p.moves_out, p.peak, occupied};
  std::copy(v, v + 12, out);
  return HM_OK;
}

int64_t hm_pt_allocated_pages(const hm_pagetable* pt, int tier, int64_t* out, int64_t cap) {
  const Pool* p = pt ? const_cast<hm_pagetable*>(pt)->pool_of_tier(tier) : nullptr;
  if (!p) return 0;
  int64_t k = 0;
  for (int64_t i = 0; i < p->num; ++i) {
    if (!p->pages[(size_t)i].allocated) continue;
    if (k < cap && out) out[k] = p->first + i;
    ++k;
  }
  return k;
}

int64_t hm_pt_free_pages(const hm_pagetable* pt, int tier, int64_t* out, int64_t cap) {
  const Pool* p = pt ? const_cast<hm_pagetable*>(pt)->pool_of_tier(tier) : nullptr;
  if (!p) return 0;
  int64_t k = 0;
  for (int64_t pid : p->free_ids) {
    if (k < cap && out) out[k] = pid;
    ++k;
  }
  return k;
}

int hm_pt_page_info(const hm_pagetable* pt, int64_t pid, int64_t out[11]) {
  if (!pt || !out) return hm_set_error(HM_ERR_INVALID, "null argument");
  const Pool* p = pt->pool_of_page(pid);
  if (!p) return hm_set_error(HM_ERR_KEY, "unknown page id %lld", (long long)pid);
  const PageRec& pr = p->page(pid);
  out[0] = p->tier;
  out[1] = p->page_bytes;
  out[2] = pr.n;
  for (int i = 0; i < 2; ++i) {
    const bool has = i < pr.n;
    out[3 + 4 * i] = has ? pr.occ[i].tid : -1;
    out[4 + 4 * i] = has ? pr.occ[i].bytes : 0;
    out[5 + 4 * i] = has ? (pr.occ[i].shareable ? 1 : 0) : 0;
    out[6 + 4 * i] = has ? pr.occ[i].offset : 0;
  }
  return HM_OK;
}

int64_t hm_pt_tensor_ids(const hm_pagetable* pt, int64_t* out, int64_t cap) {
  if (!pt) return 0;
  int64_t k = 0;
  for (const auto& kv : pt->tensors) {
    if (k < cap && out) out[k] = kv.first;
    ++k;
  }
  return k;
}

int hm_pt_tensor_info(const hm_pagetable* pt, int64_t tid, int64_t out[4]) {
  if (!pt || !out) return hm_set_error(HM_ERR_INVALID, "null argument");
  auto it = pt->tensors.find(tid);
  if (it == pt->tensors.end()) return hm_set_error(HM_ERR_KEY, "unknown tensor %lld", (long long)tid);
  out[0] = it->second.kind;
  out[1] = it->second.bytes;
  out[2] = pt->tensor_tier(it->second);
  out[3] = (int64_t)it->second.pages.size();
  return HM_OK;
}

int64_t hm_pt_tensor_pages(const hm_pagetable* pt, int64_t tid, int64_t* out, int64_t cap) {
  if (!pt) return -1;
  auto it = pt->tensors.find(tid);
  if (it == pt->tensors.end()) {
    hm_set_error(HM_ERR_KEY, "unknown tensor %lld", (long long)tid);
    return -1;
  }
  const auto& pg = it->second.pages;
  for (int64_t i = 0; i < (int64_t)pg.size() && i < cap && out; ++i) out[i] = pg[(size_t)i];
  return (int64_t)pg.size();
}

int64_t hm_pt_tensor_segments(const hm_pagetable* pt, int64_t tid, int64_t* out3, int64_t cap) {
  if (!pt) return -1;
  auto it = pt->tensors.find(tid);
  if (it == pt->tensors.end()) {
    hm_set_error(HM_ERR_KEY, "unknown tensor %lld", (long long)tid);
    return -1;
  }
  const auto& pg = it->second.pages;
  for (int64_t i = 0; i < (int64_t)pg.size() && i < cap && out3; ++i) {
    const int64_t pid = pg[(size_t)i];
    const Pool* p = pt->pool_of_page(pid);
    const PageRec& pr = p->page(pid);
    int64_t off = 0, bytes = 0;
    for (int j = 0; j < pr.n; ++j)
      if (pr.occ[j].tid == tid) { off = pr.occ[j].offset; bytes = pr.occ[j].bytes; break; }
    out3[3 * i + 0] = pid;
    out3[3 * i + 1] = off;
    out3[3 * i + 2] = bytes;
  }
  return (int64_t)pg.size();
}

}  // extern "C"
