// Host runtime of cumstream_b200: device-resident series and window state,
// cached layouts and launch plans, and the extern "C" entry points declared
// in include/cumstream_b200.h.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <numeric>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <map>
#include <unordered_map>
#include <memory>
#include <functional>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "common.hpp"
#include "kernels.cuh"
#include "layout.hpp"
#include "nccl_shim.hpp"

namespace csb {

namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_rows_read{0};

struct DevLayout {
  Layout host;
  DevBuf<uint64_t> offset;
  DevBuf<uint16_t> index;
  DevBuf<uint64_t> prefix;
  DevBuf<double> mult;
  std::vector<double> mult_host;  // the same, for the report's block fold on the host
  DevBuf<uint32_t> diag;  // blocks with equal neighbouring coordinates
  uint32_t ndiag = 0;
  std::vector<uint32_t> diag_host;
  // [first, count) of the diagonal-block list inside block range [lo, hi)
  std::pair<uint32_t, uint32_t> diag_range(uint64_t lo, uint64_t hi) const {
    const auto a = std::lower_bound(diag_host.begin(), diag_host.end(), lo);
    const auto b = std::lower_bound(diag_host.begin(), diag_host.end(), hi);
    return {static_cast<uint32_t>(a - diag_host.begin()), static_cast<uint32_t>(b - a)};
  }
  LayoutDev view() const {
    LayoutDev v;
    v.offset = offset.ptr;
    v.index = index.ptr;
    v.prefix = prefix.ptr;
    v.order = host.order;
    v.grid = host.grid;
    v.nblocks = host.nblocks;
    return v;
  }
};

struct Device {
  int id = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // low-order kernel beside the top pair
  cudaEvent_t fork = nullptr, join = nullptr;
  cudaEvent_t nfork = nullptr, njoin = nullptr;  // exact norm partials of C_s beside moms2cums of order s + 1
  std::mutex mu;
  std::map<std::tuple<int, int, int>, std::shared_ptr<DevLayout>> layouts;
  std::map<std::tuple<int, int, int, int>, std::shared_ptr<MomentPlan>> plans;
  std::map<std::tuple<int, int, int>, std::shared_ptr<DevBuf<LowerElem>>> lower;
  std::map<std::tuple<int, int, int>, std::shared_ptr<DevBuf<LowerThread>>> lower2;
  std::map<std::tuple<int, int, int>, std::shared_ptr<DevBuf<uint64_t>>> subs;
  std::map<std::tuple<int, int, int>, std::shared_ptr<DevBuf<uint32_t>>> m2c_order;
  std::map<std::pair<int, int>, std::pair<std::shared_ptr<DevBuf<uint32_t>>, std::shared_ptr<DevBuf<uint32_t>>>> canon;
  std::map<std::pair<int, int>, std::pair<std::shared_ptr<DevBuf<uint2>>, std::shared_ptr<DevBuf<uint32_t>>>> mirror;
  std::map<std::pair<int, int>, std::pair<std::shared_ptr<DevBuf<uint32_t>>, std::shared_ptr<DevBuf<uint32_t>>>> copies;
  std::map<std::tuple<int, int, int, int>, std::shared_ptr<ShardPlan>> shards;
  std::shared_ptr<Comm> comm;  // csb_comm_init / csb_comm_init_ops
};

std::mutex g_dev_mu;
std::map<int, std::unique_ptr<Device>> g_devices;

int current_device_id() {
  int d = 0;
  CSB_CUDA(cudaGetDevice(&d));
  return d;
}

Device& device() {
  ensure_device();
  const int id = current_device_id();
  std::lock_guard<std::mutex> lk(g_dev_mu);
  auto& slot = g_devices[id];
  if (!slot) {
    slot = std::make_unique<Device>();
    slot->id = id;
    CSB_CUDA(cudaStreamCreateWithFlags(&slot->stream, cudaStreamNonBlocking));
    CSB_CUDA(cudaStreamCreateWithFlags(&slot->side, cudaStreamNonBlocking));
    CSB_CUDA(cudaEventCreateWithFlags(&slot->fork, cudaEventDisableTiming));
    CSB_CUDA(cudaEventCreateWithFlags(&slot->join, cudaEventDisableTiming));
    CSB_CUDA(cudaEventCreateWithFlags(&slot->nfork, cudaEventDisableTiming));
    CSB_CUDA(cudaEventCreateWithFlags(&slot->njoin, cudaEventDisableTiming));
  }
  return *slot;
}

std::shared_ptr<DevLayout> get_layout(Device& dev, int order, int n, int b) {
  std::lock_guard<std::mutex> lk(dev.mu);
  auto& slot = dev.layouts[{order, n, b}];
  if (!slot) {
    auto L = std::make_shared<DevLayout>();
    L->host = Layout(order, n, b);
    const Layout& h = L->host;
    L->offset.alloc(h.offset.size());
    L->index.alloc(h.index.size());
    L->prefix.alloc(h.prefix.size());
    L->mult.alloc(h.nblocks);
    std::vector<double> mult(h.nblocks);
    int j[20];
    for (uint64_t r = 0; r < h.nblocks; ++r) {
      for (int k = 0; k < order; ++k) j[k] = h.index[r * order + k];
      mult[r] = static_cast<double>(block_multiplicity(j, order));
    }
    h2d_sync(L->offset.ptr, h.offset.data(), L->offset.bytes());
    h2d_sync(L->index.ptr, h.index.data(), L->index.bytes());
    h2d_sync(L->prefix.ptr, h.prefix.data(), L->prefix.bytes());
    h2d_sync(L->mult.ptr, mult.data(), L->mult.bytes());
    L->mult_host = mult;
    std::vector<uint32_t> diag;
    for (uint64_t r = 0; r < h.nblocks; ++r) {
      bool runs = false;
      for (int k = 1; k < order; ++k) runs |= h.index[r * order + k] == h.index[r * order + k - 1];
      if (runs) diag.push_back(static_cast<uint32_t>(r));
    }
    L->ndiag = static_cast<uint32_t>(diag.size());
    L->diag_host = diag;
    L->diag.alloc(diag.size());
    if (!diag.empty())
      h2d_sync(L->diag.ptr, diag.data(), L->diag.bytes());
    slot = L;
  }
  return slot;
}

std::shared_ptr<ShardPlan> get_shard_plan(Device& dev, int d, int n, int b, int count) {
  auto top = get_layout(dev, d, n, b);
  auto low = get_layout(dev, d > 1 ? d - 1 : 1, n, b);
  std::lock_guard<std::mutex> lk(dev.mu);
  auto& slot = dev.shards[{d, n, b, count}];
  if (!slot) {
    auto sp = std::make_shared<ShardPlan>();
    sp->build(d, n, b, count, top->host, low->host);
    slot = sp;
  }
  return slot;
}

std::shared_ptr<MomentPlan> get_plan(Device& dev, int S, int n, int b, bool dmma, const ShardPlan* sp = nullptr,
                                     int shard_index = 0) {
  auto top = get_layout(dev, S, n, b);
  std::shared_ptr<DevLayout> low = S > 1 ? get_layout(dev, S - 1, n, b) : nullptr;
  const int count = sp ? sp->count : 1;
  std::lock_guard<std::mutex> lk(dev.mu);
  auto& slot = dev.plans[{S, n, b, (dmma ? 1 : 0) + 2 * (count * 256 + shard_index)}];
  if (!slot) {
    auto p = std::make_shared<MomentPlan>();
    if (dmma)
      p->build_dmma(S, n, b, top->host, low ? &low->host : nullptr, dmma_scratch_per_tile(), tail_windows(S, n, b), sp,
                    shard_index);
    else
      p->build(S, n, b, top->host, low ? &low->host : nullptr, kMomThreads);
    p->upload();
    slot = p;
  }
  return slot;
}

}  // namespace

void set_smem_attr(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  CSB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{kern, dev}];
  if (have >= bytes) return;
  CSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  have = bytes;
}

namespace {

// Optional per-launch event timing (csb_profile_enable); events are pooled
// (created once, returned by csb_profile_read) to keep the host cost of a
// profiled step small.

struct Profiler {
  std::mutex mu;
  bool on = false;
  struct Rec {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  };
  std::map<std::string, Rec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {  // under mu
    if (pool.empty()) {
      cudaEvent_t e = nullptr;
      CSB_CUDA(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
};
Profiler g_prof;

// Every scope is also an NVTX range (header-only NVTX 3: a no-op unless a
// tool such as nsys or ncu --nvtx is attached), so timelines show the
// step's phases by the same tags csb_profile_read uses.
struct ProfScope {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t st;
  const char* tag;
  ProfScope(const char* tag_, cudaStream_t st_) : st(st_), tag(tag_) {
    nvtxRangePushA(tag);
    if (!g_prof.on) return;
    {
      std::lock_guard<std::mutex> lk(g_prof.mu);
      a = g_prof.get();
      b = g_prof.get();
    }
    CSB_CUDA(cudaEventRecord(a, st));
  }
  ~ProfScope() {
    nvtxRangePop();
    if (!a) return;
    cudaEventRecord(b, st);
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.recs[tag].ev.emplace_back(a, b);
  }
};

// Canonical elements of order s (lexicographic) with the offset of their
// block in M_s, for the low-order kernel.
std::shared_ptr<DevBuf<LowerElem>> get_lower_elems(Device& dev, int s, int n, int b, const Layout& L) {
  std::lock_guard<std::mutex> lk(dev.mu);
  auto& slot = dev.lower[{s, n, b}];
  if (!slot) {
    std::vector<LowerElem> v;
    v.reserve(multiset_count(n, s));
    int t[8] = {0}, j[8];
    for (;;) {
      LowerElem e{};
      for (int k = 0; k < s; ++k) {
        e.idx[k] = static_cast<uint16_t>(t[k]);
        j[k] = t[k] / b;
      }
      e.blk_off = L.offset[L.rank(j)];
      v.push_back(e);
      int k = s - 1;
      while (k >= 0 && t[k] == n - 1) --k;
      if (k < 0) break;
      const int val = t[k] + 1;
      for (int l = k; l < s; ++l) t[l] = val;
    }
    auto buf = std::make_shared<DevBuf<LowerElem>>(v.size());
    h2d_sync(buf->ptr, v.data(), buf->bytes());
    slot = buf;
  }
  return slot;
}

// Sub-block offsets for moms2cums of order S: for every block j and every
// proper non-empty subset m of its positions, the offset in C_|m| of the
// block (j_k : k in m) (cumulants.cpp:163-171 reads C_|P|[i_P] there).
std::shared_ptr<DevBuf<uint64_t>> get_subs(Device& dev, int S, int n, int b) {
  std::vector<std::shared_ptr<DevLayout>> lays;
  for (int k = 1; k <= S; ++k) lays.push_back(get_layout(dev, k, n, b));
  std::lock_guard<std::mutex> lk(dev.mu);
  auto& slot = dev.subs[{S, n, b}];
  if (!slot) {
    const Layout& LS = lays[S - 1]->host;
    const int NM = (1 << S) - 1;
    std::vector<uint64_t> v(LS.nblocks * static_cast<uint64_t>(NM - 1));
    int sub[kMaxOrder];
    for (uint64_t r = 0; r < LS.nblocks; ++r)
      for (int m = 1; m < NM; ++m) {
        int cnt = 0;
        for (int k = 0; k < S; ++k)
          if (m >> k & 1) sub[cnt++] = LS.index[r * S + k];
        const Layout& Lq = lays[cnt - 1]->host;
        v[r * (NM - 1) + (m - 1)] = Lq.offset[Lq.rank(sub)];
      }
    auto buf = std::make_shared<DevBuf<uint64_t>>(v.size());
    if (!v.empty()) h2d_sync(buf->ptr, v.data(), buf->bytes());
    slot = buf;
  }
  return slot;
}

// Blocks of order S sorted by descending number of canonical entries
// (prod over runs of equal block coordinate of C(e + r - 1, r), e the run's
// extent), ties in block order: the persistent moms2cums kernel deals them
// round-robin to its CTAs.
std::shared_ptr<DevBuf<uint32_t>> get_m2c_order(Device& dev, int S, int n, int b) {
  auto lay = get_layout(dev, S, n, b);
  std::lock_guard<std::mutex> lk(dev.mu);
  auto& slot = dev.m2c_order[{S, n, b}];
  if (!slot) {
    const Layout& L = lay->host;
    std::vector<uint64_t> cost(L.nblocks);
    for (uint64_t r = 0; r < L.nblocks; ++r) {
      uint64_t c = 1;
      for (int k = 0; k < S;) {
        int e = k + 1;
        while (e < S && L.index[r * S + e] == L.index[r * S + k]) ++e;
        c *= multiset_count(L.ext(L.index[r * S + k]), e - k);
        k = e;
      }
      cost[r] = c;
    }
    std::vector<uint32_t> ord(L.nblocks);
    std::iota(ord.begin(), ord.end(), 0u);
    std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t c2) { return cost[a] > cost[c2]; });
    auto buf = std::make_shared<DevBuf<uint32_t>>(ord.size());
    if (!ord.empty()) h2d_sync(buf->ptr, ord.data(), buf->bytes());
    slot = buf;
  }
  return slot;
}

// Canonical in-block positions of a full order-S block (extents b) for each
// run pattern (bit k-1 set: j_k == j_{k-1}): offsets non-decreasing within
// runs (cumulants.cpp:163-168), C-order positions, ascending.
std::pair<const uint32_t*, const uint32_t*> get_canon(Device& dev, int S, int b) {
  std::lock_guard<std::mutex> lk(dev.mu);
  auto& slot = dev.canon[{S, b}];
  if (!slot.first) {
    uint64_t vol = 1;
    for (int k = 0; k < S; ++k) vol *= static_cast<uint64_t>(b);
    std::vector<uint32_t> list, off;
    const uint32_t npat = 1u << (S - 1);
    int o[kMaxOrder];
    for (uint32_t pat = 0; pat < npat; ++pat) {
      off.push_back(static_cast<uint32_t>(list.size()));
      for (uint64_t pos = 0; pos < vol; ++pos) {
        uint64_t rem = pos;
        for (int k = S - 1; k >= 0; --k) {
          o[k] = static_cast<int>(rem % static_cast<uint64_t>(b));
          rem /= static_cast<uint64_t>(b);
        }
        bool ok = true;
        for (int k = 1; k < S; ++k)
          if ((pat >> (k - 1) & 1) && o[k] < o[k - 1]) ok = false;
        if (ok) list.push_back(static_cast<uint32_t>(pos));
      }
    }
    off.push_back(static_cast<uint32_t>(list.size()));
    auto l = std::make_shared<DevBuf<uint32_t>>(list.size());
    auto o2 = std::make_shared<DevBuf<uint32_t>>(off.size());
    h2d_sync(l->ptr, list.data(), l->bytes());
    h2d_sync(o2->ptr, off.data(), o2->bytes());
    slot = {l, o2};
  }
  return {slot.first->ptr, slot.second->ptr};
}

// (dst, src) pairs of the symmetric copies of a full order-S block (all
// extents b) per run pattern (bit k-1: j_k == j_{k-1}): dst a non-canonical
// position, src its offsets sorted within runs (symten.cpp:195-220).  Not
// built for large blocks (the mirror kernel then sorts in place).
std::pair<const uint2*, const uint32_t*> get_mirror_lists(Device& dev, int S, int b) {
  std::lock_guard<std::mutex> lk(dev.mu);
  auto& slot = dev.mirror[{S, b}];
  if (!slot.first) {
    uint64_t vol = 1;
    for (int k = 0; k < S; ++k) vol *= static_cast<uint64_t>(b);
    const uint32_t npat = 1u << (S - 1);
    if (vol * npat > (1ull << 20)) return {nullptr, nullptr};
    std::vector<uint2> list;
    std::vector<uint32_t> off;
    int o[kMaxOrder];
    for (uint32_t pat = 0; pat < npat; ++pat) {
      off.push_back(static_cast<uint32_t>(list.size()));
      for (uint64_t pos = 0; pos < vol; ++pos) {
        uint64_t rem = pos;
        for (int k = S - 1; k >= 0; --k) {
          o[k] = static_cast<int>(rem % static_cast<uint64_t>(b));
          rem /= static_cast<uint64_t>(b);
        }
        bool canonical = true;
        for (int k = 1; k < S; ++k)
          if ((pat >> (k - 1) & 1) && o[k] < o[k - 1]) canonical = false;
        if (canonical) continue;
        for (int pass = 0; pass < S - 1; ++pass)
          for (int k = 1; k < S; ++k)
            if ((pat >> (k - 1) & 1) && o[k] < o[k - 1]) std::swap(o[k], o[k - 1]);
        uint64_t src = 0;
        for (int k = 0; k < S; ++k) src = src * static_cast<uint64_t>(b) + static_cast<uint64_t>(o[k]);
        list.push_back(make_uint2(static_cast<uint32_t>(pos), static_cast<uint32_t>(src)));
      }
    }
    off.push_back(static_cast<uint32_t>(list.size()));
    auto l = std::make_shared<DevBuf<uint2>>(std::max<size_t>(1, list.size()));
    auto o2 = std::make_shared<DevBuf<uint32_t>>(off.size());
    if (!list.empty()) h2d_sync(l->ptr, list.data(), list.size() * sizeof(uint2));
    h2d_sync(o2->ptr, off.data(), o2->bytes());
    slot = {l, o2};
  }
  return {slot.first->ptr, slot.second->ptr};
}

// Per canonical position of a full order-S block (indexed like get_canon's
// lists, patterns concatenated): its symmetric copies, as CSR (start, dst).
// The out-of-block moms2cums pass writes each copy and its norm term as
// soon as the canonical value exists.  Built where the mirror lists are.
std::pair<const uint32_t*, const uint32_t*> get_copy_lists(Device& dev, int S, int b) {
  uint64_t vol = 1;
  for (int k = 0; k < S; ++k) vol *= static_cast<uint64_t>(b);
  const uint32_t npat = 1u << (S - 1);
  if (vol * npat > (1ull << 20)) return {nullptr, nullptr};
  std::lock_guard<std::mutex> lk(dev.mu);
  auto& slot = dev.copies[{S, b}];
  if (!slot.first) {
    std::vector<uint32_t> start, dst;
    std::vector<std::vector<uint32_t>> by_src(vol);
    int o[kMaxOrder];
    for (uint32_t pat = 0; pat < npat; ++pat) {
      for (auto& v : by_src) v.clear();
      std::vector<uint32_t> canon;
      for (uint64_t pos = 0; pos < vol; ++pos) {
        uint64_t rem = pos;
        for (int k = S - 1; k >= 0; --k) {
          o[k] = static_cast<int>(rem % static_cast<uint64_t>(b));
          rem /= static_cast<uint64_t>(b);
        }
        bool canonical = true;
        for (int k = 1; k < S; ++k)
          if ((pat >> (k - 1) & 1) && o[k] < o[k - 1]) canonical = false;
        if (canonical) {
          canon.push_back(static_cast<uint32_t>(pos));
          continue;
        }
        for (int pass = 0; pass < S - 1; ++pass)
          for (int k = 1; k < S; ++k)
            if ((pat >> (k - 1) & 1) && o[k] < o[k - 1]) std::swap(o[k], o[k - 1]);
        uint64_t src = 0;
        for (int k = 0; k < S; ++k) src = src * static_cast<uint64_t>(b) + static_cast<uint64_t>(o[k]);
        by_src[src].push_back(static_cast<uint32_t>(pos));
      }
      for (uint32_t c : canon) {  // same order as get_canon's list for this pattern
        start.push_back(static_cast<uint32_t>(dst.size()));
        dst.insert(dst.end(), by_src[c].begin(), by_src[c].end());
      }
    }
    start.push_back(static_cast<uint32_t>(dst.size()));
    auto st = std::make_shared<DevBuf<uint32_t>>(start.size());
    auto ds = std::make_shared<DevBuf<uint32_t>>(std::max<size_t>(1, dst.size()));
    h2d_sync(st->ptr, start.data(), st->bytes());
    if (!dst.empty()) h2d_sync(ds->ptr, dst.data(), dst.size() * sizeof(uint32_t));
    slot = {st, ds};
  }
  return {slot.first->ptr, slot.second->ptr};
}

// Thread table of the staged low-order kernel for orders 1..ST: the
// order-ST tuples in lexicographic order, cut into runs of <= W sharing
// their (ST-1)-prefix pi; a prefix's first run also represents the tuples
// (pi_1..pi_s), s < ST, whose trailing coordinates pi_{s+1..} equal pi_s.
std::shared_ptr<DevBuf<LowerThread>> get_lower2_threads(Device& dev, int ST, int n, int W) {
  std::lock_guard<std::mutex> lk(dev.mu);
  auto& slot = dev.lower2[{ST, n, W}];
  if (!slot) {
    auto key = [](const int* t, int s) {
      uint64_t k = static_cast<uint64_t>(s);
      for (int i = 0; i < s; ++i) k = k * 65536u + static_cast<uint64_t>(t[i]);
      return k;
    };
    // lexicographic element ids of orders 1..ST-1 (the rep targets)
    std::unordered_map<uint64_t, uint32_t> ids;
    for (int s = 1; s < ST; ++s) {
      int t[8] = {0};
      uint32_t id = 0;
      for (;;) {
        ids[key(t, s)] = id++;
        int k = s - 1;
        while (k >= 0 && t[k] == n - 1) --k;
        if (k < 0) break;
        const int v = t[k] + 1;
        for (int l = k; l < s; ++l) t[l] = v;
      }
    }
    std::vector<LowerThread> v;
    int t[8] = {0};
    uint32_t id = 0;
    for (;;) {
      // t = (pi, t_ST) with t_ST = pi_last (or 0): the first tuple of pi
      const int np = ST - 1;
      const int first = np > 0 ? t[np - 1] : 0;
      if (W < 0) {
        // strided: thread q of the prefix's nthr threads owns the elements
        // t = first + q + k * nthr (k < -W), so the lanes of one prefix read
        // consecutive columns of a staged row (no shared-memory bank
        // conflicts between them); pad = the stride
        const int m = n - first, nthr = (m - W - 1) / -W;
        for (int q = 0; q < nthr; ++q) {
          LowerThread lt{};
          lt.e0 = id + static_cast<uint32_t>(q);
          for (int k = 0; k < np; ++k) lt.pidx[k] = static_cast<uint16_t>(t[k]);
          lt.t0 = static_cast<uint16_t>(first + q);
          lt.cnt = static_cast<uint16_t>((m - q + nthr - 1) / nthr);
          lt.pad = static_cast<uint32_t>(nthr);
          for (int k = 0; k < 3; ++k) lt.rep[k] = 0xffffffffu;
          if (q == 0)
            for (int s = 1; s <= np; ++s) {
              bool ok = true;
              for (int k = s; k < np; ++k) ok &= t[k] == t[s - 1];
              if (ok) lt.rep[s - 1] = ids.at(key(t, s));
            }
          v.push_back(lt);
        }
        id += static_cast<uint32_t>(m);
      }
      for (int t0 = first; W > 0 && t0 < n; t0 += W) {
        LowerThread lt{};
        lt.e0 = id;
        for (int k = 0; k < np; ++k) lt.pidx[k] = static_cast<uint16_t>(t[k]);
        lt.t0 = static_cast<uint16_t>(t0);
        lt.cnt = static_cast<uint16_t>(std::min(W, n - t0));
        for (int k = 0; k < 3; ++k) lt.rep[k] = 0xffffffffu;
        if (t0 == first)
          for (int s = 1; s <= np; ++s) {
            bool ok = true;
            for (int k = s; k < np; ++k) ok &= t[k] == t[s - 1];
            if (ok) lt.rep[s - 1] = ids.at(key(t, s));
          }
        id += lt.cnt;
        v.push_back(lt);
      }
      // next prefix pi (lexicographic)
      if (np == 0) break;
      int k = np - 1;
      while (k >= 0 && t[k] == n - 1) --k;
      if (k < 0) break;
      const int val = t[k] + 1;
      for (int l = k; l < np; ++l) t[l] = val;
    }
    require(id == multiset_count(n, ST), "lower2: element count mismatch");
    auto buf = std::make_shared<DevBuf<LowerThread>>(v.size());
    h2d_sync(buf->ptr, v.data(), buf->bytes());
    slot = buf;
  }
  return slot;
}

}  // namespace

void ensure_device() {
  int count = 0;
  const cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    fail(CSB_ERUNTIME, "cumstream_b200: no CUDA device (this library has no CPU fallback)");
  }
}

}  // namespace csb

using namespace csb;

// ---------------------------------------------------------------------------
struct csb_series {
  int n = 0, d = 0, b = 0;
  uint64_t window_len = 0;
  Device* dev = nullptr;
  std::vector<std::shared_ptr<DevLayout>> lay;  // orders 1..d
  std::vector<DevBuf<double>> data;
  // orders (bit s-1) whose symmetric copies the next run_moms2cums fills
  // from its staged blocks instead of a mirror kernel (stream step only)
  mutable uint32_t mirror_defer = 0;
};

namespace csb {
namespace {

std::unique_ptr<csb_series> make_series(int n, int d, int b) {
  require(n >= 1, "series: dim must be positive");
  require(d >= 1 && d <= kMaxOrderAny, "series: max_order must be in [1, 20]");
  require(b >= 1 && b <= n, "series: block_size must be in [1, dim]");
  Device& dev = device();
  auto s = std::make_unique<csb_series>();
  s->n = n;
  s->d = d;
  s->b = b;
  s->dev = &dev;
  for (int k = 1; k <= d; ++k) {
    s->lay.push_back(get_layout(dev, k, n, b));
    s->data.emplace_back(s->lay.back()->host.stored);
    CSB_CUDA(cudaMemsetAsync(s->data.back().ptr, 0, s->data.back().bytes(), dev.stream));
  }
  CSB_CUDA(cudaStreamSynchronize(dev.stream));
  return s;
}

void check_order(const csb_series* s, int order) {
  require(s != nullptr, "null series");
  if (order < 1 || order > s->d) fail(CSB_ERANGE, "series: order out of range");
}

// Captured step graphs hold raw scratch pointers: every (re)allocation or
// release of a scratch buffer bumps this generation, and a graph captured
// under an older one is dropped and captured again instead of replayed.
std::atomic<uint64_t> g_scratch_gen{1};

// Scratch buffer for the pass-0 stash of the update kernel (per device).
struct Scratch {
  DevBuf<double> buf;
  DevBuf<uint32_t> flags;
  ~Scratch() { g_scratch_gen.fetch_add(1, std::memory_order_relaxed); }
  double* get(uint64_t count) {
    if (buf.count < count) {
      buf.alloc(count);
      g_scratch_gen.fetch_add(1, std::memory_order_relaxed);
    }
    return buf.ptr;
  }
  DevBuf<double> tail;  // the tail kernel's per-SM stash (beside the DMMA kernel's scratch)
  double* get_tail(uint64_t count) {
    if (tail.count < count) {
      tail.alloc(count);
      g_scratch_gen.fetch_add(1, std::memory_order_relaxed);
    }
    return tail.ptr;
  }
  DevBuf<double> zeros;
  const double* get_zeros(uint64_t count) {
    if (zeros.count < count) {
      zeros.alloc(count);
      memset_sync(zeros.ptr, 0, zeros.bytes());
      g_scratch_gen.fetch_add(1, std::memory_order_relaxed);
    }
    return zeros.ptr;
  }
  uint32_t* get_flags(uint64_t count) {
    if (flags.count < count) {
      flags.alloc(count);
      memset_sync(flags.ptr, 0, flags.bytes());
      g_scratch_gen.fetch_add(1, std::memory_order_relaxed);
    }
    return flags.ptr;
  }
};
thread_local std::map<int, Scratch> g_scratch;
// Orders are processed as pairs (S, S-1): (d, d-1), (d-2, d-3), ... with a
// lone order 1 when d is odd.  Only the pair topped by d uses the fused
// multiply-add of the reference's deepest loop (moments.cpp:47).
// Orders are processed as: the top pair (S, S-1) with S = d -- the fused
// multiply-add of the reference's deepest loop (moments.cpp:47) on the
// FP64 tensor cores when possible -- and every order <= d-2 by the
// element-parallel low-order kernel (plain product + add, moments.cpp:55-57).
// Which part of the top pair this process owns.  comm is the
// NCCL communicator of the stream engine; the series-level shard entry
// points run without one (no exchange: the caller assembles shards).
struct ShardCtx {
  const ShardPlan* plan = nullptr;
  int index = 0;
  Comm* comm = nullptr;
  bool active() const { return plan && plan->count > 1; }
  uint64_t lo(int which) const { return (which ? plan->low_blk : plan->top_blk)[index]; }
  uint64_t hi(int which) const { return (which ? plan->low_blk : plan->top_blk)[index + 1]; }
};

// side_tail: work that depends only on orders <= d-2, enqueued on the side
// stream behind the low-order kernel (the stream step's C_1, C_2); returns
// whether it ran there (else the caller does it in line)
void run_moments(csb_series* m, const RowSource src[2], int npass, uint64_t K, double c,
                 cudaStream_t st, int only_order = 0, const ShardCtx& sh = ShardCtx{}, bool defer_mirror = false,
                 const std::function<void(cudaStream_t)>& side_tail = nullptr, bool* side_tail_ran = nullptr) {
  Device& dev = *m->dev;
  const int d = m->d;
  const int S = only_order ? only_order : d;
  if (S > kMaxOrder) {
    // any-order kernels: every stored element of every order from its own
    // sorted index (no pyramid, no mirror pass); not sharded
    if (sh.active()) fail(CSB_EINVAL, "sharding supports orders up to 8");
    ProfScope ps("moment_generic", st);
    for (int s = only_order ? only_order : 1; s <= S; ++s) {
      GenMomParams g;
      g.src[0] = src[0];
      g.src[1] = src[1];
      g.npass = npass;
      g.K = static_cast<uint32_t>(K);
      g.n = m->n;
      g.b = m->b;
      g.top = s == S;
      g.m = m->data[s - 1].ptr;
      g.lay = m->lay[s - 1]->view();
      g.stored = m->lay[s - 1]->host.stored;
      g.c = c;
      g.inv = 1.0 / static_cast<double>(K);
      launch_moment_generic(g, st);
    }
    return;
  }
  Scratch& sc = g_scratch[dev.id];
  const bool lower = !only_order && d > 2;
  MomParams p;
  p.src[0] = src[0];
  p.src[1] = src[1];
  p.npass = npass;
  p.K = static_cast<uint32_t>(K);
  p.n = m->n;
  p.b = m->b;
  p.L = S - 1;
  p.top = m->data[S - 1].ptr;
  p.low = (S > 1 && !only_order) ? m->data[S - 2].ptr : nullptr;
  p.c = c;
  p.inv = 1.0 / static_cast<double>(K);
  // the top pair runs on the FP64 tensor cores when the rows allow TMA
  // bulk copies; otherwise on the DFMA kernel
  const bool use_dmma = dmma_supported(p);
  // sharding applies to the DMMA plan (the DFMA fallback computes all blocks)
  const bool sharded = use_dmma && sh.active() && !only_order;
  // orders <= d-2 beside the DMMA top pair: a lean kernel on the side
  // stream (joined at the end of this call) when they are few (it is
  // latency bound and hides under the top pair); else staged, in line
  // (the TMA-staged kernel handles any count when rows are 16-byte multiples)
  const bool side = lower && d - 2 <= 4 && use_dmma &&
                    (multiset_count(m->n, d - 2) <= 60000 || m->n % 2 == 0);
  bool joined = true;
  // The side-stream launch is deferred until the top kernel is queued: the
  // block scheduler hands SMs to the top kernel's CTAs first and the few
  // low-order CTAs (TMA-staged rows) run as SMs free up in its last wave.
  // Launched first, the old register-only kernel held ~1/4 of the SMs for
  // ~180 us and cost cfg1's top kernel 31 us (measured; CSB_LOW_DEFER=0).
  std::function<void()> side_launch;
  if (lower && d - 2 <= 4) {
    const int ST = d - 2;
    // the tables are looked up inside the launch: on the side path that
    // runs after the top kernel is queued, keeping the host work before
    // the step's first (and longest) kernel short
    auto make_params = [&dev, m, ST, npass, K, c, src](int W) {
      auto th = get_lower2_threads(dev, ST, m->n, W);
      Lower2Params lp;
      lp.src[0] = src[0];
      lp.src[1] = src[1];
      lp.npass = npass;
      lp.K = static_cast<uint32_t>(K);
      lp.n = m->n;
      lp.b = m->b;
      lp.threads = th->ptr;
      lp.nthreads = static_cast<uint32_t>(th->count);
      for (int s = 1; s <= ST; ++s) {
        lp.elems[s - 1] = get_lower_elems(dev, s, m->n, m->b, m->lay[s - 1]->host)->ptr;
        lp.m[s - 1] = m->data[s - 1].ptr;
      }
      lp.c = c;
      lp.inv = 1.0 / static_cast<double>(K);
      return lp;
    };
    if (side) {
      CSB_CUDA(cudaEventRecord(dev.fork, st));  // the low orders depend only on work queued so far
      side_launch = [&dev, ST, make_params, &side_tail, side_tail_ran, m, src, npass]() {
        // many elements: a thread owns 4 consecutive ones (shared prefix work)
        // (the TMA kernel only; same test as lower_tma_supported)
        const bool tma = m->n % 2 == 0 && m->n <= 4096 && rows_aligned16(src, npass);
        const int W = tma && ST >= 2 && multiset_count(m->n, ST) > 60000 ? 4 : 1;
        // W > 1: a thread's elements are strided over its prefix (negative W
        // selects that thread table), so a prefix's lanes read consecutive
        // staged columns
        const Lower2Params lp = make_params(W > 1 ? -W : W);
        {
          std::lock_guard<std::mutex> lk(dev.mu);
          CSB_CUDA(cudaStreamWaitEvent(dev.side, dev.fork, 0));
          ProfScope pl("moment_low", dev.side);
          if (tma)
            launch_moment_lower_tma(ST, W, lp, dev.side);
          else
            launch_moment_lower_side(ST, lp, dev.side);
        }
        if (side_tail) {  // takes dev.mu itself (plan/table caches)
          side_tail(dev.side);
          if (side_tail_ran) *side_tail_ran = true;
        }
        std::lock_guard<std::mutex> lk(dev.mu);
        CSB_CUDA(cudaEventRecord(dev.join, dev.side));
      };
      joined = false;
    } else {
      ProfScope ps("moment_low", st);
      const int W = multiset_count(m->n, ST) > 60000 ? 4 : 1;
      launch_moment_lower2(ST, W, make_params(W), st);
    }
  } else if (lower) {
    // orders <= d-2 of d > 6: element-parallel kernel
    ProfScope ps("moment_low", st);
    for (int s = 1; s <= d - 2; ++s) {
      auto el = get_lower_elems(dev, s, m->n, m->b, m->lay[s - 1]->host);
      LowerParams lp;
      lp.src[0] = src[0];
      lp.src[1] = src[1];
      lp.npass = npass;
      lp.n = m->n;
      lp.b = m->b;
      lp.elems = el->ptr;
      lp.count = el->count;
      lp.m = m->data[s - 1].ptr;
      lp.c = c;
      lp.inv = 1.0 / static_cast<double>(K);
      launch_moment_lower(s, lp, st);
    }
  }
  {
    auto plan = get_plan(dev, S, m->n, m->b, use_dmma, sharded ? sh.plan : nullptr, sharded ? sh.index : 0);
    p.rows = plan->d_rows.ptr;
    p.tiles = plan->d_tiles.ptr;
    p.pairs = plan->d_pairs.ptr;
    const uint64_t ntiles = plan->tiles.size();
    if (npass == 2 || use_dmma) p.scratch = sc.get(ntiles * plan->scratch_per_tile);
    if (use_dmma) {
      p.zeros = sc.get_zeros(static_cast<uint64_t>(dmma_chunk_rows(m->n, m->b)) * m->n);
      {
        ProfScope ps("moment_top", st);  // the DMMA kernel alone (bench roofline)
        launch_moment_top_dmma(p, static_cast<int>(ntiles), st);
      }
      if (!plan->tail.empty()) {
        ProfScope ps("moment_tail", st);  // the last column window on the CUDA cores
        MomParams pt = p;
        pt.rows = plan->d_tail_rows.ptr;
        pt.tail = plan->d_tail.ptr;
        pt.tail_warps = static_cast<uint32_t>(plan->tail.size() / 32);
        pt.scratch = sc.get_tail(tail_scratch_doubles());
        launch_moment_tail(pt, st);
      }
      if (side_launch) side_launch();
      ProfScope pm("mirror", st);
      const auto& LT = m->lay[S - 1];
      auto rt = sharded ? LT->diag_range(sh.lo(0), sh.hi(0)) : std::make_pair(0u, LT->ndiag);
      // in a stream step the next moms2cums stages these blocks anyway and
      // writes their copies (same values, one pass less over M)
      const bool fuse = defer_mirror && !sharded;
      auto ml = get_mirror_lists(*m->dev, S, m->b);
      if (fuse && ml.first && m2c_fuse_ok(S, m->n, m->b))
        m->mirror_defer |= 1u << (S - 1);
      else
        launch_mirror(S, p.top, LT->view(), LT->diag.ptr + rt.first, rt.second, m->n, m->b, ml.first, ml.second, st);
      if (p.low) {
        const auto& LL = m->lay[S - 2];
        auto rl = sharded ? LL->diag_range(sh.lo(1), sh.hi(1)) : std::make_pair(0u, LL->ndiag);
        auto ml1 = get_mirror_lists(*m->dev, S - 1, m->b);
        if (fuse && ml1.first && m2c_fuse_ok(S - 1, m->n, m->b))
          m->mirror_defer |= 1u << (S - 2);
        else
          launch_mirror(S - 1, p.low, LL->view(), LL->diag.ptr + rl.first, rl.second, m->n, m->b, ml1.first,
                        ml1.second, st);
        if (sharded && sh.comm) {
          // collective C2: every rank needs all of M_{d-1} (its own blocks
          // were just updated, the rest arrive from their owners)
          std::vector<uint64_t> off(sh.plan->count), cnt(sh.plan->count);
          for (int r = 0; r < sh.plan->count; ++r) {
            off[r] = LL->host.offset[sh.plan->low_blk[r]];
            cnt[r] = LL->host.offset[sh.plan->low_blk[r + 1]] - off[r];
          }
          ProfScope pc("allgather", st);
          sh.comm->allgather_ranges(p.low, off.data(), cnt.data(), st);
        }
      }
    } else {
      ProfScope ps("moment_top", st);
      launch_moment_pair(p, static_cast<int>(ntiles), true, st);
    }
  }
  if (!joined) CSB_CUDA(cudaStreamWaitEvent(st, dev.join, 0));
}

void check_batch(uint64_t rows, uint64_t cols, const char* what) {
  if (rows < 1) fail(CSB_EINVAL, std::string(what) + ": empty batch");
  if (cols < 1) fail(CSB_EINVAL, std::string(what) + ": no columns");
  if (rows > 0xffffffffull) fail(CSB_EINVAL, std::string(what) + ": too many rows");
}

// The vector width of the reference's knorm fold as built for this host
// (-march=native): AVX-512 builds square-and-add 8 entries per chunk, AVX2
// builds 4 (the oracle pins both; symten.cpp:266).  The device reproduces
// that build bit for bit.
int host_fold_width() {
  static const int w = [] {
    __builtin_cpu_init();
    return (__builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512dq")) ? 8 : 4;
  }();
  return w;
}

// moms2cums into c, with per-block partial squared norms for every order.
struct NormScratch {
  uint32_t exact_mask = 0;  // orders whose partials are already exact (moms2cums' in-block pass)
  // one device buffer [d sums | 3 n diagonals | per-block partials of orders
  // 1..d]: the report reads it back with a single copy and folds the blocks
  // on the host (knorm's sequential block fold, symten.cpp:268: a chain of
  // nblocks dependent adds costs a CPU core a fraction of what it costs one
  // GPU thread -- cfg2: 12376 blocks, 0.097 ms in the kernel)
  DevBuf<double> all;
  std::vector<uint64_t> poff;  // d + 1 offsets of the partials inside `all`
  int pd = 0, pn = 0, pb = 0;
  void ensure(const csb_series* c);
  double* part(int s) { return all.ptr + poff[s - 1]; }
  uint64_t nblk(int s) const { return poff[s] - poff[s - 1]; }
  double* out() { return all.ptr; }
  DevBuf<double> diag;                  // gathered diagonal of a sharded C_d
  // pinned: the report's D2H is a direct DMA, not a staged pageable copy
  struct Pinned {
    double* p = nullptr;
    size_t n = 0;
    Pinned() = default;
    Pinned(const Pinned&) = delete;
    Pinned& operator=(const Pinned&) = delete;
    ~Pinned() {
      if (p) cudaFreeHost(p);
    }
    void resize(size_t k) {
      if (k <= n) return;
      if (p) cudaFreeHost(p);
      p = nullptr;
      n = 0;
      CSB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p), k * sizeof(double)));
      n = k;
    }
    double* data() { return p; }
    const double* data() const { return p; }
  } host;
};

void exact_partials(const csb_series* c, int s, double* partial, cudaStream_t st, uint64_t lo, uint64_t hi,
                    double k);

void NormScratch::ensure(const csb_series* c) {
  if (pd == c->d && pn == c->n && pb == c->b && all.ptr) return;
  pd = c->d;
  pn = c->n;
  pb = c->b;
  poff.assign(static_cast<size_t>(pd) + 1, 0);
  poff[0] = static_cast<uint64_t>(pd) + 3ull * pn;
  for (int s = 1; s <= pd; ++s) poff[s] = poff[s - 1] + c->lay[s - 1]->host.nblocks;
  all.alloc(poff[pd]);
  CSB_CUDA(cudaMemsetAsync(all.ptr, 0, all.bytes(), c->dev->stream));
  CSB_CUDA(cudaStreamSynchronize(c->dev->stream));
  host.resize(poff[pd]);
}

// orders [first, last] of moms2cums (C_1 is a copy of M_1), with per-block
// partial squared norms; the stream step may run the low orders early on
// the side stream (run_moments' side_tail) and the rest here
void run_moms2cums(const csb_series* m, csb_series* c, NormScratch& ns, cudaStream_t st,
                   const ShardCtx& sh = ShardCtx{}, int first = 1, int last = 0) {
  const int d = m->d;
  if (last <= 0) last = d;
  // (checked before any order is converted: s = 16 alone is 10^10 partitions per element)
  if (last > kMaxCumOrderAny) fail(CSB_EINVAL, "partitions: s must be in [1, 16]");
  ns.ensure(m);
  Device& dev = *m->dev;
  bool side_norms = false;
  ProfScope ps("moms2cums", st);
  const auto& L1 = m->lay[0];
  if (first <= 1) {
    launch_copy_c1(m->data[0].ptr, c->data[0].ptr, ns.part(1), L1->view(), L1->host.nblocks,
                   L1->host.stored, st);
    ns.exact_mask &= ~1u;
  }
  for (int s = std::max(2, first); s <= last; ++s) {
    if (s > kMaxCumOrder) {
      // any-order kernel: restricted growth strings walked on the device
      if (s > kMaxCumOrderAny) fail(CSB_EINVAL, "partitions: s must be in [1, 16]");
      if (sh.active()) fail(CSB_EINVAL, "sharding supports cumulants up to order 6");
      GenM2CParams g;
      g.m = m->data[s - 1].ptr;
      g.c = c->data[s - 1].ptr;
      for (int k = 1; k < s; ++k) g.lower[k - 1] = c->data[k - 1].ptr;
      for (int k = 1; k <= s; ++k) g.lay[k - 1] = m->lay[k - 1]->view();
      g.n = m->n;
      g.b = m->b;
      g.s = s;
      g.stored = m->lay[s - 1]->host.stored;
      ProfScope po("m2c_generic", st);
      launch_moms2cums_generic(g, st);
      ns.exact_mask &= ~(1u << (s - 1));
      continue;
    }
    M2CParams p;
    p.m = m->data[s - 1].ptr;
    p.c = c->data[s - 1].ptr;
    for (int k = 1; k < s; ++k) p.lower[k - 1] = c->data[k - 1].ptr;
    for (int k = 1; k <= s; ++k) p.lay[k - 1] = m->lay[k - 1]->view();
    p.n = m->n;
    p.b = m->b;
    // the block's exact norm partial inside moms2cums (one thread chains the
    // assembled block while the CTA writes it out) pays for few blocks; with
    // thousands the chain-per-lane kernel of finalize_norms is cheaper
    // (measured: cfg2 C_5, 4368 blocks, 0.293 -> 0.187 ms against +0.039 ms there;
    // cfg1/cfg2 C_4, 1365 blocks: in-kernel wins)
    p.fold_width = m->lay[s - 1]->host.nblocks > 3000 ? 0 : host_fold_width();
    p.subs = get_subs(*m->dev, s, m->n, m->b)->ptr;
    {
      uint64_t vol = 1;
      for (int k = 0; k < s; ++k) vol *= static_cast<uint64_t>(m->b);
      if (vol <= (1ull << 20)) {  // canonical-position lists for full blocks
        auto cl = get_canon(*m->dev, s, m->b);
        p.canon = cl.first;
        p.canon_off = cl.second;
        auto ml = get_mirror_lists(*m->dev, s, m->b);
        p.mlist = ml.first;
        p.mlist_off = ml.second;
        auto cp = get_copy_lists(*m->dev, s, m->b);
        p.cstart = cp.first;
        p.cdst = cp.second;
      }
    }
    if (m->mirror_defer >> (s - 1) & 1u) {
      p.mfix = m->data[s - 1].ptr;  // write M_s's copies too (run_moments deferred them)
      m->mirror_defer &= ~(1u << (s - 1));
    }
    if ((s == 6 || s == 5) && m->b == 4 && !(s == d && sh.active()))
      p.order = get_m2c_order(*m->dev, s, m->n, m->b)->ptr;  // persistent kernel
    if (s == d && sh.active()) {
      // C_d only for the owned blocks; the other partials stay zero so a
      // sum over ranks reproduces the unsharded partial array exactly
      const uint64_t lo = sh.lo(0), hi = sh.hi(0);
      CSB_CUDA(cudaMemsetAsync(ns.part(s), 0, ns.nblk(s) * sizeof(double), st));
      p.blk0 = lo;
      p.partial = ns.part(s) + lo;
      const bool exact = launch_moms2cums_v2(s, p, hi - lo, st);
      ns.exact_mask = exact ? ns.exact_mask | (1u << (s - 1)) : ns.exact_mask & ~(1u << (s - 1));
    } else {
      p.blk0 = 0;
      p.partial = ns.part(s);
      static const char* const tags[] = {"m2c_1", "m2c_2", "m2c_3", "m2c_4", "m2c_5", "m2c_6"};
      bool exact;
      {
        ProfScope po(tags[s - 1], st);
        exact = launch_moms2cums_v2(s, p, m->lay[s - 1]->host.nblocks, st);
      }
      if (!exact && s < last && s <= kMaxCumOrder && st != dev.side && !sh.active()) {
        // C_s is final: its exact norm partials on the side stream, under the
        // next order's conversion, instead of in the report's critical path
        std::lock_guard<std::mutex> lk(dev.mu);  // the side stream and its events are shared per device
        CSB_CUDA(cudaEventRecord(dev.nfork, st));
        CSB_CUDA(cudaStreamWaitEvent(dev.side, dev.nfork, 0));
        {
          ProfScope pk("norm_partials_side", dev.side);
          exact_partials(c, s, ns.part(s), dev.side, 0, m->lay[s - 1]->host.nblocks, 2.0);
        }
        CSB_CUDA(cudaEventRecord(dev.njoin, dev.side));
        side_norms = true;
        exact = true;
      }
      ns.exact_mask = exact ? ns.exact_mask | (1u << (s - 1)) : ns.exact_mask & ~(1u << (s - 1));
    }
  }
  if (side_norms) {
    std::lock_guard<std::mutex> lk(dev.mu);
    CSB_CUDA(cudaStreamWaitEvent(st, dev.njoin, 0));  // (long done when the last order ends)
  }
  c->window_len = m->window_len;
}

// Device offsets of the diagonals c_2[i,i], c_3[i,i,i], c_4[i,i,i,i].
struct DiagTables {
  DevBuf<uint64_t> off[3];
  DevBuf<uint64_t> iota;  // 0..n-1
};

DiagTables& diag_tables(const csb_series* c) {
  static thread_local std::map<std::tuple<int, int, int, int>, DiagTables> cache;
  auto& t = cache[{c->dev->id, c->n, c->b, c->d}];
  if (!t.off[0].ptr) {
    for (int q = 0; q < 3; ++q) {
      const int order = q + 2;
      if (order > c->d) continue;
      std::vector<uint64_t> off(c->n);
      int idx[8];
      for (int i = 0; i < c->n; ++i) {
        for (int k = 0; k < order; ++k) idx[k] = i;
        off[i] = c->lay[order - 1]->host.element_offset(idx);
      }
      t.off[q].alloc(c->n);
      h2d_sync(t.off[q].ptr, off.data(), t.off[q].bytes());
    }
    std::vector<uint64_t> io(c->n);
    for (int i = 0; i < c->n; ++i) io[i] = static_cast<uint64_t>(i);
    t.iota.alloc(c->n);
    h2d_sync(t.iota.ptr, io.data(), t.iota.bytes());
  }
  return t;
}

// Exact per-block norm partials of order s (all blocks, or [lo, hi) of a
// shard with zeros elsewhere, summed over ranks: x + 0 == x).
void exact_partials(const csb_series* c, int s, double* partial, cudaStream_t st, uint64_t lo, uint64_t hi,
                    double k) {
  const auto& L = c->lay[s - 1];
  if (lo > 0 || hi < L->host.nblocks) CSB_CUDA(cudaMemsetAsync(partial, 0, L->host.nblocks * sizeof(double), st));
  launch_knorm_exact(c->data[s - 1].ptr, L->view(), lo, hi - lo, k, host_fold_width(), partial, st);
}

// Norm sums of orders 1..d + diagonals, to the host: exact per-block
// partials (each block summed in storage order), then the block-order fold
// -- knorm's own sequence, so norms and nu are the reference's bit for bit.
void fold_norms_host(const csb_series* c, NormScratch& ns);

void finalize_norms(const csb_series* c, NormScratch& ns, cudaStream_t st, const ShardCtx& sh = ShardCtx{},
                    bool wait = true) {
  const int d = c->d;
  ns.ensure(c);
  {
    ProfScope ps("norm_partials", st);
    for (int s = 1; s <= d; ++s) {
      const uint64_t nb = c->lay[s - 1]->host.nblocks;
      const bool shard = sh.active() && s == d;  // C_d: only the owned blocks are valid here
      if (!(ns.exact_mask >> (s - 1) & 1u))
        exact_partials(c, s, ns.part(s), st, shard ? sh.lo(0) : 0, shard ? sh.hi(0) : nb, 2.0);
      if (shard && sh.comm) sh.comm->allreduce_sum(ns.part(s), nb, st);  // collective C3
    }
    ns.exact_mask = 0;  // (the reduced C_d partials must not be reduced again)
  }
  NormParams p;
  p.norders = d;
  p.fold = false;  // the block fold runs on the host (fold_norms_host); the kernel gathers the diagonals
  DiagTables& dt = diag_tables(c);
  for (int q = 0; q < 3; ++q) {
    p.diag_src[q] = (q + 2 <= d) ? c->data[q + 1].ptr : nullptr;
    p.diag_off[q] = dt.off[q].ptr;
  }
  if (sh.active() && d <= 4) {
    // the diagonal of C_d is sharded: owners contribute, others add zeros
    const auto& L = c->lay[d - 1];
    if (ns.diag.count < static_cast<uint64_t>(c->n)) ns.diag.alloc(c->n);
    launch_diag_pick(c->data[d - 1].ptr, dt.off[d - 2].ptr, L->host.offset[sh.lo(0)], L->host.offset[sh.hi(0)],
                     c->n, ns.diag.ptr, st);
    if (sh.comm) sh.comm->allreduce_sum(ns.diag.ptr, c->n, st);
    p.diag_src[d - 2] = ns.diag.ptr;
    p.diag_off[d - 2] = dt.iota.ptr;
  }
  p.n = c->n;
  p.out = ns.out();
  {
    ProfScope ps("norms", st);
    launch_norm_finalize(p, st);
  }
  // diagonals and every order's per-block partials in one copy
  CSB_CUDA(cudaMemcpyAsync(ns.host.data(), ns.all.ptr, ns.all.bytes(), cudaMemcpyDeviceToHost, st));
  if (wait) {
    CSB_CUDA(cudaStreamSynchronize(st));
    fold_norms_host(c, ns);
  }  // (a captured step waits after the graph launch, then folds)
}

// The blocks' partial sums folded in block order, acc = acc + mult * s
// (symten.cpp:268; the product is rounded, the reference build does not
// contract it -- this file is compiled -ffp-contract=off): the reference's
// sequence bit for bit, after finalize_norms' copy has landed.
void fold_norms_host(const csb_series* c, NormScratch& ns) {
  double* h = ns.host.data();
  for (int s = 1; s <= c->d; ++s) {
    const double* part = h + ns.poff[s - 1];
    const std::vector<double>& mult = c->lay[s - 1]->mult_host;
    const uint64_t nb = ns.nblk(s);
    double acc = 0.0;
    for (uint64_t r = 0; r < nb; ++r) {
      const double prod = mult[r] * part[r];  // rounded product, then the add (no contraction)
      acc = acc + prod;
    }
    h[s - 1] = acc;
  }
}

// make_window_report from the finalized sums (gauge.cpp:35-41,64-94,142-154).
void build_report(const csb_series* c, const NormScratch& ns, uint64_t window, csb_report* r) {
  const int d = c->d;
  if (d < 2) fail(CSB_EINVAL, "make_window_report: needs orders up to 2");
  std::memset(r, 0, sizeof(*r));
  r->window = window;
  r->rows = c->window_len;
  const double* sums = ns.host.data();
  r->norm_c1 = std::sqrt(sums[0]);
  r->norm_c2 = std::sqrt(sums[1]);
  r->n_nu = 0;
  for (int o = 3; o <= d; ++o) {
    const double n2 = r->norm_c2;
    if (n2 <= 0.0) fail(CSB_EDOMAIN, "nu: vanishing second-order cumulant norm");
    r->nu[r->n_nu++] = std::sqrt(sums[o - 1]) / std::pow(n2, 0.5 * static_cast<double>(o));
  }
  const double* c2 = sums + d;
  if (d >= 3) {
    const double* c3 = sums + d + c->n;
    double best = 0.0;
    for (int i = 0; i < c->n; ++i) {
      if (c2[i] <= 0.0) fail(CSB_EDOMAIN, "max_abs_diag_skewness: zero variance");
      best = std::max(best, std::abs(c3[i]) / std::pow(c2[i], 1.5));
    }
    r->has_skewness = 1;
    r->max_abs_skewness = best;
  }
  if (d >= 4) {
    const double* c4 = sums + d + 2 * c->n;
    double best = 0.0;
    for (int i = 0; i < c->n; ++i) {
      if (c2[i] <= 0.0) fail(CSB_EDOMAIN, "max_abs_diag_kurtosis: zero variance");
      best = std::max(best, std::abs(c4[i]) / (c2[i] * c2[i]));
    }
    r->has_kurtosis = 1;
    r->max_abs_kurtosis = best;
  }
}

double knorm_device(const csb_series* s, int order, double k, cudaStream_t st) {
  if (!(k >= 1.0)) fail(CSB_EINVAL, "knorm: k must be >= 1");
  const auto& L = s->lay[order - 1];
  DevBuf<double> partial(L->host.nblocks);
  exact_partials(s, order, partial.ptr, st, 0, L->host.nblocks, k);
  NormParams p;
  p.norders = 1;
  p.partial[0] = partial.ptr;
  p.mult[0] = L->mult.ptr;
  p.nblocks[0] = L->host.nblocks;
  p.n = 0;
  DevBuf<double> out(1);
  p.out = out.ptr;
  launch_norm_finalize(p, st);
  double acc = 0.0;
  CSB_CUDA(cudaMemcpyAsync(&acc, out.ptr, sizeof(double), cudaMemcpyDeviceToHost, st));
  CSB_CUDA(cudaStreamSynchronize(st));
  if (k == 2.0) return std::sqrt(acc);
  if (k == 1.0) return acc;
  return std::pow(acc, 1.0 / k);
}

}  // namespace
}  // namespace csb

// ---------------------------------------------------------------------------
struct csb_stream {
  csb_stream_config cfg{};
  Device* dev = nullptr;
  cudaStream_t st = nullptr;
  DevBuf<double> ring;      // window_len x dim, head = oldest row
  uint64_t head = 0;
  DevBuf<double> staging;   // update_len x dim
  // asynchronous ingestion (csb_stream_upload): two batch buffers filled on
  // a copy stream while earlier steps run; FIFO of uploaded slots
  DevBuf<double> upload[2];
  cudaStream_t copy_st = nullptr;
  cudaEvent_t uploaded[2] = {nullptr, nullptr};  // H2D of the slot done (copy stream)
  cudaEvent_t consumed[2] = {nullptr, nullptr};  // the step that read the slot done (engine stream)
  int queue[2] = {0, 0};
  int queued = 0, next_slot = 0;
  bool slot_used[2] = {false, false};
  std::unique_ptr<csb_series> M, C;
  uint64_t window = 0;
  uint64_t steps_since_resync = 0;
  NormScratch ns;
  int early_m2c = 0;  // moms2cums orders already enqueued on the side stream this step
  bool norms_valid = false;
  std::shared_ptr<ShardPlan> splan;  // shard_count > 1
  std::shared_ptr<Comm> comm;        // kept alive for the stream's lifetime
  ShardCtx sh;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  // One CUDA graph per (ring head, batch pointer, report?): a step's launch
  // sequence depends on nothing else, and the ring revisits window_len /
  // gcd(window_len, update_len) heads.  The first visit of a key runs
  // eagerly (tables, scratch and plans get built), the second is captured,
  // later ones are one cudaGraphLaunch -- the small configurations are
  // launch-bound otherwise (cfg0: ~20 launches around a 0.09 ms kernel).
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    bool seen = false;
    uint32_t exact_mask_after = 0;
    int early_m2c = 0;
    uint64_t launches = 0;
    uint64_t scratch_gen = 0;  // g_scratch_gen at capture: the graph's scratch pointers are valid under it
    std::thread::id owner;     // the capturing thread (scratch buffers are per thread)
  };
  std::map<std::tuple<uint64_t, const double*, int>, StepGraph> graphs;
  bool use_graphs = true;
  uint64_t graph_replays = 0;
  ~csb_stream() {
    for (auto& [key, g] : graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (int k = 0; k < 2; ++k) {
      if (uploaded[k]) cudaEventDestroy(uploaded[k]);
      if (consumed[k]) cudaEventDestroy(consumed[k]);
    }
    if (copy_st) {
      cudaStreamSynchronize(copy_st);
      cudaStreamDestroy(copy_st);
    }
  }
};

namespace {

template <class F>
int guard(F&& f) {
  try {
    f();
    return CSB_OK;
  } catch (const csb::Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_last_error = e.what();
    return CSB_ERUNTIME;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return CSB_ERUNTIME;
  }
}

void stream_exchange_and_update(csb_stream* s, const double* x_dev) {
  const auto& cfg = s->cfg;
  const uint64_t T = cfg.window_len, p = cfg.update_len, n = cfg.dim;
  // outgoing rows: ring[head .. head+p) with wrap (WindowBuffer::exchange, stream.cpp:39-54)
  RowSource out;
  const uint64_t first = std::min(p, T - s->head);
  out.seg0 = s->ring.ptr + s->head * n;
  out.len0 = static_cast<uint32_t>(first);
  out.seg1 = s->ring.ptr;
  out.len1 = static_cast<uint32_t>(p - first);
  const bool resync = cfg.resync_every > 0 && s->steps_since_resync + 1 >= cfg.resync_every;
  if (!resync) {
    RowSource src[2];
    src[0].seg0 = x_dev;
    src[0].len0 = static_cast<uint32_t>(p);
    src[1] = out;
    // C_1 .. C_{d-2} need only M_1 .. M_{d-2} (the low-order kernel's): on
    // the side stream, under the top pair (cfg2: C_1..C_4, 0.04 ms off the step)
    const int early = s->sh.active() ? 0 : std::min(4, cfg.max_order - 2);
    std::function<void(cudaStream_t)> tail;
    if (early >= 1)
      tail = [s, early](cudaStream_t side) { run_moms2cums(s->M.get(), s->C.get(), s->ns, side, s->sh, 1, early); };
    bool ran = false;
    run_moments(s->M.get(), src, 2, p, static_cast<double>(p) / static_cast<double>(T), s->st, 0, s->sh, true,
                tail, &ran);
    s->early_m2c = ran ? early : 0;
    g_rows_read.fetch_add(2 * p, std::memory_order_relaxed);
  } else {
    s->early_m2c = 0;
  }
  // incoming rows take the outgoing slots
  CSB_CUDA(cudaMemcpyAsync(s->ring.ptr + s->head * n, x_dev, first * n * sizeof(double),
                           cudaMemcpyDeviceToDevice, s->st));
  if (p > first)
    CSB_CUDA(cudaMemcpyAsync(s->ring.ptr, x_dev + first * n, (p - first) * n * sizeof(double),
                             cudaMemcpyDeviceToDevice, s->st));
  s->head = (s->head + p) % T;
  if (resync) {
    // moment_series(materialize()) (stream.cpp:92-95): arrival order from head
    RowSource src[2];
    src[0].seg0 = s->ring.ptr + s->head * n;
    src[0].len0 = static_cast<uint32_t>(T - s->head);
    src[0].seg1 = s->ring.ptr;
    src[0].len1 = static_cast<uint32_t>(s->head);
    run_moments(s->M.get(), src, 1, T, 0.0, s->st, 0, s->sh);
    g_rows_read.fetch_add(T, std::memory_order_relaxed);
    s->steps_since_resync = 0;
  } else {
    ++s->steps_since_resync;
  }
}

int stream_step_impl(csb_stream* s, const double* x, bool on_device, uint64_t rows, uint64_t cols,
                     csb_step_timing* timing, csb_report* report) {
  return guard([&] {
    require(s != nullptr, "step: null stream");
    const auto& cfg = s->cfg;
    if (rows != cfg.update_len || cols != static_cast<uint64_t>(cfg.dim))
      fail(CSB_EINVAL, "step: batch does not match the configured update");
    CSB_CUDA(cudaSetDevice(s->dev->id));
    const double* xd = x;
    if (!on_device) {
      CSB_CUDA(cudaMemcpyAsync(s->staging.ptr, x, rows * cols * sizeof(double), cudaMemcpyHostToDevice, s->st));
      xd = s->staging.ptr;
    }
    // the enqueue-only part of a step (no host wait): what a graph captures
    const auto enqueue = [&](bool want_report) {
      if (timing) CSB_CUDA(cudaEventRecord(s->ev[0], s->st));  // StepTiming only when asked
      {
        ProfScope pu("step_update", s->st);
        stream_exchange_and_update(s, xd);
      }
      if (timing) CSB_CUDA(cudaEventRecord(s->ev[1], s->st));
      {
        ProfScope pc("step_m2c", s->st);
        run_moms2cums(s->M.get(), s->C.get(), s->ns, s->st, s->sh, 1 + s->early_m2c);
      }
      if (timing) CSB_CUDA(cudaEventRecord(s->ev[2], s->st));
      if (want_report) {
        ProfScope pr("step_report", s->st);
        finalize_norms(s->C.get(), s->ns, s->st, s->sh, false);
      }
    };
    const bool resync = cfg.resync_every > 0 && s->steps_since_resync + 1 >= cfg.resync_every;
    const bool graphable = s->use_graphs && !timing && !g_prof.on && !s->sh.active() && !resync &&
                           s->M->mirror_defer == 0;
    csb_stream::StepGraph* sg = nullptr;
    if (graphable) {
      const auto key = std::make_tuple(s->head, xd, report ? 1 : 0);
      auto it = s->graphs.find(key);
      if (it != s->graphs.end()) sg = &it->second;
      else if (s->graphs.size() < 256) sg = &s->graphs[key];  // (callers cycling through many buffers stay eager)
    }
    if (sg && sg->exec && (sg->scratch_gen != g_scratch_gen.load(std::memory_order_relaxed) ||
                           sg->owner != std::this_thread::get_id())) {
      // a scratch buffer moved since the capture, or another thread (with its own scratch) steps now
      cudaGraphExecDestroy(sg->exec);
      sg->exec = nullptr;  // seen stays set: captured again below
    }
    if (sg && sg->exec) {
      // replay: the device work of the captured step, then its host-side bookkeeping
      CSB_CUDA(cudaGraphLaunch(sg->exec, s->st));
      s->head = (s->head + cfg.update_len) % cfg.window_len;
      ++s->steps_since_resync;
      g_rows_read.fetch_add(2 * cfg.update_len, std::memory_order_relaxed);
      s->early_m2c = sg->early_m2c;
      s->ns.exact_mask = sg->exact_mask_after;
      s->C->window_len = s->M->window_len;
      add_launches(sg->launches);
      ++s->graph_replays;
    } else if (sg && sg->seen) {
      // second visit of this key: capture the step, then run it from the graph
      const uint64_t head0 = s->head, since0 = s->steps_since_resync;
      const uint32_t mask0 = s->ns.exact_mask;
      const uint64_t l0 = launch_count();
      const uint64_t rows0 = g_rows_read.load(std::memory_order_relaxed);
      cudaGraph_t graph = nullptr;
      bool ok = cudaStreamBeginCapture(s->st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
      if (ok) {
        try {
          enqueue(report != nullptr);
        } catch (const std::exception&) {
          ok = false;
        }
        if (cudaStreamEndCapture(s->st, &graph) != cudaSuccess || !graph) ok = false;
      }
      if (ok && cudaGraphInstantiate(&sg->exec, graph, 0) != cudaSuccess) ok = false;
      if (graph) cudaGraphDestroy(graph);
      if (ok) {
        sg->scratch_gen = g_scratch_gen.load(std::memory_order_relaxed);
        sg->owner = std::this_thread::get_id();
        sg->launches = launch_count() - l0;
        sg->exact_mask_after = s->ns.exact_mask;
        sg->early_m2c = s->early_m2c;
        CSB_CUDA(cudaGraphLaunch(sg->exec, s->st));
      } else {
        // not capturable here: forget graphs for this stream and run the step eagerly
        cudaGetLastError();
        sg->exec = nullptr;
        s->use_graphs = false;
        s->head = head0;
        s->steps_since_resync = since0;
        s->ns.exact_mask = mask0;
        s->M->mirror_defer = 0;
        g_rows_read.store(rows0, std::memory_order_relaxed);
        enqueue(report != nullptr);
      }
    } else {
      if (sg) sg->seen = true;
      enqueue(report != nullptr);
    }
    s->norms_valid = false;
    ++s->window;
    if (report) {
      CSB_CUDA(cudaStreamSynchronize(s->st));
      fold_norms_host(s->C.get(), s->ns);
      s->norms_valid = true;
      build_report(s->C.get(), s->ns, s->window, report);
    }
    if (timing) {
      CSB_CUDA(cudaEventSynchronize(s->ev[2]));
      float a = 0, b = 0;
      CSB_CUDA(cudaEventElapsedTime(&a, s->ev[0], s->ev[1]));
      CSB_CUDA(cudaEventElapsedTime(&b, s->ev[1], s->ev[2]));
      timing->update_s = a * 1e-3;
      timing->moms2cums_s = b * 1e-3;
    }
  });
}

}  // namespace

extern "C" {

int csb_version(void) { return 1; }
const char* csb_last_error(void) { return g_last_error.c_str(); }

int csb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int csb_set_device(int d) {
  return guard([&] {
    ensure_device();
    CSB_CUDA(cudaSetDevice(d));
  });
}

uint64_t csb_rows_read(void) { return g_rows_read.load(std::memory_order_relaxed); }

int csb_layout_size(int order, int dim, int block, uint64_t* stored, uint64_t* blocks) {
  return guard([&] {
    require(stored && blocks, "layout_size: null output");
    Layout L(order, dim, block);
    *stored = L.stored;
    *blocks = L.nblocks;
  });
}

int csb_block_multiplicity(const int* j, int order, uint64_t* out) {
  return guard([&] {
    require(order >= 1, "block_multiplicity: empty index");
    require(order <= 20, "block_multiplicity: order too large for exact count");
    for (int k = 1; k < order; ++k)
      require(j[k - 1] <= j[k], "block_multiplicity: index not non-decreasing");
    *out = block_multiplicity(j, order);
  });
}

int csb_series_create(int dim, int max_order, int block, csb_series** out) {
  return guard([&] {
    require(out != nullptr, "series_create: null output");
    *out = make_series(dim, max_order, block).release();
  });
}

int csb_series_destroy(csb_series* s) {
  return guard([&] { delete s; });
}

int csb_series_copy(csb_series* dst, const csb_series* src) {
  return guard([&] {
    require(dst && src, "series_copy: null series");
    require(dst->n == src->n && dst->d == src->d && dst->b == src->b, "series_copy: shape mismatch");
    for (int k = 0; k < src->d; ++k)
      CSB_CUDA(cudaMemcpyAsync(dst->data[k].ptr, src->data[k].ptr, src->data[k].bytes(),
                               cudaMemcpyDeviceToDevice, src->dev->stream));
    CSB_CUDA(cudaStreamSynchronize(src->dev->stream));
    dst->window_len = src->window_len;
  });
}

int csb_series_shape(const csb_series* s, int* dim, int* max_order, int* block, uint64_t* wl) {
  return guard([&] {
    require(s != nullptr, "null series");
    if (dim) *dim = s->n;
    if (max_order) *max_order = s->d;
    if (block) *block = s->b;
    if (wl) *wl = s->window_len;
  });
}

int csb_series_set_window_len(csb_series* s, uint64_t wl) {
  return guard([&] {
    require(s != nullptr, "null series");
    s->window_len = wl;
  });
}

int csb_series_stored(const csb_series* s, int order, uint64_t* stored) {
  return guard([&] {
    check_order(s, order);
    *stored = s->lay[order - 1]->host.stored;
  });
}

int csb_series_device_ptr(const csb_series* s, int order, double** dev) {
  return guard([&] {
    check_order(s, order);
    *dev = s->data[order - 1].ptr;
  });
}

int csb_series_upload(csb_series* s, int order, const double* host, uint64_t count) {
  return guard([&] {
    check_order(s, order);
    require(count == s->lay[order - 1]->host.stored, "series_upload: size mismatch");
    h2d_sync(s->data[order - 1].ptr, host, count * sizeof(double));
  });
}

int csb_series_download(const csb_series* s, int order, double* host, uint64_t count) {
  return guard([&] {
    check_order(s, order);
    require(count == s->lay[order - 1]->host.stored, "series_download: size mismatch");
    CSB_CUDA(cudaStreamSynchronize(s->dev->stream));
    CSB_CUDA(cudaMemcpy(host, s->data[order - 1].ptr, count * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

int csb_series_gather(const csb_series* s, int order, const uint64_t* offsets, uint64_t count, double* host) {
  return guard([&] {
    check_order(s, order);
    require(count == 0 || (offsets && host), "series_gather: null argument");
    if (!count) return;
    const uint64_t stored = s->lay[order - 1]->host.stored;
    for (uint64_t i = 0; i < count; ++i)
      if (offsets[i] >= stored) fail(CSB_ERANGE, "series_gather: offset out of range");
    cudaStream_t st = s->dev->stream;
    DevBuf<uint64_t> off(count);
    DevBuf<double> out(count);
    CSB_CUDA(cudaMemcpyAsync(off.ptr, offsets, count * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    launch_gather(s->data[order - 1].ptr, off.ptr, count, out.ptr, st);
    CSB_CUDA(cudaMemcpyAsync(host, out.ptr, count * sizeof(double), cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
  });
}

static void moment_series_impl(csb_series* out, const double* xd, uint64_t rows, uint64_t,
                               const ShardCtx& sh = ShardCtx{}) {
  RowSource src[2];
  src[0].seg0 = xd;
  src[0].len0 = static_cast<uint32_t>(rows);
  run_moments(out, src, 1, rows, 0.0, out->dev->stream, 0, sh);
  out->window_len = rows;
  g_rows_read.fetch_add(rows, std::memory_order_relaxed);
}

int csb_moment_series(csb_series* out, const double* x, uint64_t rows, uint64_t cols) {
  return guard([&] {
    require(out != nullptr, "moment_series: null series");
    check_batch(rows, cols, "moment_series");
    require(cols == static_cast<uint64_t>(out->n), "moment_series: dimension mismatch");
    DevBuf<double> xd(rows * cols);
    CSB_CUDA(cudaMemcpyAsync(xd.ptr, x, xd.bytes(), cudaMemcpyHostToDevice, out->dev->stream));
    moment_series_impl(out, xd.ptr, rows, cols);
    CSB_CUDA(cudaStreamSynchronize(out->dev->stream));
  });
}

int csb_moment_series_dev(csb_series* out, const double* x, uint64_t rows, uint64_t cols) {
  return guard([&] {
    require(out != nullptr, "moment_series: null series");
    check_batch(rows, cols, "moment_series");
    require(cols == static_cast<uint64_t>(out->n), "moment_series: dimension mismatch");
    moment_series_impl(out, x, rows, cols);
    CSB_CUDA(cudaStreamSynchronize(out->dev->stream));
  });
}

int csb_moment_tensor(csb_series* out, int order, const double* x, uint64_t rows, uint64_t cols) {
  return guard([&] {
    check_order(out, order);
    check_batch(rows, cols, "moment_tensor");
    require(cols == static_cast<uint64_t>(out->n), "moment_tensor: dimension mismatch");
    DevBuf<double> xd(rows * cols);
    CSB_CUDA(cudaMemcpyAsync(xd.ptr, x, xd.bytes(), cudaMemcpyHostToDevice, out->dev->stream));
    RowSource src[2];
    src[0].seg0 = xd.ptr;
    src[0].len0 = static_cast<uint32_t>(rows);
    run_moments(out, src, 1, rows, 0.0, out->dev->stream, order);
    g_rows_read.fetch_add(rows, std::memory_order_relaxed);
    CSB_CUDA(cudaStreamSynchronize(out->dev->stream));
  });
}

static void update_impl(csb_series* m, const double* in, const double* outg, uint64_t rows) {
  RowSource src[2];
  src[0].seg0 = in;
  src[0].len0 = static_cast<uint32_t>(rows);
  src[1].seg0 = outg;
  src[1].len0 = static_cast<uint32_t>(rows);
  run_moments(m, src, 2, rows, static_cast<double>(rows) / static_cast<double>(m->window_len),
              m->dev->stream);
  g_rows_read.fetch_add(2 * rows, std::memory_order_relaxed);
}

static void check_update(const csb_series* m, uint64_t rows, uint64_t cols) {
  require(m != nullptr, "moments_update: null series");
  check_batch(rows, cols, "moments_update");
  if (rows > m->window_len) fail(CSB_EINVAL, "moments_update: batch longer than the window");
  if (cols != static_cast<uint64_t>(m->n)) fail(CSB_EINVAL, "moments_update: dimension mismatch");
}

int csb_moments_update(csb_series* m, const double* in, const double* outg, uint64_t rows, uint64_t cols) {
  return guard([&] {
    check_update(m, rows, cols);
    DevBuf<double> xd(2 * rows * cols);
    const uint64_t nb = rows * cols * sizeof(double);
    CSB_CUDA(cudaMemcpyAsync(xd.ptr, in, nb, cudaMemcpyHostToDevice, m->dev->stream));
    CSB_CUDA(cudaMemcpyAsync(xd.ptr + rows * cols, outg, nb, cudaMemcpyHostToDevice, m->dev->stream));
    update_impl(m, xd.ptr, xd.ptr + rows * cols, rows);
    CSB_CUDA(cudaStreamSynchronize(m->dev->stream));
  });
}

int csb_moments_update_dev(csb_series* m, const double* in, const double* outg, uint64_t rows, uint64_t cols) {
  return guard([&] {
    check_update(m, rows, cols);
    update_impl(m, in, outg, rows);
    CSB_CUDA(cudaStreamSynchronize(m->dev->stream));
  });
}

int csb_moms2cums(const csb_series* m, csb_series* c) {
  return guard([&] {
    require(m && c, "moms2cums: null series");
    require(m->d >= 1, "moms2cums: empty series");
    require(m->n == c->n && m->d == c->d && m->b == c->b, "moms2cums: series tensors disagree on shape");
    NormScratch ns;
    run_moms2cums(m, c, ns, m->dev->stream);
    CSB_CUDA(cudaStreamSynchronize(m->dev->stream));
  });
}

int csb_combine(const csb_series* m1, uint64_t s1, const csb_series* m2, uint64_t s2, csb_series* out) {
  return guard([&] {
    require(m1 && m2 && out, "combine: null series");
    if (m1->d != m2->d) fail(CSB_EINVAL, "combine: order mismatch");
    if (s1 + s2 == 0) fail(CSB_EINVAL, "combine: empty combination");
    if (m1->n != m2->n || m1->b != m2->b || out->n != m1->n || out->b != m1->b || out->d != m1->d)
      fail(CSB_EINVAL, "combine: shape mismatch");
    const double w1 = static_cast<double>(s1) / static_cast<double>(s1 + s2);
    const double w2 = static_cast<double>(s2) / static_cast<double>(s1 + s2);
    for (int k = 0; k < m1->d; ++k)
      launch_combine(m1->data[k].ptr, m2->data[k].ptr, w1, w2, out->data[k].ptr, m1->data[k].count,
                     m1->dev->stream);
    out->window_len = s1 + s2;
    CSB_CUDA(cudaStreamSynchronize(m1->dev->stream));
  });
}

int csb_knorm(const csb_series* s, int order, double k, double* out) {
  return guard([&] {
    check_order(s, order);
    *out = knorm_device(s, order, k, s->dev->stream);
  });
}

int csb_nu(const csb_series* c, int d, double* out) {
  return guard([&] {
    require(c != nullptr, "nu: null series");
    if (d < 3 || d > c->d) fail(CSB_EINVAL, "nu: order must be in [3, max_order]");
    const double n2 = knorm_device(c, 2, 2.0, c->dev->stream);
    if (n2 <= 0.0) fail(CSB_EDOMAIN, "nu: vanishing second-order cumulant norm");
    *out = knorm_device(c, d, 2.0, c->dev->stream) / std::pow(n2, 0.5 * static_cast<double>(d));
  });
}

int csb_window_report(const csb_series* c, uint64_t window, csb_report* out) {
  return guard([&] {
    require(c && out, "window_report: null argument");
    if (c->d < 2) fail(CSB_EINVAL, "make_window_report: needs orders up to 2");
    NormScratch ns;
    finalize_norms(c, ns, c->dev->stream);
    build_report(c, ns, window, out);
  });
}

int csb_stream_prime(const csb_stream_config* cfg, const double* first, uint64_t rows, uint64_t cols,
                     csb_stream** out) {
  return guard([&] {
    require(cfg && out, "prime: null argument");
    // StreamConfig::validate (stream.cpp:18-27)
    if (cfg->dim < 1) fail(CSB_EINVAL, "StreamConfig: dim must be positive");
    if (cfg->max_order < 2) fail(CSB_EINVAL, "StreamConfig: max_order must be >= 2");
    if (cfg->window_len < 1) fail(CSB_EINVAL, "StreamConfig: window_len must be positive");
    if (cfg->update_len < 1 || cfg->update_len > cfg->window_len)
      fail(CSB_EINVAL, "StreamConfig: update_len must be in [1, window_len]");
    if (cfg->block_size < 1 || cfg->block_size > cfg->dim)
      fail(CSB_EINVAL, "StreamConfig: block_size must be in [1, dim]");
    if (cfg->workers < 0) fail(CSB_EINVAL, "StreamConfig: workers must be >= 0");
    if (rows != cfg->window_len || cols != static_cast<uint64_t>(cfg->dim))
      fail(CSB_EINVAL, "prime: batch does not match the configured window");
    auto s = std::make_unique<csb_stream>();
    s->cfg = *cfg;
    s->dev = &device();
    s->st = s->dev->stream;
    if (cfg->shard_count > 1) {
      if (cfg->shard_index < 0 || cfg->shard_index >= cfg->shard_count)
        fail(CSB_EINVAL, "StreamConfig: shard_index must be in [0, shard_count)");
      if (cfg->max_order > kMaxCumOrder) fail(CSB_EINVAL, "StreamConfig: sharding supports orders up to 6");
      const auto& cm = s->dev->comm;
      if (!cm || cm->nranks != cfg->shard_count || cm->rank != cfg->shard_index)
        fail(CSB_EINVAL, "prime: shard_count > 1 needs csb_comm_init(shard_count, shard_index, id) first");
      s->comm = cm;
      s->splan = get_shard_plan(*s->dev, cfg->max_order, cfg->dim, cfg->block_size, cfg->shard_count);
      s->sh.plan = s->splan.get();
      s->sh.index = cfg->shard_index;
      s->sh.comm = s->comm.get();
    }
    s->M = make_series(cfg->dim, cfg->max_order, cfg->block_size);
    s->C = make_series(cfg->dim, cfg->max_order, cfg->block_size);
    s->ring.alloc(rows * cols);
    s->staging.alloc(cfg->update_len * cols);
    for (auto& e : s->ev) CSB_CUDA(cudaEventCreate(&e));
    CSB_CUDA(cudaMemcpyAsync(s->ring.ptr, first, s->ring.bytes(), cudaMemcpyHostToDevice, s->st));
    s->head = 0;
    moment_series_impl(s->M.get(), s->ring.ptr, rows, cols, s->sh);
    run_moms2cums(s->M.get(), s->C.get(), s->ns, s->st, s->sh);
    s->window = 1;
    s->steps_since_resync = 0;
    CSB_CUDA(cudaStreamSynchronize(s->st));
    *out = s.release();
  });
}

int csb_stream_upload(csb_stream* s, const double* x, uint64_t rows, uint64_t cols) {
  return guard([&] {
    require(s != nullptr && x != nullptr, "upload: null argument");
    if (rows != s->cfg.update_len || cols != static_cast<uint64_t>(s->cfg.dim))
      fail(CSB_EINVAL, "upload: batch does not match the configured update");
    if (s->queued == 2) fail(CSB_EINVAL, "upload: two batches already uploaded and not stepped");
    CSB_CUDA(cudaSetDevice(s->dev->id));
    if (!s->copy_st) {
      CSB_CUDA(cudaStreamCreateWithFlags(&s->copy_st, cudaStreamNonBlocking));
      for (int k = 0; k < 2; ++k) {
        s->upload[k].alloc(rows * cols);
        CSB_CUDA(cudaEventCreateWithFlags(&s->uploaded[k], cudaEventDisableTiming));
        CSB_CUDA(cudaEventCreateWithFlags(&s->consumed[k], cudaEventDisableTiming));
      }
    }
    const int slot = s->next_slot;
    s->next_slot ^= 1;
    // the step that last read this slot must be done with it
    if (s->slot_used[slot]) CSB_CUDA(cudaStreamWaitEvent(s->copy_st, s->consumed[slot], 0));
    CSB_CUDA(cudaMemcpyAsync(s->upload[slot].ptr, x, rows * cols * sizeof(double), cudaMemcpyHostToDevice,
                             s->copy_st));
    CSB_CUDA(cudaEventRecord(s->uploaded[slot], s->copy_st));
    s->queue[s->queued++] = slot;
  });
}

int csb_stream_step_uploaded(csb_stream* s, csb_step_timing* t, csb_report* r) {
  int rc = guard([&] {
    require(s != nullptr, "step_uploaded: null stream");
    if (s->queued == 0) fail(CSB_EINVAL, "step_uploaded: no batch uploaded");
    CSB_CUDA(cudaStreamWaitEvent(s->st, s->uploaded[s->queue[0]], 0));
  });
  if (rc != CSB_OK) return rc;
  const int slot = s->queue[0];
  rc = stream_step_impl(s, s->upload[slot].ptr, true, s->cfg.update_len, static_cast<uint64_t>(s->cfg.dim), t, r);
  return guard([&] {
    CSB_CUDA(cudaEventRecord(s->consumed[slot], s->st));
    s->slot_used[slot] = true;
    s->queue[0] = s->queue[1];
    --s->queued;
    if (rc != CSB_OK) fail(rc, csb_last_error());
  });
}

int csb_stream_destroy(csb_stream* st) {
  return guard([&] { delete st; });
}

int csb_stream_step(csb_stream* s, const double* x, uint64_t rows, uint64_t cols, csb_step_timing* t,
                    csb_report* r) {
  return stream_step_impl(s, x, false, rows, cols, t, r);
}

int csb_stream_step_dev(csb_stream* s, const double* x, uint64_t rows, uint64_t cols, csb_step_timing* t,
                        csb_report* r) {
  return stream_step_impl(s, x, true, rows, cols, t, r);
}

int csb_stream_report(csb_stream* s, csb_report* r) {
  return guard([&] {
    require(s && r, "stream_report: null argument");
    if (!s->norms_valid) {
      finalize_norms(s->C.get(), s->ns, s->st, s->sh);
      s->norms_valid = true;
    }
    build_report(s->C.get(), s->ns, s->window, r);
  });
}

int csb_stream_moments(csb_stream* s, const csb_series** m) {
  return guard([&] {
    require(s && m, "null argument");
    CSB_CUDA(cudaStreamSynchronize(s->st));
    *m = s->M.get();
  });
}

int csb_stream_cumulants(csb_stream* s, const csb_series** c) {
  return guard([&] {
    require(s && c, "null argument");
    CSB_CUDA(cudaStreamSynchronize(s->st));
    *c = s->C.get();
  });
}

int csb_stream_window(const csb_stream* s, uint64_t* w) {
  return guard([&] {
    require(s && w, "null argument");
    *w = s->window;
  });
}

int csb_stream_materialize(const csb_stream* s, double* host, uint64_t count) {
  return guard([&] {
    require(s && host, "null argument");
    const uint64_t T = s->cfg.window_len, n = s->cfg.dim;
    require(count == T * n, "materialize: size mismatch");
    CSB_CUDA(cudaStreamSynchronize(s->st));
    const uint64_t tail = T - s->head;
    CSB_CUDA(cudaMemcpy(host, s->ring.ptr + s->head * n, tail * n * sizeof(double), cudaMemcpyDeviceToHost));
    if (s->head)
      CSB_CUDA(cudaMemcpy(host + tail * n, s->ring.ptr, s->head * n * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

int csb_stream_use_graphs(csb_stream* s, int on) {
  return guard([&] {
    require(s != nullptr, "use_graphs: null stream");
    s->use_graphs = on != 0;
  });
}

int csb_stream_graph_replays(const csb_stream* s, uint64_t* replays) {
  return guard([&] {
    require(s && replays, "graph_replays: null argument");
    *replays = s->graph_replays;
  });
}

int csb_stream_gather_shards(csb_stream* s) {
  return guard([&] {
    require(s != nullptr, "gather_shards: null stream");
    if (!s->sh.active()) return;  // the whole tensors already live here
    CSB_CUDA(cudaSetDevice(s->dev->id));
    const int d = s->cfg.max_order;
    const auto& L = s->M->lay[d - 1];
    const int G = s->sh.plan->count;
    // rank r owns the blocks [top_blk[r], top_blk[r+1]) of order d: one
    // contiguous range of the flat block storage (blocks are in lex order)
    std::vector<uint64_t> off(G), cnt(G);
    for (int r = 0; r < G; ++r) {
      off[r] = L->host.offset[s->sh.plan->top_blk[r]];
      cnt[r] = L->host.offset[s->sh.plan->top_blk[r + 1]] - off[r];
    }
    s->sh.comm->allgather_ranges(s->M->data[d - 1].ptr, off.data(), cnt.data(), s->st);
    s->sh.comm->allgather_ranges(s->C->data[d - 1].ptr, off.data(), cnt.data(), s->st);
    CSB_CUDA(cudaStreamSynchronize(s->st));
  });
}

int csb_stream_norm_partials(csb_stream* s, int order, double* host, uint64_t count, uint64_t* first_block) {
  return guard([&] {
    require(s && host, "null argument");
    if (order < 1 || order > s->cfg.max_order) fail(CSB_ERANGE, "norm_partials: order out of range");
    if (!s->norms_valid) {  // the exact partials are made with the report
      finalize_norms(s->C.get(), s->ns, s->st, s->sh);
      s->norms_valid = true;
    }
    require(count == s->ns.nblk(order), "norm_partials: size mismatch");
    CSB_CUDA(cudaStreamSynchronize(s->st));
    CSB_CUDA(cudaMemcpy(host, s->ns.part(order), count * sizeof(double), cudaMemcpyDeviceToHost));
    // a sharded stream's order-d partials are allreduced: the whole array is valid
    if (first_block) *first_block = 0;
  });
}

int csb_comm_unique_id(unsigned char* out) {
  return guard([&] {
    require(out != nullptr, "comm_unique_id: null output");
    nccl::get_unique_id(out);
  });
}

int csb_comm_init(int nranks, int rank, const unsigned char* id) {
  return guard([&] {
    require(id != nullptr && nranks >= 1 && rank >= 0 && rank < nranks, "comm_init: bad arguments");
    Device& dev = device();
    dev.comm.reset();  // live streams keep theirs
    dev.comm = make_nccl_comm(nranks, rank, id);  // one rank is a valid (trivial) communicator
  });
}

int csb_comm_init_ops(int nranks, int rank, const csb_comm_ops* ops) {
  return guard([&] {
    require(ops != nullptr && nranks >= 1 && rank >= 0 && rank < nranks, "comm_init_ops: bad arguments");
    Device& dev = device();
    dev.comm.reset();
    if (nranks > 1) dev.comm = make_ops_comm(nranks, rank, *ops);
  });
}

int csb_comm_selftest(uint64_t count) {
  return guard([&] {
    Device& dev = device();
    require(dev.comm != nullptr, "comm_selftest: no communicator (csb_comm_init first)");
    require(count >= 1 && count <= (1u << 24), "comm_selftest: count must be in [1, 2^24]");
    Comm& cm = *dev.comm;
    const int G = cm.nranks;
    const auto value = [](int r, uint64_t i) { return static_cast<double>(r + 1) + 1e-3 * static_cast<double>(i % 997); };
    // collective C2's shape: rank r owns [r * count, (r + 1) * count); the rest starts as NaN
    std::vector<double> h(static_cast<size_t>(G) * count, std::nan(""));
    for (uint64_t i = 0; i < count; ++i) h[static_cast<size_t>(cm.rank) * count + i] = value(cm.rank, i);
    DevBuf<double> buf(h.size());
    CSB_CUDA(cudaMemcpyAsync(buf.ptr, h.data(), buf.bytes(), cudaMemcpyHostToDevice, dev.stream));
    std::vector<uint64_t> off(G), cnt(G, count);
    for (int r = 0; r < G; ++r) off[r] = static_cast<uint64_t>(r) * count;
    cm.allgather_ranges(buf.ptr, off.data(), cnt.data(), dev.stream);
    CSB_CUDA(cudaMemcpyAsync(h.data(), buf.ptr, buf.bytes(), cudaMemcpyDeviceToHost, dev.stream));
    CSB_CUDA(cudaStreamSynchronize(dev.stream));
    for (int r = 0; r < G; ++r)
      for (uint64_t i = 0; i < count; ++i)
        if (h[static_cast<size_t>(r) * count + i] != value(r, i))
          fail(CSB_ERUNTIME, "comm_selftest: allgather_ranges returned a wrong value for rank " + std::to_string(r));
    // collective C3's shape: elementwise sum over ranks
    std::vector<double> a(count);
    for (uint64_t i = 0; i < count; ++i) a[i] = value(cm.rank, i);
    CSB_CUDA(cudaMemcpyAsync(buf.ptr, a.data(), count * sizeof(double), cudaMemcpyHostToDevice, dev.stream));
    cm.allreduce_sum(buf.ptr, count, dev.stream);
    CSB_CUDA(cudaMemcpyAsync(a.data(), buf.ptr, count * sizeof(double), cudaMemcpyDeviceToHost, dev.stream));
    CSB_CUDA(cudaStreamSynchronize(dev.stream));
    for (uint64_t i = 0; i < count; ++i) {
      double want = 0.0;
      for (int r = 0; r < G; ++r) want += value(r, i);
      if (std::fabs(a[i] - want) > 1e-12 * want) fail(CSB_ERUNTIME, "comm_selftest: allreduce_sum returned a wrong value");
    }
  });
}

int csb_comm_destroy(void) {
  return guard([&] {
    device().comm.reset();
  });
}

int csb_shard_range(int max_order, int dim, int block, int shard_index, int shard_count, int which,
                    uint64_t* blk_lo, uint64_t* blk_hi, uint64_t* elem_lo, uint64_t* elem_hi) {
  return guard([&] {
    require(max_order >= 2 && max_order <= kMaxOrder, "shard_range: max_order must be in [2, 8]");
    require(shard_count >= 1 && shard_index >= 0 && shard_index < shard_count, "shard_range: bad shard");
    require(which == 0 || which == 1, "shard_range: which must be 0 (order d) or 1 (order d-1)");
    Layout top(max_order, dim, block), low(max_order - 1, dim, block);
    ShardPlan sp;
    sp.build(max_order, dim, block, shard_count, top, low);
    const auto& bl = which ? sp.low_blk : sp.top_blk;
    const Layout& L = which ? low : top;
    if (blk_lo) *blk_lo = bl[shard_index];
    if (blk_hi) *blk_hi = bl[shard_index + 1];
    if (elem_lo) *elem_lo = L.offset[bl[shard_index]];
    if (elem_hi) *elem_hi = L.offset[bl[shard_index + 1]];
  });
}

int csb_moments_update_shard(csb_series* m, const double* in, const double* outg, uint64_t rows, uint64_t cols,
                             int shard_index, int shard_count) {
  return guard([&] {
    check_update(m, rows, cols);
    require(shard_count >= 1 && shard_index >= 0 && shard_index < shard_count, "moments_update_shard: bad shard");
    auto sp = get_shard_plan(*m->dev, m->d, m->n, m->b, shard_count);
    ShardCtx sh{sp.get(), shard_index, nullptr};
    DevBuf<double> xd(2 * rows * cols);
    const uint64_t nb = rows * cols * sizeof(double);
    CSB_CUDA(cudaMemcpyAsync(xd.ptr, in, nb, cudaMemcpyHostToDevice, m->dev->stream));
    CSB_CUDA(cudaMemcpyAsync(xd.ptr + rows * cols, outg, nb, cudaMemcpyHostToDevice, m->dev->stream));
    RowSource src[2];
    src[0].seg0 = xd.ptr;
    src[0].len0 = static_cast<uint32_t>(rows);
    src[1].seg0 = xd.ptr + rows * cols;
    src[1].len0 = static_cast<uint32_t>(rows);
    run_moments(m, src, 2, rows, static_cast<double>(rows) / static_cast<double>(m->window_len), m->dev->stream, 0,
                sh);
    g_rows_read.fetch_add(2 * rows, std::memory_order_relaxed);
    CSB_CUDA(cudaStreamSynchronize(m->dev->stream));
  });
}

int csb_moms2cums_shard(const csb_series* m, csb_series* c, int shard_index, int shard_count) {
  return guard([&] {
    require(m && c, "moms2cums_shard: null series");
    require(m->n == c->n && m->d == c->d && m->b == c->b, "moms2cums: series tensors disagree on shape");
    require(shard_count >= 1 && shard_index >= 0 && shard_index < shard_count, "moms2cums_shard: bad shard");
    auto sp = get_shard_plan(*m->dev, m->d, m->n, m->b, shard_count);
    ShardCtx sh{sp.get(), shard_index, nullptr};
    NormScratch ns;
    run_moms2cums(m, c, ns, m->dev->stream, sh);
    CSB_CUDA(cudaStreamSynchronize(m->dev->stream));
  });
}

uint64_t csb_launch_count(void) { return csb::launch_count(); }

int csb_top_kernel(int dim, int max_order, int block, char* out, uint64_t cap) {
  return guard([&] {
    require(out && cap > 0, "top_kernel: null output");
    require(dim >= 1 && block >= 1 && block <= dim && max_order >= 1 && max_order <= kMaxOrderAny,
            "top_kernel: bad shape");
    if (max_order > kMaxOrder) {
      std::snprintf(out, cap, "%s", "moment_generic_kernel (any order, one thread per stored element)");
      return;
    }
    MomParams p;
    p.n = dim;
    p.b = block;
    p.L = max_order - 1;
    p.npass = 1;  // aligned rows assumed
    std::string name = dmma_supported(p) ? dmma_kernel_name(dim, block) : "moment_pair_kernel (DFMA)";
    std::snprintf(out, cap, "%s", name.c_str());
  });
}

int csb_profile_enable(int on) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.on = on != 0;
  });
}

int csb_profile_read(const char* tag, double* total_ms, uint64_t* launches) {
  return guard([&] {
    require(tag && total_ms && launches, "profile_read: null argument");
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    {
      std::lock_guard<std::mutex> lk(g_prof.mu);
      ev.swap(g_prof.recs[tag].ev);
    }
    double tot = 0.0;
    for (auto& [a, b] : ev) {
      CSB_CUDA(cudaEventSynchronize(b));
      float ms = 0.f;
      CSB_CUDA(cudaEventElapsedTime(&ms, a, b));
      tot += ms;
    }
    {
      std::lock_guard<std::mutex> lk(g_prof.mu);
      for (auto& [a, b] : ev) {
        g_prof.pool.push_back(a);
        g_prof.pool.push_back(b);
      }
    }
    *total_ms = tot;
    *launches = ev.size();
  });
}

int csb_stream_cuda_stream(csb_stream* s, void** cs) {
  return guard([&] {
    require(s && cs, "null argument");
    *cs = s->st;
  });
}

}  // extern "C"
