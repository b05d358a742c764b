#include "layout.hpp"

#include <algorithm>
#include <map>
#include <tuple>
#include <cstdlib>
#include <array>
#include <numeric>

namespace csb {

Layout::Layout(int order_, int dim_, int block_) : order(order_), dim(dim_), block(block_) {
  require(order >= 1 && order <= 20, "SymTensor: order must be in [1, 20]");
  require(dim >= 1, "SymTensor: dim must be positive");
  require(block >= 1 && block <= dim, "SymTensor: block_size must be in [1, dim]");
  require(dim <= 65535, "cumstream_b200: dim must be <= 65535");
  grid = (dim + block - 1) / block;
  // lexicographic multiset ranker over the block grid (symten.cpp:31-45)
  prefix.assign(static_cast<std::size_t>(order) * (grid + 1), 0);
  for (int rem = 0; rem < order; ++rem) {
    uint64_t acc = 0;
    for (int v = 0; v <= grid; ++v) {
      prefix[static_cast<std::size_t>(rem) * (grid + 1) + v] = acc;
      if (v < grid) acc += multiset_count(grid - v, rem);
    }
  }
  nblocks = multiset_count(grid, order);
  index.reserve(nblocks * order);
  offset.reserve(nblocks + 1);
  int j[20] = {0};
  uint64_t off = 0;
  for (;;) {
    uint64_t vol = 1;
    for (int k = 0; k < order; ++k) {
      index.push_back(static_cast<uint16_t>(j[k]));
      vol *= static_cast<uint64_t>(ext(j[k]));
    }
    offset.push_back(off);
    off += vol;
    int k = order - 1;
    while (k >= 0 && j[k] == grid - 1) --k;
    if (k < 0) break;
    const int v = j[k] + 1;
    for (int l = k; l < order; ++l) j[l] = v;
  }
  offset.push_back(off);
  stored = off;
}

uint64_t Layout::rank(const int* j) const {
  uint64_t acc = 0;
  int lo = 0;
  for (int i = 0; i < order; ++i) {
    const int rem = order - 1 - i;
    acc += prefix[static_cast<std::size_t>(rem) * (grid + 1) + j[i]] -
           prefix[static_cast<std::size_t>(rem) * (grid + 1) + lo];
    lo = j[i];
  }
  return acc;
}

uint64_t Layout::element_offset(const int* i) const {
  int j[20];
  for (int k = 0; k < order; ++k) j[k] = i[k] / block;
  const uint64_t r = rank(j);
  uint64_t off = 0;
  for (int k = 0; k < order; ++k)
    off = off * static_cast<uint64_t>(ext(j[k])) + static_cast<uint64_t>(i[k] - j[k] * block);
  return offset[r] + off;
}

uint64_t block_multiplicity(const int* j, int d) {
  uint64_t num = 1;
  for (int i = 2; i <= d; ++i) num *= static_cast<uint64_t>(i);
  for (int s = 0; s < d;) {
    int e = s + 1;
    while (e < d && j[e] == j[s]) ++e;
    for (int i = 2; i <= e - s; ++i) num /= static_cast<uint64_t>(i);
    s = e;
  }
  return num;
}

std::vector<std::vector<PrefixRow>> MomentPlan::enumerate(int S_, int n_, int b_, const Layout& top,
                                                          const Layout* low) {
  S = S_;
  L = S_ - 1;
  n = n_;
  b = b_;
  rows.clear();
  tiles.clear();
  const int grid = top.grid;
  // canonical L-tuples in lexicographic order, bucketed by J = i_L / b
  std::vector<std::vector<PrefixRow>> byJ(grid);
  if (L == 0) {
    PrefixRow r{};
    r.top_base = 0;
    r.low_off = 0;
    r.vprime = 1;
    r.poff = 0;
    byJ[0].push_back(r);
    return byJ;
  }
  int t[8] = {0};
  int jj[8], full[8];
  for (;;) {
    PrefixRow r{};
    uint32_t vprime = 1, poff = 0;
    for (int k = 0; k < L; ++k) {
      r.idx[k] = static_cast<uint16_t>(t[k]);
      jj[k] = t[k] / b;
      const int e = top.ext(jj[k]);
      vprime *= static_cast<uint32_t>(e);
      poff = poff * static_cast<uint32_t>(e) + static_cast<uint32_t>(t[k] - jj[k] * b);
    }
    const int J = jj[L - 1];
    for (int k = 0; k < L; ++k) full[k] = jj[k];
    full[L] = J;
    r.top_base = top.offset[top.rank(full)];
    r.low_off = low ? low->offset[low->rank(jj)] + poff : 0;
    r.vprime = vprime;
    r.poff = poff;
    byJ[J].push_back(r);
    int k = L - 1;
    while (k >= 0 && t[k] == n - 1) --k;
    if (k < 0) break;
    const int v = t[k] + 1;
    for (int l = k; l < L; ++l) t[l] = v;
  }
  return byJ;
}

PrefixRow MomentPlan::make_row(const int* t, const Layout& top, const Layout* low) const {
  PrefixRow r{};
  int jj[8], full[8];
  uint32_t vprime = 1, poff = 0;
  for (int k = 0; k < L; ++k) {
    r.idx[k] = static_cast<uint16_t>(t[k]);
    jj[k] = t[k] / b;
    const int e = top.ext(jj[k]);
    vprime *= static_cast<uint32_t>(e);
    poff = poff * static_cast<uint32_t>(e) + static_cast<uint32_t>(t[k] - jj[k] * b);
  }
  for (int k = 0; k < L; ++k) full[k] = jj[k];
  full[L] = jj[L - 1];
  r.top_base = top.offset[top.rank(full)];
  r.low_off = low ? low->offset[low->rank(jj)] + poff : 0;
  r.vprime = vprime;
  r.poff = poff;
  // bit 0 of the spare idx slot: equal neighbouring block coordinates among
  // (j_1..j_L), i.e. the prefix block has internal symmetry copies
  uint16_t runs = 0;
  for (int k = 1; k < L; ++k) runs |= jj[k] == jj[k - 1];
  r.idx[7] = runs;
  return r;
}

void ShardPlan::build(int d_, int n_, int b_, int count_, const Layout& top, const Layout& low) {
  d = d_;
  n = n_;
  b = b_;
  count = std::max(1, count_);
  // prefix length: the (d-2)-prefix pi of a DMMA group fixes the first d-2
  // block coordinates; 2 (d = 4) or 3 (d >= 5) gives enough granularity
  plen = std::max(0, std::min(d >= 5 ? 3 : 2, d - 2));
  const int g = top.grid;
  prefix_rank = plen > 0 ? std::make_shared<Layout>(plen, g, 1) : nullptr;
  const uint64_t nprefix = plen == 0 ? 1 : prefix_rank->nblocks;
  std::vector<double> w(nprefix, 0.0);
  auto prank = [&](const uint16_t* j) -> uint64_t {
    if (plen == 0) return 0;
    int t[3];
    for (int k = 0; k < plen; ++k) t[k] = j[k];
    return prefix_rank->rank(t);
  };
  for (uint64_t r = 0; r < top.nblocks; ++r) {
    const uint16_t* j = &top.index[r * d];
    // canonical entries of the block: prod over runs C(e + len - 1, len)
    double c = 1.0;
    for (int a = 0; a < d;) {
      int e2 = a + 1;
      while (e2 < d && j[e2] == j[a]) ++e2;
      c *= static_cast<double>(multiset_count(top.ext(j[a]), e2 - a));
      a = e2;
    }
    w[prank(j)] += c;
  }
  // contiguous min-max partition of the prefix sequence into `count`
  // ranges (binary search on the largest range weight, greedy fill)
  double total = 0.0, wmax = 0.0;
  for (double v : w) {
    total += v;
    wmax = std::max(wmax, v);
  }
  auto fits = [&](double cap) {
    int used = 1;
    double acc = 0.0;
    for (double v : w) {
      if (acc + v > cap) {
        ++used;
        acc = 0.0;
      }
      acc += v;
    }
    return used <= count;
  };
  double lo = std::max(wmax, total / count), hi = total;
  for (int it = 0; it < 100 && hi - lo > 1e-9 * total; ++it) {
    const double mid = 0.5 * (lo + hi);
    (fits(mid) ? hi : lo) = mid;
  }
  shard_of_prefix.assign(nprefix, 0);
  {
    int cur = 0;
    double acc = 0.0;
    for (uint64_t p = 0; p < nprefix; ++p) {
      // open a new range when the cap is exceeded, or when the remaining
      // prefixes are needed to give every later shard at least one
      if (cur < count - 1 && (acc + w[p] > hi || nprefix - p <= static_cast<uint64_t>(count - 1 - cur))) {
        if (acc > 0.0) {
          ++cur;
          acc = 0.0;
        }
      }
      shard_of_prefix[p] = cur;
      acc += w[p];
    }
  }
  auto bounds = [&](const Layout& L, std::vector<uint64_t>& out) {
    out.assign(count + 1, L.nblocks);
    out[0] = 0;
    int last = 0;
    for (uint64_t r = 0; r < L.nblocks; ++r) {
      const int sh = plen == 0 ? 0 : shard_of_prefix[prank(&L.index[r * L.order])];
      while (last < sh) out[++last] = r;
    }
  };
  bounds(top, top_blk);
  bounds(low, low_blk);
}

int ShardPlan::owner(const int* jp) const {
  if (plen == 0) return 0;
  return shard_of_prefix[prefix_rank->rank(jp)];
}

void MomentPlan::build_dmma(int S_, int n_, int b_, const Layout& top, const Layout* low, uint64_t scratch,
                            int tail_windows, const ShardPlan* shard, int shard_index, int sm_count) {
  S = S_;
  L = S_ - 1;
  n = n_;
  b = b_;
  rows.clear();
  tiles.clear();
  pairs.clear();
  dmma = true;
  require(L >= 2 && L <= 7, "build_dmma: order out of range");
  const int LM1 = L - 1;
  // all (L-1)-tuples pi in lexicographic order
  std::vector<std::array<uint16_t, 6>> pis;
  {
    int t[8] = {0};
    for (;;) {
      std::array<uint16_t, 6> a{};
      for (int k = 0; k < LM1; ++k) a[k] = static_cast<uint16_t>(t[k]);
      pis.push_back(a);
      int k = LM1 - 1;
      while (k >= 0 && t[k] == n - 1) --k;
      if (k < 0) break;
      const int v = t[k] + 1;
      for (int l = k; l < LM1; ++l) t[l] = v;
    }
  }
  const int nh = (n + 7) / 8;
  auto owned = [&](const std::array<uint16_t, 6>& pi) {
    if (!shard || shard->count <= 1) return true;
    int jp[3] = {0, 0, 0};
    for (int k = 0; k < shard->plen; ++k) jp[k] = pi[k] / b;
    return shard->owner(jp) == shard_index;  // else another shard's blocks
  };
  // the last window (columns [8h, n), at most one 8-wide tile): CUDA-core
  // tasks, grouped by the first last index s so a warp's lanes share the
  // loop structure
  tail.clear();
  tail_rows.clear();
  // whole 8-column chunks right of a window are needed by the rectangle
  // tasks: a second tail window only when n is a multiple of 8
  tail_windows = std::max(0, std::min({tail_windows, nh, n % 8 == 0 ? 2 : 1}));
  const int nh_dmma = nh - tail_windows;
  {
    // tasks grouped by (kind, run length, s) so a warp's lanes share them
    std::map<std::tuple<int, int, int>, std::vector<TailTask>> groups;
    int t[8];
    for (int h = nh_dmma; h < nh; ++h) {
      const int lo = 8 * h, hi = std::min(8 * h + 8, n);
      for (const auto& pi : pis) {
        const int last = pi[LM1 - 1];
        if (last >= hi || !owned(pi)) continue;
        const int s = std::max(last, lo);
        const uint32_t row0 = static_cast<uint32_t>(tail_rows.size());
        for (int k = 0; k < LM1; ++k) t[k] = pi[k];
        for (int a = s; a < hi; ++a) {
          t[LM1] = a;
          tail_rows.push_back(make_row(t, top, low));
        }
        TailTask tk{};
        for (int k = 0; k < 6; ++k) tk.pidx[k] = pi[k];
        tk.s = static_cast<uint16_t>(s);
        tk.e = static_cast<uint16_t>(hi);
        tk.c0 = static_cast<uint16_t>(s);
        tk.kind = TAIL_TRI;
        tk.row0 = row0;
        groups[{TAIL_TRI, hi - s, s}].push_back(tk);
        // the full 8-column chunks right of the window, by sub-runs of <= 4
        for (int c0 = hi; c0 < n; c0 += 8)
          for (int a = s; a < hi;) {
            const int e = std::min(hi, std::max(a + 1, ((a + 4) / 4) * 4));  // 4-aligned sub-runs
            TailTask r = tk;
            r.s = static_cast<uint16_t>(a);
            r.e = static_cast<uint16_t>(e);
            r.c0 = static_cast<uint16_t>(c0);
            r.kind = TAIL_RECT;
            r.row0 = row0 + static_cast<uint32_t>(a - s);
            groups[{TAIL_RECT, e - a, a}].push_back(r);
            a = e;
          }
      }
    }
    // longest tasks first: CTAs are handed out in order, one per SM, and a
    // CTA of 8-row triangles runs ~9x longer than one of single rows, so the
    // last wave should be made of the cheap ones
    std::vector<std::pair<int, const std::vector<TailTask>*>> order;
    for (const auto& [key, v] : groups) {
      const int rl = std::get<1>(key);
      const int per_row = std::get<0>(key) == TAIL_TRI ? LM1 - 1 + 2 * rl + rl * (rl + 1) / 2 : LM1 - 1 + 9 * rl;
      order.emplace_back(per_row, &v);
    }
    std::stable_sort(order.begin(), order.end(), [](const auto& a, const auto& b) { return a.first > b.first; });
    for (const auto& [cost, vp] : order) {
      const auto& v = *vp;
      for (const auto& tk : v) tail.push_back(tk);
      TailTask pad = v.front();
      pad.row0 = kNoRow;
      for (size_t k = v.size(); k % 32; ++k) tail.push_back(pad);
    }
  }
  struct Win {
    uint32_t rs0, nrs;
    int h;
  };
  std::vector<Win> windows;
  for (int h = 0; h < nh_dmma; ++h) {
    const int hi = std::min(8 * h + 8, n);
    const uint32_t rs0 = static_cast<uint32_t>(pairs.size() / 32);
    int t[8];
    for (const auto& pi : pis) {
      const int last = pi[LM1 - 1];
      if (last >= hi) continue;  // every row of this window has i_L < i_{L-1}
      if (!owned(pi)) continue;
      for (int k = 0; k < LM1; ++k) t[k] = pi[k];
      // pairs (a, a + 1) start at even a (16-byte aligned column pairs: the
      // producer loads x[a0], x[a0 + 1] with one LDS.128); when the first
      // canonical a is odd, the pair's first slot is masked (hi is even)
      const int a_lo = std::max(last, 8 * h);
      for (int a = a_lo & ~1; a < hi; a += 2) {
        DmmaPair pr{};
        for (int k = 0; k < 6; ++k) pr.pidx[k] = pi[k];
        pr.a0 = static_cast<uint16_t>(a);
        pr.a1 = static_cast<uint16_t>(a + 1);
        pairs.push_back(pr);
        if (a >= a_lo) {
          t[LM1] = a;
          rows.push_back(make_row(t, top, low));
        } else {
          rows.push_back(PrefixRow{});  // masked slot
        }
        t[LM1] = a + 1;
        rows.push_back(make_row(t, top, low));
      }
    }
    while (pairs.size() % 32) {  // pad the window's last row set
      pairs.push_back(DmmaPair{});
      rows.push_back(PrefixRow{});
      rows.push_back(PrefixRow{});
    }
    const uint32_t nrs = static_cast<uint32_t>(pairs.size() / 32) - rs0;
    if (!nrs) continue;
    windows.push_back({rs0, nrs, h});
  }
  // R row sets per CTA, up to kMaxNc column tiles per DMMA warp (8 warps):
  // each row set's tiles spread over 4/R sub-partitions; the base choice keeps
  // the busiest sub-partition's share per row set smallest.  When that leaves
  // fewer CTAs than SMs (cfg0: ~45 row sets, 12 CTAs at R = 4), R is halved:
  // the rows of a pass are a serial chain, so a small problem's time is set by
  // one CTA's DMMAs per row step, and fewer row sets per CTA shorten exactly that.
  constexpr int kMaxNc = 3;
  auto base_r = [](int ncg) { return ncg <= 6 ? 4 : ncg <= 12 ? 2 : 1; };
  int shrink = 0;
  for (; shrink < 2; ++shrink) {
    uint64_t ctas = 0;
    for (const auto& w : windows) {
      const int ncg = (n - 8 * w.h + 7) / 8;
      const int R = std::max(1, base_r(ncg) >> shrink);
      const int per_cta = kMaxNc * 8 / R;
      ctas += static_cast<uint64_t>((ncg + per_cta - 1) / per_cta) * ((w.nrs + R - 1) / R);
    }
    if (ctas >= static_cast<uint64_t>(sm_count)) break;
  }
  for (const auto& w : windows) {
    const int h = w.h;
    const uint32_t rs0 = w.rs0, nrs = w.nrs;
    const int ncg = (n - 8 * h + 7) / 8;
    const int R = std::max(1, base_r(ncg) >> shrink);
    const int per_cta = kMaxNc * 8 / R;
    const int nranges = (ncg + per_cta - 1) / per_cta;
    for (int q = 0; q < nranges; ++q) {
      const int c0 = q * ncg / nranges, c1 = (q + 1) * ncg / nranges;
      for (uint32_t s0 = 0; s0 < nrs; s0 += static_cast<uint32_t>(R)) {
        MomTile tl{};
        tl.row0 = rs0 + s0;
        tl.nrows = std::min<uint32_t>(static_cast<uint32_t>(R), nrs - s0);
        tl.J = static_cast<uint32_t>(h);
        tl.col0 = static_cast<uint32_t>(8 * h + 8 * c0);
        tl.ncols = static_cast<uint32_t>(c1 - c0);
        tl.low = (q == 0 && low) ? 1u : 0u;
        tl.pad0 = static_cast<uint32_t>(R);
        tiles.push_back(tl);
      }
    }
  }
  // longest tiles first (the hardware dispatches in blockIdx order): a
  // tile's time is set by its widest DMMA warp
  auto width = [](const MomTile& t) { return (t.ncols + (4 / t.pad0) - 1) / (4 / t.pad0); };
  std::stable_sort(tiles.begin(), tiles.end(),
                   [&](const MomTile& a, const MomTile& c) { return width(a) > width(c); });
  for (size_t i = 0; i < tiles.size(); ++i) tiles[i].pad1 = static_cast<uint32_t>(i);
  scratch_per_tile = scratch;
}

void MomentPlan::build(int S_, int n_, int b_, const Layout& top, const Layout* low, int threads) {
  auto byJ = enumerate(S_, n_, b_, top, low);
  const int grid = top.grid;
  constexpr int kMaxTileRows = 1024;
  for (int J = 0; J < grid; ++J) {
    const auto& R = byJ[J];
    if (R.empty()) continue;
    const uint32_t col0 = static_cast<uint32_t>(J * b);
    const uint32_t ncols = static_cast<uint32_t>(n - J * b);
    const int cg = static_cast<int>((ncols + 7) / 8);
    int rg_max = std::max(1, threads / cg);
    rg_max = std::min(rg_max, kMaxTileRows / 8);
    const uint64_t cap = static_cast<uint64_t>(rg_max) * 8;
    const uint64_t nt = (R.size() + cap - 1) / cap;
    uint64_t per = (R.size() + nt - 1) / nt;
    per = (per + 7) / 8 * 8;
    const uint32_t base = static_cast<uint32_t>(rows.size());
    rows.insert(rows.end(), R.begin(), R.end());
    for (uint64_t r0 = 0; r0 < R.size(); r0 += per) {
      MomTile t{};
      t.row0 = base + static_cast<uint32_t>(r0);
      t.nrows = static_cast<uint32_t>(std::min<uint64_t>(per, R.size() - r0));
      t.J = static_cast<uint32_t>(J);
      t.col0 = col0;
      t.ncols = ncols;
      t.low = (L > 0 && low) ? 1u : 0u;
      tiles.push_back(t);
    }
  }
  // largest tiles first (the hardware dispatches in blockIdx order)
  std::stable_sort(tiles.begin(), tiles.end(), [](const MomTile& a, const MomTile& c) {
    return static_cast<uint64_t>(a.nrows) * a.ncols > static_cast<uint64_t>(c.nrows) * c.ncols;
  });
  scratch_per_tile = static_cast<uint64_t>(threads) * 64;
}

void MomentPlan::upload() {
  d_rows.alloc(rows.size());
  d_tiles.alloc(tiles.size());
  d_pairs.alloc(pairs.size());
  if (!pairs.empty())
    h2d_sync(d_pairs.ptr, pairs.data(), d_pairs.bytes());
  if (!rows.empty())
    h2d_sync(d_rows.ptr, rows.data(), d_rows.bytes());
  if (!tiles.empty())
    h2d_sync(d_tiles.ptr, tiles.data(), d_tiles.bytes());
  d_tail.alloc(tail.size());
  d_tail_rows.alloc(tail_rows.size());
  if (!tail.empty()) h2d_sync(d_tail.ptr, tail.data(), d_tail.bytes());
  if (!tail_rows.empty()) h2d_sync(d_tail_rows.ptr, tail_rows.data(), d_tail_rows.bytes());
}

}  // namespace csb
