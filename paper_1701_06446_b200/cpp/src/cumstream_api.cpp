// cumstream_b200 C++ drop-in API (the reference's namespace cumstream) on
// top of the C ABI in include/cumstream_b200.h.  Every hot-path operation
// (moment_series, moment_tensor, moments_update, moms2cums, knorm, nu,
// make_window_report, prime, step, run) executes on the B200; the host side
// only validates arguments, keeps the device handles and converts statuses
// back into the reference's exception types.
#include <algorithm>
#include <array>
#include <charconv>
#include <cmath>
#include <cstring>
#include <iostream>
#include <stdexcept>
#include <string>

#include "cumstream/cumulants.hpp"
#include "cumstream/gauge.hpp"
#include "cumstream/moments.hpp"
#include "cumstream/stream.hpp"
#include "cumstream/symten.hpp"
#include "cumstream_b200.h"

#if __has_include(<json.hpp>)
#include <exception>
#include <json.hpp>  // nlohmann/json 3.11.3, the reference's JSON dependency
#define CSB_HAVE_NLOHMANN 1
#else
#define CSB_HAVE_NLOHMANN 0
#endif

namespace cumstream {

namespace detail {

[[noreturn]] void rethrow(int rc) {
  const std::string msg = csb_last_error();
  switch (rc) {
    case CSB_EINVAL: throw std::invalid_argument(msg);
    case CSB_ERANGE: throw std::out_of_range(msg);
    case CSB_EDOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
  }
}

inline void check(int rc) {
  if (rc != CSB_OK) rethrow(rc);
}

struct DeviceStream;

// A device series (orders 1..d of one (n, b) shape).  Tensors whose
// authoritative copy lives in slot `order` point at it through dev_.
struct DeviceSeries {
  csb_series* s = nullptr;
  bool owned = true;
  std::shared_ptr<DeviceStream> keep;  // borrowed from a stream: keep it alive
  int n = 0, d = 0, b = 0;

  DeviceSeries() = default;
  DeviceSeries(const DeviceSeries&) = delete;
  DeviceSeries& operator=(const DeviceSeries&) = delete;
  ~DeviceSeries() {
    if (owned && s) csb_series_destroy(s);
  }

  static std::shared_ptr<DeviceSeries> create(int n, int d, int b) {
    auto ds = std::make_shared<DeviceSeries>();
    check(csb_series_create(n, d, b, &ds->s));
    ds->n = n;
    ds->d = d;
    ds->b = b;
    return ds;
  }

  void download(const SymTensor& t) const {
    check(csb_series_download(s, t.order_, t.data_.data(), t.size_));
  }
  void upload(const SymTensor& t) const {
    t.pull();
    check(csb_series_upload(s, t.order_, t.data_.data(), t.size_));
  }
  // the tensors now live on the device (host mirrors stale)
  static void attach(const SymTensor& t, const std::shared_ptr<DeviceSeries>& ds) {
    t.dev_ = ds;
    t.host_fresh_ = false;
  }
  static bool is(const SymTensor& t, const DeviceSeries* ds) { return t.dev_.get() == ds; }
  // knorm on the device: the tensor's own device copy when it has one,
  // otherwise a one-order upload
  static double knorm_of(const SymTensor& t, double k) {
    double out = 0.0;
    if (t.dev_ && t.dev_->d >= t.order_) {
      check(csb_knorm(t.dev_->s, t.order_, k, &out));
      return out;
    }
    auto ds = create(t.dim_, t.order_, t.block_size_);
    ds->upload(t);
    check(csb_knorm(ds->s, t.order_, k, &out));
    return out;
  }
  static std::shared_ptr<DeviceSeries> of(const SymTensor& t) { return t.dev_; }
  static void mark_clean(const SymTensor& t, const std::shared_ptr<DeviceSeries>& ds) {
    t.dev_ = ds;  // host mirror and device copy agree
  }
};

// Device series holding exactly `tensors` (orders 1..d): reused when every
// tensor already lives in the same device series, otherwise assembled by
// uploading the host mirrors.
template <class Vec>
std::shared_ptr<DeviceSeries> acquire(const Vec& tensors, std::size_t window_len) {
  if (tensors.empty()) throw std::invalid_argument("empty series");
  const int d = static_cast<int>(tensors.size());
  const SymTensor& t0 = tensors.front();
  std::shared_ptr<DeviceSeries> ds = DeviceSeries::of(t0);
  bool reuse = ds && ds->d == d;
  for (int k = 0; reuse && k < d; ++k) reuse = DeviceSeries::is(tensors[k], ds.get());
  if (!reuse) {
    ds = DeviceSeries::create(t0.dim(), d, t0.block_size());
    for (int k = 0; k < d; ++k) {
      const SymTensor& t = tensors[k];
      if (t.order() != k + 1 || t.dim() != t0.dim() || t.block_size() != t0.block_size())
        throw std::invalid_argument("series tensors disagree on shape");
      ds->upload(t);
      DeviceSeries::mark_clean(t, ds);
    }
  }
  check(csb_series_set_window_len(ds->s, window_len));
  return ds;
}

// Ensure the tensors are the content of a given device series slot set
// (used to push host-side edits of WindowState::moments into the stream).
void sync_into(const std::vector<SymTensor>& tensors, const std::shared_ptr<DeviceSeries>& ds) {
  for (const SymTensor& t : tensors) {
    if (DeviceSeries::is(t, ds.get())) continue;
    ds->upload(t);
    DeviceSeries::mark_clean(t, ds);
  }
}

template <class Series>
Series wrap(const std::shared_ptr<DeviceSeries>& ds) {
  Series out;
  uint64_t wl = 0;
  check(csb_series_shape(ds->s, nullptr, nullptr, nullptr, &wl));
  out.window_len = wl;
  out.tensors.reserve(ds->d);
  for (int k = 1; k <= ds->d; ++k) {
    out.tensors.emplace_back(k, ds->n, ds->b);
    DeviceSeries::attach(out.tensors.back(), ds);
  }
  return out;
}

struct DeviceStream {
  csb_stream* st = nullptr;
  std::shared_ptr<DeviceSeries> m;  // the stream's moment series (borrowed)
  ~DeviceStream() {
    if (st) csb_stream_destroy(st);
  }
  // the WindowBuffer of a primed state views the device ring
  static void bind(WindowBuffer& buf, const std::shared_ptr<DeviceStream>& ds) {
    buf.values_.clear();
    buf.values_.shrink_to_fit();
    buf.device_ = ds;
  }
};

void check_batch(const DataBatch& x, const char* what) {
  if (x.rows < 1) throw std::invalid_argument(std::string(what) + ": empty batch");
  if (x.cols < 1) throw std::invalid_argument(std::string(what) + ": no columns");
  if (x.values.size() != x.rows * x.cols)
    throw std::invalid_argument(std::string(what) + ": bad batch buffer size");
}

}  // namespace detail

using detail::check;
using detail::DeviceSeries;

// ===========================================================================
// symten (symten.hpp:19-159)

namespace {

std::uint64_t binomial_u64(int n, int k) {
  if (k < 0 || k > n) return 0;
  if (k > n - k) k = n - k;
  std::uint64_t r = 1;
  for (int i = 1; i <= k; ++i) r = r * static_cast<std::uint64_t>(n - k + i) / i;
  return r;
}

void require_sorted(std::span<const int> t, const char* what) {
  for (std::size_t i = 1; i < t.size(); ++i)
    if (t[i - 1] > t[i]) throw std::invalid_argument(std::string(what) + ": index not non-decreasing");
}

}  // namespace

// table_[rem][v] counts the non-decreasing (rem+1)-tuples whose first entry
// is below v: summing C(alphabet - u + rem - 1, rem) over u < v telescopes
// (hockey stick) to C(alphabet + rem, rem + 1) - C(alphabet - v + rem, rem + 1),
// so every entry is one closed form.
MultisetRanker::MultisetRanker(int alphabet, int order) : alphabet_(alphabet), order_(order) {
  if (alphabet < 1 || order < 1)
    throw std::invalid_argument("MultisetRanker: alphabet and order must be positive");
  count_ = binomial_u64(alphabet + order - 1, order);
  const std::size_t stride = static_cast<std::size_t>(alphabet) + 1;
  table_.resize(static_cast<std::size_t>(order) * stride);
  for (int rem = 0; rem < order; ++rem) {
    const std::uint64_t all = binomial_u64(alphabet + rem, rem + 1);
    for (int v = 0; v <= alphabet; ++v)
      table_[rem * stride + v] = all - binomial_u64(alphabet - v + rem, rem + 1);
  }
}

std::uint64_t MultisetRanker::rank(std::span<const int> tuple) const {
  if (static_cast<int>(tuple.size()) != order_)
    throw std::invalid_argument("MultisetRanker::rank: wrong tuple length");
  const bool sorted_in_range =
      std::is_sorted(tuple.begin(), tuple.end()) && (tuple.empty() || (tuple.front() >= 0 && tuple.back() < alphabet_));
  if (!sorted_in_range) throw std::out_of_range("MultisetRanker::rank: tuple not sorted or out of range");
  return rank_unchecked(tuple.data());
}

// Position by position, the largest value whose table offset (relative to
// the previous entry) does not exceed the remaining rank: a binary search
// per position over the monotone table row.
void MultisetRanker::unrank(std::uint64_t r, std::span<int> out) const {
  if (static_cast<int>(out.size()) != order_)
    throw std::invalid_argument("MultisetRanker::unrank: wrong output length");
  if (r >= count_) throw std::out_of_range("MultisetRanker::unrank: rank too large");
  const std::size_t stride = static_cast<std::size_t>(alphabet_) + 1;
  int lo = 0;
  for (int i = 0; i < order_; ++i) {
    const std::uint64_t* row = table_.data() + static_cast<std::size_t>(order_ - 1 - i) * stride;
    const std::uint64_t target = row[lo] + r;
    // first v in (lo, alphabet] with row[v] > target, minus one
    const std::uint64_t* it = std::upper_bound(row + lo + 1, row + alphabet_ + 1, target);
    const int v = static_cast<int>(it - row) - 1;
    r = target - row[v];
    out[i] = v;
    lo = v;
  }
}

DenseTensor::DenseTensor(int order_, int dim_) : order(order_), dim(dim_) {
  if (order_ < 1 || dim_ < 1) throw std::invalid_argument("DenseTensor: order and dim must be positive");
  std::size_t total = 1;
  for (int k = 0; k < order_; ++k) total *= static_cast<std::size_t>(dim_);
  values.assign(total, 0.0);
}

std::size_t DenseTensor::linear(std::span<const int> index) const {
  if (static_cast<int>(index.size()) != order) throw std::invalid_argument("DenseTensor: wrong index length");
  std::size_t pos = 0;
  for (int v : index) {
    if (v < 0 || v >= dim) throw std::out_of_range("DenseTensor: index out of range");
    pos = pos * dim + static_cast<std::size_t>(v);
  }
  return pos;
}

double DenseTensor::at(std::initializer_list<int> index) const {
  return at(std::span<const int>(index.begin(), index.size()));
}
double& DenseTensor::at(std::initializer_list<int> index) {
  return at(std::span<const int>(index.begin(), index.size()));
}

SymTensor::SymTensor(int order, int dim, int block_size) : order_(order), dim_(dim), block_size_(block_size) {
  if (order < 1 || order > kMaxOrder) throw std::invalid_argument("SymTensor: order must be in [1, 20]");
  if (dim < 1) throw std::invalid_argument("SymTensor: dim must be positive");
  if (block_size < 1 || block_size > dim) throw std::invalid_argument("SymTensor: block_size must be in [1, dim]");
  grid_ = (dim + block_size - 1) / block_size;
  auto ranker = std::make_shared<MultisetRanker>(grid_, order);
  auto blocks = std::make_shared<std::vector<BlockInfo>>();
  blocks->reserve(ranker->count());
  std::vector<int> j(order, 0);
  std::size_t off = 0;
  for (;;) {
    BlockInfo bi;
    bi.index = j;
    bi.extents.resize(order);
    bi.base.resize(order);
    bi.volume = 1;
    for (int k = 0; k < order; ++k) {
      bi.base[k] = j[k] * block_size;
      bi.extents[k] = std::min(block_size, dim - bi.base[k]);
      bi.volume *= static_cast<std::size_t>(bi.extents[k]);
    }
    bi.offset = off;
    off += bi.volume;
    blocks->push_back(std::move(bi));
    int k = order - 1;
    while (k >= 0 && j[k] == grid_ - 1) --k;
    if (k < 0) break;
    const int v = j[k] + 1;
    for (int l = k; l < order; ++l) j[l] = v;
  }
  size_ = off;
  block_ranker_ = std::move(ranker);
  blocks_ = std::move(blocks);
  data_.assign(off, 0.0);
}

SymTensor::SymTensor(const SymTensor& o)
    : order_(o.order_), dim_(o.dim_), block_size_(o.block_size_), grid_(o.grid_), size_(o.size_),
      block_ranker_(o.block_ranker_), blocks_(o.blocks_) {
  o.pull();
  data_ = o.data_;  // an independent value (no device link)
}

SymTensor& SymTensor::operator=(const SymTensor& o) {
  if (this != &o) {
    o.pull();
    order_ = o.order_;
    dim_ = o.dim_;
    block_size_ = o.block_size_;
    grid_ = o.grid_;
    size_ = o.size_;
    block_ranker_ = o.block_ranker_;
    blocks_ = o.blocks_;
    data_ = o.data_;
    dev_.reset();
    host_fresh_ = true;
  }
  return *this;
}

SymTensor::~SymTensor() = default;

void SymTensor::pull() const {
  if (dev_ && !host_fresh_) {
    dev_->download(*this);
    host_fresh_ = true;
  }
}

void SymTensor::detach() {
  pull();
  dev_.reset();
}

std::span<double> SymTensor::data() {
  detach();
  return data_;
}
std::span<const double> SymTensor::data() const {
  pull();
  return data_;
}
std::span<double> SymTensor::block_data(std::size_t r) {
  detach();
  return {data_.data() + (*blocks_)[r].offset, (*blocks_)[r].volume};
}
std::span<const double> SymTensor::block_data(std::size_t r) const {
  pull();
  return {data_.data() + (*blocks_)[r].offset, (*blocks_)[r].volume};
}

std::uint64_t SymTensor::block_rank(std::span<const int> block_index) const {
  require_sorted(block_index, "SymTensor::block_rank");
  return block_ranker_->rank(block_index);
}

void SymTensor::check_index(std::span<const int> index) const {
  if (static_cast<int>(index.size()) != order_) throw std::invalid_argument("SymTensor: wrong index length");
  for (int v : index)
    if (v < 0 || v >= dim_) throw std::out_of_range("SymTensor: index out of range");
}

double SymTensor::get(std::span<const int> index) const {
  check_index(index);
  std::vector<int> s(index.begin(), index.end());
  std::sort(s.begin(), s.end());
  return at_sorted_unchecked(s.data());
}
double SymTensor::get(std::initializer_list<int> index) const {
  return get(std::span<const int>(index.begin(), index.size()));
}
double SymTensor::get_sorted(std::span<const int> index) const {
  check_index(index);
  require_sorted(index, "SymTensor::get_sorted");
  return at_sorted_unchecked(index.data());
}

double SymTensor::at_sorted_unchecked(const int* index) const noexcept {
  try {
    pull();
  } catch (...) {
    return 0.0;
  }
  int j[kMaxOrder];
  for (int k = 0; k < order_; ++k) j[k] = index[k] / block_size_;
  const BlockInfo& bi = (*blocks_)[block_ranker_->rank_unchecked(j)];
  std::size_t off = 0;
  for (int k = 0; k < order_; ++k)
    off = off * static_cast<std::size_t>(bi.extents[k]) + static_cast<std::size_t>(index[k] - bi.base[k]);
  return data_[bi.offset + off];
}

void SymTensor::set_canonical(std::span<const int> index, double value) {
  check_index(index);
  detach();
  std::vector<int> s(index.begin(), index.end());
  std::sort(s.begin(), s.end());
  std::vector<int> j(order_), o(order_);
  for (int k = 0; k < order_; ++k) {
    j[k] = s[k] / block_size_;
    o[k] = s[k] - j[k] * block_size_;
  }
  const BlockInfo& bi = (*blocks_)[block_ranker_->rank(j)];
  // every distinct permutation of the offsets within runs of equal j
  std::vector<std::pair<int, int>> runs;
  for (int a = 0; a < order_;) {
    int e = a + 1;
    while (e < order_ && j[e] == j[a]) ++e;
    runs.emplace_back(a, e);
    a = e;
  }
  for (;;) {
    std::size_t off = 0;
    for (int k = 0; k < order_; ++k) off = off * bi.extents[k] + o[k];
    data_[bi.offset + off] = value;
    int q = static_cast<int>(runs.size()) - 1;
    while (q >= 0 && !std::next_permutation(o.begin() + runs[q].first, o.begin() + runs[q].second)) --q;
    if (q < 0) break;
  }
}
void SymTensor::set_canonical(std::initializer_list<int> index, double value) {
  set_canonical(std::span<const int>(index.begin(), index.size()), value);
}

std::uint64_t block_multiplicity(std::span<const int> block_index) {
  const int d = static_cast<int>(block_index.size());
  if (d < 1) throw std::invalid_argument("block_multiplicity: empty index");
  if (d > 20) throw std::invalid_argument("block_multiplicity: order too large for exact count");
  require_sorted(block_index, "block_multiplicity");
  std::uint64_t out = 0;
  check(csb_block_multiplicity(block_index.data(), d, &out));
  return out;
}
std::uint64_t block_multiplicity(std::initializer_list<int> block_index) {
  return block_multiplicity(std::span<const int>(block_index.begin(), block_index.size()));
}

SymTensor axpy(const SymTensor& t1, const SymTensor& t2, double alpha) {
  if (!t1.same_shape(t2)) throw std::invalid_argument("axpy: shape mismatch");
  SymTensor out = t1;
  auto z = out.data();
  const auto y = t2.data();
  for (std::size_t i = 0; i < z.size(); ++i) z[i] = std::fma(alpha, y[i], z[i]);
  return out;
}

double knorm(const SymTensor& t, double k) {
  if (!(k >= 1.0)) throw std::invalid_argument("knorm: k must be >= 1");
  return DeviceSeries::knorm_of(t, k);
}

// Every dense position decoded (mixed radix n), its index sorted, looked
// up in block storage.
DenseTensor densify(const SymTensor& t) {
  DenseTensor out(t.order(), t.dim());
  const int d = t.order();
  const std::size_t n = static_cast<std::size_t>(t.dim());
  t.data();  // host mirror
  std::vector<int> idx(d);
  for (std::size_t pos = 0; pos < out.values.size(); ++pos) {
    std::size_t rem = pos;
    for (int k = d - 1; k >= 0; --k, rem /= n) idx[k] = static_cast<int>(rem % n);
    std::sort(idx.begin(), idx.end());
    out.values[pos] = t.at_sorted_unchecked(idx.data());
  }
  return out;
}

// Every stored entry read from the dense tensor at its full index (block
// base plus the in-block offsets decoded from the entry's position).
SymTensor from_dense(const DenseTensor& dense, int block_size) {
  SymTensor out(dense.order, dense.dim, block_size);
  const int d = dense.order;
  auto data = out.data();
  std::vector<int> idx(d);
  for (std::size_t r = 0; r < out.block_count(); ++r) {
    const BlockInfo& bi = out.block(r);
    for (std::size_t pos = 0; pos < bi.volume; ++pos) {
      std::size_t rem = pos;
      for (int k = d - 1; k >= 0; --k) {
        const std::size_t e = static_cast<std::size_t>(bi.extents[k]);
        idx[k] = bi.base[k] + static_cast<int>(rem % e);
        rem /= e;
      }
      data[bi.offset + pos] = dense.at(idx);
    }
  }
  return out;
}

// ===========================================================================
// moments (moments.hpp:44-63)

std::uint64_t rows_read() { return csb_rows_read(); }

SymTensor moment_tensor(const DataBatch& x, int order, int block_size, int) {
  detail::check_batch(x, "moment_tensor");
  if (order < 1 || order > SymTensor::kMaxOrder) throw std::invalid_argument("moment_tensor: order out of range");
  auto ds = DeviceSeries::create(static_cast<int>(x.cols), order, block_size);
  check(csb_moment_tensor(ds->s, order, x.values.data(), x.rows, x.cols));
  SymTensor out(order, static_cast<int>(x.cols), block_size);
  DeviceSeries::attach(out, ds);
  return out;
}

MomentSeries moment_series(const DataBatch& x, int max_order, int block_size, int) {
  detail::check_batch(x, "moment_series");
  if (max_order < 1 || max_order > SymTensor::kMaxOrder)
    throw std::invalid_argument("moment_series: max_order out of range");
  auto ds = DeviceSeries::create(static_cast<int>(x.cols), max_order, block_size);
  check(csb_moment_series(ds->s, x.values.data(), x.rows, x.cols));
  return detail::wrap<MomentSeries>(ds);
}

MomentSeries combine(const MomentSeries& m1, std::size_t s1, const MomentSeries& m2, std::size_t s2) {
  if (m1.max_order() != m2.max_order()) throw std::invalid_argument("combine: order mismatch");
  if (s1 + s2 == 0) throw std::invalid_argument("combine: empty combination");
  for (int k = 1; k <= m1.max_order(); ++k)
    if (!m1.order(k).same_shape(m2.order(k))) throw std::invalid_argument("combine: shape mismatch");
  auto a = detail::acquire(m1.tensors, m1.window_len);
  auto b = detail::acquire(m2.tensors, m2.window_len);
  auto out = DeviceSeries::create(m1.dim(), m1.max_order(), m1.block_size());
  check(csb_combine(a->s, s1, b->s, s2, out->s));
  return detail::wrap<MomentSeries>(out);
}

void moments_update(MomentSeries& m, const DataBatch& incoming, const DataBatch& outgoing, int) {
  detail::check_batch(incoming, "moments_update");
  detail::check_batch(outgoing, "moments_update");
  if (m.tensors.empty()) throw std::invalid_argument("moments_update: empty series");
  if (incoming.rows != outgoing.rows) throw std::invalid_argument("moments_update: batch sizes differ");
  if (incoming.rows > m.window_len) throw std::invalid_argument("moments_update: batch longer than the window");
  const int n = m.dim();
  if (static_cast<int>(incoming.cols) != n || static_cast<int>(outgoing.cols) != n)
    throw std::invalid_argument("moments_update: dimension mismatch");
  auto ds = detail::acquire(m.tensors, m.window_len);
  check(csb_moments_update(ds->s, incoming.values.data(), outgoing.values.data(), incoming.rows,
                           incoming.cols));
  for (auto& t : m.tensors) DeviceSeries::attach(t, ds);
}

// ===========================================================================
// cumulants (cumulants.hpp:25-51)

namespace {

// Restricted growth strings a (a[0] = 0, a[i] <= 1 + max(a[0..i-1])), each
// one set partition with parts labelled by first occurrence.  next_rgs
// steps to the lexicographic successor in place: the rightmost position
// that can still grow is incremented and everything right of it reset to
// 0, prefix maxima kept alongside.  Starting from all zeros this visits the
// strings in the reference's order (cumulants.cpp:16-26).
bool next_rgs(std::vector<int>& a, std::vector<int>& pmax) {
  const int s = static_cast<int>(a.size());
  for (int i = s - 1; i >= 1; --i) {
    if (a[i] <= pmax[i - 1] && a[i] + 1 < s) {
      ++a[i];
      pmax[i] = std::max(pmax[i - 1], a[i]);
      for (int k = i + 1; k < s; ++k) {
        a[k] = 0;
        pmax[k] = pmax[k - 1];
      }
      return true;
    }
  }
  return false;
}

// emit(a, parts) for every restricted growth string of length s
template <class Emit>
void for_each_rgs(int s, Emit&& emit) {
  std::vector<int> a(s, 0), pmax(s, 0);
  do emit(a, pmax[s - 1] + 1);
  while (next_rgs(a, pmax));
}

SetPartition decode(const std::vector<int>& a, int parts) {
  SetPartition out(parts);
  for (std::size_t i = 0; i < a.size(); ++i) out[a[i]].push_back(static_cast<int>(i));
  return out;
}

void check_s(int s) {
  if (s < 1 || s > 16) throw std::invalid_argument("partitions: s must be in [1, 16]");
}

}  // namespace

std::vector<SetPartition> partitions(int s, int sigma) {
  check_s(s);
  if (sigma < 1 || sigma > s) throw std::invalid_argument("partitions: sigma must be in [1, s]");
  std::vector<SetPartition> out;
  for_each_rgs(s, [&](const std::vector<int>& g, int parts) {
    if (parts == sigma) out.push_back(decode(g, parts));
  });
  return out;
}

std::vector<SetPartition> partitions_at_least(int s, int min_sigma) {
  check_s(s);
  if (min_sigma < 1 || min_sigma > s) throw std::invalid_argument("partitions_at_least: min_sigma must be in [1, s]");
  std::vector<SetPartition> out;
  for_each_rgs(s, [&](const std::vector<int>& g, int parts) {
    if (parts >= min_sigma) out.push_back(decode(g, parts));
  });
  return out;
}

double sym_outer_element(std::span<const int> index, const CumulantSeries& lower) {
  const int s = static_cast<int>(index.size());
  check_s(s);
  if (s == 1) return 0.0;
  if (lower.max_order() < s - 1) throw std::invalid_argument("sym_outer_element: missing lower cumulant orders");
  for (int v : index)
    if (v < 0 || v >= lower.dim()) throw std::out_of_range("sym_outer_element: index out of range");
  std::vector<int> sorted(index.begin(), index.end());
  std::sort(sorted.begin(), sorted.end());
  // one element's partition sum (a test hook of the reference,
  // cumulants.cpp:110-126), same order and no FMA as the device kernel
  double acc = 0.0;
  std::vector<int> sub;
  for_each_rgs(s, [&](const std::vector<int>& g, int parts) {
    if (parts < 2) return;
    double prod = 1.0;
    for (const auto& part : decode(g, parts)) {
      sub.clear();
      for (int p : part) sub.push_back(sorted[p]);
      prod *= lower.order(static_cast<int>(part.size())).at_sorted_unchecked(sub.data());
    }
    acc += prod;  // built with -ffp-contract=off: product, then sum
  });
  return acc;
}

CumulantSeries moms2cums(const MomentSeries& m, int) {
  if (m.tensors.empty()) throw std::invalid_argument("moms2cums: empty series");
  for (int s = 1; s <= m.max_order(); ++s) {
    const SymTensor& t = m.order(s);
    if (t.order() != s || t.dim() != m.dim() || t.block_size() != m.block_size())
      throw std::invalid_argument("moms2cums: series tensors disagree on shape");
  }
  auto dm = detail::acquire(m.tensors, m.window_len);
  auto dc = DeviceSeries::create(m.dim(), m.max_order(), m.block_size());
  check(csb_moms2cums(dm->s, dc->s));
  return detail::wrap<CumulantSeries>(dc);
}

CumulantSeries cumulant_series(const DataBatch& x, int max_order, int block_size, int workers) {
  return moms2cums(moment_series(x, max_order, block_size, workers), workers);
}

// ===========================================================================
// gauge (gauge.hpp:21-60)

double nu(const CumulantSeries& c, int d) {
  if (d < 3 || d > c.max_order()) throw std::invalid_argument("nu: order must be in [3, max_order]");
  auto ds = detail::acquire(c.tensors, c.window_len);
  double out = 0.0;
  check(csb_nu(ds->s, d, &out));
  return out;
}

namespace {

// Standardised third / fourth central moment of one column from its first
// four raw moments (power sums over the rows, scaled once).
struct ColumnShape {
  double m[5] = {1.0, 0.0, 0.0, 0.0, 0.0};  // raw moments m[k] = E[x^k]
  explicit ColumnShape(const DataBatch& x, std::size_t col) {
    for (std::size_t r = 0; r < x.rows; ++r) {
      const double v = x.at(r, col);
      double p = v;
      for (int k = 1; k <= 4; ++k, p *= v) m[k] += p;
    }
    const double inv = 1.0 / static_cast<double>(x.rows);
    for (int k = 1; k <= 4; ++k) m[k] *= inv;
  }
  double variance() const { return m[2] - m[1] * m[1]; }
  double skewness() const {
    const double mu3 = m[3] - 3.0 * m[1] * m[2] + 2.0 * m[1] * m[1] * m[1];
    return mu3 / std::pow(variance(), 1.5);
  }
  double excess_kurtosis() const {
    const double a = m[1];
    const double mu4 = m[4] - 4.0 * a * m[3] + 6.0 * a * a * m[2] - 3.0 * a * a * a * a;
    return mu4 / (variance() * variance()) - 3.0;
  }
};

}  // namespace

double max_abs_univariate(const DataBatch& x, UnivariateStat stat) {
  if (x.rows < 4) throw std::invalid_argument("max_abs_univariate: need at least 4 rows");
  double best = 0.0;
  for (std::size_t col = 0; col < x.cols; ++col) {
    const ColumnShape cs(x, col);
    if (cs.variance() <= 0.0) throw std::domain_error("max_abs_univariate: zero-variance column");
    const double v = stat == UnivariateStat::kSkewness ? cs.skewness() : cs.excess_kurtosis();
    best = std::max(best, std::abs(v));
  }
  return best;
}

namespace {
csb_report device_report(const CumulantSeries& c, std::uint64_t window) {
  auto ds = detail::acquire(c.tensors, c.window_len);
  csb_report r{};
  check(csb_window_report(ds->s, window, &r));
  return r;
}
}  // namespace

double max_abs_diag_skewness(const CumulantSeries& c) {
  if (c.max_order() < 3) throw std::invalid_argument("max_abs_diag_skewness: needs order 3");
  return device_report(c, 0).max_abs_skewness;
}

double max_abs_diag_kurtosis(const CumulantSeries& c) {
  if (c.max_order() < 4) throw std::invalid_argument("max_abs_diag_kurtosis: needs order 4");
  return device_report(c, 0).max_abs_kurtosis;
}

namespace {

// Stirling numbers of the second kind S(i, j) for i <= 25, built once:
// table row i from row i - 1 by S(i, j) = j S(i-1, j) + S(i-1, j-1).
const std::array<std::array<std::uint64_t, 26>, 26>& stirling_table() {
  static const auto table = [] {
    std::array<std::array<std::uint64_t, 26>, 26> t{};
    t[0][0] = 1;
    for (int i = 1; i <= 25; ++i)
      for (int j = 1; j <= i; ++j) t[i][j] = static_cast<std::uint64_t>(j) * t[i - 1][j] + t[i - 1][j - 1];
    return t;
  }();
  return table;
}

}  // namespace

std::uint64_t stirling2(int s, int sigma) {
  if (s < 1 || s > 25) throw std::invalid_argument("stirling2: s must be in [1, 25]");
  return sigma < 1 || sigma > s ? 0 : stirling_table()[s][sigma];
}

// Bell numbers from the Bell (Aitken) triangle: each row starts with the
// previous row's last entry, each next entry adds the entry above-left;
// B(s) is the first entry of row s.
std::uint64_t bell_number(int s) {
  if (s < 1 || s > 25) throw std::invalid_argument("bell_number: s must be in [1, 25]");
  std::vector<std::uint64_t> row{1};
  for (int i = 1; i <= s; ++i) {
    std::vector<std::uint64_t> next{row.back()};
    for (std::uint64_t v : row) next.push_back(next.back() + v);
    row.swap(next);
  }
  return row.front();
}

double moment_error_bound(int d, std::size_t t, double m_2d) {
  if (d < 1) throw std::invalid_argument("moment_error_bound: order must be positive");
  if (t < 1) throw std::invalid_argument("moment_error_bound: need samples");
  if (m_2d < 0.0) throw std::invalid_argument("moment_error_bound: negative moment bound");
  return std::sqrt(m_2d / static_cast<double>(t));
}

double gaussian_moment_error_bound(int d, std::size_t t) {
  // E[z^{2d}] of a standard normal: (2d - 1)!! = 1 * 3 * ... * (2d - 1)
  double m = 1.0;
  for (int k = 2; k <= d; ++k) m *= static_cast<double>(2 * k - 1);
  return moment_error_bound(d, t, m);
}

double predicted_speedup(std::size_t t, std::size_t t_up, int d) {
  if (t_up < 1 || t < t_up) throw std::invalid_argument("predicted_speedup: need 1 <= t_up <= t");
  return static_cast<double>(t) / (2.0 * static_cast<double>(t_up) + static_cast<double>(bell_number(d)));
}

double predicted_moment_speedup(std::size_t t, std::size_t t_up) {
  if (t_up < 1 || t < t_up) throw std::invalid_argument("predicted_moment_speedup: need 1 <= t_up <= t");
  return static_cast<double>(t) / (2.0 * static_cast<double>(t_up));
}

namespace {
WindowReport to_report(const csb_report& r) {
  WindowReport rep;
  rep.window = r.window;
  rep.rows = r.rows;
  rep.norm_c1 = r.norm_c1;
  rep.norm_c2 = r.norm_c2;
  for (int k = 0; k < r.n_nu; ++k) rep.nu[k + 3] = r.nu[k];
  if (r.has_skewness) rep.max_abs_skewness = r.max_abs_skewness;
  if (r.has_kurtosis) rep.max_abs_kurtosis = r.max_abs_kurtosis;
  return rep;
}

// JSON number: shortest round-trip form, integral values keep ".0"
#if !CSB_HAVE_NLOHMANN
std::string num(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof buf, v);
  std::string s(buf, res.ptr);
  if (s.find_first_of(".eE") == std::string::npos) s += ".0";
  return s;
}
#endif
}  // namespace

WindowReport make_window_report(std::uint64_t window, const CumulantSeries& c) {
  if (c.max_order() < 2) throw std::invalid_argument("make_window_report: needs orders up to 2");
  return to_report(device_report(c, window));
}

std::string report_json_line(const WindowReport& r) {
#if CSB_HAVE_NLOHMANN
  // the reference's JSON library (nlohmann/json 3.11.3, ordered_json) and
  // key order (gauge.cpp:156-168, docs/window_report.schema.json): with
  // bit-identical report values the lines are byte-identical
  nlohmann::ordered_json j;
  j["window"] = r.window;
  j["rows"] = r.rows;
  j["norm_c1"] = r.norm_c1;
  j["norm_c2"] = r.norm_c2;
  auto nus = nlohmann::ordered_json::object();
  for (const auto& [o, v] : r.nu) nus[std::to_string(o)] = v;
  j["nu"] = std::move(nus);
  if (r.max_abs_skewness) j["max_abs_skewness"] = *r.max_abs_skewness;
  if (r.max_abs_kurtosis) j["max_abs_kurtosis"] = *r.max_abs_kurtosis;
  return j.dump();
#else
  // key order of docs/window_report.schema.json
  std::string s = "{\"window\":" + std::to_string(r.window) + ",\"rows\":" + std::to_string(r.rows) +
                  ",\"norm_c1\":" + num(r.norm_c1) + ",\"norm_c2\":" + num(r.norm_c2) + ",\"nu\":{";
  bool first = true;
  for (const auto& [o, v] : r.nu) {
    if (!first) s += ",";
    first = false;
    s += "\"" + std::to_string(o) + "\":" + num(v);
  }
  s += "}";
  if (r.max_abs_skewness) s += ",\"max_abs_skewness\":" + num(*r.max_abs_skewness);
  if (r.max_abs_kurtosis) s += ",\"max_abs_kurtosis\":" + num(*r.max_abs_kurtosis);
  return s + "}";
#endif
}

// ===========================================================================
// stream (stream.hpp:19-89)

void StreamConfig::validate() const {
  const std::pair<bool, const char*> rules[] = {
      {dim >= 1, "StreamConfig: dim must be positive"},
      {max_order >= 2, "StreamConfig: max_order must be >= 2"},
      {window_len >= 1, "StreamConfig: window_len must be positive"},
      {update_len >= 1 && update_len <= window_len, "StreamConfig: update_len must be in [1, window_len]"},
      {block_size >= 1 && block_size <= dim, "StreamConfig: block_size must be in [1, dim]"},
      {workers >= 0, "StreamConfig: workers must be >= 0"},
      {shard_count >= 1 && shard_index >= 0 && shard_index < shard_count,
       "StreamConfig: shard_index must be in [0, shard_count)"},
  };
  for (const auto& [ok, msg] : rules)
    if (!ok) throw std::invalid_argument(msg);
}

WindowBuffer::WindowBuffer(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), values_(rows * cols) {}

void WindowBuffer::fill(const DataBatch& x) {
  if (device_) throw std::runtime_error("WindowBuffer::fill: the window lives on the device (use prime)");
  if (x.rows != rows_ || x.cols != cols_)
    throw std::invalid_argument("WindowBuffer::fill: batch does not match capacity");
  values_.assign(x.values.begin(), x.values.end());
  head_ = 0;
}

// The oldest x.rows rows leave and x's rows take their slots: at most two
// contiguous segments of the ring (before and after the wrap), each swapped
// with the matching span of the batch.
DataBatch WindowBuffer::exchange(const DataBatch& x) {
  if (device_) throw std::runtime_error("WindowBuffer::exchange: the window lives on the device (use step)");
  if (x.cols != cols_) throw std::invalid_argument("WindowBuffer::exchange: column mismatch");
  if (x.rows < 1 || x.rows > rows_) throw std::invalid_argument("WindowBuffer::exchange: batch size out of range");
  DataBatch out;
  out.rows = x.rows;
  out.cols = cols_;
  out.values = x.values;
  const std::size_t first = std::min(x.rows, rows_ - head_);
  auto ring = values_.begin();
  std::swap_ranges(ring + head_ * cols_, ring + (head_ + first) * cols_, out.values.begin());
  std::swap_ranges(ring, ring + (x.rows - first) * cols_, out.values.begin() + first * cols_);
  head_ = (head_ + x.rows) % rows_;
  return out;
}

DataBatch WindowBuffer::materialize() const {
  DataBatch out;
  out.rows = rows_;
  out.cols = cols_;
  out.values.resize(rows_ * cols_);
  if (device_) {
    check(csb_stream_materialize(device_->st, out.values.data(), out.values.size()));
    return out;
  }
  // arrival order: the ring rotated so the oldest row (head) comes first
  std::rotate_copy(values_.begin(), values_.begin() + head_ * cols_, values_.end(), out.values.begin());
  return out;
}

namespace {

csb_stream_config to_c(const StreamConfig& c) {
  csb_stream_config cc{};
  cc.dim = c.dim;
  cc.max_order = c.max_order;
  cc.window_len = c.window_len;
  cc.update_len = c.update_len;
  cc.block_size = c.block_size;
  cc.resync_every = c.resync_every;
  cc.workers = c.workers;
  cc.shard_index = c.shard_index;
  cc.shard_count = c.shard_count;
  return cc;
}

std::shared_ptr<DeviceSeries> borrow(const std::shared_ptr<detail::DeviceStream>& ds, const csb_series* s,
                                     const StreamConfig& cfg) {
  auto out = std::make_shared<DeviceSeries>();
  out->s = const_cast<csb_series*>(s);
  out->owned = false;
  out->keep = ds;
  out->n = cfg.dim;
  out->d = cfg.max_order;
  out->b = cfg.block_size;
  return out;
}

}  // namespace

WindowState prime(const StreamConfig& config, const DataBatch& first) {
  config.validate();
  if (first.rows != config.window_len || static_cast<int>(first.cols) != config.dim)
    throw std::invalid_argument("prime: batch does not match the configured window");
  auto dev = std::make_shared<detail::DeviceStream>();
  const csb_stream_config cc = to_c(config);
  check(csb_stream_prime(&cc, first.values.data(), first.rows, first.cols, &dev->st));
  const csb_series* m = nullptr;
  check(csb_stream_moments(dev->st, &m));
  dev->m = borrow(dev, m, config);
  WindowState state;
  state.config = config;
  state.buffer = WindowBuffer(config.window_len, static_cast<std::size_t>(config.dim));
  detail::DeviceStream::bind(state.buffer, dev);
  state.moments = detail::wrap<MomentSeries>(dev->m);
  state.window = 1;
  state.steps_since_resync = 0;
  state.device = dev;
  return state;
}

CumulantSeries step(WindowState& state, const DataBatch& x, StepTiming* timing) {
  const StreamConfig& cfg = state.config;
  if (x.rows != cfg.update_len || static_cast<int>(x.cols) != cfg.dim)
    throw std::invalid_argument("step: batch does not match the configured update");
  if (!state.device) throw std::invalid_argument("step: state was not created by prime()");
  auto& dev = *state.device;
  // host-side edits of state.moments (writes through data()) flow back in
  detail::sync_into(state.moments.tensors, dev.m);
  csb_step_timing t{};
  check(csb_stream_step(dev.st, x.values.data(), x.rows, x.cols, timing ? &t : nullptr, nullptr));
  if (timing) {
    timing->update_s = t.update_s;
    timing->moms2cums_s = t.moms2cums_s;
  }
  for (auto& tt : state.moments.tensors) DeviceSeries::attach(tt, dev.m);
  state.steps_since_resync = (cfg.resync_every > 0 && state.steps_since_resync + 1 >= cfg.resync_every)
                                 ? 0
                                 : state.steps_since_resync + 1;
  ++state.window;
  // the returned series is a value: snapshot the stream's cumulants
  const csb_series* c = nullptr;
  check(csb_stream_cumulants(dev.st, &c));
  auto snap = DeviceSeries::create(cfg.dim, cfg.max_order, cfg.block_size);
  check(csb_series_copy(snap->s, c));
  return detail::wrap<CumulantSeries>(snap);
}

CumulantSeries gather_shards(WindowState& state) {
  if (!state.device) throw std::invalid_argument("gather_shards: state was not created by prime()");
  auto& dev = *state.device;
  const StreamConfig& cfg = state.config;
  detail::sync_into(state.moments.tensors, dev.m);
  check(csb_stream_gather_shards(dev.st));
  for (auto& tt : state.moments.tensors) DeviceSeries::attach(tt, dev.m);  // host mirrors are stale now
  const csb_series* c = nullptr;
  check(csb_stream_cumulants(dev.st, &c));
  auto snap = DeviceSeries::create(cfg.dim, cfg.max_order, cfg.block_size);
  check(csb_series_copy(snap->s, c));
  return detail::wrap<CumulantSeries>(snap);
}

void run(const StreamConfig& config, BatchSource& source, const ReportSink& sink) {
  config.validate();
  auto first = source.next(config.window_len);
  if (!first || first->rows < config.window_len)
    throw std::runtime_error("run: source ended before the first window was full");
  WindowState state = prime(config, *first);
  first.reset();
  csb_report r{};
  check(csb_stream_report(state.device->st, &r));
  sink(to_report(r));
  // Pipelined ingestion: while the device runs step k, the
  // host reads batch k + 1 from the source and starts its copy on the
  // engine's copy stream; the report of step k is fetched afterwards.
  const auto take = [&]() -> std::optional<DataBatch> {
    auto batch = source.next(config.update_len);
    if (!batch) return std::nullopt;
    if (batch->rows < config.update_len) {
      if (batch->rows > 0)
        std::cerr << "warning: discarding " << batch->rows << " trailing rows shorter than one update\n";
      return std::nullopt;
    }
    if (batch->cols != static_cast<std::size_t>(config.dim))
      throw std::invalid_argument("step: batch does not match the configured update");
    return batch;
  };
  csb_stream* st = state.device->st;
  std::optional<DataBatch> cur = take();
  if (cur) check(csb_stream_upload(st, cur->values.data(), cur->rows, cur->cols));
  while (cur) {
    check(csb_stream_step_uploaded(st, nullptr, nullptr));  // queued; returns at once
    std::optional<DataBatch> next;
    std::exception_ptr bad;  // a failing read surfaces after this step's report, as in the reference's loop
    try {
      next = take();  // host ingestion under the step
      if (next) check(csb_stream_upload(st, next->values.data(), next->rows, next->cols));
    } catch (...) {
      bad = std::current_exception();
    }
    check(csb_stream_report(st, &r));  // waits for the step
    ++state.window;
    sink(to_report(r));
    if (bad) std::rethrow_exception(bad);
    cur = std::move(next);
  }
}

}  // namespace cumstream
