// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference library (cumstream, compiled in
// place from /root/reference/proj/src by oracle/Makefile with
// -Dcumstream=cumstream_ref so it can share a process with the product).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load the resulting oracle/_ref/*.so.
//
// Every entry point is a flat-array restatement of one reference call:
//   ref_moment_series   -> cumstream::moment_series   (include/cumstream/moments.hpp:52)
//   ref_moments_update  -> cumstream::moments_update  (moments.hpp:62)
//   ref_moms2cums       -> cumstream::moms2cums       (cumulants.hpp:47)
//   ref_knorm           -> cumstream::knorm           (symten.hpp:156)
//   ref_nu              -> cumstream::nu              (gauge.hpp:21)
//   ref_report          -> cumstream::make_window_report (gauge.hpp:57)
//   ref_stream_*        -> cumstream::prime / step    (stream.hpp:69,73)
// Tensors cross the boundary as one flat block-storage array per order,
// exactly SymTensor::data() (symten.hpp:122).
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "cumstream/cumulants.hpp"
#include "cumstream/gauge.hpp"
#include "cumstream/moments.hpp"
#include "cumstream/parallel.hpp"
#include "cumstream/stream.hpp"
#include "cumstream/symten.hpp"

namespace cs = cumstream_ref;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::out_of_range& e) {
    return fail(e, 2);
  } catch (const std::domain_error& e) {
    return fail(e, 3);
  } catch (const std::exception& e) {
    return fail(e, 4);
  }
}

cs::DataBatch batch(const double* x, std::size_t rows, std::size_t cols) {
  cs::DataBatch b;
  b.rows = rows;
  b.cols = cols;
  b.values.assign(x, x + rows * cols);
  return b;
}

void load(cs::SymTensor& t, const double* src) {
  auto d = t.data();
  std::memcpy(d.data(), src, d.size() * sizeof(double));
}

void store(const cs::SymTensor& t, double* dst) {
  auto d = t.data();
  std::memcpy(dst, d.data(), d.size() * sizeof(double));
}

template <class Series>
Series series_from(const double* const* orders, std::size_t window_len, int n, int d, int b) {
  Series s;
  s.window_len = window_len;
  for (int k = 1; k <= d; ++k) {
    cs::SymTensor t(k, n, b);
    load(t, orders[k - 1]);
    s.tensors.push_back(std::move(t));
  }
  return s;
}

struct RefStream {
  cs::WindowState state;
  cs::CumulantSeries last;
};

void fill_report(const cs::WindowReport& r, double* out) {
  // out: [window, rows, norm_c1, norm_c2, skew (nan if absent), kurt, nu3..nu_d]
  out[0] = static_cast<double>(r.window);
  out[1] = static_cast<double>(r.rows);
  out[2] = r.norm_c1;
  out[3] = r.norm_c2;
  out[4] = r.max_abs_skewness ? *r.max_abs_skewness : __builtin_nan("");
  out[5] = r.max_abs_kurtosis ? *r.max_abs_kurtosis : __builtin_nan("");
  int i = 6;
  for (const auto& kv : r.nu) out[i++] = kv.second;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_layout_size(int order, int dim, int block, std::uint64_t* stored, std::uint64_t* blocks) {
  return guard([&] {
    cs::SymTensor t(order, dim, block);
    *stored = t.size();
    *blocks = t.block_count();
  });
}

// Block table: for each stored block r, index[order] and offset.
int ref_block_table(int order, int dim, int block, int* index_out, std::uint64_t* offset_out) {
  return guard([&] {
    cs::SymTensor t(order, dim, block);
    for (std::size_t r = 0; r < t.block_count(); ++r) {
      const auto& bi = t.block(r);
      for (int k = 0; k < order; ++k) index_out[r * order + k] = bi.index[k];
      offset_out[r] = bi.offset;
    }
  });
}

int ref_moment_series(const double* x, std::size_t rows, std::size_t cols, int d, int b,
                      int workers, double* const* out) {
  return guard([&] {
    const cs::MomentSeries m = cs::moment_series(batch(x, rows, cols), d, b, workers);
    for (int s = 1; s <= d; ++s) store(m.order(s), out[s - 1]);
  });
}

int ref_moment_tensor(const double* x, std::size_t rows, std::size_t cols, int order, int b,
                      int workers, double* out) {
  return guard([&] {
    store(cs::moment_tensor(batch(x, rows, cols), order, b, workers), out);
  });
}

int ref_moments_update(double* const* m, std::size_t window_len, const double* in,
                       const double* outg, std::size_t rows, std::size_t cols, int d, int b,
                       int workers) {
  return guard([&] {
    auto ms = series_from<cs::MomentSeries>(m, window_len, static_cast<int>(cols), d, b);
    cs::moments_update(ms, batch(in, rows, cols), batch(outg, rows, cols), workers);
    for (int s = 1; s <= d; ++s) store(ms.order(s), m[s - 1]);
  });
}

int ref_moms2cums(const double* const* m, double* const* c, std::size_t window_len, int n, int d,
                  int b, int workers) {
  return guard([&] {
    const auto ms = series_from<cs::MomentSeries>(m, window_len, n, d, b);
    const cs::CumulantSeries cu = cs::moms2cums(ms, workers);
    for (int s = 1; s <= d; ++s) store(cu.order(s), c[s - 1]);
  });
}

int ref_knorm(const double* t, int order, int n, int b, double k, double* out) {
  return guard([&] {
    cs::SymTensor st(order, n, b);
    load(st, t);
    *out = cs::knorm(st, k);
  });
}

int ref_nu(const double* const* c, int n, int d, int b, int order, double* out) {
  return guard([&] {
    const auto cu = series_from<cs::CumulantSeries>(c, 1, n, d, b);
    *out = cs::nu(cu, order);
  });
}

int ref_report(const double* const* c, std::size_t window_len, int n, int d, int b,
               std::uint64_t window, double* out) {
  return guard([&] {
    const auto cu = series_from<cs::CumulantSeries>(c, window_len, n, d, b);
    fill_report(cs::make_window_report(window, cu), out);
  });
}

int ref_sym_outer_element(const int* index, int s, const double* const* c, int n, int d, int b,
                          double* out) {
  return guard([&] {
    const auto cu = series_from<cs::CumulantSeries>(c, 1, n, d, b);
    *out = cs::sym_outer_element(std::vector<int>(index, index + s), cu);
  });
}

// Packed partitions of {0..s-1} into exactly sigma parts, RGS order:
// per partition, per part: [len, members...].  Returns the count in *count
// and the packed ints in out (cap ints).
int ref_partitions(int s, int sigma, int* out, std::size_t cap, std::size_t* used,
                   std::size_t* count) {
  return guard([&] {
    const auto ps = cs::partitions(s, sigma);
    std::size_t w = 0;
    for (const auto& p : ps)
      for (const auto& part : p) {
        if (w + 1 + part.size() > cap) throw std::length_error("ref_partitions: cap");
        out[w++] = static_cast<int>(part.size());
        for (int v : part) out[w++] = v;
      }
    *used = w;
    *count = ps.size();
  });
}

std::uint64_t ref_rows_read() { return cs::rows_read(); }
std::uint64_t ref_bell_number(int s) { return cs::bell_number(s); }
std::uint64_t ref_stirling2(int s, int sigma) { return cs::stirling2(s, sigma); }
double ref_predicted_speedup(std::size_t t, std::size_t t_up, int d) {
  return cs::predicted_speedup(t, t_up, d);
}
int ref_resolve_workers(int requested) { return cs::resolve_workers(requested); }

int ref_stream_prime(int n, int d, std::size_t t, std::size_t t_up, int b,
                     std::size_t resync_every, int workers, const double* first, void** handle) {
  return guard([&] {
    cs::StreamConfig cfg;
    cfg.dim = n;
    cfg.max_order = d;
    cfg.window_len = t;
    cfg.update_len = t_up;
    cfg.block_size = b;
    cfg.resync_every = resync_every;
    cfg.workers = workers;
    auto* s = new RefStream;
    try {
      s->state = cs::prime(cfg, batch(first, t, static_cast<std::size_t>(n)));
      s->last = cs::moms2cums(s->state.moments, workers);
    } catch (...) {
      delete s;
      throw;
    }
    *handle = s;
  });
}

// One step; report_out as in ref_report; timing_out = [update_s, moms2cums_s].
int ref_stream_step(void* handle, const double* x, std::size_t rows, std::size_t cols,
                    double* timing_out, double* report_out) {
  return guard([&] {
    auto* s = static_cast<RefStream*>(handle);
    cs::StepTiming tm;
    s->last = cs::step(s->state, batch(x, rows, cols), &tm);
    if (timing_out) {
      timing_out[0] = tm.update_s;
      timing_out[1] = tm.moms2cums_s;
    }
    if (report_out) fill_report(cs::make_window_report(s->state.window, s->last), report_out);
  });
}

int ref_stream_report(void* handle, double* report_out) {
  return guard([&] {
    auto* s = static_cast<RefStream*>(handle);
    fill_report(cs::make_window_report(s->state.window, s->last), report_out);
  });
}

int ref_stream_moments(void* handle, int order, double* out) {
  return guard([&] { store(static_cast<RefStream*>(handle)->state.moments.order(order), out); });
}

int ref_stream_cumulants(void* handle, int order, double* out) {
  return guard([&] { store(static_cast<RefStream*>(handle)->last.order(order), out); });
}

int ref_stream_materialize(void* handle, double* out) {
  return guard([&] {
    const auto b = static_cast<RefStream*>(handle)->state.buffer.materialize();
    std::memcpy(out, b.values.data(), b.values.size() * sizeof(double));
  });
}

void ref_stream_free(void* handle) { delete static_cast<RefStream*>(handle); }

}  // extern "C"
