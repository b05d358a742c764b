// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// The reference's own `process` path, driven through its public API only
// (csv.hpp CsvBatchSource, stream.hpp run, gauge.hpp report_json_line;
// /root/reference/proj/src/stream.cpp:110-132, gauge.cpp:156-168), with the
// same command line as paper_1701_06446_b200/cpp/tests/process_main.cpp so
// tests/test_gpu_report_exact.py can compare the two JSONL outputs byte
// for byte.  Built by `make -C oracle ref` from the reference sources in
// place (never copied), next to the reference shim libraries.
//   ref_process_v4 CSV DIM ORDER WINDOW UPDATE BLOCK [DUMPDIR]
// With DUMPDIR, every window's cumulants are also written as
// DUMPDIR/window_<w>.json with the reference's to_json (serialize.cpp:61-75,
// indent 1: the --dump-cumulants layout of tools/cumstream.cpp:90-96).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <stdexcept>
#include <string>

#include "cumstream/csv.hpp"
#include "cumstream/gauge.hpp"
#include "cumstream/serialize.hpp"
#include "cumstream/stream.hpp"

int main(int argc, char** argv) {
  if (argc != 7 && argc != 8) {
    std::fprintf(stderr, "usage: %s CSV DIM ORDER WINDOW UPDATE BLOCK [DUMPDIR]\n", argv[0]);
    return 1;
  }
  cumstream::StreamConfig cfg;
  cfg.dim = std::atoi(argv[2]);
  cfg.max_order = std::atoi(argv[3]);
  cfg.window_len = std::strtoull(argv[4], nullptr, 10);
  cfg.update_len = std::strtoull(argv[5], nullptr, 10);
  cfg.block_size = std::atoi(argv[6]);
  cfg.resync_every = 0;
  try {
    std::ifstream in(argv[1]);
    cumstream::CsvBatchSource source(in, cfg.dim);
    if (argc == 8) {
      const std::string dir = argv[7];
      const auto emit = [&](std::uint64_t w, const cumstream::CumulantSeries& c) {
        std::cout << cumstream::report_json_line(cumstream::make_window_report(w, c)) << "\n";
        std::ofstream f(dir + "/window_" + std::to_string(w) + ".json");
        f << cumstream::to_json(c, w, 1) << "\n";
      };
      auto first = source.next(cfg.window_len);
      if (!first || first->rows < cfg.window_len) throw std::runtime_error("short input");
      cumstream::WindowState state = cumstream::prime(cfg, *first);
      emit(state.window, cumstream::moms2cums(state.moments));
      for (auto b = source.next(cfg.update_len); b && b->rows == cfg.update_len; b = source.next(cfg.update_len)) {
        const cumstream::CumulantSeries c = cumstream::step(state, *b);
        emit(state.window, c);
      }
      return 0;
    }
    cumstream::run(cfg, source,
                   [](const cumstream::WindowReport& r) { std::cout << cumstream::report_json_line(r) << "\n"; });
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  }
  return 0;
}
