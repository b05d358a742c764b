// The `cumstream process` path end to end (the
// shape of the reference's acceptance check 8, tests/acceptance.cpp:397):
// rows written to a CSV file, streamed back through CsvBatchSource into
// run(), one report_json_line per window.  Checks: two runs give
// byte-identical JSONL with one line per window, and the lines equal those
// of prime()/step() fed the same batches directly (CSV round trip exact).
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "cumstream/csv.hpp"
#include "cumstream/cumulants.hpp"
#include "cumstream/gauge.hpp"
#include "cumstream/serialize.hpp"
#include "cumstream/stream.hpp"

using namespace cumstream;

// process CSV DIM ORDER WINDOW UPDATE BLOCK [DUMPDIR]: the stream of a CSV
// file, one report line per window on stdout (the same CLI as
// oracle/ref_process.cpp, which drives the reference library:
// tests/test_gpu_report_exact.py compares the two outputs byte for byte).
// With DUMPDIR each window's cumulants go to DUMPDIR/window_<w>.json
// (to_json, indent 1: the reference CLI's --dump-cumulants,
// tools/cumstream.cpp:90-96), gathered from the shards when there are any.
int process_file(int argc, char** argv) {
  if (argc != 7 && argc != 8) {
    std::fprintf(stderr, "usage: %s CSV DIM ORDER WINDOW UPDATE BLOCK [DUMPDIR]\n", argv[0]);
    return 1;
  }
  StreamConfig cfg;
  cfg.dim = std::atoi(argv[2]);
  cfg.max_order = std::atoi(argv[3]);
  cfg.window_len = std::strtoull(argv[4], nullptr, 10);
  cfg.update_len = std::strtoull(argv[5], nullptr, 10);
  cfg.block_size = std::atoi(argv[6]);
  cfg.resync_every = 0;
  try {
    std::ifstream in(argv[1]);
    CsvBatchSource source(in, cfg.dim);
    if (argc == 8) {
      const std::string dir = argv[7];
      const auto emit = [&](std::uint64_t w, const CumulantSeries& c) {
        std::cout << report_json_line(make_window_report(w, c)) << "\n";
        std::ofstream f(dir + "/window_" + std::to_string(w) + ".json");
        f << to_json(c, w, 1) << "\n";
      };
      auto first = source.next(cfg.window_len);
      if (!first || first->rows < cfg.window_len) throw std::runtime_error("short input");
      WindowState state = prime(cfg, *first);
      emit(state.window, gather_shards(state));
      for (auto b = source.next(cfg.update_len); b && b->rows == cfg.update_len; b = source.next(cfg.update_len)) {
        step(state, *b);
        emit(state.window, gather_shards(state));
      }
      return 0;
    }
    run(cfg, source, [](const WindowReport& r) { std::cout << report_json_line(r) << "\n"; });
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  }
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1) return process_file(argc, argv);
  namespace fs = std::filesystem;
  const fs::path dir = fs::temp_directory_path() / "cumstream_b200_process";
  fs::create_directories(dir);
  const fs::path csv = dir / "stream.csv";
  StreamConfig cfg;
  cfg.dim = 6;
  cfg.max_order = 4;
  cfg.window_len = 400;
  cfg.update_len = 100;
  cfg.block_size = 2;
  const int windows = 6;
  std::vector<DataBatch> batches;
  {
    std::mt19937_64 mt(808);
    std::normal_distribution<double> g(0.0, 1.0);
    std::ofstream f(csv);
    for (int k = 0; k < windows; ++k) {
      DataBatch b;
      b.rows = k == 0 ? cfg.window_len : cfg.update_len;
      b.cols = cfg.dim;
      b.values.resize(b.rows * b.cols);
      for (auto& v : b.values) v = g(mt) * 1.5 + 0.25;
      write_csv(f, b);
      batches.push_back(std::move(b));
    }
  }
  const auto run_once = [&]() {
    std::ifstream in(csv);
    CsvBatchSource source(in, cfg.dim);
    std::ostringstream out;
    run(cfg, source, [&](const WindowReport& r) { out << report_json_line(r) << "\n"; });
    return out.str();
  };
  try {
    const std::string a = run_once(), b = run_once();
    std::ostringstream direct;
    WindowState st = prime(cfg, batches[0]);
    direct << report_json_line(make_window_report(st.window, moms2cums(st.moments))) << "\n";
    for (int k = 1; k < windows; ++k) {
      const CumulantSeries c = step(st, batches[k]);
      direct << report_json_line(make_window_report(st.window, c)) << "\n";
    }
    std::size_t lines = 0;
    for (char ch : a) lines += ch == '\n';
    const bool same = !a.empty() && a == b;
    const bool match = a == direct.str();
    std::cout << a;
    if (a != direct.str()) std::cout << "direct prime/step lines:\n" << direct.str();
    std::printf("runs byte-identical: %s; lines: %zu (want %d); equal to prime/step: %s\n", same ? "yes" : "no",
                lines, windows, match ? "yes" : "no");
    return same && match && lines == static_cast<std::size_t>(windows) ? 0 : 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  }
}
