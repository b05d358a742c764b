// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// The reference's own `process` path, driven through its public API only
// (csv.hpp CsvBatchSource, stream.hpp run, gauge.hpp report_json_line;
// /root/reference/proj/src/stream.cpp:110-132, gauge.cpp:156-168), with the
// same command line as paper_1701_06446_b200/cpp/tests/process_main.cpp so
// tests/test_gpu_report_exact.py can compare the two JSONL outputs byte
// for byte.  Built by `make -C oracle ref` from the reference sources in
// place (never copied), next to the reference shim libraries.
//   ref_process_v4 CSV DIM ORDER WINDOW UPDATE BLOCK
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>

#include "cumstream/csv.hpp"
#include "cumstream/gauge.hpp"
#include "cumstream/stream.hpp"

int main(int argc, char** argv) {
  if (argc != 7) {
    std::fprintf(stderr, "usage: %s CSV DIM ORDER WINDOW UPDATE BLOCK\n", argv[0]);
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
    cumstream::run(cfg, source,
                   [](const cumstream::WindowReport& r) { std::cout << cumstream::report_json_line(r) << "\n"; });
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 2;
  }
  return 0;
}
