// CSV row source and writer (csv.hpp): host-side ingestion in front of the
// device stream (run() pulls batches from a BatchSource).
#include "cumstream/csv.hpp"

#include <charconv>
#include <istream>
#include <ostream>
#include <stdexcept>
#include <string>

namespace cumstream {
namespace {

bool blank(const std::string& s) {
  for (char c : s)
    if (c != ' ' && c != '\t' && c != '\r') return false;
  return true;
}

// fields of one line into out (cols of them), else a runtime_error
void parse_line(const std::string& s, std::size_t line, std::size_t cols, double* out) {
  std::size_t field = 0, i = 0;
  const std::size_t n = s.size();
  while (true) {
    std::size_t j = s.find(',', i);
    if (j == std::string::npos) j = n;
    std::size_t a = i, b = j;
    while (a < b && (s[a] == ' ' || s[a] == '\t')) ++a;
    while (b > a && (s[b - 1] == ' ' || s[b - 1] == '\t' || s[b - 1] == '\r')) --b;
    if (field >= cols)
      throw std::runtime_error("csv: expected " + std::to_string(cols) + " fields, got more on line " +
                               std::to_string(line));
    double v = 0.0;
    const char* first = s.data() + a;
    if (a < b && *first == '+') ++first;  // from_chars takes no leading '+'
    const auto r = std::from_chars(first, s.data() + b, v);
    if (a == b || r.ec != std::errc() || r.ptr != s.data() + b)
      throw std::runtime_error("csv: unparsable number on line " + std::to_string(line));
    out[field++] = v;
    if (j == n) break;
    i = j + 1;
  }
  if (field != cols)
    throw std::runtime_error("csv: expected " + std::to_string(cols) + " fields, got " + std::to_string(field) +
                             " on line " + std::to_string(line));
}

}  // namespace

CsvBatchSource::CsvBatchSource(std::istream& in, std::size_t cols, bool skip_header) : in_(in), cols_(cols) {
  if (cols == 0) throw std::invalid_argument("CsvBatchSource: cols must be positive");
  if (skip_header) {
    std::string h;
    if (std::getline(in_, h)) ++line_;
  }
}

std::optional<DataBatch> CsvBatchSource::next(std::size_t rows) {
  if (drained_) return std::nullopt;
  DataBatch b;
  b.cols = cols_;
  b.values.reserve(rows * cols_);
  std::string s;
  while (b.rows < rows && std::getline(in_, s)) {
    ++line_;
    if (blank(s)) continue;
    b.values.resize((b.rows + 1) * cols_);
    parse_line(s, line_, cols_, b.values.data() + b.rows * cols_);
    ++b.rows;
  }
  if (b.rows < rows) drained_ = true;
  return b;
}

void write_csv(std::ostream& out, const DataBatch& x) {
  char buf[64];
  std::string line;
  for (std::size_t r = 0; r < x.rows; ++r) {
    line.clear();
    for (std::size_t c = 0; c < x.cols; ++c) {
      if (c) line += ',';
      const auto res = std::to_chars(buf, buf + sizeof buf, x.at(r, c));
      line.append(buf, res.ptr);
    }
    line += '\n';
    out << line;
  }
}

}  // namespace cumstream
