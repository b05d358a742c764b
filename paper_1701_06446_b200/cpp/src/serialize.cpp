// JSON dumps of block tensors / cumulant series (serialize.hpp).  Host-side
// formatting of the downloaded block storage and a small parser for the
// same shape; follows the reference's format (src/serialize.cpp:13-75 of
// the reference: key names, block order, error type), not its code.
#include "cumstream/serialize.hpp"

#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <istream>
#include <iterator>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include <json.hpp>  // nlohmann/json 3.11.3, the reference's JSON dependency (number formatting only)

namespace cumstream {
namespace {

[[noreturn]] void bad(const std::string& what) { throw std::runtime_error("sym_tensor_from_json: " + what); }

// Numbers go through the number formatter of the reference's JSON library
// (nlohmann/json 3.11.3, Grisu2: round-trip exact, and the shortest form
// except in rare cases) so a dump equals the reference's byte for byte --
// std::to_chars' always-shortest digits differ from it in those rare cases.
std::string number(double v) {
  if (!std::isfinite(v)) return "null";  // JSON has no inf/nan (nlohmann writes null too)
  char buf[64];
  const char* end = nlohmann::detail::to_chars(buf, buf + sizeof buf, v);
  return std::string(static_cast<const char*>(buf), end);
}

// Writer with nlohmann-like layout: compact for indent < 0, else one
// element per line indented by `indent` spaces per level.
struct Writer {
  int indent;
  std::string out;
  void nl(int level) {
    if (indent < 0) return;
    out += '\n';
    out.append(static_cast<std::size_t>(indent * level), ' ');
  }
  void key(const char* k, int level, bool first) {
    if (!first) out += ',';
    nl(level);
    out += '"';
    out += k;
    out += indent < 0 ? "\":" : "\": ";
  }
  void tensor(const SymTensor& t, int level) {
    out += '{';
    key("order", level + 1, true);
    out += std::to_string(t.order());
    key("dim", level + 1, false);
    out += std::to_string(t.dim());
    key("block_size", level + 1, false);
    out += std::to_string(t.block_size());
    key("blocks", level + 1, false);
    out += '[';
    for (std::size_t r = 0; r < t.block_count(); ++r) {
      if (r) out += ',';
      nl(level + 2);
      out += '[';
      const auto v = t.block_data(r);
      for (std::size_t i = 0; i < v.size(); ++i) {
        if (i) out += ',';
        nl(level + 3);
        out += number(v[i]);
      }
      if (!v.empty()) nl(level + 2);
      out += ']';
    }
    if (t.block_count()) nl(level + 1);
    out += ']';
    nl(level);
    out += '}';
  }
};

// Minimal JSON reader for the tensor object (values: integers, numbers,
// arrays, nested objects are skipped if their key is unknown).
struct Reader {
  const std::string& s;
  std::size_t i = 0;
  explicit Reader(const std::string& text) : s(text) {}
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  bool eat(char c) {
    ws();
    if (i < s.size() && s[i] == c) {
      ++i;
      return true;
    }
    return false;
  }
  void need(char c) {
    if (!eat(c)) bad(std::string("expected '") + c + "'");
  }
  std::string str() {
    need('"');
    std::string k;
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\') {
        if (++i >= s.size()) bad("bad escape");
      }
      k += s[i++];
    }
    need('"');
    return k;
  }
  double num() {
    ws();
    if (s.compare(i, 4, "null") == 0) {
      i += 4;
      return std::nan("");
    }
    const char* b = s.c_str() + i;
    char* e = nullptr;
    const double v = std::strtod(b, &e);
    if (e == b) bad("expected a number");
    i += static_cast<std::size_t>(e - b);
    return v;
  }
  long long integer() {
    const double v = num();
    if (!(v == std::floor(v)) || std::fabs(v) > 1e15) bad("expected an integer");
    return static_cast<long long>(v);
  }
  void skip() {  // any value
    ws();
    if (i >= s.size()) bad("unexpected end");
    if (s[i] == '"') {
      str();
    } else if (eat('{')) {
      if (eat('}')) return;
      do {
        str();
        need(':');
        skip();
      } while (eat(','));
      need('}');
    } else if (eat('[')) {
      if (eat(']')) return;
      do skip();
      while (eat(','));
      need(']');
    } else if (s.compare(i, 4, "true") == 0 || s.compare(i, 4, "null") == 0) {
      i += 4;
    } else if (s.compare(i, 5, "false") == 0) {
      i += 5;
    } else {
      num();
    }
  }
  std::vector<std::vector<double>> blocks() {
    std::vector<std::vector<double>> out;
    need('[');
    if (eat(']')) return out;
    do {
      need('[');
      std::vector<double> blk;
      if (!eat(']')) {
        do blk.push_back(num());
        while (eat(','));
        need(']');
      }
      out.push_back(std::move(blk));
    } while (eat(','));
    need(']');
    return out;
  }
};

SymTensor parse_tensor(const std::string& text) {
  Reader rd(text);
  long long order = -1, dim = -1, bsz = -1;
  std::vector<std::vector<double>> blocks;
  bool have_blocks = false;
  rd.need('{');
  if (!rd.eat('}')) {
    do {
      const std::string k = rd.str();
      rd.need(':');
      if (k == "order")
        order = rd.integer();
      else if (k == "dim")
        dim = rd.integer();
      else if (k == "block_size")
        bsz = rd.integer();
      else if (k == "blocks") {
        blocks = rd.blocks();
        have_blocks = true;
      } else
        rd.skip();
    } while (rd.eat(','));
    rd.need('}');
  }
  rd.ws();
  if (rd.i != text.size()) bad("trailing characters");
  if (order < 1 || dim < 1 || bsz < 1 || !have_blocks) bad("missing or invalid order/dim/block_size/blocks");
  if (order > SymTensor::kMaxOrder || bsz > dim) bad("shape out of range");
  auto make = [&]() -> SymTensor {
    try {
      return SymTensor(static_cast<int>(order), static_cast<int>(dim), static_cast<int>(bsz));
    } catch (const std::exception& e) {
      bad(e.what());
    }
  };
  SymTensor t = make();
  if (blocks.size() != t.block_count()) bad("block count does not match the shape");
  for (std::size_t r = 0; r < blocks.size(); ++r) {
    auto dst = t.block_data(r);
    if (blocks[r].size() != dst.size()) bad("block volume does not match the shape");
    for (std::size_t e = 0; e < dst.size(); ++e) dst[e] = blocks[r][e];
  }
  return t;
}

}  // namespace

std::string to_json(const SymTensor& t, int indent) {
  Writer w{indent, {}};
  w.tensor(t, 0);
  return w.out;
}

SymTensor sym_tensor_from_json(const std::string& text) { return parse_tensor(text); }

SymTensor sym_tensor_from_json(std::istream& in) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return parse_tensor(text);
}

std::string to_json(const CumulantSeries& c, std::uint64_t window, int indent) {
  Writer w{indent, {}};
  w.out += '{';
  w.key("window", 1, true);
  w.out += std::to_string(window);
  w.key("rows", 1, false);
  w.out += std::to_string(c.window_len);
  w.key("tensors", 1, false);
  w.out += '[';
  for (std::size_t k = 0; k < c.tensors.size(); ++k) {
    if (k) w.out += ',';
    w.nl(2);
    w.tensor(c.tensors[k], 2);
  }
  if (!c.tensors.empty()) w.nl(1);
  w.out += ']';
  w.nl(0);
  w.out += '}';
  return w.out;
}

}  // namespace cumstream
