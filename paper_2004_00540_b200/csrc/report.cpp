// report.cpp -- RunReport JSON (reference report.hpp:64-88).
//
// Writer: fixed field order, schema_version first, the timing block last, so
// two identical runs differ only in that block.  Numbers: integers in decimal,
// doubles as the shortest text that parses back to the same value
// (std::to_chars), so serialize -> parse is an exact round trip.  Points of
// the path entries are written with a table-free integer formatter into one
// preallocated buffer (4096 targets x thousands of points is tens of MB).
// Parser: a small recursive-descent JSON reader into a value tree, then a
// strict mapping onto the record types (every field required, unknown schema
// versions rejected); malformed text raises ParseError with line and column.
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <memory>
#include <string>

#include "actmap/errors.hpp"
#include "actmap/report.hpp"

namespace actmap {

std::uint32_t LayerRule::layers_for(std::uint32_t n) const {
  if (fixed) return *fixed;
  const double l = std::ceil(ratio * n);
  return l < 1.0 ? 1u : (l > 4294967295.0 ? 4294967295u : static_cast<std::uint32_t>(l));
}

namespace {

constexpr int kSchemaVersion = 1;

// ------------------------------------------------------------------ writer
class Writer {
 public:
  std::string out;
  void raw(std::string_view s) { out.append(s); }
  void key(std::string_view k) {
    str(k);
    out.push_back(':');
    fresh_ = true;
  }
  void u(std::uint64_t v) {
    comma();
    char b[24];
    out.append(b, std::to_chars(b, b + sizeof b, v).ptr);
  }
  void i(std::int64_t v) {
    comma();
    char b[24];
    out.append(b, std::to_chars(b, b + sizeof b, v).ptr);
  }
  void d(double v) {
    comma();
    if (!std::isfinite(v)) {  // JSON has no inf / nan: written as null and read back as nan
      out.append("null");
      return;
    }
    char b[40];
    out.append(b, std::to_chars(b, b + sizeof b, v).ptr);
  }
  void b(bool v) {
    comma();
    out.append(v ? "true" : "false");
  }
  void null() {
    comma();
    out.append("null");
  }
  void str(std::string_view s) {
    comma();
    out.push_back('"');
    for (unsigned char ch : s) {
      if (ch == '"' || ch == '\\') {
        out.push_back('\\');
        out.push_back((char)ch);
      } else if (ch < 0x20) {
        char e[8];
        std::snprintf(e, sizeof e, "\\u%04x", ch);
        out.append(e);
      } else {
        out.push_back((char)ch);
      }
    }
    out.push_back('"');
  }
  void coord(Coord c) {
    comma();
    out.push_back('[');
    fresh_ = true;
    u(c.row);
    u(c.col);
    out.push_back(']');
  }
  void open(char c) {
    comma();
    out.push_back(c);
    fresh_ = true;
  }
  void close(char c) {
    out.push_back(c);
    fresh_ = false;
  }
  // points: [[r,c],...] straight into the buffer
  void points(const std::vector<Coord>& p) {
    comma();
    out.push_back('[');
    const size_t at = out.size();
    out.resize(at + p.size() * 24 + 1);
    char* o = out.data() + at;
    for (size_t k = 0; k < p.size(); ++k) {
      if (k) *o++ = ',';
      *o++ = '[';
      o = std::to_chars(o, o + 10, p[k].row).ptr;
      *o++ = ',';
      o = std::to_chars(o, o + 10, p[k].col).ptr;
      *o++ = ']';
    }
    out.resize(o - out.data());
    out.push_back(']');
  }

 private:
  bool fresh_ = true;  // next value needs no separating comma
  void comma() {
    if (!fresh_ && !out.empty() && out.back() != ':') out.push_back(',');
    fresh_ = false;
  }
};

const char* mode_name(Mode m) { return m == Mode::kBatched ? "batched" : "iterative"; }
const char* method_name(Method m) { return m == Method::kSimple ? "simple" : "euclidean"; }
const char* rule_name(CornerRule r) { return r == CornerRule::kStrict ? "strict" : "permissive"; }
const char* stop_name(AutoStop s) {
  return s == AutoStop::kFilled ? "filled" : s == AutoStop::kStalled ? "stalled" : "cap";
}

void write_bound(Writer& w, const LayerBound& b) {
  w.open('{');
  w.key("worst_case");
  w.u(b.worst_case);
  w.key("heuristic_low");
  w.u(b.heuristic_low);
  w.key("heuristic_high");
  w.u(b.heuristic_high);
  w.close('}');
}

void write_opt_coord(Writer& w, const std::optional<Coord>& c) {
  if (c) w.coord(*c);
  else w.null();
}

void write_opt_double(Writer& w, const std::optional<double>& v) {
  if (v) w.d(*v);
  else w.null();
}

void write_validation(Writer& w, const ValidationReport& v) {
  w.open('{');
  w.key("layers_used");
  w.u(v.layers_used);
  w.key("termination");
  w.str(stop_name(v.termination));
  w.key("bounds");
  write_bound(w, v.bounds);
  w.key("activity");
  w.open('{');
  w.key("violations");
  w.u(v.activity.violations);
  w.key("samples");
  w.points(v.activity.samples);
  w.close('}');
  w.key("kernels_checked");
  w.b(v.kernels_checked);
  w.key("kernels_equal");
  w.b(v.kernels_equal);
  w.key("kernel_mismatch");
  write_opt_coord(w, v.kernel_mismatch);
  w.key("targets");
  w.open('[');
  for (const TargetValidation& t : v.targets) {
    w.open('{');
    w.key("target");
    w.coord(t.target);
    w.key("covered");
    w.b(t.covered);
    w.key("simple_steps");
    w.u(t.simple_steps);
    w.key("bfs_hops");
    w.u(t.bfs_hops);
    w.key("step_optimal");
    w.b(t.step_optimal);
    w.key("nearest_ok_simple");
    w.b(t.nearest_ok_simple);
    w.key("euclidean_length");
    w.d(t.euclidean_length);
    w.key("octile_distance");
    w.d(t.octile_distance);
    w.key("euclidean_excess");
    w.d(t.euclidean_excess);
    w.key("excess_positive");
    w.b(t.excess_positive);
    w.key("octile_reachable");
    w.b(t.octile_reachable);
    w.key("nearest_ok_euclidean");
    w.b(t.nearest_ok_euclidean);
    w.close('}');
  }
  w.close(']');
  w.key("covered_targets");
  w.u(v.covered_targets);
  w.key("step_failures");
  w.u(v.step_failures);
  w.key("positive_excess_count");
  w.u(v.positive_excess_count);
  w.key("max_excess");
  w.d(v.max_excess);
  w.key("octile_unreachable_count");
  w.u(v.octile_unreachable_count);
  w.key("nearest_failures");
  w.u(v.nearest_failures);
  w.key("findings");
  w.open('[');
  for (const std::string& f : v.findings) w.str(f);
  w.close(']');
  w.key("passed");
  w.b(v.passed());
  w.close('}');
}

void write_bench(Writer& w, const BenchReport& b) {
  w.open('{');
  w.key("samples");
  w.open('[');
  for (const BenchSample& s : b.samples) {
    w.open('{');
    w.key("n");
    w.u(s.n);
    w.key("layers");
    w.u(s.layers);
    w.key("mode");
    w.str(mode_name(s.mode));
    w.key("threads");
    w.u(s.threads);
    w.key("repeats");
    w.u(s.repeats);
    w.key("median_ms");
    w.d(s.median_ms);
    w.key("min_ms");
    w.d(s.min_ms);
    w.key("skipped");
    w.b(s.skipped);
    w.close('}');
  }
  w.close(']');
  w.key("fit");
  if (b.fit) {
    w.open('{');
    w.key("slope_vs_nodes");
    write_opt_double(w, b.fit->slope_vs_nodes);
    w.key("slope_vs_layers");
    write_opt_double(w, b.fit->slope_vs_layers);
    w.key("coefficient");
    w.d(b.fit->coefficient);
    w.key("max_rel_residual");
    w.d(b.fit->max_rel_residual);
    w.close('}');
  } else {
    w.null();
  }
  w.key("mode_compare");
  if (b.mode_compare) {
    w.open('{');
    w.key("batched_median_ms");
    w.d(b.mode_compare->batched_median_ms);
    w.key("iterative_median_ms");
    w.d(b.mode_compare->iterative_median_ms);
    w.key("ratio");
    w.d(b.mode_compare->ratio);
    w.close('}');
  } else {
    w.null();
  }
  w.close('}');
}

// ------------------------------------------------------------------ parser
struct Value;
using Object = std::vector<std::pair<std::string, Value>>;
using Array = std::vector<Value>;
struct Value {
  enum Kind { kNull, kBool, kNumber, kString, kArray, kObject, kCoords } kind = kNull;
  bool boolean = false;
  std::string text;  // number token or string contents
  std::shared_ptr<Array> arr;
  std::shared_ptr<Object> obj;
  std::shared_ptr<std::vector<Coord>> pairs;  // kCoords: an array of [row, col] read in one pass
};

class Reader {
 public:
  explicit Reader(std::string_view t) : s_(t) {}
  Value document() {
    Value v = value(0);
    ws();
    if (p_ != s_.size()) fail("trailing characters after the report");
    return v;
  }
  [[noreturn]] void fail(const std::string& what) const {
    size_t line = 1, col = 1;
    for (size_t k = 0; k < p_ && k < s_.size(); ++k) {
      if (s_[k] == '\n') ++line, col = 1;
      else ++col;
    }
    throw ParseError("run report: " + what, line, col);
  }

 private:
  std::string_view s_;
  size_t p_ = 0;
  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\t' || s_[p_] == '\n' || s_[p_] == '\r')) ++p_;
  }
  bool eat(char c) {
    ws();
    if (p_ < s_.size() && s_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  bool word(std::string_view w) {
    if (s_.substr(p_, w.size()) == w) {
      p_ += w.size();
      return true;
    }
    return false;
  }
  // [[r,c],...] of unsigned 32-bit integers straight into a vector (path points: millions of pairs);
  // false (position restored) when the text has any other shape, which the generic reader then handles
  bool coord_array(Value& out) {
    const size_t start = p_;
    auto num = [&](uint32_t& x) {
      ws();
      const auto r = std::from_chars(s_.data() + p_, s_.data() + s_.size(), x);
      if (r.ec != std::errc() || r.ptr == s_.data() + p_) return false;
      p_ = r.ptr - s_.data();
      return true;
    };
    auto pairs = std::make_shared<std::vector<Coord>>();
    bool ok = eat('[');
    if (ok && !eat(']')) {
      do {
        Coord c;
        ok = eat('[') && num(c.row) && eat(',') && num(c.col) && eat(']');
        if (ok) pairs->push_back(c);
      } while (ok && eat(','));
      ok = ok && eat(']');
    }
    if (!ok) {
      p_ = start;
      return false;
    }
    out.kind = Value::kCoords;
    out.pairs = std::move(pairs);
    return true;
  }
  Value value(int depth) {
    if (depth > 64) fail("nesting too deep");
    ws();
    Value v;
    if (p_ >= s_.size()) fail("unexpected end of text");
    const char c = s_[p_];
    if (c == '{') {
      ++p_;
      v.kind = Value::kObject;
      v.obj = std::make_shared<Object>();
      if (eat('}')) return v;
      do {
        ws();
        if (p_ >= s_.size() || s_[p_] != '"') fail("expected a key");
        std::string k = string();
        expect(':');
        Value x;
        if ((k == "points" || k == "samples") && coord_array(x)) v.obj->emplace_back(std::move(k), std::move(x));
        else v.obj->emplace_back(std::move(k), value(depth + 1));
      } while (eat(','));
      expect('}');
    } else if (c == '[') {
      ++p_;
      v.kind = Value::kArray;
      v.arr = std::make_shared<Array>();
      if (eat(']')) return v;
      do v.arr->push_back(value(depth + 1));
      while (eat(','));
      expect(']');
    } else if (c == '"') {
      v.kind = Value::kString;
      v.text = string();
    } else if (word("true")) {
      v.kind = Value::kBool;
      v.boolean = true;
    } else if (word("false")) {
      v.kind = Value::kBool;
    } else if (word("null")) {
      v.kind = Value::kNull;
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      const size_t b = p_;
      ++p_;
      while (p_ < s_.size() && (std::isdigit((unsigned char)s_[p_]) || s_[p_] == '.' || s_[p_] == 'e' ||
                                s_[p_] == 'E' || s_[p_] == '+' || s_[p_] == '-'))
        ++p_;
      v.kind = Value::kNumber;
      v.text = std::string(s_.substr(b, p_ - b));
    } else {
      fail("unexpected character");
    }
    return v;
  }
  std::string string() {
    ++p_;  // opening quote
    std::string o;
    while (true) {
      if (p_ >= s_.size()) fail("unterminated string");
      const char c = s_[p_++];
      if (c == '"') break;
      if (c != '\\') {
        o.push_back(c);
        continue;
      }
      if (p_ >= s_.size()) fail("unterminated escape");
      const char e = s_[p_++];
      switch (e) {
        case '"': o.push_back('"'); break;
        case '\\': o.push_back('\\'); break;
        case '/': o.push_back('/'); break;
        case 'b': o.push_back('\b'); break;
        case 'f': o.push_back('\f'); break;
        case 'n': o.push_back('\n'); break;
        case 'r': o.push_back('\r'); break;
        case 't': o.push_back('\t'); break;
        case 'u': {
          if (p_ + 4 > s_.size()) fail("bad \\u escape");
          unsigned cp = 0;
          for (int k = 0; k < 4; ++k) {
            const char h = s_[p_++];
            cp = cp * 16 + (h >= '0' && h <= '9' ? h - '0' : h >= 'a' && h <= 'f' ? h - 'a' + 10
                            : h >= 'A' && h <= 'F' ? h - 'A' + 10 : 99);
            if (cp >= 0x10000) fail("bad \\u escape");
          }
          if (cp < 0x80) {
            o.push_back((char)cp);
          } else if (cp < 0x800) {
            o.push_back((char)(0xC0 | (cp >> 6)));
            o.push_back((char)(0x80 | (cp & 0x3F)));
          } else {
            o.push_back((char)(0xE0 | (cp >> 12)));
            o.push_back((char)(0x80 | ((cp >> 6) & 0x3F)));
            o.push_back((char)(0x80 | (cp & 0x3F)));
          }
          break;
        }
        default: fail("bad escape");
      }
    }
    return o;
  }
};

// strict mapping of the value tree onto the records
[[noreturn]] void bad(const std::string& what) { throw InvalidInputError("run report: " + what); }

const Value& field(const Value& o, const char* k) {
  if (o.kind != Value::kObject) bad(std::string("expected an object holding \"") + k + "\"");
  for (const auto& kv : *o.obj)
    if (kv.first == k) return kv.second;
  bad(std::string("missing field \"") + k + "\"");
}
const Array& arr(const Value& v, const char* what) {
  // "[]" under a "points" / "samples" key reads as an empty coordinate array: it is also an empty array
  static const Array kEmpty;
  if (v.kind == Value::kCoords && v.pairs->empty()) return kEmpty;
  if (v.kind != Value::kArray) bad(std::string(what) + " must be an array");
  return *v.arr;
}
std::uint64_t u64(const Value& v, const char* what, std::uint64_t max = ~0ull) {
  std::uint64_t x = 0;
  if (v.kind != Value::kNumber) bad(std::string(what) + " must be a number");
  const auto r = std::from_chars(v.text.data(), v.text.data() + v.text.size(), x);
  if (r.ec != std::errc() || r.ptr != v.text.data() + v.text.size() || x > max)
    bad(std::string(what) + " must be an unsigned integer in range");
  return x;
}
std::uint32_t u32(const Value& v, const char* what) { return (std::uint32_t)u64(v, what, 0xFFFFFFFFull); }
double dbl(const Value& v, const char* what) {
  if (v.kind == Value::kNull) return std::nan("");
  if (v.kind != Value::kNumber) bad(std::string(what) + " must be a number");
  double x = 0;
  const auto r = std::from_chars(v.text.data(), v.text.data() + v.text.size(), x);
  if (r.ec != std::errc() || r.ptr != v.text.data() + v.text.size()) bad(std::string(what) + " is not a number");
  return x;
}
bool boolean(const Value& v, const char* what) {
  if (v.kind != Value::kBool) bad(std::string(what) + " must be true or false");
  return v.boolean;
}
std::string str(const Value& v, const char* what) {
  if (v.kind != Value::kString) bad(std::string(what) + " must be a string");
  return v.text;
}
Coord coord(const Value& v, const char* what) {
  const Array& a = arr(v, what);
  if (a.size() != 2) bad(std::string(what) + " must be [row, col]");
  return Coord{u32(a[0], what), u32(a[1], what)};
}
std::optional<Coord> opt_coord(const Value& v, const char* what) {
  if (v.kind == Value::kNull) return std::nullopt;
  return coord(v, what);
}
std::optional<double> opt_dbl(const Value& v, const char* what) {
  if (v.kind == Value::kNull) return std::nullopt;
  return dbl(v, what);
}
std::vector<Coord> coords(const Value& v, const char* what) {
  if (v.kind == Value::kCoords) return *v.pairs;
  const Array& a = arr(v, what);
  std::vector<Coord> o;
  o.reserve(a.size());
  for (const Value& x : a) o.push_back(coord(x, what));
  return o;
}
template <class E>
E pick(const Value& v, const char* what, std::initializer_list<std::pair<const char*, E>> names) {
  const std::string s = str(v, what);
  for (const auto& [n, e] : names)
    if (s == n) return e;
  bad(std::string(what) + ": unknown value \"" + s + "\"");
}
Mode mode_of(const Value& v) { return pick<Mode>(v, "mode", {{"batched", Mode::kBatched}, {"iterative", Mode::kIterative}}); }
LayerBound bound_of(const Value& v) {
  return LayerBound{u64(field(v, "worst_case"), "worst_case"), u32(field(v, "heuristic_low"), "heuristic_low"),
                    u32(field(v, "heuristic_high"), "heuristic_high")};
}

}  // namespace

std::string serialize_run_report(const RunReport& r) {
  Writer w;
  size_t pts = 0;
  for (const TargetReport& t : r.paths) pts += t.points.size();
  w.out.reserve(1024 + r.paths.size() * 160 + pts * 14);
  w.open('{');
  w.key("schema_version");
  w.i(r.schema_version);
  w.key("command");
  w.str(r.command);
  w.key("scene");
  w.open('{');
  w.key("width");
  w.u(r.scene.width);
  w.key("height");
  w.u(r.scene.height);
  w.key("obstacles");
  w.u(r.scene.obstacles);
  w.key("sources");
  w.u(r.scene.sources);
  w.key("targets");
  w.u(r.scene.targets);
  w.close('}');
  w.key("config");
  w.open('{');
  w.key("layers");
  if (r.config.layers) w.u(*r.config.layers);
  else w.null();
  w.key("auto_cap");
  w.u(r.config.auto_cap);
  w.key("mode");
  w.str(mode_name(r.config.mode));
  w.key("method");
  w.str(method_name(r.config.method));
  w.key("seed");
  w.u(r.config.seed);
  w.key("corner_rule");
  w.str(rule_name(r.config.corner_rule));
  w.key("threads");
  w.u(r.config.threads);
  w.close('}');
  w.key("layers_used");
  w.u(r.layers_used);
  w.key("termination");
  w.str(r.termination);
  w.key("max_activity");
  w.u(r.max_activity);
  w.key("bounds");
  if (r.bounds) write_bound(w, *r.bounds);
  else w.null();
  w.key("paths");
  w.open('[');
  for (const TargetReport& t : r.paths) {
    w.open('{');
    w.key("target");
    w.coord(t.target);
    w.key("covered");
    w.b(t.covered);
    w.key("reached_source");
    write_opt_coord(w, t.reached_source);
    w.key("steps");
    w.u(t.steps);
    w.key("euclidean_length");
    w.d(t.euclidean_length);
    w.key("points");
    w.points(t.points);
    w.close('}');
  }
  w.close(']');
  w.key("validation");
  if (r.validation) write_validation(w, *r.validation);
  else w.null();
  w.key("bench");
  if (r.bench) write_bench(w, *r.bench);
  else w.null();
  w.key("timing");  // last: the only block that differs between identical runs
  w.open('{');
  w.key("parse_ms");
  w.d(r.timing.parse_ms);
  w.key("propagate_ms");
  w.d(r.timing.propagate_ms);
  w.key("reconstruct_ms");
  w.d(r.timing.reconstruct_ms);
  w.key("validate_ms");
  w.d(r.timing.validate_ms);
  w.key("total_ms");
  w.d(r.timing.total_ms);
  w.close('}');
  w.close('}');
  w.out.push_back('\n');
  return std::move(w.out);
}

RunReport parse_run_report(std::string_view text) {
  Reader rd(text);
  const Value doc = rd.document();
  RunReport r;
  const Value& ver = field(doc, "schema_version");
  if (ver.kind != Value::kNumber || ver.text != std::to_string(kSchemaVersion))
    bad("unsupported schema_version " + ver.text + " (this library reads " + std::to_string(kSchemaVersion) + ")");
  r.schema_version = kSchemaVersion;
  r.command = str(field(doc, "command"), "command");
  const Value& sc = field(doc, "scene");
  r.scene = SceneSummary{u32(field(sc, "width"), "width"), u32(field(sc, "height"), "height"),
                         u64(field(sc, "obstacles"), "obstacles"), u64(field(sc, "sources"), "sources"),
                         u64(field(sc, "targets"), "targets")};
  const Value& cf = field(doc, "config");
  const Value& lay = field(cf, "layers");
  if (lay.kind != Value::kNull) r.config.layers = u32(lay, "layers");
  r.config.auto_cap = u32(field(cf, "auto_cap"), "auto_cap");
  r.config.mode = mode_of(field(cf, "mode"));
  r.config.method =
      pick<Method>(field(cf, "method"), "method", {{"simple", Method::kSimple}, {"euclidean", Method::kEuclidean}});
  r.config.seed = u64(field(cf, "seed"), "seed");
  r.config.corner_rule = pick<CornerRule>(field(cf, "corner_rule"), "corner_rule",
                                          {{"strict", CornerRule::kStrict}, {"permissive", CornerRule::kPermissive}});
  r.config.threads = u32(field(cf, "threads"), "threads");
  r.layers_used = u32(field(doc, "layers_used"), "layers_used");
  r.termination = str(field(doc, "termination"), "termination");
  r.max_activity = u32(field(doc, "max_activity"), "max_activity");
  const Value& bd = field(doc, "bounds");
  if (bd.kind != Value::kNull) r.bounds = bound_of(bd);
  for (const Value& t : arr(field(doc, "paths"), "paths")) {
    TargetReport tr;
    tr.target = coord(field(t, "target"), "target");
    tr.covered = boolean(field(t, "covered"), "covered");
    tr.reached_source = opt_coord(field(t, "reached_source"), "reached_source");
    tr.steps = u64(field(t, "steps"), "steps");
    tr.euclidean_length = dbl(field(t, "euclidean_length"), "euclidean_length");
    tr.points = coords(field(t, "points"), "points");
    r.paths.push_back(std::move(tr));
  }
  const Value& va = field(doc, "validation");
  if (va.kind != Value::kNull) {
    ValidationReport v;
    v.layers_used = u32(field(va, "layers_used"), "layers_used");
    v.termination = pick<AutoStop>(field(va, "termination"), "termination",
                                   {{"filled", AutoStop::kFilled}, {"stalled", AutoStop::kStalled},
                                    {"cap", AutoStop::kCapReached}});
    v.bounds = bound_of(field(va, "bounds"));
    const Value& ac = field(va, "activity");
    v.activity.violations = u64(field(ac, "violations"), "violations");
    v.activity.samples = coords(field(ac, "samples"), "samples");
    v.kernels_checked = boolean(field(va, "kernels_checked"), "kernels_checked");
    v.kernels_equal = boolean(field(va, "kernels_equal"), "kernels_equal");
    v.kernel_mismatch = opt_coord(field(va, "kernel_mismatch"), "kernel_mismatch");
    for (const Value& t : arr(field(va, "targets"), "targets")) {
      TargetValidation x;
      x.target = coord(field(t, "target"), "target");
      x.covered = boolean(field(t, "covered"), "covered");
      x.simple_steps = u64(field(t, "simple_steps"), "simple_steps");
      x.bfs_hops = u32(field(t, "bfs_hops"), "bfs_hops");
      x.step_optimal = boolean(field(t, "step_optimal"), "step_optimal");
      x.nearest_ok_simple = boolean(field(t, "nearest_ok_simple"), "nearest_ok_simple");
      x.euclidean_length = dbl(field(t, "euclidean_length"), "euclidean_length");
      x.octile_distance = dbl(field(t, "octile_distance"), "octile_distance");
      x.euclidean_excess = dbl(field(t, "euclidean_excess"), "euclidean_excess");
      x.excess_positive = boolean(field(t, "excess_positive"), "excess_positive");
      x.octile_reachable = boolean(field(t, "octile_reachable"), "octile_reachable");
      x.nearest_ok_euclidean = boolean(field(t, "nearest_ok_euclidean"), "nearest_ok_euclidean");
      v.targets.push_back(x);
    }
    v.covered_targets = u64(field(va, "covered_targets"), "covered_targets");
    v.step_failures = u64(field(va, "step_failures"), "step_failures");
    v.positive_excess_count = u64(field(va, "positive_excess_count"), "positive_excess_count");
    v.max_excess = dbl(field(va, "max_excess"), "max_excess");
    v.octile_unreachable_count = u64(field(va, "octile_unreachable_count"), "octile_unreachable_count");
    v.nearest_failures = u64(field(va, "nearest_failures"), "nearest_failures");
    for (const Value& f : arr(field(va, "findings"), "findings")) v.findings.push_back(str(f, "findings"));
    (void)boolean(field(va, "passed"), "passed");  // derived (ValidationReport::passed)
    r.validation = std::move(v);
  }
  const Value& be = field(doc, "bench");
  if (be.kind != Value::kNull) {
    BenchReport b;
    for (const Value& s : arr(field(be, "samples"), "samples")) {
      BenchSample x;
      x.n = u32(field(s, "n"), "n");
      x.layers = u32(field(s, "layers"), "layers");
      x.mode = mode_of(field(s, "mode"));
      x.threads = u32(field(s, "threads"), "threads");
      x.repeats = u32(field(s, "repeats"), "repeats");
      x.median_ms = dbl(field(s, "median_ms"), "median_ms");
      x.min_ms = dbl(field(s, "min_ms"), "min_ms");
      x.skipped = boolean(field(s, "skipped"), "skipped");
      b.samples.push_back(x);
    }
    const Value& fit = field(be, "fit");
    if (fit.kind != Value::kNull)
      b.fit = ScalingFit{opt_dbl(field(fit, "slope_vs_nodes"), "slope_vs_nodes"),
                         opt_dbl(field(fit, "slope_vs_layers"), "slope_vs_layers"),
                         dbl(field(fit, "coefficient"), "coefficient"),
                         dbl(field(fit, "max_rel_residual"), "max_rel_residual")};
    const Value& mc = field(be, "mode_compare");
    if (mc.kind != Value::kNull)
      b.mode_compare = ModeComparison{dbl(field(mc, "batched_median_ms"), "batched_median_ms"),
                                      dbl(field(mc, "iterative_median_ms"), "iterative_median_ms"),
                                      dbl(field(mc, "ratio"), "ratio")};
    r.bench = std::move(b);
  }
  const Value& tm = field(doc, "timing");
  r.timing = Timings{dbl(field(tm, "parse_ms"), "parse_ms"), dbl(field(tm, "propagate_ms"), "propagate_ms"),
                     dbl(field(tm, "reconstruct_ms"), "reconstruct_ms"), dbl(field(tm, "validate_ms"), "validate_ms"),
                     dbl(field(tm, "total_ms"), "total_ms")};
  return r;
}

}  // namespace actmap
