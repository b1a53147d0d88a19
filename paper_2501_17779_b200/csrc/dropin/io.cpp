// Curve and result file formats (reference: proj/src/io.cpp:44-151), restated
// with a minimal JSON codec for the two schemas involved:
//   curve:   {"closed": true, "nodes": [[x, y], ...]}
//   results: flat objects of numbers / bools / one number array (gamma).
// Keys are written in lexicographic order and numbers in the shortest
// round-trip form, as nlohmann::json::dump() (the reference's writer) does;
// readers accept any JSON whitespace, key order and extra keys.
#include "curvalign/io.hpp"

#include <cctype>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <utility>

namespace curvalign {

namespace {

std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

void write_file(const std::string& path, const std::string& content) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write file: " + path);
  out << content;
}

void drop_closing_duplicate(Curve& c) {  // io.cpp:28-33
  if (c.size() >= 2 && c.nodes.front().x == c.nodes.back().x && c.nodes.front().y == c.nodes.back().y)
    c.nodes.pop_back();
}

// 17 significant digits, default float format (io.cpp:35-40: CSV cells)
std::string fmt17(double v) {
  std::ostringstream ss;
  ss.precision(17);
  ss << v;
  return ss.str();
}

// JSON number: shortest round-trip digits; integral values keep a ".0" as
// nlohmann's dump does; non-finite -> null
std::string jnum(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

// ---- minimal JSON reader (values: object, array, number, string, bool, null)
struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  double num = 0.0;
  bool b = false;
  std::string str;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;
};

struct JParser {
  std::string s;  // owned: callers pass temporaries (read_file)
  size_t i = 0;
  explicit JParser(std::string text) : s(std::move(text)) {}
  [[noreturn]] void fail(const char* what) {
    throw std::runtime_error(std::string("JSON parse error (") + what + ") at offset " + std::to_string(i));
  }
  void ws() {
    while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
  }
  bool lit(const char* w) {
    size_t k = 0;
    while (w[k] && i + k < s.size() && s[i + k] == w[k]) ++k;
    if (w[k]) return false;
    i += k;
    return true;
  }
  JVal value() {
    ws();
    if (i >= s.size()) fail("unexpected end");
    JVal v;
    const char c = s[i];
    if (c == '{') {
      v.kind = JVal::Obj;
      ++i;
      ws();
      if (i < s.size() && s[i] == '}') {
        ++i;
        return v;
      }
      for (;;) {
        ws();
        if (i >= s.size() || s[i] != '"') fail("expected key");
        const std::string k = string();
        ws();
        if (i >= s.size() || s[i] != ':') fail("expected ':'");
        ++i;
        v.obj[k] = value();
        ws();
        if (i < s.size() && s[i] == ',') {
          ++i;
          continue;
        }
        if (i < s.size() && s[i] == '}') {
          ++i;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = JVal::Arr;
      ++i;
      ws();
      if (i < s.size() && s[i] == ']') {
        ++i;
        return v;
      }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (i < s.size() && s[i] == ',') {
          ++i;
          continue;
        }
        if (i < s.size() && s[i] == ']') {
          ++i;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = JVal::Str;
      v.str = string();
      return v;
    }
    if (lit("true")) {
      v.kind = JVal::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.kind = JVal::Bool;
      return v;
    }
    if (lit("null")) return v;
    // number
    const char* p0 = s.c_str() + i;
    char* end = nullptr;
    v.num = std::strtod(p0, &end);
    if (end == p0) fail("bad value");
    i += (size_t)(end - p0);
    v.kind = JVal::Num;
    return v;
  }
  std::string string() {
    ++i;  // opening quote
    std::string out;
    while (i < s.size() && s[i] != '"') {
      if (s[i] == '\\' && i + 1 < s.size()) {
        out += s[i + 1];
        i += 2;
      } else {
        out += s[i++];
      }
    }
    if (i >= s.size()) fail("unterminated string");
    ++i;
    return out;
  }
};

}  // namespace

// strtod with std::stod's acceptance rules: leading blanks skipped, trailing
// characters ignored, no digits or overflow -> failure
bool parse_num(const std::string& t, double* v) {
  const char* p = t.c_str();
  char* end = nullptr;
  errno = 0;
  *v = std::strtod(p, &end);
  return end != p && errno != ERANGE;
}

Curve read_curve_csv(const std::string& path) {  // io.cpp:44-71
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open file: " + path);
  Curve c;
  bool header_allowed = true;  // only the first non-empty line may be a header
  for (std::string line; std::getline(in, line);) {
    if (line.empty() || line == "\r") continue;
    const std::size_t comma = line.find(',');
    // "x,y" split at the first comma; the y field is the rest of the line and must be non-empty
    if (comma == std::string::npos || comma + 1 == line.size())
      throw std::runtime_error("malformed CSV line in " + path + ": " + line);
    double x, y;
    const bool ok = parse_num(line.substr(0, comma), &x) && parse_num(line.substr(comma + 1), &y);
    const bool header = !ok && header_allowed;
    header_allowed = false;
    if (header) continue;
    if (!ok) throw std::runtime_error("malformed CSV line in " + path + ": " + line);
    c.nodes.emplace_back(x, y);
  }
  drop_closing_duplicate(c);
  validate_curve(c, 4);
  return c;
}

std::string curve_to_csv(const Curve& c) {
  std::ostringstream ss;
  ss << "x,y\n";
  for (const Point2& p : c.nodes) ss << fmt17(p.x) << "," << fmt17(p.y) << "\n";
  return ss.str();
}

void write_curve_csv(const std::string& path, const Curve& c) { write_file(path, curve_to_csv(c)); }

Curve read_curve_json(const std::string& path) {  // io.cpp:83-96
  JParser jp(read_file(path));
  const JVal j = jp.value();
  const auto it = j.kind == JVal::Obj ? j.obj.find("nodes") : j.obj.end();
  if (it == j.obj.end() || it->second.kind != JVal::Arr)
    throw std::runtime_error("curve JSON must contain a \"nodes\" array: " + path);
  Curve c;
  for (const JVal& e : it->second.arr) {
    if (e.kind != JVal::Arr || e.arr.size() != 2 || e.arr[0].kind != JVal::Num || e.arr[1].kind != JVal::Num)
      throw std::runtime_error("curve JSON nodes must be [x, y] pairs: " + path);
    c.nodes.emplace_back(e.arr[0].num, e.arr[1].num);
  }
  drop_closing_duplicate(c);
  validate_curve(c, 4);
  return c;
}

std::string curve_to_json(const Curve& c) {
  std::string s = "{\"closed\":true,\"nodes\":[";
  for (std::size_t i = 0; i < c.size(); ++i) {
    if (i) s += ",";
    s += "[" + jnum(c.nodes[i].x) + "," + jnum(c.nodes[i].y) + "]";
  }
  return s + "]}";
}

void write_curve_json(const std::string& path, const Curve& c) { write_file(path, curve_to_json(c)); }

Curve load_curve(const std::string& path) {  // io.cpp:107-111
  const auto dot = path.find_last_of('.');
  const std::string ext = dot == std::string::npos ? "" : path.substr(dot + 1);
  return ext == "json" ? read_curve_json(path) : read_curve_csv(path);
}

std::string alignment_to_json(const RigidAlignment& a) {  // io.cpp:113-120
  return "{\"energy\":" + jnum(a.energy) + ",\"shift\":" + std::to_string(a.shift) + ",\"t0\":" + jnum(a.t0) +
         ",\"theta\":" + jnum(a.rotation.theta()) + ",\"trace\":" + jnum(a.trace) + "}";
}

std::string elastic_to_json(const ElasticMatch& m) {  // io.cpp:122-131
  std::string g = "[";
  for (std::size_t i = 0; i < m.gamma.gamma.size(); ++i) g += (i ? "," : "") + jnum(m.gamma.gamma[i]);
  g += "]";
  return std::string("{\"converged\":") + (m.converged ? "true" : "false") + ",\"distance\":" + jnum(m.distance) +
         ",\"gamma\":" + g + ",\"iterations\":" + std::to_string(m.iterations) + ",\"t0\":" + jnum(m.t0) +
         ",\"theta\":" + jnum(m.rotation.theta()) + "}";
}

std::string matrix_to_csv(const std::vector<std::string>& names, const std::vector<std::vector<double>>& d) {
  if (names.size() != d.size()) throw std::invalid_argument("matrix_to_csv: name count mismatch");
  std::ostringstream ss;
  ss << "id";
  for (const std::string& n : names) ss << "," << n;
  ss << "\n";
  for (std::size_t i = 0; i < d.size(); ++i) {
    if (d[i].size() != names.size()) throw std::invalid_argument("matrix_to_csv: ragged matrix");
    ss << names[i];
    for (double v : d[i]) ss << "," << (std::isnan(v) ? std::string("nan") : fmt17(v));
    ss << "\n";
  }
  return ss.str();
}

}  // namespace curvalign
