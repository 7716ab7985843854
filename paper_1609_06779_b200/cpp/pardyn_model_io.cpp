// Model validation and JSON model files of the pardyn drop-in API
// (SURVEY.md §8f row 4). Host-side only.
//
//   validate_chain   proj/core/src/model.cpp:75-115 (ModelError messages)
//   load_chain       proj/core/src/model.cpp:254-310 (field checks, messages)
//   save_chain       proj/core/src/model.cpp:312-337 (2-space indented, the
//                    reference's field order; every double printed with the
//                    shortest digits that parse back to the same value, so a
//                    save/load round trip reproduces the chain exactly)
//
// The reference uses nlohmann::ordered_json; this file carries a small
// recursive-descent JSON reader (objects, arrays, numbers, strings, literals)
// sufficient for the model format.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/pardyn/pardyn.hpp"
#include "records.hpp"

namespace pardyn {

namespace {

std::string link_prefix(int k) { return "link " + std::to_string(k); }

bool finite3(const Vec3& v) { return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]); }

}  // namespace

// Smallest eigenvalue of a symmetric 3x3 (cyclic Jacobi), the
// SelfAdjointEigenSolver minCoeff of model.cpp:96 and spatial.cpp:83.
double detail::sym3_min_eig(const Mat3& a) {
  double m[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) m[r][c] = 0.5 * (a(r, c) + a(c, r));
  for (int sweep = 0; sweep < 64; ++sweep) {
    const double off = m[0][1] * m[0][1] + m[0][2] * m[0][2] + m[1][2] * m[1][2];
    if (off < 1e-300) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (m[p][q] == 0.0) continue;
        const double th = (m[q][q] - m[p][p]) / (2.0 * m[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {
          const double x = m[k][p], y = m[k][q];
          m[k][p] = c * x - s * y;
          m[k][q] = s * x + c * y;
        }
        for (int k = 0; k < 3; ++k) {
          const double x = m[p][k], y = m[q][k];
          m[p][k] = c * x - s * y;
          m[q][k] = s * x + c * y;
        }
      }
  }
  return std::min(m[0][0], std::min(m[1][1], m[2][2]));
}

// SE3Transform::is_valid (spatial.cpp:36-41)
bool SE3Transform::is_valid(double tol) const {
  if (!rotation.allFinite() || !translation.allFinite()) return false;
  const Mat3 gram = rotation.transpose() * rotation;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      if (std::fabs(gram(r, c) - (r == c ? 1.0 : 0.0)) > tol) return false;
  const Mat3& R = rotation;
  const double det = R(0, 0) * (R(1, 1) * R(2, 2) - R(1, 2) * R(2, 1)) -
                     R(0, 1) * (R(1, 0) * R(2, 2) - R(1, 2) * R(2, 0)) +
                     R(0, 2) * (R(1, 0) * R(2, 1) - R(1, 1) * R(2, 0));
  return det > 0.0;
}

namespace {

// ---------------------------------------------------------------- JSON reader
struct Json {
  enum Kind { kNull, kBool, kNumber, kString, kArray, kObject } kind = kNull;
  bool b = false;
  double num = 0.0;
  bool integer = false;  // number token without fraction / exponent
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;
  const Json* find(const char* key) const {
    for (const auto& kv : obj)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
};

class Reader {
 public:
  explicit Reader(const std::string& s) : s_(s) {}
  Json document() {
    Json v = value();
    ws();
    if (i_ != s_.size()) fail("unexpected trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& what) const {
    std::size_t line = 1, col = 1;
    for (std::size_t k = 0; k < i_ && k < s_.size(); ++k) {
      if (s_[k] == '\n') {
        ++line;
        col = 1;
      } else {
        ++col;
      }
    }
    throw std::runtime_error("parse error at line " + std::to_string(line) + ", column " + std::to_string(col) +
                             ": " + what);
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r')) ++i_;
  }
  bool lit(const char* w) {
    const std::size_t n = std::char_traits<char>::length(w);
    if (s_.compare(i_, n, w) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }
  Json value() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end of input");
    const char c = s_[i_];
    Json v;
    if (c == '{') {
      v.kind = Json::kObject;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == '}') {
        ++i_;
        return v;
      }
      for (;;) {
        ws();
        if (i_ >= s_.size() || s_[i_] != '"') fail("expected a string key");
        std::string key = string();
        ws();
        if (i_ >= s_.size() || s_[i_] != ':') fail("expected ':'");
        ++i_;
        v.obj.emplace_back(std::move(key), value());
        ws();
        if (i_ < s_.size() && s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < s_.size() && s_[i_] == '}') {
          ++i_;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.kind = Json::kArray;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == ']') {
        ++i_;
        return v;
      }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (i_ < s_.size() && s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (i_ < s_.size() && s_[i_] == ']') {
          ++i_;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.kind = Json::kString;
      v.str = string();
      return v;
    }
    if (lit("true")) {
      v.kind = Json::kBool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.kind = Json::kBool;
      return v;
    }
    if (lit("null")) return v;
    if (c == '-' || (c >= '0' && c <= '9')) {
      const std::size_t start = i_;
      bool integer = true;
      if (s_[i_] == '-') ++i_;
      while (i_ < s_.size() && ((s_[i_] >= '0' && s_[i_] <= '9') || s_[i_] == '.' || s_[i_] == 'e' ||
                                s_[i_] == 'E' || s_[i_] == '+' || s_[i_] == '-')) {
        if (s_[i_] == '.' || s_[i_] == 'e' || s_[i_] == 'E') integer = false;
        ++i_;
      }
      const std::string tok = s_.substr(start, i_ - start);
      char* end = nullptr;
      v.num = std::strtod(tok.c_str(), &end);
      if (end != tok.c_str() + tok.size()) fail("invalid number '" + tok + "'");
      v.kind = Json::kNumber;
      v.integer = integer;
      return v;
    }
    fail(std::string("unexpected character '") + c + "'");
  }
  std::string string() {
    ++i_;  // opening quote
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      if (s_[i_] == '\\' && i_ + 1 < s_.size()) {
        const char e = s_[i_ + 1];
        out.push_back(e == 'n' ? '\n' : e == 't' ? '\t' : e);
        i_ += 2;
      } else {
        out.push_back(s_[i_++]);
      }
    }
    if (i_ >= s_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  const std::string& s_;
  std::size_t i_ = 0;
};

const Json& need(const Json& j, const char* field, const std::string& where) {
  const Json* v = j.kind == Json::kObject ? j.find(field) : nullptr;
  if (!v) throw ModelError(where + ": missing field '" + field + "'");
  return *v;
}

double need_number(const Json& j, const char* field, const std::string& where) {
  const Json& v = need(j, field, where);
  if (v.kind != Json::kNumber) throw ModelError(where + ": field '" + field + "' must be a number");
  return v.num;
}

std::vector<double> need_array(const Json& j, const char* field, std::size_t len, const std::string& where) {
  const Json& v = need(j, field, where);
  if (v.kind != Json::kArray || v.arr.size() != len)
    throw ModelError(where + ": field '" + field + "' must be an array of " + std::to_string(len) + " numbers");
  std::vector<double> out;
  for (const Json& e : v.arr) {
    if (e.kind != Json::kNumber) throw ModelError(where + ": field '" + field + "' must contain only numbers");
    out.push_back(e.num);
  }
  return out;
}

// Shortest decimal that parses back to exactly v (JSON number syntax).
std::string num(double v) {
  char buf[40];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof buf, "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s = buf;
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";  // keep it a float token, like nlohmann
  return s;
}

void put_array(std::ostream& o, const double* v, int k, const std::string& ind) {
  o << "[\n";
  for (int i = 0; i < k; ++i) o << ind << "  " << num(v[i]) << (i + 1 < k ? ",\n" : "\n");
  o << ind << "]";
}

}  // namespace

void validate_chain(const RobotChain& chain) {
  if (chain.links.empty()) throw ModelError("chain must have at least one link");
  if (!finite3(chain.gravity)) throw ModelError("gravity must be finite");
  for (int k = 0; k < chain.size(); ++k) {
    const LinkSpec& link = chain.links[k];
    if (!(link.mass > 0.0) || !std::isfinite(link.mass)) throw ModelError(link_prefix(k) + ": mass must be positive");
    if (!finite3(link.com)) throw ModelError(link_prefix(k) + ": com must be finite");
    bool fin = true;
    double asym = 0.0, scale = 0.0;
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        fin = fin && std::isfinite(link.inertia_rot(r, c));
        asym = std::max(asym, std::fabs(link.inertia_rot(r, c) - link.inertia_rot(c, r)));
        scale = std::max(scale, std::fabs(link.inertia_rot(r, c)));
      }
    if (!fin || asym > 1e-9 * std::max(1.0, scale))
      throw ModelError(link_prefix(k) + ": rotational inertia must be symmetric");
    if (!(detail::sym3_min_eig(link.inertia_rot) > 0.0))
      throw ModelError(link_prefix(k) + ": rotational inertia must be positive definite");
    bool sfin = true;
    double norm = 0.0;
    for (double v : link.joint_screw.stacked()) {
      sfin = sfin && std::isfinite(v);
      norm += v * v;
    }
    if (!sfin) throw ModelError(link_prefix(k) + ": joint_screw must be finite");
    norm = std::sqrt(norm);
    if (std::fabs(norm - 1.0) > 1e-9)
      throw ModelError(link_prefix(k) + ": joint_screw must have unit norm (got " + std::to_string(norm) + ")");
    if (!link.home_transform.is_valid(1e-9))
      throw ModelError(link_prefix(k) + ": home_transform rotation must be orthonormal with determinant +1");
  }
}

RobotChain load_chain(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ModelError("cannot open model file '" + path + "'");
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string text = ss.str();
  Json doc;
  try {
    doc = Reader(text).document();
  } catch (const std::runtime_error& e) {
    throw ModelError("model file '" + path + "': " + e.what());
  }
  const std::string where = "model file '" + path + "'";
  const Json& n_field = need(doc, "n", where);
  if (n_field.kind != Json::kNumber || !n_field.integer) throw ModelError(where + ": field 'n' must be an integer");
  const int n = static_cast<int>(n_field.num);
  RobotChain chain;
  const std::vector<double> g = need_array(doc, "gravity", 3, where);
  chain.gravity = Vec3(g[0], g[1], g[2]);
  const Json& links = need(doc, "links", where);
  if (links.kind != Json::kArray) throw ModelError(where + ": field 'links' must be an array");
  if (static_cast<int>(links.arr.size()) != n)
    throw ModelError(where + ": field 'n' (= " + std::to_string(n) + ") does not match the length of 'links' (= " +
                     std::to_string(links.arr.size()) + ")");
  chain.links.resize(links.arr.size());
  for (std::size_t k = 0; k < links.arr.size(); ++k) {
    const Json& j = links.arr[k];
    const std::string lw = link_prefix(static_cast<int>(k));
    if (j.kind != Json::kObject) throw ModelError(lw + ": must be an object");
    LinkSpec& l = chain.links[k];
    l.mass = need_number(j, "mass", lw);
    const std::vector<double> com = need_array(j, "com", 3, lw);
    const std::vector<double> ir = need_array(j, "inertia_rot", 9, lw);
    const std::vector<double> sc = need_array(j, "joint_screw", 6, lw);
    l.com = Vec3(com[0], com[1], com[2]);
    l.inertia_rot = Mat3::FromRowMajor(ir.data());
    l.joint_screw = Twist(Vec3(sc[0], sc[1], sc[2]), Vec3(sc[3], sc[4], sc[5]));
    const Json& home = need(j, "home_transform", lw);
    if (home.kind != Json::kObject) throw ModelError(lw + ": field 'home_transform' must be an object");
    const std::vector<double> hr = need_array(home, "rotation", 9, lw);
    const std::vector<double> ht = need_array(home, "translation", 3, lw);
    l.home_transform.rotation = Mat3::FromRowMajor(hr.data());
    l.home_transform.translation = Vec3(ht[0], ht[1], ht[2]);
  }
  validate_chain(chain);
  return chain;
}

void save_chain(const RobotChain& chain, const std::string& path) {
  std::ostringstream o;
  o << "{\n  \"n\": " << chain.size() << ",\n  \"gravity\": ";
  put_array(o, chain.gravity.data(), 3, "  ");
  o << ",\n  \"links\": [";
  for (std::size_t k = 0; k < chain.links.size(); ++k) {
    const LinkSpec& l = chain.links[k];
    const std::string ind = "      ";
    o << (k ? ",\n" : "\n") << "    {\n" << ind << "\"mass\": " << num(l.mass) << ",\n" << ind << "\"com\": ";
    double rec[PD_LINK_FIELDS];
    detail::to_record(l, rec);  // row-major fields, the file's order
    put_array(o, rec + 1, 3, ind);
    o << ",\n" << ind << "\"inertia_rot\": ";
    put_array(o, rec + 4, 9, ind);
    o << ",\n" << ind << "\"joint_screw\": ";
    put_array(o, rec + 13, 6, ind);
    o << ",\n" << ind << "\"home_transform\": {\n" << ind << "  \"rotation\": ";
    put_array(o, rec + 19, 9, ind + "  ");
    o << ",\n" << ind << "  \"translation\": ";
    put_array(o, rec + 28, 3, ind + "  ");
    o << "\n" << ind << "}\n    }";
  }
  o << (chain.links.empty() ? "]\n}\n" : "\n  ]\n}\n");
  std::ofstream out(path);
  if (!out) throw ModelError("cannot open model file '" + path + "' for writing");
  out << o.str();
  if (!out) throw ModelError("failed writing model file '" + path + "'");
}

}  // namespace pardyn
