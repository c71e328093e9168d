// model_io.cpp — fitted-model wire format, host side:
// the reference's binary "SGMM4D01" layout (gmm_io.cpp:71-118, little-endian
// u32 M, f32 weights[M], f32 means[M*4], f32 packed covariances[M*10]) and
// its JSON mirror (gmm_io.cpp:120-177, fields "weights", "means",
// "covariances_packed" at full double precision), with the same post-load
// checks (finalize_loaded, gmm_io.cpp:43-69): non-empty, finite, positive
// weights summing to 1 within 1e-6 (then renormalised), SPD covariances.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/gmmb.h"

namespace {

thread_local std::string g_io_err;

struct IoErr {
  int code;  // 1 I/O (format / truncated), 3 numerical
  std::string msg;
};

const char kMagic[8] = {'S', 'G', 'M', 'M', '4', 'D', '0', '1'};

void put_u32(std::ostream& os, uint32_t v) {
  const char b[4] = {static_cast<char>(v & 0xff), static_cast<char>((v >> 8) & 0xff),
                     static_cast<char>((v >> 16) & 0xff), static_cast<char>((v >> 24) & 0xff)};
  os.write(b, 4);
}
void put_f32(std::ostream& os, double v) {
  const float f = static_cast<float>(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  put_u32(os, u);
}
uint32_t get_u32(std::istream& is) {
  unsigned char b[4];
  is.read(reinterpret_cast<char*>(b), 4);
  if (!is) throw IoErr{1, "model file truncated"};
  return static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8) |
         (static_cast<uint32_t>(b[2]) << 16) | (static_cast<uint32_t>(b[3]) << 24);
}
double get_f32(std::istream& is) {
  const uint32_t u = get_u32(is);
  float f;
  std::memcpy(&f, &u, 4);
  return static_cast<double>(f);
}

// kernels.cpp:10-25 cholesky4 (validation only)
bool spd4(const double* c10) {
  static const int row[10] = {0, 1, 1, 2, 2, 2, 3, 3, 3, 3};
  static const int col[10] = {0, 0, 1, 0, 1, 2, 0, 1, 2, 3};
  double a[4][4], l[4][4] = {};
  for (int q = 0; q < 10; ++q) a[row[q]][col[q]] = a[col[q]][row[q]] = c10[q];
  for (int j = 0; j < 4; ++j) {
    double d = a[j][j];
    for (int k = 0; k < j; ++k) d -= l[j][k] * l[j][k];
    if (!(d > 0.0) || !std::isfinite(d)) return false;
    l[j][j] = std::sqrt(d);
    for (int i = j + 1; i < 4; ++i) {
      double s = a[i][j];
      for (int k = 0; k < j; ++k) s -= l[i][k] * l[j][k];
      l[i][j] = s / l[j][j];
    }
  }
  return true;
}

void finalize_loaded(std::vector<double>& w, const std::vector<double>& mu,
                     const std::vector<double>& cov) {
  const size_t m = w.size();
  if (m < 1) throw IoErr{1, "model has no components"};
  bool finite = true;
  for (double v : w) finite = finite && std::isfinite(v);
  for (double v : mu) finite = finite && std::isfinite(v);
  for (double v : cov) finite = finite && std::isfinite(v);
  if (!finite) throw IoErr{3, "loaded model contains non-finite values"};
  double sum = 0.0, wmin = INFINITY;
  for (double v : w) {
    sum += v;
    wmin = std::fmin(wmin, v);
  }
  if (wmin <= 0.0) throw IoErr{3, "loaded model has non-positive weights"};
  if (std::abs(sum - 1.0) > 1e-6)
    throw IoErr{3, "loaded weights sum to " + std::to_string(sum) + ", beyond the 1e-6 tolerance"};
  for (double& v : w) v /= sum;
  for (size_t b = 0; b < m; ++b) {
    if (!spd4(&cov[b * 10]))
      throw IoErr{3, "loaded covariance of component " + std::to_string(b) +
                         " is not positive definite"};
  }
}

// ---- minimal JSON reader for the mirror format ----------------------------
struct Json {
  enum Kind { Num, Arr, Obj, Other } kind = Other;
  double num = 0.0;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;
  const Json* get(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct Parser {
  const std::string& s;
  size_t i = 0;
  explicit Parser(const std::string& t) : s(t) {}
  [[noreturn]] void fail() { throw IoErr{1, "malformed JSON"}; }
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\r' || s[i] == '\t')) ++i;
  }
  std::string str() {
    if (s[i] != '"') fail();
    std::string out;
    for (++i; i < s.size() && s[i] != '"'; ++i) {
      if (s[i] == '\\') ++i;
      if (i < s.size()) out.push_back(s[i]);
    }
    if (i >= s.size()) fail();
    ++i;
    return out;
  }
  Json value() {
    ws();
    if (i >= s.size()) fail();
    Json j;
    if (s[i] == '[') {
      j.kind = Json::Arr;
      ++i;
      ws();
      if (s[i] == ']') {
        ++i;
        return j;
      }
      while (true) {
        j.arr.push_back(value());
        ws();
        if (s[i] == ',') ++i;
        else if (s[i] == ']') { ++i; return j; }
        else fail();
      }
    }
    if (s[i] == '{') {
      j.kind = Json::Obj;
      ++i;
      ws();
      if (s[i] == '}') {
        ++i;
        return j;
      }
      while (true) {
        ws();
        std::string k = str();
        ws();
        if (s[i] != ':') fail();
        ++i;
        j.obj.emplace_back(k, value());
        ws();
        if (s[i] == ',') ++i;
        else if (s[i] == '}') { ++i; return j; }
        else fail();
      }
    }
    if (s[i] == '"') {
      str();
      return j;
    }
    char* end = nullptr;
    j.num = std::strtod(s.c_str() + i, &end);
    if (end == s.c_str() + i) fail();
    j.kind = Json::Num;
    i = static_cast<size_t>(end - s.c_str());
    return j;
  }
};

template <typename F>
int guarded_io(F&& f) {
  try {
    f();
    return 0;
  } catch (const IoErr& e) {
    g_io_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_io_err = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* gmmb_io_last_error(void) { return g_io_err.c_str(); }

int gmmb_save_model(const char* path, int m, const double* w, const double* mu,
                    const double* cov) {
  return guarded_io([&] {
    std::ofstream os(path, std::ios::binary);
    if (!os) throw IoErr{1, std::string("cannot open ") + path + " for writing"};
    os.write(kMagic, 8);
    put_u32(os, static_cast<uint32_t>(m));
    for (int b = 0; b < m; ++b) put_f32(os, w[b]);
    for (int b = 0; b < m * 4; ++b) put_f32(os, mu[b]);
    for (int b = 0; b < m * 10; ++b) put_f32(os, cov[b]);
    if (!os) throw IoErr{1, std::string("write failed for ") + path};
  });
}

int gmmb_load_model(const char* path, int capacity, double* w, double* mu, double* cov,
                    int* m_out) {
  return guarded_io([&] {
    std::ifstream is(path, std::ios::binary);
    if (!is) throw IoErr{1, std::string("cannot open ") + path};
    char magic[8];
    is.read(magic, 8);
    if (!is || std::memcmp(magic, kMagic, 8) != 0)
      throw IoErr{1, std::string("bad magic in ") + path};
    const uint32_t m = get_u32(is);
    if (m == 0) throw IoErr{1, "model declares zero components"};
    std::vector<double> vw(m), vmu(static_cast<size_t>(m) * 4), vc(static_cast<size_t>(m) * 10);
    for (auto& v : vw) v = get_f32(is);
    for (auto& v : vmu) v = get_f32(is);
    for (auto& v : vc) v = get_f32(is);
    finalize_loaded(vw, vmu, vc);
    if (m_out) *m_out = static_cast<int>(m);
    if (static_cast<int>(m) > capacity) throw IoErr{2, "output capacity smaller than the model"};
    std::memcpy(w, vw.data(), sizeof(double) * m);
    std::memcpy(mu, vmu.data(), sizeof(double) * m * 4);
    std::memcpy(cov, vc.data(), sizeof(double) * m * 10);
  });
}

int gmmb_save_model_json(const char* path, int m, const double* w, const double* mu,
                         const double* cov) {
  return guarded_io([&] {
    std::ofstream os(path);
    if (!os) throw IoErr{1, std::string("cannot open ") + path + " for writing"};
    char buf[64];
    auto num = [&](double v) {
      std::snprintf(buf, sizeof(buf), "%.17g", v);
      return std::string(buf);
    };
    os << "{\n  \"covariances_packed\": [";
    for (int b = 0; b < m; ++b) {
      os << (b ? ",\n    [" : "\n    [");
      for (int k = 0; k < 10; ++k) os << (k ? ", " : "") << num(cov[b * 10 + k]);
      os << "]";
    }
    os << "\n  ],\n  \"means\": [";
    for (int b = 0; b < m; ++b) {
      os << (b ? ",\n    [" : "\n    [");
      for (int d = 0; d < 4; ++d) os << (d ? ", " : "") << num(mu[b * 4 + d]);
      os << "]";
    }
    os << "\n  ],\n  \"weights\": [";
    for (int b = 0; b < m; ++b) os << (b ? ", " : "") << num(w[b]);
    os << "]\n}\n";
    if (!os) throw IoErr{1, std::string("write failed for ") + path};
  });
}

int gmmb_load_model_json(const char* path, int capacity, double* w, double* mu, double* cov,
                         int* m_out) {
  return guarded_io([&] {
    std::ifstream is(path);
    if (!is) throw IoErr{1, std::string("cannot open ") + path};
    std::stringstream ss;
    ss << is.rdbuf();
    const std::string text = ss.str();
    Parser p(text);
    const Json j = p.value();
    const Json* jw = j.get("weights");
    const Json* jm = j.get("means");
    const Json* jc = j.get("covariances_packed");
    if (j.kind != Json::Obj || !jw || !jm || !jc)
      throw IoErr{1, std::string("missing model fields in ") + path};
    const size_t m = jw->arr.size();
    if (m == 0 || jm->arr.size() != m || jc->arr.size() != m)
      throw IoErr{1, std::string("inconsistent field sizes in ") + path};
    std::vector<double> vw(m), vmu(m * 4), vc(m * 10);
    for (size_t b = 0; b < m; ++b) {
      if (jw->arr[b].kind != Json::Num || jm->arr[b].arr.size() != 4 ||
          jc->arr[b].arr.size() != 10)
        throw IoErr{1, std::string("bad row size in ") + path};
      vw[b] = jw->arr[b].num;
      // every element must be a number (the reference's get<double>() raises
      // GmmFormatError on anything else, gmm_io.cpp)
      for (int d = 0; d < 4; ++d) {
        if (jm->arr[b].arr[d].kind != Json::Num)
          throw IoErr{1, std::string("malformed model data in ") + path};
        vmu[b * 4 + d] = jm->arr[b].arr[d].num;
      }
      for (int k = 0; k < 10; ++k) {
        if (jc->arr[b].arr[k].kind != Json::Num)
          throw IoErr{1, std::string("malformed model data in ") + path};
        vc[b * 10 + k] = jc->arr[b].arr[k].num;
      }
    }
    finalize_loaded(vw, vmu, vc);
    if (m_out) *m_out = static_cast<int>(m);
    if (static_cast<int>(m) > capacity) throw IoErr{2, "output capacity smaller than the model"};
    std::memcpy(w, vw.data(), sizeof(double) * m);
    std::memcpy(mu, vmu.data(), sizeof(double) * m * 4);
    std::memcpy(cov, vc.data(), sizeof(double) * m * 10);
  });
}

}  // extern "C"
