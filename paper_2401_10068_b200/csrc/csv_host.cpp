// csv_host.cpp -- host side of the dataset file format (reference cli.py:47-56):
// cv_write_dataset_csv formats every value exactly as Python's repr(float) does, so a
// dataset written here is byte-identical to the reference's writer; rows are formatted
// by a pool of threads and written in order.  Also the host entry of the shared
// decimal parser (numparse.cuh), used by the tests to pin it against Python's float().
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cavi.h"
#include "numparse.cuh"

namespace {

// repr(float) (CPython float_repr_style 'short': the shortest round-trip digits, fixed
// notation when -4 < decpt <= 16, else d.ddde+XX with at least two exponent digits).
int py_repr(double x, char* out) {
  char* o = out;
  if (x != x) return std::sprintf(out, "nan");
  if (x == __builtin_inf()) return std::sprintf(out, "inf");
  if (x == -__builtin_inf()) return std::sprintf(out, "-inf");
  if (x == 0.0) return std::sprintf(out, std::signbit(x) ? "-0.0" : "0.0");
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
  *res.ptr = 0;
  const char* p = buf;
  if (*p == '-') {
    *o++ = '-';
    ++p;
  }
  char digits[32] = {0};
  int nd = 0;
  for (; *p && *p != 'e'; ++p)
    if (*p != '.') digits[nd++] = *p;
  const int e10 = std::atoi(p + 1);  // value = d.ddd x 10^e10
  const int decpt = e10 + 1;          // value = 0.ddd x 10^decpt
  if (decpt <= -4 || decpt > 16) {
    *o++ = digits[0];
    if (nd > 1) {
      *o++ = '.';
      std::memcpy(o, digits + 1, nd - 1);
      o += nd - 1;
    }
    o += std::sprintf(o, "e%c%02d", e10 < 0 ? '-' : '+', e10 < 0 ? -e10 : e10);
  } else if (decpt <= 0) {
    *o++ = '0';
    *o++ = '.';
    for (int k = 0; k < -decpt; ++k) *o++ = '0';
    std::memcpy(o, digits, nd);
    o += nd;
  } else if (decpt >= nd) {
    std::memcpy(o, digits, nd);
    o += nd;
    for (int k = nd; k < decpt; ++k) *o++ = '0';
    *o++ = '.';
    *o++ = '0';
  } else {
    std::memcpy(o, digits, decpt);
    o += decpt;
    *o++ = '.';
    std::memcpy(o, digits + decpt, nd - decpt);
    o += nd - decpt;
  }
  *o = 0;
  return (int)(o - out);
}

}  // namespace

namespace cavi {
int set_error(int code, const char* msg);  // cavi.cu: the message cv_last_error() returns
}

extern "C" {

int32_t cv_format_repr(double x, char* out) { return py_repr(x, out); }

int32_t cv_parse_number_host(const char* s, int64_t n, double* out) {
  if (!s || !out) return -1;
  return cavi::num::parse_double(s, s + n, out);
}

int32_t cv_write_dataset_csv(const char* path, const double* r, const double* mu, const double* D, int64_t V,
                             int32_t d, int32_t threads) {
  if (!path || !r || !mu || !D || V < 0 || d < 1) {
    return cavi::set_error(CV_ERR_ARG, "bad arguments");
  }
  FILE* fh = std::fopen(path, "wb");
  if (!fh) {
    return cavi::set_error(CV_ERR_ARG, (std::string(path) + ": " + std::strerror(errno)).c_str());
  }
  std::string head = "r";
  for (int q = 0; q <= d; ++q) head += ",d_" + std::to_string(q + 1);  // N = d + 1 networks
  head += "\n";
  std::fwrite(head.data(), 1, head.size(), fh);
  int T = threads > 0 ? threads : (int)std::thread::hardware_concurrency();
  if (T < 1) T = 1;
  const int64_t kRows = 1 << 16;  // rows per task
  std::vector<std::string> out(T);
  for (int64_t base = 0; base < V; base += kRows * T) {
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) {
      const int64_t lo = base + t * kRows;
      const int64_t hi = lo + kRows < V ? lo + kRows : V;
      out[t].clear();
      if (lo >= V) continue;
      pool.emplace_back([&, t, lo, hi] {
        std::string& s = out[t];
        s.reserve((size_t)(hi - lo) * (size_t)(24 * (d + 2)));
        char b[40];
        for (int64_t i = lo; i < hi; ++i) {
          s.append(b, py_repr(r[i], b));
          const double m = mu[i];
          for (int j = 0; j < d; ++j) {  // untransform: d_j = D_j + mu (model.py:192-197)
            s.push_back(',');
            s.append(b, py_repr(D[i * d + j] + m, b));
          }
          s.push_back(',');
          s.append(b, py_repr(m, b));
          s.push_back('\n');
        }
      });
    }
    for (auto& th : pool) th.join();
    for (int t = 0; t < T; ++t) std::fwrite(out[t].data(), 1, out[t].size(), fh);
  }
  if (std::fclose(fh) != 0) {
    return cavi::set_error(CV_ERR_ARG, (std::string(path) + ": write failed").c_str());
  }
  return CV_OK;
}

}  // extern "C"
