// File formats on either side of the evaluation path, native:
//
//   SFS1 snapshots        snapshots.py:1-72   read_snapshot / write_snapshot
//   points CSV            fields.py:146-174   write_points_csv / read_points_csv
//   rectilinear fields    fields.py:67-95     write_field
//   legacy VTK            fields.py:119-143   write_vtk_rectilinear
//
// Every writer produces the reference's bytes exactly (numbers via Python's
// repr() rules, CSV rows as Python's csv module writes them) and every
// reader accepts what the reference's readers accept, with the same
// ValueError texts.  Device buffers stream through two pinned chunks so the
// file read (write) of one chunk overlaps the copy of the other; CSV parsing
// and formatting are split across host threads at line boundaries.
#include <fcntl.h>
#include <locale.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "vfn_internal.cuh"

namespace vfn {
namespace {

constexpr size_t kChunk = size_t(16) << 20;  // pinned staging chunk

int io_fail(const std::string& path, const char* what) {
  return fail(VFN_ERR_IO, path + ": " + what + ": " + std::strerror(errno));
}

// ------------------------------------------------------------ raw file I/O
struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

int read_full(int fd, int64_t off, void* dst, size_t n, const std::string& path) {
  char* p = static_cast<char*>(dst);
  while (n) {
    ssize_t r = ::pread(fd, p, n, off);
    if (r < 0) {
      if (errno == EINTR) continue;
      return io_fail(path, "read failed");
    }
    if (r == 0) return fail(VFN_ERR_IO, path + ": unexpected end of file");
    p += r;
    off += r;
    n -= (size_t)r;
  }
  return VFN_OK;
}

int write_full(int fd, const void* src, size_t n, const std::string& path) {
  const char* p = static_cast<const char*>(src);
  while (n) {
    ssize_t w = ::write(fd, p, n);
    if (w < 0) {
      if (errno == EINTR) continue;
      return io_fail(path, "write failed");
    }
    p += w;
    n -= (size_t)w;
  }
  return VFN_OK;
}

int open_write(const std::string& path, Fd& f) {
  f.fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
  return f.fd < 0 ? io_fail(path, "cannot open for writing") : VFN_OK;
}

// Two pinned chunks + their events, for streaming between a file and HBM.
struct Staging {
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  ~Staging() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (buf[i]) cudaFreeHost(buf[i]);
    }
  }
  int init(size_t bytes) {
    for (int i = 0; i < 2; ++i) {
      VFN_CUDA(cudaHostAlloc(&buf[i], std::max<size_t>(bytes, 1), cudaHostAllocDefault));
      VFN_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    return VFN_OK;
  }
};

// file [off, off + n) -> device dst: the read of chunk i+1 overlaps the H2D
// copy of chunk i.
int file_to_device(int fd, int64_t off, size_t n, void* dst, cudaStream_t s, const std::string& path) {
  Staging st;
  VFN_CHECK(st.init(std::min(n, kChunk)));
  size_t done = 0;
  for (int i = 0; done < n; ++i) {
    const int b = i & 1;
    const size_t len = std::min(kChunk, n - done);
    VFN_CUDA(cudaEventSynchronize(st.ev[b]));  // chunk i-2's copy has drained the buffer
    VFN_CHECK(read_full(fd, off + (int64_t)done, st.buf[b], len, path));
    VFN_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + done, st.buf[b], len, cudaMemcpyHostToDevice, s));
    VFN_CUDA(cudaEventRecord(st.ev[b], s));
    done += len;
  }
  VFN_CUDA(cudaStreamSynchronize(s));
  return VFN_OK;
}

// device src -> file: the D2H copy of chunk i+1 overlaps the write of chunk i.
int device_to_file(int fd, const void* src, size_t n, cudaStream_t s, const std::string& path) {
  if (n == 0) return VFN_OK;
  Staging st;
  VFN_CHECK(st.init(std::min(n, kChunk)));
  const size_t nchunks = (n + kChunk - 1) / kChunk;
  auto issue = [&](size_t i) -> int {
    const size_t off = i * kChunk, len = std::min(kChunk, n - off);
    VFN_CUDA(cudaMemcpyAsync(st.buf[i & 1], static_cast<const char*>(src) + off, len,
                             cudaMemcpyDeviceToHost, s));
    VFN_CUDA(cudaEventRecord(st.ev[i & 1], s));
    return VFN_OK;
  };
  VFN_CHECK(issue(0));
  for (size_t i = 0; i < nchunks; ++i) {
    if (i + 1 < nchunks) VFN_CHECK(issue(i + 1));
    VFN_CUDA(cudaEventSynchronize(st.ev[i & 1]));
    const size_t off = i * kChunk, len = std::min(kChunk, n - off);
    VFN_CHECK(write_full(fd, st.buf[i & 1], len, path));
  }
  return VFN_OK;
}

// pageable host -> device through pinned chunks (used for parsed tables)
int host_to_device(const void* src, size_t n, void* dst, cudaStream_t s) {
  if (n == 0) return VFN_OK;
  Staging st;
  VFN_CHECK(st.init(std::min(n, kChunk)));
  size_t done = 0;
  for (int i = 0; done < n; ++i) {
    const int b = i & 1;
    const size_t len = std::min(kChunk, n - done);
    VFN_CUDA(cudaEventSynchronize(st.ev[b]));
    std::memcpy(st.buf[b], static_cast<const char*>(src) + done, len);
    VFN_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + done, st.buf[b], len, cudaMemcpyHostToDevice, s));
    VFN_CUDA(cudaEventRecord(st.ev[b], s));
    done += len;
  }
  VFN_CUDA(cudaStreamSynchronize(s));
  return VFN_OK;
}

int pick_threads(size_t work_bytes) {
  const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
  const size_t by_size = work_bytes / (size_t(1) << 20) + 1;  // >= 1 MB per thread
  return (int)std::min<size_t>({(size_t)hc, (size_t)64, by_size});
}

template <typename F>
void parallel_for(int nt, F&& f) {
  if (nt <= 1) {
    f(0);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(nt - 1);
  for (int t = 1; t < nt; ++t) th.emplace_back(f, t);
  f(0);
  for (auto& x : th) x.join();
}

// ------------------------------------------------------- Python repr rules
// repr(float) with float_repr_style 'short': the shortest digit string that
// round-trips (std::to_chars gives the same digits as Python's dtoa mode 0),
// fixed notation when -4 < decpt <= 16, else d[.ddd]e(+|-)XX.
char* py_repr(double v, char* p) {
  if (std::isnan(v)) {
    std::memcpy(p, "nan", 3);
    return p + 3;
  }
  if (std::signbit(v)) {
    *p++ = '-';
    v = -v;
  }
  if (std::isinf(v)) {
    std::memcpy(p, "inf", 3);
    return p + 3;
  }
  if (v == 0.0) {
    std::memcpy(p, "0.0", 3);
    return p + 3;
  }
  char buf[40];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
  char dig[24];
  int nd = 0;
  const char* q = buf;
  dig[nd++] = *q++;
  if (*q == '.') {
    ++q;
    while (*q != 'e') dig[nd++] = *q++;
  }
  ++q;  // 'e'
  const bool eneg = *q == '-';
  ++q;  // sign
  int e = 0;
  while (q < r.ptr) e = 10 * e + (*q++ - '0');
  if (eneg) e = -e;
  const int decpt = e + 1;
  if (decpt <= -4 || decpt > 16) {
    *p++ = dig[0];
    if (nd > 1) {
      *p++ = '.';
      std::memcpy(p, dig + 1, nd - 1);
      p += nd - 1;
    }
    *p++ = 'e';
    *p++ = e < 0 ? '-' : '+';
    const int ae = e < 0 ? -e : e;
    if (ae < 10) *p++ = '0';
    p = std::to_chars(p, p + 8, ae).ptr;
  } else if (decpt <= 0) {
    *p++ = '0';
    *p++ = '.';
    for (int i = 0; i < -decpt; ++i) *p++ = '0';
    std::memcpy(p, dig, nd);
    p += nd;
  } else if (decpt >= nd) {
    std::memcpy(p, dig, nd);
    p += nd;
    for (int i = nd; i < decpt; ++i) *p++ = '0';
    *p++ = '.';
    *p++ = '0';
  } else {
    std::memcpy(p, dig, decpt);
    p += decpt;
    *p++ = '.';
    std::memcpy(p, dig + decpt, nd - decpt);
    p += nd - decpt;
  }
  return p;
}

// repr(bytes) for the bad-magic message (snapshots.py:57)
std::string py_bytes_repr(const unsigned char* b, int n) {
  bool has_sq = false, has_dq = false;
  for (int i = 0; i < n; ++i) {
    has_sq |= b[i] == '\'';
    has_dq |= b[i] == '"';
  }
  const char quote = (has_sq && !has_dq) ? '"' : '\'';
  std::string s = "b";
  s += quote;
  static const char* hex = "0123456789abcdef";
  for (int i = 0; i < n; ++i) {
    const unsigned char c = b[i];
    if (c == (unsigned char)quote || c == '\\') {
      s += '\\';
      s += (char)c;
    } else if (c == '\t') {
      s += "\\t";
    } else if (c == '\n') {
      s += "\\n";
    } else if (c == '\r') {
      s += "\\r";
    } else if (c < 0x20 || c >= 0x7f) {
      s += "\\x";
      s += hex[c >> 4];
      s += hex[c & 15];
    } else {
      s += (char)c;
    }
  }
  s += quote;
  return s;
}

// ------------------------------------------------------------ SFS1 layout
// struct "<4sI6d3I3Bd" (snapshots.py:31): 79 bytes, no padding.
constexpr int kHdr = 79;

void pack_header(const vfn_snapshot_info& in, unsigned char* h) {
  std::memcpy(h, "SFS1", 4);
  const uint32_t ver = 1;
  std::memcpy(h + 4, &ver, 4);
  for (int d = 0; d < 3; ++d) {  // a1 b1 a2 b2 a3 b3
    std::memcpy(h + 8 + 16 * d, &in.a[d], 8);
    std::memcpy(h + 16 + 16 * d, &in.b[d], 8);
  }
  for (int d = 0; d < 3; ++d) {
    const uint32_t n = (uint32_t)in.shape[d];
    std::memcpy(h + 56 + 4 * d, &n, 4);
  }
  for (int d = 0; d < 3; ++d) h[68 + d] = in.mirror[d] ? 1 : 0;
  std::memcpy(h + 71, &in.time, 8);
}

// read_snapshot's checks in its order (snapshots.py:50-71)
int read_info(int fd, const std::string& path, vfn_snapshot_info* info) {
  struct stat sb;
  if (::fstat(fd, &sb) != 0) return io_fail(path, "stat failed");
  const int64_t size = sb.st_size;
  if (size < kHdr) return fail(VFN_ERR_INVALID, path + ": truncated snapshot header");
  unsigned char h[kHdr];
  VFN_CHECK(read_full(fd, 0, h, kHdr, path));
  if (std::memcmp(h, "SFS1", 4) != 0)
    return fail(VFN_ERR_INVALID, path + ": not a snapshot file (bad magic " + py_bytes_repr(h, 4) + ")");
  uint32_t ver;
  std::memcpy(&ver, h + 4, 4);
  if (ver != 1) return fail(VFN_ERR_INVALID, path + ": unsupported snapshot version " + std::to_string(ver));
  uint32_t n[3];
  for (int d = 0; d < 3; ++d) {
    std::memcpy(&info->a[d], h + 8 + 16 * d, 8);
    std::memcpy(&info->b[d], h + 16 + 16 * d, 8);
    std::memcpy(&n[d], h + 56 + 4 * d, 4);
    info->shape[d] = n[d];
    info->mirror[d] = h[68 + d] != 0;
  }
  std::memcpy(&info->time, h + 71, 8);
  const unsigned __int128 count = (unsigned __int128)n[0] * n[1] * n[2];
  if ((unsigned __int128)(size - kHdr) != 16 * count)
    return fail(VFN_ERR_INVALID, path + ": payload size " + std::to_string(size - kHdr) +
                                     " does not match " + std::to_string(n[0]) + "x" +
                                     std::to_string(n[1]) + "x" + std::to_string(n[2]) +
                                     " complex values");
  return VFN_OK;
}

int open_read(const char* path, Fd& f) {
  f.fd = ::open(path, O_RDONLY | O_CLOEXEC);
  return f.fd < 0 ? io_fail(path, "cannot open") : VFN_OK;
}

// ------------------------------------------------------------ CSV reading
// Python float(): surrounding whitespace, optional sign, decimal or
// exponent form, inf / infinity / nan in any case; correctly rounded.
const char* const kWs = " \t\n\v\f\r";

bool parse_py_float(const char* b, const char* e, double* out) {
  while (b < e && std::strchr(kWs, *b) && *b) ++b;
  while (e > b && std::strchr(kWs, e[-1]) && e[-1]) --e;
  if (b == e) return false;
  bool neg = false;
  if (*b == '+' || *b == '-') {
    neg = *b == '-';
    ++b;
  }
  if (b == e || *b == '+' || *b == '-') return false;
  // from_chars would accept "nan(...)"; Python does not
  for (const char* q = b; q < e; ++q)
    if (*q == '(' || *q == ')') return false;
  // PEP 515: single underscores between digits are accepted and dropped
  std::string nodash;
  if (std::find(b, e, '_') != e) {
    for (const char* q = b; q < e; ++q) {
      if (*q != '_') continue;
      if (q == b || q + 1 == e || !std::isdigit((unsigned char)q[-1]) || !std::isdigit((unsigned char)q[1]))
        return false;
    }
    nodash.reserve(e - b);
    for (const char* q = b; q < e; ++q)
      if (*q != '_') nodash += *q;
    b = nodash.data();
    e = b + nodash.size();
  }
  double v = 0.0;
  const auto r = std::from_chars(b, e, v, std::chars_format::general);
  if (r.ptr != e) return false;
  if (r.ec == std::errc::result_out_of_range) {
    // overflow -> inf, underflow -> correctly rounded subnormal / 0 (strtod)
    static locale_t cloc = newlocale(LC_NUMERIC_MASK, "C", (locale_t)0);
    std::string tmp(b, e);
    v = strtod_l(tmp.c_str(), nullptr, cloc);
  } else if (r.ec != std::errc()) {
    return false;
  }
  *out = neg ? -v : v;
  return true;
}

// Python's csv reader (excel dialect, non-strict) on one record starting at
// p: fields into `f`, returns the position after the record's terminator.
// Handles quoted fields ("" escapes, embedded line breaks).
const char* csv_record(const char* p, const char* end, std::vector<std::string>& f) {
  f.clear();
  if (p >= end) return p;
  std::string cur;
  bool any = false;  // record has at least one field
  enum { START, UNQ, QUO, QUO_Q } st = START;
  while (p < end) {
    const char c = *p;
    if (st == QUO) {
      if (c == '"') st = QUO_Q;
      else cur += c;
      ++p;
      continue;
    }
    if (st == QUO_Q && c == '"') {  // doubled quote inside a quoted field
      cur += '"';
      st = QUO;
      ++p;
      continue;
    }
    if (c == ',') {
      f.push_back(cur);
      cur.clear();
      any = true;
      st = START;
      ++p;
      continue;
    }
    if (c == '\n' || c == '\r') {
      ++p;
      if (c == '\r' && p < end && *p == '\n') ++p;
      if (any || st != START) f.push_back(cur);
      return p;
    }
    if (st == START && c == '"') {
      st = QUO;
      ++p;
      continue;
    }
    cur += c;  // unquoted text, or text after a closing quote (non-strict)
    if (st == START || st == QUO_Q) st = UNQ;
    ++p;
  }
  if (any || st != START) f.push_back(cur);
  return p;
}

std::string py_str_repr(const std::string& s) {
  // enough of repr(str) for the conversion error message
  const char quote = (s.find('\'') != std::string::npos && s.find('"') == std::string::npos) ? '"' : '\'';
  std::string o(1, quote);
  for (char c : s) {
    if (c == quote || c == '\\') {
      o += '\\';
      o += c;
    } else if (c == '\n') {
      o += "\\n";
    } else if (c == '\r') {
      o += "\\r";
    } else if (c == '\t') {
      o += "\\t";
    } else {
      o += c;
    }
  }
  return o + quote;
}

// ------------------------------------------------------------ CSV writing
// csv.writer QUOTE_MINIMAL for a header field (fields.py:151-153)
std::string csv_quote(const std::string& s, bool only_field) {
  if (s.empty()) return only_field ? "\"\"" : "";
  if (s.find_first_of(",\"\r\n") == std::string::npos) return s;
  std::string o = "\"";
  for (char c : s) {
    if (c == '"') o += '"';
    o += c;
  }
  return o + "\"";
}

}  // namespace
}  // namespace vfn

// parsed table: column-major doubles
struct vfn_table {
  std::vector<std::string> names;
  int64_t rows = 0;
  std::vector<double> data;  // data[c * rows + r]
};

using namespace vfn;

extern "C" {

int vfn_snapshot_info_read(const char* path, vfn_snapshot_info* info) {
  if (!path || !info) return fail(VFN_ERR_INVALID, "null argument");
  Fd f;
  VFN_CHECK(open_read(path, f));
  return read_info(f.fd, path, info);
}

int vfn_snapshot_read(const char* path, vfn_snapshot_info* info, double* values, int64_t capacity,
                      int on_device, int device, void* stream) {
  if (!path || !info) return fail(VFN_ERR_INVALID, "null argument");
  Fd f;
  VFN_CHECK(open_read(path, f));
  VFN_CHECK(read_info(f.fd, path, info));
  const int64_t count = info->shape[0] * info->shape[1] * info->shape[2];
  if (count == 0) return VFN_OK;
  if (!values) return fail(VFN_ERR_INVALID, "null values buffer");
  if (capacity < count) return fail(VFN_ERR_INVALID, "values buffer too small for the snapshot payload");
  const size_t bytes = (size_t)count * 16;
  if (!on_device) return read_full(f.fd, kHdr, values, bytes, path);
  DeviceGuard guard(device);
  return file_to_device(f.fd, kHdr, bytes, values, reinterpret_cast<cudaStream_t>(stream), path);
}

int vfn_snapshot_write(const char* path, const vfn_snapshot_info* info, const double* values,
                       int on_device, int device, void* stream) {
  if (!path || !info) return fail(VFN_ERR_INVALID, "null argument");
  for (int d = 0; d < 3; ++d)
    if (info->shape[d] < 0 || info->shape[d] > 0xffffffffLL)
      return fail(VFN_ERR_INVALID, "argument out of range");  // struct.error for 'I'
  const int64_t count = info->shape[0] * info->shape[1] * info->shape[2];
  if (count && !values) return fail(VFN_ERR_INVALID, "null values buffer");
  unsigned char h[kHdr];
  pack_header(*info, h);
  Fd f;
  VFN_CHECK(open_write(path, f));
  VFN_CHECK(write_full(f.fd, h, kHdr, path));
  const size_t bytes = (size_t)count * 16;
  if (!on_device) return write_full(f.fd, values, bytes, path);
  DeviceGuard guard(device);
  return device_to_file(f.fd, values, bytes, reinterpret_cast<cudaStream_t>(stream), path);
}

int vfn_csv_read(const char* path, vfn_table** out, int64_t* rows, int* cols) {
  if (!path || !out || !rows || !cols) return fail(VFN_ERR_INVALID, "null argument");
  *out = nullptr;
  Fd f;
  VFN_CHECK(open_read(path, f));
  struct stat sb;
  if (::fstat(f.fd, &sb) != 0) return io_fail(path, "stat failed");
  std::string text((size_t)sb.st_size, '\0');
  if (sb.st_size) VFN_CHECK(read_full(f.fd, 0, text.data(), text.size(), path));
  const char* p = text.data();
  const char* end = p + text.size();
  const std::string spath = path;
  if (p == end) return fail(VFN_ERR_INVALID, spath + ": empty points file, expected a header row");

  auto t = new vfn_table();
  std::vector<std::string> hdr;
  const char* body = csv_record(p, end, hdr);
  const int nc = (int)hdr.size();
  t->names = hdr;
  auto strip = [](std::string s) {
    const size_t b = s.find_first_not_of(kWs), e = s.find_last_not_of(kWs);
    return b == std::string::npos ? std::string() : s.substr(b, e - b + 1);
  };
  for (auto& s : t->names) s = strip(s);

  const bool quoted = std::find(body, end, '"') != end;
  const std::string ragged = spath + ": ragged CSV";
  auto conv_error = [&](const std::string& field) {
    return fail(VFN_ERR_INVALID, "could not convert string to float: " + py_str_repr(field));
  };
  if (quoted) {
    // general path: sequential, any quoting
    std::vector<std::vector<double>> cols_v(nc);
    std::vector<std::string> rec;
    const char* q = body;
    int64_t r = 0;
    while (q < end) {
      q = csv_record(q, end, rec);
      if (rec.empty()) continue;
      if ((int)rec.size() != nc) {
        delete t;
        return fail(VFN_ERR_INVALID, ragged);
      }
      for (int c = 0; c < nc; ++c) {
        double v;
        if (!parse_py_float(rec[c].data(), rec[c].data() + rec[c].size(), &v)) {
          delete t;
          return conv_error(rec[c]);
        }
        cols_v[c].push_back(v);
      }
      ++r;
    }
    t->rows = r;
    t->data.resize((size_t)nc * r);
    for (int c = 0; c < nc; ++c) std::copy(cols_v[c].begin(), cols_v[c].end(), t->data.begin() + (size_t)c * r);
  } else {
    // fast path: chunks at line boundaries, count rows, then parse in place
    const size_t blen = (size_t)(end - body);
    const int nt = pick_threads(blen);
    std::vector<const char*> cut(nt + 1);
    cut[0] = body;
    cut[nt] = end;
    for (int i = 1; i < nt; ++i) {
      const char* c = std::max(cut[i - 1], body + blen * i / nt);
      const char* nl = std::find(c, end, '\n');
      cut[i] = nl == end ? end : nl + 1;
    }
    // a line: [b, e) without its terminator; empty lines are skipped
    auto for_lines = [](const char* b, const char* e, auto&& fn) {
      while (b < e) {
        const char* l = b;
        while (b < e && *b != '\n' && *b != '\r') ++b;
        const char* le = b;
        if (b < e) {
          if (*b == '\r' && b + 1 < e && b[1] == '\n') ++b;
          ++b;
        }
        if (le > l && !fn(l, le)) return false;
      }
      return true;
    };
    std::vector<int64_t> cnt(nt + 1, 0);
    parallel_for(nt, [&](int i) {
      int64_t n = 0;
      for_lines(cut[i], cut[i + 1], [&](const char*, const char*) {
        ++n;
        return true;
      });
      cnt[i + 1] = n;
    });
    for (int i = 0; i < nt; ++i) cnt[i + 1] += cnt[i];
    const int64_t R = cnt[nt];
    t->rows = R;
    if (R && nc == 0) {
      delete t;
      return fail(VFN_ERR_INVALID, ragged);
    }
    t->data.resize((size_t)nc * R);
    double* D = t->data.data();
    // per-thread first error: (row, kind, field)
    std::vector<int64_t> err_row(nt, INT64_MAX);
    std::vector<int> err_kind(nt, 0);
    std::vector<std::string> err_field(nt);
    parallel_for(nt, [&](int i) {
      int64_t r = cnt[i];
      for_lines(cut[i], cut[i + 1], [&](const char* l, const char* le) {
        int c = 0;
        const char* fb = l;
        while (true) {
          const char* fe = std::find(fb, le, ',');
          if (c >= nc) {
            err_row[i] = r, err_kind[i] = 1;
            return false;
          }
          double v;
          if (!parse_py_float(fb, fe, &v)) {
            err_row[i] = r, err_kind[i] = 2, err_field[i] = std::string(fb, fe);
            return false;
          }
          D[(size_t)c * R + r] = v;
          ++c;
          if (fe == le) break;
          fb = fe + 1;
        }
        if (c != nc) {
          err_row[i] = r, err_kind[i] = 1;
          return false;
        }
        ++r;
        return true;
      });
    });
    int worst = -1;
    for (int i = 0; i < nt; ++i)
      if (err_row[i] != INT64_MAX && (worst < 0 || err_row[i] < err_row[worst])) worst = i;
    if (worst >= 0) {
      const int kind = err_kind[worst];
      const std::string field = err_field[worst];
      delete t;
      return kind == 1 ? fail(VFN_ERR_INVALID, ragged) : conv_error(field);
    }
  }
  *rows = t->rows;
  *cols = nc;
  *out = t;
  return VFN_OK;
}

int vfn_table_name(const vfn_table* t, int col, const char** name) {
  if (!t || !name) return fail(VFN_ERR_INVALID, "null argument");
  if (col < 0 || col >= (int)t->names.size()) return fail(VFN_ERR_INVALID, "column index out of range");
  *name = t->names[col].c_str();
  return VFN_OK;
}

int vfn_table_column(const vfn_table* t, int col, double* out) {
  if (!t || (!out && t->rows)) return fail(VFN_ERR_INVALID, "null argument");
  if (col < 0 || col >= (int)t->names.size()) return fail(VFN_ERR_INVALID, "column index out of range");
  std::copy_n(t->data.data() + (size_t)col * t->rows, t->rows, out);
  return VFN_OK;
}

int vfn_table_points(const vfn_table* t, const int cols[3], double* points, int on_device, int device,
                     void* stream) {
  if (!t || !cols || (!points && t->rows)) return fail(VFN_ERR_INVALID, "null argument");
  for (int d = 0; d < 3; ++d)
    if (cols[d] < 0 || cols[d] >= (int)t->names.size()) return fail(VFN_ERR_INVALID, "column index out of range");
  const int64_t R = t->rows;
  if (R == 0) return VFN_OK;
  std::vector<double> tmp;
  double* dst = points;
  if (on_device) {
    tmp.resize((size_t)R * 3);
    dst = tmp.data();
  }
  const double* c0 = t->data.data() + (size_t)cols[0] * R;
  const double* c1 = t->data.data() + (size_t)cols[1] * R;
  const double* c2 = t->data.data() + (size_t)cols[2] * R;
  const int nt = pick_threads((size_t)R * 24);
  parallel_for(nt, [&](int i) {
    const int64_t b = R * i / nt, e = R * (i + 1) / nt;
    for (int64_t r = b; r < e; ++r) {
      dst[3 * r] = c0[r];
      dst[3 * r + 1] = c1[r];
      dst[3 * r + 2] = c2[r];
    }
  });
  if (!on_device) return VFN_OK;
  DeviceGuard guard(device);
  return host_to_device(tmp.data(), tmp.size() * sizeof(double), points, reinterpret_cast<cudaStream_t>(stream));
}

int vfn_table_destroy(vfn_table* t) {
  delete t;
  return VFN_OK;
}

int vfn_csv_write(const char* path, const double* points, int64_t M, int ncols, const char* const* names,
                  const void* const* columns, const int64_t* strides, const int* kinds) {
  if (!path || M < 0 || ncols < 0 || (M && !points)) return fail(VFN_ERR_INVALID, "null argument");
  if (ncols && (!names || !columns || !strides || !kinds)) return fail(VFN_ERR_INVALID, "null argument");
  for (int c = 0; c < ncols; ++c) {
    if (!names[c] || (M && !columns[c])) return fail(VFN_ERR_INVALID, "null column");
    if (kinds[c] < 0 || kinds[c] > 2) return fail(VFN_ERR_INVALID, "column kind must be 0 (float64), 1 (int64) or 2 (bool)");
  }
  std::string head;
  const int nf = 3 + ncols;
  const char* fixed[3] = {"x1", "x2", "x3"};
  for (int c = 0; c < nf; ++c) {
    if (c) head += ',';
    head += csv_quote(c < 3 ? fixed[c] : names[c - 3], nf == 1);
  }
  head += "\r\n";
  Fd f;
  VFN_CHECK(open_write(path, f));
  VFN_CHECK(write_full(f.fd, head.data(), head.size(), path));
  if (M == 0) return VFN_OK;
  // rows are formatted in blocks by all host threads, written in order
  const int64_t kBlock = 1 << 16;
  const int nt = pick_threads((size_t)M * nf * 24);
  std::vector<std::string> buf(nt);
  for (int64_t b0 = 0; b0 < M; b0 += kBlock * nt) {
    parallel_for(nt, [&](int i) {
      std::string& s = buf[i];
      s.clear();
      const int64_t b = std::min(M, b0 + kBlock * i), e = std::min(M, b0 + kBlock * (i + 1));
      s.resize((size_t)(e - b) * (size_t)nf * 26 + 16);
      char* p = s.data();
      for (int64_t r = b; r < e; ++r) {
        p = py_repr(points[3 * r], p);
        *p++ = ',';
        p = py_repr(points[3 * r + 1], p);
        *p++ = ',';
        p = py_repr(points[3 * r + 2], p);
        for (int c = 0; c < ncols; ++c) {
          *p++ = ',';
          if (kinds[c] == 0) {
            p = py_repr(static_cast<const double*>(columns[c])[r * strides[c]], p);
          } else if (kinds[c] == 1) {
            p = std::to_chars(p, p + 24, static_cast<const int64_t*>(columns[c])[r * strides[c]]).ptr;
          } else {
            const bool v = static_cast<const uint8_t*>(columns[c])[r * strides[c]] != 0;
            std::memcpy(p, v ? "True" : "False", v ? 4 : 5);
            p += v ? 4 : 5;
          }
        }
        *p++ = '\r';
        *p++ = '\n';
      }
      s.resize((size_t)(p - s.data()));
    });
    for (int i = 0; i < nt; ++i) VFN_CHECK(write_full(f.fd, buf[i].data(), buf[i].size(), path));
  }
  return VFN_OK;
}

int vfn_density(int device, const double* values, int64_t n, double* rho, int on_device, void* stream) {
  if (n < 0 || (n && (!values || !rho))) return fail(VFN_ERR_INVALID, "null argument");
  if (n == 0) return VFN_OK;
  if (!on_device) return fail(VFN_ERR_INVALID, "vfn_density works on device buffers");
  DeviceGuard guard(device);
  return launch_density(reinterpret_cast<const double2*>(values), n, rho, reinterpret_cast<cudaStream_t>(stream));
}

int vfn_field_write(const char* hdr_path, const char* psi_path, const char* rho_path, const char* psi_name,
                    const char* rho_name, const int64_t shape[3], const double* const coords[3],
                    const double* values, const double* density, int has_time, double time, int on_device,
                    int device, void* stream) {
  if (!hdr_path || !psi_path || !rho_path || !psi_name || !rho_name || !shape || !coords)
    return fail(VFN_ERR_INVALID, "null argument");
  for (int d = 0; d < 3; ++d)
    if (shape[d] < 0 || (shape[d] && !coords[d])) return fail(VFN_ERR_INVALID, "bad grid");
  const int64_t n = shape[0] * shape[1] * shape[2];
  if (n && (!values || !density)) return fail(VFN_ERR_INVALID, "null payload");
  // header text (fields.py:80-91)
  std::string h = "format = rectilinear-field-v1\n";
  h += "size = " + std::to_string(shape[0]) + " " + std::to_string(shape[1]) + " " + std::to_string(shape[2]) + "\n";
  h += "order = row-major third-index-fastest\n";
  h += std::string("payload_psi = ") + psi_name + "  # complex, interleaved (re, im) f64, little-endian\n";
  h += std::string("payload_rho = ") + rho_name + "  # f64, little-endian\n";
  char num[40];
  if (has_time) h += "time = " + std::string(num, py_repr(time, num)) + "\n";
  for (int d = 0; d < 3; ++d) {
    h += "coords_" + std::to_string(d + 1) + " =";
    if (shape[d] == 0) h += " ";  // " ".join([]) after "= "
    for (int64_t i = 0; i < shape[d]; ++i) {
      h += ' ';
      h.append(num, py_repr(coords[d][i], num));
    }
    h += "\n";
  }
  // fields.py:92-94: header, then psi, then rho
  {
    Fd f;
    VFN_CHECK(open_write(hdr_path, f));
    VFN_CHECK(write_full(f.fd, h.data(), h.size(), hdr_path));
  }
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  {
    Fd f;
    VFN_CHECK(open_write(psi_path, f));
    if (on_device) {
      DeviceGuard guard(device);
      VFN_CHECK(device_to_file(f.fd, values, (size_t)n * 16, s, psi_path));
    } else {
      VFN_CHECK(write_full(f.fd, values, (size_t)n * 16, psi_path));
    }
  }
  {
    Fd f;
    VFN_CHECK(open_write(rho_path, f));
    if (on_device) {
      DeviceGuard guard(device);
      VFN_CHECK(device_to_file(f.fd, density, (size_t)n * 8, s, rho_path));
    } else {
      VFN_CHECK(write_full(f.fd, density, (size_t)n * 8, rho_path));
    }
  }
  return VFN_OK;
}

int vfn_vtk_write(const char* path, const char* title, const int64_t shape[3], const double* const coords[3],
                  int nscalars, const char* const* names, const double* const* scalars, int on_device, int device,
                  void* stream) {
  if (!path || !title || !shape || !coords || nscalars < 0 || (nscalars && (!names || !scalars)))
    return fail(VFN_ERR_INVALID, "null argument");
  const int64_t n = shape[0] * shape[1] * shape[2];
  std::string h = "# vtk DataFile Version 3.0\n";
  h += std::string(title) + "\nBINARY\nDATASET RECTILINEAR_GRID\n";
  h += "DIMENSIONS " + std::to_string(shape[0]) + " " + std::to_string(shape[1]) + " " + std::to_string(shape[2]) + "\n";
  Fd f;
  VFN_CHECK(open_write(path, f));
  VFN_CHECK(write_full(f.fd, h.data(), h.size(), path));
  const char axis[3] = {'X', 'Y', 'Z'};
  for (int d = 0; d < 3; ++d) {
    std::string t = std::string(1, axis[d]) + "_COORDINATES " + std::to_string(shape[d]) + " double\n";
    std::vector<uint64_t> be((size_t)shape[d]);
    for (int64_t i = 0; i < shape[d]; ++i) {
      uint64_t u;
      std::memcpy(&u, &coords[d][i], 8);
      be[i] = __builtin_bswap64(u);
    }
    t.append(reinterpret_cast<const char*>(be.data()), be.size() * 8);
    t += "\n";
    VFN_CHECK(write_full(f.fd, t.data(), t.size(), path));
  }
  const std::string pd = "POINT_DATA " + std::to_string(n) + "\n";
  VFN_CHECK(write_full(f.fd, pd.data(), pd.size(), path));
  const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  DevBuf packed;
  std::vector<uint32_t> host;
  for (int k = 0; k < nscalars; ++k) {
    if (!names[k] || (n && !scalars[k])) return fail(VFN_ERR_INVALID, "null scalar");
    const std::string sh = std::string("SCALARS ") + names[k] + " float 1\nLOOKUP_TABLE default\n";
    VFN_CHECK(write_full(f.fd, sh.data(), sh.size(), path));
    if (n) {
      if (on_device) {
        DeviceGuard guard(device);
        VFN_CHECK(packed.ensure((size_t)n * 4));
        VFN_CHECK(launch_vtk_pack(scalars[k], shape, packed.as<uint32_t>(), s));
        VFN_CHECK(device_to_file(f.fd, packed.ptr, (size_t)n * 4, s, path));
      } else {
        // host-resident scalars: the same layout on the host threads
        host.resize((size_t)n);
        const double* in = scalars[k];
        const int64_t s0 = shape[0], s1 = shape[1], s2 = shape[2];
        const int nt = pick_threads((size_t)n * 8);
        parallel_for(nt, [&](int i) {
          const int64_t b = n * i / nt, e = n * (i + 1) / nt;
          for (int64_t o = b; o < e; ++o) {
            const int64_t x = o % s0, y = (o / s0) % s1, z = o / (s0 * s1);
            const float v = (float)in[(x * s1 + y) * s2 + z];
            uint32_t u;
            std::memcpy(&u, &v, 4);
            host[o] = __builtin_bswap32(u);
          }
        });
        VFN_CHECK(write_full(f.fd, host.data(), host.size() * 4, path));
      }
    }
    VFN_CHECK(write_full(f.fd, "\n", 1, path));
  }
  return VFN_OK;
}

}  // extern "C"
