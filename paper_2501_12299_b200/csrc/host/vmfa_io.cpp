// vmfa_io.cpp — the reference's on-disk containers,
// host-only part of libvmfa_b200.so:
//   * MFAD dataset    io.hpp:12-16, io.cpp:91-125
//   * MFAM checkpoint io.hpp:18-23, io.cpp:127-179 (Lambda stored row-major
//     D x H per component, io.cpp:139-144)
//   * MFAK variational-state sidecar (this project): K, g and g_count, so a
//     run resumes exactly where a checkpoint left it.
// All little-endian (the byte-order helpers swap on big-endian hosts, like
// io.cpp:24-63). Dataset and state loads take a row range, so every rank of a
// multi-GPU job reads only its own shard.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../vmfa_internal.hpp"
#include "vmfa_b200.h"

namespace {

constexpr uint32_t kDatasetVersion = 1;     // io.cpp:21
constexpr uint32_t kCheckpointVersion = 1;  // io.cpp:22
constexpr uint32_t kStateVersion = 1;
constexpr int64_t kDatasetHeader = 4 + 4 + 8 + 4 + 1 + 7;  // magic, version, N, D, dtype, reserved
constexpr int64_t kStateHeader = 4 + 4 + 8 + 4 + 4 + 4;    // magic, version, N, C', C, G

bool host_little() {
  const uint16_t one = 1;
  unsigned char b;
  std::memcpy(&b, &one, 1);
  return b == 1;
}

struct File {
  FILE* f = nullptr;
  std::string path;
  ~File() {
    if (f) std::fclose(f);
  }
};

int open_file(File& fh, const char* path, const char* mode) {
  if (!path) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "null path");
  fh.path = path;
  fh.f = std::fopen(path, mode);
  if (!fh.f) return vmfa_b200::fail(VMFA_ERR_IO, "cannot open %s", path);
  return VMFA_OK;
}

// raw little-endian element arrays
template <class T>
int write_arr(File& fh, const T* v, size_t n) {
  if (host_little()) {
    if (n && std::fwrite(v, sizeof(T), n, fh.f) != n)
      return vmfa_b200::fail(VMFA_ERR_IO, "write failed for %s", fh.path.c_str());
    return VMFA_OK;
  }
  for (size_t i = 0; i < n; ++i) {
    unsigned char b[sizeof(T)];
    std::memcpy(b, v + i, sizeof(T));
    for (size_t k = 0; k < sizeof(T) / 2; ++k) std::swap(b[k], b[sizeof(T) - 1 - k]);
    if (std::fwrite(b, 1, sizeof(T), fh.f) != sizeof(T))
      return vmfa_b200::fail(VMFA_ERR_IO, "write failed for %s", fh.path.c_str());
  }
  return VMFA_OK;
}
template <class T>
int read_arr(File& fh, T* v, size_t n, const char* what) {
  if (n && std::fread(v, sizeof(T), n, fh.f) != n)
    return vmfa_b200::fail(VMFA_ERR_TRUNCATED_FILE, "%s: unexpected end of file (%s)", fh.path.c_str(), what);
  if (!host_little())
    for (size_t i = 0; i < n; ++i) {
      unsigned char b[sizeof(T)];
      std::memcpy(b, v + i, sizeof(T));
      for (size_t k = 0; k < sizeof(T) / 2; ++k) std::swap(b[k], b[sizeof(T) - 1 - k]);
      std::memcpy(v + i, b, sizeof(T));
    }
  return VMFA_OK;
}
template <class T>
int write_le(File& fh, T v) {
  return write_arr(fh, &v, 1);
}
template <class T>
int read_le(File& fh, T* v, const char* what) {
  return read_arr(fh, v, 1, what);
}

int expect_magic(File& fh, const char* magic) {  // io.cpp:65-72
  char buf[4];
  if (std::fread(buf, 1, 4, fh.f) != 4)
    return vmfa_b200::fail(VMFA_ERR_TRUNCATED_FILE, "%s: file shorter than its magic", fh.path.c_str());
  if (std::memcmp(buf, magic, 4) != 0)
    return vmfa_b200::fail(VMFA_ERR_BAD_MAGIC, "%s: expected magic %s", fh.path.c_str(), magic);
  return VMFA_OK;
}

int seek(File& fh, int64_t off) {
  if (std::fseek(fh.f, static_cast<long>(off), SEEK_SET) != 0)
    return vmfa_b200::fail(VMFA_ERR_TRUNCATED_FILE, "%s: seek past the end", fh.path.c_str());
  return VMFA_OK;
}

#define IO_TRY(expr)               \
  do {                             \
    const int r_ = (expr);         \
    if (r_ != VMFA_OK) return r_;  \
  } while (0)

int dataset_header(File& fh, int64_t* N, int* D) {  // io.cpp:106-120
  IO_TRY(expect_magic(fh, "MFAD"));
  uint32_t version = 0, d = 0;
  uint64_t n = 0;
  uint8_t dtype = 0;
  IO_TRY(read_le(fh, &version, "version"));
  if (version != kDatasetVersion)
    return vmfa_b200::fail(VMFA_ERR_UNSUPPORTED_VERSION, "dataset version %u", version);
  IO_TRY(read_le(fh, &n, "N"));
  IO_TRY(read_le(fh, &d, "D"));
  IO_TRY(read_le(fh, &dtype, "dtype"));
  if (dtype != 0) return vmfa_b200::fail(VMFA_ERR_UNSUPPORTED_VERSION, "dataset dtype %u", dtype);
  char reserved[7];
  if (std::fread(reserved, 1, 7, fh.f) != 7)
    return vmfa_b200::fail(VMFA_ERR_TRUNCATED_FILE, "%s: dataset header truncated", fh.path.c_str());
  if (n < 1 || d < 1) return vmfa_b200::fail(VMFA_ERR_IO, "%s: dataset header declares empty data", fh.path.c_str());
  *N = static_cast<int64_t>(n);
  *D = static_cast<int>(d);
  return VMFA_OK;
}

int checkpoint_header(File& fh, int* C, int* D, int* H) {  // io.cpp:155-167
  IO_TRY(expect_magic(fh, "MFAM"));
  uint32_t version = 0, c = 0, d = 0, h = 0;
  IO_TRY(read_le(fh, &version, "version"));
  if (version != kCheckpointVersion)
    return vmfa_b200::fail(VMFA_ERR_UNSUPPORTED_VERSION, "checkpoint version %u", version);
  IO_TRY(read_le(fh, &c, "C"));
  IO_TRY(read_le(fh, &d, "D"));
  IO_TRY(read_le(fh, &h, "H"));
  const int ci = static_cast<int>(c), di = static_cast<int>(d), hi = static_cast<int>(h);
  if (ci < 1 || di < 1 || hi < 1 || hi > di)
    return vmfa_b200::fail(VMFA_ERR_IO, "%s: checkpoint header declares invalid sizes", fh.path.c_str());
  *C = ci, *D = di, *H = hi;
  return VMFA_OK;
}

int state_header(File& fh, int64_t* N, int* Cp, int* C, int* G) {
  IO_TRY(expect_magic(fh, "MFAK"));
  uint32_t version = 0, cp = 0, c = 0, g = 0;
  uint64_t n = 0;
  IO_TRY(read_le(fh, &version, "version"));
  if (version != kStateVersion) return vmfa_b200::fail(VMFA_ERR_UNSUPPORTED_VERSION, "state version %u", version);
  IO_TRY(read_le(fh, &n, "N"));
  IO_TRY(read_le(fh, &cp, "C'"));
  IO_TRY(read_le(fh, &c, "C"));
  IO_TRY(read_le(fh, &g, "G"));
  if (n < 1 || cp < 1 || c < 1 || g < 1 || cp > c || g > c)
    return vmfa_b200::fail(VMFA_ERR_IO, "%s: state header declares invalid sizes", fh.path.c_str());
  *N = static_cast<int64_t>(n), *Cp = static_cast<int>(cp), *C = static_cast<int>(c), *G = static_cast<int>(g);
  return VMFA_OK;
}

}  // namespace

extern "C" {

int vmfa_save_dataset(const char* path, const float* X, int64_t N, int D) {
  if (!X || N < 1 || D < 1) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_save_dataset: empty data");
  File fh;
  IO_TRY(open_file(fh, path, "wb"));
  if (std::fwrite("MFAD", 1, 4, fh.f) != 4) return vmfa_b200::fail(VMFA_ERR_IO, "write failed for %s", path);
  IO_TRY(write_le<uint32_t>(fh, kDatasetVersion));
  IO_TRY(write_le<uint64_t>(fh, static_cast<uint64_t>(N)));
  IO_TRY(write_le<uint32_t>(fh, static_cast<uint32_t>(D)));
  IO_TRY(write_le<uint8_t>(fh, 0));  // dtype 0 = 32-bit float
  const char reserved[7] = {};
  if (std::fwrite(reserved, 1, 7, fh.f) != 7) return vmfa_b200::fail(VMFA_ERR_IO, "write failed for %s", path);
  IO_TRY(write_arr(fh, X, static_cast<size_t>(N) * D));
  if (std::fflush(fh.f) != 0) return vmfa_b200::fail(VMFA_ERR_IO, "write failed for %s", path);
  return VMFA_OK;
}

int vmfa_dataset_info(const char* path, int64_t* N, int* D) {
  if (!N || !D) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "null output");
  File fh;
  IO_TRY(open_file(fh, path, "rb"));
  return dataset_header(fh, N, D);
}

int vmfa_load_dataset(const char* path, int64_t row_begin, int64_t rows, int D, float* X) {
  File fh;
  IO_TRY(open_file(fh, path, "rb"));
  int64_t n = 0;
  int d = 0;
  IO_TRY(dataset_header(fh, &n, &d));
  if (d != D || row_begin < 0 || rows < 0 || row_begin + rows > n || (!X && rows > 0))
    return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_load_dataset: rows [%lld, %lld) / D %d outside the file's %lld x %d",
                           static_cast<long long>(row_begin), static_cast<long long>(row_begin + rows), D,
                           static_cast<long long>(n), d);
  IO_TRY(seek(fh, kDatasetHeader + row_begin * static_cast<int64_t>(D) * 4));
  return read_arr(fh, X, static_cast<size_t>(rows) * D, "rows");
}

// MfaParams::validate (model.cpp:14-41) before writing (io.cpp:129)
int vmfa_save_checkpoint(const char* path, int C, int D, int H, const double* pi, const double* mu,
                         const double* lambda, const double* dnoise) {
  if (C < 1 || D < 1 || H < 1 || H > D) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "invalid model sizes C/D/H");
  if (!pi || !mu || !lambda || !dnoise) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "null parameter array");
  const size_t CD = static_cast<size_t>(C) * D;
  for (size_t i = 0; i < CD * H; ++i)
    if (!std::isfinite(lambda[i])) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "non-finite loadings");
  double psum = 0.0;
  for (int c = 0; c < C; ++c) {
    if (!std::isfinite(pi[c])) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "non-finite parameters");
    if (pi[c] < 0.0) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "negative mixing proportion");
    psum += pi[c];
  }
  for (size_t i = 0; i < CD; ++i) {
    if (!std::isfinite(mu[i]) || !std::isfinite(dnoise[i]))
      return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "non-finite parameters");
    if (dnoise[i] <= 0.0) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "noise variance at or below zero");
  }
  if (std::abs(psum - 1.0) > 1e-12) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "mixing proportions do not sum to 1");
  File fh;
  IO_TRY(open_file(fh, path, "wb"));
  if (std::fwrite("MFAM", 1, 4, fh.f) != 4) return vmfa_b200::fail(VMFA_ERR_IO, "write failed for %s", path);
  IO_TRY(write_le<uint32_t>(fh, kCheckpointVersion));
  IO_TRY(write_le<uint32_t>(fh, static_cast<uint32_t>(C)));
  IO_TRY(write_le<uint32_t>(fh, static_cast<uint32_t>(D)));
  IO_TRY(write_le<uint32_t>(fh, static_cast<uint32_t>(H)));
  IO_TRY(write_arr(fh, pi, C));
  IO_TRY(write_arr(fh, mu, CD));
  // Lambda: this ABI's per-component D x H column-major block -> the file's
  // row-major D x H (io.cpp:139-144)
  std::vector<double> rowmajor(static_cast<size_t>(D) * H);
  for (int c = 0; c < C; ++c) {
    const double* lam = lambda + static_cast<size_t>(c) * D * H;
    for (int d = 0; d < D; ++d)
      for (int h = 0; h < H; ++h) rowmajor[static_cast<size_t>(d) * H + h] = lam[static_cast<size_t>(h) * D + d];
    IO_TRY(write_arr(fh, rowmajor.data(), rowmajor.size()));
  }
  IO_TRY(write_arr(fh, dnoise, CD));
  if (std::fflush(fh.f) != 0) return vmfa_b200::fail(VMFA_ERR_IO, "write failed for %s", path);
  return VMFA_OK;
}

int vmfa_checkpoint_info(const char* path, int* C, int* D, int* H) {
  if (!C || !D || !H) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "null output");
  File fh;
  IO_TRY(open_file(fh, path, "rb"));
  return checkpoint_header(fh, C, D, H);
}

int vmfa_load_checkpoint(const char* path, int C, int D, int H, double* pi, double* mu, double* lambda,
                         double* dnoise) {
  File fh;
  IO_TRY(open_file(fh, path, "rb"));
  int c = 0, d = 0, h = 0;
  IO_TRY(checkpoint_header(fh, &c, &d, &h));
  if (c != C || d != D || h != H)
    return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_load_checkpoint: file holds C=%d D=%d H=%d", c, d, h);
  if (!pi || !mu || !lambda || !dnoise) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "null parameter array");
  const size_t CD = static_cast<size_t>(C) * D;
  IO_TRY(read_arr(fh, pi, C, "pi"));
  IO_TRY(read_arr(fh, mu, CD, "mu"));
  std::vector<double> rowmajor(static_cast<size_t>(D) * H);
  for (int k = 0; k < C; ++k) {
    IO_TRY(read_arr(fh, rowmajor.data(), rowmajor.size(), "Lambda"));
    double* lam = lambda + static_cast<size_t>(k) * D * H;
    for (int dd = 0; dd < D; ++dd)
      for (int hh = 0; hh < H; ++hh) lam[static_cast<size_t>(hh) * D + dd] = rowmajor[static_cast<size_t>(dd) * H + hh];
  }
  return read_arr(fh, dnoise, CD, "dnoise");
}

int vmfa_save_state(const char* path, int64_t N, int Cp, int C, int G, const int32_t* K, const int32_t* g,
                    const int32_t* g_count) {
  if (N < 1 || Cp < 1 || C < 1 || G < 1 || Cp > C || G > C || !K || !g || !g_count)
    return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_save_state: invalid sizes or null arrays");
  File fh;
  IO_TRY(open_file(fh, path, "wb"));
  if (std::fwrite("MFAK", 1, 4, fh.f) != 4) return vmfa_b200::fail(VMFA_ERR_IO, "write failed for %s", path);
  IO_TRY(write_le<uint32_t>(fh, kStateVersion));
  IO_TRY(write_le<uint64_t>(fh, static_cast<uint64_t>(N)));
  IO_TRY(write_le<uint32_t>(fh, static_cast<uint32_t>(Cp)));
  IO_TRY(write_le<uint32_t>(fh, static_cast<uint32_t>(C)));
  IO_TRY(write_le<uint32_t>(fh, static_cast<uint32_t>(G)));
  IO_TRY(write_arr(fh, K, static_cast<size_t>(N) * Cp));
  IO_TRY(write_arr(fh, g, static_cast<size_t>(C) * G));
  IO_TRY(write_arr(fh, g_count, static_cast<size_t>(C)));
  if (std::fflush(fh.f) != 0) return vmfa_b200::fail(VMFA_ERR_IO, "write failed for %s", path);
  return VMFA_OK;
}

int vmfa_state_info(const char* path, int64_t* N, int* Cp, int* C, int* G) {
  if (!N || !Cp || !C || !G) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "null output");
  File fh;
  IO_TRY(open_file(fh, path, "rb"));
  return state_header(fh, N, Cp, C, G);
}

int vmfa_load_state(const char* path, int64_t row_begin, int64_t rows, int Cp, int C, int G, int32_t* K,
                    int32_t* g, int32_t* g_count) {
  File fh;
  IO_TRY(open_file(fh, path, "rb"));
  int64_t n = 0;
  int cp = 0, c = 0, gg = 0;
  IO_TRY(state_header(fh, &n, &cp, &c, &gg));
  if (cp != Cp || c != C || gg != G || row_begin < 0 || rows < 0 || row_begin + rows > n)
    return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "vmfa_load_state: file holds N=%lld C'=%d C=%d G=%d",
                           static_cast<long long>(n), cp, c, gg);
  if ((rows > 0 && !K) || !g || !g_count) return vmfa_b200::fail(VMFA_ERR_INVALID_ARGUMENT, "null state array");
  IO_TRY(seek(fh, kStateHeader + row_begin * static_cast<int64_t>(Cp) * 4));
  IO_TRY(read_arr(fh, K, static_cast<size_t>(rows) * Cp, "K"));
  IO_TRY(seek(fh, kStateHeader + n * static_cast<int64_t>(Cp) * 4));
  IO_TRY(read_arr(fh, g, static_cast<size_t>(C) * G, "g"));
  return read_arr(fh, g_count, static_cast<size_t>(C), "g_count");
}

}  // extern "C"
