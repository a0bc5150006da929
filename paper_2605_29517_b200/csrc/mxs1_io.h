// Native reader for the reference's "MXS1" embedding files (maxsim/streamio.py:1-163).
//
// Header (little-endian): magic "MXS1", u16 version (1), u8 elem (0 f32, 1 f16, 2 i8),
// u8 layout (0 dense, 1 packed, 2 quantized); then dense / quantized: B, L, dim (u64);
// packed: B, dim (u64) and cu_seqlens[B + 1] (u64).  Payload: row-major elements
// (dense B*L*dim, packed cu[B]*dim); quantized appends B*L f32 scales.
//
// Host-side only: the reader parses the header once, keeps the packed offset table, and copies
// any document range straight into a caller-provided (typically pinned) host buffer with
// pread(2) -- several threads for large ranges -- so the streaming scorer can overlap file I/O,
// the H2D copy and the kernels.  Validation and error classes follow _parse_header
// (maxsim/streamio.py:103-134) and _read_exact (:96-100).
#pragma once
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace mxs_io {

enum Elem { kF32 = 0, kF16 = 1, kI8 = 2 };
enum Layout { kDense = 0, kPacked = 1, kQuantized = 2 };

struct Mxs1File {
  int fd = -1;
  int elem = 0, layout = 0;
  int64_t n_docs = 0, length = 0, dim = 0;
  int64_t payload_offset = 0;
  int64_t file_size = 0;
  std::vector<int64_t> cu;  // packed only
  std::string path;
};

inline int elem_size(int elem) { return elem == kF32 ? 4 : (elem == kF16 ? 2 : 1); }

// Payload bytes of n_docs x length x dim elements (+ n_docs x length f32 scales when quantized);
// false when a header field is negative (top bit set) or the product overflows int64.
inline bool payload_bytes(int64_t n_docs, int64_t length, int64_t dim, int64_t es, bool scales, int64_t* out) {
  if (n_docs < 0 || length < 0 || dim < 0) return false;
  int64_t rows = 0, elems = 0, bytes = 0, sbytes = 0;
  if (__builtin_mul_overflow(n_docs, length, &rows)) return false;
  if (__builtin_mul_overflow(rows, dim, &elems)) return false;
  if (__builtin_mul_overflow(elems, es, &bytes)) return false;
  if (scales) {
    if (__builtin_mul_overflow(rows, (int64_t)4, &sbytes)) return false;
    if (__builtin_add_overflow(bytes, sbytes, &bytes)) return false;
  }
  *out = bytes;
  return true;
}

// Reads exactly n bytes at off (any number of pread calls); returns bytes read.
inline int64_t pread_all(int fd, void* dst, int64_t n, int64_t off) {
  int64_t done = 0;
  char* p = static_cast<char*>(dst);
  while (done < n) {
    const ssize_t r = ::pread(fd, p + done, (size_t)(n - done), (off_t)(off + done));
    if (r < 0) return -1;
    if (r == 0) break;
    done += r;
  }
  return done;
}

// Large ranges are split over a few threads (page cache / NVMe parallelism).
inline int64_t pread_parallel(int fd, void* dst, int64_t n, int64_t off) {
  constexpr int64_t kPiece = 32ll << 20;
  // page-cache -> pinned copies are host-memory-bandwidth bound: use up to 16 cores
  const int64_t hw = std::max(1u, std::thread::hardware_concurrency());
  const int nt = (int)std::min<int64_t>(std::min<int64_t>(16, hw), (n + kPiece - 1) / kPiece);
  if (nt <= 1) return pread_all(fd, dst, n, off);
  std::vector<std::thread> th;
  std::vector<int64_t> got(nt, 0);
  const int64_t per = (n + nt - 1) / nt;
  for (int i = 0; i < nt; ++i) {
    const int64_t a = i * per, b = std::min(n, a + per);
    th.emplace_back([&, i, a, b] { got[i] = (b > a) ? pread_all(fd, static_cast<char*>(dst) + a, b - a, off + a) : 0; });
  }
  int64_t total = 0;
  bool bad = false;
  for (int i = 0; i < nt; ++i) {
    th[i].join();
    if (got[i] < 0) bad = true;
    total += got[i] > 0 ? got[i] : 0;
  }
  return bad ? -1 : total;
}

}  // namespace mxs_io
