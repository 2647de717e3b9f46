// BAKM matrix files straight into (pinned) host memory (
// reference matio.py:17-57).  Host-only code: parallel pread of a byte range,
// so a config-3-size file (34 GB) lands in the pinned buffer that the
// pipelined GRAM upload (bak.py) streams to the GPU, with no intermediate
// numpy copy and no single-threaded read.
//
// File layout (matio.py:3-5,17-20): 16-byte little-endian header
// {"BAKM", u32 rows, u32 cols, u32 precision tag 32|64}, then the scalars in
// column-major order.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <thread>
#include <vector>

#include "bak_common.cuh"

using namespace bak;

namespace {

int pread_all(int fd, char* dst, int64_t bytes, int64_t off) {
  while (bytes > 0) {
    const ssize_t n = pread(fd, dst, static_cast<size_t>(bytes > (1LL << 30) ? (1LL << 30) : bytes), off);
    if (n < 0) {
      if (errno == EINTR) continue;
      return errno;
    }
    if (n == 0) return -1;  // short file
    dst += n;
    off += n;
    bytes -= n;
  }
  return 0;
}

}  // namespace

// Reads header fields; returns BAK_OK or BAK_EINVAL (message in bak_last_error):
// "truncated header", "bad magic", "unknown precision tag", file size too short.
extern "C" int bak_bakm_header(const char* path, int64_t* rows, int64_t* cols, int* tag, int64_t* file_bytes) {
  g_err_clear();
  if (!path || !rows || !cols || !tag) {
    set_error("bak_bakm_header: bad arguments");
    return BAK_EINVAL;
  }
  const int fd = open(path, O_RDONLY);
  if (fd < 0) {
    set_error("%s: %s", path, strerror(errno));
    return BAK_EINVAL;
  }
  unsigned char h[16];
  const int rc = pread_all(fd, reinterpret_cast<char*>(h), 16, 0);
  struct stat sb;
  fstat(fd, &sb);
  close(fd);
  if (rc != 0) {
    set_error("%s: truncated header", path);
    return BAK_EINVAL;
  }
  if (std::memcmp(h, "BAKM", 4) != 0) {
    set_error("%s: bad magic", path);
    return BAK_EINVAL;
  }
  auto u32 = [&](int o) {
    return static_cast<uint32_t>(h[o]) | (static_cast<uint32_t>(h[o + 1]) << 8) |
           (static_cast<uint32_t>(h[o + 2]) << 16) | (static_cast<uint32_t>(h[o + 3]) << 24);
  };
  *rows = u32(4);
  *cols = u32(8);
  *tag = static_cast<int>(u32(12));
  if (file_bytes) *file_bytes = static_cast<int64_t>(sb.st_size);
  if (*tag != 32 && *tag != 64) {
    set_error("%s: unknown precision tag %d", path, *tag);
    return BAK_EINVAL;
  }
  return BAK_OK;
}

// Parallel pread of [offset, offset + bytes) into dst (any host memory;
// pinned for the GPU path).  nthreads <= 0: hardware concurrency, capped at 16.
extern "C" int bak_file_read(const char* path, int64_t offset, void* dst, int64_t bytes, int nthreads) {
  g_err_clear();
  if (!path || (!dst && bytes > 0) || offset < 0 || bytes < 0) {
    set_error("bak_file_read: bad arguments");
    return BAK_EINVAL;
  }
  const int fd = open(path, O_RDONLY);
  if (fd < 0) {
    set_error("%s: %s", path, strerror(errno));
    return BAK_EINVAL;
  }
  if (nthreads <= 0) nthreads = static_cast<int>(std::thread::hardware_concurrency());
  if (nthreads > 16) nthreads = 16;
  if (nthreads < 1) nthreads = 1;
  const int64_t min_chunk = 64LL << 20;
  if (bytes < min_chunk * 2) nthreads = 1;
  std::vector<int> err(nthreads, 0);
  std::vector<std::thread> th;
  const int64_t per = (bytes + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    const int64_t b0 = t * per, b1 = b0 + per < bytes ? b0 + per : bytes;
    if (b1 <= b0) break;
    th.emplace_back([&, t, b0, b1] {
      err[t] = pread_all(fd, static_cast<char*>(dst) + b0, b1 - b0, offset + b0);
    });
  }
  for (auto& t : th) t.join();
  close(fd);
  for (int e : err) {
    if (e == -1) {
      set_error("%s: file is short", path);
      return BAK_EINVAL;
    }
    if (e != 0) {
      set_error("%s: %s", path, strerror(e));
      return BAK_EINVAL;
    }
  }
  return BAK_OK;
}
