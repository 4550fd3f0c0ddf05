// scan2d_t2dm.cpp -- T2DM tensor files (include/scan2d_t2dm.h).
//
// Format and checks follow the reference's tensor I/O (tensor_io.hpp:11-16,
// tensor_io.cpp:78-151); version 2 lifts the 3-dimension cap
// (tensor_io.cpp:17) for batched tensors.  Host code only.
#include "../../include/scan2d_t2dm.h"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <vector>

namespace {

constexpr unsigned char kMagic[4] = {'T', '2', 'D', 'M'};
constexpr int kMaxNdimV1 = 3;

size_t elem_size(int dtype) { return dtype == 1 ? 8 : 4; }

bool count_of(const scan2d_tensor* t, size_t* n) {
  size_t c = 1;
  for (int i = 0; i < t->ndim; ++i) {
    const uint64_t d = t->dims[i];
    if (d == 0 || d > (uint64_t(1) << 32)) return false;
    if (c > std::numeric_limits<size_t>::max() / d) return false;
    c *= static_cast<size_t>(d);
  }
  *n = c;
  return true;
}

bool valid(const scan2d_tensor* t, size_t* n) {
  if (t == nullptr || (t->dtype != 0 && t->dtype != 1)) return false;
  if (t->ndim < 1 || t->ndim > SCAN2D_T2DM_MAX_NDIM) return false;
  if (!count_of(t, n)) return false;
  return *n == 0 || t->data != nullptr;
}

void put_u64(uint64_t v, unsigned char* o) {
  for (int i = 0; i < 8; ++i) o[i] = static_cast<unsigned char>(v >> (8 * i));
}
uint64_t get_u64(const unsigned char* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
  return v;
}

}  // namespace

extern "C" {

size_t scan2d_t2dm_encoded_bytes(const scan2d_tensor* t) {
  size_t n = 0;
  if (!valid(t, &n)) return 0;
  return 8 + 8 * static_cast<size_t>(t->ndim) + n * elem_size(t->dtype);
}

int scan2d_t2dm_encode(const scan2d_tensor* t, void* buf, size_t cap, size_t* len) {
  size_t n = 0;
  if (!valid(t, &n)) return SCAN2D_T2DM_BAD_SHAPE;
  const size_t total = scan2d_t2dm_encoded_bytes(t);
  if (buf == nullptr || cap < total) return SCAN2D_T2DM_IO;
  unsigned char* o = static_cast<unsigned char*>(buf);
  std::memcpy(o, kMagic, 4);
  o[4] = static_cast<unsigned char>(t->ndim <= kMaxNdimV1 ? 1 : 2);  // version
  o[5] = static_cast<unsigned char>(t->dtype);
  o[6] = static_cast<unsigned char>(t->ndim);
  o[7] = 0;
  o += 8;
  for (int i = 0; i < t->ndim; ++i, o += 8) put_u64(t->dims[i], o);
  // payload, little endian (the host is little endian: a byte copy)
  if (n) std::memcpy(o, t->data, n * elem_size(t->dtype));
  if (len) *len = total;
  return SCAN2D_T2DM_OK;
}

int scan2d_t2dm_decode(const void* buf, size_t len, scan2d_tensor* out, size_t* err_offset) {
  size_t off_dummy = 0;
  size_t& eo = err_offset ? *err_offset : off_dummy;
  eo = 0;
  if (out == nullptr) return SCAN2D_T2DM_IO;
  std::memset(out, 0, sizeof(*out));
  const unsigned char* p = static_cast<const unsigned char*>(buf);
  if (len < 8) {
    eo = len;
    return SCAN2D_T2DM_TRUNCATED;
  }
  if (std::memcmp(p, kMagic, 4) != 0) return eo = 0, SCAN2D_T2DM_BAD_MAGIC;
  const int version = p[4];
  if (version != 1 && version != 2) return eo = 4, SCAN2D_T2DM_BAD_VERSION;
  if (p[5] > 1) return eo = 5, SCAN2D_T2DM_BAD_DTYPE;
  const int ndim = p[6];
  const int max_nd = version == 1 ? kMaxNdimV1 : SCAN2D_T2DM_MAX_NDIM;
  if (ndim < 1 || ndim > max_nd) return eo = 6, SCAN2D_T2DM_BAD_SHAPE;
  scan2d_tensor t{};
  t.dtype = p[5];
  t.ndim = ndim;
  size_t off = 8, count = 1;
  for (int i = 0; i < ndim; ++i) {
    if (len < off + 8) return eo = len, SCAN2D_T2DM_TRUNCATED;
    const uint64_t d = get_u64(p + off);
    if (d == 0 || d > (uint64_t(1) << 32)) return eo = off, SCAN2D_T2DM_BAD_SHAPE;
    if (count > std::numeric_limits<size_t>::max() / d) return eo = off, SCAN2D_T2DM_BAD_SHAPE;
    t.dims[i] = d;
    count *= static_cast<size_t>(d);
    off += 8;
  }
  const size_t es = elem_size(t.dtype);
  if (count > (std::numeric_limits<size_t>::max() - off) / es) return eo = off, SCAN2D_T2DM_BAD_SHAPE;
  if (len < off + count * es) return eo = len, SCAN2D_T2DM_TRUNCATED;
  const unsigned char* pay = p + off;
  for (size_t k = 0; k < count; ++k) {
    bool fin;
    if (es == 4) {
      float v;
      std::memcpy(&v, pay + 4 * k, 4);
      fin = std::isfinite(v);
    } else {
      double v;
      std::memcpy(&v, pay + 8 * k, 8);
      fin = std::isfinite(v);
    }
    if (!fin) return eo = off + k * es, SCAN2D_T2DM_NON_FINITE;
  }
  t.data = std::malloc(count * es ? count * es : 1);
  if (t.data == nullptr) return SCAN2D_T2DM_IO;
  std::memcpy(t.data, pay, count * es);
  *out = t;
  return SCAN2D_T2DM_OK;
}

int scan2d_t2dm_write(const char* path, const scan2d_tensor* t, size_t* bytes_written) {
  const size_t total = scan2d_t2dm_encoded_bytes(t);
  if (total == 0) return SCAN2D_T2DM_BAD_SHAPE;
  std::vector<unsigned char> buf(total);
  size_t len = 0;
  int rc = scan2d_t2dm_encode(t, buf.data(), buf.size(), &len);
  if (rc != SCAN2D_T2DM_OK) return rc;
  FILE* f = path ? std::fopen(path, "wb") : nullptr;
  if (f == nullptr) return SCAN2D_T2DM_IO;
  const size_t w = std::fwrite(buf.data(), 1, len, f);
  const int cl = std::fclose(f);
  if (w != len || cl != 0) return SCAN2D_T2DM_IO;
  if (bytes_written) *bytes_written = len;
  return SCAN2D_T2DM_OK;
}

int scan2d_t2dm_read(const char* path, scan2d_tensor* out, size_t* err_offset) {
  FILE* f = path ? std::fopen(path, "rb") : nullptr;
  if (f == nullptr) return SCAN2D_T2DM_IO;
  std::vector<unsigned char> buf;
  unsigned char chunk[1 << 16];
  size_t r;
  while ((r = std::fread(chunk, 1, sizeof(chunk), f)) > 0) buf.insert(buf.end(), chunk, chunk + r);
  const bool err = std::ferror(f) != 0;
  std::fclose(f);
  if (err) return SCAN2D_T2DM_IO;
  return scan2d_t2dm_decode(buf.data(), buf.size(), out, err_offset);
}

void scan2d_t2dm_free(scan2d_tensor* t) {
  if (t == nullptr) return;
  std::free(t->data);
  t->data = nullptr;
}

const char* scan2d_t2dm_status_string(int status) {
  switch (status) {
    case SCAN2D_T2DM_OK: return "ok";
    case SCAN2D_T2DM_BAD_MAGIC: return "bad magic";
    case SCAN2D_T2DM_BAD_VERSION: return "unsupported version";
    case SCAN2D_T2DM_BAD_DTYPE: return "unsupported dtype";
    case SCAN2D_T2DM_BAD_SHAPE: return "bad shape";
    case SCAN2D_T2DM_TRUNCATED: return "truncated";
    case SCAN2D_T2DM_NON_FINITE: return "non-finite entry";
    case SCAN2D_T2DM_IO: return "i/o error";
    default: return "unknown status";
  }
}

}  // extern "C"
