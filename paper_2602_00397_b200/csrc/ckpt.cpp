// Native reader of the reference's single-file `.ffwd` checkpoints (checkpoint.py:1-22,
// read_checkpoint :207-263).  The file is memory-mapped; the directory is parsed and
// validated with the reference's rules (magic, version, duplicate names, dtype, byte
// counts, payload bounds) and tensors are exposed as zero-copy pointers into the
// mapping, so a loader can stream them to the GPU without an intermediate copy.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_set>
#include <vector>

#include "ffwd_b200.h"

namespace {

struct Entry {
  std::string name;
  std::vector<uint32_t> dims;
  uint64_t offset, nbytes;
};

struct Ckpt {
  int fd = -1;
  const uint8_t* base = nullptr;
  size_t size = 0;
  uint32_t version = 0;
  std::string config;
  std::vector<Entry> entries;
  const uint8_t* payload = nullptr;
  uint64_t payload_len = 0;
};

thread_local std::string t_err;

int ckfail(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return FFWD_ERR_VALIDATION;
}

struct Cursor {
  const uint8_t* p;
  size_t n, pos = 0;
  const char* path;
  int err = 0;
  bool take(void* out, size_t k, const char* what) {
    if (err) return false;
    if (pos + k > n) {
      err = ckfail("checkpoint %s truncated while reading %s (need %zu bytes at offset %zu, "
                   "have %zu)", path, what, k, pos, n);
      return false;
    }
    if (out) std::memcpy(out, p + pos, k);
    pos += k;
    return true;
  }
};

}  // namespace

extern "C" {

FFWD_API const char* ffwd_ckpt_last_error(void) { return t_err.c_str(); }

FFWD_API int ffwd_ckpt_open(const char* path, void** handle) {
  t_err.clear();
  *handle = nullptr;
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) return ckfail("cannot open %s", path);
  struct stat st;
  if (fstat(fd, &st) != 0) {
    ::close(fd);
    return ckfail("cannot stat %s", path);
  }
  auto* ck = new Ckpt;
  ck->fd = fd;
  ck->size = static_cast<size_t>(st.st_size);
  if (ck->size > 0) {
    void* m = mmap(nullptr, ck->size, PROT_READ, MAP_PRIVATE, fd, 0);
    if (m == MAP_FAILED) {
      ::close(fd);
      delete ck;
      return ckfail("cannot map %s", path);
    }
    ck->base = static_cast<const uint8_t*>(m);
  }
  auto bail = [&](int rc) {
    if (ck->base) munmap(const_cast<uint8_t*>(ck->base), ck->size);
    ::close(fd);
    delete ck;
    return rc;
  };
  Cursor c{ck->base, ck->size, 0, path};
  char magic[4] = {0, 0, 0, 0};
  if (!c.take(magic, 4, "magic")) return bail(c.err);
  if (std::memcmp(magic, "FFWD", 4) != 0)
    return bail(ckfail("%s is not an engine checkpoint (magic %.4s, expected FFWD)", path, magic));
  if (!c.take(&ck->version, 4, "version")) return bail(c.err);
  if (ck->version != 1)
    return bail(ckfail("%s: unsupported checkpoint version %u", path, ck->version));
  uint32_t clen = 0;
  if (!c.take(&clen, 4, "config length")) return bail(c.err);
  if (c.pos + clen > c.n) {
    c.take(nullptr, clen, "config JSON");
    return bail(c.err);
  }
  ck->config.assign(reinterpret_cast<const char*>(ck->base + c.pos), clen);
  c.pos += clen;
  uint32_t nt = 0;
  if (!c.take(&nt, 4, "tensor count")) return bail(c.err);
  std::unordered_set<std::string> names;
  for (uint32_t t = 0; t < nt; ++t) {
    uint16_t nl = 0;
    if (!c.take(&nl, 2, "tensor name length")) return bail(c.err);
    if (c.pos + nl > c.n) {
      c.take(nullptr, nl, "tensor name");
      return bail(c.err);
    }
    Entry e;
    e.name.assign(reinterpret_cast<const char*>(ck->base + c.pos), nl);
    c.pos += nl;
    if (!names.insert(e.name).second)
      return bail(ckfail("%s: duplicate tensor name '%s'", path, e.name.c_str()));
    char dt[4];
    if (!c.take(dt, 4, "tensor dtype")) return bail(c.err);
    if (std::memcmp(dt, "f32 ", 4) != 0)
      return bail(ckfail("%s: tensor %s has unsupported dtype %.4s", path, e.name.c_str(), dt));
    uint8_t nd = 0;
    if (!c.take(&nd, 1, "tensor ndim")) return bail(c.err);
    uint64_t count = 1;
    for (int i = 0; i < nd; ++i) {
      uint32_t v = 0;
      if (!c.take(&v, 4, "tensor dim")) return bail(c.err);
      e.dims.push_back(v);
      count *= v;
    }
    if (!c.take(&e.offset, 8, "tensor offset") || !c.take(&e.nbytes, 8, "tensor size"))
      return bail(c.err);
    const uint64_t expected = 4 * count;  // ndim 0: one element
    if (e.nbytes != expected)
      return bail(ckfail("%s: tensor %s wants %llu bytes, directory says %llu", path,
                         e.name.c_str(), static_cast<unsigned long long>(expected),
                         static_cast<unsigned long long>(e.nbytes)));
    ck->entries.push_back(std::move(e));
  }
  if (!c.take(&ck->payload_len, 8, "payload length")) return bail(c.err);
  if (c.pos + ck->payload_len > c.n) {
    c.take(nullptr, ck->payload_len, "payload");
    return bail(c.err);
  }
  ck->payload = ck->base + c.pos;
  for (const Entry& e : ck->entries)
    if (e.offset + e.nbytes > ck->payload_len)
      return bail(ckfail("%s: tensor %s extends past the payload (%llu+%llu > %llu)", path,
                         e.name.c_str(), static_cast<unsigned long long>(e.offset),
                         static_cast<unsigned long long>(e.nbytes),
                         static_cast<unsigned long long>(ck->payload_len)));
  *handle = ck;
  return FFWD_OK;
}

FFWD_API void ffwd_ckpt_close(void* handle) {
  auto* ck = static_cast<Ckpt*>(handle);
  if (!ck) return;
  if (ck->base) munmap(const_cast<uint8_t*>(ck->base), ck->size);
  if (ck->fd >= 0) ::close(ck->fd);
  delete ck;
}

FFWD_API const char* ffwd_ckpt_config(void* handle, size_t* len) {
  auto* ck = static_cast<Ckpt*>(handle);
  *len = ck->config.size();
  return ck->config.data();
}

FFWD_API int ffwd_ckpt_num_tensors(void* handle) {
  return static_cast<int>(static_cast<Ckpt*>(handle)->entries.size());
}

// Name, shape and a host pointer (into the mapping) of tensor i.  dims holds up to 8.
FFWD_API int ffwd_ckpt_tensor(void* handle, int i, const char** name, int* ndim, uint32_t* dims,
                              const float** data, uint64_t* nbytes) {
  auto* ck = static_cast<Ckpt*>(handle);
  if (i < 0 || i >= static_cast<int>(ck->entries.size()))
    return ckfail("tensor index %d out of range", i);
  const Entry& e = ck->entries[i];
  if (e.dims.size() > 8) return ckfail("tensor %s has %zu dims (max 8)", e.name.c_str(), e.dims.size());
  *name = e.name.c_str();
  *ndim = static_cast<int>(e.dims.size());
  for (size_t k = 0; k < e.dims.size(); ++k) dims[k] = e.dims[k];
  *data = reinterpret_cast<const float*>(ck->payload + e.offset);
  *nbytes = e.nbytes;
  return FFWD_OK;
}

}  // extern "C"
