// S2DCKPT1 checkpoint save / load straight from the device shards
// (save_checkpoint / load_checkpoint, src/embedding.cpp:133-219;
// Trainer::save_tables / load_tables, src/trainer.cpp:875-896).
//
// File: "S2DCKPT1", u32 table count, then per table u32 version (1),
// u32 table_id, u64 rows, u64 dim, f32 weights[rows*dim], f32 moments[rows],
// little-endian.  Every table's offset follows from the registered shapes,
// so the ranks of DP group 0 (the replica the reference saves) each write
// their own row ranges in place with pwrite -- no gather through one host --
// into path.tmp, which local rank 0 of group 0 creates, sizes and finally
// renames once every writer has passed a world barrier.  Loading reads each
// rank's owned rows back with pread on every replica (the reference copies
// the file into all replicas).  bf16 shards are widened to f32 on save
// (exact) and rounded to nearest-even on load.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstdio>
#include <cstring>
#include <vector>

#include "ctx.h"

namespace s2d {
namespace {

constexpr char kMagic[8] = {'S', '2', 'D', 'C', 'K', 'P', 'T', '1'};
constexpr uint32_t kVersion = 1;
constexpr uint64_t kHeader = 8 + 4;
constexpr uint64_t kTableHeader = 4 + 4 + 8 + 8;
constexpr uint64_t kChunkBytes = 64ull << 20;

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

void io_error(const std::string& what, const std::string& path) {
  throw Error(S2D_ERUNTIME, what + ": " + path + " (" + std::strerror(errno) + ")");
}

void pwrite_all(int fd, const void* p, uint64_t n, uint64_t off, const std::string& path) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    const ssize_t k = ::pwrite(fd, c, n, (off_t)off);
    if (k <= 0) io_error("checkpoint write failed", path);
    c += k;
    n -= (uint64_t)k;
    off += (uint64_t)k;
  }
}

void pread_all(int fd, void* p, uint64_t n, uint64_t off, const std::string& path) {
  char* c = static_cast<char*>(p);
  while (n) {
    const ssize_t k = ::pread(fd, c, n, (off_t)off);
    if (k < 0) io_error("checkpoint read failed", path);
    if (k == 0) throw Error(S2D_ERUNTIME, "checkpoint truncated: " + path);
    c += k;
    n -= (uint64_t)k;
    off += (uint64_t)k;
  }
}

}  // namespace

// byte offset of table f's header in the file
static std::vector<uint64_t> table_offsets(const std::vector<s2d_table_desc>& t) {
  std::vector<uint64_t> off(t.size() + 1);
  off[0] = kHeader;
  for (size_t f = 0; f < t.size(); ++f)
    off[f + 1] = off[f] + kTableHeader + (uint64_t)t[f].rows * t[f].dim * 4 + (uint64_t)t[f].rows * 4;
  return off;
}

// Host-synchronous barrier over every rank; returns how many ranks passed
// `failed` != 0, so a local IO error becomes an error on every rank instead
// of a hang.
int Ctx::world_barrier(int failed) {
  S2D_CUDA(cudaStreamSynchronize(stream));
  if (T <= 1) return failed ? 1 : 0;
  bar_buf.ensure(16);
  int* h = err_host.as<int>() + 1;  // pinned scratch next to the fault word
  *h = failed ? 1 : 0;
  S2D_CUDA(cudaMemcpyAsync(bar_buf.p, h, 4, cudaMemcpyHostToDevice, stream));
  world.allreduce_i32(bar_buf.as<int32_t>(), ncclSum, stream);
  S2D_CUDA(cudaMemcpyAsync(h, bar_buf.p, 4, cudaMemcpyDeviceToHost, stream));
  S2D_CUDA(cudaStreamSynchronize(stream));
  return *h;
}

void Ctx::save_tables(const char* path_c) {
  if (!F) throw Error(S2D_EINVAL, "register tables first");
  if (!path_c || !*path_c) throw Error(S2D_EINVAL, "empty checkpoint path");
  S2D_CUDA(cudaSetDevice(device));
  const std::string path(path_c), tmp = path + ".tmp";
  const std::vector<uint64_t> off = table_offsets(tables);
  const bool writer = group == 0, creator = group == 0 && local == 0;
  std::string why;
  auto stage = [&](auto&& fn) {  // run fn, then agree across ranks on success
    int bad = 0;
    try {
      fn();
    } catch (const std::exception& e) {
      why = e.what();
      bad = 1;
    }
    if (world_barrier(bad)) throw Error(S2D_ERUNTIME, why.empty() ? "checkpoint save failed on another rank" : why);
  };
  // 1. the creator lays out the file: magic, count, table headers, full size
  stage([&] {
    if (!creator) return;
    Fd f;
    f.fd = ::open(tmp.c_str(), O_CREAT | O_TRUNC | O_WRONLY, 0644);
    if (f.fd < 0) io_error("cannot open checkpoint", tmp);
    if (::ftruncate(f.fd, (off_t)off[F]) != 0) io_error("checkpoint write failed", tmp);
    pwrite_all(f.fd, kMagic, 8, 0, tmp);
    pwrite_all(f.fd, &F, 4, 8, tmp);
    for (uint32_t t = 0; t < F; ++t) {
      const uint32_t ver = kVersion, id = tables[t].table_id;
      const uint64_t rows = tables[t].rows, dim = tables[t].dim;
      pwrite_all(f.fd, &ver, 4, off[t], tmp);
      pwrite_all(f.fd, &id, 4, off[t] + 4, tmp);
      pwrite_all(f.fd, &rows, 8, off[t] + 8, tmp);
      pwrite_all(f.fd, &dim, 8, off[t] + 16, tmp);
    }
  });
  // 2. every rank of group 0 writes its owned rows in place
  stage([&] {
    if (!writer) return;
    Fd f;
    f.fd = ::open(tmp.c_str(), O_WRONLY);
    if (f.fd < 0) io_error("cannot open checkpoint", tmp);
    std::vector<float> w, v;
    for (uint32_t t = 0; t < F; ++t) {
      const uint32_t lo = feats[t].lo, hi = feats[t].hi, dim = feats[t].dim;
      const uint32_t step = (uint32_t)std::max<uint64_t>(1, kChunkBytes / ((uint64_t)dim * 4));
      for (uint32_t r = lo; r < hi; r += step) {
        const uint32_t e = (uint32_t)std::min<uint64_t>((uint64_t)r + step, hi);
        w.resize((size_t)(e - r) * dim);
        v.resize(e - r);
        shard_io(t, r, e, w.data(), v.data(), false);
        pwrite_all(f.fd, w.data(), w.size() * 4, off[t] + kTableHeader + (uint64_t)r * dim * 4, tmp);
        pwrite_all(f.fd, v.data(), v.size() * 4,
                   off[t] + kTableHeader + (uint64_t)tables[t].rows * dim * 4 + (uint64_t)r * 4, tmp);
      }
    }
    if (::fsync(f.fd) != 0) io_error("checkpoint sync failed", tmp);
  });
  // 3. publish
  stage([&] {
    if (creator && std::rename(tmp.c_str(), path.c_str()) != 0) io_error("cannot rename checkpoint", tmp);
  });
}

void Ctx::load_tables(const char* path_c) {
  if (!F) throw Error(S2D_EINVAL, "register tables first");
  if (!path_c || !*path_c) throw Error(S2D_EINVAL, "empty checkpoint path");
  S2D_CUDA(cudaSetDevice(device));
  const std::string path(path_c);
  Fd f;
  f.fd = ::open(path.c_str(), O_RDONLY);
  if (f.fd < 0) io_error("cannot open checkpoint", path);
  char magic[8];
  pread_all(f.fd, magic, 8, 0, path);
  if (std::memcmp(magic, kMagic, 8) != 0) throw Error(S2D_ERUNTIME, "not a checkpoint file: " + path);
  uint32_t count = 0;
  pread_all(f.fd, &count, 4, 8, path);
  if (count != F) throw Error(S2D_ERUNTIME, "checkpoint table count mismatch");
  // walk the headers with the file's own shapes, then check them
  uint64_t o = kHeader;
  std::vector<uint64_t> at(F);
  for (uint32_t t = 0; t < F; ++t) {
    uint32_t ver = 0, id = 0;
    uint64_t rows = 0, dim = 0;
    pread_all(f.fd, &ver, 4, o, path);
    if (ver != kVersion) throw Error(S2D_ERUNTIME, "unsupported checkpoint version " + std::to_string(ver));
    pread_all(f.fd, &id, 4, o + 4, path);
    pread_all(f.fd, &rows, 8, o + 8, path);
    pread_all(f.fd, &dim, 8, o + 16, path);
    if (rows != tables[t].rows || dim != tables[t].dim)
      throw Error(S2D_ERUNTIME, "checkpoint shape mismatch for table " + std::to_string(t));
    at[t] = o;
    o += kTableHeader + rows * dim * 4 + rows * 4;
  }
  struct stat st {};
  if (::fstat(f.fd, &st) != 0) io_error("cannot stat checkpoint", path);
  if ((uint64_t)st.st_size < o) throw Error(S2D_ERUNTIME, "checkpoint truncated: " + path);
  std::vector<float> w, v;
  for (uint32_t t = 0; t < F; ++t) {
    const uint32_t lo = feats[t].lo, hi = feats[t].hi, dim = feats[t].dim;
    const uint32_t step = (uint32_t)std::max<uint64_t>(1, kChunkBytes / ((uint64_t)dim * 4));
    for (uint32_t r = lo; r < hi; r += step) {
      const uint32_t e = std::min<uint64_t>((uint64_t)r + step, hi);
      w.resize((size_t)(e - r) * dim);
      v.resize(e - r);
      pread_all(f.fd, w.data(), w.size() * 4, at[t] + kTableHeader + (uint64_t)r * dim * 4, path);
      pread_all(f.fd, v.data(), v.size() * 4,
                at[t] + kTableHeader + (uint64_t)tables[t].rows * dim * 4 + (uint64_t)r * 4, path);
      shard_io(t, r, e, w.data(), v.data(), true);
    }
  }
  if (M > 1 && dirty.p) S2D_CUDA(cudaMemsetAsync(dirty.p, 0, n_slots, stream));  // replicas now agree
  S2D_CUDA(cudaStreamSynchronize(stream));
}

}  // namespace s2d
