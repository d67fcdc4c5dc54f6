// PLXS dataset shard files (the reference's on-disk format, shard_io.hpp:
// 26-414): a byte-identical writer and a reader that streams sections
// straight into device memory.
//
// File layout (little endian): "PLXS", u32 version 1, u32 precision (4|8),
// u32 reserved, u64 ranges[6] (row0,row1,col0,col1,fcol0,fcol1), then
// (u64 offset, u64 size) for the four sections — CSR even, CSR odd,
// features, labels — and the sections back to back. Each section carries an
// FNV-1a 64 checksum in the JSON manifest (kept by shard_io.py).
//
// Device reads go through a pinned double buffer: chunk c+1 is read from the
// file while chunk c is copied to HBM (cudaMemcpyAsync) and, on a full-range
// read, hashed — the reference verifies checksums only when a read covers a
// whole section (shard_io.hpp:126-129) and so does this reader.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "pk_common.cuh"
#include "plexus_b200.h"

namespace pk {
namespace {

constexpr uint32_t kShardVersion = 1;
constexpr int kSections = 4;

// FNV-1a 64 (common.hpp:52-71)
struct Fnv1a64 {
  u64 state = 0xcbf29ce484222325ull;
  void update(const void* data, size_t n) {
    const auto* p = static_cast<const unsigned char*>(data);
    u64 s = state;
    for (size_t i = 0; i < n; ++i) {
      s ^= p[i];
      s *= 0x100000001b3ull;
    }
    state = s;
  }
};

[[noreturn]] void io_fail(int code, const std::string& msg) { throw Error(code, msg); }

struct Section {
  u64 off = 0, size = 0;
};

}  // namespace

struct PlxsFile {
  std::string path;
  std::FILE* f = nullptr;
  u32 precision = 0;
  u64 ranges[6] = {};
  Section sec[kSections];
  u64 bytes_read = 0;
  ~PlxsFile() {
    if (f) std::fclose(f);
  }

  void read_at(u64 off, void* dst, size_t n) {
    if (n == 0) return;
    if (std::fseek(f, static_cast<long>(off), SEEK_SET) != 0 ||
        std::fread(dst, 1, n, f) != n)
      io_fail(PK_ERR_IO_TRUNCATED, path + ": truncated file");
    bytes_read += n;
  }
  // bounds-checked read inside section s (shard_io.hpp:261-268)
  void section_read(int s, u64 offset, void* dst, size_t n, Fnv1a64* h) {
    if (offset + n > sec[s].size)
      io_fail(PK_ERR_IO_TRUNCATED, path + ": truncated section " + std::to_string(s));
    read_at(sec[s].off + offset, dst, n);
    if (h) h->update(dst, n);
  }
  // the same into device memory, chunked through a pinned double buffer
  void section_read_device(int s, u64 offset, void* dst, size_t n, Fnv1a64* h,
                           cudaStream_t st);
  void check_digest(int s, const Fnv1a64& h, u64 expected) const {
    if (h.state != expected)
      io_fail(PK_ERR_IO_CHECKSUM, path + ": checksum mismatch in section " + std::to_string(s));
  }
};

namespace {

struct Staging {
  static constexpr size_t kChunk = size_t{32} << 20;
  unsigned char* buf[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  Staging() {
    for (int i = 0; i < 2; ++i) {
      PK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&buf[i]), kChunk, cudaHostAllocDefault));
      PK_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
  }
  ~Staging() {
    for (int i = 0; i < 2; ++i) {
      if (buf[i]) cudaFreeHost(buf[i]);
      if (done[i]) cudaEventDestroy(done[i]);
    }
  }
};

Staging& staging() {
  static thread_local Staging s;
  return s;
}

}  // namespace

void PlxsFile::section_read_device(int s, u64 offset, void* dst, size_t n, Fnv1a64* h,
                                   cudaStream_t st) {
  if (offset + n > sec[s].size)
    io_fail(PK_ERR_IO_TRUNCATED, path + ": truncated section " + std::to_string(s));
  Staging& sg = staging();
  auto* out = static_cast<unsigned char*>(dst);
  int slot = 0;
  for (size_t done = 0; done < n; done += Staging::kChunk, slot ^= 1) {
    const size_t len = std::min(Staging::kChunk, n - done);
    PK_CUDA(cudaEventSynchronize(sg.done[slot]));  // the copy that used this slot is over
    read_at(sec[s].off + offset + done, sg.buf[slot], len);
    if (h) h->update(sg.buf[slot], len);
    PK_CUDA(cudaMemcpyAsync(out + done, sg.buf[slot], len, cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaEventRecord(sg.done[slot], st));
  }
  PK_CUDA(cudaStreamSynchronize(st));
}

}  // namespace pk

using namespace pk;

struct pk_plxs {
  PlxsFile file;
};

namespace {

std::string write_csr_section(const pk_plxs_csr_host* c, u32 precision) {
  std::string out;
  auto put = [&](const void* p, size_t n) { out.append(static_cast<const char*>(p), n); };
  const u64 head[3] = {c->rows, c->cols, c->nnz};
  put(head, sizeof(head));
  put(c->row_ptr, (c->rows + 1) * sizeof(u64));
  put(c->col_idx, c->nnz * sizeof(u32));
  put(c->values, c->nnz * precision);
  return out;
}

}  // namespace

extern "C" {

int pk_plxs_write(const char* path, const uint64_t ranges[6], uint32_t precision,
                  const pk_plxs_csr_host* even, const pk_plxs_csr_host* odd,
                  uint64_t f_rows, uint64_t f_cols, const void* features,
                  uint64_t label_count, const uint32_t* labels_row,
                  const uint32_t* labels_col, const uint8_t* mask_row,
                  const uint8_t* mask_col, uint64_t checksums_out[4]) {
  return guard([&] {
    check(path && ranges && even && odd && checksums_out, "plxs write: null argument");
    check(precision == 4 || precision == 8, "plxs write: precision must be 4 or 8");
    std::string sections[kSections];
    sections[0] = write_csr_section(even, precision);
    sections[1] = write_csr_section(odd, precision);
    {
      const u64 head[2] = {f_rows, f_cols};
      sections[2].append(reinterpret_cast<const char*>(head), sizeof(head));
      sections[2].append(static_cast<const char*>(features), f_rows * f_cols * precision);
    }
    {
      std::string& l = sections[3];
      l.append(reinterpret_cast<const char*>(&label_count), sizeof(u64));
      l.append(reinterpret_cast<const char*>(labels_row), label_count * sizeof(u32));
      l.append(reinterpret_cast<const char*>(labels_col), label_count * sizeof(u32));
      l.append(reinterpret_cast<const char*>(mask_row), label_count);
      l.append(reinterpret_cast<const char*>(mask_col), label_count);
    }
    std::string header("PLXS", 4);
    auto put32 = [&](u32 v) { header.append(reinterpret_cast<const char*>(&v), 4); };
    auto put64 = [&](u64 v) { header.append(reinterpret_cast<const char*>(&v), 8); };
    put32(kShardVersion);
    put32(precision);
    put32(0);
    for (int i = 0; i < 6; ++i) put64(ranges[i]);
    u64 offset = header.size() + kSections * 2 * sizeof(u64);
    for (int s = 0; s < kSections; ++s) {
      put64(offset);
      put64(sections[s].size());
      Fnv1a64 h;
      h.update(sections[s].data(), sections[s].size());
      checksums_out[s] = h.state;
      offset += sections[s].size();
    }
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) io_fail(PK_ERR_IO_WRITE, std::string("cannot write shard file ") + path);
    out.write(header.data(), static_cast<std::streamsize>(header.size()));
    for (const auto& sct : sections) out.write(sct.data(), static_cast<std::streamsize>(sct.size()));
    out.flush();
    if (!out) io_fail(PK_ERR_IO_WRITE, std::string("write failed for ") + path);
  });
}

int pk_plxs_open(const char* path, const uint64_t expect_ranges[6], uint32_t precision,
                 pk_plxs** out) {
  return guard([&] {
    check(path && out, "plxs open: null argument");
    *out = nullptr;
    auto h = std::make_unique<pk_plxs>();
    PlxsFile& f = h->file;
    f.path = path;
    f.f = std::fopen(path, "rb");
    if (!f.f) io_fail(PK_ERR_IO_MISSING, std::string("missing shard file ") + path);
    char magic[4];
    f.read_at(0, magic, 4);
    if (std::memcmp(magic, "PLXS", 4) != 0) io_fail(PK_ERR_IO_FORMAT, f.path + ": not a shard file");
    u32 meta[3];
    f.read_at(4, meta, sizeof(meta));
    if (meta[0] != kShardVersion) io_fail(PK_ERR_IO_FORMAT, f.path + ": unsupported version");
    f.precision = meta[1];
    if (precision && f.precision != precision)
      io_fail(PK_ERR_IO_MANIFEST, f.path + ": precision disagrees with manifest");
    f.read_at(16, f.ranges, sizeof(f.ranges));
    if (expect_ranges)
      for (int i = 0; i < 6; ++i)
        if (f.ranges[i] != expect_ranges[i])
          io_fail(PK_ERR_IO_MANIFEST, f.path + ": block ranges disagree with manifest");
    u64 secs[2 * kSections];
    f.read_at(64, secs, sizeof(secs));
    for (int s = 0; s < kSections; ++s) f.sec[s] = Section{secs[2 * s], secs[2 * s + 1]};
    *out = h.release();
  });
}

int pk_plxs_close(pk_plxs* h) {
  delete h;
  return PK_OK;
}

int pk_plxs_info(const pk_plxs* h, uint64_t ranges_out[6], uint32_t* precision,
                 uint64_t* bytes_read) {
  return guard([&] {
    check(h != nullptr, "plxs info: null handle");
    if (ranges_out) std::memcpy(ranges_out, h->file.ranges, sizeof(h->file.ranges));
    if (precision) *precision = h->file.precision;
    if (bytes_read) *bytes_read = h->file.bytes_read;
  });
}

int pk_plxs_csr_extent(pk_plxs* h, int sec, uint64_t r0, uint64_t r1, uint64_t* rows,
                       uint64_t* cols, uint64_t* nnz, uint64_t* e0, uint64_t* e1) {
  return guard([&] {
    check(h && (sec == 0 || sec == 1), "read_csr_rows: bad section");
    PlxsFile& f = h->file;
    const u64 nrows = f.ranges[1] - f.ranges[0], ncols = f.ranges[3] - f.ranges[2];
    check(r0 <= r1 && r1 <= nrows, "read_csr_rows: row range out of bounds");
    const u64 counted = f.bytes_read;  // a sizing probe: not part of the read's IO
    u64 head[3];
    f.section_read(sec, 0, head, sizeof(head), nullptr);
    if (head[0] != nrows || head[1] != ncols)
      io_fail(PK_ERR_IO_MANIFEST, f.path + ": CSR section shape disagrees with manifest");
    u64 b[2];
    f.section_read(sec, sizeof(head) + r0 * sizeof(u64), &b[0], sizeof(u64), nullptr);
    f.section_read(sec, sizeof(head) + r1 * sizeof(u64), &b[1], sizeof(u64), nullptr);
    check(b[0] <= b[1] && b[1] <= head[2], "read_csr_rows: corrupt row pointers");
    f.bytes_read = counted;
    if (rows) *rows = nrows;
    if (cols) *cols = ncols;
    if (nnz) *nnz = head[2];
    if (e0) *e0 = b[0];
    if (e1) *e1 = b[1];
  });
}

// Rows [r0, r1) of section `sec` (read_csr_rows, shard_io.hpp:120-151):
// row_ptr (host, rebased to 0), col_idx / values into host or device memory.
// A full-range read is hashed in file order and checked against `expected`.
int pk_plxs_read_csr_rows(pk_plxs* h, int sec, uint64_t r0, uint64_t r1, uint64_t expected,
                          uint64_t* row_ptr, uint32_t* col_idx, void* values, int device,
                          void* stream) {
  return guard([&] {
    check(h && (sec == 0 || sec == 1) && row_ptr, "read_csr_rows: bad arguments");
    PlxsFile& f = h->file;
    const u64 rows = f.ranges[1] - f.ranges[0];
    check(r0 <= r1 && r1 <= rows, "read_csr_rows: row range out of bounds");
    const bool full = r0 == 0 && r1 == rows;
    Fnv1a64 hash;
    Fnv1a64* hp = full ? &hash : nullptr;
    u64 head[3];
    f.section_read(sec, 0, head, sizeof(head), hp);
    f.section_read(sec, sizeof(head) + r0 * sizeof(u64), row_ptr, (r1 - r0 + 1) * sizeof(u64),
                   hp);
    const u64 e0 = row_ptr[0], e1 = row_ptr[r1 - r0], nnz = head[2];
    check(e0 <= e1 && e1 <= nnz, "read_csr_rows: corrupt row pointers");
    const u64 idx_base = sizeof(head) + (rows + 1) * sizeof(u64);
    const u64 val_base = idx_base + nnz * sizeof(u32);
    const size_t prec = f.precision;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (device) {
      f.section_read_device(sec, idx_base + e0 * sizeof(u32), col_idx, (e1 - e0) * sizeof(u32),
                            hp, st);
      f.section_read_device(sec, val_base + e0 * prec, values, (e1 - e0) * prec, hp, st);
    } else {
      f.section_read(sec, idx_base + e0 * sizeof(u32), col_idx, (e1 - e0) * sizeof(u32), hp);
      f.section_read(sec, val_base + e0 * prec, values, (e1 - e0) * prec, hp);
    }
    if (hp) f.check_digest(sec, hash, expected);
    for (u64 i = 0; i <= r1 - r0; ++i) row_ptr[i] -= e0;
  });
}

// Feature rows [r0, r1) of the file's column chunk (read_feature_rows,
// shard_io.hpp:158-176), host or device destination, row-major cols wide.
int pk_plxs_read_feature_rows(pk_plxs* h, uint64_t r0, uint64_t r1, uint64_t expected,
                              void* dst, int device, void* stream) {
  return guard([&] {
    check(h != nullptr, "read_feature_rows: null handle");
    PlxsFile& f = h->file;
    const u64 rows = f.ranges[1] - f.ranges[0], cols = f.ranges[5] - f.ranges[4];
    check(r0 <= r1 && r1 <= rows, "read_feature_rows: row range out of bounds");
    const bool full = r0 == 0 && r1 == rows;
    Fnv1a64 hash;
    Fnv1a64* hp = full ? &hash : nullptr;
    u64 head[2];
    f.section_read(2, 0, head, sizeof(head), hp);
    if (head[0] != rows || head[1] != cols)
      io_fail(PK_ERR_IO_MANIFEST, f.path + ": feature section shape disagrees with manifest");
    const u64 off = sizeof(head) + r0 * cols * f.precision;
    const size_t n = (r1 - r0) * cols * f.precision;
    if (device)
      f.section_read_device(2, off, dst, n, hp, static_cast<cudaStream_t>(stream));
    else
      f.section_read(2, off, dst, n, hp);
    if (hp) f.check_digest(2, hash, expected);
  });
}

// Label / mask rows [r0, r1) in both permutation orders (read_labels,
// shard_io.hpp:183-213), host memory.
int pk_plxs_read_labels(pk_plxs* h, uint64_t r0, uint64_t r1, uint64_t expected,
                        uint32_t* labels_row, uint32_t* labels_col, uint8_t* mask_row,
                        uint8_t* mask_col) {
  return guard([&] {
    check(h != nullptr, "read_labels: null handle");
    PlxsFile& f = h->file;
    const u64 rows = f.ranges[1] - f.ranges[0];
    check(r0 <= r1 && r1 <= rows, "read_labels: row range out of bounds");
    const bool full = r0 == 0 && r1 == rows;
    Fnv1a64 hash;
    Fnv1a64* hp = full ? &hash : nullptr;
    u64 count;
    f.section_read(3, 0, &count, sizeof(count), hp);
    if (count != rows)
      io_fail(PK_ERR_IO_MANIFEST, f.path + ": label section length disagrees with manifest");
    const u64 n = r1 - r0;
    u64 base = sizeof(u64);
    f.section_read(3, base + r0 * sizeof(u32), labels_row, n * sizeof(u32), hp);
    base += count * sizeof(u32);
    f.section_read(3, base + r0 * sizeof(u32), labels_col, n * sizeof(u32), hp);
    base += count * sizeof(u32);
    f.section_read(3, base + r0, mask_row, n, hp);
    base += count;
    f.section_read(3, base + r0, mask_col, n, hp);
    if (hp) f.check_digest(3, hash, expected);
  });
}

}  // extern "C"
