// columnio.cpp — native batch reader for the columnar input format
// (reference columnio.py:1-20 layout, decode columnio.py:224-265, batching
// columnio.py:268-303, reader columnio.py:328-409).
//
// The Python layer parses the file headers and plans this shard's chunks
// (round-robin by global chunk index, columnio.py:306-325); this file is the
// data plane: pread + raw-DEFLATE inflate + column decode on a pool of
// decoder threads (chunks decode out of order, are consumed in order), and an
// assembler thread that slices fixed-row batches across chunk boundaries into
// reusable batch buffers — pinned host memory when the batches are headed for
// the GPU, so each column crosses PCIe with one async copy.  Byte-string
// columns are delivered packed (string offsets + one blob) so hashing never
// touches Python objects.  Batch order never depends on scheduling.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>
#include <zlib.h>

#include <condition_variable>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "sparsekit_b200.h"

namespace skb {
int set_error(int code, const char* msg, int64_t arg);  // runtime.cu
void clear_error();
}

namespace {

enum : int32_t { kF32 = 0, kI64 = 1, kBytes = 2 };

struct IoError {
  std::string msg;
};

[[noreturn]] void fail(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw IoError{buf};
}

// growable byte buffer, optionally page-locked (cudaHostAlloc)
struct HostBuf {
  uint8_t* p = nullptr;
  size_t cap = 0, size = 0;
  bool pinned = false;
  HostBuf() = default;
  explicit HostBuf(bool pin) : pinned(pin) {}
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  ~HostBuf() { release(); }
  void release() {
    if (!p) return;
    if (pinned)
      cudaFreeHost(p);
    else
      free(p);
    p = nullptr;
    cap = 0;
  }
  void reserve(size_t n) {
    if (n <= cap) return;
    size_t c = cap ? cap : 4096;
    while (c < n) c += c / 2 + 4096;
    uint8_t* q = nullptr;
    if (pinned) {
      if (cudaHostAlloc(reinterpret_cast<void**>(&q), c, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        fail("cudaHostAlloc(%zu) failed", c);
      }
    } else {
      q = static_cast<uint8_t*>(malloc(c));
      if (!q) fail("out of host memory (%zu bytes)", c);
    }
    if (size) memcpy(q, p, size);
    release();
    p = q;
    cap = c;
  }
  void resize(size_t n) {
    reserve(n);
    size = n;
  }
  template <class T> T* as() { return reinterpret_cast<T*>(p); }
};

struct Column {
  std::string name;
  int32_t dtype;
  bool ragged;
  bool selected;
};

struct ChunkRef {
  int64_t path, offset, len, rows, index;
};

// one decoded column of one chunk: row lengths + values (or packed strings)
struct ChunkCol {
  std::vector<int64_t> offs;   // rows + 1, chunk-local
  std::vector<uint8_t> vals;   // f32 / i64 payload, or the string blob
  std::vector<int64_t> soffs;  // bytes: count + 1 string offsets into vals
};

struct Chunk {
  int64_t rows = 0;
  std::vector<ChunkCol> cols;  // selected columns only
};

// one assembled batch (selected columns, reader-owned buffers)
struct Batch {
  int64_t rows = 0;
  std::vector<std::unique_ptr<HostBuf>> offs, vals, soffs;
  std::vector<int64_t> nvals;
};

int64_t rd64(const uint8_t* p) {
  int64_t v;
  memcpy(&v, p, 8);
  return v;
}

void read_exact(int fd, int64_t off, int64_t len, std::vector<uint8_t>& out, const std::string& path,
                int64_t chunk) {
  out.resize(len);
  int64_t got = 0;
  while (got < len) {
    ssize_t r = pread(fd, out.data() + got, len - got, off + got);
    if (r < 0) fail("%s: chunk %lld: read error", path.c_str(), (long long)chunk);
    if (r == 0) break;
    got += r;
  }
  if (got != len) fail("%s: chunk %lld: truncated chunk", path.c_str(), (long long)chunk);
}

void inflate_raw(const uint8_t* src, size_t n, std::vector<uint8_t>& out, size_t raw_len, const Column& c) {
  out.resize(raw_len);
  z_stream zs{};
  if (inflateInit2(&zs, -15) != Z_OK) fail("column '%s': inflateInit2 failed", c.name.c_str());
  zs.next_in = const_cast<Bytef*>(src);
  zs.avail_in = (uInt)n;
  // inflate everything; the produced size is checked against raw_len below
  size_t produced = 0;
  int rc;
  do {
    if (produced == out.size()) out.resize(out.size() * 2 + 64);
    zs.next_out = out.data() + produced;
    zs.avail_out = (uInt)(out.size() - produced);
    rc = inflate(&zs, Z_NO_FLUSH);
    produced = out.size() - zs.avail_out;
    if (rc == Z_STREAM_END) break;
    if (rc != Z_OK) {
      const char* m = zs.msg ? zs.msg : "corrupt stream";
      int code = rc == Z_BUF_ERROR ? -5 : rc;
      inflateEnd(&zs);
      fail("column '%s': bad DEFLATE data: Error %d while decompressing data: %s", c.name.c_str(), code, m);
    }
  } while (zs.avail_in > 0 || zs.avail_out == 0);
  const bool ended = rc == Z_STREAM_END;
  inflateEnd(&zs);
  if (!ended)
    fail("column '%s': bad DEFLATE data: Error -5 while decompressing data: incomplete or truncated stream",
         c.name.c_str());
  out.resize(produced);
}

void decode_values(const uint8_t* p, size_t n, int64_t count, const Column& c, ChunkCol& cc) {
  if (c.dtype == kF32 || c.dtype == kI64) {
    const size_t w = c.dtype == kF32 ? 4 : 8;
    if (n != w * (size_t)count)
      fail("%s payload length mismatch", c.dtype == kF32 ? "float32" : "int64");
    cc.vals.assign(p, p + n);
    return;
  }
  if (n < 8 * (size_t)count) fail("byte-string payload shorter than its length array");
  cc.soffs.resize(count + 1);
  cc.soffs[0] = 0;
  int64_t total = 0;
  for (int64_t i = 0; i < count; ++i) {
    const int64_t ln = rd64(p + 8 * i);
    total += ln;
    cc.soffs[i + 1] = total;
  }
  if (total != (int64_t)(n - 8 * (size_t)count)) fail("byte-string payload length mismatch");
  cc.vals.assign(p + 8 * count, p + n);
}

void check_offsets(const std::vector<int64_t>& o, int64_t count) {
  if (o[0] != 0) fail("row_offsets must start at 0");
  for (size_t i = 1; i < o.size(); ++i)
    if (o[i] < o[i - 1]) fail("row_offsets must be nondecreasing");
  (void)count;
}

// decode one chunk (columnio.py:224-265)
void decode_chunk(const std::vector<Column>& cols, const std::vector<uint8_t>& blob, int64_t rows, Chunk& out) {
  size_t pos = 0;
  out.rows = rows;
  out.cols.clear();
  std::vector<uint8_t> raw;
  for (const Column& c : cols) {
    if (pos + 17 > blob.size()) fail("column '%s': truncated column header", c.name.c_str());
    const uint8_t flag = blob[pos];
    const int64_t raw_len = rd64(&blob[pos + 1]);
    const int64_t stored_len = rd64(&blob[pos + 9]);
    pos += 17;
    if (stored_len < 0 || pos + (size_t)stored_len > blob.size())
      fail("column '%s': truncated payload", c.name.c_str());
    if (c.selected) {
      const uint8_t* p = &blob[pos];
      size_t n = (size_t)stored_len;
      if (flag) {
        inflate_raw(p, n, raw, raw_len > 0 ? (size_t)raw_len : 64, c);
        p = raw.data();
        n = raw.size();
      }
      if ((int64_t)n != raw_len) fail("column '%s': raw length mismatch", c.name.c_str());
      ChunkCol cc;
      if (c.ragged) {
        const size_t need = 8 * (size_t)(rows + 1);
        if (n < need) fail("column '%s': truncated offsets", c.name.c_str());
        cc.offs.resize(rows + 1);
        memcpy(cc.offs.data(), p, need);
        const int64_t count = cc.offs[rows];
        if (count < 0) fail("row_offsets must be nondecreasing");
        decode_values(p + need, n - need, count, c, cc);
        check_offsets(cc.offs, count);
      } else {
        cc.offs.resize(rows + 1);
        for (int64_t i = 0; i <= rows; ++i) cc.offs[i] = i;
        decode_values(p, n, rows, c, cc);
      }
      out.cols.push_back(std::move(cc));
    }
    pos += (size_t)stored_len;
  }
  if (pos != blob.size()) fail("trailing bytes after last column");
}

size_t elem_bytes(int32_t dtype) { return dtype == kF32 ? 4 : dtype == kI64 ? 8 : 1; }

struct Reader {
  std::vector<std::string> paths;
  std::vector<int> fds;
  std::vector<ChunkRef> chunks;
  std::vector<Column> cols;
  std::vector<int> sel;  // indices of selected columns
  int64_t batch_rows;
  size_t depth;
  bool pinned;
  int device = 0;  // CUDA device the pinned batch buffers are allocated for

  // decode pool: chunk k's result lands in slot k % window
  size_t window;
  struct Slot {
    int64_t chunk = -1;
    bool done = false;
    bool failed = false;
    std::string err;
    Chunk data;
  };
  std::vector<Slot> slots;
  int64_t next_decode = 0;  // next chunk index a decoder may claim
  int64_t consumed = 0;     // chunks handed to the assembler
  std::mutex m;
  std::condition_variable cv_dec, cv_asm, cv_out;
  bool stopping = false;
  std::vector<std::thread> decoders;
  std::thread assembler;

  // assembled batches
  std::deque<Batch*> ready;
  std::vector<Batch*> free_batches;
  std::vector<std::unique_ptr<Batch>> all_batches;
  bool finished = false;
  bool asm_failed = false;
  std::string asm_err;
  Batch* current = nullptr;

  ~Reader() { shutdown(); }

  void shutdown() {
    {
      std::lock_guard<std::mutex> g(m);
      stopping = true;
    }
    cv_dec.notify_all();
    cv_asm.notify_all();
    cv_out.notify_all();
    for (auto& t : decoders)
      if (t.joinable()) t.join();
    if (assembler.joinable()) assembler.join();
    decoders.clear();
    for (int fd : fds)
      if (fd >= 0) close(fd);
    fds.clear();
  }

  void decoder_loop() {
    std::vector<uint8_t> blob;
    while (true) {
      int64_t k;
      {
        std::unique_lock<std::mutex> g(m);
        cv_dec.wait(g, [&] { return stopping || (next_decode < (int64_t)chunks.size() &&
                                                 next_decode < consumed + (int64_t)window); });
        if (stopping) return;
        k = next_decode++;
      }
      Slot& s = slots[k % window];
      Chunk c;
      std::string err;
      bool bad = false;
      try {
        const ChunkRef& r = chunks[k];
        read_exact(fds[r.path], r.offset, r.len, blob, paths[r.path], r.index);
        try {
          decode_chunk(cols, blob, r.rows, c);
        } catch (const IoError& e) {
          fail("%s: chunk %lld: %s", paths[r.path].c_str(), (long long)r.index, e.msg.c_str());
        }
      } catch (const IoError& e) {
        bad = true;
        err = e.msg;
      }
      {
        std::lock_guard<std::mutex> g(m);
        s.chunk = k;
        s.data = std::move(c);
        s.failed = bad;
        s.err = err;
        s.done = true;
      }
      cv_asm.notify_all();
    }
  }

  Batch* take_free_batch() {  // with m held by caller's unique_lock
    Batch* b;
    if (!free_batches.empty()) {
      b = free_batches.back();
      free_batches.pop_back();
    } else {
      all_batches.emplace_back(new Batch());
      b = all_batches.back().get();
      for (size_t j = 0; j < sel.size(); ++j) {
        b->offs.emplace_back(new HostBuf(pinned));
        b->vals.emplace_back(new HostBuf(pinned));
        b->soffs.emplace_back(new HostBuf(pinned));
      }
      b->nvals.assign(sel.size(), 0);
    }
    return b;
  }

  // assembler: in-order chunks -> fixed-row batches (columnio.py:268-303)
  void assembler_loop() {
    if (pinned) cudaSetDevice(device);  // pinned allocations from this thread
    std::deque<Chunk> pending;
    int64_t head_row = 0;  // rows of pending.front() already emitted
    int64_t avail = 0;     // rows pending
    auto emit = [&](int64_t count) -> bool {
      Batch* b;
      {
        std::unique_lock<std::mutex> g(m);
        cv_out.wait(g, [&] { return stopping || ready.size() < depth; });
        if (stopping) return false;
        b = take_free_batch();
      }
      b->rows = count;
      for (size_t j = 0; j < sel.size(); ++j) {
        const Column& c = cols[sel[j]];
        const size_t eb = elem_bytes(c.dtype);
        // pass 1: sizes
        int64_t nv = 0, nbytes = 0, left = count, hr = head_row;
        for (size_t q = 0; q < pending.size() && left > 0; ++q) {
          const ChunkCol& cc = pending[q].cols[j];
          const int64_t r0 = q == 0 ? hr : 0, take = std::min(left, pending[q].rows - r0);
          const int64_t e0 = cc.offs[r0], e1 = cc.offs[r0 + take];
          nv += e1 - e0;
          nbytes += c.dtype == kBytes ? cc.soffs[e1] - cc.soffs[e0] : (e1 - e0) * (int64_t)eb;
          left -= take;
        }
        b->offs[j]->resize(8 * (count + 1));
        b->vals[j]->resize(nbytes);
        if (c.dtype == kBytes) b->soffs[j]->resize(8 * (nv + 1));
        int64_t* o = b->offs[j]->as<int64_t>();
        int64_t* so = c.dtype == kBytes ? b->soffs[j]->as<int64_t>() : nullptr;
        uint8_t* v = b->vals[j]->p;
        int64_t ro = 0, eo = 0, bo = 0;
        o[0] = 0;
        if (so) so[0] = 0;
        left = count;
        for (size_t q = 0; q < pending.size() && left > 0; ++q) {
          const ChunkCol& cc = pending[q].cols[j];
          const int64_t r0 = q == 0 ? head_row : 0, take = std::min(left, pending[q].rows - r0);
          const int64_t e0 = cc.offs[r0];
          for (int64_t r = 1; r <= take; ++r) o[ro + r] = eo + (cc.offs[r0 + r] - e0);
          const int64_t ne = cc.offs[r0 + take] - e0;
          if (c.dtype == kBytes) {
            const int64_t b0 = cc.soffs[e0];
            for (int64_t e = 1; e <= ne; ++e) so[eo + e] = bo + (cc.soffs[e0 + e] - b0);
            const int64_t nb = cc.soffs[e0 + ne] - b0;
            if (nb) memcpy(v + bo, cc.vals.data() + b0, nb);
            bo += nb;
          } else {
            if (ne) memcpy(v + eo * eb, cc.vals.data() + e0 * eb, ne * eb);
          }
          ro += take;
          eo += ne;
          left -= take;
        }
        b->nvals[j] = nv;
      }
      // consume the rows
      int64_t left = count;
      while (left > 0) {
        const int64_t r = pending.front().rows - head_row;
        if (r <= left) {
          left -= r;
          pending.pop_front();
          head_row = 0;
        } else {
          head_row += left;
          left = 0;
        }
      }
      avail -= count;
      {
        std::lock_guard<std::mutex> g(m);
        ready.push_back(b);
      }
      cv_out.notify_all();
      return true;
    };
    for (int64_t k = 0; k < (int64_t)chunks.size(); ++k) {
      Chunk c;
      {
        std::unique_lock<std::mutex> g(m);
        Slot& s = slots[k % window];
        cv_asm.wait(g, [&] { return stopping || (s.done && s.chunk == k); });
        if (stopping) return;
        if (s.failed) {
          asm_failed = true;
          asm_err = s.err;
          finished = true;
          cv_out.notify_all();
          return;
        }
        c = std::move(s.data);
        s.done = false;
        consumed = k + 1;
      }
      cv_dec.notify_all();
      // drop empty chunks' columns cheaply; they add no rows
      avail += c.rows;
      if (c.rows) pending.push_back(std::move(c));
      while (avail >= batch_rows)
        if (!emit(batch_rows)) return;
    }
    if (avail > 0 && !emit(avail)) return;
    std::lock_guard<std::mutex> g(m);
    finished = true;
    cv_out.notify_all();
  }

  void start(int threads) {
    window = (size_t)std::max(2, 2 * threads);
    slots.resize(window);
    for (int t = 0; t < threads; ++t) decoders.emplace_back(&Reader::decoder_loop, this);
    assembler = std::thread(&Reader::assembler_loop, this);
  }

  // returns rows of the next batch (0 at end); throws IoError
  int64_t next() {
    std::unique_lock<std::mutex> g(m);
    if (current) {
      free_batches.push_back(current);
      current = nullptr;
    }
    cv_out.notify_all();
    cv_out.wait(g, [&] { return !ready.empty() || finished; });
    if (!ready.empty()) {
      current = ready.front();
      ready.pop_front();
      cv_out.notify_all();
      return current->rows;
    }
    if (asm_failed) throw IoError{asm_err};
    return 0;
  }
};

int io_fail(const std::string& msg) { return skb::set_error(SKB_E_IO, msg.c_str(), 0); }
int arg_fail(int64_t arg, const char* msg) { return skb::set_error(SKB_E_ARG, msg, arg); }

}  // namespace

extern "C" {

int skb_reader_open(const char* const* paths, int64_t npaths, const int64_t* chunks, int64_t nchunks,
                    const char* const* col_names, const int32_t* col_dtype, const int32_t* col_ragged,
                    const int32_t* col_selected, int64_t ncols, int64_t batch_rows, int64_t prefetch_depth,
                    int32_t threads, int32_t pinned, int32_t device, skb_reader_t* out) {
  skb::clear_error();
  if (!out || batch_rows < 1 || npaths < 0 || nchunks < 0 || ncols < 0)
    return arg_fail(batch_rows, "skb_reader_open: bad arguments");
  auto r = std::make_unique<Reader>();
  for (int64_t i = 0; i < npaths; ++i) {
    r->paths.emplace_back(paths[i]);
    const int fd = open(paths[i], O_RDONLY);
    if (fd < 0) return io_fail(std::string(paths[i]) + ": cannot open");
    r->fds.push_back(fd);
  }
  for (int64_t i = 0; i < nchunks; ++i) {
    const int64_t* c = chunks + 5 * i;
    if (c[0] < 0 || c[0] >= npaths || c[2] < 0 || c[3] < 0) return arg_fail(i, "skb_reader_open: bad chunk descriptor");
    r->chunks.push_back(ChunkRef{c[0], c[1], c[2], c[3], c[4]});
  }
  for (int64_t j = 0; j < ncols; ++j) {
    if (col_dtype[j] < kF32 || col_dtype[j] > kBytes) return arg_fail(j, "skb_reader_open: bad column dtype");
    r->cols.push_back(Column{col_names[j], col_dtype[j], col_ragged[j] != 0, col_selected[j] != 0});
    if (col_selected[j]) r->sel.push_back((int)j);
  }
  r->batch_rows = batch_rows;
  r->depth = (size_t)std::max<int64_t>(1, prefetch_depth);
  r->pinned = pinned != 0;
  r->device = device;
  r->start(std::max(1, threads));
  *out = reinterpret_cast<skb_reader_t>(r.release());
  return SKB_OK;
}

int skb_reader_next(skb_reader_t h, int64_t* rows) {
  skb::clear_error();
  if (!h || !rows) return arg_fail(0, "skb_reader_next: null argument");
  try {
    *rows = reinterpret_cast<Reader*>(h)->next();
  } catch (const IoError& e) {
    return io_fail(e.msg);
  }
  return SKB_OK;
}

int skb_reader_column(skb_reader_t h, int64_t j, const int64_t** row_offsets, const void** values,
                      int64_t* n_values, const int64_t** str_offsets, int64_t* blob_bytes) {
  Reader* r = reinterpret_cast<Reader*>(h);
  if (!r || !r->current || j < 0 || j >= (int64_t)r->sel.size())
    return arg_fail(j, "skb_reader_column: no current batch or bad column");
  Batch* b = r->current;
  const Column& c = r->cols[r->sel[j]];
  *row_offsets = b->offs[j]->as<int64_t>();
  *values = b->vals[j]->p;
  *n_values = b->nvals[j];
  *str_offsets = c.dtype == kBytes ? b->soffs[j]->as<int64_t>() : nullptr;
  *blob_bytes = c.dtype == kBytes ? (int64_t)b->vals[j]->size : 0;
  return SKB_OK;
}

int skb_reader_close(skb_reader_t h) {
  delete reinterpret_cast<Reader*>(h);
  return SKB_OK;
}

}  // extern "C"
