// ingest.cu -- fvecs straight into device memory.
//
// rnnd::load_fvecs (dataset.cpp:30-95) reads the whole file into a host
// vector and then copies it.  Here the file is read in chunks of whole
// records into two pinned staging buffers; each chunk is validated in file
// order with the reference's checks and messages (parse_vecs,
// dataset.cpp:55-78: truncated record header, non-positive record
// dimension, record dimension mismatch, truncated record payload, then
// non-finite value, :89), packed in place (the 4-byte record headers
// dropped) and sent to the device store with an asynchronous H2D copy while
// the next chunk is read.  Host code only.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "ctx.hpp"

namespace rnndg {

namespace {

constexpr size_t kChunkBytes = size_t(32) << 20;

uint32_t get_u32_le(const unsigned char* p) {
  return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

// pinned staging buffers + completion events; the destructor waits for the
// copies still reading from them, so an error mid-file is safe
struct Staging {
  cudaStream_t stream;
  unsigned char* buf[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  explicit Staging(cudaStream_t s, size_t bytes) : stream(s) {
    for (int i = 0; i < 2; ++i) {
      RNNDG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&buf[i]), bytes, cudaHostAllocDefault));
      RNNDG_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
  }
  ~Staging() {
    cudaStreamSynchronize(stream);
    for (int i = 0; i < 2; ++i) {
      if (done[i]) cudaEventDestroy(done[i]);
      if (buf[i]) cudaFreeHost(buf[i]);
    }
  }
};

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

}  // namespace

void op_load_fvecs(rnndg_ctx* c, const char* path_c, uint64_t* n_out, uint32_t* d_out) {
  const std::string path(path_c);
  File file;
  file.f = std::fopen(path_c, "rb");
  if (!file.f) throw DataError(path + ": cannot open");
  if (fseeko(file.f, 0, SEEK_END) != 0) throw DataError(path + ": cannot read");
  const off_t size_o = ftello(file.f);
  if (size_o < 0) throw DataError(path + ": cannot read");
  if (fseeko(file.f, 0, SEEK_SET) != 0) throw DataError(path + ": cannot read");
  const uint64_t size = uint64_t(size_o);
  if (size == 0) throw DataError(path + ": empty file");
  if (size < 4) throw DataError(path + ": truncated record header");
  unsigned char head[4];
  if (std::fread(head, 1, 4, file.f) != 4) throw DataError(path + ": read failed");
  const int32_t rd = int32_t(get_u32_le(head));
  if (rd <= 0) throw DataError(path + ": non-positive record dimension");
  const uint32_t dim = uint32_t(rd);
  if (fseeko(file.f, 0, SEEK_SET) != 0) throw DataError(path + ": cannot read");
  const uint64_t rec = 4 + 4 * uint64_t(dim);
  const uint64_t nfull = size / rec;
  const uint64_t rest = size % rec;
  if (nfull >= (1ull << 31)) throw ParamError("load_fvecs: n must be < 2^31");

  // The store is replaced in place: invalidate the context first, so a
  // DataError part-way through the file (non-finite value, dimension
  // mismatch, truncated payload) leaves no store and no graph behind (later
  // calls fail with RNNDG_EPARAM) instead of a half-overwritten store or a
  // pointer into a buffer ensure() has just reallocated.
  c->x = nullptr;
  c->n = 0;
  c->nv = 0;
  c->v0 = 0;
  c->partitioned = false;
  c->has_graph = false;
  c->xp_src = nullptr;
  c->x_own.ensure(nfull ? nfull * dim : 1);
  float* dst = c->x_own.p;
  const uint64_t chunk_rows = kChunkBytes / rec > 0 ? kChunkBytes / rec : 1;
  Staging st(c->stream, size_t(chunk_rows * rec));
  uint64_t row0 = 0;
  for (int k = 0; row0 < nfull; ++k) {
    const int b = k & 1;
    RNNDG_CUDA(cudaEventSynchronize(st.done[b]));  // the copy out of this buffer is done
    const uint64_t rows = nfull - row0 < chunk_rows ? nfull - row0 : chunk_rows;
    unsigned char* buf = st.buf[b];
    if (std::fread(buf, 1, size_t(rows * rec), file.f) != size_t(rows * rec))
      throw DataError(path + ": read failed");
    for (uint64_t r = 0; r < rows; ++r) {
      const unsigned char* recp = buf + r * rec;
      const int32_t h = int32_t(get_u32_le(recp));
      if (h <= 0) throw DataError(path + ": non-positive record dimension");
      if (uint32_t(h) != dim) throw DataError(path + ": record dimension mismatch");
      float* out = reinterpret_cast<float*>(buf) + r * dim;
      // packed row r starts 4*(r+1) bytes before its payload: copy forward
      std::memmove(out, recp + 4, size_t(dim) * 4);
      for (uint32_t i = 0; i < dim; ++i)
        if (!std::isfinite(out[i])) throw DataError(path + ": non-finite value");
    }
    RNNDG_CUDA(cudaMemcpyAsync(dst + row0 * dim, buf, size_t(rows * dim * 4),
                               cudaMemcpyHostToDevice, c->stream));
    RNNDG_CUDA(cudaEventRecord(st.done[b], c->stream));
    row0 += rows;
  }
  if (rest) {  // a partial record at the end (parse_vecs' checks, in order)
    if (rest < 4) throw DataError(path + ": truncated record header");
    unsigned char h4[4];
    if (std::fread(h4, 1, 4, file.f) != 4) throw DataError(path + ": read failed");
    const int32_t h = int32_t(get_u32_le(h4));
    if (h <= 0) throw DataError(path + ": non-positive record dimension");
    if (uint32_t(h) != dim) throw DataError(path + ": record dimension mismatch");
    throw DataError(path + ": truncated record payload");
  }
  RNNDG_CUDA(cudaStreamSynchronize(c->stream));
  c->x = c->x_own.p;
  c->n = nfull;
  c->d = dim;
  c->v0 = 0;
  c->nv = nfull;
  c->partitioned = false;
  c->has_graph = false;
  c->xp_src = nullptr;  // chain-blocked copy is stale
  if (n_out) *n_out = nfull;
  if (d_out) *d_out = dim;
}

}  // namespace rnndg
