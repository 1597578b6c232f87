// gk_sg.cu -- serialized-graph cache straight to HBM.
//
// Reads / writes the reference's binary layout (proj/include/gapkit/io.hpp:
// 328-456, pinned by test_io.cc:174-203): "GAPB", u8 version 1, u8 flags
// (bit0 directed, bit1 weighted), u64 n, u64 m, out_offsets (n+1) x u64,
// out_neighbors m x u32, [out_weights m x i32], [in_offsets, in_neighbors,
// [in_weights]] when directed.  The arrays stream through two pinned staging
// buffers: the file read of chunk i+1 overlaps the H2D copy of chunk i, so a
// scale-27 .sg (~18 GB) loads at disk speed with no host-sized copy of the
// graph.  Weights are skipped (BFS is unweighted); the same invariants the
// reference's ReadSerialized checks (io.hpp:451-452) are checked on the
// device copy's offsets.
#include <cstdio>
#include <cstring>
#include <string>

#include "gk_internal.cuh"

namespace gk {
namespace {

constexpr size_t kStage = size_t(64) << 20;  // bytes per staging buffer

struct Stager {
  char* buf[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  cudaStream_t s = nullptr;
  ~Stager() {
    for (int i = 0; i < 2; i++) {
      if (done[i]) cudaEventDestroy(done[i]);
      if (buf[i]) cudaFreeHost(buf[i]);
    }
    if (s) cudaStreamDestroy(s);
  }
  cudaError_t init() {
    cudaError_t e;
    for (int i = 0; i < 2; i++) {
      if ((e = cudaHostAlloc(&buf[i], kStage, cudaHostAllocDefault))) return e;
      if ((e = cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming))) return e;
    }
    return cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  }
};

// fread `bytes` from f into device memory dst (nullptr: skip), double-buffered.
// Returns "" on success, else an error message.
std::string stream_in(FILE* f, Stager& st, char* dst, size_t bytes) {
  if (!dst) {
    if (fseeko(f, (off_t)bytes, SEEK_CUR) != 0) return "truncated array data";
    return "";
  }
  size_t done = 0;
  int k = 0;
  while (done < bytes) {
    const size_t chunk = bytes - done < kStage ? bytes - done : kStage;
    cudaEventSynchronize(st.done[k]);  // the copy that last used buf[k] has finished
    if (fread(st.buf[k], 1, chunk, f) != chunk) return "truncated array data";
    if (cudaMemcpyAsync(dst + done, st.buf[k], chunk, cudaMemcpyHostToDevice, st.s) != cudaSuccess)
      return "H2D copy failed";
    cudaEventRecord(st.done[k], st.s);
    done += chunk;
    k ^= 1;
  }
  return "";
}

std::string stream_out(FILE* f, Stager& st, const char* src, size_t bytes) {
  size_t done = 0;
  while (done < bytes) {
    const size_t chunk = bytes - done < kStage ? bytes - done : kStage;
    if (cudaMemcpyAsync(st.buf[0], src + done, chunk, cudaMemcpyDeviceToHost, st.s) != cudaSuccess ||
        cudaStreamSynchronize(st.s) != cudaSuccess)
      return "D2H copy failed";
    if (fwrite(st.buf[0], 1, chunk, f) != chunk) return "write failed";
    done += chunk;
  }
  return "";
}

__global__ void k_check_offsets(const int64_t* off, int64_t n, int64_t m, unsigned long long* bad) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (long long)gridDim.x * blockDim.x)
    if (off[v] > off[v + 1] || off[v + 1] > m) atomicAdd(bad, 1ull);
  if (blockIdx.x == 0 && threadIdx.x == 0 && (off[0] != 0 || off[n] != m)) atomicAdd(bad, 1ull);
}

}  // namespace

int sg_load(const char* path, int64_t* n_out, int64_t* m_out, int* directed_out, int64_t** off,
            uint32_t** nb, int64_t** in_off, uint32_t** in_nb, std::string* err) {
  FILE* f = fopen(path, "rb");
  if (!f) {
    *err = std::string("cannot open graph file: ") + path;
    return 2;
  }
  unsigned char hdr[22];
  int code = 0;
  Stager st;
  uint64_t n = 0, m = 0;
  bool directed = false, weighted = false;
  unsigned long long* bad = nullptr;
  *off = nullptr;
  *nb = nullptr;
  *in_off = nullptr;
  *in_nb = nullptr;
  auto fail = [&](int c, const std::string& m_) {
    *err = std::string(path) + ": " + m_;
    code = c;
  };
  if (fread(hdr, 1, 4, f) != 4 || memcmp(hdr, "GAPB", 4) != 0) {
    fail(3, "not a serialized graph (bad magic)");  // io.hpp:398-400
  } else if (fread(hdr + 4, 1, 18, f) != 18) {
    fail(4, "truncated array data");
  } else if (hdr[4] != 1) {
    fail(5, "unsupported version " + std::to_string(hdr[4]));  // io.hpp:403-405
  } else if (hdr[5] & ~3u) {
    fail(6, "unknown flag bits");
  } else {
    directed = hdr[5] & 1;
    weighted = hdr[5] & 2;
    memcpy(&n, hdr + 6, 8);
    memcpy(&m, hdr + 14, 8);
  }
  if (!code && n > (uint64_t(1) << 31)) {
    fail(2, "more than 2^31 vertices (parents are int32)");
  } else if (!code && m > (uint64_t(1) << 40)) {  // also keeps the size arithmetic below from overflowing
    fail(4, "declared arc count out of range");
  } else if (!code) {
    fseeko(f, 0, SEEK_END);
    const uint64_t actual = (uint64_t)ftello(f);
    fseeko(f, 22, SEEK_SET);
    const uint64_t sides = directed ? 2 : 1;
    const uint64_t expected = 22 + sides * ((n + 1) * 8 + m * 4 + (weighted ? m * 4 : 0));
    if (actual < expected) fail(4, "file shorter than its declared arrays");  // io.hpp:415-421
  }
  if (!code && st.init() != cudaSuccess) fail(7, "cannot allocate staging buffers");
  const size_t ob = (n + 1) * 8 + 16, nbb = (m ? m : 1) * 4 + kNbPad;
  if (!code && (cudaMalloc(off, ob) || cudaMalloc(nb, nbb))) fail(8, "device allocation failed");
  std::string e;
  if (!code && !(e = stream_in(f, st, (char*)*off, (n + 1) * 8)).empty()) fail(4, e);
  if (!code && !(e = stream_in(f, st, (char*)*nb, m * 4)).empty()) fail(4, e);
  if (!code && weighted && !(e = stream_in(f, st, nullptr, m * 4)).empty()) fail(4, e);
  if (!code && directed) {
    if (cudaMalloc(in_off, ob) || cudaMalloc(in_nb, nbb)) fail(8, "device allocation failed");
    if (!code && !(e = stream_in(f, st, (char*)*in_off, (n + 1) * 8)).empty()) fail(4, e);
    if (!code && !(e = stream_in(f, st, (char*)*in_nb, m * 4)).empty()) fail(4, e);
  }
  fclose(f);
  if (!code) {
    cudaStreamSynchronize(st.s);
    cudaMalloc(&bad, sizeof(unsigned long long));
    cudaMemset(bad, 0, sizeof(unsigned long long));
    k_check_offsets<<<148 * 4, 256, 0, st.s>>>(*off, (int64_t)n, (int64_t)m, bad);
    if (directed) k_check_offsets<<<148 * 4, 256, 0, st.s>>>(*in_off, (int64_t)n, (int64_t)m, bad);
    unsigned long long hb = 0;
    cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, st.s);
    cudaStreamSynchronize(st.s);
    cudaFree(bad);
    if (hb) fail(9, "invalid graph data: offsets not monotone / out of range");  // io.hpp:451-452
  }
  if (code) {
    cudaFree(*off);
    cudaFree(*nb);
    cudaFree(*in_off);
    cudaFree(*in_nb);
    *off = nullptr;
    *nb = nullptr;
    *in_off = nullptr;
    *in_nb = nullptr;
    return code;
  }
  *n_out = (int64_t)n;
  *m_out = (int64_t)m;
  *directed_out = directed ? 1 : 0;
  return 0;
}

int sg_save(const char* path, int64_t n, int64_t m, int directed, const int64_t* off, const uint32_t* nb,
            const int64_t* in_off, const uint32_t* in_nb, std::string* err) {
  FILE* f = fopen(path, "wb");
  if (!f) {
    *err = std::string("cannot open file for writing: ") + path;
    return 2;
  }
  Stager st;
  unsigned char hdr[22];
  memcpy(hdr, "GAPB", 4);
  hdr[4] = 1;
  hdr[5] = directed ? 1 : 0;
  const uint64_t un = (uint64_t)n, um = (uint64_t)m;
  memcpy(hdr + 6, &un, 8);
  memcpy(hdr + 14, &um, 8);
  std::string e;
  if (st.init() != cudaSuccess) e = "cannot allocate staging buffers";
  if (e.empty() && fwrite(hdr, 1, 22, f) != 22) e = "write failed";
  if (e.empty()) e = stream_out(f, st, (const char*)off, (size_t)(n + 1) * 8);
  if (e.empty()) e = stream_out(f, st, (const char*)nb, (size_t)m * 4);
  if (e.empty() && directed) e = stream_out(f, st, (const char*)in_off, (size_t)(n + 1) * 8);
  if (e.empty() && directed) e = stream_out(f, st, (const char*)in_nb, (size_t)m * 4);
  if (fclose(f) != 0 && e.empty()) e = "write failed";
  if (!e.empty()) {
    *err = std::string(path) + ": " + e;
    return 4;
  }
  return 0;
}

}  // namespace gk
