// fnv_pipeline.cuh -- the per-step row digest (fnv_kernels.cuh, nibble
// decomposition) with its buffers and its captured graph, for any engine
// whose current row is described by a RingArgs: positions x[buf] and
// velocities v[buf] in ID order, the row starting at id (N - W) mod N, with
// buf and W read from the device control block at run time.  Used by the
// single-GPU ring (engine.cu: the live state) and the grid engine (grid.cu:
// its compacted rank-ordered row, W = 0).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "fnv_kernels.cuh"

namespace nb200 {

class FnvRowDigest {
 public:
  FnvRowDigest() = default;
  FnvRowDigest(const FnvRowDigest&) = delete;
  FnvRowDigest& operator=(const FnvRowDigest&) = delete;
  ~FnvRowDigest() {
    if (graph_) cudaGraphExecDestroy(graph_);
    for (uint8_t* p : maps_) cudaFree(p);
    for (uint8_t* p : pre_) cudaFree(p);
    for (uint8_t* p : lb_) cudaFree(p);
    cudaFree(top_);
    cudaFree(lo4_);
    cudaFree(hi4_);
    cudaFree(sub_);
    for (int b = 0; b < 2; ++b) {
      cudaFree(A_[b]);
      cudaFree(D_[b]);
    }
    cudaFree(hash_);
  }

  bool started() const { return hash_ != nullptr; }

  // Folds the row into the device digest: one graph launch.  The first call
  // allocates for n cars (vbytes-byte velocities), seeds the digest with
  // `host_hash` and captures the graph over `args` (which must keep
  // describing the row: the kernels read buf and W from args.ctl).  Returns
  // the kernel launches the graph made.
  uint32_t fold(const RingArgs& args, uint32_t n, int vbytes, cudaStream_t stream, uint64_t host_hash) {
    if (!hash_) start(n, vbytes, host_hash);
    if (!graph_) {
      cudaGraph_t g;
      ck(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
      launches_ = enqueue(args, n, stream);
      ck(cudaStreamEndCapture(stream, &g), "cudaStreamEndCapture");
      ck(cudaGraphInstantiate(&graph_, g, 0), "cudaGraphInstantiate");
      ck(cudaGraphDestroy(g), "cudaGraphDestroy");
    }
    ck(cudaGraphLaunch(graph_, stream), "cudaGraphLaunch(digest)");
    return launches_;
  }

  // The same fold without a graph, for a row of n <= capacity values whose
  // length changes from call to call (checksum batches of small rings: the
  // rows of k steps laid end to end); the first call sizes the buffers for
  // `capacity` values.
  uint32_t fold_direct(const RingArgs& args, uint32_t n, uint32_t capacity, int vbytes, cudaStream_t stream,
                       uint64_t host_hash) {
    if (!hash_) start(capacity, vbytes, host_hash);
    if (n > n_) throw std::logic_error("digest row longer than its capacity");
    return enqueue(args, n, stream);
  }

  // The device digest into *out (synchronises the stream); false before the
  // first fold.
  bool pull(cudaStream_t stream, uint64_t* out) const {
    if (!hash_) return false;
    unsigned long long h = 0;
    ck(cudaMemcpyAsync(&h, hash_, 8, cudaMemcpyDeviceToHost, stream), "cudaMemcpyAsync(digest)");
    ck(cudaStreamSynchronize(stream), "cudaStreamSynchronize(digest)");
    *out = h;
    return true;
  }

 private:
  static void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  }

  void start(uint32_t n, int vbytes, uint64_t host_hash) {
    n_ = n;
    vbytes_ = vbytes;
    alloc();
    ck(cudaMalloc(&hash_, 8), "cudaMalloc(digest)");
    const unsigned long long h = host_hash;
    ck(cudaMemcpy(hash_, &h, 8, cudaMemcpyHostToDevice), "cudaMemcpy(digest)");
  }

  // slots and chunks of a row of n values (fnv_row)
  static uint32_t slots_of(uint32_t n) {
    const uint32_t nu = (n + kFnvSlot - 1) / kFnvSlot;
    return 2 * ((nu + 1 + kFnvSlotsPerChunk - 1) / kFnvSlotsPerChunk * kFnvSlotsPerChunk);
  }

  void alloc() {
    nslots_ = slots_of(n_);
    chunks_ = nslots_ / kFnvSlotsPerChunk;
    for (uint32_t m = chunks_;;) {
      uint8_t *maps = nullptr, *pre = nullptr, *lb = nullptr;
      ck(cudaMalloc(&maps, size_t(m) * 16), "cudaMalloc(maps)");
      ck(cudaMalloc(&pre, size_t(m) * 16), "cudaMalloc(pre)");
      ck(cudaMalloc(&lb, m), "cudaMalloc(lb)");
      maps_.push_back(maps);
      pre_.push_back(pre);
      lb_.push_back(lb);
      count_.push_back(m);
      if (m <= 256) break;
      m = (m + 255) / 256;
    }
    ck(cudaMalloc(&top_, 16), "cudaMalloc(top)");
    ck(cudaMalloc(&lo4_, chunks_), "cudaMalloc(lo4)");
    ck(cudaMalloc(&hi4_, chunks_), "cudaMalloc(hi4)");
    ck(cudaMalloc(&sub_, size_t(chunks_) * (kFnvSlotsPerChunk - 1) * 16), "cudaMalloc(sub)");
    for (int b = 0; b < 2; ++b) {
      ck(cudaMalloc(&A_[b], size_t(nslots_) * 8), "cudaMalloc(A)");
      ck(cudaMalloc(&D_[b], size_t(nslots_) * 8), "cudaMalloc(D)");
    }
  }

  // Composition tree over maps_[0] (filled by pass A or B; `chunks` maps):
  // up, then down from the digest's nibble at `shift`, the level-0 result
  // into `out`.
  uint32_t tree(uint32_t chunks, int shift, uint8_t* out, cudaStream_t stream) {
    uint32_t nl = 0;
    std::vector<uint32_t> count;
    for (uint32_t m = chunks;; m = (m + 255) / 256) {
      count.push_back(m);
      if (m <= 256) break;
    }
    const size_t levels = count.size();
    for (size_t i = 0; i < levels; ++i, ++nl) {
      const uint32_t groups = (count[i] + 255) / 256;
      fnv_up16_kernel<<<(groups + kUpGroups - 1) / kUpGroups, 16 * kUpGroups, 0, stream>>>(
          maps_[i], count[i], pre_[i], i + 1 < levels ? maps_[i + 1] : top_);
    }
    for (size_t i = levels; i-- > 0; ++nl) {
      fnv_down16_kernel<<<(count[i] + 255) / 256, 256, 0, stream>>>(
          pre_[i], count[i], i + 1 < levels ? lb_[i + 1] : nullptr, hash_, shift, i == 0 ? out : lb_[i]);
    }
    return nl;
  }

  uint32_t enqueue(const RingArgs& args, uint32_t n, cudaStream_t stream) {
    uint32_t nl = 0;
    const uint32_t nslots = slots_of(n), chunks = nslots / kFnvSlotsPerChunk;
    const int cgrid = static_cast<int>((chunks + kFnvTPB - 1) / kFnvTPB);
    if (vbytes_ == 1) fnv_nib_kernel<uint8_t, 0><<<cgrid, kFnvTPB, 0, stream>>>(args, nullptr, maps_[0], nullptr);
    else fnv_nib_kernel<uint32_t, 0><<<cgrid, kFnvTPB, 0, stream>>>(args, nullptr, maps_[0], nullptr);
    nl += 1 + tree(chunks, 0, lo4_, stream);
    if (vbytes_ == 1) fnv_nib_kernel<uint8_t, 1><<<cgrid, kFnvTPB, 0, stream>>>(args, lo4_, maps_[0], sub_);
    else fnv_nib_kernel<uint32_t, 1><<<cgrid, kFnvTPB, 0, stream>>>(args, lo4_, maps_[0], sub_);
    nl += 1 + tree(chunks, 4, hi4_, stream);
    const int sgrid = static_cast<int>((nslots + kFnvTPB - 1) / kFnvTPB);
    if (vbytes_ == 1)
      fnv_exact_kernel<uint8_t><<<sgrid, kFnvTPB, 0, stream>>>(args, lo4_, hi4_, sub_, A_[0], D_[0]);
    else
      fnv_exact_kernel<uint32_t><<<sgrid, kFnvTPB, 0, stream>>>(args, lo4_, hi4_, sub_, A_[0], D_[0]);
    ++nl;
    int in = 0;
    for (uint32_t m = nslots; m > 1; m = (m + 255) / 256, in ^= 1, ++nl)
      fnv_affine_reduce<<<(m + 255) / 256, 256, 0, stream>>>(A_[in], D_[in], m, A_[in ^ 1], D_[in ^ 1]);
    fnv_affine_apply<<<1, 1, 0, stream>>>(A_[in], D_[in], hash_);
    ck(cudaGetLastError(), "digest kernels");
    return nl + 1;
  }

  uint32_t n_ = 0, nslots_ = 0, chunks_ = 0, launches_ = 0;
  int vbytes_ = 1;
  unsigned long long* hash_ = nullptr;
  std::vector<uint8_t*> maps_;   // level 0: chunk maps; level i+1: groups of 256 of level i
  std::vector<uint8_t*> pre_;    // prefix tables per level
  std::vector<uint8_t*> lb_;     // incoming nibble per map, levels >= 1
  std::vector<uint32_t> count_;  // maps per level
  uint8_t* lo4_ = nullptr;       // incoming low nibble per chunk (pass A)
  uint8_t* hi4_ = nullptr;       // incoming high nibble per chunk (pass B)
  uint8_t* sub_ = nullptr;       // bytes at the slot boundaries inside a chunk (pass B)
  uint8_t* top_ = nullptr;       // the top group's composed map (unused)
  unsigned long long* A_[2] = {nullptr, nullptr};
  unsigned long long* D_[2] = {nullptr, nullptr};
  cudaGraphExec_t graph_ = nullptr;
};

}  // namespace nb200
