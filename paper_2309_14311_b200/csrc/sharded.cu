// sharded.cu -- ShardedRing: one ring split into contiguous car segments
// (DESIGN.md section 6).
//
// Shard g holds global ids [lo_g, lo_g+1) with lo_g = floor(g*N/G) -- the
// reference's own block formula (src/engine.cpp:31-42) -- plus a 16-car halo
// inline after its cars.  Each launch advances every shard K steps with the
// temporal-blocked kernel (tb_kernel.cuh, sharded mode); the shards then
// exchange one 2 KB record each (first cars + the origin-cone slots they
// own) and every shard plans the next launch from the same window
// (shard_kernels.cuh).  Default exchange: the step kernel's last block
// stores the record into every shard's HBM (peer pointers; IPC-mapped
// across processes) and raises a flag the plan kernel waits on.  Collective
// exchange (construction, set_state, or NASCH_B200_XCHG=collective): pack ->
// NCCL all-gather (one process per GPU) or stream-ordered peer copies
// (shards of one process) -> plan.  Shards of one process may share ONE GPU,
// which is how the sharded path is tested bit-exactly here.  Draws are
// indexed by global rank, so the trajectory is bit-identical for any shard
// count, as the reference's is for any OpenMP team size.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: the library is opened at run time

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <exception>
#include <vector>

#include "engine.hpp"
#include "host_simd.hpp"
#include "minstd.hpp"
#include "fnv_kernels.cuh"
#include "shard_kernels.cuh"
#include "step_kernels.cuh"
#include "tb_config.hpp"
#include "tb_kernel.cuh"

namespace nb200 {

namespace {

void check_s(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  }
}
#define CKS(call) check_s((call), #call)

constexpr int kTPB = kTbTPB;
constexpr int kCPT = kTbCPT;
constexpr int kHalo = kTbHalo;
constexpr uint32_t kLoad = kTbLoad;
constexpr uint32_t kStore = kTbStore;

// NCCL entry points, resolved from libnccl.so.2 at first use (no link-time
// dependency: the library loads on machines without NCCL).
struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;

  static NcclApi& get() {
    static NcclApi api;
    if (!api.handle) api.open();
    return api;
  }
  // The NCCL already in the process if there is one (e.g. PyTorch's, which
  // may be newer than the system's: loading the system copy first would
  // shadow it -- same soname -- for a later `import torch`), else
  // NASCH_B200_NCCL_LIB, else the default search path.  Opened RTLD_LOCAL:
  // our lookups go through dlsym, nothing is exported to the process.
  void open() {
    handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!handle) {
      const char* env = std::getenv("NASCH_B200_NCCL_LIB");
      if (env && *env) handle = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    }
    if (!handle) handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!handle) throw std::runtime_error(std::string("cannot load libnccl.so.2: ") + dlerror());
    get_unique_id = reinterpret_cast<decltype(get_unique_id)>(dlsym(handle, "ncclGetUniqueId"));
    comm_init_rank = reinterpret_cast<decltype(comm_init_rank)>(dlsym(handle, "ncclCommInitRank"));
    all_gather = reinterpret_cast<decltype(all_gather)>(dlsym(handle, "ncclAllGather"));
    all_reduce = reinterpret_cast<decltype(all_reduce)>(dlsym(handle, "ncclAllReduce"));
    broadcast = reinterpret_cast<decltype(broadcast)>(dlsym(handle, "ncclBroadcast"));
    comm_destroy = reinterpret_cast<decltype(comm_destroy)>(dlsym(handle, "ncclCommDestroy"));
    error_string = reinterpret_cast<decltype(error_string)>(dlsym(handle, "ncclGetErrorString"));
    if (!get_unique_id || !comm_init_rank || !all_gather || !all_reduce || !broadcast || !comm_destroy ||
        !error_string)
      throw std::runtime_error("libnccl.so.2 lacks a required symbol");
  }
  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess) throw std::runtime_error(std::string("NCCL error in ") + what + ": " + error_string(r));
  }
};

}  // namespace

bool ShardedRing::can_shard(const SimParams& p, unsigned shards) {
  try {
    p.validate();
  } catch (...) {
    return false;
  }
  if (shards < 2 || p.road_length > 2147483647ull) return false;
  const uint64_t vmax_eff = std::min<uint64_t>(p.v_max, p.road_length - 1);
  const char* ks = std::getenv("NASCH_B200_K");
  const long kreq = ks && *ks ? std::strtol(ks, nullptr, 10) : kPlanMax;
  uint64_t K = static_cast<uint64_t>(std::max<long>(1, std::min<long>(kreq, std::min(kPlanMax, kTbHalo))));
  K = std::min<uint64_t>(K, kConeMax / (vmax_eff + 1));
  const uint64_t min_seg = p.car_count / shards;  // floor partition: smallest segment
  return K >= 2 && p.road_length > K * vmax_eff && p.car_count >= K * (vmax_eff + 1) && min_seg >= 64;
}

void nccl_unique_id(void* out128) {
  NcclApi& api = NcclApi::get();
  ncclUniqueId id;
  api.check(api.get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof id);
}

struct ShardedRing::Impl {
  struct Shard {
    uint32_t g = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_packed = nullptr, ev_done = nullptr;
    uint32_t gofs = 0, nl = 0, npad = 0;
    int grid = 1;
    uint32_t* x[2] = {nullptr, nullptr};
    void* v[2] = {nullptr, nullptr};
    Ctl* ctl = nullptr;
    StepRec* rec = nullptr;
    uint32_t* blkpow = nullptr;
    uint32_t* thrpow = nullptr;
    uint32_t* send = nullptr;
    uint32_t* recv = nullptr;
    // peer-memory exchange: [kFlagWords flags][2][G][kXchgWords] receive area
    uint32_t* xarea = nullptr;
    void** ptab = nullptr;            // device [2G]: every shard's rec area, then flag array
    std::vector<void*> ipc_opened;    // peer areas mapped with cudaIpcOpenMemHandle
    uint32_t* lo_dev = nullptr;
    RingArgs args{};
    StepRec* hrec = nullptr;
    Ctl* hctl = nullptr;
    // on-device checksum: chunk tables of this shard's pieces of the row
    unsigned long long* fT[2] = {nullptr, nullptr};
    unsigned long long* fP[2] = {nullptr, nullptr};
    unsigned long long* hpiece = nullptr;  // pinned: up to 4 pieces x (256 + 1)
    // pinned staging of this shard's segment: set_state narrowing and
    // segment snapshots (allocated on first use)
    uint32_t* hx_stage = nullptr;
    void* hv_stage = nullptr;
    // device copy of the segment for an asynchronous segment snapshot
    uint32_t* snap_x = nullptr;
    void* snap_v = nullptr;
  };

  SimParams params;
  uint32_t n = 0, L = 0, vmax_eff = 0, K = 1;
  int vbytes = 1;
  unsigned G = 1;
  std::vector<uint32_t> lo;  // G+1 segment starts
  bool use_nccl = false;
  ncclComm_t comm = nullptr;
  // Steady-state exchange: records pushed into peer HBM by the step
  // kernel's last block (tb_body<PUSH>), flags awaited by the plan kernel.
  // Construction / set_state always exchange through the collective path
  // (peer copies or NCCL all-gather), which also absorbs any skew between
  // the ranks' host threads.
  bool p2p = false;
  uint32_t xseq = 0;  // launches published through the peer exchange
  // One process per GPU: this rank's per-step crossing counts and the
  // planned (whole-ring) counts of drained steps not yet checked; their sum
  // over the ranks must equal the plan (verify_ranks, at every collective
  // synchronisation point).
  // The drained steps' local velocity sums go through the same all-reduce,
  // so every rank ends up with the WHOLE ring's per-step series.
  std::vector<uint32_t> pend_c, pend_plan;
  std::vector<uint64_t> pend_sv;
  uint64_t pend_first = 0;
  uint64_t* dcheck = nullptr;  // device scratch for the all-reduce
  size_t dcheck_cap = 0;
  // One process per GPU: a failure detected outside a collective call
  // (drain) is kept here and raised on EVERY rank at the next collective
  // synchronisation point (verify_ranks), so no rank is left waiting in a
  // collective its peer never reaches.  Once raised, the engine is
  // poisoned: every later call repeats the error.
  std::string local_err, poisoned;
  // asynchronous segment snapshot (one process per GPU)
  cudaStream_t snap_stream = nullptr;
  cudaEvent_t snap_ready = nullptr;
  std::thread snap_thread;
  std::exception_ptr snap_error;
  unsigned long long* dhash_x = nullptr;  // checksum piece exchange (one process per GPU)
  std::vector<Shard> sh;  // shards held by this process
  bool exchanged_once = false;
  ~Impl();

  uint64_t steps_done = 0, drained = 0, series_base = 0;
  uint64_t hash = kFnvBasis;
  bool checksum_on = true;
  uint64_t sumv0 = 0;
  std::vector<uint64_t> sumv_host, wraps_host;
  uint32_t W_host = 0, buf_host = 0;
  uint64_t launches = 0;
  std::vector<Frame> frames;
  uint32_t* hx = nullptr;  // global ID-ordered staging (in-process mode)
  void* hv = nullptr;

  void init_common(const SimParams& p, unsigned world) {
    p.validate();
    params = p;
    if (p.road_length > 2147483647ull)
      throw std::invalid_argument("length above 2^31-1 is not supported by the B200 engine");
    if (world < 1) throw std::invalid_argument("worker count must be at least 1");
    n = static_cast<uint32_t>(p.car_count);
    L = static_cast<uint32_t>(p.road_length);
    vmax_eff = static_cast<uint32_t>(std::min<uint64_t>(p.v_max, p.road_length - 1));
    vbytes = vmax_eff <= 255 ? 1 : 4;
    G = world;
    const char* ks = std::getenv("NASCH_B200_K");
    long kreq = ks && *ks ? std::strtol(ks, nullptr, 10) : kPlanMax;
    K = static_cast<uint32_t>(std::max<long>(1, std::min<long>(kreq, std::min(kPlanMax, kTbHalo))));
    K = std::min<uint32_t>(K, kConeMax / (vmax_eff + 1));
    lo.resize(G + 1);
    for (unsigned g = 0; g <= G; ++g) lo[g] = static_cast<uint32_t>(uint64_t(g) * n / G);
    uint32_t min_seg = n;
    for (unsigned g = 0; g < G; ++g) min_seg = std::min(min_seg, lo[g + 1] - lo[g]);
    if (K < 2 || uint64_t(L) <= uint64_t(K) * vmax_eff || uint64_t(n) < uint64_t(K) * (vmax_eff + 1) ||
        min_seg < 64)
      throw std::invalid_argument("ring too small to shard (need >= 64 cars per shard and "
                                  "length > 2*vmax)");
    int ndev = 0;
    const cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
      throw std::runtime_error(std::string("no CUDA device available for the B200 engine (") +
                               cudaGetErrorString(e) + ")");
  }

  template <typename VT>
  void occupancy(int* per_sm) {
    CKS(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, nasch_tb_kernel<VT, kTPB, kCPT, kHalo, kTbWT>,
                                                      kTPB, 0));
  }

  void make_shard(uint32_t g, int device) {
    sh.emplace_back();  // registered first: ~Impl frees whatever gets allocated
    Shard& s = sh.back();
    s.g = g;
    s.device = device;
    CKS(cudaSetDevice(device));
    s.gofs = lo[g];
    s.nl = lo[g + 1] - lo[g];
    const uint32_t ntiles = (s.nl + kStore - 1) / kStore;
    s.npad = ntiles * kStore + kLoad + 64;
    CKS(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    CKS(cudaEventCreateWithFlags(&s.ev_packed, cudaEventDisableTiming));
    CKS(cudaEventCreateWithFlags(&s.ev_done, cudaEventDisableTiming));
    for (int b = 0; b < 2; ++b) {
      CKS(cudaMalloc(&s.x[b], size_t(s.npad) * 4));
      CKS(cudaMalloc(&s.v[b], size_t(s.npad) * vbytes));
    }
    CKS(cudaMalloc(&s.ctl, sizeof(Ctl)));
    CKS(cudaMalloc(&s.rec, sizeof(StepRec) * kRecCap));
    CKS(cudaMalloc(&s.send, kXchgWords * 4));
    CKS(cudaMalloc(&s.recv, size_t(G) * kXchgWords * 4));
    const size_t xbytes = (kFlagWords + 2 * size_t(G) * kXchgWords) * 4;
    CKS(cudaMalloc(&s.xarea, xbytes));
    CKS(cudaMemset(s.xarea, 0, xbytes));
    CKS(cudaMalloc(&s.ptab, 2 * size_t(G) * sizeof(void*)));
    CKS(cudaMalloc(&s.lo_dev, (G + 1) * 4));
    CKS(cudaMemcpy(s.lo_dev, lo.data(), (G + 1) * 4, cudaMemcpyHostToDevice));
    CKS(cudaMallocHost(&s.hrec, sizeof(StepRec) * kRecCap));
    CKS(cudaMallocHost(&s.hctl, sizeof(Ctl)));
    int sms = 0, per_sm = 0;
    CKS(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    if (vbytes == 1) occupancy<uint8_t>(&per_sm); else occupancy<uint32_t>(&per_sm);
    const char* we = std::getenv("NASCH_B200_WAVES");
    const long waves = std::max<long>(1, we && *we ? std::strtol(we, nullptr, 10) : kTbWaves);
    s.grid = static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>(ntiles, uint64_t(sms) * std::max(per_sm, 1) * uint64_t(waves))));
    std::vector<uint32_t> blk(s.grid), thr(kTPB);
    const uint32_t a_tile = powmod(kA, kStore);
    blk[0] = 1;
    for (int b = 1; b < s.grid; ++b) blk[b] = mulmod(blk[b - 1], a_tile);
    for (int t = 0; t < kTPB; ++t) thr[t] = powmod(kA, TbLarge::offset(t));
    CKS(cudaMalloc(&s.blkpow, blk.size() * 4));
    CKS(cudaMalloc(&s.thrpow, thr.size() * 4));
    CKS(cudaMemcpy(s.blkpow, blk.data(), blk.size() * 4, cudaMemcpyHostToDevice));
    CKS(cudaMemcpy(s.thrpow, thr.data(), thr.size() * 4, cudaMemcpyHostToDevice));
    RingArgs& a = s.args;
    a.x[0] = s.x[0];
    a.x[1] = s.x[1];
    a.v[0] = s.v[0];
    a.v[1] = s.v[1];
    a.n = n;
    a.L = L;
    a.vmax = vmax_eff;
    a.tp = deceleration_threshold(params.p);
    a.s0 = seeded(params.seed);
    a.an = powmod(kA, n);
    a.an_inv = powmod(kA, kOrder - (n % kOrder));
    a.a1 = powmod(kA, (1 + kOrder - (n % kOrder)) % kOrder);
    a.g = powmod(kA, uint64_t(s.grid) * kStore);
    a.kplan = K;
    a.nl = s.nl;
    a.gofs = s.gofs;
    a.agofs = powmod(kA, s.gofs);
    a.sharded = 1;
    a.blkpow = s.blkpow;
    a.thrpow = s.thrpow;
    a.ctl = s.ctl;
    a.rec = s.rec;
    const int ib = std::max(1, std::min<int>((s.npad + kTPB - 1) / kTPB, 4096));
    for (int b = 0; b < 2; ++b) {
      if (vbytes == 1)
        shard_init_kernel<uint8_t><<<ib, kTPB, 0, s.stream>>>(s.x[b], static_cast<uint8_t*>(s.v[b]), s.nl, s.npad, s.gofs, n, L);
      else
        shard_init_kernel<uint32_t><<<ib, kTPB, 0, s.stream>>>(s.x[b], static_cast<uint32_t*>(s.v[b]), s.nl, s.npad, s.gofs, n, L);
    }
    CKS(cudaGetLastError());
  }

  // ---- peer-memory exchange setup ------------------------------------
  static bool p2p_wanted() {
    const char* e = std::getenv("NASCH_B200_XCHG");
    return !(e && std::strcmp(e, "collective") == 0);
  }

  // Shards of this process: plain device pointers, peer access enabled
  // between distinct GPUs (NVLink); any pair that cannot map the other's
  // memory keeps the collective exchange.
  void setup_p2p_local() {
    if (!p2p_wanted() || G > kFlagWords) return;
    for (const Shard& a : sh)
      for (const Shard& b : sh) {
        if (a.device == b.device) continue;
        int ok = 0;
        CKS(cudaDeviceCanAccessPeer(&ok, a.device, b.device));
        if (!ok) return;
      }
    for (const Shard& a : sh)
      for (const Shard& b : sh) {
        if (a.device == b.device) continue;
        CKS(cudaSetDevice(a.device));
        const cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else CKS(e);
      }
    std::vector<void*> tab(2 * size_t(G));
    for (unsigned h = 0; h < G; ++h) {
      tab[h] = sh[h].xarea + kFlagWords;
      tab[G + h] = sh[h].xarea;
    }
    for (Shard& s : sh) {
      CKS(cudaSetDevice(s.device));
      CKS(cudaMemcpy(s.ptab, tab.data(), tab.size() * sizeof(void*), cudaMemcpyHostToDevice));
    }
    p2p = true;
  }

  // One shard per process: the ranks swap cudaIpcMemHandle_t of their
  // receive areas over the NCCL communicator, map every peer's area, and
  // agree (a second all-gather) to switch only if every rank mapped every
  // peer.
  void setup_p2p_ipc() {
    if (!p2p_wanted() || G > kFlagWords) return;
    Shard& s = sh[0];
    NcclApi& api = NcclApi::get();
    CKS(cudaSetDevice(s.device));
    constexpr size_t kSlot = 128;  // one cudaIpcMemHandle_t (64 B) + status, per rank
    static_assert(sizeof(cudaIpcMemHandle_t) <= kSlot - 8, "handle slot");
    std::vector<unsigned char> mine(kSlot, 0), all(kSlot * G, 0);
    cudaIpcMemHandle_t h{};
    const bool got = cudaIpcGetMemHandle(&h, s.xarea) == cudaSuccess;
    if (!got) cudaGetLastError();
    std::memcpy(mine.data(), &h, sizeof h);
    mine[kSlot - 1] = got ? 1 : 0;
    unsigned char* dbuf = nullptr;
    CKS(cudaMalloc(&dbuf, kSlot * (G + 1)));
    struct Free {
      unsigned char* p;
      ~Free() { cudaFree(p); }
    } guard{dbuf};
    CKS(cudaMemcpy(dbuf, mine.data(), kSlot, cudaMemcpyHostToDevice));
    api.check(api.all_gather(dbuf, dbuf + kSlot, kSlot, ncclUint8, comm, s.stream), "ncclAllGather(ipc)");
    CKS(cudaStreamSynchronize(s.stream));
    CKS(cudaMemcpy(all.data(), dbuf + kSlot, kSlot * G, cudaMemcpyDeviceToHost));
    std::vector<void*> tab(2 * size_t(G), nullptr);
    bool ok = true;
    for (unsigned r = 0; r < G && ok; ++r) {
      if (r == s.g) {
        tab[r] = s.xarea;
        continue;
      }
      if (!all[kSlot * r + kSlot - 1]) {
        ok = false;
        break;
      }
      cudaIpcMemHandle_t ph;
      std::memcpy(&ph, all.data() + kSlot * r, sizeof ph);
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, ph, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = false;
        break;
      }
      s.ipc_opened.push_back(p);
      tab[r] = p;
    }
    // agree: every rank switches, or none does
    const uint32_t flag = ok ? 1u : 0u;
    CKS(cudaMemcpy(dbuf, &flag, 4, cudaMemcpyHostToDevice));
    api.check(api.all_gather(dbuf, dbuf + kSlot, 4, ncclUint8, comm, s.stream), "ncclAllGather(ipc ok)");
    CKS(cudaStreamSynchronize(s.stream));
    std::vector<uint32_t> oks(G);
    CKS(cudaMemcpy(oks.data(), dbuf + kSlot, 4 * size_t(G), cudaMemcpyDeviceToHost));
    for (uint32_t v : oks) ok = ok && v == 1u;
    if (!ok) return;  // the opened mappings are released by ~Impl
    std::vector<void*> dev(2 * size_t(G));
    for (unsigned r = 0; r < G; ++r) {
      dev[r] = static_cast<uint32_t*>(tab[r]) + kFlagWords;
      dev[G + r] = tab[r];
    }
    CKS(cudaMemcpy(s.ptab, dev.data(), dev.size() * sizeof(void*), cudaMemcpyHostToDevice));
    p2p = true;
  }

  // ---- the per-launch pipeline ---------------------------------------
  void pack_all() {
    for (Shard& s : sh) {
      CKS(cudaSetDevice(s.device));
      if (!use_nccl && exchanged_once) {
        // nobody may still be copying our previous record
        for (const Shard& o : sh) CKS(cudaStreamWaitEvent(s.stream, o.ev_done, 0));
      }
      if (vbytes == 1) shard_pack_kernel<uint8_t><<<1, kConeMax, 0, s.stream>>>(s.args, s.send);
      else shard_pack_kernel<uint32_t><<<1, kConeMax, 0, s.stream>>>(s.args, s.send);
      CKS(cudaGetLastError());
      CKS(cudaEventRecord(s.ev_packed, s.stream));
      ++launches;
    }
  }

  void exchange_all() {
    const size_t bytes = size_t(kXchgWords) * 4;
    if (use_nccl) {
      NcclApi& api = NcclApi::get();
      for (Shard& s : sh) {
        CKS(cudaSetDevice(s.device));
        api.check(api.all_gather(s.send, s.recv, bytes, ncclUint8, comm, s.stream), "ncclAllGather");
      }
      return;
    }
    for (Shard& s : sh) {
      CKS(cudaSetDevice(s.device));
      for (const Shard& o : sh) {
        CKS(cudaStreamWaitEvent(s.stream, o.ev_packed, 0));
        CKS(cudaMemcpyPeerAsync(s.recv + size_t(o.g) * kXchgWords, s.device, o.send, o.device, bytes,
                                s.stream));
      }
    }
  }

  void plan_all() {
    for (Shard& s : sh) {
      CKS(cudaSetDevice(s.device));
      if (vbytes == 1)
        shard_plan_kernel<uint8_t><<<1, kConeMax, 0, s.stream>>>(s.args, s.recv, s.lo_dev, G, s.g, nullptr, 0u);
      else
        shard_plan_kernel<uint32_t><<<1, kConeMax, 0, s.stream>>>(s.args, s.recv, s.lo_dev, G, s.g, nullptr, 0u);
      CKS(cudaGetLastError());
      CKS(cudaEventRecord(s.ev_done, s.stream));
      ++launches;
    }
    exchanged_once = true;
  }

  void exchange_and_plan() {
    pack_all();
    exchange_all();
    plan_all();
  }

  void launch(uint32_t k) {
    if (p2p) {
      launch_p2p(k);
      steps_done += k;
      return;
    }
    for (Shard& s : sh) {
      CKS(cudaSetDevice(s.device));
      if (vbytes == 1) nasch_tb_kernel<uint8_t, kTPB, kCPT, kHalo, kTbWT><<<s.grid, kTPB, 0, s.stream>>>(s.args, k);
      else nasch_tb_kernel<uint32_t, kTPB, kCPT, kHalo, kTbWT><<<s.grid, kTPB, 0, s.stream>>>(s.args, k);
      CKS(cudaGetLastError());
      ++launches;
    }
    exchange_and_plan();
    steps_done += k;
  }

  // Two kernels per launch and no host-side exchange: the step kernel
  // publishes the record into every shard's HBM; the plan kernel waits on
  // the flags.  Shards of one process additionally order the plan after
  // every shard's step kernel with events, so no kernel ever waits on a
  // kernel that might not be running (several shards may share one GPU).
  void launch_p2p(uint32_t k) {
    const uint32_t seq = ++xseq;
    for (Shard& s : sh) {
      CKS(cudaSetDevice(s.device));
      XchgArgs xa;
      xa.rec = reinterpret_cast<uint32_t* const*>(s.ptab);
      xa.flag = reinterpret_cast<uint32_t* const*>(s.ptab + G);
      xa.g = s.g;
      xa.G = G;
      xa.seq = seq;
      if (vbytes == 1)
        nasch_tb_push_kernel<uint8_t, kTPB, kCPT, kHalo, kTbWT><<<s.grid, kTPB, 0, s.stream>>>(s.args, k, xa);
      else
        nasch_tb_push_kernel<uint32_t, kTPB, kCPT, kHalo, kTbWT><<<s.grid, kTPB, 0, s.stream>>>(s.args, k, xa);
      CKS(cudaGetLastError());
      if (!use_nccl) CKS(cudaEventRecord(s.ev_packed, s.stream));
      ++launches;
    }
    for (Shard& s : sh) {
      CKS(cudaSetDevice(s.device));
      if (!use_nccl)
        for (const Shard& o : sh) CKS(cudaStreamWaitEvent(s.stream, o.ev_packed, 0));
      const uint32_t* rec = s.xarea + kFlagWords;
      if (vbytes == 1)
        shard_plan_kernel<uint8_t><<<1, kConeMax, 0, s.stream>>>(s.args, rec, s.lo_dev, G, s.g, s.xarea, seq);
      else
        shard_plan_kernel<uint32_t><<<1, kConeMax, 0, s.stream>>>(s.args, rec, s.lo_dev, G, s.g, s.xarea, seq);
      CKS(cudaGetLastError());
      CKS(cudaEventRecord(s.ev_done, s.stream));
      ++launches;
    }
  }

  void reset_ctl() {
    for (Shard& s : sh) {
      CKS(cudaSetDevice(s.device));
      Ctl c{};
      c.t = steps_done;
      c.W = 0;
      c.buf = buf_host;
      c.E = mulmod(seeded(params.seed), powmod(kA, draw_exponent(steps_done, n, 0)));
      c.E2 = mulmod(c.E, s.args.an_inv);
      *s.hctl = c;
      CKS(cudaMemcpyAsync(s.ctl, s.hctl, sizeof(Ctl), cudaMemcpyHostToDevice, s.stream));
      CKS(cudaMemsetAsync(s.rec, 0, sizeof(StepRec) * kRecCap, s.stream));
    }
    W_host = 0;
    exchange_and_plan();
  }

  void sync_all() {
    for (Shard& s : sh) {
      CKS(cudaSetDevice(s.device));
      CKS(cudaStreamSynchronize(s.stream));
    }
  }

  // Per-step records of [drained, steps_done), summed over local shards.
  // Local only (no collective): with one process per GPU the records wait
  // in pend_* for verify_ranks, and any inconsistency is deferred there.
  void drain() {
    if (drained == steps_done) return;
    const uint64_t first = drained, count = steps_done - drained;
    for (Shard& s : sh) {
      CKS(cudaSetDevice(s.device));
      uint64_t done = 0;
      while (done < count) {
        const uint64_t slot = (first + done) % kRecCap;
        const uint64_t seg = std::min<uint64_t>(count - done, kRecCap - slot);
        CKS(cudaMemcpyAsync(s.hrec + done, s.rec + slot, seg * sizeof(StepRec), cudaMemcpyDeviceToHost, s.stream));
        done += seg;
      }
      CKS(cudaMemcpyAsync(s.hctl, s.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s.stream));
    }
    sync_all();
    for (const Shard& s : sh) {
      std::string e;
      if (s.hctl->err == 3u)
        e = "peer exchange timed out on shard " + std::to_string(s.g) +
            " (a rank stopped publishing; engine state is invalid)";
      else if (s.hctl->t != steps_done)
        e = "device step counter out of sync on shard " + std::to_string(s.g);
      else if (s.hctl->W != sh[0].hctl->W || s.hctl->buf != sh[0].hctl->buf)
        e = "shards disagree on the rank offset";
      if (e.empty()) continue;
      if (!use_nccl) throw std::runtime_error(e);
      if (local_err.empty()) local_err = e;
    }
    for (uint64_t k = 0; k < count; ++k) {
      uint64_t sv = 0, c = 0;
      for (const Shard& s : sh) {
        sv += s.hrec[k].sumv;
        c += s.hrec[k].c;
      }
      if (use_nccl) {
        if (pend_c.empty()) pend_first = first + k;
        pend_c.push_back(static_cast<uint32_t>(c));
        pend_plan.push_back(sh[0].hrec[k].cplan);
        pend_sv.push_back(sv);
        continue;
      }
      if (c != sh[0].hrec[k].cplan)
        throw std::runtime_error("origin-cone plan contradicted at step " + std::to_string(first + k) +
                                 " (engine state is invalid)");
      sumv_host.push_back(sv);
      wraps_host.push_back(c);
    }
    W_host = sh[0].hctl->W;
    buf_host = sh[0].hctl->buf;
    drained = steps_done;
  }

  void check_poison() const {
    if (!poisoned.empty()) throw std::runtime_error(poisoned);
  }

  // Collective with one process per GPU (every rank calls it at the same
  // point of the same call sequence: the end of advance, synchronize, the
  // series / observables / state accessors, set_state): one all-reduce of
  // the drained steps' crossing counts, velocity sums and an error flag.
  // The ring's crossing totals are compared with the plan, the velocity
  // sums become the whole ring's series, and a failure seen by any rank is
  // raised by all of them.  Other modes: drain only.
  void verify_ranks() {
    check_poison();
    drain();
    if (!use_nccl) return;
    Shard& s = sh[0];
    CKS(cudaSetDevice(s.device));
    const size_t n = pend_c.size();
    const size_t words = 2 * n + 1;
    if (words > dcheck_cap) {
      if (dcheck) CKS(cudaFree(dcheck));
      dcheck = nullptr;
      CKS(cudaMalloc(&dcheck, words * 8));
      dcheck_cap = words;
    }
    std::vector<uint64_t> buf(words);
    for (size_t k = 0; k < n; ++k) {
      buf[k] = pend_c[k];
      buf[n + k] = pend_sv[k];
    }
    buf[2 * n] = local_err.empty() ? 0u : 1u;
    NcclApi& api = NcclApi::get();
    CKS(cudaMemcpyAsync(dcheck, buf.data(), words * 8, cudaMemcpyHostToDevice, s.stream));
    api.check(api.all_reduce(dcheck, dcheck, words, ncclUint64, ncclSum, comm, s.stream),
              "ncclAllReduce(step records)");
    CKS(cudaMemcpyAsync(buf.data(), dcheck, words * 8, cudaMemcpyDeviceToHost, s.stream));
    CKS(cudaStreamSynchronize(s.stream));
    const uint64_t first = pend_first;
    std::vector<uint32_t> plan;
    plan.swap(pend_plan);
    pend_c.clear();
    pend_sv.clear();
    if (buf[2 * n]) {
      poisoned = local_err.empty() ? "another rank of the distributed ring failed (engine state is invalid)"
                                   : local_err + " (raised on every rank; engine state is invalid)";
      throw std::runtime_error(poisoned);
    }
    for (size_t k = 0; k < n; ++k)
      if (buf[k] != plan[k]) {
        poisoned = "origin-cone plan contradicted at step " + std::to_string(first + k) +
                   " (summed over the ranks; engine state is invalid)";
        throw std::runtime_error(poisoned);
      }
    for (size_t k = 0; k < n; ++k) {
      sumv_host.push_back(buf[n + k]);
      wraps_host.push_back(plan[k]);
    }
  }

  void ensure_full_staging() {
    if (hx) return;
    CKS(cudaMallocHost(&hx, size_t(n) * 4));
    CKS(cudaMallocHost(&hv, size_t(n) * vbytes));
  }

  void ensure_stage(Shard& s) {
    if (s.hx_stage) return;
    CKS(cudaMallocHost(&s.hx_stage, size_t(s.nl) * 4 + 64));
    CKS(cudaMallocHost(&s.hv_stage, size_t(s.nl) * vbytes + 64));
  }

  // Device -> pinned staging of the ids [id0, id0 + cnt) held at (dx, dv),
  // placed at their ranks (rank = (id + W) mod N: at most two pieces).
  void d2h_at_ranks(const uint32_t* dx, const void* dv, uint32_t id0, uint32_t cnt, cudaStream_t st) {
    const uint32_t r0 = static_cast<uint32_t>((uint64_t(id0) + W_host) % n);
    const uint32_t m1 = std::min<uint32_t>(cnt, n - r0);
    const char* dvb = static_cast<const char*>(dv);
    char* hvb = static_cast<char*>(hv);
    CKS(cudaMemcpyAsync(hx + r0, dx, size_t(m1) * 4, cudaMemcpyDeviceToHost, st));
    CKS(cudaMemcpyAsync(hvb + size_t(r0) * vbytes, dvb, size_t(m1) * vbytes, cudaMemcpyDeviceToHost, st));
    if (m1 < cnt) {
      CKS(cudaMemcpyAsync(hx, dx + m1, size_t(cnt - m1) * 4, cudaMemcpyDeviceToHost, st));
      CKS(cudaMemcpyAsync(hvb, dvb + size_t(m1) * vbytes, size_t(cnt - m1) * vbytes, cudaMemcpyDeviceToHost, st));
    }
  }

  // The whole ring in rank order into the pinned staging (hx, hv); needs
  // drained == steps_done.  Segments of this process: stream-ordered D2H
  // straight to their ranks.  One process per GPU (collective: every rank
  // calls it): segment r is broadcast from rank r into every other rank's
  // idle ping-pong buffer (NCCL over NVLink) and copied down by the ranks
  // that want the ring (`want`); the others only take part.
  void gather_rank_order(bool want) {
    if (want) ensure_full_staging();
    if (!use_nccl) {
      for (Shard& s : sh) {
        CKS(cudaSetDevice(s.device));
        d2h_at_ranks(s.x[buf_host], s.v[buf_host], s.gofs, s.nl, s.stream);
      }
      sync_all();
      return;
    }
    Shard& s = sh[0];
    CKS(cudaSetDevice(s.device));
    NcclApi& api = NcclApi::get();
    const unsigned idle = buf_host ^ 1u;
    for (unsigned r = 0; r < G; ++r) {
      const uint32_t nl_r = lo[r + 1] - lo[r];
      uint32_t* xb = r == s.g ? s.x[buf_host] : s.x[idle];
      void* vb = r == s.g ? s.v[buf_host] : s.v[idle];
      api.check(api.broadcast(xb, xb, size_t(nl_r) * 4, ncclUint8, static_cast<int>(r), comm, s.stream),
                "ncclBroadcast(state x)");
      api.check(api.broadcast(vb, vb, size_t(nl_r) * vbytes, ncclUint8, static_cast<int>(r), comm, s.stream),
                "ncclBroadcast(state v)");
      if (want) d2h_at_ranks(xb, vb, lo[r], nl_r, s.stream);
    }
    CKS(cudaStreamSynchronize(s.stream));
  }

  uint32_t hvel(size_t i) const {
    return vbytes == 1 ? static_cast<const uint8_t*>(hv)[i] : static_cast<const uint32_t*>(hv)[i];
  }

  bool frame_due() const {
    return params.output_mode != OutputMode::none && steps_done < params.steps &&
           steps_done % params.output_stride == 0;
  }

  // src/engine.cpp:81-86 -- every rank records the whole ring (collective
  // with one process per GPU, like the reference's frames in one process).
  void record_frame() {
    drain();
    gather_rank_order(true);
    Frame f;
    f.step = steps_done;
    f.positions.resize(n);
    f.velocities.resize(n);
    widen_staging(f.positions.data(), f.velocities.data());
    frames.push_back(std::move(f));
  }

  // Rank-ordered staging -> caller's u64 arrays (either may be null).
  void widen_staging(uint64_t* positions, uint64_t* velocities) const {
    parallel_chunks(n, [&](size_t a, size_t b) {
      if (positions) widen_u32(hx + a, positions + a, b - a);
      if (velocities) {
        if (vbytes == 1) widen_u8(static_cast<const uint8_t*>(hv) + a, velocities + a, b - a);
        else widen_u32(static_cast<const uint32_t*>(hv) + a, velocities + a, b - a);
      }
    });
  }

  // This process's segment (one process per GPU) in id order, D2H from
  // (dx, dv) in 16M-car pieces on `st`, each widened into the caller's
  // arrays while the next one is in flight.
  void segment_to_host(Shard& s, const uint32_t* dx, const void* dv, uint64_t* positions, uint64_t* velocities,
                       cudaStream_t st) {
    ensure_stage(s);
    constexpr uint32_t kChunk = 1u << 24;
    std::vector<cudaEvent_t> evs;
    for (uint32_t c0 = 0; c0 < s.nl; c0 += kChunk) {
      const uint32_t m = std::min<uint32_t>(kChunk, s.nl - c0);
      cudaEvent_t ev;
      CKS(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      if (positions) CKS(cudaMemcpyAsync(s.hx_stage + c0, dx + c0, size_t(m) * 4, cudaMemcpyDeviceToHost, st));
      if (velocities)
        CKS(cudaMemcpyAsync(static_cast<char*>(s.hv_stage) + size_t(c0) * vbytes,
                            static_cast<const char*>(dv) + size_t(c0) * vbytes, size_t(m) * vbytes,
                            cudaMemcpyDeviceToHost, st));
      CKS(cudaEventRecord(ev, st));
      evs.push_back(ev);
    }
    cudaError_t err = cudaSuccess;
    for (size_t i = 0; i < evs.size(); ++i) {
      if (err == cudaSuccess) err = cudaEventSynchronize(evs[i]);
      if (err == cudaSuccess) {
        const size_t c0 = i * size_t(kChunk), m = std::min<size_t>(kChunk, s.nl - c0);
        parallel_chunks(m, [&](size_t a, size_t b) {
          a += c0;
          b += c0;
          if (positions) widen_u32(s.hx_stage + a, positions + a, b - a);
          if (velocities) {
            if (vbytes == 1) widen_u8(static_cast<const uint8_t*>(s.hv_stage) + a, velocities + a, b - a);
            else widen_u32(static_cast<const uint32_t*>(s.hv_stage) + a, velocities + a, b - a);
          }
        });
      }
      cudaEventDestroy(evs[i]);
    }
    CKS(err);
  }

  // u32 form (nasch_sim_state_segment32): positions by DMA straight into a
  // page-locked caller array (else through the staging), u8 velocities
  // widened to u32 on the host as each piece lands.
  void segment_to_host32(Shard& s, uint32_t* positions, uint32_t* velocities) {
    ensure_stage(s);
    cudaPointerAttributes pa{};
    const bool direct_x =
        positions && cudaPointerGetAttributes(&pa, positions) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    const uint32_t* dx = s.x[buf_host];
    const void* dv = s.v[buf_host];
    constexpr uint32_t kChunk = 1u << 24;
    std::vector<cudaEvent_t> evs;
    for (uint32_t c0 = 0; c0 < s.nl; c0 += kChunk) {
      const uint32_t m = std::min<uint32_t>(kChunk, s.nl - c0);
      cudaEvent_t ev;
      CKS(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      if (velocities)
        CKS(cudaMemcpyAsync(static_cast<char*>(s.hv_stage) + size_t(c0) * vbytes,
                            static_cast<const char*>(dv) + size_t(c0) * vbytes, size_t(m) * vbytes,
                            cudaMemcpyDeviceToHost, s.stream));
      if (positions)
        CKS(cudaMemcpyAsync((direct_x ? positions : s.hx_stage) + c0, dx + c0, size_t(m) * 4,
                            cudaMemcpyDeviceToHost, s.stream));
      CKS(cudaEventRecord(ev, s.stream));
      evs.push_back(ev);
    }
    cudaError_t err = cudaSuccess;
    for (size_t i = 0; i < evs.size(); ++i) {
      if (err == cudaSuccess) err = cudaEventSynchronize(evs[i]);
      if (err == cudaSuccess) {
        const size_t c0 = i * size_t(kChunk), m = std::min<size_t>(kChunk, s.nl - c0);
        parallel_chunks(m, [&](size_t a, size_t b) {
          a += c0;
          b += c0;
          if (positions && !direct_x) std::memcpy(positions + a, s.hx_stage + a, (b - a) * 4);
          if (velocities) {
            if (vbytes == 1) widen_u8_u32(static_cast<const uint8_t*>(s.hv_stage) + a, velocities + a, b - a);
            else std::memcpy(velocities + a, static_cast<const uint32_t*>(s.hv_stage) + a, (b - a) * 4);
          }
        });
      }
      cudaEventDestroy(evs[i]);
    }
    CKS(err);
  }

  void snap_join() {
    if (snap_thread.joinable()) snap_thread.join();
    if (snap_error) {
      std::exception_ptr e = snap_error;
      snap_error = nullptr;
      std::rethrow_exception(e);
    }
  }

  // Segment snapshot: the rank of the segment's first car, after a local
  // drain (no collective: each rank writes its own piece).
  uint64_t segment_first_rank() const { return (uint64_t(sh[0].gofs) + W_host) % n; }

  void state_segment(uint64_t* positions, uint64_t* velocities, uint64_t* first_rank, bool async) {
    check_poison();
    snap_join();
    drain();
    Shard& s = sh[0];
    CKS(cudaSetDevice(s.device));
    if (first_rank) *first_rank = segment_first_rank();
    if (!async) {
      segment_to_host(s, s.x[buf_host], s.v[buf_host], positions, velocities, s.stream);
      return;
    }
    // device copy now (stream-ordered before the next step), D2H and
    // widening on a host thread while the ring keeps stepping
    if (!s.snap_x) {
      CKS(cudaMalloc(&s.snap_x, size_t(s.nl) * 4));
      CKS(cudaMalloc(&s.snap_v, size_t(s.nl) * vbytes));
      CKS(cudaStreamCreateWithFlags(&snap_stream, cudaStreamNonBlocking));
      CKS(cudaEventCreateWithFlags(&snap_ready, cudaEventDisableTiming));
    }
    CKS(cudaMemcpyAsync(s.snap_x, s.x[buf_host], size_t(s.nl) * 4, cudaMemcpyDeviceToDevice, s.stream));
    CKS(cudaMemcpyAsync(s.snap_v, s.v[buf_host], size_t(s.nl) * vbytes, cudaMemcpyDeviceToDevice, s.stream));
    CKS(cudaEventRecord(snap_ready, s.stream));
    snap_thread = std::thread([this, &s, positions, velocities] {
      try {
        CKS(cudaSetDevice(s.device));
        CKS(cudaStreamWaitEvent(snap_stream, snap_ready, 0));
        segment_to_host(s, s.snap_x, s.snap_v, positions, velocities, snap_stream);
      } catch (...) {
        snap_error = std::current_exception();
      }
    });
  }

  // The trajectory checksum without moving the ring: each shard reduces its
  // pieces of the rank-ordered row (positions, then velocities; at most two
  // contiguous id ranges each) to one FNV chunk map on its own GPU
  // (fnv_kernels.cuh), and the host composes the <= 4G maps in row order
  // and applies the result to the running digest.
  void gpu_hash_step() {
    const uint32_t head = (n - W_host) % n;
    struct Piece {
      uint64_t row0;
      size_t shard, slot;
    };
    std::vector<Piece> pieces;
    for (size_t si = 0; si < sh.size(); ++si) {
      Shard& s = sh[si];
      CKS(cudaSetDevice(s.device));
      if (!s.fT[0]) {
        const size_t maxch = (s.nl + kFnvChunk - 1) / kFnvChunk;
        for (int b = 0; b < 2; ++b) {
          CKS(cudaMalloc(&s.fT[b], maxch * 256 * sizeof(unsigned long long)));
          CKS(cudaMalloc(&s.fP[b], maxch * sizeof(unsigned long long)));
        }
        CKS(cudaMallocHost(&s.hpiece, 4 * 257 * sizeof(unsigned long long)));
      }
      // local id ranges in row order: split where the rank-0 car sits
      std::pair<uint32_t, uint32_t> rng[2];
      int nr = 0;
      if (head > s.gofs && head < s.gofs + s.nl) {
        rng[nr++] = {head - s.gofs, s.nl};
        rng[nr++] = {0, head - s.gofs};
      } else {
        rng[nr++] = {0, s.nl};
      }
      size_t slot = 0;
      for (int field = 0; field < 2; ++field) {
        for (int q = 0; q < nr; ++q) {
          const uint32_t a = rng[q].first, cnt = rng[q].second - rng[q].first;
          const uint64_t r0 = (uint64_t(s.gofs) + a + n - head) % n;
          const uint32_t nch = (cnt + kFnvChunk - 1) / kFnvChunk;
          if (field == 0) {
            fnv_slice_chunk_kernel<uint32_t><<<nch, 256, 0, s.stream>>>(s.x[buf_host] + a, cnt, s.fT[0], s.fP[0]);
          } else if (vbytes == 1) {
            fnv_slice_chunk_kernel<uint8_t><<<nch, 256, 0, s.stream>>>(
                static_cast<const uint8_t*>(s.v[buf_host]) + a, cnt, s.fT[0], s.fP[0]);
          } else {
            fnv_slice_chunk_kernel<uint32_t><<<nch, 256, 0, s.stream>>>(
                static_cast<const uint32_t*>(s.v[buf_host]) + a, cnt, s.fT[0], s.fP[0]);
          }
          CKS(cudaGetLastError());
          int in = 0;
          for (uint32_t m = nch; m > 1; m = (m + 1) / 2) {
            fnv_compose_kernel<<<(m + 1) / 2, 256, 0, s.stream>>>(s.fT[in], s.fP[in], m, s.fT[in ^ 1], s.fP[in ^ 1]);
            in ^= 1;
          }
          CKS(cudaMemcpyAsync(s.hpiece + slot * 257, s.fT[in], 256 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, s.stream));
          CKS(cudaMemcpyAsync(s.hpiece + slot * 257 + 256, s.fP[in], sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, s.stream));
          pieces.push_back({field ? n + r0 : r0, si, slot});
          ++slot;
        }
      }
    }
    sync_all();
    // One process per GPU: every rank's piece maps go to every rank (one
    // all-gather of fixed 4-piece records), and all ranks compose the same
    // row, so the checksum is available on each of them.
    std::vector<unsigned long long> all;  // [rank][piece][row0, 256 T, P]
    if (use_nccl) {
      constexpr size_t kRec = 4 * 258;
      Shard& s = sh[0];
      std::vector<unsigned long long> mine(kRec, ~0ull);
      for (const Piece& pc : pieces) {
        unsigned long long* d = mine.data() + pc.slot * 258;
        d[0] = pc.row0;
        std::memcpy(d + 1, s.hpiece + pc.slot * 257, 257 * sizeof(unsigned long long));
      }
      if (!dhash_x) CKS(cudaMalloc(&dhash_x, (G + 1) * kRec * sizeof(unsigned long long)));
      NcclApi& api = NcclApi::get();
      CKS(cudaMemcpyAsync(dhash_x, mine.data(), kRec * 8, cudaMemcpyHostToDevice, s.stream));
      api.check(api.all_gather(dhash_x, dhash_x + kRec, kRec, ncclUint64, comm, s.stream), "ncclAllGather(checksum)");
      all.resize(G * kRec);
      CKS(cudaMemcpyAsync(all.data(), dhash_x + kRec, all.size() * 8, cudaMemcpyDeviceToHost, s.stream));
      CKS(cudaStreamSynchronize(s.stream));
      pieces.clear();
      for (size_t r = 0; r < G; ++r)
        for (size_t q = 0; q < 4; ++q) {
          const unsigned long long* d = all.data() + (r * 4 + q) * 258;
          if (d[0] != ~0ull) pieces.push_back({d[0], r, q});
        }
    }
    auto piece_map = [&](const Piece& pc) -> const unsigned long long* {
      return use_nccl ? all.data() + (pc.shard * 4 + pc.slot) * 258 + 1 : sh[pc.shard].hpiece + pc.slot * 257;
    };
    std::sort(pieces.begin(), pieces.end(), [](const Piece& a, const Piece& b) { return a.row0 < b.row0; });
    // compose in row order: (P1, T1) then (P2, T2) = (P2 P1, l -> P2 T1[l] + T2[(P1 l + T1[l]) & 0xff])
    unsigned long long P = 1, T[256];
    for (int l = 0; l < 256; ++l) T[l] = 0;
    for (const Piece& pc : pieces) {
      const unsigned long long* t2 = piece_map(pc);
      const unsigned long long p2 = t2[256];
      unsigned long long nt[256];
      for (int l = 0; l < 256; ++l) nt[l] = p2 * T[l] + t2[(P * static_cast<unsigned long long>(l) + T[l]) & 0xffu];
      P = p2 * P;
      std::memcpy(T, nt, sizeof T);
    }
    hash = P * hash + T[hash & 0xffu];
  }


  void enqueue_steps(uint64_t count) {
    while (count > 0) {
      if (steps_done - drained + K > kRecCap / 2) drain();
      const uint32_t k = static_cast<uint32_t>(std::min<uint64_t>(count, K));
      launch(k);
      count -= k;
    }
  }

  void advance(uint64_t steps, bool sync) {
    check_poison();
    const uint64_t count = std::min(steps, params.steps - steps_done);
    if (count == 0) {
      if (sync) verify_ranks();
      return;
    }
    if (!checksum_on) {
      uint64_t left = count;
      while (left > 0) {
        uint64_t chunk = left;
        if (params.output_mode != OutputMode::none) {
          const uint64_t stride = params.output_stride;
          chunk = std::min(chunk, (steps_done / stride + 1) * stride - steps_done);
        }
        enqueue_steps(chunk);
        left -= chunk;
        if (frame_due()) record_frame();
      }
      if (sync) verify_ranks();
      return;
    }
    for (uint64_t k = 0; k < count; ++k) {
      launch(1);
      drain();
      gpu_hash_step();
      if (frame_due()) record_frame();
    }
    verify_ranks();
  }

  // Validates and narrows one segment's rank-ordered input (xs, vs: the
  // segment's cars, element 0 first) into the shard's pinned staging while
  // earlier 16M-car pieces are in flight to its idle ping-pong buffer.
  // Returns the first violated rule (0 none; see narrow_validate) and adds
  // the segment's velocity sum.
  template <typename T>
  int stage_segment(Shard& s, const T* xs, const T* vs, unsigned dst, uint64_t* vsum) {
    ensure_stage(s);
    CKS(cudaSetDevice(s.device));
    const uint64_t vlim = std::min<uint64_t>(params.v_max, vmax_eff);
    std::atomic<int> err{0};
    std::atomic<uint64_t> sum{0};
    constexpr size_t kChunk = size_t(1) << 24;
    for (size_t c0 = 0; c0 < s.nl && !err.load(); c0 += kChunk) {
      const size_t c1 = std::min<size_t>(s.nl, c0 + kChunk);
      parallel_chunks(c1 - c0, [&](size_t a, size_t b) {
        a += c0;
        b += c0;
        int e = 0;
        uint64_t acc = 0;
        if constexpr (std::is_same<T, uint64_t>::value) {
          e = narrow_validate(xs, vs, a, b, L, params.v_max, vlim, s.hx_stage, s.hv_stage, vbytes);
          if (!e) {
            if (vbytes == 1)
              for (size_t i = a; i < b; ++i) acc += static_cast<const uint8_t*>(s.hv_stage)[i];
            else
              for (size_t i = a; i < b; ++i) acc += static_cast<const uint32_t*>(s.hv_stage)[i];
          }
        } else {
          e = narrow_validate32(xs, vs, a, b, L, params.v_max, vlim, s.hx_stage, s.hv_stage, vbytes);
        }
        if (!e && !std::is_same<T, uint64_t>::value) {
          if (vbytes == 1)
            for (size_t i = a; i < b; ++i) acc += static_cast<const uint8_t*>(s.hv_stage)[i];
          else
            for (size_t i = a; i < b; ++i) acc += static_cast<const uint32_t*>(s.hv_stage)[i];
        }
        sum += acc;
        if (e) {
          int expected = 0;
          err.compare_exchange_strong(expected, e);
        }
      });
      CKS(cudaMemcpyAsync(s.x[dst] + c0, s.hx_stage + c0, (c1 - c0) * 4, cudaMemcpyHostToDevice, s.stream));
      CKS(cudaMemcpyAsync(static_cast<char*>(s.v[dst]) + c0 * vbytes,
                          static_cast<const char*>(s.hv_stage) + c0 * vbytes, (c1 - c0) * vbytes,
                          cudaMemcpyHostToDevice, s.stream));
    }
    *vsum += sum.load();
    return err.load();
  }

  // set_state.  `segment_only`: the input holds this process's segment only
  // (one process per GPU: ids [first, first + count) of shard_range);
  // otherwise the whole rank-ordered ring, of which each shard reads only
  // its own ids.  Every rank validates and converts only its own cars
  // (AVX-512, pipelined with the upload into the idle ping-pong buffer);
  // the links between segments (last car of g < first car of g+1) and the
  // error codes are agreed in one small all-gather, so every rank accepts
  // or rejects the state together and a rejected state leaves the ring
  // untouched.
  template <typename T>
  void load_state(const T* xin, const T* vin, size_t cnt, bool segment_only) {
    snap_join();
    verify_ranks();  // collective with one process per GPU
    const bool own_only = use_nccl && segment_only;
    int e = cnt != (own_only ? size_t(sh[0].nl) : size_t(n)) ? 5 : 0;
    const unsigned dst = buf_host ^ 1u;
    uint64_t vsum = 0;
    std::vector<uint64_t> firstx(sh.size(), 0), lastx(sh.size(), 0);
    for (size_t i = 0; i < sh.size() && !e; ++i) {
      Shard& s = sh[i];
      const size_t off = own_only ? 0 : s.gofs;
      e = stage_segment(s, xin + off, vin + off, dst, &vsum);
      firstx[i] = xin[off];
      lastx[i] = xin[off + s.nl - 1];
    }
    sync_all();
    if (!use_nccl) {
      for (size_t i = 0; i + 1 < sh.size() && !e; ++i)
        if (lastx[i] >= firstx[i + 1]) e = 2;
    } else {
      // [err, first x, last x, velocity sum] of every rank
      Shard& s = sh[0];
      CKS(cudaSetDevice(s.device));
      uint64_t mine[4] = {uint64_t(e), firstx[0], lastx[0], vsum};
      uint64_t* dbuf = nullptr;
      CKS(cudaMalloc(&dbuf, 4 * 8 * (size_t(G) + 1)));
      struct Free {
        uint64_t* p;
        ~Free() { cudaFree(p); }
      } guard{dbuf};
      std::vector<uint64_t> all(4 * size_t(G));
      CKS(cudaMemcpyAsync(dbuf, mine, 32, cudaMemcpyHostToDevice, s.stream));
      NcclApi& api = NcclApi::get();
      api.check(api.all_gather(dbuf, dbuf + 4, 4, ncclUint64, comm, s.stream), "ncclAllGather(set_state)");
      CKS(cudaMemcpyAsync(all.data(), dbuf + 4, all.size() * 8, cudaMemcpyDeviceToHost, s.stream));
      CKS(cudaStreamSynchronize(s.stream));
      e = 0;
      vsum = 0;
      for (unsigned r = 0; r < G && !e; ++r) e = static_cast<int>(all[4 * r]);
      for (unsigned r = 0; r + 1 < G && !e; ++r)
        if (all[4 * r + 2] >= all[4 * (r + 1) + 1]) e = 2;
      for (unsigned r = 0; r < G; ++r) vsum += all[4 * r + 3];
    }
    switch (e) {
      case 1: throw std::invalid_argument("position out of range [0, length)");
      case 2: throw std::invalid_argument("positions must be strictly increasing");
      case 3: throw std::invalid_argument("velocity above vmax");
      case 4: throw std::invalid_argument("velocity above length-1 (B200 engine restriction)");
      case 5:
        throw std::invalid_argument(own_only ? "segment length must equal this rank's shard_range count"
                                             : "state length must equal ncars");
      default: break;
    }
    buf_host = dst;
    reset_ctl();
    sync_all();
    sumv0 = vsum;
    series_base = steps_done;
    sumv_host.clear();
    wraps_host.clear();
    if (steps_done == 0) {
      frames.clear();
      if (frame_due()) record_frame();
    }
  }

  void finish_construction() {
    reset_ctl();
    sync_all();
    if (!use_nccl) ensure_full_staging();
    else checksum_on = false;  // off by default (one all-gather per step when switched on)
    if (frame_due()) record_frame();
  }
};

ShardedRing::ShardedRing(const SimParams& params, unsigned shards) : impl_(new Impl) {
  Impl& d = *impl_;
  d.init_common(params, shards);
  int ndev = 0;
  CKS(cudaGetDeviceCount(&ndev));
  int cur = 0;
  CKS(cudaGetDevice(&cur));
  for (unsigned g = 0; g < shards; ++g) d.make_shard(g, ndev > 1 ? static_cast<int>(g % ndev) : cur);
  d.setup_p2p_local();
  CKS(cudaSetDevice(cur));
  d.finish_construction();
}

ShardedRing::ShardedRing(const SimParams& params, unsigned rank, unsigned world, const void* nccl_id)
    : impl_(new Impl) {
  Impl& d = *impl_;
  d.init_common(params, world);
  if (rank >= world) throw std::invalid_argument("rank must be below world size");
  int cur = 0;
  CKS(cudaGetDevice(&cur));
  d.use_nccl = true;
  NcclApi& api = NcclApi::get();
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof id);
  api.check(api.comm_init_rank(&d.comm, static_cast<int>(world), id, static_cast<int>(rank)),
            "ncclCommInitRank");
  d.make_shard(rank, cur);
  d.setup_p2p_ipc();
  d.finish_construction();
}

// Released by Impl's destructor (shards are registered before their
// allocations), so nothing leaks if construction throws.
ShardedRing::~ShardedRing() = default;

ShardedRing::Impl::~Impl() {
  Impl& d = *this;
  if (d.snap_thread.joinable()) d.snap_thread.join();
  if (d.snap_ready) cudaEventDestroy(d.snap_ready);
  if (d.snap_stream) cudaStreamDestroy(d.snap_stream);
  for (auto& s : d.sh) {
    cudaSetDevice(s.device);
    if (s.stream) cudaStreamSynchronize(s.stream);
    for (int b = 0; b < 2; ++b) {
      cudaFree(s.x[b]);
      cudaFree(s.v[b]);
    }
    cudaFree(s.ctl);
    cudaFree(s.rec);
    cudaFree(s.blkpow);
    cudaFree(s.thrpow);
    for (int b = 0; b < 2; ++b) {
      cudaFree(s.fT[b]);
      cudaFree(s.fP[b]);
    }
    cudaFreeHost(s.hpiece);
    cudaFree(s.send);
    cudaFree(s.recv);
    for (void* p : s.ipc_opened) cudaIpcCloseMemHandle(p);
    cudaFree(s.xarea);
    cudaFree(s.ptab);
    cudaFree(s.lo_dev);
    cudaFreeHost(s.hrec);
    cudaFreeHost(s.hctl);
    cudaFreeHost(s.hx_stage);
    cudaFreeHost(s.hv_stage);
    cudaFree(s.snap_x);
    cudaFree(s.snap_v);
    if (s.ev_packed) cudaEventDestroy(s.ev_packed);
    if (s.ev_done) cudaEventDestroy(s.ev_done);
    if (s.stream) cudaStreamDestroy(s.stream);
  }
  if (!d.sh.empty()) cudaSetDevice(d.sh[0].device);
  cudaFree(d.dcheck);
  cudaFree(d.dhash_x);
  if (d.comm) NcclApi::get().comm_destroy(d.comm);
  cudaFreeHost(d.hx);
  cudaFreeHost(d.hv);
}

void ShardedRing::set_state(const uint64_t* x, const uint64_t* v, size_t n) {
  impl_->load_state(x, v, n, false);
}
void ShardedRing::set_state32(const uint32_t* x, const uint32_t* v, size_t n) {
  impl_->load_state(x, v, n, false);
}
void ShardedRing::set_state_segment(const uint64_t* x, const uint64_t* v, size_t n) {
  impl_->load_state(x, v, n, true);
}
void ShardedRing::advance(uint64_t steps) { impl_->advance(steps, true); }
void ShardedRing::enqueue(uint64_t steps) { impl_->advance(steps, false); }
void ShardedRing::synchronize() { impl_->verify_ranks(); }
uint64_t ShardedRing::steps_done() const { return impl_->steps_done; }
uint64_t ShardedRing::checksum() const { return impl_->hash; }
const std::vector<Frame>& ShardedRing::frames() const { return impl_->frames; }
const SimParams& ShardedRing::params() const { return impl_->params; }

// Collective with one process per GPU: the whole ring's velocity sum.
void ShardedRing::observables(double* density, double* mean_velocity, double* flow) {
  Impl& d = *impl_;
  d.verify_ranks();
  const uint64_t total = d.sumv_host.empty() ? d.sumv0 : d.sumv_host.back();
  const double n = static_cast<double>(d.params.car_count);
  const double mean = static_cast<double>(total) / n;
  const double dens = n / static_cast<double>(d.params.road_length);
  if (density) *density = dens;
  if (mean_velocity) *mean_velocity = mean;
  if (flow) *flow = dens * mean;
}

// Collective with one process per GPU: every rank passing a non-null array
// receives the whole ring in rank order (segments broadcast over NCCL).
void ShardedRing::state(uint64_t* positions, uint64_t* velocities) {
  Impl& d = *impl_;
  d.snap_join();
  d.verify_ranks();
  const bool want = positions || velocities;
  d.gather_rank_order(want);
  if (want) d.widen_staging(positions, velocities);
}

// Not collective: this process's segment (the whole ring, rank order, when
// the process holds every segment).
void ShardedRing::state_segment(uint64_t* positions, uint64_t* velocities, uint64_t* first_rank) {
  Impl& d = *impl_;
  if (!d.use_nccl) {
    state(positions, velocities);
    if (first_rank) *first_rank = 0;
    return;
  }
  d.state_segment(positions, velocities, first_rank, false);
}

void ShardedRing::state_segment32(uint32_t* positions, uint32_t* velocities, uint64_t* first_rank) {
  Impl& d = *impl_;
  if (!d.use_nccl) {
    RingEngine::state_segment32(positions, velocities, first_rank);
    return;
  }
  d.check_poison();
  d.snap_join();
  d.drain();
  Impl::Shard& s = d.sh[0];
  CKS(cudaSetDevice(s.device));
  if (first_rank) *first_rank = d.segment_first_rank();
  d.segment_to_host32(s, positions, velocities);
}

void ShardedRing::state_segment_async(uint64_t* positions, uint64_t* velocities, uint64_t* first_rank) {
  Impl& d = *impl_;
  if (!d.use_nccl) {
    state_segment(positions, velocities, first_rank);
    return;
  }
  d.state_segment(positions, velocities, first_rank, true);
}

void ShardedRing::state_wait() { impl_->snap_join(); }

size_t ShardedRing::sumv_series(uint64_t* out, size_t cap) {
  Impl& d = *impl_;
  d.verify_ranks();
  const size_t k = std::min(cap, d.sumv_host.size());
  if (out) std::memcpy(out, d.sumv_host.data(), k * sizeof(uint64_t));
  return d.sumv_host.size();
}

size_t ShardedRing::wrap_series(uint64_t* out, size_t cap) {
  Impl& d = *impl_;
  d.verify_ranks();
  const size_t k = std::min(cap, d.wraps_host.size());
  if (out) std::memcpy(out, d.wraps_host.data(), k * sizeof(uint64_t));
  return d.wraps_host.size();
}

void ShardedRing::set_checksum(bool enabled) { impl_->checksum_on = enabled; }
void* ShardedRing::cuda_stream() const { return impl_->sh.empty() ? nullptr : impl_->sh[0].stream; }
uint64_t ShardedRing::kernel_launches() const { return impl_->launches; }
int ShardedRing::exchange_mode() const { return impl_->p2p ? 2 : 1; }
int ShardedRing::steps_per_launch() const { return static_cast<int>(impl_->K); }

void ShardedRing::shard_range(uint64_t* first, uint64_t* count) const {
  const Impl& d = *impl_;
  if (d.use_nccl && d.G > 1) {
    if (first) *first = d.sh[0].gofs;
    if (count) *count = d.sh[0].nl;
  } else {
    if (first) *first = 0;
    if (count) *count = d.n;
  }
}

}  // namespace nb200
