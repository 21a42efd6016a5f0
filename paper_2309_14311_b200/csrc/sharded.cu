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
#include <vector>

#include "engine.hpp"
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
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;

  static NcclApi& get() {
    static NcclApi api;
    if (!api.handle) api.open();
    return api;
  }
  void open() {
    handle = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!handle) throw std::runtime_error(std::string("cannot load libnccl.so.2: ") + dlerror());
    get_unique_id = reinterpret_cast<decltype(get_unique_id)>(dlsym(handle, "ncclGetUniqueId"));
    comm_init_rank = reinterpret_cast<decltype(comm_init_rank)>(dlsym(handle, "ncclCommInitRank"));
    all_gather = reinterpret_cast<decltype(all_gather)>(dlsym(handle, "ncclAllGather"));
    all_reduce = reinterpret_cast<decltype(all_reduce)>(dlsym(handle, "ncclAllReduce"));
    comm_destroy = reinterpret_cast<decltype(comm_destroy)>(dlsym(handle, "ncclCommDestroy"));
    error_string = reinterpret_cast<decltype(error_string)>(dlsym(handle, "ncclGetErrorString"));
    if (!get_unique_id || !comm_init_rank || !all_gather || !all_reduce || !comm_destroy || !error_string)
      throw std::runtime_error("libnccl.so.2 lacks a required symbol");
  }
  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess) throw std::runtime_error(std::string("NCCL error in ") + what + ": " + error_string(r));
  }
};

template <typename F>
void par_chunks(size_t n, F&& f) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const unsigned nt = static_cast<unsigned>(std::min<size_t>(std::min(hw, 32u), n / (1u << 20) + 1));
  if (nt <= 1) {
    f(size_t(0), n);
    return;
  }
  const size_t chunk = (n + nt - 1) / nt;
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t) {
    const size_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

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
  uint64_t K = static_cast<uint64_t>(std::max<long>(1, std::min<long>(kreq, kPlanMax)));
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
  std::vector<uint32_t> pend_c, pend_plan;
  uint64_t pend_first = 0;
  uint32_t* dcheck = nullptr;  // device scratch for the all-reduce
  size_t dcheck_cap = 0;
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
    K = static_cast<uint32_t>(std::max<long>(1, std::min<long>(kreq, kPlanMax)));
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
      if (s.hctl->err == 3u)
        throw std::runtime_error("peer exchange timed out on shard " + std::to_string(s.g) +
                                 " (a rank stopped publishing; engine state is invalid)");
      if (s.hctl->t != steps_done)
        throw std::runtime_error("device step counter out of sync on shard " + std::to_string(s.g));
      if (s.hctl->W != sh[0].hctl->W || s.hctl->buf != sh[0].hctl->buf)
        throw std::runtime_error("shards disagree on the rank offset");
    }
    for (uint64_t k = 0; k < count; ++k) {
      uint64_t sv = 0, c = 0;
      for (const Shard& s : sh) {
        sv += s.hrec[k].sumv;
        c += s.hrec[k].c;
      }
      if (!use_nccl && c != sh[0].hrec[k].cplan)
        throw std::runtime_error("origin-cone plan contradicted at step " + std::to_string(first + k) +
                                 " (engine state is invalid)");
      if (use_nccl) {
        if (pend_c.empty()) pend_first = first + k;
        pend_c.push_back(static_cast<uint32_t>(c));
        pend_plan.push_back(sh[0].hrec[k].cplan);
      }
      sumv_host.push_back(sv);
      wraps_host.push_back(use_nccl ? sh[0].hrec[k].cplan : c);
    }
    W_host = sh[0].hctl->W;
    buf_host = sh[0].hctl->buf;
    drained = steps_done;
  }

  // Collective (every rank calls it at the same point of the same call
  // sequence: the end of advance and synchronize): all-reduce the drained
  // steps' crossing counts and compare the ring's totals with the plan.
  void verify_ranks() {
    if (!use_nccl || pend_c.empty()) return;
    Shard& s = sh[0];
    CKS(cudaSetDevice(s.device));
    const size_t n = pend_c.size();
    if (n > dcheck_cap) {
      if (dcheck) CKS(cudaFree(dcheck));
      dcheck = nullptr;
      CKS(cudaMalloc(&dcheck, n * 4));
      dcheck_cap = n;
    }
    NcclApi& api = NcclApi::get();
    CKS(cudaMemcpyAsync(dcheck, pend_c.data(), n * 4, cudaMemcpyHostToDevice, s.stream));
    api.check(api.all_reduce(dcheck, dcheck, n, ncclUint32, ncclSum, comm, s.stream), "ncclAllReduce(crossings)");
    std::vector<uint32_t> tot(n);
    CKS(cudaMemcpyAsync(tot.data(), dcheck, n * 4, cudaMemcpyDeviceToHost, s.stream));
    CKS(cudaStreamSynchronize(s.stream));
    const uint64_t first = pend_first;
    pend_c.clear();
    std::vector<uint32_t> plan;
    plan.swap(pend_plan);
    for (size_t k = 0; k < n; ++k)
      if (tot[k] != plan[k])
        throw std::runtime_error("origin-cone plan contradicted at step " + std::to_string(first + k) +
                                 " (summed over the ranks; engine state is invalid)");
  }

  void require_local(const char* what) const {
    if (use_nccl && G > 1)
      throw std::invalid_argument(std::string(what) + " needs the whole ring; this process holds one "
                                  "shard of a distributed ring");
  }

  // Whole ring in rank order into the staging buffers (in-process mode).
  void fetch_rank_order() {
    require_local("state");
    std::vector<uint32_t> gx(n);
    std::vector<uint8_t> gv8(vbytes == 1 ? n : 0);
    std::vector<uint32_t> gv32(vbytes == 4 ? n : 0);
    for (Shard& s : sh) {
      CKS(cudaSetDevice(s.device));
      CKS(cudaMemcpyAsync(gx.data() + s.gofs, s.x[buf_host], size_t(s.nl) * 4, cudaMemcpyDeviceToHost, s.stream));
      if (vbytes == 1)
        CKS(cudaMemcpyAsync(gv8.data() + s.gofs, s.v[buf_host], s.nl, cudaMemcpyDeviceToHost, s.stream));
      else
        CKS(cudaMemcpyAsync(gv32.data() + s.gofs, s.v[buf_host], size_t(s.nl) * 4, cudaMemcpyDeviceToHost, s.stream));
    }
    sync_all();
    const uint32_t head = (n - W_host) % n;
    par_chunks(n, [&](size_t a, size_t b) {
      for (size_t k = a; k < b; ++k) {
        size_t id = head + k;
        if (id >= n) id -= n;
        hx[k] = gx[id];
        if (vbytes == 1) static_cast<uint8_t*>(hv)[k] = gv8[id];
        else static_cast<uint32_t*>(hv)[k] = gv32[id];
      }
    });
  }

  uint32_t hvel(size_t i) const {
    return vbytes == 1 ? static_cast<const uint8_t*>(hv)[i] : static_cast<const uint32_t*>(hv)[i];
  }

  bool frame_due() const {
    return params.output_mode != OutputMode::none && steps_done < params.steps &&
           steps_done % params.output_stride == 0;
  }

  void record_frame_staged() {
    Frame f;
    f.step = steps_done;
    f.positions.assign(hx, hx + n);
    f.velocities.resize(n);
    for (uint32_t i = 0; i < n; ++i) f.velocities[i] = hvel(i);
    frames.push_back(std::move(f));
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
    const uint64_t count = std::min(steps, params.steps - steps_done);
    if (count == 0) return;
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
        if (frame_due()) {
          drain();
          fetch_rank_order();
          record_frame_staged();
        }
      }
      if (sync) {
        drain();
        verify_ranks();
      }
      return;
    }
    for (uint64_t k = 0; k < count; ++k) {
      launch(1);
      drain();
      gpu_hash_step();
      if (frame_due()) {
        fetch_rank_order();
        record_frame_staged();
      }
    }
    verify_ranks();
  }

  template <typename T>
  void load_state(const T* xin, const T* vin, size_t cnt) {
    if (cnt != n) throw std::invalid_argument("state length must equal ncars");
    std::atomic<int> err{0};
    std::atomic<uint64_t> vsum{0};
    const uint64_t vlim = std::min<uint64_t>(params.v_max, vmax_eff);
    par_chunks(n, [&](size_t a, size_t b) {
      int e = 0;
      uint64_t s = 0;
      for (size_t i = a; i < b && !e; ++i) {
        const uint64_t xi = xin[i], vi = vin[i];
        if (xi >= L) e = 1;
        else if (i && static_cast<uint64_t>(xin[i - 1]) >= xi) e = 2;
        else if (vi > params.v_max) e = 3;
        else if (vi > vlim) e = 4;
        s += vi;
      }
      vsum += s;
      if (e) {
        int expected = 0;
        err.compare_exchange_strong(expected, e);
      }
    });
    switch (err.load()) {
      case 1: throw std::invalid_argument("position out of range [0, length)");
      case 2: throw std::invalid_argument("positions must be strictly increasing");
      case 3: throw std::invalid_argument("velocity above vmax");
      case 4: throw std::invalid_argument("velocity above length-1 (B200 engine restriction)");
      default: break;
    }
    drain();
    verify_ranks();
    for (Shard& s : sh) {
      CKS(cudaSetDevice(s.device));
      std::vector<uint32_t> sx(s.nl);
      std::vector<uint8_t> sv8(vbytes == 1 ? s.nl : 0);
      std::vector<uint32_t> sv32(vbytes == 4 ? s.nl : 0);
      for (uint32_t i = 0; i < s.nl; ++i) {
        sx[i] = static_cast<uint32_t>(xin[s.gofs + i]);
        if (vbytes == 1) sv8[i] = static_cast<uint8_t>(vin[s.gofs + i]);
        else sv32[i] = static_cast<uint32_t>(vin[s.gofs + i]);
      }
      CKS(cudaMemcpyAsync(s.x[buf_host], sx.data(), size_t(s.nl) * 4, cudaMemcpyHostToDevice, s.stream));
      if (vbytes == 1)
        CKS(cudaMemcpyAsync(s.v[buf_host], sv8.data(), s.nl, cudaMemcpyHostToDevice, s.stream));
      else
        CKS(cudaMemcpyAsync(s.v[buf_host], sv32.data(), size_t(s.nl) * 4, cudaMemcpyHostToDevice, s.stream));
      CKS(cudaStreamSynchronize(s.stream));
    }
    reset_ctl();
    sync_all();
    sumv0 = vsum.load();
    series_base = steps_done;
    sumv_host.clear();
    wraps_host.clear();
    if (steps_done == 0 && !(use_nccl && G > 1)) {
      frames.clear();
      if (frame_due()) {
        fetch_rank_order();
        record_frame_staged();
      }
    }
  }

  void finish_construction() {
    reset_ctl();
    sync_all();
    if (!(use_nccl && G > 1)) {
      CKS(cudaMallocHost(&hx, size_t(n) * 4));
      CKS(cudaMallocHost(&hv, size_t(n) * vbytes));
      if (frame_due()) {
        fetch_rank_order();
        record_frame_staged();
      }
    } else {
      checksum_on = false;  // off by default (one all-gather per step when switched on)
    }
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

void ShardedRing::set_state(const uint64_t* x, const uint64_t* v, size_t n) { impl_->load_state(x, v, n); }
void ShardedRing::set_state32(const uint32_t* x, const uint32_t* v, size_t n) { impl_->load_state(x, v, n); }
void ShardedRing::advance(uint64_t steps) { impl_->advance(steps, true); }
void ShardedRing::enqueue(uint64_t steps) { impl_->advance(steps, false); }
void ShardedRing::synchronize() {
  impl_->drain();
  impl_->verify_ranks();
}
uint64_t ShardedRing::steps_done() const { return impl_->steps_done; }
uint64_t ShardedRing::checksum() const { return impl_->hash; }
const std::vector<Frame>& ShardedRing::frames() const { return impl_->frames; }
const SimParams& ShardedRing::params() const { return impl_->params; }

void ShardedRing::observables(double* density, double* mean_velocity, double* flow) {
  Impl& d = *impl_;
  d.require_local("observables");
  d.drain();
  const uint64_t total = d.sumv_host.empty() ? d.sumv0 : d.sumv_host.back();
  const double n = static_cast<double>(d.params.car_count);
  const double mean = static_cast<double>(total) / n;
  const double dens = n / static_cast<double>(d.params.road_length);
  if (density) *density = dens;
  if (mean_velocity) *mean_velocity = mean;
  if (flow) *flow = dens * mean;
}

void ShardedRing::state(uint64_t* positions, uint64_t* velocities) {
  Impl& d = *impl_;
  d.drain();
  d.fetch_rank_order();
  par_chunks(d.n, [&](size_t a, size_t b) {
    for (size_t i = a; i < b; ++i) {
      if (positions) positions[i] = d.hx[i];
      if (velocities) velocities[i] = d.hvel(i);
    }
  });
}

size_t ShardedRing::sumv_series(uint64_t* out, size_t cap) {
  Impl& d = *impl_;
  d.drain();
  const size_t k = std::min(cap, d.sumv_host.size());
  if (out) std::memcpy(out, d.sumv_host.data(), k * sizeof(uint64_t));
  return d.sumv_host.size();
}

size_t ShardedRing::wrap_series(uint64_t* out, size_t cap) {
  Impl& d = *impl_;
  d.drain();
  const size_t k = std::min(cap, d.wraps_host.size());
  if (out) std::memcpy(out, d.wraps_host.data(), k * sizeof(uint64_t));
  return d.wraps_host.size();
}

void ShardedRing::set_checksum(bool enabled) {

  impl_->checksum_on = enabled;
}
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
