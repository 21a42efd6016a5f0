// engine.cu -- host side of the B200 ring engine (GpuRing) and the uniform
// initial-state generator.
//
// Mode selection (per simulation, fixed at construction):
//   warp ring -- N <= 512: ring_warp_kernel, one warp, cars in registers,
//                whole chunks of steps per launch (resident_kernel.cuh);
//                256 < N <= 512: ring_quad_kernel, the same on four warps.
//   resident  -- N <= 4096: ring_resident_kernel, one CTA, shared memory
//                (only where the distributed-resident kernel does not apply).
//   DR        -- 4096 < N <= ~560k: ring_dr_kernel, the ring in registers
//                across all SMs, a planner CTA one epoch ahead
//                (dr_kernel.cuh, cone_warp.cuh).
//   TB        -- larger rings: nasch_tb_kernel, K steps per launch from
//                registers with the origin-cone plan (tb_kernel.cuh).
//   K1        -- nasch_step_kernel, one step per launch: rings no other
//                mode admits (e.g. vmax too large for a K >= 2 cone).
// All are bit-identical to the reference; tests force each one
// (NASCH_B200_DR / _RESIDENT / _WARPRING / _K / _TILE).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <atomic>
#include <cmath>
#include <exception>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <condition_variable>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <type_traits>
#include <vector>

#include "engine.hpp"
#include "host_simd.hpp"
#include "minstd.hpp"
#include "step_kernels.cuh"
#include "tb_config.hpp"
#include "tb_kernel.cuh"
#include "resident_kernel.cuh"
#include "dr_kernel.cuh"
#include "fnv_pipeline.cuh"

namespace nb200 {

namespace {

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  }
}
#define CK(call) check((call), #call)

constexpr int kTPB = 256;
// single-step kernel geometry
constexpr int kCPT1 = 8;
constexpr uint32_t kTile1 = kTPB * kCPT1;
// temporal-blocked kernel geometry: tb_config.hpp
constexpr int kGraphLaunches = 16;
// resident small-ring kernel
constexpr int kResidentTPB = 1024;
constexpr uint32_t kResidentChunk = kRecCap / 4;  // steps per resident launch

long env_long(const char* name, long fallback) {
  const char* s = std::getenv(name);
  if (!s || !*s) return fallback;
  return std::strtol(s, nullptr, 10);
}

}  // namespace

struct GpuRing::Impl {
  SimParams params;
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t n = 0, L = 0, vmax_eff = 0, npad = 0;
  int vbytes = 1;   // 1 => u8 velocities, 4 => u32
  bool tb = false;  // temporal-blocked mode
  bool resident = false;  // small ring: one CTA runs whole chunks of steps
  bool warp_ring = true;  // tiny rings (N <= 512): one warp, cars in registers
  bool quad_all = false;  // NASCH_B200_QUADRING=2: every N <= 512 on four warps (tests)
  bool quad_ring = true;  // 256 < N <= 512 (and ragged 128 < N <= 256): four warps (ring_quad_kernel)
  bool medium = false;    // TB with 512-car tiles (medium rings)
  bool dr = false;        // distributed-resident medium ring (dr_kernel.cuh)
  uint32_t dr_G = 0, dr_cpt = 0;
  int dr_geom = 0;  // index into kDrGeoms
  Ctl* dplans = nullptr;
  DrSync* dsync = nullptr;
  uint32_t* dmbox = nullptr;
  uint32_t* dseg = nullptr;
  ~Impl();
  uint32_t K = 1;   // steps per TB launch
  uint32_t* x[2] = {nullptr, nullptr};
  void* v[2] = {nullptr, nullptr};
  uint32_t* blkpow = nullptr;
  uint32_t* thrpow = nullptr;
  // Temporal-blocked rings also keep the one-step kernel's geometry: with the
  // checksum on every step's row is hashed, so they step one launch at a
  // time with nasch_step_kernel (HBM-bound, ~0.35 ms on 2e8 cars against
  // ~0.58 ms for a one-step TB launch) and re-plan before the next TB launch.
  RingArgs args1{};
  int grid1 = 0;
  uint32_t* blkpow1 = nullptr;
  uint32_t* thrpow1 = nullptr;
  bool plan_stale = false;  // one-step launches ran since the last TB plan
  // streamed job (job32): the input state's own buffers, streams, events
  uint32_t* jx = nullptr;
  void* jv = nullptr;
  cudaStream_t jstream[3] = {nullptr, nullptr, nullptr};  // x upload, v upload, download
  Ctl* jctl = nullptr;  // pinned: the control block after the job's plan
  unsigned long long* dcode = nullptr;  // set_state32: first position-rule violation (device)
  unsigned long long* hcode = nullptr;  // ... its pinned host copy
  Ctl* ctl = nullptr;
  StepRec* rec = nullptr;
  unsigned long long* dsum = nullptr;
  int grid = 1;
  RingArgs args{};
  cudaGraphExec_t graph = nullptr;

  // host bookkeeping
  uint64_t steps_done = 0;  // steps enqueued
  uint64_t drained = 0;     // steps whose records are in the host series
  uint64_t hash = kFnvBasis;
  bool checksum_on = true;
  uint64_t sumv0 = 0;       // velocity sum of the state at the last set_state
  std::vector<uint64_t> sumv_host;  // [k] = sum v after step series_base+k+1
  std::vector<uint64_t> wraps_host;
  uint64_t series_base = 0;
  uint32_t W_host = 0;      // rank offset after `drained` steps
  uint32_t buf_host = 0;    // buffer holding the state after `drained` steps
  uint64_t launches = 0;
  std::vector<Frame> frames;

  // pinned staging
  uint32_t* hx = nullptr;
  void* hv = nullptr;

  // asynchronous snapshots (state_async): device copy of the state, a copy
  // stream, pinned staging and the host thread widening into the caller's
  // arrays
  uint32_t* snap_x = nullptr;
  void* snap_v = nullptr;
  uint32_t* snap_hx = nullptr;
  void* snap_hv = nullptr;
  cudaStream_t snap_stream = nullptr;
  cudaEvent_t snap_ready = nullptr;
  std::thread snap_thread;
  std::exception_ptr snap_error;

  void snap_join() {
    if (snap_thread.joinable()) snap_thread.join();
    if (snap_error) {
      std::exception_ptr e = snap_error;
      snap_error = nullptr;
      std::rethrow_exception(e);
    }
  }
  StepRec* hrec = nullptr;
  Ctl* hctl = nullptr;

  template <typename VT, int TPB, int CPT, bool QDRAW = false>
  void launch_dr_cpt(uint32_t k) {
    DrArgs da{dplans, dmbox, dsync, dseg, dr_G, K};
    void* kargs[] = {&args, &da, &k};
    CK(cudaMemsetAsync(dsync, 0, (2 + dr_G) * sizeof(unsigned int), stream));
    CK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&ring_dr_kernel<VT, TPB, CPT, QDRAW>),
                                   dim3(dr_G + 1), dim3(TPB), kargs, 0, stream));
  }
  template <typename VT>
  void launch_dr(uint32_t k) {
    switch (dr_geom) {
      case 0: launch_dr_cpt<VT, kDrTPB, 4>(k); break;
      case 1: launch_dr_cpt<VT, kDrTPB, 8>(k); break;
      case 2: launch_dr_cpt<VT, kDrTPB, 16>(k); break;
      case 3: launch_dr_cpt<VT, kDrTPB, 20, true>(k); break;
      case 4: launch_dr_cpt<VT, kDrTPB, 24, true>(k); break;
      default: launch_dr_cpt<VT, kDrTPB, 32, true>(k); break;
    }
  }

  template <typename VT>
  void launch_tb(uint32_t k) {
    if (medium) nasch_tb_kernel<VT, kTbmTPB, kTbmCPT, kTbHalo, false><<<grid, kTbmTPB, 0, stream>>>(args, k);
    else nasch_tb_kernel<VT, kTbTPB, kTbCPT, kTbHalo, kTbWT><<<grid, kTbTPB, 0, stream>>>(args, k);
    // the next launch's plan, when its cone does not fit the step kernel's
    // last block (K (vmax + 1) > threads per block)
    if (!tb_plan_inline(K, vmax_eff, medium ? kTbmTPB : kTbTPB)) {
      cone_init_kernel<VT, 256><<<1, 256, 0, stream>>>(args);
      ++launches;
    }
  }

  // One launch advancing k steps (k == 1 in single-step mode; any k in
  // resident mode).
  // ring_quad_kernel: CPW = 1, 2 or 4 cars per thread on four warps.
  template <typename VT>
  void launch_quad(uint32_t k) {
    const uint32_t cpw = n <= 128 ? 1 : n <= 256 ? 2 : 4;  // (NASCH_B200_QUADRING=2 sends every N <= 512 here)
    const bool exact = n % cpw == 0;
    if (cpw == 1) ring_quad_kernel<VT, 1, true><<<1, 128, 0, stream>>>(args, k);
    else if (cpw == 2 && exact) ring_quad_kernel<VT, 2, true><<<1, 128, 0, stream>>>(args, k);
    else if (cpw == 2) ring_quad_kernel<VT, 2, false><<<1, 128, 0, stream>>>(args, k);
    else if (exact) ring_quad_kernel<VT, 4, true><<<1, 128, 0, stream>>>(args, k);
    else ring_quad_kernel<VT, 4, false><<<1, 128, 0, stream>>>(args, k);
  }

  void launch(uint32_t k) {
    if (dr) {
      launch_dr<uint8_t>(k);  // DR needs K(vmax+1) <= 256: u8 velocities
    } else if (tb) {
      if (vbytes == 1) launch_tb<uint8_t>(k); else launch_tb<uint32_t>(k);
    } else if (resident) {
      // Block width by ring size: a per-step barrier across 32 warps costs
      // more than a few extra cars per thread on a tiny ring (C1: 200 cars).
      // (measured, tools/c1_probe.py: four warps 283 ns per step at N = 500
      // against 513 on one warp with 16 cars per lane; N = 203: 264 / 321;
      // N = 200, the EXACT one-warp instantiation: 273 / 250; N = 100: 265 / 195)
      if (quad_ring && n <= 512 && (quad_all || n > 256 || (n > 128 && n % 8 != 0))) {
        if (vbytes == 1) launch_quad<uint8_t>(k); else launch_quad<uint32_t>(k);
      } else if (vbytes == 1) {
        if (warp_ring && n <= 128) {
          if (n % 4 == 0) ring_warp_kernel<uint8_t, 4, true><<<1, 32, 0, stream>>>(args, k);
          else ring_warp_kernel<uint8_t, 4><<<1, 32, 0, stream>>>(args, k);
        } else if (warp_ring && n <= 256) {
          if (n % 8 == 0) ring_warp_kernel<uint8_t, 8, true><<<1, 32, 0, stream>>>(args, k);
          else ring_warp_kernel<uint8_t, 8><<<1, 32, 0, stream>>>(args, k);
        } else if (warp_ring && n <= 512) {
          if (n % 16 == 0) ring_warp_kernel<uint8_t, 16, true><<<1, 32, 0, stream>>>(args, k);
          else ring_warp_kernel<uint8_t, 16><<<1, 32, 0, stream>>>(args, k);
        }
        else if (n <= 256) ring_resident_kernel<uint8_t, 256><<<1, 256, 0, stream>>>(args, k);
        else ring_resident_kernel<uint8_t, kResidentTPB><<<1, kResidentTPB, 0, stream>>>(args, k);
      } else {
        if (warp_ring && n <= 128) ring_warp_kernel<uint32_t, 4><<<1, 32, 0, stream>>>(args, k);
        else if (warp_ring && n <= 256) ring_warp_kernel<uint32_t, 8><<<1, 32, 0, stream>>>(args, k);
        else if (warp_ring && n <= 512) ring_warp_kernel<uint32_t, 16><<<1, 32, 0, stream>>>(args, k);
        else if (n <= 256) ring_resident_kernel<uint32_t, 256><<<1, 256, 0, stream>>>(args, k);
        else ring_resident_kernel<uint32_t, kResidentTPB><<<1, kResidentTPB, 0, stream>>>(args, k);
      }
    } else {
      if (vbytes == 1) {
        nasch_step_kernel<uint8_t, kTPB, kCPT1><<<grid, kTPB, 0, stream>>>(args);
      } else {
        nasch_step_kernel<uint32_t, kTPB, kCPT1><<<grid, kTPB, 0, stream>>>(args);
      }
    }
    ++launches;
  }

  uint32_t steps_per_launch() const { return (resident || dr) ? kResidentChunk : tb ? K : 1u; }

  // One step of a temporal-blocked ring by the one-step kernel (its own grid
  // and draw-multiplier tables, args1): it advances the control block (t, W,
  // E, buf) exactly as a 1-step TB launch would, but leaves no plan.
  void launch_single() {
    if (vbytes == 1) nasch_step_kernel<uint8_t, kTPB, kCPT1><<<grid1, kTPB, 0, stream>>>(args1);
    else nasch_step_kernel<uint32_t, kTPB, kCPT1><<<grid1, kTPB, 0, stream>>>(args1);
    ++launches;
    plan_stale = true;
  }

  // The origin-cone plan for the current step (after one-step launches).
  void replan() {
    if (dr) cone_init_kernel<uint8_t, kDrTPB><<<1, kDrTPB, 0, stream>>>(args);  // the DR planner's width
    else if (vbytes == 1) cone_init_kernel<uint8_t, 256><<<1, 256, 0, stream>>>(args);
    else cone_init_kernel<uint32_t, 256><<<1, 256, 0, stream>>>(args);
    CK(cudaGetLastError());
    ++launches;
    plan_stale = false;
  }

  void build_graph() {
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < kGraphLaunches; ++i) launch(steps_per_launch());
    launches -= kGraphLaunches;
    CK(cudaStreamEndCapture(stream, &g));
    CK(cudaGraphInstantiate(&graph, g, 0));
    CK(cudaGraphDestroy(g));
  }

  // Control block for the current state (W = 0: ids are ranks again).
  void reset_ctl() {
    Ctl c{};
    c.t = steps_done;
    c.W = 0;
    c.buf = buf_host;
    c.E = mulmod(seeded(params.seed), powmod(kA, draw_exponent(steps_done, n, 0)));
    c.E2 = mulmod(c.E, args.an_inv);
    *hctl = c;
    CK(cudaMemcpyAsync(ctl, hctl, sizeof(Ctl), cudaMemcpyHostToDevice, stream));
    CK(cudaMemsetAsync(rec, 0, sizeof(StepRec) * kRecCap, stream));
    if (dr) {  // the DR planner's width
      cone_init_kernel<uint8_t, kDrTPB><<<1, kDrTPB, 0, stream>>>(args);
      CK(cudaGetLastError());
    } else if (tb) {
      // the first plan: K (vmax + 1) <= 256 cone cars
      if (vbytes == 1) cone_init_kernel<uint8_t, 256><<<1, 256, 0, stream>>>(args);
      else cone_init_kernel<uint32_t, 256><<<1, 256, 0, stream>>>(args);
      CK(cudaGetLastError());
    }
    W_host = 0;
    plan_stale = false;
  }

  void compute_sumv0() {
    CK(cudaMemsetAsync(dsum, 0, sizeof(unsigned long long), stream));
    const int blocks = std::max(1, std::min<int>((n + kTPB - 1) / kTPB, 1024));
    if (vbytes == 1) {
      sum_velocity_kernel<uint8_t><<<blocks, kTPB, 0, stream>>>(static_cast<uint8_t*>(v[buf_host]), n, dsum);
    } else {
      sum_velocity_kernel<uint32_t><<<blocks, kTPB, 0, stream>>>(static_cast<uint32_t*>(v[buf_host]), n, dsum);
    }
    CK(cudaGetLastError());
    unsigned long long s = 0;
    CK(cudaMemcpyAsync(&s, dsum, sizeof s, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    sumv0 = s;
  }

  // Pull per-step records of steps [drained, steps_done) into the host series.
  void drain() {
    if (drained == steps_done) return;
    const uint64_t first = drained, count = steps_done - drained;
    uint64_t done = 0;
    while (done < count) {  // records live at t mod kRecCap
      const uint64_t slot = (first + done) % kRecCap;
      const uint64_t seg = std::min<uint64_t>(count - done, kRecCap - slot);
      CK(cudaMemcpyAsync(hrec + done, rec + slot, seg * sizeof(StepRec), cudaMemcpyDeviceToHost, stream));
      done += seg;
    }
    CK(cudaMemcpyAsync(hctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (hctl->err == 3) {
      throw std::runtime_error("distributed-resident launch aborted: a CTA waited more than ~2 s for a "
                               "neighbour or the planner (engine state is invalid)");
    }
    if (hctl->err) {
      throw std::runtime_error("origin-cone plan contradicted at step " +
                               std::to_string(hctl->err_step) + " (engine state is invalid)");
    }
    if (hctl->t != steps_done) {
      throw std::runtime_error("device step counter out of sync (" + std::to_string(hctl->t) +
                               " vs " + std::to_string(steps_done) + ")");
    }
    for (uint64_t k = 0; k < count; ++k) {
      sumv_host.push_back(hrec[k].sumv);
      wraps_host.push_back(hrec[k].c);
    }
    W_host = hctl->W;
    buf_host = hctl->buf;
    drained = steps_done;
  }

  // Current state in rank order into pinned staging (hx, hv); requires
  // drained == steps_done.
  void fetch_rank_order() {
    const int cur = static_cast<int>(buf_host);
    const uint32_t head = (n - W_host) % n;  // id of the rank-0 car
    const uint32_t first = n - head;         // ids head..n-1 -> ranks 0..first-1
    CK(cudaMemcpyAsync(hx, x[cur] + head, size_t(first) * 4, cudaMemcpyDeviceToHost, stream));
    if (head) CK(cudaMemcpyAsync(hx + first, x[cur], size_t(head) * 4, cudaMemcpyDeviceToHost, stream));
    char* hvb = static_cast<char*>(hv);
    const char* dv = static_cast<const char*>(v[cur]);
    CK(cudaMemcpyAsync(hvb, dv + size_t(head) * vbytes, size_t(first) * vbytes, cudaMemcpyDeviceToHost, stream));
    if (head)
      CK(cudaMemcpyAsync(hvb + size_t(first) * vbytes, dv, size_t(head) * vbytes, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
  }

  uint32_t hvel(size_t i) const {
    return vbytes == 1 ? static_cast<const uint8_t*>(hv)[i] : static_cast<const uint32_t*>(hv)[i];
  }

  // output = pgm: the frame as its raster row only, built on the device
  // from the current state (a memset and a scatter of N zero bytes into an
  // L-byte row), then copied to the host -- L bytes per frame instead of
  // 16 N bytes of u64 positions and velocities rendered on the host.
  uint8_t* draster = nullptr;
  void record_frame_raster() {
    if (!draster) CK(cudaMalloc(&draster, L));
    const int cur = static_cast<int>(buf_host);
    CK(cudaMemsetAsync(draster, 0xff, L, stream));
    raster_kernel<<<std::max(1u, std::min(148u * 8u, (n + 255) / 256)), 256, 0, stream>>>(x[cur], n, draster);
    CK(cudaGetLastError());
    ++launches;
    Frame f;
    f.step = steps_done;
    f.raster.resize(L);
    CK(cudaMemcpyAsync(f.raster.data(), draster, L, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    frames.push_back(std::move(f));
  }

  void record_frame_staged() {
    Frame f;
    f.step = steps_done;
    f.positions.assign(hx, hx + n);
    f.velocities.resize(n);
    for (uint32_t i = 0; i < n; ++i) f.velocities[i] = hvel(i);
    frames.push_back(std::move(f));
  }

  bool frame_due() const {
    return params.output_mode != OutputMode::none && steps_done < params.steps &&
           steps_done % params.output_stride == 0;
  }

  // src/engine.cpp:81-86
  void record_frame_if_due() {
    if (!frame_due()) return;
    drain();
    if (params.output_mode == OutputMode::pgm) {
      record_frame_raster();
      return;
    }
    fetch_rank_order();
    record_frame_staged();
  }

  // Enqueue `count` steps: graph chains of full launches, then a remainder
  // launch.  Keeps the undrained record window well inside kRecCap (each
  // launch's last block zeroes the slots of the next plan).
  void enqueue_steps(uint64_t count) {
    if (plan_stale) replan();
    const uint64_t per = steps_per_launch();
    if (resident || dr) {  // whole chunks in one launch; no graph needed
      while (count > 0) {
        const uint32_t k = static_cast<uint32_t>(std::min<uint64_t>(count, per));
        if (steps_done - drained + k > kRecCap / 2) drain();
        launch(k);
        CK(cudaGetLastError());
        steps_done += k;
        count -= k;
      }
      return;
    }
    const uint64_t chunk = per * kGraphLaunches;
    while (count > 0) {
      if (steps_done - drained + std::min(count, chunk) > kRecCap / 2) drain();
      if (count >= chunk) {
        if (!graph) build_graph();
        CK(cudaGraphLaunch(graph, stream));
        launches += kGraphLaunches;
        steps_done += chunk;
        count -= chunk;
      } else {
        const uint32_t k = static_cast<uint32_t>(std::min(count, per));
        launch(k);
        CK(cudaGetLastError());
        steps_done += k;
        count -= k;
      }
    }
  }

  void advance(uint64_t steps, bool sync) {
    const uint64_t count = std::min(steps, params.steps - steps_done);
    if (count == 0) return;
    // Small rings whose every few steps are hashed or recorded: rows dumped
    // by the step kernels, digested and turned into frames a batch at a time
    // (frames alone only on the resident rings: a medium ring's multi-step
    // launches and its device raster are faster than dumping every row)
    if (dump_rows() > 0 && (checksum_on || (params.output_mode != OutputMode::none && resident))) {
      dump_batched(count);
      if (sync) drain();
      return;
    }
    if (!checksum_on) {
      // Run at full speed between frame steps (every output_stride steps,
      // src/engine.cpp:81-86); each frame is one rank-ordered D2H.
      uint64_t left = count;
      while (left > 0) {
        uint64_t chunk = left;
        if (params.output_mode != OutputMode::none) {
          const uint64_t stride = params.output_stride;
          const uint64_t next = (steps_done / stride + 1) * stride;  // next frame step
          chunk = std::min(chunk, next - steps_done);
        }
        enqueue_steps(chunk);
        left -= chunk;
        if (frame_due() && params.output_mode == OutputMode::pgm) {
          drain();
          record_frame_raster();
        } else if (frame_due()) {
          // overlapped with the next chunk: device copy now, host copy and
          // widening into the frame on the snapshot thread
          frames.emplace_back();
          Frame& f = frames.back();
          f.step = steps_done;
          f.positions.resize(n);
          f.velocities.resize(n);
          snap_start(f.positions.data(), f.velocities.data());
        }
      }
      if (sync) drain();
      return;
    }
    // The checksum folds every step's row (src/engine.cpp:173-181): one
    // step per launch, each followed by the on-device FNV fold
    // (fnv_kernels.cuh) -- no host round trip unless a frame is due.
    for (uint64_t k = 0; k < count; ++k) {
      if (tb) launch_single();
      else launch(1);
      CK(cudaGetLastError());
      ++steps_done;
      fnv_fold();
      if (frame_due()) {
        record_frame_if_due();
      } else if (steps_done - drained > kRecCap / 2) {
        drain();
      }
    }
    if (sync) drain();
  }

  // ---- checksum batches (rings up to ~1M cars) -------------------------
  // The digest is one FNV-1a over every step's row laid end to end, so k
  // rows can be digested in ONE pass of the pipeline (FnvRowDigest over the
  // positions-only array of 2 N k u32 values) instead of one pass per step,
  // whose ~20 launches dominate a small ring's step (C1: 89 us per step,
  // slower than the reference's CPU).  Small rings dump their rows from the
  // resident kernels (RingArgs::dump, k steps per launch); medium rings step
  // with the one-step kernel and dump_row_kernel.
  static constexpr uint64_t kDumpBytes = uint64_t(256) << 20;
  static constexpr uint64_t kDumpMaxRows = 4096;
  uint32_t* dstage = nullptr;  // [rows][2N] u32 rank-ordered rows
  Ctl* dctl0 = nullptr;        // W = 0, buf = 0: the batch as one row

  static constexpr uint64_t kDumpGraphRows = 512;
  cudaGraphExec_t gbatch = nullptr;
  uint64_t gbatch_launches = 0;

  // k one-step launches, each followed by the dump of its row (slot i)
  void enqueue_dumped_steps(uint64_t k) {
    const int g = static_cast<int>(std::min<uint64_t>(148 * 8, (n + 255) / 256));
    for (uint64_t i = 0; i < k; ++i) {
      launch_single();
      if (vbytes == 1) dump_row_kernel<uint8_t><<<g, 256, 0, stream>>>(args, dstage + i * 2 * n);
      else dump_row_kernel<uint32_t><<<g, 256, 0, stream>>>(args, dstage + i * 2 * n);
      ++launches;
    }
  }

  uint64_t dump_rows() const {
    if (!(resident || ((tb || dr) && grid1 > 0))) return 0;
    const uint64_t rows = std::min<uint64_t>(kDumpMaxRows, kDumpBytes / (8ull * n));
    return rows >= 8 ? rows : 0;
  }

  uint32_t* hrows = nullptr;   // pinned: frame rows copied down from a batch

  void dump_batched(uint64_t count) {
    const uint64_t B = dump_rows();
    if (!dstage) {
      CK(cudaMalloc(&dstage, size_t(B) * 2 * n * 4));
      CK(cudaMalloc(&dctl0, sizeof(Ctl)));
      CK(cudaMemset(dctl0, 0, sizeof(Ctl)));
    }
    RingArgs rowargs{};
    rowargs.x[0] = rowargs.x[1] = dstage;
    rowargs.v[0] = rowargs.v[1] = dstage;
    rowargs.ctl = dctl0;
    rowargs.fnv_pos_only = 1;
    while (count > 0) {
      const uint64_t k = std::min(count, B);
      if (steps_done - drained + k > kRecCap / 2) drain();
      if (resident) {
        const uint32_t* keep = args.dump;
        args.dump = dstage;
        launch(static_cast<uint32_t>(k));
        args.dump = const_cast<uint32_t*>(keep);
      } else if (k == B && B <= kDumpGraphRows) {
        // full batches replay one captured graph of B (step, dump) pairs:
        // the per-kernel launch latency, not the work, sets a medium ring's
        // step time here
        if (!gbatch) {
          cudaGraph_t gr;
          CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
          const uint64_t l0 = launches;
          enqueue_dumped_steps(B);
          gbatch_launches = launches - l0;
          launches = l0;
          CK(cudaStreamEndCapture(stream, &gr));
          CK(cudaGraphInstantiate(&gbatch, gr, 0));
          CK(cudaGraphDestroy(gr));
        }
        CK(cudaGraphLaunch(gbatch, stream));
        launches += gbatch_launches;
        plan_stale = true;
      } else {
        enqueue_dumped_steps(k);
      }
      CK(cudaGetLastError());
      const uint64_t before = steps_done;
      steps_done += k;
      if (checksum_on) {
        rowargs.n = static_cast<uint32_t>(2 * n * k);
        launches += digest.fold_direct(rowargs, rowargs.n, static_cast<uint32_t>(2 * n * B), 4, stream, hash);
      }
      if (params.output_mode != OutputMode::none) record_batch_frames(before, k);
      count -= k;
    }
  }

  // Frames (src/engine.cpp:81-86: steps s with s % stride == 0, s < T) among
  // the batch's rows (row j = the state after step before + j + 1), copied
  // down in one span and widened to the reference's u64 frames.
  void record_batch_frames(uint64_t before, uint64_t k) {
    const uint64_t stride = params.output_stride;
    uint64_t s = (before / stride + 1) * stride;
    if (s > before + k || s >= params.steps) return;
    const uint64_t last = std::min<uint64_t>(before + k, params.steps - 1) / stride * stride;
    const uint64_t j0 = s - before - 1, j1 = last - before - 1;
    if (!hrows) CK(cudaMallocHost(&hrows, size_t(dump_rows()) * 2 * n * 4));
    CK(cudaMemcpyAsync(hrows, dstage + j0 * 2 * n, size_t(j1 - j0 + 1) * 2 * n * 4, cudaMemcpyDeviceToHost,
                       stream));
    CK(cudaStreamSynchronize(stream));
    for (; s <= last; s += stride) {
      const uint32_t* row = hrows + (s - before - 1 - j0) * 2 * n;
      Frame f;
      f.step = s;
      f.positions.assign(row, row + n);
      f.velocities.assign(row + n, row + 2 * n);
      frames.push_back(std::move(f));
    }
  }

  // Starts an asynchronous rank-ordered snapshot into (positions,
  // velocities): a device copy stream-ordered before any later step, then
  // D2H + widening on a host thread (see GpuRing::state_async).
  void snap_start(uint64_t* positions, uint64_t* velocities) {
  Impl& d = *this;
  d.snap_join();  // one snapshot in flight: the staging buffers are reused
  d.drain();
  if (!d.snap_x) {
    CK(cudaMalloc(&d.snap_x, size_t(d.n) * 4));
    CK(cudaMalloc(&d.snap_v, size_t(d.n) * d.vbytes));
  }
  if (!d.snap_hx) {
    CK(cudaMallocHost(&d.snap_hx, size_t(d.n) * 4));
    CK(cudaMallocHost(&d.snap_hv, size_t(d.n) * d.vbytes));
    CK(cudaStreamCreateWithFlags(&d.snap_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&d.snap_ready, cudaEventDisableTiming));
  }
  const int cur = static_cast<int>(d.buf_host);
  CK(cudaMemcpyAsync(d.snap_x, d.x[cur], size_t(d.n) * 4, cudaMemcpyDeviceToDevice, d.stream));
  CK(cudaMemcpyAsync(d.snap_v, d.v[cur], size_t(d.n) * d.vbytes, cudaMemcpyDeviceToDevice, d.stream));
  CK(cudaEventRecord(d.snap_ready, d.stream));
  const uint32_t n = d.n, head = (d.n - d.W_host) % d.n;
  const int vbytes = d.vbytes, device = d.device;
  d.snap_thread = std::thread([&d, positions, velocities, n, head, vbytes, device] {
    try {
      CK(cudaSetDevice(device));
      CK(cudaStreamWaitEvent(d.snap_stream, d.snap_ready, 0));
      // rank r holds id (head + r) mod n: two contiguous pieces
      constexpr uint32_t kChunk = 1u << 24;
      struct Piece { uint32_t r0, r1, id0; cudaEvent_t ev; };
      std::vector<Piece> pieces;
      for (uint32_t r0 = 0; r0 < n;) {
        const uint32_t id0 = head + r0 < n ? head + r0 : head + r0 - n;
        const uint32_t r1 = std::min<uint32_t>({n, r0 + kChunk, r0 + (n - id0)});
        Piece pc{r0, r1, id0, nullptr};
        CK(cudaEventCreateWithFlags(&pc.ev, cudaEventDisableTiming));
        const size_t m = r1 - r0;
        if (positions)
          CK(cudaMemcpyAsync(d.snap_hx + r0, d.snap_x + id0, m * 4, cudaMemcpyDeviceToHost, d.snap_stream));
        if (velocities)
          CK(cudaMemcpyAsync(static_cast<char*>(d.snap_hv) + size_t(r0) * vbytes,
                             static_cast<const char*>(d.snap_v) + size_t(id0) * vbytes, m * vbytes,
                             cudaMemcpyDeviceToHost, d.snap_stream));
        CK(cudaEventRecord(pc.ev, d.snap_stream));
        pieces.push_back(pc);
        r0 = r1;
      }
      cudaError_t err = cudaSuccess;
      for (const Piece& pc : pieces) {
        if (err == cudaSuccess) err = cudaEventSynchronize(pc.ev);
        if (err == cudaSuccess) {
          parallel_chunks(pc.r1 - pc.r0, [&](size_t lo, size_t hi) {
            lo += pc.r0;
            hi += pc.r0;
            if (positions) widen_u32(d.snap_hx + lo, positions + lo, hi - lo);
            if (velocities) {
              if (vbytes == 1) widen_u8(static_cast<const uint8_t*>(d.snap_hv) + lo, velocities + lo, hi - lo);
              else widen_u32(static_cast<const uint32_t*>(d.snap_hv) + lo, velocities + lo, hi - lo);
            }
          });
        }
        cudaEventDestroy(pc.ev);
      }
      CK(err);
    } catch (...) {
      d.snap_error = std::current_exception();
    }
  });
}

  // ---- on-device trajectory checksum ---------------------------------
  // Per step (fnv_kernels.cuh, nibble decomposition): pass A (low-nibble
  // chunk maps) and its composition tree up and down (every chunk's incoming
  // low nibble), pass B (high-nibble maps from it) and its tree (every
  // chunk's incoming low byte), pass C (one exact 64-bit run per slot), the
  // slots' affine maps reduced and applied -- all graph-captured, no host
  // round trip.
  FnvRowDigest digest;

  // Folds the current state's row into the device digest (one graph launch).
  void fnv_fold() { launches += digest.fold(args, n, vbytes, stream, hash); }

  void pull_hash() {
    uint64_t h = 0;
    if (digest.pull(stream, &h)) hash = h;
  }

  // ---- streamed end-to-end job (nasch_sim_job32) -----------------------
  // set_state32(xin, vin) + advance(k) + state32(xout, vout) for k <= K (one
  // temporal-blocked launch) with page-locked arrays, overlapped by ranges
  // of the ring: the positions upload on one stream and the narrowed
  // velocities on another, chunk by chunk; the launch runs as kJobChunks
  // range launches (nasch_tb_range_kernel), range c as soon as chunks c and
  // c+1 (its halo) have landed; each range's cars go back on a third stream
  // into their rank order (the final rank offset is known from the origin-
  // cone plan, computed once chunk 0 and the last chunk are up).  The input
  // lives in its own buffers (jx, jv) until the job validated, so a
  // rejected input leaves the ring as it was; the rules and their order are
  // set_state32's (positions on the device, velocities on the host).
  // Returns false when the streamed form does not apply (the caller then
  // runs the three calls).
  static constexpr uint32_t kJobChunks = 16;  // 4: 41 ms, 8: 35-43, 12: 33, 16: 32, 24: 32, 32: 33 on C3 (NASCH_B200_JOB_CHUNKS)
  bool job32(const uint32_t* xin, const uint32_t* vin, uint64_t steps, uint32_t* xout, uint32_t* vout) {
    const uint64_t k64 = std::min<uint64_t>(steps, params.steps - steps_done);
    auto pinned = [](const void* p) {
      cudaPointerAttributes pa{};
      const bool ok = p && cudaPointerGetAttributes(&pa, p) == cudaSuccess && pa.type == cudaMemoryTypeHost;
      cudaGetLastError();
      return ok;
    };
    if (!jx || checksum_on || params.output_mode != OutputMode::none || k64 == 0 || k64 > K ||
        !pinned(xin) || !pinned(xout) || !vin || !vout)
      return false;
    const uint32_t k = static_cast<uint32_t>(k64);
    drain();
    snap_join();
    if (plan_stale) replan();  // (the saved control block below must be current)
    CK(cudaStreamSynchronize(stream));

    const int cur = static_cast<int>(buf_host);
    CK(cudaMemcpy(hctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost));
    const Ctl saved = *hctl;  // restored if the input is rejected
    RingArgs ja = args;       // reads the job's input buffers, writes the idle ping-pong buffer
    ja.x[cur] = jx;
    ja.v[cur] = jv;
    const uint32_t ntiles = (n + kTbStore - 1) / kTbStore;
    const uint32_t chunks = static_cast<uint32_t>(std::max<long>(2, env_long("NASCH_B200_JOB_CHUNKS", kJobChunks)));
    const uint32_t tpc = (ntiles + chunks - 1) / chunks;  // tiles per chunk
    const uint32_t nch = (ntiles + tpc - 1) / tpc;
    auto cfirst = [&](uint32_t c) { return std::min<uint64_t>(uint64_t(c) * tpc * kTbStore, n); };
    std::vector<cudaEvent_t> ev;
    const bool trace = std::getenv("NASCH_B200_JOB_TRACE") != nullptr;
    std::vector<std::pair<std::string, cudaEvent_t>> tev;
    cudaEvent_t t_start = nullptr;
    const auto host_t0 = std::chrono::steady_clock::now();
    auto host_ms = [&] {
      return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
    };
    if (trace) {
      CK(cudaEventCreate(&t_start));
      CK(cudaEventRecord(t_start, stream));
    }
    auto event = [&](cudaStream_t st) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, trace ? cudaEventDefault : cudaEventDisableTiming));
      CK(cudaEventRecord(e, st));
      ev.push_back(e);
      if (trace) tev.emplace_back(st == jstream[0] ? "x_up" : st == jstream[1] ? "v_up" : st == jstream[2] ? "down" : "comp", e);
      return e;
    };
    // upload order: chunk 0 and the last chunk first (the origin cone needs
    // the first K and the last K vmax ids), then the rest in order
    std::vector<cudaEvent_t> eup(nch), ecomp(nch), edown(nch);
    const uint64_t vlim = std::min<uint64_t>(params.v_max, vmax_eff);
    std::atomic<unsigned long long> vcode{~0ull};
    auto narrow_up = [&](uint32_t c) {
      const uint64_t a = cfirst(c), b = cfirst(c + 1);
      parallel_chunks(b - a, [&](size_t lo, size_t hi) {
        const uint64_t code = narrow_v32(vin, a + lo, a + hi, params.v_max, vlim, hv, vbytes);
        unsigned long long m = vcode.load();
        while (code < m && !vcode.compare_exchange_weak(m, code)) {
        }
      });
      // one upload stream, chunk after chunk (H2D copies of two streams
      // measured serialised: the velocities only moved after every position)
      CK(cudaMemcpyAsync(jx + a, xin + a, (b - a) * 4, cudaMemcpyHostToDevice, jstream[0]));
      CK(cudaMemcpyAsync(static_cast<char*>(jv) + a * vbytes, static_cast<char*>(hv) + a * vbytes,
                         (b - a) * vbytes, cudaMemcpyHostToDevice, jstream[0]));
      eup[c] = event(jstream[0]);
      if (trace) std::fprintf(stderr, "[job32] chunk %u enqueued at host %.2f ms\n", c, host_ms());
    };
    auto wait_chunk = [&](uint32_t c) { CK(cudaStreamWaitEvent(stream, eup[c], 0)); };
    // the control block for the loaded state (W = 0), cleared records, the
    // origin-cone plan from chunk 0 and the last chunk
    narrow_up(0);
    if (nch > 1) narrow_up(nch - 1);
    wait_chunk(0);
    if (nch > 1) wait_chunk(nch - 1);
    {
      Ctl c{};
      c.t = steps_done;
      c.W = 0;
      c.buf = static_cast<unsigned int>(cur);
      c.E = mulmod(seeded(params.seed), powmod(kA, draw_exponent(steps_done, n, 0)));
      c.E2 = mulmod(c.E, args.an_inv);
      *hctl = c;
      CK(cudaMemcpyAsync(ctl, hctl, sizeof(Ctl), cudaMemcpyHostToDevice, stream));
      CK(cudaMemsetAsync(rec, 0, sizeof(StepRec) * kRecCap, stream));
      if (vbytes == 1) cone_init_kernel<uint8_t, 256><<<1, 256, 0, stream>>>(ja);
      else cone_init_kernel<uint32_t, 256><<<1, 256, 0, stream>>>(ja);
      CK(cudaGetLastError());
      ++launches;
      CK(cudaMemcpyAsync(jctl, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, stream));
    }
    cudaEvent_t eplan = event(stream);
    // range launches, each once its chunk and the next have landed
    const int rgrid_max = grid;
    auto launch_range = [&](uint32_t c) {
      TbRange rg{};
      rg.tile0 = c * tpc;
      rg.tile_end = std::min(ntiles, (c + 1) * tpc);
      const uint32_t gr = std::max<uint32_t>(1, std::min<uint32_t>(rg.tile_end - rg.tile0, rgrid_max));
      rg.gpow = powmod(kA, uint64_t(gr) * kTbStore);
      rg.a_tile0 = powmod(kA, uint64_t(rg.tile0) * kTbStore);
      rg.epi = c + 1 == nch ? 1u : 0u;
      if (vbytes == 1)
        nasch_tb_range_kernel<uint8_t, kTbTPB, kTbCPT, kTbHalo, kTbWT><<<gr, kTbTPB, 0, stream>>>(ja, k, rg);
      else
        nasch_tb_range_kernel<uint32_t, kTbTPB, kTbCPT, kTbHalo, kTbWT><<<gr, kTbTPB, 0, stream>>>(ja, k, rg);
      CK(cudaGetLastError());
      ++launches;
      ecomp[c] = event(stream);
    };
    // downloads: once the plan has given the final rank offset
    bool have_head = false;
    uint32_t head_f = 0, W_f = 0;
    uint32_t next_down = 0, launched = 0;
    auto try_head = [&](bool block) {
      if (have_head) return;
      if (!block && cudaEventQuery(eplan) != cudaSuccess) {
        cudaGetLastError();
        return;
      }
      CK(cudaEventSynchronize(eplan));
      uint64_t w = uint64_t(jctl->Wk[k - 1]) + jctl->ck[k - 1];
      if (w >= n) w -= n;
      W_f = static_cast<uint32_t>(w);
      head_f = (n - W_f) % n;
      have_head = true;
    };
    // [a, b) of ids -> up to two rank pieces (r0, id0, m)
    auto pieces_of = [&](uint64_t a, uint64_t b, auto&& fn) {
      if (a >= b) return;
      if (a >= head_f) fn(a - head_f, a, b - a);
      else if (b <= head_f) fn(a + n - head_f, a, b - a);
      else {
        fn(a + n - head_f, a, head_f - a);
        fn(0, head_f, b - head_f);
      }
    };
    const int dst = cur ^ 1;
    auto issue_downloads = [&]() {
      for (; next_down < launched; ++next_down) {
        const uint32_t c = next_down;
        CK(cudaStreamWaitEvent(jstream[2], ecomp[c], 0));
        pieces_of(cfirst(c), cfirst(c + 1), [&](uint64_t r0, uint64_t id0, uint64_t m) {
          CK(cudaMemcpyAsync(reinterpret_cast<char*>(hx) + r0 * vbytes, static_cast<const char*>(v[dst]) + id0 * vbytes,
                             m * vbytes, cudaMemcpyDeviceToHost, jstream[2]));
        });
        pieces_of(cfirst(c), cfirst(c + 1), [&](uint64_t r0, uint64_t id0, uint64_t m) {
          CK(cudaMemcpyAsync(xout + r0, x[dst] + id0, m * 4, cudaMemcpyDeviceToHost, jstream[2]));
        });
        edown[c] = event(jstream[2]);
      }
    };
    for (uint32_t c = 1; c + 1 < nch; ++c) {
      narrow_up(c);
      wait_chunk(c);
      launch_range(c - 1);
      ++launched;
      try_head(false);
      if (have_head) issue_downloads();
    }
    if (nch > 1) {
      launch_range(nch - 2);  // its halo is the last chunk's start (up)
      ++launched;
    }
    launch_range(nch - 1);  // the wrap tiles read chunk 0; the epilogue
    ++launched;
    // the position rules over the whole input (velocities: vcode above)
    CK(cudaMemsetAsync(dcode, 0xff, sizeof(unsigned long long), stream));
    validate_positions_kernel<<<148 * 8, 256, 0, stream>>>(jx, n, L, dcode);
    CK(cudaGetLastError());
    ++launches;
    CK(cudaMemcpyAsync(hcode, dcode, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
    cudaEvent_t evalid = event(stream);
    try_head(true);
    issue_downloads();
    // widen each chunk's velocities into rank order as it lands
    cudaError_t err = cudaSuccess;
    for (uint32_t c = 0; c < nch; ++c) {
      if (err == cudaSuccess) err = cudaEventSynchronize(edown[c]);
      if (err != cudaSuccess) break;
      pieces_of(cfirst(c), cfirst(c + 1), [&](uint64_t r0, uint64_t, uint64_t m) {
        parallel_chunks(m, [&](size_t lo, size_t hi) {
          if (vbytes == 1) widen_u8_u32(reinterpret_cast<const uint8_t*>(hx) + r0 + lo, vout + r0 + lo, hi - lo);
          else std::memcpy(vout + r0 + lo, reinterpret_cast<const uint32_t*>(hx) + r0 + lo, (hi - lo) * 4);
        });
      });
    }
    if (err == cudaSuccess) err = cudaEventSynchronize(evalid);
    if (trace) {
      std::fprintf(stderr, "[job32] host done %.2f ms;", host_ms());
      for (auto& te : tev) {
        float ms = 0;
        cudaEventElapsedTime(&ms, t_start, te.second);
        std::fprintf(stderr, " %s %.2f", te.first.c_str(), ms);
      }
      std::fprintf(stderr, "\n");
      cudaEventDestroy(t_start);
    }
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    CK(err);
    CK(cudaStreamSynchronize(stream));
    const unsigned long long code = std::min<unsigned long long>(*hcode, vcode.load());
    if (code != ~0ull) {
      // rejected: the ring is as it was (its buffers were never written)
      *hctl = saved;
      CK(cudaMemcpyAsync(ctl, hctl, sizeof(Ctl), cudaMemcpyHostToDevice, stream));
      CK(cudaStreamSynchronize(stream));
      plan_stale = true;  // the records of the planned steps are stale: re-plan and clear
      switch (static_cast<int>(code & 3u) + 1) {
        case 1: throw std::invalid_argument("position out of range [0, length)");
        case 2: throw std::invalid_argument("positions must be strictly increasing");
        case 3: throw std::invalid_argument("velocity above vmax");
        default: throw std::invalid_argument("velocity above length-1 (B200 engine restriction)");
      }
    }
    // accepted: the state loaded (set_state's bookkeeping) and k steps done
    series_base = steps_done;
    sumv_host.clear();
    wraps_host.clear();
    sumv0 = 0;
    steps_done += k;
    plan_stale = true;  // the next K-step launch needs its own plan
    drain();            // records, control block (buf, W, t, plan check)
    if (W_host != W_f) throw std::runtime_error("job: rank offset differs from the plan (engine state is invalid)");
    return true;
  }

  // Validates a rank-ordered state (strictly ascending positions < L,
  // velocities <= vmax -- the invariants of acceptance.cpp:118-123 -- and
  // <= L-1) while narrowing it into the pinned staging buffers, in parallel
  // host chunks, then uploads it.
  //
  // Pipelined: 16M-car chunks are converted on all host cores while the
  // previous chunk is in flight to the device.  The upload goes to the idle
  // ping-pong buffer, which becomes current only once every chunk
  // validated, so a rejected state leaves the simulation untouched.
  template <typename T>
  void load_state(const T* hx_in, const T* hv_in) {
    drain();
    std::atomic<int> err{0};
    const uint64_t vlim = std::min<uint64_t>(params.v_max, vmax_eff);
    const int dst = static_cast<int>(buf_host ^ 1u);
    constexpr size_t kChunk = size_t(1) << 24;
    // u32 positions in page-locked memory (cudaMallocHost / cudaHostRegister,
    // e.g. a pinned torch tensor) go to the device straight from the
    // caller's array: validated on the host, no staging copy.
    bool direct_x = false;
    if constexpr (std::is_same<T, uint32_t>::value) {
      cudaPointerAttributes pa{};
      direct_x = cudaPointerGetAttributes(&pa, hx_in) == cudaSuccess && pa.type == cudaMemoryTypeHost;
      cudaGetLastError();
    }
    // Page-locked u32 positions never pass through the host: all of them
    // are queued for DMA at once and validated on the device (rules 1-2);
    // the host only narrows and checks the velocities (rules 3-4) chunk by
    // chunk behind them, and the earliest violation of either wins.  Host
    // memory traffic: 2.0 GB instead of 2.8 GB on BASELINE config 3.
    if constexpr (std::is_same<T, uint32_t>::value) {
      if (direct_x) {
        CK(cudaMemcpyAsync(x[dst], hx_in, size_t(n) * 4, cudaMemcpyHostToDevice, stream));
        if (!dcode) {
          CK(cudaMalloc(&dcode, sizeof(unsigned long long)));
          CK(cudaMallocHost(&hcode, sizeof(unsigned long long)));
        }
        CK(cudaMemsetAsync(dcode, 0xff, sizeof(unsigned long long), stream));
        validate_positions_kernel<<<148 * 8, 256, 0, stream>>>(x[dst], n, L, dcode);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(hcode, dcode, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
        std::atomic<unsigned long long> vcode{~0ull};
        for (size_t c0 = 0; c0 < n && vcode.load() == ~0ull; c0 += kChunk) {
          const size_t c1 = std::min<size_t>(n, c0 + kChunk);
          parallel_chunks(c1 - c0, [&](size_t a, size_t b) {
            const uint64_t c = narrow_v32(hv_in, c0 + a, c0 + b, params.v_max, vlim, hv, vbytes);
            unsigned long long cur_min = vcode.load();
            while (c < cur_min && !vcode.compare_exchange_weak(cur_min, c)) {
            }
          });
          CK(cudaMemcpyAsync(static_cast<char*>(v[dst]) + c0 * vbytes, static_cast<char*>(hv) + c0 * vbytes,
                             (c1 - c0) * vbytes, cudaMemcpyHostToDevice, stream));
        }
        CK(cudaStreamSynchronize(stream));
        const unsigned long long code = std::min<unsigned long long>(*hcode, vcode.load());
        if (code != ~0ull) err.store(static_cast<int>(code & 3u) + 1);
      }
    }
    for (size_t c0 = 0; c0 < n && !err.load() && !direct_x; c0 += kChunk) {
      const size_t c1 = std::min<size_t>(n, c0 + kChunk);
      parallel_chunks(c1 - c0, [&](size_t a, size_t b) {
        int e = 0;
        if constexpr (std::is_same<T, uint64_t>::value) {
          e = narrow_validate(hx_in, hv_in, c0 + a, c0 + b, L, params.v_max, vlim, hx, hv, vbytes);
        } else {
          e = narrow_validate32(hx_in, hv_in, c0 + a, c0 + b, L, params.v_max, vlim, hx, hv, vbytes);
        }
        if (e) {
          int expected = 0;
          err.compare_exchange_strong(expected, e);
        }
      });
      CK(cudaMemcpyAsync(x[dst] + c0, hx + c0, (c1 - c0) * 4, cudaMemcpyHostToDevice, stream));
      CK(cudaMemcpyAsync(static_cast<char*>(v[dst]) + c0 * vbytes, static_cast<char*>(hv) + c0 * vbytes,
                         (c1 - c0) * vbytes, cudaMemcpyHostToDevice, stream));
    }
    CK(cudaStreamSynchronize(stream));
    switch (err.load()) {
      case 1: throw std::invalid_argument("position out of range [0, length)");
      case 2: throw std::invalid_argument("positions must be strictly increasing");
      case 3: throw std::invalid_argument("velocity above vmax");
      case 4: throw std::invalid_argument("velocity above length-1 (B200 engine restriction)");
      default: break;
    }
    buf_host ^= 1u;
    reset_ctl();
    compute_sumv0();
    series_base = steps_done;
    sumv_host.clear();
    wraps_host.clear();
    if (steps_done == 0) {
      frames.clear();
      record_frame_if_due();
    }
  }
};

GpuRing::GpuRing(const SimParams& params) : impl_(new Impl) {
  Impl& d = *impl_;
  params.validate();
  d.params = params;
  if (params.road_length > 2147483647ull) {
    throw std::invalid_argument("length above 2^31-1 is not supported by the B200 engine");
  }
  int ndev = 0;
  const cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    throw std::runtime_error(std::string("no CUDA device available for the B200 engine (") +
                             cudaGetErrorString(e) + ")");
  }
  CK(cudaGetDevice(&d.device));
  d.n = static_cast<uint32_t>(params.car_count);
  d.L = static_cast<uint32_t>(params.road_length);
  d.vmax_eff = static_cast<uint32_t>(std::min<uint64_t>(params.v_max, params.road_length - 1));
  d.vbytes = d.vmax_eff <= 255 ? 1 : 4;

  // Temporal blocking: K steps per launch when the origin cone fits one
  // block and the ring holds at least two full tiles.
  int sms = 0, per_sm = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d.device));
  // Medium rings (fewer than ~4 large tiles per SM) use 512-car tiles so
  // every SM gets work; NASCH_B200_TILE=large|medium forces one.
  const char* tile_env = std::getenv("NASCH_B200_TILE");
  const uint32_t large_tiles = (d.n + kTbStore - 1) / kTbStore;
  d.medium = tile_env ? std::string(tile_env) == "medium" : large_tiles < 4u * uint32_t(sms);
  const int tb_tpb = d.medium ? kTbmTPB : kTbTPB;
  const uint32_t tb_load = d.medium ? kTbmLoad : kTbLoad;
  const long kreq = env_long("NASCH_B200_K", kPlanMax);
  uint32_t K = static_cast<uint32_t>(std::max<long>(1, std::min<long>(kreq, std::min(kPlanMax, kTbHalo))));
  // the plan simulates K (vmax + 1) cone cars on at most 256 threads
  // (inline in the launch's last block when they fit it, tb_plan_inline)
  K = std::min<uint32_t>(K, 256u / (d.vmax_eff + 1));
  (void)tb_tpb;
  d.tb = K >= 2 && d.n >= std::max(4096u, 2 * tb_load) && uint64_t(d.L) > uint64_t(K) * d.vmax_eff;
  d.K = d.tb ? K : 1;
  if (!d.tb) d.medium = false;
  // Small rings run whole chunks of steps in one shared-memory-resident CTA
  // (NASCH_B200_RESIDENT=0 forces the one-step-per-launch kernel instead).
  d.resident = !d.tb && d.n <= kResidentMaxCars && env_long("NASCH_B200_RESIDENT", 1) != 0;
  d.warp_ring = env_long("NASCH_B200_WARPRING", 1) != 0;
  d.quad_ring = env_long("NASCH_B200_QUADRING", 1) != 0;
  d.quad_all = env_long("NASCH_B200_QUADRING", 1) == 2;
  // Medium rings: the distributed-resident kernel (dr_kernel.cuh) keeps the
  // ring in registers on every SM for whole chunks of steps
  // (NASCH_B200_DR=0 disables it).
  std::vector<uint32_t> dr_seg;
  // From 513 cars up (NASCH_B200_DR_MIN raises it): 0.44 us per step from
  // 600 cars on, where the one-CTA shared-memory kernel takes 0.9-1.3 us
  // (tools/small_ring_sweep.py); that kernel remains the path of rings the DR
  // conditions below exclude (u32 velocities, L <= 2 K vmax).
  const long dr_min = std::max(512l, env_long("NASCH_B200_DR_MIN", 512));
  if (d.n > uint64_t(dr_min) && env_long("NASCH_B200_DR", 1) != 0) {
    // 32-step epochs (C2: 4.0e11 vs 3.4e11 at 16 with the four-warp cone)
    const long kreq_dr = env_long("NASCH_B200_K", kDrKMax);
    uint32_t Kd = static_cast<uint32_t>(std::max<long>(1, std::min<long>(kreq_dr, kDrKMax)));
    // the planner simulates 2K-step cones of 2K*(vmax+1) <= 512 cars; the
    // initial plan is one 256-thread block's K-step cone
    Kd = std::min<uint32_t>(Kd, 256 / (d.vmax_eff + 1));
    int coop = 0;
    CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, d.device));
    const uint32_t Gw = std::max<uint32_t>(1, std::min<uint32_t>(uint32_t(sms) - 1, (d.n + 255) / 256));
    // balanced, 16-aligned segments of at least kDrHalo cars (N >= 256 G)
    const uint32_t segsz = (d.n + Gw - 1) / Gw + 16;  // largest segment
    uint32_t cptd = 0;
    // cars per thread by segment size, smallest capacity first (512-thread
    // blocks with 4 or 8 cars per thread measured 3-4 % slower on C2);
    // NASCH_B200_DR_GEOM forces one (index) for experiments
    struct G2 { int tpb; uint32_t cpt; uint32_t cap; const void* fn; };
    // (20 / 24 / 32 cars per thread: the draw as one per-thread base times
    // 2 a^c, QDRAW in dr_kernel.cuh -- rings of 0.56M..1.17M cars)
    const G2 geoms[6] = {
        {kDrTPB, 4, dr_capacity<kDrTPB, 4>(), reinterpret_cast<const void*>(&ring_dr_kernel<uint8_t, kDrTPB, 4>)},
        {kDrTPB, 8, dr_capacity<kDrTPB, 8>(), reinterpret_cast<const void*>(&ring_dr_kernel<uint8_t, kDrTPB, 8>)},
        {kDrTPB, 16, dr_capacity<kDrTPB, 16>(), reinterpret_cast<const void*>(&ring_dr_kernel<uint8_t, kDrTPB, 16>)},
        {kDrTPB, 20, dr_capacity<kDrTPB, 20>(),
         reinterpret_cast<const void*>(&ring_dr_kernel<uint8_t, kDrTPB, 20, true>)},
        {kDrTPB, 24, dr_capacity<kDrTPB, 24>(),
         reinterpret_cast<const void*>(&ring_dr_kernel<uint8_t, kDrTPB, 24, true>)},
        {kDrTPB, 32, dr_capacity<kDrTPB, 32>(),
         reinterpret_cast<const void*>(&ring_dr_kernel<uint8_t, kDrTPB, 32, true>)}};
    const long gforce = env_long("NASCH_B200_DR_GEOM", -1);
    int gi = -1;
    for (int i = 0; i < 6; ++i)
      if ((gforce < 0 || gforce == i) && gi < 0 && segsz <= geoms[i].cap) gi = i;
    if (gi >= 0) cptd = geoms[gi].cpt;
    if (coop && sms >= 2 && cptd && Kd >= 2 && d.vbytes == 1 && uint64_t(d.L) > 2ull * Kd * d.vmax_eff) {
      int occ = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, geoms[gi].fn, geoms[gi].tpb, 0));
      const uint32_t G = Gw;
      if (occ >= 1 && G + 1 <= uint32_t(sms) * uint32_t(occ)) {
        d.dr = true;
        // bound on any single inter-CTA wait (dr_kernel.cuh), seconds
        const long to_s = std::max(1l, env_long("NASCH_B200_DR_TIMEOUT_S", 60));
        const unsigned long long to_ns = static_cast<unsigned long long>(to_s) * 1000000000ull;
        CK(cudaMemcpyToSymbol(c_dr_timeout_ns, &to_ns, sizeof to_ns));
        d.tb = d.medium = d.resident = false;
        d.K = Kd;
        d.dr_G = G;
        d.dr_cpt = cptd;
        d.dr_geom = gi;
        for (uint32_t g = 0; g < G; ++g) dr_seg.push_back(static_cast<uint32_t>(uint64_t(g) * d.n / G) & ~15u);
        dr_seg.push_back(d.n);
      }
    }
  }
  const uint32_t tile = d.tb ? (d.medium ? kTbmStore : kTbStore) : kTile1;
  const uint32_t cpt = d.tb ? (d.medium ? kTbmCPT : kTbCPT) : kCPT1;
  const int tpb = d.tb ? tb_tpb : kTPB;
  const uint32_t ntiles = (d.n + tile - 1) / tile;
  d.npad = ntiles * tile + std::max(kTbLoad, kTile1);  // vector loads of the last tile stay in bounds

  CK(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
  for (int b = 0; b < 2; ++b) {
    CK(cudaMalloc(&d.x[b], size_t(d.npad) * 4));
    CK(cudaMalloc(&d.v[b], size_t(d.npad) * d.vbytes));
  }
  CK(cudaMalloc(&d.ctl, sizeof(Ctl)));
  CK(cudaMalloc(&d.rec, sizeof(StepRec) * kRecCap));
  CK(cudaMalloc(&d.dsum, sizeof(unsigned long long)));
  CK(cudaMallocHost(&d.hx, size_t(d.n) * 4));
  CK(cudaMallocHost(&d.hv, size_t(d.n) * d.vbytes));
  CK(cudaMallocHost(&d.hrec, sizeof(StepRec) * kRecCap));
  CK(cudaMallocHost(&d.hctl, sizeof(Ctl)));

  // Persistent grid: resident blocks on every SM, never more than tiles.
  if (d.tb && d.medium) {
    if (d.vbytes == 1) {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nasch_tb_kernel<uint8_t, kTbmTPB, kTbmCPT, kTbHalo, false>, kTbmTPB, 0));
    } else {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nasch_tb_kernel<uint32_t, kTbmTPB, kTbmCPT, kTbHalo, false>, kTbmTPB, 0));
    }
  } else if (d.tb) {
    if (d.vbytes == 1) {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nasch_tb_kernel<uint8_t, kTbTPB, kTbCPT, kTbHalo, kTbWT>, kTbTPB, 0));
    } else {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nasch_tb_kernel<uint32_t, kTbTPB, kTbCPT, kTbHalo, kTbWT>, kTbTPB, 0));
    }
  } else if (d.vbytes == 1) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nasch_step_kernel<uint8_t, kTPB, kCPT1>, kTPB, 0));
  } else {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nasch_step_kernel<uint32_t, kTPB, kCPT1>, kTPB, 0));
  }
  // Temporal-blocked kernels: several block waves (tb_config.hpp kTbWaves);
  // the one-step kernel stays persistent (HBM-bound, one wave).
  // Block tiles (0.56M-2.3M cars): 2 waves -- fewer, longer-lived blocks pay
  // the per-block plan load and velocity-sum reduction less often (measured,
  // tools/tile_ab.py: N = 1e6 1.88 -> 1.69 us per step, 2e6 2.96 -> 2.54).
  const uint32_t waves =
      d.tb ? static_cast<uint32_t>(std::max<long>(1, env_long("NASCH_B200_WAVES", d.medium ? 2 : kTbWaves))) : 1u;
  d.grid = static_cast<int>(std::max<uint64_t>(
      1, std::min<uint64_t>(ntiles, uint64_t(sms) * std::max(per_sm, 1) * waves)));
  // Test knob: force a grid size, to show results do not depend on the
  // launch geometry (the reference's W-invariance, test_engine.cpp:136-152).
  const long gwant = env_long("NASCH_B200_GRID", 0);
  if (gwant > 0) d.grid = static_cast<int>(std::min<long>(gwant, 1 << 20));

  // Geometry-dependent draw multipliers a^(first id of block / thread).
  std::vector<uint32_t> blk(d.grid), thr(tpb);
  const uint32_t a_tile = powmod(kA, tile);
  blk[0] = 1;
  for (int b = 1; b < d.grid; ++b) blk[b] = mulmod(blk[b - 1], a_tile);
  for (int t = 0; t < tpb; ++t) {
    const uint32_t ofs = !d.tb ? t * cpt : d.medium ? TbMedium::offset(t) : TbLarge::offset(t);
    thr[t] = powmod(kA, ofs);
  }
  CK(cudaMalloc(&d.blkpow, blk.size() * 4));
  CK(cudaMalloc(&d.thrpow, thr.size() * 4));
  CK(cudaMemcpy(d.blkpow, blk.data(), blk.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d.thrpow, thr.data(), thr.size() * 4, cudaMemcpyHostToDevice));

  RingArgs& a = d.args;
  a.x[0] = d.x[0];
  a.x[1] = d.x[1];
  a.v[0] = d.v[0];
  a.v[1] = d.v[1];
  a.n = d.n;
  a.L = d.L;
  a.vmax = d.vmax_eff;
  a.tp = deceleration_threshold(params.p);
  a.s0 = seeded(params.seed);
  a.an = powmod(kA, d.n);
  a.an_inv = powmod(kA, kOrder - (d.n % kOrder));
  a.a1 = powmod(kA, (1 + kOrder - (d.n % kOrder)) % kOrder);
  a.g = powmod(kA, uint64_t(d.grid) * tile);
  a.kplan = (d.tb || d.dr) ? d.K : 0;
  a.nl = d.n;
  a.gofs = 0;
  a.agofs = 1;
  a.sharded = 0;
  a.blkpow = d.blkpow;
  a.thrpow = d.thrpow;
  a.ctl = d.ctl;
  a.rec = d.rec;

  if (d.dr) {
    CK(cudaMalloc(&d.dplans, 2 * sizeof(Ctl)));
    CK(cudaMalloc(&d.dsync, (2 + d.dr_G) * sizeof(unsigned int)));
    CK(cudaMalloc(&d.dmbox, size_t(3) * d.dr_G * 2 * kDrHalo * sizeof(uint32_t)));
    CK(cudaMalloc(&d.dseg, dr_seg.size() * 4));
    CK(cudaMemcpy(d.dseg, dr_seg.data(), dr_seg.size() * 4, cudaMemcpyHostToDevice));
  }

  if (d.tb && !d.medium && d.n >= (1u << 22)) {
    // the streamed job's input buffers (job32), allocated here so a job
    // never pays for them (the velocities come back through the staging hx)
    CK(cudaMalloc(&d.jx, size_t(d.npad) * 4));
    CK(cudaMalloc(&d.jv, size_t(d.npad) * d.vbytes));
    for (cudaStream_t& js : d.jstream) CK(cudaStreamCreateWithFlags(&js, cudaStreamNonBlocking));
    CK(cudaMallocHost(&d.jctl, sizeof(Ctl)));
    CK(cudaMalloc(&d.dcode, sizeof(unsigned long long)));
    CK(cudaMallocHost(&d.hcode, sizeof(unsigned long long)));
  }
  if (d.tb || d.dr) {  // the one-step kernel's geometry (checksum mode, GpuRing::Impl::launch_single)
    int per1 = 0;
    if (d.vbytes == 1) {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, nasch_step_kernel<uint8_t, kTPB, kCPT1>, kTPB, 0));
    } else {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, nasch_step_kernel<uint32_t, kTPB, kCPT1>, kTPB, 0));
    }
    const uint32_t ntiles1 = (d.n + kTile1 - 1) / kTile1;
    d.grid1 = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(ntiles1, uint64_t(sms) * std::max(per1, 1))));
    std::vector<uint32_t> blk1(d.grid1), thr1(kTPB);
    const uint32_t a_tile1 = powmod(kA, kTile1);
    blk1[0] = 1;
    for (int b = 1; b < d.grid1; ++b) blk1[b] = mulmod(blk1[b - 1], a_tile1);
    for (int t = 0; t < kTPB; ++t) thr1[t] = powmod(kA, uint64_t(t) * kCPT1);
    CK(cudaMalloc(&d.blkpow1, blk1.size() * 4));
    CK(cudaMalloc(&d.thrpow1, thr1.size() * 4));
    CK(cudaMemcpy(d.blkpow1, blk1.data(), blk1.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d.thrpow1, thr1.data(), thr1.size() * 4, cudaMemcpyHostToDevice));
    d.args1 = a;
    d.args1.blkpow = d.blkpow1;
    d.args1.thrpow = d.thrpow1;
    d.args1.g = powmod(kA, uint64_t(d.grid1) * kTile1);
    d.args1.kplan = 0;
  }

  // init_state (model.cpp:30-40) on the device.
  const int ib = std::max(1, std::min<int>((d.npad + kTPB - 1) / kTPB, 4096));
  for (int b = 0; b < 2; ++b) {
    if (d.vbytes == 1) {
      init_state_kernel<uint8_t><<<ib, kTPB, 0, d.stream>>>(d.x[b], static_cast<uint8_t*>(d.v[b]), d.n, d.npad, d.L);
    } else {
      init_state_kernel<uint32_t><<<ib, kTPB, 0, d.stream>>>(d.x[b], static_cast<uint32_t*>(d.v[b]), d.n, d.npad, d.L);
    }
  }
  CK(cudaGetLastError());
  d.buf_host = 0;
  d.reset_ctl();
  d.sumv0 = 0;
  CK(cudaStreamSynchronize(d.stream));
  d.record_frame_if_due();
}

// Resources are released by Impl's destructor, so a constructor that throws
// half way (e.g. out of device memory) leaks nothing.
GpuRing::Impl::~Impl() {
  if (snap_thread.joinable()) snap_thread.join();
  cudaSetDevice(device);
  cudaFree(snap_x);
  cudaFree(snap_v);
  cudaFreeHost(snap_hx);
  cudaFreeHost(snap_hv);
  if (snap_ready) cudaEventDestroy(snap_ready);
  if (snap_stream) cudaStreamDestroy(snap_stream);
  if (stream) cudaStreamSynchronize(stream);
  if (graph) cudaGraphExecDestroy(graph);
  for (int b = 0; b < 2; ++b) {
    cudaFree(x[b]);
    cudaFree(v[b]);
  }
  cudaFree(ctl);
  cudaFree(rec);
  cudaFree(dsum);
  cudaFree(blkpow);
  cudaFree(thrpow);
  cudaFree(blkpow1);
  cudaFree(thrpow1);
  cudaFree(dcode);
  cudaFreeHost(hcode);
  cudaFree(draster);
  cudaFree(dstage);
  cudaFree(dctl0);
  cudaFreeHost(hrows);
  if (gbatch) cudaGraphExecDestroy(gbatch);
  cudaFree(jx);
  cudaFree(jv);
  for (cudaStream_t js : jstream)
    if (js) cudaStreamDestroy(js);
  cudaFreeHost(jctl);
  cudaFree(dplans);
  cudaFree(dsync);
  cudaFree(dmbox);
  cudaFree(dseg);
  cudaFreeHost(hx);
  cudaFreeHost(hv);
  cudaFreeHost(hrec);
  cudaFreeHost(hctl);
  if (stream) cudaStreamDestroy(stream);
}

GpuRing::~GpuRing() = default;

void GpuRing::set_state(const uint64_t* x, const uint64_t* v, size_t n) {
  Impl& d = *impl_;
  CK(cudaSetDevice(d.device));
  if (n != d.n) throw std::invalid_argument("state length must equal ncars");
  d.load_state<uint64_t>(x, v);
}

void GpuRing::set_state32(const uint32_t* x, const uint32_t* v, size_t n) {
  Impl& d = *impl_;
  CK(cudaSetDevice(d.device));
  if (n != d.n) throw std::invalid_argument("state length must equal ncars");
  d.load_state<uint32_t>(x, v);
}

void GpuRing::job32(const uint32_t* xin, const uint32_t* vin, size_t n, uint64_t steps, uint32_t* xout,
                    uint32_t* vout) {
  Impl& d = *impl_;
  CK(cudaSetDevice(d.device));
  if (n != d.n) throw std::invalid_argument("state length must equal ncars");
  if (d.job32(xin, vin, steps, xout, vout)) return;
  RingEngine::job32(xin, vin, n, steps, xout, vout);
}

void GpuRing::advance(uint64_t steps) {
  CK(cudaSetDevice(impl_->device));
  impl_->advance(steps, true);
}

void GpuRing::enqueue(uint64_t steps) {
  CK(cudaSetDevice(impl_->device));
  impl_->advance(steps, false);
}

void GpuRing::synchronize() {
  CK(cudaSetDevice(impl_->device));
  impl_->drain();
}

uint64_t GpuRing::steps_done() const { return impl_->steps_done; }
uint64_t GpuRing::checksum() const {
  CK(cudaSetDevice(impl_->device));
  impl_->pull_hash();
  return impl_->hash;
}
const std::vector<Frame>& GpuRing::frames() const {
  impl_->snap_join();  // the last frame may still be in flight
  return impl_->frames;
}
const SimParams& GpuRing::params() const { return impl_->params; }

void GpuRing::observables(double* density, double* mean_velocity, double* flow) {
  Impl& d = *impl_;
  CK(cudaSetDevice(d.device));
  d.drain();
  const uint64_t total = d.sumv_host.empty() ? d.sumv0 : d.sumv_host.back();
  const double n = static_cast<double>(d.params.car_count);
  const double mean = static_cast<double>(total) / n;
  const double dens = n / static_cast<double>(d.params.road_length);
  if (density) *density = dens;
  if (mean_velocity) *mean_velocity = mean;
  if (flow) *flow = dens * mean;
}

void GpuRing::state(uint64_t* positions, uint64_t* velocities) {
  Impl& d = *impl_;
  CK(cudaSetDevice(d.device));
  d.drain();
  // Pipelined: rank-order chunks are copied to pinned staging one after the
  // other and each is widened to u64 on all host cores as soon as its copy
  // lands, while the next is in flight.
  constexpr uint32_t kChunk = 1u << 24;
  const int cur = static_cast<int>(d.buf_host);
  const uint32_t head = (d.n - d.W_host) % d.n;  // id of the rank-0 car
  const uint32_t* xs = d.x[cur];
  const void* vs = d.v[cur];
  struct Piece { uint32_t r0, r1; cudaEvent_t ev; };
  std::vector<Piece> pieces;
  for (uint32_t r0 = 0; r0 < d.n;) {
    const uint32_t id0 = head + r0 < d.n ? head + r0 : head + r0 - d.n;
    const uint32_t r1 = std::min<uint32_t>({d.n, r0 + kChunk, r0 + (d.n - id0)});
    Piece p{r0, r1, nullptr};
    CK(cudaEventCreateWithFlags(&p.ev, cudaEventDisableTiming));
    const size_t m = r1 - r0;
    if (positions) CK(cudaMemcpyAsync(d.hx + r0, xs + id0, m * 4, cudaMemcpyDeviceToHost, d.stream));
    if (velocities)
      CK(cudaMemcpyAsync(static_cast<char*>(d.hv) + size_t(r0) * d.vbytes,
                         static_cast<const char*>(vs) + size_t(id0) * d.vbytes, m * d.vbytes,
                         cudaMemcpyDeviceToHost, d.stream));
    CK(cudaEventRecord(p.ev, d.stream));
    pieces.push_back(p);
    r0 = r1;
  }
  cudaError_t err = cudaSuccess;
  for (const Piece& p : pieces) {
    if (err == cudaSuccess) err = cudaEventSynchronize(p.ev);
    if (err == cudaSuccess) {
      parallel_chunks(p.r1 - p.r0, [&](size_t lo, size_t hi) {
        lo += p.r0;
        hi += p.r0;
        if (positions) widen_u32(d.hx + lo, positions + lo, hi - lo);
        if (velocities) {
          if (d.vbytes == 1) widen_u8(static_cast<const uint8_t*>(d.hv) + lo, velocities + lo, hi - lo);
          else widen_u32(static_cast<const uint32_t*>(d.hv) + lo, velocities + lo, hi - lo);
        }
      });
    }
    cudaEventDestroy(p.ev);
  }
  CK(err);
}

// u32 form (BASELINE's int32 state format): positions are the device's own
// format, so they go by DMA straight into a page-locked caller array (else
// through the pinned staging and a parallel copy); u8 velocities land in the
// staging and are widened to u32 on all host cores as each piece arrives.
// Half the host bytes of the u64 form.  On BASELINE config 3 (1 GB over
// PCIe, 1.6 GB of u32 output) it takes ~23 ms, bound by host memory writes
// (the positions' DMA and the velocity widening share them: measured 15 ms
// for the positions alone, 8 ms for the velocities alone, whatever the
// widening thread count).
void GpuRing::state32(uint32_t* positions, uint32_t* velocities) {
  Impl& d = *impl_;
  CK(cudaSetDevice(d.device));
  d.drain();
  auto pinned = [](const void* p) {
    cudaPointerAttributes pa{};
    const bool ok = p && cudaPointerGetAttributes(&pa, p) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();  // a pageable pointer may leave an error behind on older drivers
    return ok;
  };
  const bool direct_x = pinned(positions);
  const bool direct_v = d.vbytes == 4 && pinned(velocities);
  constexpr uint32_t kChunk = 1u << 24;
  const int cur = static_cast<int>(d.buf_host);
  const uint32_t head = (d.n - d.W_host) % d.n;  // id of the rank-0 car
  const uint32_t* xs = d.x[cur];
  const void* vs = d.v[cur];
  struct Piece { uint32_t r0, r1; cudaEvent_t ev; };
  std::vector<Piece> pieces;
  // velocities first (the host widens each piece while the rest -- and all
  // the positions -- are still in flight), then the positions
  for (int pass = 0; pass < 2; ++pass) {
    for (uint32_t r0 = 0; r0 < d.n;) {
      const uint32_t id0 = head + r0 < d.n ? head + r0 : head + r0 - d.n;
      const uint32_t r1 = std::min<uint32_t>({d.n, r0 + kChunk, r0 + (d.n - id0)});
      const size_t m = r1 - r0;
      if (pass == 0 && velocities) {
        Piece p{r0, r1, nullptr};
        CK(cudaEventCreateWithFlags(&p.ev, cudaEventDisableTiming));
        CK(cudaMemcpyAsync(direct_v ? static_cast<void*>(velocities + r0)
                                    : static_cast<void*>(static_cast<char*>(d.hv) + size_t(r0) * d.vbytes),
                           static_cast<const char*>(vs) + size_t(id0) * d.vbytes, m * d.vbytes,
                           cudaMemcpyDeviceToHost, d.stream));
        CK(cudaEventRecord(p.ev, d.stream));
        pieces.push_back(p);
      }
      if (pass == 1 && positions) {
        Piece p{r0, r1, nullptr};
        CK(cudaEventCreateWithFlags(&p.ev, cudaEventDisableTiming));
        CK(cudaMemcpyAsync((direct_x ? positions : d.hx) + r0, xs + id0, m * 4, cudaMemcpyDeviceToHost,
                           d.stream));
        CK(cudaEventRecord(p.ev, d.stream));
        pieces.push_back(p);
      }
      r0 = r1;
    }
  }
  const size_t nvp = velocities ? pieces.size() - (positions ? (pieces.size() / 2) : 0) : 0;  // velocity pieces

  cudaError_t err = cudaSuccess;
  for (size_t k = 0; k < pieces.size(); ++k) {
    const Piece& p = pieces[k];
    const bool is_v = k < nvp;
    if (err == cudaSuccess) err = cudaEventSynchronize(p.ev);
    if (err == cudaSuccess && (is_v ? !direct_v : !direct_x)) {
      parallel_chunks(p.r1 - p.r0, [&](size_t lo, size_t hi) {
        lo += p.r0;
        hi += p.r0;
        if (!is_v) std::memcpy(positions + lo, d.hx + lo, (hi - lo) * 4);
        else if (d.vbytes == 1) widen_u8_u32(static_cast<const uint8_t*>(d.hv) + lo, velocities + lo, hi - lo);
        else std::memcpy(velocities + lo, static_cast<const uint32_t*>(d.hv) + lo, (hi - lo) * 4);
      });
    }
    cudaEventDestroy(p.ev);
  }
  CK(err);
}

// The device copy is stream-ordered before any later step, so the caller may
// advance at once; the D2H of that copy and the widening run on a host
// thread meanwhile (BASELINE config 5: a 6e7-car snapshot every 1000 steps).
void GpuRing::state_async(uint64_t* positions, uint64_t* velocities) {
  CK(cudaSetDevice(impl_->device));
  impl_->snap_start(positions, velocities);
}

void GpuRing::state_wait() { impl_->snap_join(); }

size_t GpuRing::sumv_series(uint64_t* out, size_t cap) {
  Impl& d = *impl_;
  CK(cudaSetDevice(d.device));
  d.drain();
  const size_t k = std::min(cap, d.sumv_host.size());
  if (out) std::memcpy(out, d.sumv_host.data(), k * sizeof(uint64_t));
  return d.sumv_host.size();
}

size_t GpuRing::wrap_series(uint64_t* out, size_t cap) {
  Impl& d = *impl_;
  CK(cudaSetDevice(d.device));
  d.drain();
  const size_t k = std::min(cap, d.wraps_host.size());
  if (out) std::memcpy(out, d.wraps_host.data(), k * sizeof(uint64_t));
  return d.wraps_host.size();
}

void GpuRing::set_checksum(bool enabled) { impl_->checksum_on = enabled; }
bool GpuRing::checksum_enabled() const { return impl_->checksum_on; }
void* GpuRing::cuda_stream() const { return impl_->stream; }
uint64_t GpuRing::kernel_launches() const { return impl_->launches; }
int GpuRing::velocity_bytes() const { return impl_->vbytes; }
int GpuRing::steps_per_launch() const { return static_cast<int>(impl_->steps_per_launch()); }
void GpuRing::shard_range(uint64_t* first, uint64_t* count) const {
  if (first) *first = 0;
  if (count) *count = impl_->params.car_count;
}

// Selection sampling (Knuth Vol. 2, Algorithm S): cell c is chosen with
// probability need/(L - c), which yields every N-subset of [0, L) with
// equal probability, already sorted.  splitmix64 streams, Lemire's
// multiply-shift for the bounded draw.  Velocities come from a second
// stream.  Deterministic for (L, N, vmax_init, seed).
void fill_uniform_state(uint64_t L, uint64_t N, uint64_t vmax_init, uint64_t seed,
                        uint32_t* x, uint32_t* v) {
  if (N > L || L > 0xffffffffull) throw std::invalid_argument("need N <= L < 2^32");
  auto mix = [](uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  };
  uint64_t s = seed * 0x2545f4914f6cdd1dull + 0x1234567ull;
  uint64_t need = N;
  uint64_t k = 0;
  for (uint64_t c = 0; c < L && need > 0; ++c) {
    const uint64_t left = L - c;
    if (need == left) {  // must take every remaining cell
      for (uint64_t r = c; r < L; ++r) x[k++] = static_cast<uint32_t>(r);
      break;
    }
    const uint64_t r = mix(s) >> 32;  // 32 random bits
    if (((r * left) >> 32) < need) {
      x[k++] = static_cast<uint32_t>(c);
      --need;
    }
  }
  uint64_t sv = seed ^ 0xa5a5a5a5deadbeefull;
  for (uint64_t i = 0; i < N; ++i) {
    v[i] = vmax_init ? static_cast<uint32_t>(((mix(sv) >> 32) * (vmax_init + 1)) >> 32) : 0u;
  }
}

}  // namespace nb200

#ifdef NB_TB_TRACE
extern "C" int nasch_b200_tb_trace(unsigned long long* out, int reset) {
  if (reset) {
    std::vector<unsigned long long> init(64 * 8, 0);
    for (int i = 0; i < 64; ++i) init[i * 8 + 0] = init[i * 8 + 2] = ~0ull;
    return cudaMemcpyToSymbol(nb200::g_tb_trace, init.data(), init.size() * 8) == cudaSuccess ? 0 : 1;
  }
  return cudaMemcpyFromSymbol(out, nb200::g_tb_trace, 64 * 8 * 8) == cudaSuccess ? 0 : 1;
}
#endif

#ifdef NB_DR_TRACE
extern "C" int nasch_b200_dr_trace(unsigned long long* out, size_t n) {
  return cudaMemcpyFromSymbol(out, nb200::g_dr_trace, std::min<size_t>(n, 256 * 8) * 8) == cudaSuccess ? 0 : 1;
}
extern "C" int nasch_b200_cone_cycles(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, nb200::g_cone_cycles, 16) == cudaSuccess ? 0 : 1;
}
extern "C" int nasch_b200_dr_wtrace(unsigned long long* out, size_t n) {
  return cudaMemcpyFromSymbol(out, nb200::g_dr_wtrace, std::min<size_t>(n, 64 * 160 * 4) * 8) == cudaSuccess ? 0 : 1;
}
#endif
