// cone_warp.cuh -- the origin-cone planner (step_kernels.cuh, cone_simulate)
// run by ONE warp with no block barriers: cone slot i = lane * CPW + c lives
// in lane `lane`'s registers, leaders cross lanes by shuffle and the
// per-step crossing count is a warp reduction.  Used by the distributed-
// resident planner (dr_kernel.cuh), whose epochs wait on it.
//
// Slots, draws and outputs are exactly those of cone_simulate: slot i holds
// the car of id (h + N - M + i) mod N with h the rank-0 id, M = kk * vmax
// rear cars (every car that can reach the origin within kk steps) and kk
// leaders ahead; the front slot's missing leader corrupts at most kk slots
// from the front, never the counted rear ones.
#pragma once
#include <cstdint>

#include "step_kernels.cuh"

namespace nb200 {

// Shared-memory power tables of the planner: lin[i] = a^i, step2[c] =
// 2 a^c and step2[kConeSlots + c] = 2 a^(c + N) (the per-step draw-base
// update E' = E a^c [a^N unless W wraps], doubled for mulmod_x2).
constexpr uint32_t kConeSlots = 512;  // 32 lanes x up to 16 cars
struct ConeTab {
  uint32_t lin[kConeSlots];
  uint32_t step2[2 * kConeSlots];
};

// Only lin and step2[0, kConeSlots): for a block planning rings of
// different N (the N-dependent factor is then one more mulmod).
__device__ __forceinline__ void cone_tab_fill_lin(ConeTab& tab) {
  const uint32_t a256 = mulmod(c_pow.lin[255], kA);
  for (uint32_t i = threadIdx.x; i < kConeSlots; i += blockDim.x) {
    const uint32_t a = i < 256 ? c_pow.lin[i] : mulmod(c_pow.lin[i - 256], a256);
    tab.lin[i] = a;
    tab.step2[i] = a << 1;
  }
}

__device__ __forceinline__ void cone_tab_fill(ConeTab& tab, const RingArgs& ra) {
  const uint32_t a256 = mulmod(c_pow.lin[255], kA);
  for (uint32_t i = threadIdx.x; i < kConeSlots; i += blockDim.x) {
    const uint32_t a = i < 256 ? c_pow.lin[i] : mulmod(c_pow.lin[i - 256], a256);
    tab.lin[i] = a;
    tab.step2[i] = a << 1;
    tab.step2[kConeSlots + i] = mulmod(a, ra.an) << 1;
  }
}

// Simulates kk <= 64 steps of the cone (M rear cars + kk leaders) from step
// t with rank offset W over (X, V); writes plan steps [ofs, ofs + kout) --
// W, E, E2 and the crossing count of each -- into out->Wk/Ek/E2k/ck, plus
// out->kplan/E/E2.  Returns (in every lane) W after ofs steps, the first
// planned step's.  Requires M + kk <= 32 * CPW, kout <= 32 and ofs + kout <= kk.
//
// The serial chain of a step is crossing count -> E_{j+1} -> draws ->
// velocities -> crossings: one table lookup and two mulmod_x2; each car's
// multiplier for either side of the rank seam (a^id, a^(id-N)) is
// precomputed, so the seam test selects a register, not a product.
template <typename VT, int CPW, bool kTabN = true>
__device__ uint32_t cone_warp_run(const RingArgs& ra, const uint32_t* X, const VT* V, uint64_t t, uint32_t W,
                                  uint32_t kk, uint32_t M, uint32_t ofs, uint32_t kout, Ctl* out,
                                  const ConeTab& tab) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t N = ra.n, L = ra.L, vmax = ra.vmax, tp = ra.tp;
  const uint32_t C = M + kk;
  const uint32_t id0 = cone_slot_id(N, W, M, 0);
  const uint32_t aid0 = powmod_warp(id0);
  uint32_t E = mulmod(ra.s0, powmod_warp(draw_exponent(t, N, W)));
  uint32_t x[CPW], v[CPW], apA[CPW], apB[CPW], idv[CPW];
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    const uint32_t i = lane * CPW + c;
    const bool act = i < C;
    uint32_t id = id0 + (act ? i : 0u);  // < 2^32: id0 < N < 2^31, i < 256
    const bool wrapped = id >= N;
    if (wrapped) id -= N;
    idv[c] = id;
    x[c] = act ? __ldcg(X + id) : 0u;
    v[c] = act ? static_cast<uint32_t>(__ldcg(V + id)) : 0u;
    uint32_t a = mulmod(aid0, tab.lin[act ? i : 0u]);
    if (wrapped) a = mulmod(a, ra.an_inv);
    apA[c] = a << 1;                         // ids below the seam: E a^id
    apB[c] = mulmod(a, ra.an_inv) << 1;      // at or past it: E a^(id-N)
  }
  const uint32_t an_inv2 = ra.an_inv << 1;
  uint32_t rear = 0;  // bit c: slot counts toward the step's crossings
#pragma unroll
  for (int c = 0; c < CPW; ++c) rear |= (lane * CPW + c < M) ? (1u << c) : 0u;
  // E_{j+1} = E_j * a^c_j [* a^N unless W wraps]: lane l precomputes the
  // candidate for c_j = l while the cars move, so the chain after the
  // crossing count is one shuffle (c_j >= 32 or a wrap: the table path).
  const uint32_t candm = kTabN ? tab.step2[kConeSlots + lane] : 0u;
  const uint32_t an2 = ra.an << 1;
  uint32_t Wj = W, Wofs = W;
  uint32_t rW = 0, rE = 0, rE2 = 0, rc = 0;  // lane j keeps plan step ofs + j
  for (uint32_t j = 0; j < kk; ++j) {
    const uint32_t bound = N - Wj;
    uint32_t xn = __shfl_down_sync(0xffffffffu, x[0], 1);
    if (lane == 31) xn = x[CPW - 1];
    const uint32_t cand = kTabN ? mulmod_x2(candm, E) : mulmod_x2(an2, mulmod_x2(tab.step2[lane], E));
    uint32_t cnt = 0;
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      const uint32_t s = mulmod_x2(idv[c] < bound ? apA[c] : apB[c], E);
      const uint32_t xl = (c + 1 < CPW) ? x[c + 1] : xn;
      // car_rule with the modular headway / position as unsigned min's
      uint32_t d = xl - x[c];
      d = min(d, d + L);
      const int vc = static_cast<int>(min(min(v[c] + 1, vmax), d - 1));
      const int vn = max(vc - (s < tp ? 1 : 0), 0);
      v[c] = static_cast<uint32_t>(vn);
      const uint32_t xs = x[c] + v[c];
      x[c] = min(xs, xs - L);
      cnt += ((rear >> c) & 1u) && xs >= L ? 1u : 0u;
    }
    const uint32_t cj = __reduce_add_sync(0xffffffffu, cnt);
    if (j == ofs) Wofs = Wj;
    if (j >= ofs && lane == j - ofs) {
      rW = Wj;
      rE = E;
      rE2 = mulmod_x2(an_inv2, E);
      rc = cj;
    }
    uint32_t Wn = Wj + cj;
    const bool wrap = Wn >= N;
    if (wrap) Wn -= N;
    const uint32_t fast = __shfl_sync(0xffffffffu, cand, cj & 31u);
    if (cj < 32 && !wrap) {
      E = fast;
    } else if (kTabN) {
      E = mulmod_x2(tab.step2[cj + (wrap ? 0u : kConeSlots)], E);  // cj <= M < kConeSlots
    } else {  // table without the a^N half (cone_tab_fill_lin)
      E = mulmod_x2(tab.step2[cj], E);
      if (!wrap) E = mulmod_x2(an2, E);
    }
    Wj = Wn;
    if (j + 1 == ofs + kout) break;
  }
  if (lane < kout) {
    out->Wk[lane] = rW;
    out->Ek[lane] = rE;
    out->E2k[lane] = rE2;
    out->ck[lane] = rc;
  }
  if (lane == 0) {
    out->kplan = kout;
    out->E = rE;
    out->E2 = rE2;
  }
  return Wofs;
}

// The rear slots need only the cars that can reach the origin within kk
// steps: of the last kk*vmax ranks, the suffix with x >= L - kk*vmax (cars
// behind them cannot cross and never influence them -- influence runs from
// leader to follower).  At moderate density that is a fraction of kk*vmax,
// and the per-lane work shrinks with it.  Requires L > kk*vmax.
template <typename VT, bool kTabN = true>
__device__ uint32_t cone_warp(const RingArgs& ra, const uint32_t* X, const VT* V, uint64_t t, uint32_t W,
                              uint32_t kk, uint32_t ofs, uint32_t kout, Ctl* out, const ConeTab& tab) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t N = ra.n, L = ra.L;
  const uint32_t Mmax = kk * ra.vmax;
  const uint32_t id0 = cone_slot_id(N, W, Mmax, 0);
  uint32_t cnt = 0;
  for (uint32_t i = lane; i < Mmax; i += 32) {
    uint32_t id = id0 + i;
    if (id >= N) id -= N;
    cnt += __ldcg(X + id) >= L - Mmax ? 1u : 0u;
  }
  const uint32_t M = __reduce_add_sync(0xffffffffu, cnt);
  const uint32_t C = M + kk;
  if (C <= 64) return cone_warp_run<VT, 2, kTabN>(ra, X, V, t, W, kk, M, ofs, kout, out, tab);
  if (C <= 128) return cone_warp_run<VT, 4, kTabN>(ra, X, V, t, W, kk, M, ofs, kout, out, tab);
  if (C <= 256) return cone_warp_run<VT, 8, kTabN>(ra, X, V, t, W, kk, M, ofs, kout, out, tab);
  return cone_warp_run<VT, 16, kTabN>(ra, X, V, t, W, kk, M, ofs, kout, out, tab);
}

// ---- four-warp variant ------------------------------------------------------
//
// The same cone simulation spread over 4 warps (128 threads, CPW slots each),
// synchronised by one named barrier per step: a lone warp issues every car
// of the cone itself and is issue-latency bound (~250 ns per step); four
// warps share the cars and each carries the short per-step bookkeeping
// (count -> E) redundantly.  Per step each warp publishes its crossing count
// and its first car's new position in parity-alternating slots.
constexpr int kConeMwThreads = 128;

#ifdef NB_DR_TRACE
// Diagnostic build: cycles spent in the cone step loop and steps run.
__device__ unsigned long long g_cone_cycles[2];
#endif

__device__ __forceinline__ void cone_mw_bar() {
  asm volatile("bar.sync 1, 128;" ::: "memory");
}

// Slot i of the cone is superset entry sofs + i, whose car (x, v) the
// caller staged in shared memory (sx, sv); aid0 = a^(id of slot 0), E0 the
// draw base of step t.
template <int CPW>
__device__ uint32_t cone_mw_run(const RingArgs& ra, const uint32_t* sx, const uint32_t* sv, uint32_t sofs,
                                uint32_t id0, uint32_t aid0, uint32_t E0, uint32_t W, uint32_t kk, uint32_t M,
                                uint32_t ofs, uint32_t kout, Ctl* out, const ConeTab& tab) {
  __shared__ uint4 s_cnt[2];  // per-warp crossing counts, one 16-byte load
  __shared__ uint32_t s_lead[2][4];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t N = ra.n, L = ra.L, vmax = ra.vmax, tp = ra.tp;
  const uint32_t C = M + kk;
  uint32_t x[CPW], v[CPW], apA[CPW], apB[CPW], idv[CPW];
  uint32_t E = E0;
  uint32_t rear = 0;
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    const uint32_t i = tid * CPW + c;
    const bool act = i < C;
    uint32_t id = id0 + (act ? i : 0u);
    const bool wrapped = id >= N;
    if (wrapped) id -= N;
    idv[c] = id;
    x[c] = act ? sx[sofs + i] : 0u;
    v[c] = act ? sv[sofs + i] : 0u;
    uint32_t a = mulmod(aid0, tab.lin[act ? i : 0u]);
    if (wrapped) a = mulmod(a, ra.an_inv);
    apA[c] = a << 1;
    apB[c] = mulmod(a, ra.an_inv) << 1;
    rear |= (i < M) ? (1u << c) : 0u;
  }
  if (lane == 0) s_lead[0][warp] = x[0];
  cone_mw_bar();
#ifdef NB_DR_TRACE
  const long long c_start = clock64();
#endif
  const uint32_t an_inv2 = ra.an_inv << 1;
  const uint32_t candm = tab.step2[kConeSlots + lane];
  uint32_t Wj = W, Wofs = W;
  uint32_t rW = 0, rE = 0, rE2 = 0, rc = 0;  // warp 0, lane j: plan step ofs + j
  for (uint32_t j = 0; j < kk; ++j) {
    const uint32_t par = j & 1u;
    const uint32_t bound = N - Wj;
    uint32_t xn = __shfl_down_sync(0xffffffffu, x[0], 1);
    if (lane == 31) xn = warp < 3 ? s_lead[par][warp + 1] : x[CPW - 1];
    const uint32_t cand = mulmod_x2(candm, E);
    uint32_t cnt = 0;
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      const uint32_t s = mulmod_x2(idv[c] < bound ? apA[c] : apB[c], E);
      const uint32_t xl = (c + 1 < CPW) ? x[c + 1] : xn;
      uint32_t d = xl - x[c];
      d = min(d, d + L);
      const int vc = static_cast<int>(min(min(v[c] + 1, vmax), d - 1));
      const int vn = max(vc - (s < tp ? 1 : 0), 0);
      v[c] = static_cast<uint32_t>(vn);
      const uint32_t xs = x[c] + v[c];
      x[c] = min(xs, xs - L);
      cnt += ((rear >> c) & 1u) && xs >= L ? 1u : 0u;
    }
    const uint32_t wc = CPW == 1 ? __popc(__ballot_sync(0xffffffffu, cnt != 0))
                                 : __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) {
      reinterpret_cast<uint32_t*>(&s_cnt[par])[warp] = wc;
      s_lead[par ^ 1u][warp] = x[0];
    }
    cone_mw_bar();
    const uint4 c4 = s_cnt[par];
    const uint32_t cj = (c4.x + c4.y) + (c4.z + c4.w);
    if (j == ofs) Wofs = Wj;
    if (warp == 0 && j >= ofs && lane == j - ofs) {
      rW = Wj;
      rE = E;
      rE2 = mulmod_x2(an_inv2, E);
      rc = cj;
    }
    uint32_t Wn = Wj + cj;
    const bool wrap = Wn >= N;
    if (wrap) Wn -= N;
    const uint32_t fast = __shfl_sync(0xffffffffu, cand, cj & 31u);
    E = (cj < 32 && !wrap) ? fast : mulmod_x2(tab.step2[cj + (wrap ? 0u : kConeSlots)], E);
    Wj = Wn;
    if (j + 1 == ofs + kout) break;
  }
#ifdef NB_DR_TRACE
  if (tid == 0) {
    atomicAdd(&g_cone_cycles[0], static_cast<unsigned long long>(clock64() - c_start));
    atomicAdd(&g_cone_cycles[1], static_cast<unsigned long long>(ofs + kout));
  }
#endif
  if (warp == 0) {
    if (lane < kout) {
      out->Wk[lane] = rW;
      out->Ek[lane] = rE;
      out->E2k[lane] = rE2;
      out->ck[lane] = rc;
    }
    if (lane == 0) {
      out->kplan = kout;
      out->E = rE;
      out->E2 = rE2;
    }
  }
  return Wofs;
}

// Entry for threads 0..127 of a block (tables with the a^N half).  One
// L2 round trip: the whole superset (the last kk*vmax ranks and kk leaders)
// is staged in shared memory, the active-zone size M counted from it, and
// the two big powers computed while the loads are in flight.
template <typename VT>
__device__ uint32_t cone_mw(const RingArgs& ra, const uint32_t* X, const VT* V, uint64_t t, uint32_t W,
                            uint32_t kk, uint32_t ofs, uint32_t kout, Ctl* out, const ConeTab& tab) {
  __shared__ uint32_t s_x[kConeSlots], s_v[kConeSlots];
  __shared__ uint32_t s_m[4], s_pow[2];
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t N = ra.n, L = ra.L;
  const uint32_t Mmax = kk * ra.vmax;
  const uint32_t S = Mmax + kk;  // <= kConeSlots
  const uint32_t id0max = cone_slot_id(N, W, Mmax, 0);
  uint32_t cnt = 0;
  for (uint32_t i = tid; i < S; i += kConeMwThreads) {
    uint32_t id = id0max + i;
    if (id >= N) id -= N;
    const uint32_t xi = __ldcg(X + id);
    s_x[i] = xi;
    s_v[i] = static_cast<uint32_t>(__ldcg(V + id));
    cnt += (i < Mmax && xi >= L - Mmax) ? 1u : 0u;
  }
  if (warp < 2) {
    const uint32_t r = warp == 0 ? powmod_warp(id0max) : powmod_warp(draw_exponent(t, N, W));
    if (lane == 0) s_pow[warp] = r;
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (lane == 0) s_m[warp] = cnt;
  cone_mw_bar();
  const uint32_t M = s_m[0] + s_m[1] + s_m[2] + s_m[3];
  const uint32_t sofs = Mmax - M;  // the cone starts M ranks before rank 0
  uint32_t id0 = id0max + sofs;
  if (id0 >= N) id0 -= N;
  // a^id0 = a^id0max * a^sofs (times a^-N when id0 wrapped past N-1)
  uint32_t aid0 = mulmod(s_pow[0], tab.lin[sofs]);
  if (id0max + sofs >= N) aid0 = mulmod(aid0, ra.an_inv);
  const uint32_t E0 = mulmod(ra.s0, s_pow[1]);
  const uint32_t C = M + kk;
  if (C <= 128) return cone_mw_run<1>(ra, s_x, s_v, sofs, id0, aid0, E0, W, kk, M, ofs, kout, out, tab);
  if (C <= 256) return cone_mw_run<2>(ra, s_x, s_v, sofs, id0, aid0, E0, W, kk, M, ofs, kout, out, tab);
  return cone_mw_run<4>(ra, s_x, s_v, sofs, id0, aid0, E0, W, kk, M, ofs, kout, out, tab);
}

}  // namespace nb200
