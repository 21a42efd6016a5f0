/*
 * nasch_oracle.c -- CPU restatement of the reference NaSch hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 engine: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  The product library
 * (paper_2309_14311_b200/libnasch_b200.so) never links or calls it.
 *
 * Every function restates one piece of the reference implementation
 * (/root/reference/proj, cited as file:line) in plain C with the same
 * 64-bit integer and binary64 arithmetic, so results are bit-identical:
 *
 *   minstd LCG            src/lcg.hpp:21-56, src/lcg.cpp:5-39
 *   init_state            src/model.cpp:30-40
 *   gap_ahead             src/model.hpp:60-65
 *   step_serial           src/model.cpp:42-75   (normative step rule)
 *   step_grid_serial      src/model.cpp:99-129  (cell-array oracle)
 *   FNV-1a-64 row hash    src/engine.hpp:12-36, src/engine.cpp:11-21
 *   measure               src/model.cpp:131-142
 *
 * Parity is pinned against the reference's own golden vectors
 * (tests/test_lcg.cpp, test_model.cpp, test_engine.cpp, test_capi.cpp)
 * and against oracle/_ref (the reference sources compiled unmodified);
 * see tests/test_oracle.py.
 */
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

#define OR_A 48271ull       /* lcg.hpp:22 kDefaultMultiplier */
#define OR_M 2147483647ull  /* lcg.hpp:23 kDefaultModulus = 2^31-1 */
#define OR_FNV_BASIS 14695981039346656037ull /* engine.hpp:12 */
#define OR_FNV_PRIME 1099511628211ull        /* engine.hpp:13 */

/* lcg.cpp:11-16 -- state = seed mod m; 0 escapes to 1 (c = 0). */
uint64_t or_lcg_seeded(uint64_t seed) {
  uint64_t s = seed % OR_M;
  return s == 0 ? 1 : s;
}

/* lcg.hpp:37-46 -- s' = (a*s + c) mod m with c = 0. */
uint64_t or_lcg_next(uint64_t* state) {
  *state = (OR_A * *state) % OR_M;
  return *state;
}

/* lcg.hpp:50-52 -- binary64 quotient state/m. */
double or_uniform01(uint64_t* state) {
  return (double)or_lcg_next(state) / (double)OR_M;
}

/* lcg.cpp:22-39 -- square-and-multiply on the affine pair (A, C).  The
 * default generator has c = 0, but the pair is kept to mirror the
 * reference's general form. */
void or_jump_coefficients(uint64_t draws, uint64_t* out_mul, uint64_t* out_add) {
  uint64_t mul = 1 % OR_M, add = 0;
  uint64_t bmul = OR_A % OR_M, badd = 0;
  for (uint64_t k = draws; k > 0; k >>= 1) {
    if (k & 1) {
      mul = (bmul * mul) % OR_M;
      add = (bmul * add + badd) % OR_M;
    }
    badd = (bmul * badd + badd) % OR_M;
    bmul = (bmul * bmul) % OR_M;
  }
  *out_mul = mul;
  *out_add = add;
}

/* lcg.cpp:18-20 + lcg.hpp:54-56 -- jump = apply(jump_coefficients). */
uint64_t or_lcg_jump(uint64_t state, uint64_t draws) {
  uint64_t mul, add;
  or_jump_coefficients(draws, &mul, &add);
  return (mul * state + add) % OR_M;
}

/* model.cpp:30-40 -- x_i = floor(i*L/N), v_i = 0. */
void or_init_state(uint64_t L, uint64_t N, uint64_t* x, uint64_t* v) {
  for (uint64_t i = 0; i < N; ++i) {
    x[i] = i * L / N;
    v[i] = 0;
  }
}

/* model.hpp:60-65 */
uint64_t or_gap_ahead(const uint64_t* x, size_t n, uint64_t L, size_t i) {
  uint64_t ahead = x[i + 1 == n ? 0 : i + 1];
  return (ahead + L - x[i] - 1) % L;
}

static uint64_t or_min(uint64_t a, uint64_t b) { return a < b ? a : b; }

/* Rotate the last k elements of a[0..n) to the front (std::rotate with
 * middle = end - k, model.cpp:70-73). */
static void or_rotate_suffix(uint64_t* a, size_t n, size_t k, uint64_t* tmp) {
  if (k == 0 || k == n) return;
  memcpy(tmp, a + (n - k), k * sizeof(uint64_t));
  memmove(a + k, a, (n - k) * sizeof(uint64_t));
  memcpy(a, tmp, k * sizeof(uint64_t));
}

/* model.cpp:42-75 -- the normative synchronous step.  One draw per car
 * in ascending (rank) order, evaluated before the `v > 0` test so it is
 * always consumed.  `tmp` must hold n values (rotation scratch). */
size_t or_step_serial(uint64_t* x, uint64_t* v, size_t n, uint64_t L,
                      uint64_t vmax, double p, uint64_t* rng, uint64_t* tmp) {
  for (size_t i = 0; i < n; ++i) {
    uint64_t vi = or_min(v[i] + 1, vmax);
    vi = or_min(vi, or_gap_ahead(x, n, L, i));
    double u = or_uniform01(rng);
    if (u < p && vi > 0) --vi;
    v[i] = vi;
  }
  size_t wrapped = 0;
  for (size_t i = 0; i < n; ++i) {
    uint64_t xi = x[i] + v[i];
    if (xi >= L) {
      xi -= L;
      ++wrapped;
    }
    x[i] = xi;
  }
  or_rotate_suffix(x, n, wrapped, tmp);
  or_rotate_suffix(v, n, wrapped, tmp);
  return wrapped;
}

/* model.cpp:99-129 -- cell-array step; cells[x] = velocity or -1.
 * Draws are consumed in ascending cell order (= rank order). */
void or_step_grid_serial(int64_t* cells, uint64_t L, uint64_t vmax, double p,
                         uint64_t* rng) {
  size_t n = 0;
  for (uint64_t x = 0; x < L; ++x) n += cells[x] != -1;
  uint64_t* occ = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  uint64_t* vel = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  size_t k = 0;
  for (uint64_t x = 0; x < L; ++x)
    if (cells[x] != -1) occ[k++] = x;
  for (size_t i = 0; i < n; ++i) {
    uint64_t x = occ[i];
    uint64_t ahead = occ[i + 1 == n ? 0 : i + 1];
    uint64_t gap = (ahead + L - x - 1) % L;
    uint64_t vi = or_min((uint64_t)cells[x] + 1, vmax);
    vi = or_min(vi, gap);
    double u = or_uniform01(rng);
    if (u < p && vi > 0) --vi;
    vel[i] = vi;
  }
  for (uint64_t x = 0; x < L; ++x) cells[x] = -1;
  for (size_t i = 0; i < n; ++i) cells[(occ[i] + vel[i]) % L] = (int64_t)vel[i];
  free(occ);
  free(vel);
}

/* engine.hpp:15-36 -- FNV-1a 64 over the 8 little-endian bytes of one
 * value.  Restated bytewise (the reference's <2^32 fast path is an
 * algebraic shortcut of exactly this, test_engine.cpp:85-98). */
uint64_t or_fnv1a64_value(uint64_t hash, uint64_t value) {
  for (int b = 0; b < 8; ++b) {
    hash = (hash ^ (value & 0xffu)) * OR_FNV_PRIME;
    value >>= 8;
  }
  return hash;
}

/* engine.cpp:11-21 -- positions then velocities, rank order. */
uint64_t or_hash_row(uint64_t hash, const uint64_t* x, const uint64_t* v, size_t n) {
  for (size_t i = 0; i < n; ++i) hash = or_fnv1a64_value(hash, x[i]);
  for (size_t i = 0; i < n; ++i) hash = or_fnv1a64_value(hash, v[i]);
  return hash;
}

/* model.cpp:131-142 -- exact integer sum, then binary64. */
double or_mean_velocity(const uint64_t* v, size_t n) {
  uint64_t total = 0;
  for (size_t i = 0; i < n; ++i) total += v[i];
  return (double)total / (double)n;
}

/*
 * engine.cpp:101-184 semantics (== step_serial per test_engine.cpp:117-134)
 * for `steps` steps from the given rank-ordered state.  `rng` is the
 * generator state before the first draw of the first step (for a fresh
 * run: or_lcg_seeded(seed); to resume at step t: jump by t*N).
 * Optional outputs: per-step exact sum of velocities after each step,
 * per-step crossing count, the running checksum (FNV over every step's
 * row, starting from *checksum).
 */
int or_run(uint64_t L, uint64_t vmax, double p, uint64_t* rng, uint64_t steps,
           uint64_t* x, uint64_t* v, size_t n, uint64_t* sumv_series,
           uint64_t* wrap_series, uint64_t* checksum) {
  uint64_t* tmp = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
  if (!tmp) return 1;
  for (uint64_t t = 0; t < steps; ++t) {
    size_t w = or_step_serial(x, v, n, L, vmax, p, rng, tmp);
    if (wrap_series) wrap_series[t] = w;
    if (sumv_series) {
      uint64_t s = 0;
      for (size_t i = 0; i < n; ++i) s += v[i];
      sumv_series[t] = s;
    }
    if (checksum) *checksum = or_hash_row(*checksum, x, v, n);
  }
  free(tmp);
  return 0;
}

/*
 * The BASELINE.json input generator: seeded
 * uniform DISTINCT sorted positions by selection sampling over the cells
 * 0..L-1 (cell c is taken with probability need/left, decided on 32
 * splitmix64 bits as floor(r * left / 2^32) < need), and velocities
 * uniform in [0, vmax_init] from a second splitmix64 stream.  This is not
 * a reference function -- the reference only has init_state -- but the
 * generator that feeds BOTH arms of the benchmark; it is restated here so
 * the reference arm (bench.py --impl reference) never loads the product
 * library.  tests/test_oracle.py checks it equal to
 * nasch_fill_uniform_state of libnasch_b200.so.  Returns 0, or 1 if
 * N > L or L >= 2^32.
 */
static uint64_t or_splitmix64(uint64_t* s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

int or_fill_uniform_state(uint64_t L, uint64_t N, uint64_t vmax_init, uint64_t seed,
                          uint32_t* x, uint32_t* v) {
  if (N > L || L > 0xffffffffull) return 1;
  uint64_t s = seed * 0x2545f4914f6cdd1dull + 0x1234567ull;
  uint64_t need = N, k = 0, c = 0;
  while (need > 0 && c < L) {
    const uint64_t left = L - c;
    if (need == left) { /* every remaining cell is taken */
      while (c < L) x[k++] = (uint32_t)c++;
      break;
    }
    const uint64_t r = or_splitmix64(&s) >> 32;
    if (((r * left) >> 32) < need) {
      x[k++] = (uint32_t)c;
      --need;
    }
    ++c;
  }
  uint64_t sv = seed ^ 0xa5a5a5a5deadbeefull;
  for (uint64_t i = 0; i < N; ++i)
    v[i] = vmax_init ? (uint32_t)(((or_splitmix64(&sv) >> 32) * (vmax_init + 1)) >> 32) : 0u;
  return 0;
}
