/* nasch.h -- C interface of the B200 NaSch engine (libnasch_b200.so).
 *
 * Drop-in for the reference's C ABI /root/reference/proj/include/nasch/nasch.h
 * (36 symbols, reference nasch.h:16-127): same names, signatures, enum
 * values, ownership and error conventions.  Each declaration below cites
 * the reference declaration it replaces.  The agent engine runs on the
 * current CUDA device; there is no CPU fallback -- without a GPU,
 * nasch_sim_new* fails with NASCH_ERR_INVALID.
 *
 * Every fallible entry point returns a nasch_status; on failure
 * nasch_last_error() describes it for the calling thread.  Handles are
 * opaque and owned by the caller until the matching _free.
 */
#ifndef NASCH_H
#define NASCH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* reference nasch.h:16-21 */
typedef enum nasch_status {
  NASCH_OK = 0,
  NASCH_ERR_INVALID = 1, /* bad argument, parameter combination or device failure */
  NASCH_ERR_PARSE = 2,   /* malformed parameter text */
  NASCH_ERR_IO = 3       /* file could not be read or written */
} nasch_status;

/* reference nasch.h:23-27 */
typedef enum nasch_output_mode {
  NASCH_OUTPUT_NONE = 0,
  NASCH_OUTPUT_ASCII = 1,
  NASCH_OUTPUT_PGM = 2
} nasch_output_mode;

/* reference nasch.h:29-32, plus the explicit CUDA kind (additive: the
 * reference rejects unknown kinds, capi.cpp:203-207). */
typedef enum nasch_engine_kind {
  NASCH_ENGINE_AGENT = 0,          /* car-array engine (runs on the GPU here) */
  NASCH_ENGINE_GRID_REFERENCE = 1, /* cell-array engine, workers must be 1 */
  NASCH_ENGINE_CUDA = 2            /* same as AGENT, named explicitly */
} nasch_engine_kind;

typedef struct nasch_params nasch_params;
typedef struct nasch_sim nasch_sim;

/* reference nasch.h:37-40 */
const char* nasch_last_error(void);

/* ---- parameter sets (reference nasch.h:42-78) ------------------------ */

/* reference nasch.h:44-47: defaults vmax=5, p=0.13, output=none, stride=1. */
nasch_status nasch_params_new(nasch_params** out);
/* reference nasch.h:49-55: `key = value` text / file. */
nasch_status nasch_params_parse(const char* text, nasch_params** out,
                                unsigned* out_threads);
nasch_status nasch_params_load(const char* path, nasch_params** out,
                               unsigned* out_threads);
void nasch_params_free(nasch_params* params);

/* reference nasch.h:58-66 */
nasch_status nasch_params_set_length(nasch_params* params, uint64_t length);
nasch_status nasch_params_set_ncars(nasch_params* params, uint64_t ncars);
nasch_status nasch_params_set_vmax(nasch_params* params, uint64_t vmax);
nasch_status nasch_params_set_p(nasch_params* params, double p);
nasch_status nasch_params_set_steps(nasch_params* params, uint64_t steps);
nasch_status nasch_params_set_seed(nasch_params* params, uint64_t seed);
nasch_status nasch_params_set_output(nasch_params* params,
                                     nasch_output_mode mode);
nasch_status nasch_params_set_stride(nasch_params* params, uint64_t stride);

/* reference nasch.h:68-75 (0 / NONE for a NULL set) */
uint64_t nasch_params_length(const nasch_params* params);
uint64_t nasch_params_ncars(const nasch_params* params);
uint64_t nasch_params_vmax(const nasch_params* params);
double nasch_params_p(const nasch_params* params);
uint64_t nasch_params_steps(const nasch_params* params);
uint64_t nasch_params_seed(const nasch_params* params);
nasch_output_mode nasch_params_output(const nasch_params* params);
uint64_t nasch_params_stride(const nasch_params* params);

/* reference nasch.h:77-78 */
nasch_status nasch_params_validate(const nasch_params* params);

/* ---- simulations (reference nasch.h:80-122) -------------------------- */

/* reference nasch.h:82-86.  workers >= 1; results are bit-identical for
 * every value (the B200 engine is geometry-independent). */
nasch_status nasch_sim_new(const nasch_params* params, unsigned workers,
                           nasch_sim** out);
/* reference nasch.h:88-90 */
nasch_status nasch_sim_new_kind(const nasch_params* params, unsigned workers,
                                nasch_engine_kind kind, nasch_sim** out);
void nasch_sim_free(nasch_sim* sim);

/* reference nasch.h:93-97: synchronous; clamps at the configured total. */
nasch_status nasch_sim_advance(nasch_sim* sim, uint64_t steps);
nasch_status nasch_sim_run(nasch_sim* sim);

/* reference nasch.h:99-107 (0 for NULL) */
uint64_t nasch_sim_steps_done(const nasch_sim* sim);
uint64_t nasch_sim_checksum(const nasch_sim* sim);
uint64_t nasch_sim_draws(const nasch_sim* sim);
uint64_t nasch_sim_frame_count(const nasch_sim* sim);

/* reference nasch.h:109-113 */
nasch_status nasch_sim_observables(const nasch_sim* sim, double* out_density,
                                   double* out_mean_velocity,
                                   double* out_flow);

/* reference nasch.h:115-118: increasing-position order. */
nasch_status nasch_sim_state(const nasch_sim* sim, uint64_t* positions,
                             uint64_t* velocities, size_t capacity);

/* reference nasch.h:120-122 */
nasch_status nasch_sim_write_ascii(const nasch_sim* sim, const char* path);
nasch_status nasch_sim_write_pgm(const nasch_sim* sim, const char* path);

/* reference nasch.h:126-127 */
unsigned nasch_physical_cores(void);

/* ---- B200 extensions (additive; absent from the reference) ----------- */

/* Replaces the current state with a rank-ordered one: strictly increasing
 * positions < length, velocities <= vmax (and <= length-1).  steps_done,
 * draws and checksum are kept, so it doubles as checkpoint restore; the
 * velocity series restarts.  The reference can only start from its
 * equally spaced init (engine.cpp:52). */
nasch_status nasch_sim_set_state(nasch_sim* sim, const uint64_t* positions,
                                 const uint64_t* velocities, size_t count);
nasch_status nasch_sim_set_state32(nasch_sim* sim, const uint32_t* positions,
                                   const uint32_t* velocities, size_t count);

/* nasch_sim_state (reference nasch.h:115-118) into u32 arrays, BASELINE's
 * int32 state format: half the host bytes of the u64 form; positions reach
 * a page-locked array by DMA with no host pass.  Same rules otherwise. */
nasch_status nasch_sim_state32(const nasch_sim* sim, uint32_t* positions,
                               uint32_t* velocities, size_t capacity);

/* One job end to end: nasch_sim_set_state32(positions_in, velocities_in,
 * count) + nasch_sim_advance(steps) + nasch_sim_state32(positions_out,
 * velocities_out, capacity), with the same results, series and errors as
 * the three calls (a rejected input leaves the simulation as it was).  With
 * page-locked arrays and steps within one temporal-blocked launch the
 * upload, the steps and the download overlap by ranges of the ring; the
 * three calls otherwise.  Either output may be NULL. */
nasch_status nasch_sim_job32(nasch_sim* sim, const uint32_t* positions_in,
                             const uint32_t* velocities_in, size_t count,
                             uint64_t steps, uint32_t* positions_out,
                             uint32_t* velocities_out, size_t capacity);

/* nasch_sim_state (reference nasch.h:115-118) split in two: _async copies
 * the current state on the device and returns; the host transfer and
 * widening into the caller's arrays proceed while the caller advances the
 * simulation, and are complete when nasch_sim_state_wait returns.  At most
 * one snapshot is in flight (a second _async waits for the first).  The
 * arrays must stay valid until the wait. */
nasch_status nasch_sim_state_async(nasch_sim* sim, uint64_t* positions,
                                   uint64_t* velocities, size_t capacity);
nasch_status nasch_sim_state_wait(nasch_sim* sim);

/* The per-step trajectory checksum needs every step's state on the host
 * (serial FNV-1a, engine.cpp:173-181).  On by default, as in the
 * reference; pass 0 to stop folding further steps (checksum() then keeps
 * the value reached). */
nasch_status nasch_sim_set_checksum(nasch_sim* sim, int enabled);

/* Exact velocity sum / mean velocity after each completed step since the
 * last set_state (or since step 0).  *count receives the series length;
 * at most `capacity` values are written. */
nasch_status nasch_sim_sumv_series(const nasch_sim* sim, uint64_t* out,
                                   size_t capacity, size_t* count);
nasch_status nasch_sim_mean_velocity_series(const nasch_sim* sim, double* out,
                                            size_t capacity, size_t* count);
/* Number of cars that crossed the origin in each step. */
nasch_status nasch_sim_wrap_series(const nasch_sim* sim, uint64_t* out,
                                   size_t capacity, size_t* count);

/* Asynchronous advance on the engine's CUDA stream; nasch_sim_synchronize
 * completes it.  Steps that need host work (checksum, frames) still
 * synchronise internally. */
nasch_status nasch_sim_enqueue(nasch_sim* sim, uint64_t steps);
nasch_status nasch_sim_synchronize(nasch_sim* sim);

/* The cudaStream_t the engine launches on (for event timing). */
void* nasch_sim_cuda_stream(const nasch_sim* sim);
/* Kernel launches issued by this simulation so far. */
uint64_t nasch_sim_kernel_launches(const nasch_sim* sim);
/* Steps one step-kernel launch advances (temporal-blocking depth K, or 1
 * for rings too small to block; env NASCH_B200_K caps K). */
unsigned nasch_sim_steps_per_launch(const nasch_sim* sim);

/* Seeded synthetic input: N distinct uniformly chosen cells of [0, L)
 * in increasing order, velocities uniform in [0, vmax_init].  Host-only. */
nasch_status nasch_fill_uniform_state(uint64_t length, uint64_t ncars,
                                      uint64_t vmax_init, uint64_t seed,
                                      uint32_t* positions, uint32_t* velocities);

/* Build identification string. */
const char* nasch_b200_version(void);

/* The integer form of the deceleration test: a draw s decelerates iff
 * s < threshold, which equals double(s)/double(2^31-1) < p for every s
 * (src/model.cpp:51). */
uint32_t nasch_b200_draw_threshold(double p);

/* ---- one ring over several GPUs (extension) ------------------------------
 * nasch_sim_new_kind(params, G, NASCH_ENGINE_CUDA, &sim) with G > 1 splits
 * the ring into G contiguous car segments (the reference's block formula,
 * engine.cpp:31-42) over the visible GPUs of this process; the trajectory is
 * bit-identical for every G.  One process per GPU instead: rank 0 calls
 * nasch_nccl_unique_id, the launcher broadcasts the 128 bytes, and every rank
 * calls nasch_sim_new_distributed.  A distributed sim steps its own segment;
 * the calls that see the whole ring are COLLECTIVE -- every rank makes them,
 * in the same order: advance/run, synchronize, set_state, state,
 * observables, the sumv / mean-velocity / wrap series (whole-ring values on
 * every rank: one all-reduce of the drained steps' records), and frame
 * capture inside advance (every rank records whole-ring frames).  state()
 * broadcasts each segment over NCCL; a rank passing NULL arrays only takes
 * part.  enqueue and the segment calls below are local.  A failure one rank
 * detects outside a collective is raised on every rank at the next
 * collective call.  The trajectory checksum is off by default;
 * nasch_sim_set_checksum(sim, 1) on every rank turns it on (each step's FNV
 * chunk maps are all-gathered over NCCL and every rank composes the
 * whole-ring digest). */
nasch_status nasch_nccl_unique_id(void* out128);
nasch_status nasch_sim_new_distributed(const nasch_params* params, unsigned rank,
                                       unsigned world, const void* nccl_id,
                                       nasch_sim** out);
/* Global car ids this process holds: [first, first + count). */
nasch_status nasch_sim_shard_range(const nasch_sim* sim, uint64_t* first,
                                   uint64_t* count);
/* How the segments exchange their halo and origin-cone records each
 * launch: 0 = one segment (nothing to exchange), 1 = collective (stream-
 * ordered peer copies in one process, NCCL all-gather across processes),
 * 2 = peer memory (the step kernel's last block stores the record into
 * every segment's HBM over NVLink and raises a flag; the default when the
 * GPUs can map each other's memory; env NASCH_B200_XCHG=collective forces
 * 1).  Construction and set_state always use the collective path. */
unsigned nasch_sim_exchange_mode(const nasch_sim* sim);
/* Segment snapshot: the cars this process
 * holds (nasch_sim_shard_range), widened to u64, element k at rank
 * (*first_rank + k) mod N -- each rank writes its own piece of a snapshot
 * with no collective.  On a sim holding the whole ring: nasch_sim_state
 * with *first_rank = 0.  The _async form copies the segment on the device
 * and returns; nasch_sim_state_wait completes the host copy. */
nasch_status nasch_sim_state_segment(nasch_sim* sim, uint64_t* positions,
                                     uint64_t* velocities, size_t capacity,
                                     uint64_t* first_rank);
nasch_status nasch_sim_state_segment32(nasch_sim* sim, uint32_t* positions,
                                       uint32_t* velocities, size_t capacity,
                                       uint64_t* first_rank);
nasch_status nasch_sim_state_segment_async(nasch_sim* sim, uint64_t* positions,
                                           uint64_t* velocities, size_t capacity,
                                           uint64_t* first_rank);
/* Collective set_state from each rank's own segment of the new rank-ordered
 * state (count = this rank's shard_range count); validation of the links
 * between segments and of every rule is agreed over NCCL, so all ranks
 * accept or reject together.  On a sim holding the whole ring: set_state. */
nasch_status nasch_sim_set_state_segment(nasch_sim* sim, const uint64_t* positions,
                                         const uint64_t* velocities, size_t count);

/* ---- ensembles of independent rings (extension) ------------------------
 * One handle advances many independent simulations at once -- BASELINE
 * config 4's fundamental-diagram sweep.  Each ring is exactly the
 * single-ring model with its own parameter set and minstd stream; rings
 * that fit one SM's shared memory (about 57k cars, vmax <= 255) run in one
 * persistent launch, the others on their own engine.  For multi-GPU runs
 * each rank builds an ensemble of its share of the rings. */
typedef struct nasch_ensemble nasch_ensemble;
nasch_status nasch_ensemble_new(const nasch_params* const* params, size_t count,
                                nasch_ensemble** out);
void nasch_ensemble_free(nasch_ensemble* ens);
size_t nasch_ensemble_size(const nasch_ensemble* ens);
nasch_status nasch_ensemble_set_state32(nasch_ensemble* ens, size_t ring,
                                        const uint32_t* positions,
                                        const uint32_t* velocities, size_t count);
/* Every ring's state at once: rings concatenated in ring order, ring r's
 * count = its ncars (total = sum of ncars); validated on all host cores,
 * one upload.  Same rules as nasch_ensemble_set_state32. */
nasch_status nasch_ensemble_set_state_all32(nasch_ensemble* ens, const uint32_t* positions,
                                            const uint32_t* velocities, size_t total);
/* Every ring advances min(steps, its remaining steps). */
nasch_status nasch_ensemble_advance(nasch_ensemble* ens, uint64_t steps);
nasch_status nasch_ensemble_enqueue(nasch_ensemble* ens, uint64_t steps);
nasch_status nasch_ensemble_synchronize(nasch_ensemble* ens);
uint64_t nasch_ensemble_steps_done(const nasch_ensemble* ens, size_t ring);
/* Per ring: exact sum over completed steps of the velocity sum
 * (time-averaged flux = total / (steps * length)). */
nasch_status nasch_ensemble_sumv_totals(const nasch_ensemble* ens, uint64_t* out,
                                        size_t capacity);
/* Per ring: velocity sum after the last completed step. */
nasch_status nasch_ensemble_sumv_last(const nasch_ensemble* ens, uint64_t* out,
                                      size_t capacity);
nasch_status nasch_ensemble_state(const nasch_ensemble* ens, size_t ring,
                                  uint64_t* positions, uint64_t* velocities,
                                  size_t capacity);
void* nasch_ensemble_cuda_stream(const nasch_ensemble* ens);
uint64_t nasch_ensemble_kernel_launches(const nasch_ensemble* ens);

#ifdef __cplusplus
}
#endif

#endif /* NASCH_H */
