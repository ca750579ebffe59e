/*
 * b200tally.h -- C ABI of the B200-native PUMI-Tally hot path
 * (libb200tally.so, built from paper_2504_19048_b200/csrc/).
 *
 * The boundary is the paper's PIMPL interface (Listing 2 at
 * PAPER.md:265-270) as restated by the reference's Python facade
 * meshtally.MeshTally (tally.py:203-286):
 *
 *   PumiTally(mesh, num_particles, ...)            -> bt_create
 *   initialize_particle_location(double*, size)    -> bt_initialize_particle_location
 *   move_to_next_location(double*, int8_t*, double*, size)
 *                                                  -> bt_move_to_next_location
 *   MeshTally.finalize_batch / flux / grid         -> bt_finalize_batch, bt_read_tally
 *
 * Plain pointers and sizes only.  Buffers are HOST memory when mem_kind ==
 * BT_MEM_HOST (pinned or pageable; copied in and out on the handle's stream)
 * or DEVICE memory on the handle's GPU when mem_kind == BT_MEM_DEVICE
 * (zero-copy, e.g. a torch CUDA tensor's data_ptr()).  Caller buffers are never
 * retained past the call.  Every function returns a bt_status; the message
 * of the last failure on the calling thread is bt_last_error().
 *
 * A handle is not re-entrant; one host thread drives it.  All calls are
 * synchronous with respect to the host unless documented otherwise.
 */
#ifndef B200TALLY_H
#define B200TALLY_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bt_tally bt_tally;

/* Status codes; the Python layer maps them to the reference's exception
 * classes (tally.py:219-222, particles.py:65-73, search.py:513-516). */
typedef enum {
    BT_OK = 0,
    BT_EINVAL = 1,    /* ValueError: bad size / count > capacity / bad argument */
    BT_ERUNTIME = 2,  /* RuntimeError: sweep guard exceeded, no source weight */
    BT_ECUDA = 3,     /* RuntimeError: CUDA failure (message names the call) */
    BT_EINDEX = 4,    /* IndexError: group out of [0, num_groups) */
    BT_ENOMEM = 5     /* MemoryError: device allocation failed */
} bt_status;

enum { BT_MEM_HOST = 0, BT_MEM_DEVICE = 1 };

/* localization modes for bt_initialize_particle_location */
enum {
    BT_LOCATE_GRID = 0, /* uniform-grid candidate search, lowest containing id */
    BT_LOCATE_WALK = 1  /* reference semantics: centroid-0 walk + tie-break
                           (search.py:557-601), bit-exact incl. lost points */
};

/* tally arrays for bt_read_tally / bt_tally_device_ptr */
enum {
    BT_TALLY_BATCH = 0,     /* unfinalized per-bin totals (tally.py:101-104) */
    BT_TALLY_SUM = 1,       /* running sum of normalised batch tallies */
    BT_TALLY_SUM_SQ = 2,    /* running sum of squares */
    BT_TALLY_COL_BATCH = 3, /* collision estimator (bt_transport_run) */
    BT_TALLY_COL_SUM = 4,
    BT_TALLY_COL_SUM_SQ = 5
};

/* options for bt_set_option */
enum {
    BT_OPT_MAX_SWEEPS = 0,   /* sweep guard; <0 -> 2*E + 1000 (search.py:449-450) */
    BT_OPT_DIGEST = 1,       /* 1: record per-particle (element, face) digests */
    BT_OPT_SORT = 2,         /* 1: hand particles to warps in element order */
    BT_OPT_WARP_AGG = 3,     /* __match_any_sync aggregation of tally atomics:
                                0 adaptive (default: when a warp's lanes score the same
                                bins), 1 always, 2 never */
    BT_OPT_BLOCKS_PER_SM = 4, /* walk register budget: 1..3 resident 256-thread CTAs/SM */
    BT_OPT_STAGED = 5,        /* refill: 0 v1 (per-lane loads), 1 stage kernel + cp.async work
                                 list, 2 direct (warp-claimed chunks read from the particle
                                 arrays, no stage kernel) */
    BT_OPT_MOVE_CHUNKS = 6,   /* host inputs: copy/walk pipeline depth (0 = auto, <= 16) */
    BT_OPT_LOCATE_LANES = 7,  /* grid localization: lanes per particle 1..32 (0 = default 2) */
    BT_OPT_EXACT_ONLY = 8,    /* 1: no fp32 pre-filters -- grid localization tests every
                                 candidate exactly, and (with BT_OPT_DIGEST) every exit search
                                 runs the reference's literal arithmetic; for validation */
    BT_OPT_DEFER_INIT = 9,    /* host positions, grid mode, >= 2^20 particles: 1 = the
                                 initialize call returns once the DMA (from the front) and
                                 host threads (from the back, into pinned staging) have read
                                 the caller's buffer; the parked part is copied and localized
                                 by the next call (the move: chunk by chunk, ahead of the walk
                                 chunks that need it); 0 (default, measured faster end to
                                 end): copy it all in the initialize call */
    BT_OPT_STREAM_MOVE = 10   /* host inputs, direct refill, >= 2^22 particles: 1 (default) =
                                 ONE walk launch consumes the move's input chunks as the copy
                                 stream lands them (a stream memory write after each chunk);
                                 0 = one walk launch per chunk */
};

/* Mirrors meshtally.search.TraceSummary (search.py:150-157). */
typedef struct {
    int64_t sweeps;
    int64_t events;
    int64_t reached;
    int64_t boundary_exits;
    int64_t stuck_recoveries;
    int64_t stuck_terminations;
} bt_summary;

/*
 * Upload a mesh and allocate a fixed-capacity particle batch + tally on
 * `device` (MeshTally.__init__, tally.py:211-229; create_batch,
 * create_workspace, create_grid).  Arrays are host memory in the reference
 * layout (TetMesh, mesh.py:73-83): vertices (V,3) f64, elements (E,4) i32,
 * adj_elem (E,4) i32 (-1 = boundary), adj_face (E,4) i8, bbox (2,3) f64,
 * centroid0 = centroids[0] (3) f64 (the localization trial point).
 */
bt_status bt_create(const double *vertices, int64_t num_vertices, const int32_t *elements,
                    const int32_t *adj_elem, const int8_t *adj_face, int64_t num_elements,
                    const double *bbox, const double *centroid0, int64_t num_particles,
                    int32_t num_groups, int32_t device, bt_tally **out);

/*
 * One handle over several GPUs of this process (SURVEY §8b "ndev", §8e;
 * PAPER.md:296): `num_devices` ordinals in `devices`; particles are sharded in
 * contiguous ranges [r*ceil(N/P), (r+1)*ceil(N/P)), the mesh is replicated,
 * each GPU keeps a private tally, and bt_finalize_batch sums the tallies with
 * one NCCL all-reduce over NVLink (ncclCommInitAll; peer copies when NCCL is
 * absent or an ordinal repeats) before the on-device finalize.  Every entry
 * point takes the multi-GPU handle and fans out on one host thread per GPU:
 * host arrays are GLOBAL (the handle slices them), summaries are summed
 * (sweeps: max), particle/digest readouts are gathered, BT_TALLY_BATCH is the
 * sum over GPUs, the source weight follows the reference's rule on the whole
 * move.  Device-memory arguments, the transport and the callback path need a
 * one-GPU handle (BT_EINVAL otherwise); bt_shard exposes the per-GPU handles.
 */
bt_status bt_create_multi(const double *vertices, int64_t num_vertices, const int32_t *elements,
                          const int32_t *adj_elem, const int8_t *adj_face, int64_t num_elements,
                          const double *bbox, const double *centroid0, int64_t num_particles,
                          int32_t num_groups, const int32_t *devices, int32_t num_devices,
                          bt_tally **out);

/* Number of per-GPU shards (1 for a bt_create handle) and shard `index`'s
 * handle and particle range [lo, hi). */
bt_status bt_num_shards(bt_tally *h, int32_t *n);
bt_status bt_shard(bt_tally *h, int32_t index, bt_tally **shard, int64_t *lo, int64_t *hi);

bt_status bt_destroy(bt_tally *h);

/*
 * initialize_particle_location(double* pos, int64_t size)
 * (tally.py:239-245 -> search.py:557-601).  size = number of doubles
 * (3 * count); size % 3 != 0 or count > capacity -> BT_EINVAL.  Resets the
 * batch's recorded source weight.  `summary` (nullable) receives the trial
 * walk's counters in BT_LOCATE_WALK mode, zeros in grid mode.  With HOST
 * positions in grid mode the call returns once the positions have been
 * copied; the localization kernel completes asynchronously, ordered before
 * every later call on the handle (so the next move's input copies overlap it).
 */
bt_status bt_initialize_particle_location(bt_tally *h, const double *positions, int64_t size,
                                          int32_t mem_kind, int32_t mode, bt_summary *summary);

/*
 * move_to_next_location(double* dest, int8_t* flying, double* weights,
 * int64_t size) (tally.py:247-271; load_step particles.py:57-89;
 * trace_and_score search.py:492-517).  size = count of particles; dest holds
 * 3*count doubles (xyz interleaved); groups is nullable (keeps previous
 * groups).  On the first move of a batch the source weight is recorded as the
 * sum of weights of flying particles.  count == 0 -> BT_OK with an all-zero
 * summary (the Python facade returns None).
 */
bt_status bt_move_to_next_location(bt_tally *h, const double *destinations, const int8_t *flying,
                                   const double *weights, const int32_t *groups, int64_t size,
                                   int32_t mem_kind, bt_summary *summary);

/* finalize_batch (tally.py:273-279, _finalize tally.py:83-95).
 * source_weight <= 0 -> use the recorded one (BT_ERUNTIME if none). */
bt_status bt_finalize_batch(bt_tally *h, double source_weight);

/* Copy a tally array (E*G doubles) to host `out` (n must equal E*G). */
bt_status bt_read_tally(bt_tally *h, int32_t which, double *out, int64_t n);

/* Device pointer of a tally array (for an NCCL reduce across GPUs). */
bt_status bt_tally_device_ptr(bt_tally *h, int32_t which, void **ptr);

/* Source weight recorded on the first move of the current batch. */
bt_status bt_get_source_weight(bt_tally *h, double *w);
bt_status bt_set_source_weight(bt_tally *h, double w);
bt_status bt_batches_completed(bt_tally *h, int64_t *n);

/* Particle state readout, [0, count); any output pointer may be NULL. */
bt_status bt_read_particles(bt_tally *h, int64_t count, double *position, int32_t *element,
                            int8_t *alive, int8_t *entry_face, int8_t *stuck, int8_t *outcome,
                            double *seg_total);

/* Per-particle digest + scored-event count of the LAST move (BT_OPT_DIGEST). */
bt_status bt_read_digest(bt_tally *h, int64_t count, uint64_t *digest, int64_t *events);

bt_status bt_set_option(bt_tally *h, int32_t key, int64_t value);

/* Device time of the last call's walk kernel(s), CUDA events on the
 * handle's stream, and the number of kernels the library launched. */
bt_status bt_last_timing(bt_tally *h, float *walk_ms, float *call_ms, int64_t *kernels);

/* Device pointers of the persistent particle state (position (N,3) f64,
 * element i32, alive i8) so a device-side driver (e.g. a transport step in
 * torch) can build the next move's destinations without a host round trip.
 * Valid until bt_destroy; write access only between calls. */
bt_status bt_particle_device_ptrs(bt_tally *h, double **position, int32_t **element,
                                  int8_t **alive);

/* Snapshot / restore of the per-particle state (device-to-device); used by
 * the benchmark to replay one move over an identical start state. */
bt_status bt_save_state(bt_tally *h);
bt_status bt_restore_state(bt_tally *h);

/* Device ordinal and sizes. */
bt_status bt_info(bt_tally *h, int32_t *device, int64_t *num_elements, int64_t *capacity,
                  int32_t *num_groups);

/*
 * Face adjacency of a tet mesh on `device` (build_adjacency, mesh.py:188-235):
 * elements (E,4) i32 host in; adj_elem (E,4) i32 and adj_face (E,4) i8 host
 * out, -1 on the boundary.  Face f of an element is opposite local vertex f.
 * BT_EINVAL (MalformedMeshError) for a face shared by 3+ elements, an element
 * listing a face twice, a duplicated element, or an out-of-range vertex id.
 * Two stable device radix sorts of the face keys (c, then (a,b)).
 */
bt_status bt_build_adjacency(const int32_t *elements, int64_t num_elements, int64_t num_vertices,
                             int32_t device, int32_t *adj_elem, int8_t *adj_face);

/*
 * Listing-1 callback path (trace_batch, search.py:453-489):
 * lockstep sweeps with a caller decision point between the proposal and the
 * commit.  bt_load_step loads a step like load_step (particles.py:57-89);
 * bt_trace_begin checks localization (search.py:440-446); then per sweep
 * bt_trace_propose compacts the flying particles (ascending ids), computes
 * every proposal (_sweep_events, search.py:278-372) and returns the event
 * arrays as DEVICE pointers, valid until bt_trace_commit; the caller may
 * rewrite next_element / particle_done (redirect, kill, resurrect); then
 * bt_trace_commit applies them (_commit_events, search.py:375-419).
 * The loop ends when bt_trace_propose reports flying == 0.
 */
typedef struct {
    int64_t count;            /* events this sweep (ascending particle id) */
    int64_t *particle;
    int32_t *element;
    int8_t *exit_face;        /* -1: the segment ends at the destination */
    double *segment_start;    /* (count,3) */
    double *segment_end;      /* (count,3) */
    double *segment_length;
    int32_t *next_element;    /* writable */
    int8_t *particle_done;    /* writable */
    int32_t *next_proposed;   /* boundary = exit_face >= 0 && next_proposed < 0 */
} bt_sweep_events;

bt_status bt_load_step(bt_tally *h, const double *destinations, const int8_t *flying,
                       const double *weights, const int32_t *groups, int64_t count,
                       int32_t mem_kind);
bt_status bt_trace_begin(bt_tally *h, int32_t score, int64_t max_sweeps);
bt_status bt_trace_propose(bt_tally *h, bt_sweep_events *events, int64_t *flying);
bt_status bt_trace_commit(bt_tally *h);
bt_status bt_trace_end(bt_tally *h, bt_summary *summary);

/* Flux of the track-length (estimator 0) or collision (1) tally on the
 * device (flux, tally.py:123-152): mean (E,G) = (sum/n)/volume, rel_error =
 * sqrt(var/n)/batch_mean (0 where the mean is 0 or n < 2). */
bt_status bt_flux(bt_tally *h, int32_t estimator, const double *volumes, double *mean,
                  double *rel_error);

/* cudaMemcpy for bindings without a CUDA runtime: kind 0 device->host,
 * 1 host->device, 2 device->device. */
bt_status bt_memcpy(void *dst, const void *src, int64_t bytes, int32_t kind);

/* Totals of bt_transport_run, mirroring transport.RunResult (transport.py:422-442). */
typedef struct {
    double source_weight;
    double leaked_weight;
    double absorbed_weight;
    double stuck_weight;
    double track_length_total;
    int64_t collisions;
    int64_t events;
    int64_t sweeps;
    float ms_localization;
    float ms_transport;
} bt_transport_totals;

/*
 * Fixed-source analog multigroup transport on the device (transport.run,
 * transport.py:445-549): per batch, source sampling in
 * `box` (2,3) with isotropic (fixed_direction NULL) or fixed directions,
 * localization, then every particle's whole history in one persistent kernel
 * (flight -> walk with track-length scoring -> collision estimator +
 * scatter/absorb), finalized into the handle's track and collision tallies.
 * Random draws are philox4x64-10 keyed (seed, batch, particle, block)
 * exactly as rng.py:58-64.  Cross sections: sigma_t (G), scatter probability
 * per group (G) and the group CDF (G,G) (XSData, transport.py:83-99).
 */
bt_status bt_transport_run(bt_tally *h, const double *sigma_t, const double *scatter_prob,
                           const double *group_cdf, int32_t num_groups, int64_t num_particles,
                           int64_t num_batches, uint64_t seed, const double *box,
                           const double *fixed_direction, bt_transport_totals *out);

/* Final per-particle direction, group and RNG block counter of the last batch. */
bt_status bt_read_transport_state(bt_tally *h, int64_t count, double *direction, int32_t *group,
                                  uint32_t *rng_block);

/* uniform_block(seed, batch, particle, block) on the device for n keys
 * (4 x u64 each) -> 4n doubles (philox KAT hook). */
bt_status bt_uniform_blocks(const uint64_t *keys, int64_t n, int32_t device, double *out);

/* The transport's log (fn 0), sin (1), cos (2) on the device for n arguments:
 * the restatement of the host libm the reference calls (csrc/glibc_math.cuh;
 * self-test hook).  BT_EINVAL when the library was built without the host
 * libm tables. */
bt_status bt_glibc_math(const double *x, int64_t n, int32_t fn, int32_t device, double *out);

/* ---- standalone tally grids and scoring (tally.py:21-80) ---------------- */

/* create_grid(num_elements, num_groups): a tally-only handle (no mesh, no
 * particles) for bt_score / bt_finalize_batch / bt_read_tally / bt_flux. */
bt_status bt_create_grid(int64_t num_elements, int32_t num_groups, int32_t device,
                         bt_tally **out);
/* score_track_length (kind 0: tally[e*G+g] += w * length) and
 * score_collision (kind 1: += w / sigma_t) for n events; BT_EINDEX for an
 * element/group out of range, BT_EINVAL for sigma_t <= 0 (nothing scored). */
bt_status bt_score(bt_tally *h, int32_t kind, const int32_t *elements, const int32_t *groups,
                   const double *weights, const double *values, int64_t n, int32_t mem_kind);
/* Overwrite a tally array (E*G doubles) from host memory (the writable grid). */
bt_status bt_write_tally(bt_tally *h, int32_t which, const double *in, int64_t n);
bt_status bt_set_batches_completed(bt_tally *h, int64_t n);

/* ---- native mesh ingest and the paper-level ABI -------- */

typedef struct bt_mesh bt_mesh;
/* read_tetmesh (mesh.py:302-331) + TetMesh.from_arrays (mesh.py:109-148):
 * text parsed on all host threads; orientation fixed (local 2<->3 swap),
 * degenerate elements rejected, volumes / centroids / bbox as the reference
 * computes them (bit-identical), adjacency on GPU `device` (< 0: host sort).
 * BT_EINVAL carries MalformedMeshError's message. */
bt_status bt_mesh_read(const char *path, int32_t device, bt_mesh **out);
bt_status bt_mesh_from_arrays(const double *vertices, int64_t num_vertices,
                              const int32_t *elements, int64_t num_elements, int32_t device,
                              bt_mesh **out);
bt_status bt_mesh_info(const bt_mesh *m, int64_t *num_vertices, int64_t *num_elements);
/* Copy out (any pointer may be NULL): vertices (V,3), elements (E,4),
 * adj_elem (E,4), adj_face (E,4), volumes (E), centroids (E,3), bbox (2,3). */
bt_status bt_mesh_arrays(const bt_mesh *m, double *vertices, int32_t *elements,
                         int32_t *adj_elem, int8_t *adj_face, double *volumes, double *centroids,
                         double *bbox);
bt_status bt_mesh_destroy(bt_mesh *m);
/* PumiTally(mesh, num_particles, ...) from a mesh object or a mesh file
 * (tally.py:224-225: a path argument is read with read_tetmesh);
 * the handle keeps a host copy of the mesh for bt_write_vtk. */
bt_status bt_create_from_mesh(const bt_mesh *m, int64_t num_particles, int32_t num_groups,
                              int32_t device, bt_tally **out);
bt_status bt_create_from_file(const char *mesh_filename, int64_t num_particles,
                              int32_t num_groups, int32_t device, bt_tally **out);
/* write(filename) (tally.py:284-286 -> write_vtk, tally.py:159-189):
 * legacy ASCII VTK of the flux, byte-identical to the reference's writer
 * (floats as Python repr).  `volumes` may be NULL for handles made from a
 * mesh object/file.  bt_write_flux_csv: write_flux_csv (tally.py:192-200). */
bt_status bt_write_vtk(bt_tally *h, const char *filename, const double *volumes);
bt_status bt_write_flux_csv(bt_tally *h, const char *filename, const double *volumes);
/* Number of visible CUDA devices (0 without a GPU or driver). */
bt_status bt_device_count(int32_t *n);
/* repr(float(x)) as Python formats it (the writers' number format). */
bt_status bt_format_double(double x, char *out, int32_t cap);

const char *bt_last_error(void);
const char *bt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* B200TALLY_H */
