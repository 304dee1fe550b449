/*
 * bh.h -- C-ABI of libbh.so, the B200-native (sm_100a) Barnes-Hut step.
 *
 * Plain pointers and sizes only.  Every pointer argument named d_* is a CUDA
 * device pointer; `stream` is a cudaStream_t (NULL = legacy default stream).
 * Calls return a bh_status; bh_last_error() gives the message of the last
 * failure on the calling thread.  Device-side failures (out-of-domain body,
 * duplicate keys, ...) are latched in a device flag and surface at the next
 * call that synchronises (bh_check, bh_build_*, bh_sim_*), exactly once.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/nbsim/<file>:<line>).  The reference is Python; its
 * "FFI" for this path is the ctypes binding in paper_2203_08966_b200/_lib.py
 * (see INTEGRATION.md).
 *
 * Layouts.  fp32 mode: bodies are float4 {x, y, z, mass} (16 B), velocities and
 * accelerations float4 {x, y, z, 0}.  fp64 mode: positions/velocities/
 * accelerations are double[n][3], masses double[n] -- the reference's own
 * `Bodies` layout (physics.py:18-51).
 */
#ifndef BH_H
#define BH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bh_handle bh_handle;

typedef enum {
  BH_OK = 0,
  BH_BAD_ARG = 1,          /* simulation.py:95-113 config validation */
  BH_OUT_OF_DOMAIN = 2,    /* morton.py:116-118 "outside domain" */
  BH_DUPLICATE_KEY = 3,    /* hashed.py:477-482 "tree resolution" */
  BH_UNSORTED = 4,         /* hashed.py:475-476 "sorted" */
  BH_DEPTH_OVERFLOW = 5,   /* octree.py:144-146 */
  BH_STACK_OVERFLOW = 6,   /* flattree.py:255 (stack cap 176); here the walk's per-warp frontier bound */
  BH_CUDA_ERROR = 7,
  BH_NCCL_ERROR = 8,
  BH_NO_TREE = 9,
  BH_OUT_OF_MEMORY = 10
} bh_status;

typedef enum { BH_FP32 = 0, BH_FP64 = 1 } bh_precision;

typedef struct {
  int64_t n_bodies;
  int64_t n_cells;       /* cells of the last build (== len(FlatTree)) */
  int64_t max_level;     /* deepest cell level of the last build */
  int64_t pp;            /* body-body interactions of the last traversal */
  int64_t pc;            /* body-cell interactions of the last traversal */
  int64_t work;          /* pp*WORK_PP + pc*WORK_PC (octree.py:23-25) */
  int64_t launches;      /* libbh kernels enqueued since the last bh_timing_reset */
  int64_t n_records;     /* fp32 walk records of the current tree (0 if none built) */
} bh_stats;

/* Phases timed with CUDA events on the caller's stream when timing is on. */
enum {
  BH_PHASE_INTEGRATE = 0, /* kick + drift + bounds reduction (+ final kick) */
  BH_PHASE_KEYS = 1,      /* R + Morton keys */
  BH_PHASE_SORT = 2,      /* radix sort of (key, index) */
  BH_PHASE_PERMUTE = 3,   /* body gather into Morton order */
  BH_PHASE_BUILD = 4,     /* lcp, scan, cell count, emit, moments, fp32 walk records */
  BH_PHASE_WALK = 5,      /* traversal */
  BH_PHASE_LET = 6,       /* locally-essential-tree marking and packing (distributed build) */
  BH_NPHASES = 7
};

/* ---- lifecycle ---------------------------------------------------------- */
int bh_create(bh_handle **out, int device, int precision);
int bh_destroy(bh_handle *h);
const char *bh_last_error(void);
int bh_version(void);
/* Synchronise `stream` and return (and clear) any latched device-side error. */
int bh_check(bh_handle *h, void *stream);

/* ---- building blocks (reference: morton.py, hashed.py, flattree.py) ----- */

/* morton.py:33-42 DomainBounds.from_positions: *d_R = 1.001*max|x| (or 1.0).
 * Result stays on the device (no host sync). */
int bh_bounds_f32(bh_handle *h, const float *d_pos4, int64_t n, double *d_R, void *stream);
int bh_bounds_f64(bh_handle *h, const double *d_pos3, int64_t n, double *d_R, void *stream);

/* morton.py:109-125 morton_keys: 63-bit keys, fp64 floor quantisation. */
int bh_morton_f32(bh_handle *h, const float *d_pos4, int64_t n, const double *d_R,
                  uint64_t *d_keys, void *stream);
int bh_morton_f64(bh_handle *h, const double *d_pos3, int64_t n, const double *d_R,
                  uint64_t *d_keys, void *stream);

/* morton.py:128-130 sort_order: stable ascending argsort of 63-bit keys. */
int bh_sort(bh_handle *h, const uint64_t *d_keys, int64_t n, uint64_t *d_keys_sorted,
            int64_t *d_perm, void *stream);

/* The single-pass u32 prefix sum the build uses (cells per body -> pre-order
 * offsets, hashed.py:489 `1 + depth[0] + sum(depth - lcp)`): exclusive
 * (inclusive != 0: inclusive) scan of d_in into d_out, mod 2^32. */
int bh_scan_u32(bh_handle *h, const uint32_t *d_in, int64_t n, uint32_t *d_out, int inclusive,
                void *stream);

/* hashed.py:448-515 build_hashed over Morton-sorted bodies (moments included).
 * The tree stays in the handle.  Synchronises once (cell count). */
int bh_build_f32(bh_handle *h, const float *d_pos4_sorted, int64_t n, const double *d_R,
                 void *stream);
int bh_build_f64(bh_handle *h, const double *d_pos3_sorted, const double *d_mass_sorted,
                 int64_t n, const double *d_R, void *stream);
int bh_tree_size(bh_handle *h, int64_t *n_cells);
/* Sync-free variant for multi-rank steps: d_out[0] = 1 if the last sync-free
 * build fits its cell capacity, else 0 (call bh_tree_size to grow the capacity
 * and build again).  Lets a caller fold the check into one host read with its
 * own device values (the replicated step reads it with its costzones cuts). */
int bh_sim_tree_fits_dev(bh_handle *h, int32_t *d_out, void *stream);
/* Bucket-mode extension: bodies with identical Morton keys share
 * one level-21 cell that is resolved body by body, instead of the reference's
 * "tree resolution" error (hashed.py:477-482).  Off by default for
 * bh_build_*; the resident bh_sim_* path enables it whenever leaf_size > 1. */
int bh_set_allow_duplicates(bh_handle *h, int allow);

/* flattree.py:34-52 FlatTree arrays of the current tree (pre-order).
 * Any pointer may be NULL to skip that array.  Shapes: centre/com [C][3],
 * quad [C][6] (xx,xy,xz,yy,yz,zz), children [C][8] (-1 = absent). */
int bh_export_tree(bh_handle *h, uint64_t *d_key, int8_t *d_level, double *d_centre,
                   double *d_side, double *d_mass, double *d_com, double *d_quad,
                   int64_t *d_count, int32_t *d_children, void *stream);

/* flattree.py:142-166 FlatTree.traverse against the current tree.
 * leaf_size <= 1 is the reference walk; leaf_size > 1 resolves cells of
 * <= leaf_size bodies that fail the MAC body by body.
 * Targets may be in any order (they are Morton-ordered internally). */
int bh_traverse_f32(bh_handle *h, const float *d_targets4, int64_t n, double theta,
                    double eps, int leaf_size, float *d_acc4, int64_t *d_work,
                    void *stream);
int bh_traverse_f64(bh_handle *h, const double *d_targets3, int64_t n, double theta,
                    double eps, int leaf_size, double *d_acc3, int64_t *d_work,
                    void *stream);

/* integrator.py:37-44 kick / drift (in place). */
int bh_kick_f32(bh_handle *h, float *d_vel4, const float *d_acc4, int64_t n, double dt, void *stream);
int bh_drift_f32(bh_handle *h, float *d_pos4, const float *d_vel4, int64_t n, double dt, void *stream);
int bh_kick_f64(bh_handle *h, double *d_vel3, const double *d_acc3, int64_t n, double dt, void *stream);
int bh_drift_f64(bh_handle *h, double *d_pos3, const double *d_vel3, int64_t n, double dt, void *stream);

/* physics.py:288-295 direct_accelerations and physics.py:322-324
 * potential_energy (O(n^2), fp64; validation / energy audit). */
int bh_direct_f64(bh_handle *h, const double *d_pos3, const double *d_mass, int64_t n,
                  double eps, double *d_acc3, void *stream);
int bh_potential_f64(bh_handle *h, const double *d_pos3, const double *d_mass, int64_t n,
                     double eps, double *d_pot, void *stream);

/* ---- resident simulation (simulation.py:478-504 `_drive`, algorithm 1) ---
 * Bodies live in the handle in Morton order between steps; `id` tracks the
 * caller's order.  load/store copy device buffers in caller order (the layout
 * of the handle's precision). */
int bh_sim_load(bh_handle *h, const void *d_pos, const void *d_vel, const double *d_mass,
                const void *d_acc, int64_t n, void *stream);
/* One force evaluation at the current positions (the bootstrap pass of
 * simulation.py:487); record_work mirrors simulation.py:394-395. */
int bh_sim_forces(bh_handle *h, double theta, double eps, int leaf_size, int record_work,
                  void *stream);
/* `steps` KDK steps: kick(dt/2), drift(dt), forces, kick(dt/2). */
int bh_sim_step(bh_handle *h, double dt, double theta, double eps, int leaf_size, int steps,
                void *stream);
int bh_sim_store(bh_handle *h, void *d_pos, void *d_vel, void *d_acc, int64_t *d_work,
                 void *stream);
/* One call from host arrays (fp32 handles): load pos4 (x, y, z, m; n x 4),
 * vel3 and acc3 (n x 3), run `steps` KDK steps (simulation.py:492-502), and
 * write the state back in the caller's order; work (optional, n int32) gets
 * the last force pass's per-body work pp + 2 pc (simulation.py:394-395,
 * octree.py:23-25).  For one step the positions are copied back under the
 * force computation.  Pinned host memory makes the copies asynchronous.  The
 * results are complete once the stream has synchronised. */
int bh_sim_step_host(bh_handle *h, float *pos4, float *vel3, float *acc3, int32_t *work, int64_t n,
                     double dt, double theta, double eps, int leaf_size, int steps, void *stream);

/* The same step in phases, for a multi-GPU driver that exchanges between them
 * (simulation.py:492-502 with the force pass split at the walk):
 *   begin_step : kick(dt/2) + drift(dt) + bounds reduction
 *   prepare    : keys, sort, body permutation, build (+ fp32 walk tree)
 *   walk_range : forces on Morton-sorted targets [begin, end) (the rank's
 *                costzones range, decomposition.py:35-57)
 *   scatter_work / end_step : work to caller order; kick(dt/2)
 * bh_sim_buffers exposes the resident device arrays (Morton order: pos, acc,
 * work; id = caller index of each sorted body; work in caller order) so the
 * driver can exchange them with NCCL. */
int bh_sim_begin_step(bh_handle *h, double dt, void *stream);
int bh_sim_prepare(bh_handle *h, double theta, double eps, int leaf_size, int bounds_ready,
                   void *stream);
int bh_sim_walk_range(bh_handle *h, double theta, double eps, int leaf_size, int64_t begin,
                      int64_t end, int record_work, void *stream);
int bh_sim_scatter_work(bh_handle *h, void *stream);
int bh_sim_end_step(bh_handle *h, double dt, void *stream);
/* Replicated ranks over NVLink peer memory (replaces the all-reduce of the zone
 * accelerations and work that follows _BroadcastTreeForces' per-rank walk,
 * simulation.py:370-416, decomposition.py:35-57): with peers set, walk_range
 * also stores its rows of acc / work into every peer's resident buffers, so
 * after a stream-ordered barrier every rank holds the full results.
 *   ipc_handles : 2 x 64 bytes (cudaIpcMemHandle_t of this handle's resident
 *                 acc and work buffers; valid until the next sim_load)
 *   set_peers   : open npeers (<= 7) such handle pairs; npeers = 0 closes them
 *   set_peer_ptrs: the same from raw device pointers (ranks in one process)
 * A load that reallocates the result buffers invalidates the mapping: walk_range
 * then fails (BH_BAD_ARG) until every rank sets its peers again. */
int bh_sim_ipc_handles(bh_handle *h, void *out128);
int bh_sim_set_peers(bh_handle *h, int npeers, const void *handles);
int bh_sim_set_peer_ptrs(bh_handle *h, int npeers, void *const *acc, void *const *work);
/* the resident acc / work device buffers (for set_peer_ptrs) */
int bh_sim_result_ptrs(bh_handle *h, void **acc, void **work);
/* Copy a Morton-order range [begin, end) of a resident array to/from a caller
 * device buffer: BH_SIM_ACC (4 components per body, handle precision),
 * BH_SIM_POS (export only), BH_SIM_WORK (int32, this pass), BH_SIM_PREV_WORK
 * (export only: the previous pass's work of each sorted body -- the costzones
 * input, decomposition.py:35-57). */
enum { BH_SIM_ACC = 0, BH_SIM_WORK = 1, BH_SIM_PREV_WORK = 2, BH_SIM_POS = 3, BH_SIM_VEL = 4,
       BH_SIM_ID = 5, BH_SIM_KEYS = 6 };
int bh_sim_export(bh_handle *h, int what, int64_t begin, int64_t end, void *d_dst, void *stream);
int bh_sim_import(bh_handle *h, int what, int64_t begin, int64_t end, const void *d_src,
                  void *stream);

/* ---- distributed build: one rank of a key-range decomposition -----------
 * (decomposition.py:35-263 costzones/migration, hashed.py:539-824 branch nodes)
 *   local_maxabs -> allreduce max -> set_R          (simulation.py:201-208)
 *   sort (keys with R) -> migrate bodies by splitter keys -> load_state -> sort
 *   build_local: the rank's tree with global leaf depths (neighbour boundary
 *     keys), shared cells marked, walk records with every branch node present
 *   branch_export / walk_records: the payloads allgathered between ranks
 *   walk_records_f32: walk own targets over the assembled global walk tree. */
int bh_sim_local_maxabs(bh_handle *h, double *out, void *stream);
int bh_sim_set_R(bh_handle *h, double R, void *stream);
int bh_sim_sort(bh_handle *h, void *stream);
/* Morton keys of the resident bodies in their current order (no sort), with
 * the R set by bh_sim_set_R: the routing keys of the migration step
 * (morton.py:109-125 on the rank's bodies; decomposition.py:84-263). */
int bh_sim_keys(bh_handle *h, uint64_t *d_keys, void *stream);
int bh_sim_load_state(bh_handle *h, const void *d_pos, const void *d_vel, const void *d_acc,
                      const int32_t *d_work, int64_t n, void *stream);
int bh_sim_build_local(bh_handle *h, double theta, int leaf_size, int has_prev, uint64_t prev_key,
                       int has_next, uint64_t next_key, int64_t *nbranch, void *stream);
int bh_sim_branch_export(bh_handle *h, uint64_t *d_key, int32_t *d_level, int64_t *d_count,
                         double *d_mom10, int32_t *d_rec, int32_t *d_lo, void *stream);
int bh_sim_walk_records(bh_handle *h, void *d_out, int64_t *n_out, void *stream);
/* Locally essential trees: for every other rank q, the cells of
 * this rank's subtrees that a target inside q's bounding box could open under a
 * conservative box-MAC, plus the bucket bodies it could resolve (replaces the
 * reference's on-demand child fetches, hashed.py:831-911).  d_boxes:
 * [nrank][nbox][6] device doubles (min xyz, max xyz; empty boxes have min > max)
 * whose union covers each rank's bodies.  let: sizes per receiver (host arrays,
 * synchronises); let_pack: the receiver's records, bodies and branch map
 * ([nbranch][2] ints: first child in the LET | -1, first body | -1). */
/* The LET exchange overlapped with the walk.  Pass A walks the
 * local part of an assembled tree while the LETs are in flight: records whose
 * d.w carries bit 30 (remote branch nodes) are not opened; each warp appends
 * (target chunk, record, m0, m1) to d_defer (int4 x cap; *d_count = entries,
 * possibly > cap = overflow).  Pass B walks those entries over the completed
 * tree, d_fcnc[record] = (first child, nchild), adding into acc and work. */
int bh_walk_records_defer_f32(bh_handle *h, const void *d_records, int64_t nrec, const float *d_bodies4,
                              const float *d_targets4, int64_t nt, double eps, int leaf_size, float *d_acc4,
                              int32_t *d_work, int32_t *d_defer, uint32_t *d_count, int64_t cap, void *stream);
int bh_walk_records_resume_f32(bh_handle *h, const void *d_records, int64_t nrec, const float *d_bodies4,
                               const float *d_targets4, int64_t nt, double eps, int leaf_size, float *d_acc4,
                               int32_t *d_work, const int32_t *d_entries, int64_t n_entries,
                               const int32_t *d_fcnc, void *stream);
/* Bounding boxes of contiguous ranges of this rank's sorted bodies (the LET
 * target region): d_start[ngroup + 1] body offsets (device int64); d_out
 * [(1 + ngroup) * 6] device doubles: the union, then one box per range
 * (empty range: min = +inf, max = -inf); 1 <= ngroup <= 256.  fp32 handles,
 * after bh_sim_sort. */
int bh_sim_target_boxes(bh_handle *h, const int64_t *d_start, int ngroup, double *d_out, void *stream);
int bh_sim_let(bh_handle *h, const double *d_boxes, int nbox, int nrank, int self,
               int64_t *rec_counts, int64_t *body_counts, void *stream);
int bh_sim_let_pack(bh_handle *h, int q, void *d_rec_out, float *d_bodies_out, int32_t *d_bmap_out,
                    void *stream);
int bh_walk_records_f32(bh_handle *h, const void *d_records, int64_t nrec, const float *d_bodies4,
                        const float *d_targets4, int64_t nt, double eps, int leaf_size,
                        float *d_acc4, int32_t *d_work, void *stream);
int bh_stats_get(bh_handle *h, bh_stats *out, void *stream);

/* ---- distributed build, host side ------------------------------------------ */
/* hashed.py:719-786: the top of the global tree from every rank's branch nodes
 * (host memory).  rows: nrows int32 rows as decomposition._pack_branches packs
 * them (key, level, count, fp64 mass/com/quad, record index, first body, walk
 * record); n_own: this rank's bodies (the bucket-sized branch nodes' bodies
 * follow them).  Writes the breadth-first top region (16-int walk records) into
 * region[cap][16] with kind[e] (0 top cell, 1 bucket-sized top cell, 2 branch
 * node: the row's record, unpatched) and row_of[e]; bb[r] = row r's first body
 * in the [own | branch bodies] list (bucket-sized rows, else -1).  Returns the
 * number of region entries, or -1 if cap is too small. */
int64_t bh_top_tree(const int32_t *rows, int64_t nrows, int64_t n_own, int leaf, double R, double theta,
                    int32_t *region, int32_t *kind, int32_t *row_of, int64_t *bb, int64_t cap);

/* ---- instrumentation ----------------------------------------------------- */
/* Enable per-phase CUDA-event timing of bh_sim_* calls (adds event records). */
int bh_timing_enable(bh_handle *h, int on);
/* Zero the per-phase accumulators and the launch counter. */
int bh_timing_reset(bh_handle *h);
/* Synchronise and return accumulated milliseconds per phase (BH_NPHASES). */
int bh_timing_get(bh_handle *h, double *ms_out, int nphases);
/* FP32 FFMA throughput microbenchmark (the roofline denominator for the walk):
 * runs a dependent-chain-free FFMA loop on every SM, returns TFLOP/s. */
int bh_ffma_peak(bh_handle *h, double *tflops_out, void *stream);
/* Page-lock (pin) a caller's host array in place so that copies to and from it
 * run at full PCIe rate (the reference's numpy Bodies arrays, integrator.py:47-58
 * through TreeForces); bh_host_unregister undoes it.  Thin wrappers of
 * cudaHostRegister / cudaHostUnregister. */
int bh_host_register(void *p, int64_t bytes);
int bh_host_unregister(void *p);
/* The same loop in fp64 (DFMA): the roofline denominator of the fp64 walk. */
int bh_dfma_peak(bh_handle *h, double *tflops_out, void *stream);

#ifdef __cplusplus
}
#endif
#endif
