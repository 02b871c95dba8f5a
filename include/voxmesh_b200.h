/*
 * voxmesh_b200.h -- C ABI of the B200-native online mesh-generation hot path.
 *
 * The reference (`voxmesh`, pure Python) has no FFI: its boundary is the
 * Python API in /root/reference/pkg/src/voxmesh/.  Each entry point below
 * replaces one reference function (cited file:line); the Python package
 * paper_1803_03949_b200 binds them with ctypes and re-exposes the reference's
 * names.  Plain pointers and sizes only; no torch types.  All calls on one
 * engine must be serialised by the caller (reference Engine is single-caller,
 * engine.py:107-119).  Every call returns a vm_status; on failure
 * vm_last_error() holds a message (thread-local).
 *
 * Device memory layout, kernels and the roofline model: DESIGN.md.
 */
#ifndef VOXMESH_B200_H
#define VOXMESH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; mapped to the reference exceptions by the Python layer */
typedef enum {
  VM_OK = 0,
  VM_ERR_CAPACITY = 1,    /* CapacityError   (store.py:150-152, :304-306) */
  VM_ERR_CONSISTENCY = 2, /* ConsistencyError (store.py:166-170,183,234,422; mesher.py:201-203,270-275) */
  VM_ERR_VALUE = 3,       /* ValueError      (store.py:260; engine.py:48,52; mesher.py:559) */
  VM_ERR_CUDA = 4,        /* CUDA runtime failure (no device, launch error, OOM) */
  VM_ERR_INPUT = 5        /* malformed arguments (shape / null pointers) */
} vm_status;

/* vertex-sharing strategies (mesher.py:45) */
enum { VM_STRATEGY_SERIAL = 0, VM_STRATEGY_CLAIM = 1, VM_STRATEGY_PARTITION = 2 };

typedef struct vm_engine vm_engine;

/* SpatialStore(cube_size, table_size, max_vertices) -- store.py:254-268 */
typedef struct {
  double cube_size;          /* metres per cube (> 0) */
  int64_t table_size;        /* hash table size; CapacityError at 2*blocks >= table_size */
  int64_t max_vertices;      /* <= 0: unlimited (VertexPool.max_vertices, store.py:104) */
  int64_t initial_blocks;    /* capacity hints for the device arenas (0 = default); */
  int64_t initial_vertices;  /* the arenas grow geometrically when a frame needs more */
  int64_t initial_triangles;
  /* spatial partition across ranks; nranks <= 1: off.
   * Blocks belong to hashed tiles of tile_blocks^3 blocks; each rank owns its
   * tiles and also computes a 1-block margin around them, so every owned
   * result is exact with no halo exchange.  Counters cover owned blocks. */
  int32_t rank;
  int32_t nranks;
  int32_t tile_blocks;       /* power of two (default 8) */
  int32_t halo_exchange;     /* 0: margin blocks integrated by this rank from the broadcast
                              * depth; 1: owned blocks only, margin blocks received from their
                              * owners before meshing (vm_partition_frame_begin / _finish) */
} vm_store_config;

/* Intrinsics (fusion.py:20-33) */
typedef struct {
  double fx, fy, cx, cy;
  int32_t width, height;
} vm_intrinsics;

/* Pose: sensor-to-world rigid transform, rotation row-major (fusion.py:36-56) */
typedef struct {
  double rotation[9];
  double translation[3];
} vm_pose;

/* resolved RunConfig fields used per frame (engine.py:27-53) */
typedef struct {
  double trunc;
  double max_range;
  double epsilon;
  int64_t weight_cap;
  int32_t refine;        /* RefineParams.enabled (refine.py:55-60) */
  int32_t frustum_only;  /* engine.py:135-138 */
  int32_t strategy;      /* VM_STRATEGY_* */
  int32_t block_gc_age;  /* > 0: opt-in block GC -- every block_gc_age frames, evict the blocks
                          * not collected for block_gc_age frames that hold no vertex and no
                          * observed sample (all weights 0); the mesh is unchanged, only
                          * blocks_active drops.  0 = off (the reference never frees a block,
                          * store.py:14) */
} vm_frame_config;

/* StatsRow non-timing columns (engine.py:71-86) + per-frame unit counts used
 * by the roofline model. */
typedef struct {
  int64_t frame;
  int64_t blocks_active;
  int64_t vertices_live;
  int64_t triangles_live;
  int64_t vertices_allocated_total;
  int64_t vertices_recycled_total;
  int64_t irregular_cube_count;
  /* per-frame unit counts */
  int64_t valid_pixels;
  int64_t nsteps;
  int64_t collected_blocks;
  int64_t new_blocks;
  int64_t scope_blocks;
  int64_t halo_blocks;
  int64_t active_cubes;
  int64_t edge_placements;
  int64_t new_vertices;
  int64_t changed_cubes;
  int64_t triangles_freed;
  int64_t triangles_allocated;
  int64_t vertices_freed;
  int64_t normals_computed;
  int64_t fallback_normals;
  int64_t refined_cubes;
  int64_t resumes;        /* arena growths that required a resume this frame */
  int64_t kernel_launches;/* kernels this library launched for the frame */
  int64_t blocks_evicted; /* block GC: blocks evicted so far (0 with block GC off) */
  int64_t overlapped;     /* 1: this frame's k_collect ran under the previous frame's k_gc_normals
                             (frame overlap, pipelined submission back to back) */
  double device_ms;       /* device time of the frame (CUDA events) */
  double fusion_ms;       /* collect + integrate (engine.py:127-132 split) */
  double meshing_ms;      /* scope .. normals (engine.py:134-144 split) */
} vm_stats;

/* Export the state of this engine's blocks (owned_only: the blocks this rank
 * owns) as dense arrays; pass coords == NULL to query *n_out first.  Arrays:
 * coords i32[n,3], tsdf f64[n,512], weight i32[n,512], type_prev/type_curr
 * u8[n,512], slot birth i32[n,1536], slot coordinate f64[n,1536], slot
 * normal f64[n,1536,3]. */
int vm_export_blocks(vm_engine *e, int32_t owned_only, int64_t *n_out, int32_t *coords, double *tsdf,
                     int32_t *weight, uint8_t *type_prev, uint8_t *type_curr, int32_t *birth,
                     double *param, double *normal);
/* Import block states exported by vm_export_blocks (allocating the blocks);
 * used to merge the ranks of a partitioned reconstruction for compaction. */
int vm_import_blocks(vm_engine *e, int64_t n, const int32_t *coords, const double *tsdf,
                     const int32_t *weight, const uint8_t *type_prev, const uint8_t *type_curr,
                     const int32_t *birth, const double *param, const double *normal);

/* AuditReport (engine.py:89-101) */
typedef struct {
  int64_t vertices_live;
  int64_t triangles_live;
  int64_t refcount_mismatches;
  int64_t duplicate_handles;
  int64_t zero_ref_live;
  int64_t conservation_ok;
} vm_audit_report;

/* pool/arena counters (store.py:113-115,185-187,204-206) */
typedef struct {
  int64_t block_count;
  int64_t block_allocations;
  int64_t vertex_count;          /* arena high-water (VertexPool.count) */
  int64_t vertex_free;           /* len(VertexPool.free) */
  int64_t vertex_recycled_total;
  int64_t vertex_allocation_events;
  int64_t triangle_count;
  int64_t triangle_free;
  int64_t triangle_recycled_total;
  int64_t irregular_cube_count;  /* incrementally maintained */
  int64_t block_capacity;        /* current device arena capacities */
  int64_t vertex_capacity;
  int64_t triangle_capacity;
  int64_t vertex_records;        /* device vertex records in use (slots ever occupied) */
  int64_t store_bytes;           /* HBM held by the stored blocks + their vertex records */
  int64_t device_bytes;          /* HBM allocated by the engine (capacities, tables, lists) */
} vm_counter_set;

/* ---- lifecycle ------------------------------------------------------- */
const char *vm_last_error(void);
const char *vm_version(void);
/* SpatialStore.__init__ (store.py:254-268) */
int vm_create(const vm_store_config *cfg, vm_engine **out);
int vm_destroy(vm_engine *e);
/* Run on a caller-owned cudaStream_t (NULL = the engine's own stream). */
int vm_set_stream(vm_engine *e, void *cuda_stream);
/* The cudaStream_t the engine's kernels run on (device inputs produced on
 * another stream must be ordered before it: the binding records an event on
 * the producer stream and makes this one wait, engine.py). */
int vm_get_stream(vm_engine *e, void **cuda_stream);
/* Order the engine's stream after the work queued so far on `producer` (a
 * cudaStream_t that wrote a device input): nothing is queued when that work
 * has already completed (so a frame can still overlap the previous one),
 * else the engine's stream waits on an event recorded there. */
int vm_order_after(vm_engine *e, void *producer);
/* Record CUDA events between the frame's kernels (per-phase device times). */
int vm_set_profiling(vm_engine *e, int on);
/* Per-kernel device times (ms) of the last frame: depth_stats, collect,
 * fuse_blocks, retype_place, gc_normals (n <= 5). Requires vm_set_profiling(e, 1). */
int vm_phase_times(vm_engine *e, double *ms, int n);
/* Diagnostics: per-CTA phase timestamps (%globaltimer, ns) of the frame
 * kernels into a caller-owned DEVICE buffer of u64[4 * 2048 * 32] (layout in
 * csrc/vm_device.cuh, kTraceCtas); NULL switches tracing off. */
int vm_set_trace(vm_engine *e, void *device_buffer);
/* Guarantee arena capacity (blocks/vertices/triangles) without growth later. */
int vm_reserve(vm_engine *e, int64_t blocks, int64_t vertices, int64_t triangles);

/* ---- the hot path ---------------------------------------------------- */
/* Engine.fuse_frame (engine.py:123-165): collect -> integrate -> scope ->
 * [frustum] -> halo -> extract (retype/refine, place, triangulate, GC,
 * normals).  depth: (h, w) f64 metres, 0 = invalid, row-major; host pointer
 * (copied to the device) or device pointer when depth_on_device != 0.
 * Synchronous: returns when the frame is complete and stats are filled. */
int vm_fuse_frame(vm_engine *e, const double *depth, int32_t h, int32_t w,
                  int32_t depth_on_device, const vm_intrinsics *intr, const vm_pose *pose,
                  const vm_frame_config *cfg, int64_t frame_index, vm_stats *out);
/* Split form of vm_fuse_frame for device timing: enqueue all frame work on the
 * stream (no host sync), then finish (sync, resume after arena growth if a
 * guard tripped, fill stats). */
int vm_fuse_frame_enqueue(vm_engine *e, const double *depth, int32_t h, int32_t w,
                          int32_t depth_on_device, const vm_intrinsics *intr,
                          const vm_pose *pose, const vm_frame_config *cfg,
                          int64_t frame_index);
int vm_fuse_frame_finish(vm_engine *e, vm_stats *out);
/* Pipelined form of vm_fuse_frame (same results, frame for frame): submit
 * starts this frame's host->device depth copy on a second stream, completes
 * the previously submitted frame (host wait, arena resume), orders this
 * frame's kernels after its copy and returns once the copy is done (the host
 * buffer may be reused) while the kernels run.  The copy of frame t+1
 * therefore overlaps the kernels of frame t.  vm_fuse_frame_result delivers
 * the stats of the oldest submitted frame not yet delivered (completing it if
 * needed); it must be called once per submitted frame, before the next
 * submit.  An error of frame t is returned by the call that completes it.
 * Every other entry point completes a pending submitted frame first. */
int vm_fuse_frame_submit(vm_engine *e, const double *depth, int32_t h, int32_t w,
                         int32_t depth_on_device, const vm_intrinsics *intr,
                         const vm_pose *pose, const vm_frame_config *cfg, int64_t frame_index);
int vm_fuse_frame_result(vm_engine *e, vm_stats *out);
/* Deferred input wait (on != 0): vm_fuse_frame_submit[_raw] returns once the
 * host->device copy of the host buffer is queued, not done; the caller calls
 * vm_input_wait before it reuses the buffer.  The Python binding delivers the
 * previous frame's row in between, so that work overlaps the copy. */
int vm_set_deferred_input_wait(vm_engine *e, int on);
/* Block until the last submitted frame's host buffer has been read. */
int vm_input_wait(vm_engine *e);
/* vm_fuse_frame_submit for a raw 16-bit depth image (native byte order, as
 * decoded from the reference's PGM files): the device converts each pixel
 * exactly as io_formats.read_depth (io_formats.py:84: raw / depth_scale in
 * f64, 0 = invalid) inside the frame's first pixel kernel, so a quarter of the
 * f64 frame's bytes cross PCIe.  Results equal vm_fuse_frame on the converted
 * frame bit for bit.  raw_on_device != 0: `raw` is a device pointer. */
int vm_fuse_frame_submit_raw(vm_engine *e, const uint16_t *raw, int32_t h, int32_t w,
                             int32_t raw_on_device, double depth_scale, const vm_intrinsics *intr,
                             const vm_pose *pose, const vm_frame_config *cfg, int64_t frame_index);

/* ---- phase-level API (tests / reference function mirrors) ------------ */
/* fusion.collect_blocks (fusion.py:70-107): allocates the touched blocks and
 * keeps them as the engine's collected list; *n_out = count. */
int vm_collect(vm_engine *e, const double *depth, int32_t h, int32_t w, int32_t depth_on_device,
               const vm_intrinsics *intr, const vm_pose *pose, double trunc, double max_range,
               int64_t *n_out);
/* copy the collected list (block coords, unordered) */
int vm_get_collected(vm_engine *e, int32_t *coords_out, int64_t n);
/* fusion.integrate_frame (fusion.py:122-168) over explicit block coords
 * (coords == NULL: the last collected list).  Absent blocks are skipped. */
int vm_integrate(vm_engine *e, const int32_t *coords, int64_t n, const double *depth, int32_t h,
                 int32_t w, int32_t depth_on_device, const vm_intrinsics *intr,
                 const vm_pose *pose, double trunc, double max_range, int64_t weight_cap);
/* mesher.meshing_scope + fused_halo (mesher.py:499-543) of the last collected
 * list, computed on the device.  Outputs are unordered; masks are 64-byte cube
 * bitmaps (bit ci = x*64+y*8+z).  Pass NULL buffers to query counts only. */
int vm_scope_halo(vm_engine *e, int64_t *n_scope, int32_t *scope_coords, uint8_t *scope_masks,
                  int64_t *n_halo, int32_t *halo_coords);
/* mesher.extract_frame (mesher.py:546-636) over an explicit scope: coords
 * (n_scope x 3) with optional 64-byte cube bitmaps (NULL = full blocks), and
 * a halo (n_halo x 3; n_halo < 0 = derive from the scope like extract_frame's
 * default).  out2 = {refined, freed}. */
int vm_extract(vm_engine *e, const int32_t *scope_coords, const uint8_t *scope_masks,
               int64_t n_scope, const int32_t *halo_coords, int64_t n_halo,
               int64_t frame_index, int32_t strategy, int32_t refine, double epsilon,
               int64_t *out2);
/* mesher.garbage_collect (mesher.py:333-356) */
int vm_garbage_collect(vm_engine *e, const int32_t *coords, int64_t n, int64_t *freed);
/* mesher.compute_normals (mesher.py:442-486) */
int vm_compute_normals(vm_engine *e, const int32_t *coords, int64_t n);
/* refine.refine_block_types / detect_disturbance evaluated by the device
 * kernel for n independent cubes: t_curr, t_prev (u8), corner tsdf (n x 8),
 * -> out (int32, -1 = None).  Used for the exhaustive Eq. 3-5 check. */
int vm_refine_eval(vm_engine *e, const uint8_t *t_curr, const uint8_t *t_prev,
                   const double *corners, int64_t n, double epsilon, int32_t *out);
/* fusion.block_in_frustum (fusion.py:171-190) evaluated on the device */
int vm_block_in_frustum(vm_engine *e, const int32_t *coords, int64_t n, const vm_pose *pose,
                        const vm_intrinsics *intr, uint8_t *out);

/* ---- store access ---------------------------------------------------- */
/* SpatialStore.get_or_allocate_block (store.py:296-320) + write the corner
 * samples (tests build fields this way); tsdf/weight (n x 512) may be NULL. */
int vm_set_blocks(vm_engine *e, const int32_t *coords, int64_t n, const double *tsdf,
                  const int32_t *weight);
/* SpatialStore.get_block existence (store.py:280-294): out[i] = 1/0 */
int vm_lookup(vm_engine *e, const int32_t *coords, int64_t n, uint8_t *out);
int vm_counters(vm_engine *e, vm_counter_set *out);
/* Snapshot of all blocks in heap order (n = block_count); any pointer may be NULL.
 * tsdf f64[n,512], weight i32[n,512], type_prev/type_curr u8[n,512],
 * edge_vertex i32[n,512,3], triangles i32[n,512,5]. */
int vm_snapshot_blocks(vm_engine *e, int64_t n, int32_t *coords, double *tsdf, int32_t *weight,
                       uint8_t *type_prev, uint8_t *type_curr, int32_t *edge_vertex,
                       int32_t *triangles);
/* vertex arena [0, vertex_count): position/normal f64[n,3], refcount, birth
 * i32[n], alive u8[n]; free stack i32[vertex_free] */
int vm_snapshot_vertices(vm_engine *e, int64_t n, double *position, double *normal,
                         int32_t *refcount, int32_t *birth, uint8_t *alive, int32_t *free_stack);
/* triangle arena [0, triangle_count): vertices i32[n,3], alive u8[n] */
int vm_snapshot_triangles(vm_engine *e, int64_t n, int32_t *vertices, uint8_t *alive,
                          int32_t *free_stack);

/* ---- outputs --------------------------------------------------------- */
/* Engine.irregular_cube_count (engine.py:169-176), full device scan */
int vm_irregular_count(vm_engine *e, int64_t *out);
/* SpatialStore.compact_mesh (store.py:388-425): two-phase; vm_compact runs the
 * device compaction and returns sizes, vm_compact_fetch copies to host. */
int vm_compact(vm_engine *e, int64_t current_frame, int64_t *n_vertices, int64_t *n_triangles);
int vm_compact_fetch(vm_engine *e, double *positions, double *normals, int64_t *ages,
                     int32_t *indices);
/* Engine.audit (engine.py:187-230) as device reductions */
int vm_audit(vm_engine *e, vm_audit_report *out);

/* ---- spatial partition across ranks ----
 * The reference is single-process; these entry points are what a rank of the
 * partitioned reconstruction calls around its collectives (the Python layer,
 * partition.py, runs them over torch.distributed: NCCL on the GPU box).
 *
 * Halo-exchange frame = begin (collect + integrate the owned blocks, pack the
 * collected boundary blocks into `send`: kVM_GHOST_RECORD bytes each), an
 * all-gather of every rank's records (max_count per rank, padded), finish
 * (adopt the records in this rank's margin, then meshing).  Engine.fuse_frame
 * (engine.py:123-165) split around the exchange.  `send` / `recv` are device
 * pointers.  If *n_send > send_cap, grow the buffer and call
 * vm_partition_repack.  *n_owned_collected: owned blocks collected. */
#define VM_GHOST_RECORD 6160
int vm_partition_frame_begin(vm_engine *e, const double *depth, int32_t h, int32_t w, int32_t depth_on_device,
                             const vm_intrinsics *intr, const vm_pose *pose, const vm_frame_config *cfg,
                             int64_t frame_index, uint8_t *send, int64_t send_cap, int64_t *n_send,
                             int64_t *n_owned_collected);
/* Sharded band walk (spatial partition): walk only pixel rows [row0, row1)
 * (row0 a multiple of 8) of the broadcast frame and list, into the device
 * buffer keys_dev (capacity cap), the packed keys of every block the band
 * samples there meet -- owned or not.  The ranks all-gather their lists;
 * vm_partition_frame_begin_keys then collects each rank's relevant blocks
 * from the union (in place of walking every pixel) and continues as
 * vm_partition_frame_begin.  The collected set equals the unsharded one. */
int vm_partition_collect_keys(vm_engine *e, const double *depth, int32_t h, int32_t w, int32_t depth_on_device,
                              const vm_intrinsics *intr, const vm_pose *pose, const vm_frame_config *cfg,
                              int64_t frame_index, int32_t row0, int32_t row1, uint64_t *keys_dev, int64_t cap,
                              int64_t *n_keys);
int vm_partition_frame_begin_keys(vm_engine *e, const uint64_t *keys_dev, int64_t n_keys, uint8_t *send,
                                  int64_t send_cap, int64_t *n_send, int64_t *n_owned_collected);
int vm_partition_repack(vm_engine *e, uint8_t *send, int64_t send_cap, int64_t *n_send);
int vm_partition_frame_finish(vm_engine *e, const uint8_t *recv, const int32_t *counts, int32_t nranks,
                              int64_t max_count, vm_stats *out);
/* Distributed compaction (store.py:388-425 over the union of the ranks'
 * owned blocks).  begin: sort this rank's owned blocks; meta: their packed
 * keys (sorted), vertex / triangle counts and 48-word slot occupancy (host
 * arrays of *n_owned entries); fill: given the merged (k-way, by key) global
 * block list -- keys, exclusive vertex / triangle bases, occupancy and its
 * per-word exclusive popcount prefix (host arrays of n_global entries) and
 * this rank's blocks' global positions -- write this rank's vertices and
 * triangles at their global positions into zero-initialised DEVICE arrays of
 * the global mesh (the ranks' arrays are then summed: disjoint ranges). */
int vm_partition_compact_begin(vm_engine *e, int64_t *n_owned);
int vm_partition_compact_meta(vm_engine *e, uint64_t *keys, int32_t *vcnt, int32_t *tcnt, uint32_t *occ);
int vm_partition_compact_fill(vm_engine *e, const uint64_t *gkeys, const int64_t *vbase, const int64_t *tbase,
                              const uint32_t *gocc, const int32_t *gocc_pre, int64_t n_global,
                              const int32_t *my_global, int64_t current_frame, double *pos, double *nrm,
                              int64_t *ages, int32_t *idx);

#ifdef __cplusplus
}
#endif
#endif /* VOXMESH_B200_H */
