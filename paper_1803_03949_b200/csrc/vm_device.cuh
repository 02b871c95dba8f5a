// vm_device.cuh -- device-side data structures and helpers for the B200
// online mesh-generation path (DESIGN.md sections 2-3).
//
// Layout ("slot-resident cube field"):
//   * block table: bucketed hash (8 CAS slots per bucket + locked overflow
//     chains) mapping packed block coordinates to a dense block index;
//   * per block (SoA, 8x8x8 cubes, C order x,y,z): tsdf f64, weight i32,
//     type_prev/type_curr u8, and per owned edge slot (3 per cube): an
//     occupancy bit, the position along the edge axis f64 and the slot's
//     vertex-record handle i32.  A vertex lives IN its edge slot (the paper's
//     "cube owns its 3 edges"): allocation = setting the occupancy bit,
//     recycling = clearing it.  Birth frame and normal live in a compact
//     vertex-record arena: a slot gets a record the first time it is occupied
//     and keeps it (re-occupation reuses it), so the arena holds the slots
//     ever used, not 1536 per block.
//   * triangles are not stored: a cube's live triangles are always
//     TRI_TABLE[type_curr] (the reference retriangulates exactly when the type
//     changes, mesher.py:283-320), so triangle lists and vertex reference
//     counts are derived from the types; counters reproduce the reference's
//     pool statistics (store.py:95-241).
//
// Numeric contract: compiled with --fmad=false; the only FMAs are explicit
// __fma_rn chains restating numpy/OpenBLAS 3x3 products (SURVEY.md appx A).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "mc_tables.inc"

namespace vm {

constexpr int kB = 8;          // cubes per block edge (store.py:26)
constexpr int kNC = 512;       // cubes per block
constexpr int kSlotsPerBucket = 8;
constexpr int kEV = kNC * 3;   // edge-vertex slots per block
constexpr long long kEmptyKey = -1LL;
constexpr int kEvicted = -3;   // hash value of a key whose block the block GC evicted (key kept)

enum { ERR_NONE = 0, ERR_CAPACITY = 1, ERR_CONSISTENCY = 2 };

// Device counters.  Persistent fields first; everything from `nvalid` on is
// reset at the start of every call (one memset).
// The frame's halo list is appended by every retype CTA at once: one counter
// would serialise ~2.5k returning atomics (~6 us at the end of the kernel), so
// appends go to kHaloShards sub-lists (shard = CTA index mod kHaloShards) of
// halo_sh_cap entries each, a full shard spilling into the general list (halo,
// nhalo), which the phase API also uses.  k_gc_normals (G_SHARDED) walks the
// shards' prefix then the general list.
constexpr int kHaloShards = 32;

struct alignas(16) Counters {
  int32_t nblocks;       // SpatialStore.block_count
  int32_t ovf_count;
  int32_t error;
  int32_t need;          // heap exhausted: the epoch of the call whose allocation ran past block_cap (0 = no)
  int64_t v_live;        // VertexPool.live_count
  int64_t v_count;       // VertexPool.count (arena high-water)
  int64_t v_recycled;
  int64_t v_events;      // VertexPool.allocation_events
  int64_t t_live;        // TrianglePool.live_count
  int64_t t_count;
  int64_t t_recycled;
  int64_t irregular;     // Engine.irregular_cube_count, maintained incrementally
  int64_t nblocks_owned; // blocks this rank owns (== nblocks unless partitioned)
  int64_t err_info[4];
  int32_t fb_pending;    // face-normal fallback records of the last frame not yet applied
  int32_t nfree;         // block GC: evicted block indices on the free list
  int64_t evicted_total; // block GC: blocks evicted so far
  int64_t a_hw;          // vertex records assigned: handles [0, a_hw) (slots keep theirs)
  int32_t need_stage;    // where a halted frame resumes: 0 k_fuse_blocks (block heap), 1 k_retype_place (records)
  int32_t pad0[3];
  // ---- per call ----------------------------------------------------------
  // The collect counters (written by k_collect / k_depth_stats and the block
  // allocations).  The next frame's k_collect may run under this frame's
  // k_gc_normals (frame overlap): so k_gc_normals saves
  // them (sv_*) and clears them at its START, before it lets the next frame
  // launch, and its commit snapshots the saved values and clears only the
  // fields from `nslab` on.
  int32_t nvalid;
  int32_t nsteps;
  int32_t ncollected;
  int32_t nnew;
  unsigned long long maxnorm_bits;
  unsigned long long t_start_ns;   // %globaltimer: k_collect (or k_depth_stats) start
  int32_t fb_next;                 // k_collect: the previous frame's fallback records handed out so far
  int32_t ds_done;                 // k_depth_stats CTAs done (an overlapped k_collect waits for all)
  int32_t pad3[2];
  // ---- per call, cleared by k_gc_normals' commit ----------------------------
  // (one 16-byte word: the meshing kernels' prologues read it with one load)
  int32_t nslab;
  int32_t nexplicit;
  int32_t nitems_live;
  int32_t nhalo;
  int32_t done_gc;
  int32_t nsend;                   // halo exchange: boundary blocks packed for the other ranks
  int64_t v_allocs;
  int64_t v_frees;
  int64_t placements;
  int64_t active;
  int64_t changed;
  int64_t t_released;
  int64_t t_allocated;
  int64_t irr_delta;
  int64_t normals;
  int64_t fallbacks;
  int64_t refined;
  int32_t nhalo_sh[kHaloShards];   // halo shard fill counts (may exceed halo_sh_cap: clamp)
  unsigned long long t_end_ns;     // k_gc_normals commit
  unsigned long long t_mesh_ns;    // k_retype_place start (after integration): fusion | meshing split
  // the frame's collect counters and block counts, saved by k_gc_normals at its start
  int32_t sv_nvalid, sv_nsteps, sv_ncollected, sv_nnew;
  unsigned long long sv_maxnorm_bits, sv_t_start_ns;
  int32_t sv_nblocks, sv_nfree;
  int64_t sv_nblocks_owned;
};
static_assert(sizeof(Counters) % 16 == 0, "snapshots are copied in 16-byte words");
static_assert(offsetof(Counters, nvalid) % 16 == 0 && offsetof(Counters, ncollected) == offsetof(Counters, nvalid) + 8 &&
              offsetof(Counters, t_start_ns) == offsetof(Counters, nvalid) + 24 &&
              offsetof(Counters, fb_next) == offsetof(Counters, nvalid) + 32, "collect region: 3 words");
static_assert(offsetof(Counters, nslab) % 16 == 0 && offsetof(Counters, nitems_live) == offsetof(Counters, nslab) + 8,
              "prologue word: nslab, nexplicit, nitems_live, nhalo");
static_assert(offsetof(Counters, sv_nvalid) % 16 == 0, "saved collect region: 16-byte words");
static_assert(offsetof(Counters, error) == 8 && offsetof(Counters, need) == 12, "head word: nblocks, ovf, error, need");

// Per-call parameters in device memory (a captured frame graph replays with
// new poses / depth pointers).
struct FrameDev {
  const double *depth;
  const uint16_t *raw;  // non-null: the frame arrived as raw u16 (read_depth): the first pixel
  double *depth_out;    //   pass fills depth_out[p] = raw[p] / depth_scale (io_formats.py:84)
  double depth_scale;
  int32_t h, w;
  double fx, fy, cx, cy;
  int32_t width, height;
  double R[9];
  double t[3];
  double trunc, max_range, epsilon;
  int64_t weight_cap;
  int32_t refine, frustum_only;
  int32_t epoch;        // monotone stamp for per-call membership sets
  int32_t frame;        // frame index (vertex birth)
  int32_t scope_mode;   // 0: collected + slabs (device scope); 1: explicit items
  int32_t nsteps_fixed; // > 0: band step count fixed by the intrinsics (k_depth_stats skipped)
  double band_step;     // 2 / (nsteps_fixed - 1) (fusion.py:96, np.linspace's step), when fixed
  int32_t block_gc_age; // > 0: opt-in block GC (k_block_gc before this frame when frame % age == 0)
  int32_t consume_fb;   // fuse_frame: k_collect applies the previous frame's fallback records
  int32_t reset_after;  // k_gc_normals' commit clears the per-call counters after its snapshot
  int32_t strategy;     // VM_STRATEGY_*: 2 = partition (8 parity passes of plain stores, k_place_parity)
  // Frame overlap: overlap != 0 -- this k_collect was
  // launched right behind the previous frame's k_gc_normals, which lets it
  // start once every gc CTA is running: it skips cudaGridDependencySynchronize
  // (it touches nothing the gc reads or writes) and runs the work that does
  // depend on the previous frame (fallback records, record ranges, the
  // snapshot publish) only after *S.gc_done reaches wait_epoch.
  int32_t overlap;
  int32_t wait_epoch;
  // host-copied input (pipelined submission): the copy stream writes in_id to
  // *in_flag after the depth; k_collect waits for it before reading the depth
  // (no event wait on the engine's stream, which would keep the frames apart)
  const unsigned long long *in_flag;
  unsigned long long in_id;
  int32_t ds_wait;      // > 0: k_collect waits until that many k_depth_stats CTAs are done (overlap)
  int32_t pad_ds;
  // spatial partition, sharded band walk: k_collect walks pixel rows
  // [row0, row1) only (row1 <= 0: all) and, with key_out set, lists the
  // distinct block keys it meets there (every block, owned or not) instead of
  // collecting them; the ranks all-gather the lists and each collects its
  // relevant blocks from the union (k_collect_keys_apply)
  int32_t row0, row1;
  unsigned long long *key_out;
  int32_t *key_count;
  int32_t key_cap;
  Counters *snap;       // non-null: k_gc_normals' commit copies the counter block here (device)
  // non-null: k_collect copies the previous frame's snapshot (pub_src) to the
  // host's mapped buffer (pub_dst) and then writes pub_id to *pub_seq, the
  // word the host waits on -- off the frame's critical path
  const Counters *pub_src;
  Counters *pub_dst;
  unsigned long long *pub_seq;
  unsigned long long pub_id;
  // non-null: k_gc_normals' commit publishes this frame's own snapshot to the
  // host (used when the next frame's input arrives by a host copy, so its
  // k_collect would publish late)
  Counters *self_dst;
  unsigned long long *self_seq;
  unsigned long long self_id;
  // halo exchange: the ranks' packed boundary blocks,
  // rank q's k-th record at ghost_recv + (q * ghost_max + k) * kGhostRec
  const uint8_t *ghost_recv;
  int32_t ghost_max, ghost_nranks;
};

// one hash slot: packed coordinate (-1 empty) and block index (-1 while the
// inserting thread has not published it yet)
// per-vertex record (the slot's handle indexes it): normal, birth frame
struct alignas(32) VertexRec {
  double nrm[3];
  int32_t birth;
  int32_t pad;
};
// vertex records one scope item can assign in a frame: its cubes own the
// edges of the 9^3 points of its tile, 3 per point
constexpr long long kRecsPerItem = 729 * 3;
constexpr long long kRecChunk = 64;

struct alignas(16) HashSlot {
  long long key;
  int32_t val;
  int32_t pad;    // epoch in which the block was last collected
};

struct DevState {
  double cube_size, extent;
  double inv_extent;    // RN(1 / extent): division-free floor with an exact fallback
  const double *rays;   // (u - cx) / fx for u < w, then (v - cy) / fy for v < h (fusion.py:29-33)
  long long table_size;
  unsigned bmask;       // nbuckets-1 if a power of two, else 0
  int32_t nbuckets;
  int32_t max_blocks;   // reference load-factor limit: 2*n < table_size
  HashSlot *slots;      // [nbuckets*8] (packed coord, block index); a bucket = one 128-B line
  int32_t *ovf_head;
  int32_t *ovf_lock;
  long long *ovf_key;
  int32_t *ovf_val;
  int32_t *ovf_next;
  int32_t *ovf_stamp;   // "collected" epoch of chain entries
  int32_t ovf_cap;
  // per-block metadata, sized max_blocks
  int4 *bcoord;
  int32_t *nbr;         // [max_blocks*27] neighbour block index (-1 absent); 13 = self
  int32_t *stamp_collect;
  int32_t *stamp_halo;
  int32_t *stamp_new;   // epoch in which the block was allocated
  uint8_t *slab_bits;
  int32_t *scope;       // scope items: collected first, then minus slabs
  int32_t *halo;
  int32_t *halo_sh;     // kHaloShards x halo_sh_cap
  int32_t halo_sh_cap;
  // heavy block storage, sized block_cap (grows)
  int32_t block_cap;
  double *tsdf;         // [cap*512]
  int32_t *weight;      // [cap*512]
  uint32_t *vmask;      // [cap*16] weight > 0, one bit per cube corner sample (C order)
  uint8_t *tp, *tc;     // [cap*512]
  int32_t *vh;          // [cap*1536] the slot's vertex record (-1: never occupied); kept when the slot empties
  uint32_t *vrb;        // [cap*48] the slot has a record (vh >= 0), as bits (staged by k_gc_normals)
  uint32_t *vocc;       // [cap*48] slot occupancy bits (read and written by k_gc_normals)
  uint32_t *vclaim;     // [cap*48] slots requested this frame (k_retype_place ORs, k_gc_normals applies + clears)
  double *vparam;       // [cap*1536] vertex coordinate along the edge axis
  VertexRec *vrec;      // [vrec_cap] vertex records (normal, birth)
  long long vrec_cap;
  // k_gc_normals hands out records from per-CTA ranges, topped up 2 kRecChunk
  // at a time (one atomic on a_hw every few frames per CTA, issued in its
  // prologue): CTA c's two free ranges [rec_chunk[4 c], rec_chunk[4 c + 1]),
  // [rec_chunk[4 c + 2], rec_chunk[4 c + 3])
  long long *rec_chunk;
  int32_t rec_chunk_ctas;
  uint32_t *item_mask;  // [cap*16] explicit scope cube masks
  // strategy "partition" only (allocated on first use): per-slot request bytes
  // written by the parity passes with plain stores, and the retype's selection
  // (one byte per tile column, bit z) of each scope item
  uint8_t *vreq;        // [cap*1536]
  uint8_t *psel;        // [cap*64]
  int4 *fallback;       // [fb_cap] fallback records of the last frame: block, slot, 4 cube types, candidate mask
  int32_t fb_cap;       //   (a bounded ring: records past it are applied inline by k_gc_normals)
  long long max_vertices;
  // spatial partition: blocks are owned by hashed tiles
  // of 2^tile_shift blocks per axis; a rank also computes a 1-block margin
  int32_t rank, nranks, tile_shift;
  // 0: margin mode -- the rank integrates its margin blocks itself from the
  //    broadcast depth; 1: halo exchange -- it integrates owned blocks only and
  //    receives the margin blocks' samples from their owners before meshing
  int32_t halo_exchange;
  uint8_t *bowned;      // [max_blocks] block owned by this rank
  int32_t *ghost_src;   // [max_blocks] scope position -> received record (halo exchange)
  int32_t *last_frame;  // [max_blocks] frame in which the block was last collected (block GC)
  int32_t *free_list;   // [max_blocks] evicted block indices (block GC)
  int32_t free_list_on; // block GC has run: allocations check the free list first
  const int32_t *ghost_counts;   // [nranks] records per rank of the current exchange
  Counters *ctr;
  int32_t *gc_done;     // epoch of the last k_gc_normals commit (outside Counters: host restores leave it)
  unsigned long long *trace;   // per-CTA phase timestamps (vm_set_trace), null = off
};

// ---------------------------------------------------------------- tracing
// Diagnostics only: with a trace buffer set, thread 0 of CTA c < kTraceCtas of
// kernel k stores %globaltimer at phase p to trace[(k * kTraceCtas + c) * kTraceSlots + p].
// Slots: 0 start, 1 prologue done, 2 + 4 * item + {0 item start, 1 resolved,
// 2 staged, 3 computed} for the first 5 items, 22..26 sub-phases of the first
// item, 27 items processed (a count), 28 item loop done, 29 / 30
// kernel-specific, 31 end.
constexpr int kTraceCtas = 2048, kTraceSlots = 32;
enum { TK_COLLECT = 0, TK_FUSE = 1, TK_RETYPE = 2, TK_GC = 3, TK_COUNT = 4 };
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#ifdef VM_TRACE   // diagnostics build only (build(trace=True)); the product build has no trace code
__device__ __forceinline__ void trace_at(const DevState &S, int k, int slot) {
  if (S.trace && threadIdx.x == 0 && blockIdx.x < kTraceCtas)
    S.trace[((size_t)k * kTraceCtas + blockIdx.x) * kTraceSlots + slot] = gtimer();
}
__device__ __forceinline__ void trace_count(const DevState &S, int k, int n) {
  if (S.trace && threadIdx.x == 0 && blockIdx.x < kTraceCtas)
    S.trace[((size_t)k * kTraceCtas + blockIdx.x) * kTraceSlots + 27] = (unsigned long long)n;
}
// per-frame kernel spans (a ring of 256 frames after the per-CTA area): entry
// [frame][2k] = kernel k's block-0 start, [2k+1] = the latest CTA end
constexpr size_t kTraceRing = (size_t)TK_COUNT * kTraceCtas * kTraceSlots;
__device__ __forceinline__ void trace_span(const DevState &S, int k, int frame, bool end) {
  if (!S.trace || threadIdx.x != 0) return;
  unsigned long long *r = S.trace + kTraceRing + (size_t)(frame & 255) * 8 + 2 * k;
  if (end) atomicMax(r + 1, gtimer());
  else if (blockIdx.x == 0) *r = gtimer();
}
// (any thread: per-warp marks)
__device__ __forceinline__ void trace_at_any(const DevState &S, int k, int slot) {
  if (S.trace && blockIdx.x < kTraceCtas) S.trace[((size_t)k * kTraceCtas + blockIdx.x) * kTraceSlots + slot] = gtimer();
}
#else
__device__ __forceinline__ void trace_span(const DevState &, int, int, bool) {}
__device__ __forceinline__ void trace_at_any(const DevState &, int, int) {}
__device__ __forceinline__ void trace_at(const DevState &, int, int) {}
__device__ __forceinline__ void trace_count(const DevState &, int, int) {}
#endif
__device__ __forceinline__ void trace_item(const DevState &S, int k, int nth, int phase) {
  if (nth < 5) trace_at(S, k, 2 + 4 * nth + phase);
}
// sub-phase marks of a CTA's first item: slots 22..26
__device__ __forceinline__ void trace_sub(const DevState &S, int k, int nth, int sub) {
  if (nth == 0) trace_at(S, k, 22 + sub);
}

// ---------------------------------------------------------------- tables
__constant__ uint8_t c_tri_count[256] = VM_TRI_COUNT_INIT;
__constant__ unsigned long long c_tri_packed[256] = VM_TRI_PACKED_INIT;
// edge geometry (mc_tables.py:44-64): owner offset (packed), axis, oriented corners
__constant__ uint8_t c_e_own[12] = {0, 1, 2, 0, 4, 5, 6, 4, 0, 1, 3, 2};
__constant__ uint8_t c_e_axis[12] = {0, 1, 0, 1, 0, 1, 0, 1, 2, 2, 2, 2};
__constant__ uint8_t c_e_start[12] = {0, 1, 3, 0, 4, 5, 7, 4, 0, 1, 2, 3};
__constant__ uint8_t c_e_end[12] = {1, 2, 2, 3, 5, 6, 6, 7, 4, 5, 6, 7};
__constant__ uint8_t c_regular[6] = {0x99, 0x66, 0x33, 0xCC, 0x0F, 0xF0};
// global-memory copies, staged into shared memory by the meshing kernels
// (coalesced loads; constant-bank reads with per-thread indices serialise)
__device__ const uint8_t g_tri_count[256] = VM_TRI_COUNT_INIT;
__constant__ uint8_t c_slab_sel[8];

// EDGE_MASK[t] (mc_tables.py:79-112) computed from the corner bits: edge e is
// active iff its two corners differ (edges (i, i+1 mod 4) of each face ring,
// then the 4 verticals (i, i + 4)); equal to the table for all 256 types
// (tests/test_tables.py)
__host__ __device__ __forceinline__ unsigned edge_mask_of(unsigned t) {
  const unsigned x = t ^ (((t >> 1) & 0x77u) | ((t << 3) & 0x88u));
  return (x & 0xFFu) | (((t ^ (t >> 4)) & 0xFu) << 8);
}

__host__ __device__ inline bool is_regular_type(unsigned t) {
  return t == 0x99 || t == 0x66 || t == 0x33 || t == 0xCC || t == 0x0F || t == 0xF0;
}

// ---------------------------------------------------------------- keys
__device__ __forceinline__ long long pack_coord(int x, int y, int z) {
  const long long off = 1LL << 20;
  return ((((long long)x + off) << 42) | (((long long)y + off) << 21) | ((long long)z + off));
}
// Bucket of a packed block coordinate.  Where a block sits in the table is
// not observable (the reference's contract is one allocation per coordinate
// and CapacityError at 2n >= table_size, store.py:296-320), so the bucket uses
// a full 64-bit mix rather than the reference's xor-of-primes slot hash
// (store.py:84-87), which clusters spatially coherent keys into shared buckets.
__device__ __forceinline__ unsigned bucket_of(const DevState &S, long long key) {
  unsigned long long h = (unsigned long long)key;
  h ^= h >> 33; h *= 0xff51afd7ed558ccdULL;
  h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ULL;
  h ^= h >> 33;
  return S.bmask ? (unsigned)h & S.bmask : (unsigned)(h % (unsigned long long)S.nbuckets);
}

template <typename T>
__device__ __forceinline__ T ld_vol(const T *p) { return *(const volatile T *)p; }

__device__ __forceinline__ void set_error(const DevState &S, int code, long long a = 0,
                                          long long b = 0, long long c = 0, long long d = 0) {
  if (atomicCAS(&S.ctr->error, 0, code) == 0) {
    S.ctr->err_info[0] = a; S.ctr->err_info[1] = b;
    S.ctr->err_info[2] = c; S.ctr->err_info[3] = d;
  }
}

__device__ __forceinline__ void add64(int64_t *p, long long v) {
  if (v) atomicAdd((unsigned long long *)p, (unsigned long long)v);
}

// ---------------------------------------------------------------- hash table
__device__ __forceinline__ int wait_val(const int32_t *p) {
  int v;
  while ((v = ld_vol(p)) == -1) __nanosleep(32);
  return v;
}

// A probe result: block index (-1 absent, -2 capacity error), the slot's
// "collected" epoch stamp as read, and where that stamp lives.
struct HashRef {
  int idx;
  int stamp;
  int32_t *stamp_ptr;
  int free_slot;   // (find, key absent) the bucket's first empty slot, -1 if full
};

// get_block with the slot's stamp: every bucket slot is one 16-byte load
// (key, index, stamp), so a probe is a single round trip in the common case
__device__ HashRef hash_find_ref(const DevState &S, int x, int y, int z) {
  const long long key = pack_coord(x, y, z);
  const unsigned b = bucket_of(S, key);
  HashSlot *kb = S.slots + (size_t)b * kSlotsPerBucket;
  int4 v[kSlotsPerBucket];   // the whole 128-B bucket in one round trip
#pragma unroll
  for (int i = 0; i < kSlotsPerBucket; i++) v[i] = __ldcg(reinterpret_cast<const int4 *>(kb + i));
  // first slot holding the key or empty (slots fill in prefix order), with
  // register selects only (no dynamically indexed local array)
  int hit = -1, idx = -1, stamp = -1, fs = -1;
  bool stop = false;
#pragma unroll
  for (int i = 0; i < kSlotsPerBucket; i++) {
    const long long k = (long long)(((unsigned long long)(unsigned)v[i].y << 32) | (unsigned)v[i].x);
    if (!stop && k == key) { hit = i; idx = v[i].z; stamp = v[i].w; }
    if (!stop && k == kEmptyKey) fs = i;   // (slots fill in prefix order: the first empty one)
    stop = stop || k == key || k == kEmptyKey;
  }
  if (hit >= 0) {
    if (idx == -1) {   // (being inserted: the stamp is written before the index is published)
      idx = wait_val(&kb[hit].val);
      stamp = ld_vol(&kb[hit].pad);
    }
    if (idx == kEvicted) return {-1, -1, nullptr, -1};   // (an evicted block reads as absent)
    return {idx, stamp, &kb[hit].pad, -1};
  }
  if (stop) return {-1, -1, nullptr, fs};
  for (int e = ld_vol(S.ovf_head + b); e >= 0; e = ld_vol(S.ovf_next + e))
    if (ld_vol(S.ovf_key + e) == key) {
      const int v = ld_vol(S.ovf_val + e);
      if (v == kEvicted) return {-1, -1, nullptr, -1};
      return {v, ld_vol(S.ovf_stamp + e), S.ovf_stamp + e, -1};
    }
  return {-1, -1, nullptr, -1};
}

// SpatialStore.get_block (store.py:280-294)
__device__ int hash_find(const DevState &S, int x, int y, int z) {
  const long long key = pack_coord(x, y, z);
  const unsigned b = bucket_of(S, key);
  const HashSlot *kb = S.slots + (size_t)b * kSlotsPerBucket;
#pragma unroll
  for (int i = 0; i < kSlotsPerBucket; i++) {
    const long long k = ld_vol(&kb[i].key);
    if (k == key) {
      int v = ld_vol(&kb[i].val);
      if (v == -1) v = wait_val(&kb[i].val);
      return v == kEvicted ? -1 : v;
    }
    if (k == kEmptyKey) return -1;  // slots fill in prefix order
  }
  for (int e = ld_vol(S.ovf_head + b); e >= 0; e = ld_vol(S.ovf_next + e))
    if (ld_vol(S.ovf_key + e) == key) {
      const int v = ld_vol(S.ovf_val + e);
      return v == kEvicted ? -1 : v;
    }
  return -1;
}

// ---------------------------------------------------------------- partition
__device__ __forceinline__ int tile_owner(const DevState &S, int tx, int ty, int tz) {
  long long h = ((long long)tx * 73856093LL) ^ ((long long)ty * 19349669LL) ^ ((long long)tz * 83492791LL);
  long long m = h % S.nranks;
  return (int)(m < 0 ? m + S.nranks : m);
}
__device__ __forceinline__ bool block_owned(const DevState &S, int x, int y, int z) {
  return S.nranks <= 1 || tile_owner(S, x >> S.tile_shift, y >> S.tile_shift, z >> S.tile_shift) == S.rank;
}
// a block whose 27-neighbourhood reaches a tile of another rank: it lies in
// that rank's margin, so its samples are sent in halo-exchange mode
__device__ __forceinline__ bool block_on_boundary(const DevState &S, int x, int y, int z) {
  const int sh = S.tile_shift;
  for (int tx = (x - 1) >> sh; tx <= (x + 1) >> sh; tx++)
    for (int ty = (y - 1) >> sh; ty <= (y + 1) >> sh; ty++)
      for (int tz = (z - 1) >> sh; tz <= (z + 1) >> sh; tz++)
        if (tile_owner(S, tx, ty, tz) != S.rank) return true;
  return false;
}

// owned, or within one block of an owned tile (the margin this rank computes)
__device__ __forceinline__ bool block_in_margin(const DevState &S, int x, int y, int z);
// the blocks this rank's band walk collects: owned + margin (margin mode) or
// owned only (halo exchange: the margin arrives from the owners)
__device__ __forceinline__ bool block_relevant(const DevState &S, int x, int y, int z) {
  if (S.nranks <= 1) return true;
  if (S.halo_exchange) return block_owned(S, x, y, z);
  return block_in_margin(S, x, y, z);
}
__device__ __forceinline__ bool block_in_margin(const DevState &S, int x, int y, int z) {
  if (S.nranks <= 1) return true;
  const int sh = S.tile_shift;
  const int x0 = (x - 1) >> sh, x1 = (x + 1) >> sh, y0 = (y - 1) >> sh, y1 = (y + 1) >> sh;
  const int z0 = (z - 1) >> sh, z1 = (z + 1) >> sh;
  for (int tx = x0; tx <= x1; tx++)
    for (int ty = y0; ty <= y1; ty++)
      for (int tz = z0; tz <= z1; tz++)
        if (tile_owner(S, tx, ty, tz) == S.rank) return true;
  return false;
}

// allocate the next block index; CapacityError at 2*n >= table_size (store.py:304-306)
__device__ int alloc_block(const DevState &S, int x, int y, int z, int epoch) {
  // block GC: reuse an evicted block's index first (its storage is initialised
  // as a fresh block's by k_fuse_blocks).  Pops only race with pops (pushes
  // happen in k_block_gc alone): a pop that finds the list empty undoes itself.
  int idx = -1;
  if (S.free_list_on && ld_vol(&S.ctr->nfree) > 0) {   // (no round trip unless block GC ever ran)
    const int k = atomicSub(&S.ctr->nfree, 1);
    if (k > 0) idx = __ldcg(S.free_list + (k - 1));
    else atomicAdd(&S.ctr->nfree, 1);
  }
  if (idx < 0) {
    idx = atomicAdd(&S.ctr->nblocks, 1);
    if (2LL * idx >= S.table_size) {
      set_error(S, ERR_CAPACITY, idx, S.table_size, 1, epoch);
      return -2;
    }
  }
  // (latched with the call's epoch: a k_collect CTA stops only for a flag left
  // by an EARLIER frame, never for one a sibling CTA of its own frame just set)
  if (idx >= S.block_cap) atomicExch(&S.ctr->need, epoch);
  S.bcoord[idx] = make_int4(x, y, z, 0);
  S.stamp_new[idx] = epoch;
  if (S.nranks > 1) {   // (single rank: every block is owned, nblocks_owned == nblocks)
    const bool own = block_owned(S, x, y, z);
    S.bowned[idx] = own;
    if (own) atomicAdd((unsigned long long *)&S.ctr->nblocks_owned, 1ull);
  } else {
    S.bowned[idx] = 1;
  }
  atomicAdd(&S.ctr->nnew, 1);   // (a statistic: result unused, no round trip)
  return idx;
}

// SpatialStore.get_or_allocate_block (store.py:296-320): lock-free in the
// bucket (CAS the key, then publish the index) and lock-based in the bucket's
// overflow chain.  Exactly one allocation per coordinate, no dropped inserts.
__device__ HashRef hash_insert_ref(const DevState &S, int x, int y, int z, int epoch);
__device__ int hash_insert(const DevState &S, int x, int y, int z, int epoch) {
  return hash_insert_ref(S, x, y, z, epoch).idx;
}
__device__ HashRef hash_insert_ref(const DevState &S, int x, int y, int z, int epoch) {
  const long long key = pack_coord(x, y, z);
  const unsigned b = bucket_of(S, key);
  HashSlot *kb = S.slots + (size_t)b * kSlotsPerBucket;
  for (int i = 0; i < kSlotsPerBucket; i++) {
    long long k = ld_vol(&kb[i].key);
    if (k == kEmptyKey) {
      k = (long long)atomicCAS((unsigned long long *)&kb[i].key, (unsigned long long)kEmptyKey,
                               (unsigned long long)key);
      if (k == kEmptyKey) {
        // publish the index: readers in this kernel use only the index (the
        // block's coordinate and stamps are read by later kernels)
        const int idx = alloc_block(S, x, y, z, epoch);
        *(volatile int32_t *)&kb[i].val = idx;
        return {idx, ld_vol(&kb[i].pad), &kb[i].pad, -1};
      }
    }
    if (k == key) {
      // an evicted block's key: the first re-inserter allocates a new block
      if (ld_vol(&kb[i].val) == kEvicted && atomicCAS(&kb[i].val, kEvicted, -1) == kEvicted) {
        const int idx = alloc_block(S, x, y, z, epoch);
        *(volatile int32_t *)&kb[i].val = idx;
        return {idx, ld_vol(&kb[i].pad), &kb[i].pad, -1};
      }
      const int v = wait_val(&kb[i].val);
      return {v, ld_vol(&kb[i].pad), &kb[i].pad, -1};
    }
  }
  int32_t *sp = nullptr;
  int found = -1;
  bool done = false;
  while (!done) {
    if (atomicCAS(S.ovf_lock + b, 0, 1) == 0) {
      __threadfence();
      for (int e = ld_vol(S.ovf_head + b); e >= 0; e = ld_vol(S.ovf_next + e))
        if (ld_vol(S.ovf_key + e) == key) {
          sp = S.ovf_stamp + e;
          found = ld_vol(S.ovf_val + e);
          if (found == kEvicted) {   // (under the bucket's lock)
            found = alloc_block(S, x, y, z, epoch);
            S.ovf_val[e] = found;
          }
          break;
        }
      if (found == -1) {
        int e = atomicAdd(&S.ctr->ovf_count, 1);
        if (e >= S.ovf_cap) {
          set_error(S, ERR_CAPACITY, e, S.ovf_cap, 2, epoch);
          found = -2;
        } else {
          found = alloc_block(S, x, y, z, epoch);
          S.ovf_key[e] = key;
          S.ovf_val[e] = found;
          S.ovf_stamp[e] = -1;
          sp = S.ovf_stamp + e;
          S.ovf_next[e] = S.ovf_head[b];
          __threadfence();
          atomicExch(S.ovf_head + b, e);
        }
      }
      __threadfence();
      atomicExch(S.ovf_lock + b, 0);
      done = true;
    } else {
      __nanosleep(64);
    }
  }
  return {found, sp ? ld_vol(sp) : -1, sp, -1};
}

// k_collect's insert of a key its find did not see, at the bucket slot the
// find saw empty (no second read of the bucket): the thread that creates the
// block marks it collected by this call itself -- stamp first, then the index
// published with release semantics, so a concurrent finder that waits for the
// index sees the stamp and does not collect it twice.  Returns the index and
// whether this thread collected it (else it falls back to the general insert
// and the caller's stamp exchange).
__device__ __forceinline__ HashRef hash_insert_collect(const DevState &S, int x, int y, int z, int epoch,
                                                       int free_slot, bool *created) {
  *created = false;
  if (free_slot >= 0) {
    const long long key = pack_coord(x, y, z);
    HashSlot *ks = S.slots + (size_t)bucket_of(S, key) * kSlotsPerBucket + free_slot;
    const long long k = (long long)atomicCAS((unsigned long long *)&ks->key, (unsigned long long)kEmptyKey,
                                             (unsigned long long)key);
    if (k == kEmptyKey) {
      const int idx = alloc_block(S, x, y, z, epoch);
      ks->pad = epoch;
      asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(&ks->val), "r"(idx) : "memory");
      *created = idx >= 0;
      return {idx, epoch, &ks->pad, -1};
    }
    if (k == key) {   // (someone else inserted it just now)
      const int v = wait_val(&ks->val);
      if (v != kEvicted) return {v, ld_vol(&ks->pad), &ks->pad, -1};
    }
  }
  return hash_insert_ref(S, x, y, z, epoch);
}

// ---------------------------------------------------------------- misc
__device__ __forceinline__ int nbr_dir(int dx, int dy, int dz) {
  return (dx + 1) * 9 + (dy + 1) * 3 + (dz + 1);
}

// floor(p / e) exactly as the correctly rounded division, without dividing in
// the common case: q = RN(p * RN(1/e)) is within ~2.2e-16 |p/e| of p/e (and of
// RN(p/e)), so unless q lies within 1e-7 of an integer (|p/e| < 2^21 here) both
// floor to the same value; near an integer the exact quotient decides.
__device__ __forceinline__ int floor_div_exact(double p, double e, double inv_e) {
  const double q = __dmul_rn(p, inv_e);
  const double f = floor(q);
  const double r = q - f;   // exact
  if (r > 1e-7 && r < 1.0 - 1e-7) return (int)f;
  return (int)floor(p / e);
}
// its common case alone: floor(RN(p * RN(1/e))); `near` is set when q lies
// within 1e-7 of an integer (the caller then takes floor(p / e))
__device__ __forceinline__ int floor_div_fast(double p, double inv_e, bool &near) {
  const double q = __dmul_rn(p, inv_e);
  const double f = floor(q);
  const double r = q - f;   // exact
  near |= !(r > 1e-7 && r < 1.0 - 1e-7);
  return (int)f;
}

// out_j = fma(a2, B[2][j], fma(a1, B[1][j], a0*B[0][j])) -- numpy `a @ B`
__device__ __forceinline__ double matvec_col(const double *a, const double *B, int j) {
  return __fma_rn(a[2], B[6 + j], __fma_rn(a[1], B[3 + j], __dmul_rn(a[0], B[j])));
}
// out_j = sum_k a_k * B[j][k]  -- numpy `a @ B.T`
__device__ __forceinline__ double matvec_row(const double *a, const double *B, int j) {
  return __fma_rn(a[2], B[3 * j + 2], __fma_rn(a[1], B[3 * j + 1], __dmul_rn(a[0], B[3 * j])));
}

// fusion.block_in_frustum (fusion.py:171-190)
__device__ bool block_in_frustum_dev(int4 c, const FrameDev &F, double extent) {
  double base[3] = {(double)c.x * extent, (double)c.y * extent, (double)c.z * extent};
  const double *t = F.t;
  if (t[0] >= base[0] && t[1] >= base[1] && t[2] >= base[2] && t[0] <= base[0] + extent &&
      t[1] <= base[1] + extent && t[2] <= base[2] + extent)
    return true;
  for (int q = 0; q < 8; q++) {
    double o[3] = {(double)((q >> 2) & 1), (double)((q >> 1) & 1), (double)(q & 1)};
    double a[3], cam[3];
    for (int j = 0; j < 3; j++) a[j] = (base[j] + o[j] * extent) - t[j];
    for (int j = 0; j < 3; j++) cam[j] = matvec_col(a, F.R, j);
    if (!(cam[2] > 0)) continue;
    double u = F.fx * cam[0] / cam[2] + F.cx;
    double v = F.fy * cam[1] / cam[2] + F.cy;
    if (u >= 0 && u < (double)F.width && v >= 0 && v < (double)F.height) return true;
  }
  return false;
}

// refine.refine_block_types for one cube (refine.py:98-135).  `small` = bit k
// set iff |corner k| < epsilon.  Returns the new type; *changed as counted by
// the reference (hit & new != current).
__device__ __forceinline__ unsigned refine_type(unsigned tc, unsigned tp, unsigned small,
                                                bool *changed) {
  *changed = false;
  if (__popc((tc ^ tp) & 0xFF) > 3) return tc;
  int best_score = 255;
  unsigned best = 0;
#pragma unroll
  for (int j = 0; j < 6; j++) {
    const unsigned reg = c_regular[j];
    const unsigned diff = (tc ^ reg) & 0xFF;
    const int dist = __popc(diff);
    if (dist > 3 || (diff & ~small)) continue;   // a disagreeing corner is not near zero
    const int score = dist * 8 + j;
    if (score < best_score) { best_score = score; best = reg; }
  }
  if (best_score < 255) {
    *changed = (tc != best);
    return best;
  }
  return tc;
}

// ---------------------------------------------------------------- reductions
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum (blockDim multiple of 32); result valid in thread 0
__device__ __forceinline__ long long block_sum(long long v, long long *sh) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  long long r = 0;
  if (wid == 0) {
    r = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : 0;
    r = warp_sum(r);
  }
  return r;
}


// Warp sums of N per-thread counters (each < 2^31 in magnitude per warp), added
// by lane k to dst[k] (a reduction, no round trip; null = skip): no barrier, so
// a warp that finishes early leaves without waiting for the rest of its CTA.
template <int N>
__device__ __forceinline__ void warp_add_counters(const int (&vals)[N], int64_t *const (&dst)[N]) {
  const int lane = threadIdx.x & 31;
  int mine = 0;
  int64_t *d = nullptr;
#pragma unroll
  for (int k = 0; k < N; k++) {
    const int v = (int)__reduce_add_sync(0xffffffffu, (unsigned)vals[k]);
    if (lane == k) { mine = v; d = dst[k]; }
  }
  if (mine && d) atomicAdd((unsigned long long *)d, (unsigned long long)(long long)mine);
}

// vertex position from its slot (mesher.py:216-235): every coordinate is
// (owner cube index) * l except the edge axis, which holds the interpolated
// value stored at placement.  Bit-identical to the reference.
__device__ __forceinline__ void slot_position(const DevState &S, int blk, int slot, double *p) {
  const int4 c = S.bcoord[blk];
  const int ci = slot / 3, axis = slot - 3 * (slot / 3);
  const int g[3] = {c.x * kB + (ci >> 6), c.y * kB + ((ci >> 3) & 7), c.z * kB + (ci & 7)};
  for (int d = 0; d < 3; d++) p[d] = __dmul_rn((double)g[d], S.cube_size);
  p[axis] = S.vparam[(size_t)blk * kEV + slot];
}

}  // namespace vm
