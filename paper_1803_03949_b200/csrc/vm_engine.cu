// vm_engine.cu -- host runtime of the B200 mesh-generation path and the C ABI
// declared in include/voxmesh_b200.h.
//
// One engine == one SpatialStore in HBM + one CUDA stream.  A frame is five
// persistent-grid kernels that read their work counts from device counters
// (no host sync inside a frame).  The only speculatively sized structure is
// the block heap: if a frame allocates past its capacity, every kernel after
// k_collect exits immediately, the host grows the heap and resumes the frame
// at k_fuse_blocks (collect + allocation is idempotent).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <array>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/voxmesh_b200.h"
#include "vm_kernels.cuh"
#include "vm_partition.cuh"

using namespace vm;

// NVTX ranges around the host-side phases (frame enqueue, settle wait,
// compaction, halo exchange) so an nsys / ncu timeline names them; free when
// no tool is attached (header-only NVTX v3).
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static thread_local std::string g_err;

static int set_err(int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t _e = (x);                                                                \
    if (_e != cudaSuccess)                                                               \
      return set_err(VM_ERR_CUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(_e), \
                     __FILE__, __LINE__);                                                \
  } while (0)

#define TRY(x)                  \
  do {                          \
    int _r = (x);               \
    if (_r != VM_OK) return _r; \
  } while (0)

enum Phase { PH_DEPTH = 0, PH_COLLECT, PH_FUSE, PH_RETYPE, PH_GC, PH_END, PH_COUNT };

struct Compacted {
  double *pos = nullptr, *nrm = nullptr;
  long long *age = nullptr;
  int32_t *idx = nullptr;
  int32_t *ev_handles = nullptr, *tri_handles = nullptr;
  int64_t nv = 0, nt = 0;
};

struct vm_engine {
  vm_store_config cfg{};
  DevState S{};
  Counters *h_ctr = nullptr;   // pinned mirror
  FrameDev *h_frame = nullptr; // pinned; passed by value to every kernel
  double *d_depth = nullptr;
  size_t depth_cap = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int32_t epoch = 0;
  int sm_count = 148;
  int grid_retype = 296, grid_gc = 296, grid_fuse = 296, grid_collect = 296, grid_parity = 296;
  void *d_scratch = nullptr;
  size_t scratch_cap = 0;
  Compacted comp;
  cudaEvent_t evs[2][PH_COUNT] = {};   // per frame slot (two frames may be in flight)
  cudaEvent_t *ev = evs[0];            // the slot being enqueued / settled
  bool profiling = false;
  int pending = 0;
  int64_t pending_frame = 0;
  // Frame slots: each enqueued frame keeps its parameters, a pinned snapshot of
  // the counters taken after its last kernel, and an event behind that copy, so
  // vm_fuse_frame_submit can queue frame t+1 before frame t is settled.
  int fslot = 0;                      // slot of the most recently enqueued frame
  FrameDev f_saved[2];                // its parameters (as launched)
  // Frame counters: k_gc_normals' commit copies them to d_snapbuf[slot]; when
  // the next frame is already queued its k_collect publishes that copy to the
  // mapped pinned h_snap[slot] and then writes the sequence word h_seq[slot]
  Counters *d_snapbuf[2] = {nullptr, nullptr};
  Counters *h_snap[2] = {nullptr, nullptr};
  unsigned long long *h_seq[2] = {nullptr, nullptr};
  Counters *d_snap[2] = {nullptr, nullptr};           // (device views of h_snap / h_seq)
  unsigned long long *d_seq[2] = {nullptr, nullptr};
  bool publish_prev = false;          // set by vm_fuse_frame_submit: the frame launched next publishes
  bool host_input = false;            // set by vm_fuse_frame_submit: this frame's depth came by a host copy
  bool in_submit = false;             // set by vm_fuse_frame_submit[_raw] around the enqueue
  bool self_pub[2] = {false, false};  // the slot's frame publishes its own snapshot (gc commit)
  unsigned long long snap_ids = 0, want_id[2] = {0, 0};
  bool ev_rec[2] = {false, false};   // the slot's frame recorded PH_DEPTH / PH_END events
  bool ctr_clean = false;            // the per-call counters are zero (a frame's commit cleared them)
  bool restore_calls = false;        // ... and hold nothing: a non-frame call restores the last frame's
  int64_t frame_of[2] = {0, 0};
  // Frame overlap: the stream's last operation is the k_gc_normals (epoch
  // ov_epoch) of a frame launch_frame queued -- the next frame's k_collect may
  // then start under it (FrameDev::overlap).  Every other entry point clears it.
  bool ov_ready = false;
  int32_t ov_epoch = 0;
  bool ov_of[2] = {false, false};   // the slot's frame was launched overlapped
  bool no_overlap = getenv("VOXMESH_B200_NO_OVERLAP") != nullptr;   // (A/B switch)
  bool host_prof = getenv("VOXMESH_B200_HOST_PROF") != nullptr;   // (diagnostics: host time per submit)
  std::vector<std::array<double, 3>> hp;   // per submit: enqueue, settle, wall since the previous submit's end
  double hp_last = 0;
  int last_resumes = 0;
  int resume_launches = 0;   // kernels the resumes of the last settled frame launched
  int frame_launches = 0;   // kernels launched by the pending / last frame
  // pipelined submission (vm_fuse_frame_submit): the next frame's depth is
  // copied on a second stream into the other slot while the pending frame runs
  cudaStream_t copy_stream = nullptr;
  double *d_slot[2] = {nullptr, nullptr};
  size_t slot_cap = 0;
  int slot = 0;
  cudaEvent_t ev_copy[2] = {nullptr, nullptr};
  cudaEvent_t ev_order = nullptr;   // vm_order_after
  bool defer_wait = false;          // vm_set_deferred_input_wait
  // device-side input flags (FrameDev::in_flag): per slot, written by the copy
  // stream after the frame's host copy
  unsigned long long *d_inseq = nullptr, *h_inseq = nullptr, in_id = 0;
  int in_slot = -1;                 // the slot the frame being enqueued waits on
  int copy_pending = -1;            // slot whose host copy the caller has not waited for yet
  uint16_t *d_raw[2] = {nullptr, nullptr};   // raw u16 frames (vm_fuse_frame_submit_raw)
  size_t raw_cap = 0;
  const uint16_t *raw_next = nullptr;          // set while a raw frame is being enqueued
  double raw_scale = 0.0;
  vm_stats settled{};       // stats of the last settled, not yet delivered frame
  int settled_valid = 0;
  // ray-norm bounds over the image, cached per (h, w, fx, fy, cx, cy)
  double norm_key[6] = {0, 0, 0, 0, 0, 0};
  double norm_lo = 0.0, norm_hi = 0.0;
  bool norm_valid = false;
  double *d_rays = nullptr;   // ray tables of the cached intrinsics (k_norm_bounds)
  size_t rays_cap = 0;
  // spatial partition: a halo-exchange frame between begin and finish, and
  // the owned-block arrays of a distributed compaction
  bool part_active = false;
  int32_t part_nc_own = 0;
  int64_t part_frame = 0;
  int32_t *d_ghost_counts = nullptr;   // [kMaxRanks]
  struct {
    unsigned long long *keys_in = nullptr, *keys_out = nullptr;
    int32_t *vals = nullptr, *order = nullptr, *vcnt = nullptr, *tcnt = nullptr;
    uint32_t *occ_bits = nullptr;
    uint16_t *occ_pre = nullptr;
    void *tmp = nullptr;
    int nb = 0, nown = 0;
  } pc;
};
constexpr int kMaxRanks = 256;

extern "C" {
static int settle(vm_engine *e);
static int settle_all(vm_engine *e);
static int settle_slot(vm_engine *e, int slot, bool succ);
}

// ------------------------------------------------------------ helpers
template <typename T>
static int dev_alloc(T **p, size_t n, int fill_byte = -2) {
  *p = nullptr;
  if (n == 0) n = 1;
  CK(cudaMalloc((void **)p, n * sizeof(T)));
  if (fill_byte != -2) CK(cudaMemset(*p, fill_byte, n * sizeof(T)));
  return VM_OK;
}

template <typename T>
static int dev_grow(T **p, size_t old_n, size_t new_n, cudaStream_t st) {
  T *q = nullptr;
  CK(cudaMalloc((void **)&q, new_n * sizeof(T)));
  if (*p && old_n) CK(cudaMemcpyAsync(q, *p, old_n * sizeof(T), cudaMemcpyDeviceToDevice, st));
  CK(cudaStreamSynchronize(st));
  if (*p) CK(cudaFree(*p));
  *p = q;
  return VM_OK;
}

static int scratch(vm_engine *e, size_t bytes, void **out) {
  if (bytes > e->scratch_cap) {
    if (e->d_scratch) CK(cudaFree(e->d_scratch));
    e->d_scratch = nullptr;
    const size_t cap = std::max(bytes, (size_t)1 << 20);
    CK(cudaMalloc(&e->d_scratch, cap));
    e->scratch_cap = cap;
  }
  *out = e->d_scratch;
  return VM_OK;
}

static inline int grid_blocks(vm_engine *e) { return e->sm_count * 4; }
static inline int grid_threads(vm_engine *e, long long n, int tpb) {
  long long g = (n + tpb - 1) / tpb;
  const long long cap = (long long)e->sm_count * 8;
  if (g < 1) g = 1;
  return (int)std::min(g, cap);
}

// every host<->device copy is ordered on the engine's (non-blocking) stream;
// a plain cudaMemcpy would run on the legacy stream, unordered with it
static int copy_sync(vm_engine *e, void *dst, const void *src, size_t bytes, cudaMemcpyKind kind) {
  if (!bytes) return VM_OK;
  CK(cudaMemcpyAsync(dst, src, bytes, kind, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  return VM_OK;
}

// Programmatic Dependent Launch: the kernel's CTAs are scheduled while the
// previous kernel of the frame drains; they wait in cudaGridDependencySynchronize()
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kern)(KArgs...), int grid, int block, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}

// k_gc_normals (its face-normal fallback records are applied by the next
// frame's k_collect, or by flush_fallbacks)
static void launch_gc(vm_engine *e, bool pdl, const int32_t *list, const int32_t *count_ptr, int count_const,
                      int mode) {
  if (pdl)
    launch_pdl(k_gc_normals, e->grid_gc, kGT, e->stream, e->S, *e->h_frame, list, count_ptr, count_const, mode);
  else
    k_gc_normals<<<e->grid_gc, kGT, 0, e->stream>>>(e->S, *e->h_frame, list, count_ptr, count_const, mode);
}

static int check_launch() {
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_err(VM_ERR_CUDA, "kernel launch failed: %s", cudaGetErrorString(err));
  return VM_OK;
}

static int grow_blocks(vm_engine *e, int64_t need) {
  DevState &S = e->S;
  int64_t cap = std::max<int64_t>((int64_t)S.block_cap * 2, need + need / 4 + 8);
  cap = std::min<int64_t>(cap, (int64_t)S.max_blocks);
  if (cap < need) cap = need;
  if (cap <= S.block_cap) return VM_OK;
  const size_t o = (size_t)S.block_cap, n = (size_t)cap;
  cudaStream_t st = e->stream;
  TRY(dev_grow(&S.tsdf, o * kNC, n * kNC, st));
  TRY(dev_grow(&S.weight, o * kNC, n * kNC, st));
  TRY(dev_grow(&S.vmask, o * (kNC / 32), n * (kNC / 32), st));
  TRY(dev_grow(&S.tp, o * kNC, n * kNC, st));
  TRY(dev_grow(&S.tc, o * kNC, n * kNC, st));
  TRY(dev_grow(&S.vh, o * kEV, n * kEV, st));
  CK(cudaMemsetAsync(S.vh + o * kEV, 0xFF, (n - o) * kEV * sizeof(int32_t), st));   // (no record yet)
  TRY(dev_grow(&S.vrb, o * (kEV / 32), n * (kEV / 32), st));
  CK(cudaMemsetAsync(S.vrb + o * (kEV / 32), 0, (n - o) * (kEV / 32) * sizeof(uint32_t), st));
  TRY(dev_grow(&S.vocc, o * (kEV / 32), n * (kEV / 32), st));
  TRY(dev_grow(&S.vclaim, o * (kEV / 32), n * (kEV / 32), st));
  TRY(dev_grow(&S.vparam, o * kEV, n * kEV, st));
  TRY(dev_grow(&S.item_mask, 0, n * 16, st));
  if (S.vreq) {   // strategy "partition" buffers (zero request bytes for the new blocks)
    TRY(dev_grow(&S.vreq, o * kEV, n * kEV, st));
    CK(cudaMemsetAsync(S.vreq + o * kEV, 0, (n - o) * kEV, st));
    TRY(dev_grow(&S.psel, 0, n * 64, st));
  }
  S.block_cap = (int32_t)cap;
  return VM_OK;
}

// Vertex-record arena: at least `need` records (grows geometrically; the
// records are addressed by handle, so a copy keeps them valid)
static int grow_records(vm_engine *e, int64_t need) {
  DevState &S = e->S;
  if (need <= S.vrec_cap) return VM_OK;
  const int64_t cap = std::max<int64_t>(need + need / 4, (int64_t)S.vrec_cap * 2);
  if (cap > INT32_MAX) return set_err(VM_ERR_CAPACITY, "vertex record arena exhausted (%lld)", (long long)need);
  TRY(dev_grow(&S.vrec, (size_t)S.vrec_cap, (size_t)cap, e->stream));
  S.vrec_cap = cap;
  return VM_OK;
}

// HBM per stored block: tsdf f64, weight i32, weight > 0
// bits, type_prev / type_curr u8 per cube; per edge slot: position f64, record
// handle i32, occupancy / request / has-record bits; the explicit-scope mask
constexpr size_t kBlockBytes = 8 * kNC + 4 * kNC + 4 * (kNC / 32) + 2 * kNC + 8 * kEV + 4 * kEV +
                               3 * 4 * (kEV / 32) + 4 * 16;
// per-block metadata, sized for the table's block limit: coordinate, neighbour
// row, epoch stamps, slab / owner bytes, ghost / GC / free-list entries, scope
// and halo list entries
constexpr size_t kBlockMetaBytes = 16 + 27 * 4 + 3 * 4 + 1 + 1 + 4 + 4 + 4 + 4 + 4;

static int read_counters(vm_engine *e) {
  CK(cudaMemcpyAsync(e->h_ctr, e->S.ctr, sizeof(Counters), cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  return VM_OK;
}

static int recover_after_error(vm_engine *e);
static int error_message(vm_engine *e);

// Report the device error flag of the call just read back (h_ctr) and clear
// it, so the store stays usable after the error as the reference's does
// (compact / audit / snapshots of the partially updated store, later frames).
static int error_from_counters(vm_engine *e) {
  const int rc = error_message(e);
  if (rc != VM_OK) {
    const std::string msg = g_err;
    recover_after_error(e);   // (best effort: the call's own error is what is reported)
    g_err = msg;
  }
  return rc;
}

static int error_message(vm_engine *e) {
  const Counters &c = *e->h_ctr;
  if (c.error == ERR_CAPACITY) {
    if (c.err_info[2] == 1)
      return set_err(VM_ERR_CAPACITY, "block table full (%lld blocks, size %lld)",
                     (long long)c.err_info[0], (long long)c.err_info[1]);
    if (c.err_info[2] == 3)
      return set_err(VM_ERR_CAPACITY, "vertex pool exhausted (%lld vertices)", (long long)c.err_info[1]);
    return set_err(VM_ERR_CAPACITY, "hash overflow chain exhausted");
  }
  if (c.error == ERR_CONSISTENCY) {
    switch (c.err_info[0]) {
      case 10:
        return set_err(VM_ERR_CONSISTENCY, "edge owner block absent during placement (cube %lld, %lld, %lld)",
                       (long long)c.err_info[1], (long long)c.err_info[2], (long long)c.err_info[3]);
      case 40: return set_err(VM_ERR_CONSISTENCY, "triangle references a vertex bound to no edge");
      case 50: return set_err(VM_ERR_CUDA, "k_gc_normals grid barrier timed out (CTAs not co-resident)");
      case 60: return set_err(VM_ERR_CUDA, "the frame's host->device depth copy did not arrive");
      default: return set_err(VM_ERR_CONSISTENCY, "consistency error %lld", (long long)c.err_info[0]);
    }
  }
  return VM_OK;
}

// After a reported error: clamp the block / overflow counts the failed
// allocations ran past, give every allocated block its storage, initialise
// (and link) the blocks a failed k_collect allocated -- its k_fuse_blocks never
// ran, so they are empty blocks as the reference leaves them after
// get_or_allocate_block raised (store.py:296-320) -- and clear the flags.
static int recover_after_error(vm_engine *e) {
  Counters &c = *e->h_ctr;
  const bool collect_time = c.error == ERR_CAPACITY && (c.err_info[2] == 1 || c.err_info[2] == 2);
  const int32_t epoch = (int32_t)c.err_info[3];
  c.nblocks = std::min<int32_t>(c.nblocks, e->S.max_blocks);
  c.ovf_count = std::min<int32_t>(c.ovf_count, e->S.ovf_cap);
  if (c.nblocks > e->S.block_cap) TRY(grow_blocks(e, c.nblocks));
  c.error = 0;
  c.need = 0;
  for (auto &v : c.err_info) v = 0;
  const size_t persist = offsetof(Counters, nvalid);
  TRY(copy_sync(e, e->S.ctr, e->h_ctr, persist, cudaMemcpyHostToDevice));
  if (collect_time && epoch > 0)
    k_init_blocks<<<grid_blocks(e), kThreadsCube, 0, e->stream>>>(e->S, epoch);
  TRY(check_launch());
  CK(cudaStreamSynchronize(e->stream));
  return VM_OK;
}

static int reset_call_counters(vm_engine *e) {
  const size_t off = offsetof(Counters, nvalid);
  CK(cudaMemsetAsync((char *)e->S.ctr + off, 0, sizeof(Counters) - off, e->stream));
  return VM_OK;
}

static inline void rec(vm_engine *e, int ph) {
  if (e->profiling) cudaEventRecord(e->ev[ph], e->stream);   // (else the kernels' own clock: t_start/t_end_ns)
}

// strategy "partition" buffers, allocated on first use (block storage size)
static int ensure_partition_bufs(vm_engine *e, int strategy) {
  DevState &S = e->S;
  if (strategy != VM_STRATEGY_PARTITION || S.vreq) return VM_OK;
  TRY(dev_alloc(&S.vreq, (size_t)S.block_cap * kEV, 0));
  TRY(dev_alloc(&S.psel, (size_t)S.block_cap * 64));
  return VM_OK;
}

// kernels of the meshing segment before k_gc_normals: k_retype_place, then for
// strategy "partition" the eight parity passes of the placement
static int meshing_launches(const FrameDev &F) { return F.strategy == VM_STRATEGY_PARTITION ? 9 : 1; }
static void launch_retype(vm_engine *e, bool pdl, const FrameDev &F) {
  const DevState &S = e->S;
  cudaStream_t st = e->stream;
  if (pdl) launch_pdl(k_retype_place, e->grid_retype, kNT, st, S, F);
  else k_retype_place<<<e->grid_retype, kNT, kRetypeSmem, st>>>(S, F);
  if (F.strategy == VM_STRATEGY_PARTITION)
    for (int p = 0; p < 8; p++) launch_pdl(k_place_parity, e->grid_parity, kNT, st, S, F, p);
}
static int gc_strategy_flag(const FrameDev &F) { return F.strategy == VM_STRATEGY_PARTITION ? G_PARTITION : 0; }

static int clear_need(vm_engine *e) {
  CK(cudaMemsetAsync(&e->S.ctr->need_stage, 0, sizeof(int32_t), e->stream));
  CK(cudaMemsetAsync(&e->S.ctr->need, 0, sizeof(int32_t), e->stream));
  return VM_OK;
}

// records a halted meshing segment may need (k_retype_place's bound, with the
// counters just read back)
static int64_t record_bound(vm_engine *e) {
  const Counters &c = *e->h_ctr;
  const int64_t items = (int64_t)c.ncollected + c.nslab + c.nexplicit;
  return c.a_hw + std::min<int64_t>(kRecsPerItem * items, (int64_t)kEV * c.nblocks) +
         4 * kRecChunk * e->S.rec_chunk_ctas + 1024;
}

// meshing segment: retype+place, gc+normals (a frame resumed for records)
static int enqueue_meshing(vm_engine *e) {
  const FrameDev F = *e->h_frame;
  rec(e, PH_RETYPE);
  launch_retype(e, true, F);
  rec(e, PH_GC);
  launch_gc(e, true, e->S.halo, &e->S.ctr->nhalo, 0,
            (int)(G_GC | G_NORMALS | G_COMMIT | G_REQUIRE_ITEMS | G_SHARDED) | gc_strategy_flag(F));
  rec(e, PH_END);
  return check_launch();
}

// frame segment after collect: fuse (init/integrate/scope), retype+place, gc+normals
static int enqueue_after_collect(vm_engine *e) {
  DevState &S = e->S;
  cudaStream_t st = e->stream;
  const int gb = grid_blocks(e);
  const FrameDev F = *e->h_frame;
  rec(e, PH_FUSE);
  launch_pdl(k_fuse_blocks, e->grid_fuse, kFB, st, S, F, (const int32_t *)S.scope,
             (const int32_t *)&S.ctr->ncollected, 0, (int)(F_INIT | F_INTEGRATE | F_SCOPE), 0);
  rec(e, PH_RETYPE);
  launch_retype(e, true, F);
  rec(e, PH_GC);
  launch_gc(e, true, S.halo, &S.ctr->nhalo, 0,
            (int)(G_GC | G_NORMALS | G_COMMIT | G_REQUIRE_ITEMS | G_SHARDED | (F.reset_after ? G_OVERLAP : 0)) |
                gc_strategy_flag(F));
  rec(e, PH_END);
  return check_launch();
}

// host side of a (possibly resumed) frame
static int complete_with_resume(vm_engine *e, int *resumes) {
  for (int guard = 0; guard < 64; guard++) {
    TRY(read_counters(e));
    TRY(error_from_counters(e));
    if (!e->h_ctr->need) return VM_OK;
    if (resumes) (*resumes)++;
    if (e->h_ctr->need_stage == 1) {   // vertex records: grow, resume at k_retype_place
      TRY(grow_records(e, record_bound(e)));
      TRY(clear_need(e));
      TRY(enqueue_meshing(e));
      e->frame_launches += 1 + meshing_launches(*e->h_frame);
      e->resume_launches += 1 + meshing_launches(*e->h_frame);
      continue;
    }
    TRY(grow_blocks(e, e->h_ctr->nblocks));
    TRY(clear_need(e));
    TRY(enqueue_after_collect(e));
    e->frame_launches += 2 + meshing_launches(*e->h_frame);
    e->resume_launches += 2 + meshing_launches(*e->h_frame);
  }
  return set_err(VM_ERR_CUDA, "resume loop did not converge");
}

static void fill_frame_host(vm_engine *e, const double *depth_dev, int32_t h, int32_t w,
                            const vm_intrinsics *intr, const vm_pose *pose) {
  FrameDev &F = *e->h_frame;
  F.consume_fb = 0;
  F.raw = nullptr;
  F.depth_out = nullptr;
  F.overlap = 0;
  F.wait_epoch = 0;
  F.in_flag = nullptr;
  F.in_id = 0;
  F.ds_wait = 0;
  F.depth = depth_dev;
  F.h = h;
  F.w = w;
  if (intr) {
    F.fx = intr->fx; F.fy = intr->fy; F.cx = intr->cx; F.cy = intr->cy;
    F.width = intr->width; F.height = intr->height;
  }
  if (pose) {
    memcpy(F.R, pose->rotation, sizeof F.R);
    memcpy(F.t, pose->translation, sizeof F.t);
  }
}

static int stage_depth(vm_engine *e, const double *depth, int32_t h, int32_t w, int on_device,
                       const double **out) {
  if (!depth || h <= 0 || w <= 0) return set_err(VM_ERR_INPUT, "depth must be a non-empty (H, W) array");
  if (on_device) {
    *out = depth;
    return VM_OK;
  }
  const size_t bytes = (size_t)h * w * sizeof(double);
  if (bytes > e->depth_cap) {
    if (e->d_depth) CK(cudaFree(e->d_depth));
    CK(cudaMalloc((void **)&e->d_depth, bytes));
    e->depth_cap = bytes;
  }
  CK(cudaMemcpyAsync(e->d_depth, depth, bytes, cudaMemcpyHostToDevice, e->stream));
  *out = e->d_depth;
  return VM_OK;
}

// upload coords into scratch and map them to block indices
static int map_coords(vm_engine *e, const int32_t *coords, int64_t n, int32_t **idx_dev, int32_t *stamp,
                      int32_t epoch, bool insert) {
  void *buf;
  TRY(scratch(e, (size_t)n * (sizeof(int3) + sizeof(int32_t)) + 256, &buf));
  int3 *dc = (int3 *)buf;
  int32_t *di = (int32_t *)((char *)buf + ((n * sizeof(int3) + 127) & ~(size_t)127));
  if (n) {
    CK(cudaMemcpyAsync(dc, coords, (size_t)n * sizeof(int3), cudaMemcpyHostToDevice, e->stream));
    if (insert)
      k_insert_coords<<<grid_threads(e, n, 128), 128, 0, e->stream>>>(e->S, dc, (int)n, di, epoch);
    else
      k_lookup_coords<<<grid_threads(e, n, 128), 128, 0, e->stream>>>(e->S, dc, (int)n, di, stamp, epoch);
    TRY(check_launch());
  }
  *idx_dev = di;
  return VM_OK;
}

// after an insertion outside a frame: grow the heap if needed, then
// initialise + link the new blocks
static int init_new_blocks(vm_engine *e) {
  TRY(read_counters(e));
  TRY(error_from_counters(e));
  if (e->h_ctr->need) {
    TRY(grow_blocks(e, e->h_ctr->nblocks));
    TRY(clear_need(e));
  }
  k_init_blocks<<<grid_blocks(e), kThreadsCube, 0, e->stream>>>(e->S, e->epoch);
  TRY(check_launch());
  TRY(read_counters(e));
  return error_from_counters(e);
}

static void free_pcompact(vm_engine *e) {
  auto &p = e->pc;
  for (void *q : {(void *)p.keys_in, (void *)p.keys_out, (void *)p.vals, (void *)p.order, (void *)p.vcnt,
                  (void *)p.tcnt, (void *)p.occ_bits, (void *)p.occ_pre, p.tmp})
    if (q) cudaFree(q);
  e->pc = {};
}

static void free_compacted(Compacted &c) {
  for (void *p : {(void *)c.pos, (void *)c.nrm, (void *)c.age, (void *)c.idx, (void *)c.ev_handles,
                  (void *)c.tri_handles})
    if (p) cudaFree(p);
  c = Compacted();
}

// store.py:388-425 on the device; with_handles also materialises the
// per-slot / per-triangle-slot dense handles of the snapshot views
static int run_compaction(vm_engine *e, int64_t frame, bool with_handles) {
  NvtxRange nvtx_("vm_compaction");
  TRY(read_counters(e));
  const int nb = e->h_ctr->nblocks;
  cudaStream_t st = e->stream;
  free_compacted(e->comp);
  if (nb == 0) return VM_OK;
  unsigned long long *keys_in, *keys_out;
  int32_t *vals_in, *order, *vcnt, *tcnt, *vbase, *tbase, *vbase_by_blk;
  uint32_t *occ_bits;
  uint16_t *occ_pre;
  CK(cudaMalloc(&keys_in, 8ull * nb));
  CK(cudaMalloc(&keys_out, 8ull * nb));
  CK(cudaMalloc(&vals_in, 4ull * nb));
  CK(cudaMalloc(&order, 4ull * nb));
  CK(cudaMalloc(&vcnt, 4ull * (nb + 1)));
  CK(cudaMalloc(&tcnt, 4ull * (nb + 1)));
  CK(cudaMalloc(&vbase, 4ull * (nb + 1)));
  CK(cudaMalloc(&tbase, 4ull * (nb + 1)));
  CK(cudaMalloc(&vbase_by_blk, 4ull * nb));
  CK(cudaMalloc(&occ_bits, 4ull * 48 * nb));
  CK(cudaMalloc(&occ_pre, 2ull * 48 * nb));
  k_block_keys<<<grid_threads(e, nb, 256), 256, 0, st>>>(e->S, nb, keys_in, vals_in);
  size_t tmp_bytes = 0, tmp2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys_in, keys_out, vals_in, order, nb, 0, 64, st);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp2, vcnt, vbase, nb + 1, st);
  tmp_bytes = std::max(tmp_bytes, tmp2);
  void *tmp;
  CK(cudaMalloc(&tmp, tmp_bytes + 16));
  cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys_in, keys_out, vals_in, order, nb, 0, 64, st);
  CK(cudaMemsetAsync(vcnt + nb, 0, 4, st));
  CK(cudaMemsetAsync(tcnt + nb, 0, 4, st));
  k_compact_count<<<grid_blocks(e), kThreadsCube, 0, st>>>(e->S, order, nb, vcnt, tcnt, occ_bits, occ_pre);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, vcnt, vbase, nb + 1, st);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, tcnt, tbase, nb + 1, st);
  k_block_base<<<grid_threads(e, nb, 256), 256, 0, st>>>(order, vbase, nb, vbase_by_blk);
  int32_t nv = 0, nt = 0;
  CK(cudaMemcpyAsync(&nv, vbase + nb, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&nt, tbase + nb, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  Compacted &c = e->comp;
  CK(cudaMalloc(&c.pos, 24ull * (nv + 1)));
  CK(cudaMalloc(&c.nrm, 24ull * (nv + 1)));
  CK(cudaMalloc(&c.age, 8ull * (nv + 1)));
  CK(cudaMalloc(&c.idx, 12ull * (nt + 1)));
  if (with_handles) {
    CK(cudaMalloc(&c.ev_handles, 4ull * kEV * nb));
    CK(cudaMalloc(&c.tri_handles, 4ull * kNC * 5 * nb));
  }
  TRY(reset_call_counters(e));
  k_compact_vertices<<<grid_blocks(e), kThreadsCube, 0, st>>>(e->S, order, nb, occ_bits, occ_pre, vbase_by_blk,
                                                              c.pos, c.nrm, c.age, (long long)frame,
                                                              c.ev_handles);
  k_compact_triangles<<<grid_blocks(e), kThreadsCube, 0, st>>>(e->S, order, nb, tbase, occ_bits, occ_pre,
                                                               vbase_by_blk, c.idx, c.tri_handles);
  TRY(check_launch());
  CK(cudaStreamSynchronize(st));
  for (void *p : {(void *)keys_in, (void *)keys_out, (void *)vals_in, (void *)order, (void *)vcnt,
                  (void *)tcnt, (void *)vbase, (void *)tbase, (void *)vbase_by_blk, (void *)occ_bits,
                  (void *)occ_pre, tmp})
    cudaFree(p);
  c.nv = nv;
  c.nt = nt;
  TRY(read_counters(e));
  return error_from_counters(e);
}


// ------------------------------------------------------------ C ABI
extern "C" {

const char *vm_last_error(void) { return g_err.c_str(); }
const char *vm_version(void) { return "voxmesh-b200 0.2.0 (sm_100a, slot-resident cube field)"; }

int vm_create(const vm_store_config *cfg, vm_engine **out) {
  if (!cfg || !out) return set_err(VM_ERR_INPUT, "null argument");
  *out = nullptr;
  if (!(cfg->cube_size > 0)) return set_err(VM_ERR_VALUE, "cube_size must be positive");
  if (cfg->table_size < 2) return set_err(VM_ERR_VALUE, "table_size must be >= 2");
  int dev = 0;
  CK(cudaGetDevice(&dev));
  vm_engine *e = new vm_engine();
  e->cfg = *cfg;
  CK(cudaDeviceGetAttribute(&e->sm_count, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
  e->own_stream = true;
  for (int k = 0; k < 2; k++) {
    for (int i = 0; i < PH_COUNT; i++) CK(cudaEventCreate(&e->evs[k][i]));
    const size_t sb = (sizeof(Counters) + 63) & ~(size_t)63;
    void *hp = nullptr, *dp = nullptr;
    CK(cudaHostAlloc(&hp, sb + 64, cudaHostAllocMapped));
    memset(hp, 0, sb + 64);
    CK(cudaHostGetDevicePointer(&dp, hp, 0));
    e->h_snap[k] = (Counters *)hp;
    e->h_seq[k] = (unsigned long long *)((char *)hp + sb);
    e->d_snap[k] = (Counters *)dp;
    e->d_seq[k] = (unsigned long long *)((char *)dp + sb);
    TRY(dev_alloc(&e->d_snapbuf[k], 1, 0));
  }
  CK(cudaMallocHost((void **)&e->h_ctr, sizeof(Counters)));
  CK(cudaMallocHost((void **)&e->h_frame, sizeof(FrameDev)));
  memset(e->h_ctr, 0, sizeof(Counters));
  memset(e->h_frame, 0, sizeof(FrameDev));
  DevState &S = e->S;
  S.cube_size = cfg->cube_size;
  S.extent = cfg->cube_size * kB;
  S.inv_extent = 1.0 / S.extent;
  S.table_size = cfg->table_size;
  S.nbuckets = (int32_t)((cfg->table_size + kSlotsPerBucket - 1) / kSlotsPerBucket);
  S.bmask = (S.nbuckets & (S.nbuckets - 1)) == 0 ? (unsigned)S.nbuckets - 1 : 0u;
  S.max_blocks = (int32_t)((cfg->table_size + 1) / 2);
  S.max_vertices = cfg->max_vertices;
  S.rank = cfg->nranks > 1 ? cfg->rank : 0;
  S.nranks = cfg->nranks > 1 ? cfg->nranks : 1;
  {
    const int tb = cfg->tile_blocks > 0 ? cfg->tile_blocks : 8;
    if (tb & (tb - 1)) return set_err(VM_ERR_VALUE, "tile_blocks must be a power of two");
    if (S.rank < 0 || S.rank >= S.nranks) return set_err(VM_ERR_VALUE, "rank out of range");
    S.tile_shift = 0;
    while ((1 << S.tile_shift) < tb) S.tile_shift++;
  }
  const size_t mb = (size_t)S.max_blocks;
  TRY(dev_alloc(&S.slots, (size_t)S.nbuckets * kSlotsPerBucket, 0xFF));
  TRY(dev_alloc(&S.ovf_head, (size_t)S.nbuckets, 0xFF));
  TRY(dev_alloc(&S.ovf_lock, (size_t)S.nbuckets, 0));
  S.ovf_cap = (int32_t)mb + 1;
  TRY(dev_alloc(&S.ovf_key, (size_t)S.ovf_cap));
  TRY(dev_alloc(&S.ovf_val, (size_t)S.ovf_cap));
  TRY(dev_alloc(&S.ovf_next, (size_t)S.ovf_cap));
  TRY(dev_alloc(&S.ovf_stamp, (size_t)S.ovf_cap, 0xFF));
  TRY(dev_alloc(&S.bcoord, mb));
  TRY(dev_alloc(&S.nbr, mb * 27, 0xFF));
  TRY(dev_alloc(&S.stamp_collect, mb, 0xFF));
  TRY(dev_alloc(&S.stamp_halo, mb, 0xFF));
  TRY(dev_alloc(&S.stamp_new, mb, 0xFF));
  TRY(dev_alloc(&S.bowned, mb, 0));
  TRY(dev_alloc(&S.ghost_src, mb));
  TRY(dev_alloc(&S.last_frame, mb, 0));
  TRY(dev_alloc(&S.free_list, mb));
  TRY(dev_alloc(&e->d_ghost_counts, kMaxRanks, 0));
  S.ghost_counts = e->d_ghost_counts;
  S.halo_exchange = (cfg->nranks > 1 && cfg->halo_exchange) ? 1 : 0;
  TRY(dev_alloc(&S.slab_bits, (mb + 4) & ~(size_t)3, 0));
  TRY(dev_alloc(&S.scope, mb));
  TRY(dev_alloc(&S.halo, mb));
  S.halo_sh_cap = (int32_t)((mb + kHaloShards - 1) / kHaloShards + 64);
  if (const char *cap = getenv("VOXMESH_B200_HALO_SHARD_CAP")) {   // (test hook: force shard spills)
    const long v = strtol(cap, nullptr, 10);
    if (v > 0 && v < S.halo_sh_cap) S.halo_sh_cap = (int32_t)v;
  }
  TRY(dev_alloc(&S.halo_sh, (size_t)kHaloShards * S.halo_sh_cap));
  TRY(dev_alloc(&S.ctr, 1, 0));
  TRY(dev_alloc(&S.gc_done, 4, 0));
  S.fb_cap = 1 << 16;   // fallback records kept for the next frame (~0.6 k per C2 frame; more are applied inline)
  if (const char *cap = getenv("VOXMESH_B200_FALLBACK_CAP")) {   // (test hook: force inline fallbacks)
    const long v = strtol(cap, nullptr, 10);
    if (v >= 0 && v < S.fb_cap) S.fb_cap = (int32_t)v;
  }
  TRY(dev_alloc(&S.fallback, (size_t)std::max(S.fb_cap, 1)));
  uint8_t slab_sel[8];   // mesher.py:518-525
  for (int m = 0; m < 8; m++) {
    uint8_t bits = 0;
    for (int o = 1; o < 8; o++)
      if ((o & ~m) == 0) bits |= (uint8_t)(1u << (o - 1));
    slab_sel[m] = bits;
  }
  CK(cudaMemcpyToSymbol(c_slab_sel, slab_sel, sizeof slab_sel));
  {
    // persistent grids: exactly the number of co-resident CTAs
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_retype_place, kNT, kRetypeSmem));
    e->grid_retype = std::max(1, occ) * e->sm_count;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gc_normals, kGT, kGcSmem));
    if (const char *g = getenv("VOXMESH_B200_GC_CTAS_PER_SM")) occ = std::min(occ, atoi(g));   // (A/B knob)
    e->grid_gc = std::max(1, occ) * e->sm_count;
    S.rec_chunk_ctas = e->grid_gc;
    TRY(dev_alloc(&S.rec_chunk, 4 * (size_t)S.rec_chunk_ctas, 0));   // (two empty record ranges per CTA)
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fuse_blocks, kFB, 0));
    e->grid_fuse = std::max(1, occ) * e->sm_count;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_collect, kCollectThreads, 0));
    if (const char *g = getenv("VOXMESH_B200_COLLECT_CTAS_PER_SM")) occ = std::min(occ, atoi(g));   // (A/B knob)
    e->grid_collect = std::max(1, occ) * e->sm_count;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_place_parity, kNT, 0));
    e->grid_parity = std::max(1, occ) * e->sm_count;
  }
  // vertex records (grow on demand; a frame short of them resumes at k_retype_place)
  S.vrec_cap = cfg->initial_vertices > 0 ? cfg->initial_vertices : (int64_t)1 << 20;
  TRY(dev_alloc(&S.vrec, (size_t)S.vrec_cap));
  S.block_cap = 0;
  const int64_t ib = cfg->initial_blocks > 0 ? cfg->initial_blocks : 1024;
  TRY(grow_blocks(e, std::min<int64_t>(ib, S.max_blocks)));
  CK(cudaDeviceSynchronize());
  *out = e;
  return VM_OK;
}

static double now_us() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
}

int vm_destroy(vm_engine *e) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return VM_OK;
  if (e->host_prof && e->hp.size() > 8) {
    double med[3];
    for (int k = 0; k < 3; k++) {
      std::vector<double> v;
      for (size_t i = 5; i < e->hp.size(); i++) v.push_back(e->hp[i][k]);
      std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
      med[k] = v[v.size() / 2];
    }
    fprintf(stderr, "[host] %zu submits, medians: enqueue %.1f us, settle %.1f us, outside the call %.1f us\n",
            e->hp.size(), med[0], med[1], med[2]);
  }
  cudaStreamSynchronize(e->stream);
  DevState &S = e->S;
  void *ptrs[] = {S.slots, S.ovf_head, S.ovf_lock, S.ovf_key, S.ovf_val, S.ovf_next, S.ovf_stamp, S.bcoord,
                  S.nbr, S.stamp_collect, S.stamp_halo, S.stamp_new, S.bowned, S.slab_bits, S.scope,
                  S.halo, S.halo_sh, S.tsdf, S.weight, S.vmask, S.tp, S.tc, S.vh, S.vrb, S.rec_chunk, S.vocc, S.vclaim, S.vparam, S.vrec, S.item_mask, S.vreq, S.psel, S.fallback, e->d_rays,
                  S.ctr, S.gc_done, e->d_inseq, e->d_depth, e->d_scratch, S.ghost_src, e->d_ghost_counts, S.last_frame, S.free_list};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  free_compacted(e->comp);
  free_pcompact(e);
  if (e->h_ctr) cudaFreeHost(e->h_ctr);
  if (e->h_inseq) cudaFreeHost(e->h_inseq);
  if (e->h_frame) cudaFreeHost(e->h_frame);
  for (int k = 0; k < 2; k++) {
    for (int i = 0; i < PH_COUNT; i++)
      if (e->evs[k][i]) cudaEventDestroy(e->evs[k][i]);
    if (e->h_snap[k]) cudaFreeHost(e->h_snap[k]);
    if (e->d_snapbuf[k]) cudaFree(e->d_snapbuf[k]);
  }
  if (e->copy_stream) cudaStreamSynchronize(e->copy_stream);
  for (int i = 0; i < 2; i++) {
    if (e->d_slot[i]) cudaFree(e->d_slot[i]);
    if (e->d_raw[i]) cudaFree(e->d_raw[i]);
    if (e->ev_copy[i]) cudaEventDestroy(e->ev_copy[i]);
  }
  if (e->copy_stream) cudaStreamDestroy(e->copy_stream);
  if (e->own_stream && e->stream) cudaStreamDestroy(e->stream);
  delete e;
  return VM_OK;
}

int vm_set_stream(vm_engine *e, void *stream) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  TRY(settle_all(e));
  CK(cudaStreamSynchronize(e->stream));
  if (e->own_stream) CK(cudaStreamDestroy(e->stream));
  if (stream) {
    e->stream = (cudaStream_t)stream;
    e->own_stream = false;
  } else {
    CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
    e->own_stream = true;
  }
  return VM_OK;
}

int vm_get_stream(vm_engine *e, void **stream) {
  if (!e || !stream) return set_err(VM_ERR_INPUT, "null argument");
  *stream = (void *)e->stream;
  return VM_OK;
}

// After a frame's host copy on the copy stream: the flag its k_collect waits
// for (the copy of a per-slot sequence value, behind the depth in stream order)
static int post_input_flag(vm_engine *e, int sl) {
  if (!e->d_inseq) {
    CK(cudaMalloc((void **)&e->d_inseq, 2 * sizeof(unsigned long long)));
    CK(cudaMemset(e->d_inseq, 0, 2 * sizeof(unsigned long long)));
    CK(cudaMallocHost((void **)&e->h_inseq, 2 * sizeof(unsigned long long)));
    e->h_inseq[0] = e->h_inseq[1] = 0;
  }
  e->h_inseq[sl] = ++e->in_id;   // (its previous copy completed: vm_input_wait ran since)
  CK(cudaMemcpyAsync(e->d_inseq + sl, e->h_inseq + sl, sizeof(unsigned long long), cudaMemcpyHostToDevice,
                     e->copy_stream));
  e->in_slot = sl;
  return VM_OK;
}

// Returning from a submit: unless the caller defers it, wait until the host
// buffer has been read (every return path, errors included)
struct InputWait {
  vm_engine *e;
  ~InputWait() {
    if (!e->defer_wait) vm_input_wait(e);
  }
};

int vm_set_deferred_input_wait(vm_engine *e, int on) {
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  TRY(vm_input_wait(e));
  e->defer_wait = on != 0;
  return VM_OK;
}

int vm_input_wait(vm_engine *e) {
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  if (e->copy_pending >= 0) {
    const int sl = e->copy_pending;
    e->copy_pending = -1;
    CK(cudaEventSynchronize(e->ev_copy[sl]));
  }
  return VM_OK;
}

int vm_order_after(vm_engine *e, void *producer) {
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  cudaStream_t p = (cudaStream_t)producer;
  if (p == e->stream) return VM_OK;
  const cudaError_t q = cudaStreamQuery(p);
  if (q == cudaSuccess) return VM_OK;   // (its work is done: nothing to order)
  if (q != cudaErrorNotReady) return set_err(VM_ERR_CUDA, "producer stream: %s", cudaGetErrorString(q));
  if (!e->ev_order) CK(cudaEventCreateWithFlags(&e->ev_order, cudaEventDisableTiming));
  CK(cudaEventRecord(e->ev_order, p));
  e->ov_ready = false;   // (an event wait on the stream: the frames stay apart)
  CK(cudaStreamWaitEvent(e->stream, e->ev_order, 0));
  return VM_OK;
}

int vm_set_trace(vm_engine *e, void *device_buffer) {
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  e->S.trace = (unsigned long long *)device_buffer;
  return VM_OK;
}

int vm_set_profiling(vm_engine *e, int on) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  e->profiling = on != 0;
  return VM_OK;
}

// per-kernel device times of the last frame (profiling mode), ms:
// depth_stats, collect, fuse_blocks, retype_place, gc_normals
int vm_phase_times(vm_engine *e, double *ms, int n) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !ms) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle(e));
  CK(cudaEventSynchronize(e->ev[PH_END]));
  for (int i = 0; i < n && i < PH_END; i++) {
    float f = 0.f;
    const cudaError_t r = cudaEventElapsedTime(&f, e->ev[i], e->ev[i + 1]);
    ms[i] = (r == cudaSuccess) ? (double)f : -1.0;
  }
  cudaGetLastError();
  return VM_OK;
}

int vm_reserve(vm_engine *e, int64_t blocks, int64_t vertices, int64_t triangles) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  TRY(settle_all(e));
  (void)triangles;   // triangles are implicit (derived from the cube types)
  if (blocks > e->S.block_cap) TRY(grow_blocks(e, std::min<int64_t>(blocks, e->S.max_blocks)));
  if (vertices > 0) TRY(grow_records(e, vertices));
  return VM_OK;
}

static void fill_stats(vm_engine *e, int64_t frame, vm_stats *out) {
  const Counters &c = *e->h_ctr;
  memset(out, 0, sizeof *out);
  out->frame = frame;
  out->blocks_active = e->S.nranks > 1 ? c.nblocks_owned : c.nblocks - c.nfree;
  out->blocks_evicted = c.evicted_total;
  out->vertices_live = c.v_live;
  out->triangles_live = c.t_live;
  out->vertices_allocated_total = c.v_count;
  out->vertices_recycled_total = c.v_recycled;
  out->irregular_cube_count = c.irregular;
  out->valid_pixels = c.nvalid;
  out->nsteps = c.nsteps;
  out->collected_blocks = c.ncollected;
  out->new_blocks = c.nnew;
  out->scope_blocks = (int64_t)c.ncollected + c.nslab;
  out->halo_blocks = c.nhalo;
  for (int k = 0; k < kHaloShards; k++) out->halo_blocks += std::min(c.nhalo_sh[k], e->S.halo_sh_cap);
  out->active_cubes = c.active;
  out->edge_placements = c.placements;
  out->new_vertices = c.v_allocs;
  out->changed_cubes = c.changed;
  out->triangles_freed = c.t_released;
  out->triangles_allocated = c.t_allocated;
  out->vertices_freed = c.v_frees;
  out->normals_computed = c.normals;
  out->fallback_normals = c.fallbacks;
  out->refined_cubes = c.refined;
  out->resumes = e->last_resumes;
  out->kernel_launches = e->frame_launches;
  float ms = 0.f;
  if (e->ev_rec[e->ev == e->evs[1]]) {
    cudaEventSynchronize(e->ev[PH_END]);
    if (cudaEventElapsedTime(&ms, e->ev[PH_DEPTH], e->ev[PH_END]) == cudaSuccess) out->device_ms = ms;
  } else if (c.t_end_ns > c.t_start_ns && c.t_start_ns) {   // submitted frame: the kernels' own clock
    out->device_ms = (double)(c.t_end_ns - c.t_start_ns) * 1e-6;
  }
  if (e->profiling) {   // segment split needs the per-kernel events
    if (cudaEventElapsedTime(&ms, e->ev[PH_DEPTH], e->ev[PH_RETYPE]) == cudaSuccess) out->fusion_ms = ms;
    if (cudaEventElapsedTime(&ms, e->ev[PH_RETYPE], e->ev[PH_END]) == cudaSuccess) out->meshing_ms = ms;
  } else if (c.t_mesh_ns > c.t_start_ns && c.t_end_ns >= c.t_mesh_ns && c.t_start_ns) {
    // the kernels' own clock: collect + integrate | retype + placement + GC + normals
    // (the reference's fusion_ms / meshing_ms segments, engine.py:127-156)
    out->fusion_ms = (double)(c.t_mesh_ns - c.t_start_ns) * 1e-6;
    out->meshing_ms = (double)(c.t_end_ns - c.t_mesh_ns) * 1e-6;
  } else {
    out->fusion_ms = out->device_ms;
    out->meshing_ms = 0.0;
  }
  cudaGetLastError();
}

// band step count for a max ray norm, exactly as k_collect computes it (fusion.py:90-94)
static int nsteps_for(double maxnorm, double trunc, double extent) {
  const double band = (2.0 * trunc) * maxnorm;
  int n = (int)std::ceil(band / (extent * 0.5)) + 1;
  return n < 2 ? 2 : n;
}

// Per-intrinsics state, recomputed when (h, w, fx, fy, cx, cy) change: the ray
// tables the pixel passes read, and the min / max ray norm over the image.
static int ensure_rays(vm_engine *e, int32_t h, int32_t w) {
  FrameDev &F = *e->h_frame;
  const double key[6] = {(double)h, (double)w, F.fx, F.fy, F.cx, F.cy};
  if (e->norm_valid && memcmp(key, e->norm_key, sizeof key) == 0) {
    e->S.rays = e->d_rays;
    return VM_OK;
  }
  const size_t need = (size_t)(h + w) * sizeof(double);
  if (need > e->rays_cap) {
    if (e->d_rays) CK(cudaFree(e->d_rays));
    CK(cudaMalloc((void **)&e->d_rays, need));
    e->rays_cap = need;
  }
  unsigned long long *d;
  TRY(scratch(e, 2 * sizeof(unsigned long long), (void **)&d));
  const unsigned long long init[2] = {~0ull, 0ull};
  unsigned long long res[2];
  CK(cudaMemcpyAsync(d, init, sizeof init, cudaMemcpyHostToDevice, e->stream));
  k_norm_bounds<<<grid_threads(e, (long long)h * w, 256), 256, 0, e->stream>>>(F, d, e->d_rays);
  CK(cudaMemcpyAsync(res, d, sizeof res, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  memcpy(&e->norm_lo, &res[0], sizeof(double));
  memcpy(&e->norm_hi, &res[1], sizeof(double));
  memcpy(e->norm_key, key, sizeof key);
  e->norm_valid = true;
  e->S.rays = e->d_rays;
  return VM_OK;
}

// The step count is a monotone function of the max norm over the valid pixels,
// which lies within [min, max] of the norm over the whole image: when both
// bounds give the same count, the frame's count is known without reading the
// depth and k_depth_stats is skipped.  Returns 0 when it is data dependent.
static int fixed_nsteps(vm_engine *e, double trunc) {
  const int lo = nsteps_for(e->norm_lo, trunc, e->S.extent), hi = nsteps_for(e->norm_hi, trunc, e->S.extent);
  return lo == hi ? lo : 0;
}

// Queue the kernels of the frame whose parameters are in slot `slot`; the
// counters are snapshotted into the slot's pinned buffer after its last kernel.
static int launch_frame(vm_engine *e, int slot) {
  NvtxRange nvtx_("vm_launch_frame");
  FrameDev &F = *e->h_frame;
  F = e->f_saved[slot];
  F.snap = e->d_snapbuf[slot];
  F.reset_after = 1;
  e->want_id[slot] = ++e->snap_ids;
  // Host-copied input: the next frame's k_collect starts only after its copy,
  // so this frame's gc commit publishes itself (a few PCIe writes at its end).
  // So does a submitted frame the next one may overlap: the gc's completion
  // is then off the critical path, while a publishing k_collect's is not
  // (its system-scope writes drain before the next kernel starts: ~1.3 us,
  // trace v11).  Else the next frame's k_collect publishes it.
  e->self_pub[slot] = e->host_input || (e->in_submit && e->own_stream && !e->profiling && !e->no_overlap);
  if (e->self_pub[slot]) {
    F.self_dst = e->d_snap[slot];
    F.self_seq = e->d_seq[slot];
    F.self_id = e->want_id[slot];
  }
  if (e->publish_prev && !e->self_pub[slot ^ 1]) {   // the pending frame's snapshot, from this k_collect
    F.pub_src = e->d_snapbuf[slot ^ 1];
    F.pub_dst = e->d_snap[slot ^ 1];
    F.pub_seq = e->d_seq[slot ^ 1];
    F.pub_id = e->want_id[slot ^ 1];
  }
  e->fslot = slot;
  e->ev = e->evs[slot];
  e->ev_rec[slot] = e->profiling;
  // Frame overlap: this frame's k_collect may run under the previous frame's
  // k_gc_normals when that kernel is the stream's last operation and nothing
  // else runs first (no counter reset, block GC or depth-stats pass, no
  // per-kernel events); a vertex-pool limit makes the gc commit raise, so it
  // keeps the frames apart too
  const bool gc_frame = F.block_gc_age > 0 && F.frame > 0 && F.frame % F.block_gc_age == 0;
  // (and only on the engine's own stream: a caller's kernel queued on a shared
  // stream between the frames could write what this k_collect reads, and it
  // skips the grid-dependency wait)
  const bool overlap = e->ov_ready && e->own_stream && e->ctr_clean && !e->profiling && !gc_frame &&
                       e->S.max_vertices <= 0 && !e->no_overlap;
  const int32_t wait_epoch = overlap ? e->ov_epoch : 0;
  e->ov_ready = false;
  if (!e->ctr_clean) TRY(reset_call_counters(e));
  cudaStream_t st = e->stream;
  rec(e, PH_DEPTH);
  e->frame_launches = 3 + meshing_launches(F);   // collect, fuse, retype (+ parity passes), gc (+ depth stats)
  if (gc_frame) {
    // opt-in block GC, before the frame allocates (its pops reuse the indices)
    e->S.free_list_on = 1;   // (allocations check the free list from now on)
    k_block_gc<<<e->sm_count * 8, 256, 0, st>>>(e->S, F.frame, F.block_gc_age);
    e->frame_launches++;
  }
  FrameDev Fc = F;   // (collect's copy: a raw frame converted by k_depth_stats is f64 now)
  Fc.overlap = overlap ? 1 : 0;
  e->ov_of[slot] = overlap;
  Fc.wait_epoch = wait_epoch;
  if (F.nsteps_fixed <= 0) {
    // the band step count needs the frame's max ray norm first: under overlap
    // this pass also starts under the previous gc (PDL, no grid-dependency
    // wait; it waits for the host copy's flag itself) and the collect waits
    // for its CTAs on a counter
    FrameDev Fd = F;
    Fd.overlap = overlap ? 1 : 0;
    if (overlap) launch_pdl(k_depth_stats, grid_blocks(e), 256, st, e->S, Fd);
    else k_depth_stats<<<grid_blocks(e), 256, 0, st>>>(e->S, Fd);
    e->frame_launches++;
    Fc.raw = nullptr;
    Fc.in_flag = nullptr;   // (k_depth_stats waited for the copy)
    Fc.ds_wait = overlap ? grid_blocks(e) : 0;
  }
  rec(e, PH_COLLECT);
  launch_pdl(k_collect, e->grid_collect, kCollectThreads, st, e->S, Fc);
  F.raw = nullptr;   // (the later kernels read the f64 depth)
  TRY(enqueue_after_collect(e));
  // the frame's gc commit publishes its counters and clears the per-call ones:
  // the next frame's kernels follow with no stream operation in between
  F.snap = nullptr;
  F.reset_after = 0;
  F.pub_src = nullptr;
  F.pub_dst = nullptr;
  F.pub_seq = nullptr;
  F.self_dst = nullptr;
  F.self_seq = nullptr;
  e->ctr_clean = true;
  e->pending = 1;
  e->pending_frame = e->frame_of[slot];
  e->ov_ready = !e->profiling;   // (the stream ends with this frame's k_gc_normals)
  e->ov_epoch = F.epoch;
  return VM_OK;
}

int vm_fuse_frame_enqueue(vm_engine *e, const double *depth, int32_t h, int32_t w, int32_t depth_on_device,
                          const vm_intrinsics *intr, const vm_pose *pose, const vm_frame_config *cfg,
                          int64_t frame_index) {
  if (!e || !intr || !pose || !cfg) return set_err(VM_ERR_INPUT, "null argument");
  if (e->pending) return set_err(VM_ERR_INPUT, "previous frame not finished");
  if (cfg->strategy < 0 || cfg->strategy > 2) return set_err(VM_ERR_VALUE, "unknown strategy %d", cfg->strategy);
  if (cfg->trunc < e->S.cube_size) return set_err(VM_ERR_VALUE, "truncation band must be at least one cube");
  const double *dd;
  if (!depth_on_device) e->ov_ready = false;   // (a host copy goes first)
  TRY(stage_depth(e, depth, h, w, depth_on_device, &dd));
  fill_frame_host(e, dd, h, w, intr, pose);
  FrameDev &F = *e->h_frame;
  F.trunc = cfg->trunc;
  F.max_range = cfg->max_range;
  F.epsilon = cfg->epsilon;
  F.weight_cap = cfg->weight_cap;
  F.refine = cfg->refine;
  F.frustum_only = cfg->frustum_only;
  F.epoch = ++e->epoch;
  F.frame = (int32_t)frame_index;
  F.scope_mode = 0;
  F.strategy = cfg->strategy;
  TRY(ensure_partition_bufs(e, cfg->strategy));
  if (!e->norm_valid) e->ov_ready = false;   // (ensure_rays launches its own kernel)
  TRY(ensure_rays(e, h, w));
  F.nsteps_fixed = fixed_nsteps(e, cfg->trunc);
  F.band_step = F.nsteps_fixed > 1 ? 2.0 / (double)(F.nsteps_fixed - 1) : 0.0;
  F.block_gc_age = cfg->block_gc_age > 0 ? cfg->block_gc_age : 0;
  F.consume_fb = 1;   // k_collect applies the previous frame's fallback records
  if (e->raw_next) {   // raw u16 frame: the first pixel kernel fills the f64 depth from it
    F.raw = e->raw_next;
    F.depth_out = const_cast<double *>(dd);
    F.depth_scale = e->raw_scale;
  }
  F.in_flag = nullptr;
  F.in_id = 0;
  if (e->in_slot >= 0) {   // (a submitted host copy: k_collect waits for its flag)
    F.in_flag = e->d_inseq + e->in_slot;
    F.in_id = e->h_inseq[e->in_slot];
    e->in_slot = -1;
  }
  const int slot = e->fslot ^ 1;
  e->f_saved[slot] = F;
  e->frame_of[slot] = frame_index;
  return launch_frame(e, slot);
}

int vm_fuse_frame_finish(vm_engine *e, vm_stats *out) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  if (!e->pending) return set_err(VM_ERR_INPUT, "no frame pending");
  e->pending = 0;
  TRY(settle_slot(e, e->fslot, false));
  if (out) *out = e->settled;
  return VM_OK;
}

int vm_fuse_frame(vm_engine *e, const double *depth, int32_t h, int32_t w, int32_t depth_on_device,
                  const vm_intrinsics *intr, const vm_pose *pose, const vm_frame_config *cfg,
                  int64_t frame_index, vm_stats *out) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  TRY(vm_fuse_frame_enqueue(e, depth, h, w, depth_on_device, intr, pose, cfg, frame_index));
  return vm_fuse_frame_finish(e, out);
}

// Complete a pending submitted frame (host wait, arena resume) and keep its
// stats for vm_fuse_frame_result.  Every call that touches the engine's state
// settles first, so a submitted frame is never observed half done.
//
// settle_slot completes the frame of slot `slot`; when `succ` the frame after it
// is already queued behind it (vm_fuse_frame_submit).  The common case is one
// event wait on the frame's counter snapshot -- the queued frame keeps the GPU
// busy meanwhile.  A frame that ran out of block heap (or failed) made every
// later kernel exit at its guard, the queued frame's included (k_collect checks
// it before any write), so its only effect was resetting the per-call
// counters: the device counters are restored from the snapshot, the frame is
// resumed as in the synchronous path, and the queued frame is launched again
// (or, when the frame failed, dropped: the engine is left as the synchronous
// path leaves it).
// The frame's counters: published by the queued successor's k_collect (wait
// on the sequence word; the GPU stays busy), else read after the stream drains.
static int wait_snapshot(vm_engine *e, int slot, bool succ) {
  volatile unsigned long long *seq = e->h_seq[slot];
  const unsigned long long want = e->want_id[slot];
  for (unsigned spins = 1; succ && *seq != want; spins++) {
    if ((spins & 1023u) == 0) {   // (a failed launch publishes nothing: watch the stream)
      const cudaError_t q = cudaStreamQuery(e->stream);
      if (q != cudaSuccess && q != cudaErrorNotReady)
        return set_err(VM_ERR_CUDA, "frame failed: %s", cudaGetErrorString(q));
      if (q == cudaSuccess && *seq != want) succ = false;
    }
  }
  if (succ) {
    std::atomic_thread_fence(std::memory_order_acquire);
    memcpy(e->h_ctr, e->h_snap[slot], sizeof(Counters));
  } else {
    TRY(copy_sync(e, e->h_ctr, e->d_snapbuf[slot], sizeof(Counters), cudaMemcpyDeviceToHost));
  }
  return VM_OK;
}

static int settle_slot(vm_engine *e, int slot, bool succ) {
  NvtxRange nvtx_("vm_settle_frame");
  TRY(wait_snapshot(e, slot, succ));
  const int launched = e->frame_launches;
  e->ev = e->evs[slot];
  e->last_resumes = 0;
  e->resume_launches = 0;
  int rc = VM_OK;
  e->restore_calls = true;   // (unhalted: the commit cleared the per-call counters)
  if (e->h_ctr->need || e->h_ctr->error) {
    e->ov_ready = false;     // (the resume queues stream operations)
    e->ctr_clean = false;    // (halted: not cleared)
    e->restore_calls = false;
    if (succ) {
      CK(cudaStreamSynchronize(e->stream));
      TRY(copy_sync(e, e->S.ctr, e->h_ctr, sizeof(Counters), cudaMemcpyHostToDevice));
      *e->h_frame = e->f_saved[slot];
      e->h_frame->raw = nullptr;
    }
    rc = complete_with_resume(e, &e->last_resumes);
  }
  if (rc == VM_OK) {
    fill_stats(e, e->frame_of[slot], &e->settled);
    e->settled.overlapped = e->ov_of[slot] && !e->last_resumes;
  }
  if (succ) {
    e->pending = 0;
    if (rc == VM_OK && e->last_resumes) {
      TRY(launch_frame(e, slot ^ 1));   // (sets pending again)
    } else if (rc == VM_OK) {
      e->pending = 1;
      e->pending_frame = e->frame_of[slot ^ 1];
      e->ev = e->evs[slot ^ 1];
      e->frame_launches = launched;
    }
    if (rc == VM_OK) {
      const FrameDev &Fs = e->f_saved[slot];
      e->settled.kernel_launches = 3 + meshing_launches(Fs) + (Fs.nsteps_fixed <= 0) +
                                   e->resume_launches +
                                   (Fs.block_gc_age > 0 && Fs.frame > 0 && Fs.frame % Fs.block_gc_age == 0);
    }
  }
  return rc;
}

static int settle(vm_engine *e) {
  if (!e->pending) return VM_OK;
  e->pending = 0;
  TRY(settle_slot(e, e->fslot, false));
  e->settled_valid = 1;
  return VM_OK;
}

// Apply pending face-normal fallback records (kept between frames for the next
// k_collect): every entry point outside the frame pipeline calls this first,
// and the ones that run k_gc_normals themselves call it again at their end.
static int flush_fallbacks(vm_engine *e) {
  k_flush_fallbacks<<<e->sm_count * 4, 128, 0, e->stream>>>(e->S);
  CK(cudaMemsetAsync(&e->S.ctr->fb_pending, 0, sizeof(int32_t), e->stream));
  return check_launch();
}

static int settle_all(vm_engine *e) {
  TRY(settle(e));
  if (e->restore_calls) {   // the last frame's per-call counters, as a synchronous frame leaves them
    const size_t off = offsetof(Counters, nvalid);
    TRY(copy_sync(e, (char *)e->S.ctr + off, (const char *)e->h_ctr + off, sizeof(Counters) - off,
                  cudaMemcpyHostToDevice));
    e->restore_calls = false;
  }
  e->ctr_clean = false;
  return flush_fallbacks(e);
}

int vm_fuse_frame_submit(vm_engine *e, const double *depth, int32_t h, int32_t w, int32_t depth_on_device,
                         const vm_intrinsics *intr, const vm_pose *pose, const vm_frame_config *cfg,
                         int64_t frame_index) {
  if (!e || !intr || !pose || !cfg) return set_err(VM_ERR_INPUT, "null argument");
  if (!depth || h <= 0 || w <= 0) return set_err(VM_ERR_INPUT, "depth must be a non-empty (H, W) array");
  if (e->settled_valid && e->pending)   // (at most one undelivered result)
    return set_err(VM_ERR_INPUT, "the previous frame's result was not taken");
  const double *dd = depth;
  int sl = -1;
  if (!depth_on_device) {
    // 1. this frame's depth goes up on the copy stream, into the slot the
    //    pending frame does not read (the frame before it has settled)
    const size_t bytes = (size_t)h * w * sizeof(double);
    if (!e->copy_stream) {
      CK(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
      for (int i = 0; i < 2; i++) CK(cudaEventCreateWithFlags(&e->ev_copy[i], cudaEventDisableTiming));
    }
    if (bytes > e->slot_cap) {
      e->ov_ready = false;
      TRY(settle(e));   // (rare) reallocation: nothing may be reading the slots
      CK(cudaStreamSynchronize(e->copy_stream));
      for (int i = 0; i < 2; i++) {
        if (e->d_slot[i]) CK(cudaFree(e->d_slot[i]));
        CK(cudaMalloc((void **)&e->d_slot[i], bytes));
      }
      e->slot_cap = bytes;
    }
    sl = e->slot ^ 1;
    CK(cudaMemcpyAsync(e->d_slot[sl], depth, bytes, cudaMemcpyHostToDevice, e->copy_stream));
    CK(cudaEventRecord(e->ev_copy[sl], e->copy_stream));
    e->copy_pending = sl;   // (waited for on every return below, or by the caller in deferred mode)
    TRY(post_input_flag(e, sl));
    dd = e->d_slot[sl];
  }
  InputWait iw_{e};
  // 2. this frame's kernels, ordered after its copy by the device-side flag
  //    (k_collect waits for it), queued behind the pending frame's; 3. the
  //    pending frame completes (its stats are kept for vm_fuse_frame_result)
  //    while this one keeps the GPU busy
  const bool prev = e->pending != 0;
  const int pslot = e->fslot;
  e->pending = 0;
  e->publish_prev = prev;
  e->host_input = sl >= 0;
  e->in_submit = true;
  const double hp0 = e->host_prof ? now_us() : 0.0;
  const int rc = vm_fuse_frame_enqueue(e, dd, h, w, 1, intr, pose, cfg, frame_index);
  const double hp1 = e->host_prof ? now_us() : 0.0;
  e->publish_prev = false;
  e->host_input = false;
  e->in_submit = false;
  if (rc != VM_OK) {   // (argument errors: nothing was queued)
    e->pending = prev;
    e->fslot = pslot;
    return rc;
  }
  if (prev) {
    TRY(settle_slot(e, pslot, true));
    e->settled_valid = 1;
  }
  if (sl >= 0) e->slot = sl;   // (the caller may reuse its buffer once the copy is done: iw_)
  if (e->host_prof) {
    const double hp2 = now_us();
    e->hp.push_back({hp1 - hp0, hp2 - hp1, e->hp_last > 0 ? hp0 - e->hp_last : 0.0});
    e->hp_last = hp2;
  }
  return VM_OK;
}

int vm_fuse_frame_submit_raw(vm_engine *e, const uint16_t *raw, int32_t h, int32_t w, int32_t raw_on_device,
                             double depth_scale, const vm_intrinsics *intr, const vm_pose *pose,
                             const vm_frame_config *cfg, int64_t frame_index) {
  if (!e || !intr || !pose || !cfg) return set_err(VM_ERR_INPUT, "null argument");
  if (!raw || h <= 0 || w <= 0) return set_err(VM_ERR_INPUT, "depth must be a non-empty (H, W) array");
  if (!(depth_scale > 0)) return set_err(VM_ERR_VALUE, "depth_scale must be positive");
  if (e->settled_valid && e->pending) return set_err(VM_ERR_INPUT, "the previous frame's result was not taken");
  const size_t npix = (size_t)h * w;
  if (!e->copy_stream) {
    CK(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; i++) CK(cudaEventCreateWithFlags(&e->ev_copy[i], cudaEventDisableTiming));
  }
  if (npix * sizeof(double) > e->slot_cap || npix * sizeof(uint16_t) > e->raw_cap) {
    e->ov_ready = false;
    TRY(settle(e));   // (rare) reallocation: nothing may be reading the slots
    CK(cudaStreamSynchronize(e->copy_stream));
    for (int i = 0; i < 2; i++) {
      if (e->d_slot[i]) CK(cudaFree(e->d_slot[i]));
      if (e->d_raw[i]) CK(cudaFree(e->d_raw[i]));
      CK(cudaMalloc((void **)&e->d_slot[i], npix * sizeof(double)));
      CK(cudaMalloc((void **)&e->d_raw[i], npix * sizeof(uint16_t)));
    }
    e->slot_cap = npix * sizeof(double);
    e->raw_cap = npix * sizeof(uint16_t);
  }
  const int sl = e->slot ^ 1;
  const uint16_t *dr = raw;
  if (!raw_on_device) {   // a quarter of the f64 frame's bytes over PCIe
    CK(cudaMemcpyAsync(e->d_raw[sl], raw, npix * sizeof(uint16_t), cudaMemcpyHostToDevice, e->copy_stream));
    CK(cudaEventRecord(e->ev_copy[sl], e->copy_stream));
    e->copy_pending = sl;
    TRY(post_input_flag(e, sl));
    dr = e->d_raw[sl];
  }
  InputWait iw_{e};
  e->raw_next = dr;
  e->raw_scale = depth_scale;
  const bool prev = e->pending != 0;
  const int pslot = e->fslot;
  e->pending = 0;
  e->publish_prev = prev;
  e->host_input = false;   // (a quarter of the bytes: the copy is done before the kernels are)
  e->in_submit = true;
  const int rc = vm_fuse_frame_enqueue(e, e->d_slot[sl], h, w, 1, intr, pose, cfg, frame_index);
  e->publish_prev = false;
  e->host_input = false;
  e->in_submit = false;
  e->raw_next = nullptr;
  if (rc != VM_OK) {
    e->pending = prev;
    e->fslot = pslot;
    return rc;
  }
  if (prev) {
    TRY(settle_slot(e, pslot, true));
    e->settled_valid = 1;
  }
  e->slot = sl;   // (the caller may reuse its buffer once the copy is done: iw_)
  return VM_OK;
}

int vm_fuse_frame_result(vm_engine *e, vm_stats *out) {
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  if (!e->settled_valid) {
    if (!e->pending) return set_err(VM_ERR_INPUT, "no frame submitted");
    e->ov_ready = false;   // (settling queues stream operations)
    TRY(settle(e));
  }
  if (out) *out = e->settled;
  e->settled_valid = 0;
  return VM_OK;
}

// ---- phase API ------------------------------------------------------------
int vm_collect(vm_engine *e, const double *depth, int32_t h, int32_t w, int32_t depth_on_device,
               const vm_intrinsics *intr, const vm_pose *pose, double trunc, double max_range,
               int64_t *n_out) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !intr || !pose) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  const double *dd;
  TRY(stage_depth(e, depth, h, w, depth_on_device, &dd));
  fill_frame_host(e, dd, h, w, intr, pose);
  FrameDev &F = *e->h_frame;
  F.trunc = trunc;
  F.max_range = max_range;
  F.epoch = ++e->epoch;
  F.scope_mode = 0;
  F.nsteps_fixed = 0;   // the phase API always runs the depth reduction
  TRY(ensure_rays(e, h, w));
  TRY(reset_call_counters(e));
  k_depth_stats<<<grid_blocks(e), 256, 0, e->stream>>>(e->S, *e->h_frame);
  k_collect<<<e->grid_collect, kCollectThreads, 0, e->stream>>>(e->S, *e->h_frame);
  TRY(check_launch());
  TRY(init_new_blocks(e));
  if (n_out) *n_out = e->h_ctr->ncollected;
  return VM_OK;
}

int vm_get_collected(vm_engine *e, int32_t *coords_out, int64_t n) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || (!coords_out && n)) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  if (n == 0) return VM_OK;
  std::vector<int32_t> idx(n);
  CK(cudaMemcpyAsync(idx.data(), e->S.scope, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToHost, e->stream));
  TRY(read_counters(e));
  std::vector<int4> bc(e->h_ctr->nblocks);
  if (!bc.empty()) TRY(copy_sync(e, bc.data(), e->S.bcoord, sizeof(int4) * bc.size(), cudaMemcpyDeviceToHost));
  for (int64_t i = 0; i < n; i++) {
    const int4 c = bc[idx[i]];
    coords_out[3 * i] = c.x;
    coords_out[3 * i + 1] = c.y;
    coords_out[3 * i + 2] = c.z;
  }
  return VM_OK;
}

int vm_integrate(vm_engine *e, const int32_t *coords, int64_t n, const double *depth, int32_t h, int32_t w,
                 int32_t depth_on_device, const vm_intrinsics *intr, const vm_pose *pose, double trunc,
                 double max_range, int64_t weight_cap) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !intr || !pose) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  const double *dd;
  TRY(stage_depth(e, depth, h, w, depth_on_device, &dd));
  fill_frame_host(e, dd, h, w, intr, pose);
  FrameDev &F = *e->h_frame;
  F.trunc = trunc;
  F.max_range = max_range;
  F.weight_cap = weight_cap;
  if (coords) {
    // fusion.py:136-168 integrates list entries in order: a repeated block is
    // integrated again, so duplicates go to separate launches
    int64_t start = 0;
    while (start < n) {
      int64_t end = start;
      std::vector<std::array<int32_t, 3>> seen;
      while (end < n && seen.size() < 4096) {
        const std::array<int32_t, 3> c = {coords[3 * end], coords[3 * end + 1], coords[3 * end + 2]};
        if (std::find(seen.begin(), seen.end(), c) != seen.end()) break;
        seen.push_back(c);
        end++;
      }
      int32_t *di;
      TRY(map_coords(e, coords + 3 * start, end - start, &di, nullptr, 0, false));
      k_fuse_blocks<<<grid_blocks(e), kFB, 0, e->stream>>>(e->S, *e->h_frame, di, nullptr,
                                                                    (int)(end - start), F_INTEGRATE);
      TRY(check_launch());
      CK(cudaStreamSynchronize(e->stream));
      start = end;
    }
  } else {
    k_fuse_blocks<<<grid_blocks(e), kFB, 0, e->stream>>>(e->S, *e->h_frame, e->S.scope,
                                                                  &e->S.ctr->ncollected, 0, F_INTEGRATE);
    TRY(check_launch());
  }
  CK(cudaStreamSynchronize(e->stream));
  return VM_OK;
}

int vm_scope_halo(vm_engine *e, int64_t *n_scope, int32_t *scope_coords, uint8_t *scope_masks,
                  int64_t *n_halo, int32_t *halo_coords) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !n_scope || !n_halo) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  CK(cudaMemsetAsync(&e->S.ctr->nslab, 0, sizeof(int32_t), e->stream));
  CK(cudaMemsetAsync(&e->S.ctr->nhalo, 0, sizeof(int32_t), e->stream));
  k_fuse_blocks<<<grid_blocks(e), kFB, 0, e->stream>>>(e->S, *e->h_frame, e->S.scope,
                                                                &e->S.ctr->ncollected, 0, F_SCOPE | F_HALO);
  TRY(check_launch());
  TRY(read_counters(e));
  const int nc = e->h_ctr->ncollected, ns = e->h_ctr->nslab, nh = e->h_ctr->nhalo;
  *n_scope = nc + ns;
  *n_halo = nh;
  std::vector<int32_t> sidx(nc + ns), hidx(nh);
  if (nc + ns) TRY(copy_sync(e, sidx.data(), e->S.scope, sizeof(int32_t) * (nc + ns), cudaMemcpyDeviceToHost));
  if (nh) TRY(copy_sync(e, hidx.data(), e->S.halo, sizeof(int32_t) * nh, cudaMemcpyDeviceToHost));
  std::vector<int4> bc(e->h_ctr->nblocks);
  if (!bc.empty()) TRY(copy_sync(e, bc.data(), e->S.bcoord, sizeof(int4) * bc.size(), cudaMemcpyDeviceToHost));
  std::vector<uint8_t> bits(ns);
  if (ns) {
    std::vector<uint8_t> all(bc.size());
    TRY(copy_sync(e, all.data(), e->S.slab_bits, all.size(), cudaMemcpyDeviceToHost));
    for (int i = 0; i < ns; i++) bits[i] = all[sidx[nc + i]];
    k_clear_slabs<<<grid_threads(e, ns, 128), 128, 0, e->stream>>>(e->S, nc, ns);
    TRY(check_launch());
    CK(cudaStreamSynchronize(e->stream));
  }
  uint8_t slab_sel[8];
  for (int m = 0; m < 8; m++) {
    uint8_t b = 0;
    for (int o = 1; o < 8; o++)
      if ((o & ~m) == 0) b |= (uint8_t)(1u << (o - 1));
    slab_sel[m] = b;
  }
  if (scope_coords)
    for (int i = 0; i < nc + ns; i++) {
      const int4 c = bc[sidx[i]];
      scope_coords[3 * i] = c.x;
      scope_coords[3 * i + 1] = c.y;
      scope_coords[3 * i + 2] = c.z;
      if (scope_masks) {
        uint8_t *m = scope_masks + (size_t)i * 64;
        memset(m, 0, 64);
        for (int ci = 0; ci < kNC; ci++) {
          bool sel = true;
          if (i >= nc) {
            const int x = ci >> 6, y = (ci >> 3) & 7, z = ci & 7;
            sel = (bits[i - nc] & slab_sel[((x == 7) << 2) | ((y == 7) << 1) | (z == 7)]) != 0;
          }
          if (sel) m[ci >> 3] |= (uint8_t)(1u << (ci & 7));
        }
      }
    }
  if (halo_coords)
    for (int i = 0; i < nh; i++) {
      const int4 c = bc[hidx[i]];
      halo_coords[3 * i] = c.x;
      halo_coords[3 * i + 1] = c.y;
      halo_coords[3 * i + 2] = c.z;
    }
  return VM_OK;
}

int vm_extract(vm_engine *e, const int32_t *scope_coords, const uint8_t *scope_masks, int64_t n_scope,
               const int32_t *halo_coords, int64_t n_halo, int64_t frame_index, int32_t strategy,
               int32_t refine, double epsilon, int64_t *out2) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  TRY(settle_all(e));
  if (strategy < 0 || strategy > 2) return set_err(VM_ERR_VALUE, "unknown strategy %d", strategy);
  if (out2) { out2[0] = 0; out2[1] = 0; }
  if (n_scope <= 0) return VM_OK;   // mesher.py:564-565
  if (n_scope > e->S.block_cap) TRY(grow_blocks(e, std::min<int64_t>(n_scope, e->S.max_blocks)));
  if (n_scope > e->S.block_cap) return set_err(VM_ERR_INPUT, "scope larger than the block table");
  FrameDev &F = *e->h_frame;
  F.refine = refine;
  F.epsilon = epsilon;
  F.frustum_only = 0;
  F.epoch = ++e->epoch;
  F.frame = (int32_t)frame_index;
  F.scope_mode = 1;
  F.strategy = strategy;
  TRY(ensure_partition_bufs(e, strategy));
  TRY(reset_call_counters(e));
  int32_t *di;
  TRY(map_coords(e, scope_coords, n_scope, &di, nullptr, 0, false));
  CK(cudaMemcpyAsync(e->S.scope, di, sizeof(int32_t) * n_scope, cudaMemcpyDeviceToDevice, e->stream));
  if (scope_masks)
    CK(cudaMemcpyAsync(e->S.item_mask, scope_masks, (size_t)n_scope * 64, cudaMemcpyHostToDevice, e->stream));
  else
    CK(cudaMemsetAsync(e->S.item_mask, 0xFF, (size_t)n_scope * 64, e->stream));
  const int32_t ni = (int32_t)n_scope;
  CK(cudaMemcpyAsync(&e->S.ctr->nexplicit, &ni, sizeof ni, cudaMemcpyHostToDevice, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  if (n_halo >= 0) {
    TRY(map_coords(e, halo_coords, n_halo, &di, e->S.stamp_halo, F.epoch, false));
    CK(cudaMemcpyAsync(e->S.halo, di, sizeof(int32_t) * n_halo, cudaMemcpyDeviceToDevice, e->stream));
    const int32_t nh = (int32_t)n_halo;
    CK(cudaMemcpyAsync(&e->S.ctr->nhalo, &nh, sizeof nh, cudaMemcpyHostToDevice, e->stream));
    CK(cudaStreamSynchronize(e->stream));
  } else {
    k_halo_from_items<<<grid_threads(e, n_scope * 27, 256), 256, 0, e->stream>>>(e->S, *e->h_frame);
    TRY(check_launch());
  }
  launch_retype(e, false, *e->h_frame);
  TRY(read_counters(e));
  for (int guard = 0; e->h_ctr->need && e->h_ctr->need_stage == 1 && guard < 8; guard++) {
    TRY(grow_records(e, record_bound(e)));   // (the retype stopped before any write)
    TRY(clear_need(e));
    launch_retype(e, false, *e->h_frame);
    TRY(read_counters(e));
  }
  // the halo given here need not hold every block a request went to: apply them all
  k_apply_claims<<<grid_threads(e, (long long)e->h_ctr->nblocks * (kEV / 32), 256), 256, 0, e->stream>>>(
      e->S, e->h_ctr->nblocks, e->h_frame->frame, (int)(e->h_frame->strategy == VM_STRATEGY_PARTITION));
  launch_gc(e, false, e->S.halo, &e->S.ctr->nhalo, 0, (int)(G_GC | G_NORMALS | G_COMMIT | G_REQUIRE_ITEMS));
  TRY(check_launch());
  TRY(flush_fallbacks(e));
  TRY(read_counters(e));
  TRY(error_from_counters(e));
  if (out2) {
    out2[0] = e->h_ctr->refined;
    out2[1] = e->h_ctr->v_frees;
  }
  return VM_OK;
}

int vm_garbage_collect(vm_engine *e, const int32_t *coords, int64_t n, int64_t *freed) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  TRY(settle_all(e));
  TRY(reset_call_counters(e));
  int32_t *di = nullptr;
  if (n > 0) TRY(map_coords(e, coords, n, &di, nullptr, 0, false));
  launch_gc(e, false, di, nullptr, (int)std::max<int64_t>(n, 0), (int)(G_GC | G_COMMIT));
  TRY(check_launch());
  TRY(read_counters(e));
  TRY(error_from_counters(e));
  if (freed) *freed = e->h_ctr->v_frees;
  return VM_OK;
}

int vm_compute_normals(vm_engine *e, const int32_t *coords, int64_t n) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  TRY(settle_all(e));
  TRY(reset_call_counters(e));
  if (n <= 0) return VM_OK;
  e->h_frame->epoch = ++e->epoch;
  int32_t *di;
  TRY(map_coords(e, coords, n, &di, e->S.stamp_halo, e->epoch, false));
  launch_gc(e, false, di, nullptr, (int)n, (int)G_NORMALS);
  TRY(flush_fallbacks(e));
  TRY(check_launch());
  TRY(read_counters(e));
  return error_from_counters(e);
}

int vm_refine_eval(vm_engine *e, const uint8_t *t_curr, const uint8_t *t_prev, const double *corners,
                   int64_t n, double epsilon, int32_t *out) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !t_curr || !t_prev || !corners || !out) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  if (n <= 0) return VM_OK;
  void *buf;
  const size_t o1 = ((size_t)n + 255) & ~(size_t)255, o2 = o1 * 2, o3 = o2 + (size_t)n * 64;
  TRY(scratch(e, o3 + (size_t)n * 4 + 256, &buf));
  char *b = (char *)buf;
  CK(cudaMemcpyAsync(b, t_curr, n, cudaMemcpyHostToDevice, e->stream));
  CK(cudaMemcpyAsync(b + o1, t_prev, n, cudaMemcpyHostToDevice, e->stream));
  CK(cudaMemcpyAsync(b + o2, corners, (size_t)n * 64, cudaMemcpyHostToDevice, e->stream));
  k_refine_eval<<<grid_threads(e, n, 256), 256, 0, e->stream>>>((uint8_t *)b, (uint8_t *)(b + o1),
                                                                 (double *)(b + o2), (int)n, epsilon,
                                                                 (int32_t *)(b + o3));
  TRY(check_launch());
  CK(cudaMemcpyAsync(out, b + o3, (size_t)n * 4, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  return VM_OK;
}

int vm_block_in_frustum(vm_engine *e, const int32_t *coords, int64_t n, const vm_pose *pose,
                        const vm_intrinsics *intr, uint8_t *out) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !coords || !pose || !intr || !out) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  if (n <= 0) return VM_OK;
  fill_frame_host(e, nullptr, 0, 0, intr, pose);
  void *buf;
  const size_t o1 = ((size_t)n * sizeof(int3) + 255) & ~(size_t)255;
  TRY(scratch(e, o1 + n + 256, &buf));
  CK(cudaMemcpyAsync(buf, coords, (size_t)n * sizeof(int3), cudaMemcpyHostToDevice, e->stream));
  k_frustum_eval<<<grid_threads(e, n, 128), 128, 0, e->stream>>>(e->S, *e->h_frame, (int3 *)buf, (int)n,
                                                                  (uint8_t *)buf + o1);
  TRY(check_launch());
  CK(cudaMemcpyAsync(out, (uint8_t *)buf + o1, n, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  return VM_OK;
}

// ---- store access -----------------------------------------------------------
int vm_set_blocks(vm_engine *e, const int32_t *coords, int64_t n, const double *tsdf, const int32_t *weight) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || (!coords && n)) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  if (n <= 0) return VM_OK;
  TRY(reset_call_counters(e));
  int32_t *di;
  TRY(map_coords(e, coords, n, &di, nullptr, ++e->epoch, true));
  std::vector<int32_t> idx(n);
  CK(cudaMemcpyAsync(idx.data(), di, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, e->stream));
  TRY(init_new_blocks(e));
  if (tsdf || weight) {
    double *dt = nullptr;
    int32_t *dw = nullptr, *didx = nullptr;
    CK(cudaMalloc((void **)&didx, sizeof(int32_t) * n));
    TRY(copy_sync(e, didx, idx.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    if (tsdf) {
      CK(cudaMalloc((void **)&dt, sizeof(double) * n * kNC));
      TRY(copy_sync(e, dt, tsdf, sizeof(double) * n * kNC, cudaMemcpyHostToDevice));
    }
    if (weight) {
      CK(cudaMalloc((void **)&dw, sizeof(int32_t) * n * kNC));
      TRY(copy_sync(e, dw, weight, sizeof(int32_t) * n * kNC, cudaMemcpyHostToDevice));
    }
    k_scatter_samples<<<grid_threads(e, n * kNC, 256), 256, 0, e->stream>>>(e->S, didx, (int)n, dt, dw);
    k_rebuild_vmask<<<grid_threads(e, n * (kNC / 32), 256), 256, 0, e->stream>>>(e->S, didx, (int)n);
    TRY(check_launch());
    CK(cudaStreamSynchronize(e->stream));
    cudaFree(didx);
    if (dt) cudaFree(dt);
    if (dw) cudaFree(dw);
  }
  return VM_OK;
}

int vm_lookup(vm_engine *e, const int32_t *coords, int64_t n, uint8_t *out) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || ((!coords || !out) && n)) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  if (n <= 0) return VM_OK;
  int32_t *di;
  TRY(map_coords(e, coords, n, &di, nullptr, 0, false));
  std::vector<int32_t> idx(n);
  CK(cudaMemcpyAsync(idx.data(), di, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  for (int64_t i = 0; i < n; i++) out[i] = idx[i] >= 0;
  return VM_OK;
}

int vm_counters(vm_engine *e, vm_counter_set *out) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !out) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  TRY(read_counters(e));
  const Counters &c = *e->h_ctr;
  out->block_count = e->S.nranks > 1 ? c.nblocks_owned : c.nblocks - c.nfree;
  out->block_allocations = out->block_count;
  out->vertex_count = c.v_count;
  out->vertex_free = c.v_count - c.v_live;
  out->vertex_recycled_total = c.v_recycled;
  out->vertex_allocation_events = c.v_events;
  out->triangle_count = c.t_count;
  out->triangle_free = c.t_count - c.t_live;
  out->triangle_recycled_total = c.t_recycled;
  out->irregular_cube_count = c.irregular;
  out->block_capacity = e->S.block_cap;
  out->vertex_capacity = e->S.vrec_cap;
  out->triangle_capacity = (int64_t)e->S.block_cap * kNC * 5;
  const DevState &S = e->S;
  // records in use: handed out minus the gc CTAs' unused ranges
  std::vector<long long> rr(4 * (size_t)S.rec_chunk_ctas);
  TRY(copy_sync(e, rr.data(), S.rec_chunk, rr.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  long long spare = 0;
  for (size_t q = 0; q < rr.size(); q += 2) spare += rr[q + 1] > rr[q] ? rr[q + 1] - rr[q] : 0;
  out->vertex_records = c.a_hw - spare;
  out->store_bytes = (int64_t)(c.nblocks - c.nfree) * (int64_t)kBlockBytes + out->vertex_records * (int64_t)sizeof(VertexRec);
  out->device_bytes = (int64_t)S.block_cap * (int64_t)kBlockBytes + S.vrec_cap * (int64_t)sizeof(VertexRec) +
                      (int64_t)S.max_blocks * (int64_t)kBlockMetaBytes +
                      (int64_t)S.nbuckets * kSlotsPerBucket * (int64_t)sizeof(HashSlot) +
                      (int64_t)S.nbuckets * 8 + (int64_t)S.ovf_cap * 20 +
                      (int64_t)kHaloShards * S.halo_sh_cap * 4 + (int64_t)S.fb_cap * 16 +
                      (S.vreq ? (int64_t)S.block_cap * (kEV + 64) : 0);
  return VM_OK;
}

// host copy of `count` rows of `row_bytes` each from a device array, keeping
// only the rows in `sel` (block GC: evicted blocks are not part of the store)
static int copy_rows(vm_engine *e, void *dst, const void *src, size_t row_bytes, int64_t count,
                     const std::vector<int> &sel) {
  if ((int64_t)sel.size() == count) return copy_sync(e, dst, src, row_bytes * count, cudaMemcpyDeviceToHost);
  std::vector<char> tmp(row_bytes * count);
  TRY(copy_sync(e, tmp.data(), src, row_bytes * count, cudaMemcpyDeviceToHost));
  for (size_t k = 0; k < sel.size(); k++) memcpy((char *)dst + k * row_bytes, tmp.data() + sel[k] * row_bytes, row_bytes);
  return VM_OK;
}

int vm_snapshot_blocks(vm_engine *e, int64_t n, int32_t *coords, double *tsdf, int32_t *weight, uint8_t *tp,
                       uint8_t *tc, int32_t *ev, int32_t *tri) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  TRY(settle_all(e));
  TRY(read_counters(e));
  const int64_t nb = e->h_ctr->nblocks, live = nb - e->h_ctr->nfree;
  if (n != live)
    return set_err(VM_ERR_INPUT, "snapshot size %lld != block count %lld", (long long)n, (long long)live);
  if (n == 0) return VM_OK;
  const DevState &S = e->S;
  if (live != nb) {   // evicted blocks (block GC) are skipped
    std::vector<int4> bc(nb);
    TRY(copy_sync(e, bc.data(), S.bcoord, sizeof(int4) * nb, cudaMemcpyDeviceToHost));
    std::vector<int> sel;
    for (int64_t i = 0; i < nb; i++)
      if (bc[i].w == 0) sel.push_back((int)i);
    if ((int64_t)sel.size() != live) return set_err(VM_ERR_CONSISTENCY, "evicted block count mismatch");
    if (coords)
      for (size_t k = 0; k < sel.size(); k++) {
        coords[3 * k] = bc[sel[k]].x; coords[3 * k + 1] = bc[sel[k]].y; coords[3 * k + 2] = bc[sel[k]].z;
      }
    if (tsdf) TRY(copy_rows(e, tsdf, S.tsdf, 8 * kNC, nb, sel));
    if (weight) TRY(copy_rows(e, weight, S.weight, 4 * kNC, nb, sel));
    if (tp) TRY(copy_rows(e, tp, S.tp, kNC, nb, sel));
    if (tc) TRY(copy_rows(e, tc, S.tc, kNC, nb, sel));
    if (ev || tri) {
      TRY(run_compaction(e, 0, true));
      if (ev) TRY(copy_rows(e, ev, e->comp.ev_handles, 4 * kEV, nb, sel));
      if (tri) TRY(copy_rows(e, tri, e->comp.tri_handles, 4 * kNC * 5, nb, sel));
    }
    return VM_OK;
  }
  if (coords) {
    std::vector<int4> bc(n);
    TRY(copy_sync(e, bc.data(), S.bcoord, sizeof(int4) * n, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; i++) {
      coords[3 * i] = bc[i].x;
      coords[3 * i + 1] = bc[i].y;
      coords[3 * i + 2] = bc[i].z;
    }
  }
  if (tsdf) TRY(copy_sync(e, tsdf, S.tsdf, sizeof(double) * n * kNC, cudaMemcpyDeviceToHost));
  if (weight) TRY(copy_sync(e, weight, S.weight, sizeof(int32_t) * n * kNC, cudaMemcpyDeviceToHost));
  if (tp) TRY(copy_sync(e, tp, S.tp, (size_t)n * kNC, cudaMemcpyDeviceToHost));
  if (tc) TRY(copy_sync(e, tc, S.tc, (size_t)n * kNC, cudaMemcpyDeviceToHost));
  if (ev || tri) {
    TRY(run_compaction(e, 0, true));
    if (ev) TRY(copy_sync(e, ev, e->comp.ev_handles, sizeof(int32_t) * n * kEV, cudaMemcpyDeviceToHost));
    if (tri) TRY(copy_sync(e, tri, e->comp.tri_handles, sizeof(int32_t) * n * kNC * 5, cudaMemcpyDeviceToHost));
  }
  return VM_OK;
}

// vertex pool view: handles 0..live-1 are the live vertices in compaction
// order, live..count-1 the free entries of the reference's arena accounting
int vm_snapshot_vertices(vm_engine *e, int64_t n, double *pos, double *nrm, int32_t *ref, int32_t *birth,
                         uint8_t *alive, int32_t *free_stack) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  TRY(settle_all(e));
  TRY(read_counters(e));
  const int64_t count = e->h_ctr->v_count, live = e->h_ctr->v_live;
  if (n != count) return set_err(VM_ERR_INPUT, "snapshot size mismatch");
  const int nb = e->h_ctr->nblocks;
  TRY(run_compaction(e, 0, true));
  if (e->comp.nv != live)
    return set_err(VM_ERR_CONSISTENCY, "live vertex count %lld != occupied slots %lld", (long long)live,
                   (long long)e->comp.nv);
  if (n) {
    if (pos) {
      if (live) TRY(copy_sync(e, pos, e->comp.pos, 24ull * live, cudaMemcpyDeviceToHost));
      memset(pos + 3 * live, 0, 24ull * (n - live));
    }
    if (nrm) {
      if (live) TRY(copy_sync(e, nrm, e->comp.nrm, 24ull * live, cudaMemcpyDeviceToHost));
      memset(nrm + 3 * live, 0, 24ull * (n - live));
    }
    if (birth) {
      std::vector<long long> age(live + 1);
      if (live) TRY(copy_sync(e, age.data(), e->comp.age, 8ull * live, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < live; i++) birth[i] = (int32_t)(-age[i]);   // compacted at frame 0
      for (int64_t i = live; i < n; i++) birth[i] = 0;
    }
    if (alive)
      for (int64_t i = 0; i < n; i++) alive[i] = i < live;
    if (ref) {
      int32_t *dref;
      CK(cudaMalloc(&dref, 4ull * (live + 1)));
      if (nb) {
        k_slot_refcounts<<<grid_threads(e, (long long)nb * kEV, 256), 256, 0, e->stream>>>(e->S, nb,
                                                                                         e->comp.ev_handles, dref);
        TRY(check_launch());
      }
      CK(cudaStreamSynchronize(e->stream));
      if (live) TRY(copy_sync(e, ref, dref, 4ull * live, cudaMemcpyDeviceToHost));
      for (int64_t i = live; i < n; i++) ref[i] = 0;
      cudaFree(dref);
    }
  }
  if (free_stack)
    for (int64_t i = live; i < count; i++) free_stack[i - live] = (int32_t)i;
  return VM_OK;
}

int vm_snapshot_triangles(vm_engine *e, int64_t n, int32_t *verts, uint8_t *alive, int32_t *free_stack) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  TRY(settle_all(e));
  TRY(read_counters(e));
  const int64_t count = e->h_ctr->t_count, live = e->h_ctr->t_live;
  if (n != count) return set_err(VM_ERR_INPUT, "snapshot size mismatch");
  TRY(run_compaction(e, 0, false));
  if (e->comp.nt != live) return set_err(VM_ERR_CONSISTENCY, "live triangle count mismatch");
  if (verts) {
    if (live) TRY(copy_sync(e, verts, e->comp.idx, 12ull * live, cudaMemcpyDeviceToHost));
    for (int64_t i = 3 * live; i < 3 * n; i++) verts[i] = -1;
  }
  if (alive)
    for (int64_t i = 0; i < n; i++) alive[i] = i < live;
  if (free_stack)
    for (int64_t i = live; i < count; i++) free_stack[i - live] = (int32_t)i;
  return VM_OK;
}

// ---- outputs ------------------------------------------------------------------
int vm_irregular_count(vm_engine *e, int64_t *out) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !out) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  TRY(read_counters(e));
  void *buf;
  TRY(scratch(e, 64, &buf));
  CK(cudaMemsetAsync(buf, 0, 8, e->stream));
  const int nb = e->h_ctr->nblocks;
  if (nb) {
    k_irregular_full<<<grid_threads(e, (long long)nb * kNC, 256), 256, 0, e->stream>>>(e->S, nb,
                                                                                   (unsigned long long *)buf);
    TRY(check_launch());
  }
  unsigned long long r = 0;
  CK(cudaMemcpyAsync(&r, buf, 8, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  *out = (int64_t)r;
  return VM_OK;
}

int vm_compact(vm_engine *e, int64_t current_frame, int64_t *n_vertices, int64_t *n_triangles) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !n_vertices || !n_triangles) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  TRY(run_compaction(e, current_frame, false));
  *n_vertices = e->comp.nv;
  *n_triangles = e->comp.nt;
  return VM_OK;
}

int vm_compact_fetch(vm_engine *e, double *pos, double *nrm, int64_t *ages, int32_t *idx) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  const Compacted &c = e->comp;
  if (c.nv) {
    if (pos) TRY(copy_sync(e, pos, c.pos, 24ull * c.nv, cudaMemcpyDeviceToHost));
    if (nrm) TRY(copy_sync(e, nrm, c.nrm, 24ull * c.nv, cudaMemcpyDeviceToHost));
    if (ages) TRY(copy_sync(e, ages, c.age, 8ull * c.nv, cudaMemcpyDeviceToHost));
  }
  if (c.nt && idx) TRY(copy_sync(e, idx, c.idx, 12ull * c.nt, cudaMemcpyDeviceToHost));
  return VM_OK;
}

int vm_export_blocks(vm_engine *e, int32_t owned_only, int64_t *n_out, int32_t *coords, double *tsdf,
                     int32_t *weight, uint8_t *tp, uint8_t *tc, int32_t *birth, double *param, double *normal) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !n_out) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  TRY(read_counters(e));
  const int nb = e->h_ctr->nblocks;
  std::vector<uint8_t> own(nb);
  if (nb) TRY(copy_sync(e, own.data(), e->S.bowned, nb, cudaMemcpyDeviceToHost));
  const DevState &S = e->S;
  std::vector<int4> bc(nb);
  if (nb) TRY(copy_sync(e, bc.data(), S.bcoord, sizeof(int4) * nb, cudaMemcpyDeviceToHost));
  std::vector<int> sel;
  for (int i = 0; i < nb; i++)
    if ((!owned_only || own[i] || e->S.nranks <= 1) && bc[i].w == 0) sel.push_back(i);
  *n_out = (int64_t)sel.size();
  if (!coords || sel.empty()) return VM_OK;
  for (size_t k = 0; k < sel.size(); k++) {
    const int i = sel[k];
    coords[3 * k] = bc[i].x; coords[3 * k + 1] = bc[i].y; coords[3 * k + 2] = bc[i].z;
    if (tsdf) TRY(copy_sync(e, tsdf + k * kNC, S.tsdf + (size_t)i * kNC, 8 * kNC, cudaMemcpyDeviceToHost));
    if (weight) TRY(copy_sync(e, weight + k * kNC, S.weight + (size_t)i * kNC, 4 * kNC, cudaMemcpyDeviceToHost));
    if (tp) TRY(copy_sync(e, tp + k * kNC, S.tp + (size_t)i * kNC, kNC, cudaMemcpyDeviceToHost));
    if (tc) TRY(copy_sync(e, tc + k * kNC, S.tc + (size_t)i * kNC, kNC, cudaMemcpyDeviceToHost));
    if (param) TRY(copy_sync(e, param + k * kEV, S.vparam + (size_t)i * kEV, 8 * kEV, cudaMemcpyDeviceToHost));
  }
  if (birth || normal) {   // per-slot views of the vertex records
    const size_t ns = sel.size();
    void *buf;
    TRY(scratch(e, ns * 4 + ns * kEV * (4 + 24) + 512, &buf));
    int32_t *d_idx = (int32_t *)buf;
    int32_t *d_birth = (int32_t *)((char *)buf + ((ns * 4 + 255) & ~(size_t)255));
    double *d_nrm = (double *)((char *)d_birth + ((ns * kEV * 4 + 255) & ~(size_t)255));
    CK(cudaMemcpyAsync(d_idx, sel.data(), ns * 4, cudaMemcpyHostToDevice, e->stream));
    k_gather_slots<<<grid_threads(e, (long long)ns * kEV, 256), 256, 0, e->stream>>>(
        S, d_idx, (int)ns, birth ? d_birth : nullptr, normal ? d_nrm : nullptr);
    TRY(check_launch());
    if (birth) TRY(copy_sync(e, birth, d_birth, ns * kEV * 4, cudaMemcpyDeviceToHost));
    if (normal) TRY(copy_sync(e, normal, d_nrm, ns * kEV * 24, cudaMemcpyDeviceToHost));
  }
  return VM_OK;
}

int vm_import_blocks(vm_engine *e, int64_t n, const int32_t *coords, const double *tsdf, const int32_t *weight,
                     const uint8_t *tp, const uint8_t *tc, const int32_t *birth, const double *param,
                     const double *normal) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || (n && !coords)) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  if (n <= 0) return VM_OK;
  TRY(reset_call_counters(e));
  int32_t *di;
  TRY(map_coords(e, coords, n, &di, nullptr, ++e->epoch, true));
  std::vector<int32_t> idx(n);
  TRY(copy_sync(e, idx.data(), di, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  TRY(init_new_blocks(e));
  const DevState &S = e->S;
  for (int64_t k = 0; k < n; k++) {
    const size_t i = (size_t)idx[k];
    if (idx[k] < 0) return set_err(VM_ERR_CAPACITY, "import: block table full");
    if (tsdf) TRY(copy_sync(e, S.tsdf + i * kNC, tsdf + k * kNC, 8 * kNC, cudaMemcpyHostToDevice));
    if (weight) {
      TRY(copy_sync(e, S.weight + i * kNC, weight + k * kNC, 4 * kNC, cudaMemcpyHostToDevice));
      uint32_t vm[kNC / 32] = {};
      for (int q = 0; q < kNC; q++)
        if (weight[k * kNC + q] > 0) vm[q >> 5] |= 1u << (q & 31);
      TRY(copy_sync(e, S.vmask + i * (kNC / 32), vm, sizeof vm, cudaMemcpyHostToDevice));
    }
    if (tp) TRY(copy_sync(e, S.tp + i * kNC, tp + k * kNC, kNC, cudaMemcpyHostToDevice));
    if (tc) TRY(copy_sync(e, S.tc + i * kNC, tc + k * kNC, kNC, cudaMemcpyHostToDevice));
    if (birth) {
      uint32_t occ[kEV / 32] = {};
      for (int q = 0; q < kEV; q++)
        if (birth[k * kEV + q] >= 0) occ[q >> 5] |= 1u << (q & 31);
      TRY(copy_sync(e, S.vocc + i * (kEV / 32), occ, sizeof occ, cudaMemcpyHostToDevice));
    }
    if (param) TRY(copy_sync(e, S.vparam + i * kEV, param + k * kEV, 8 * kEV, cudaMemcpyHostToDevice));
  }
  if (birth) {   // vertex records of the occupied slots
    int64_t occupied = 0;
    for (int64_t q = 0; q < n * kEV; q++) occupied += birth[q] >= 0;
    TRY(read_counters(e));
    TRY(grow_records(e, e->h_ctr->a_hw + occupied));
    void *buf;
    TRY(scratch(e, n * 4 + n * kEV * (4 + 24) + 512, &buf));
    int32_t *d_idx = (int32_t *)buf;
    int32_t *d_birth = (int32_t *)((char *)buf + ((n * 4 + 255) & ~(size_t)255));
    double *d_nrm = (double *)((char *)d_birth + ((n * kEV * 4 + 255) & ~(size_t)255));
    CK(cudaMemcpyAsync(d_idx, idx.data(), n * 4, cudaMemcpyHostToDevice, e->stream));
    CK(cudaMemcpyAsync(d_birth, birth, n * kEV * 4, cudaMemcpyHostToDevice, e->stream));
    if (normal) CK(cudaMemcpyAsync(d_nrm, normal, n * kEV * 24, cudaMemcpyHostToDevice, e->stream));
    k_scatter_slots<<<grid_threads(e, (long long)n * kEV, 256), 256, 0, e->stream>>>(
        e->S, d_idx, (int)n, d_birth, normal ? d_nrm : nullptr);
    TRY(check_launch());
    CK(cudaStreamSynchronize(e->stream));
  }
  return VM_OK;
}

// ---- spatial partition ------------------------------------------------------
// Halo-exchange frame, first half: collect + integrate the owned blocks and
// pack the collected boundary blocks (k_pack_boundary).  Synchronous: the
// caller needs the record count for the all-gather; a heap shortfall is
// handled here (grow, integrate again -- k_fuse_blocks stopped at its guard,
// so nothing was integrated twice).
// the frame's parameters of a partitioned frame (begin, or its key pass)
static int partition_frame_setup(vm_engine *e, const double *depth, int32_t h, int32_t w, int32_t depth_on_device,
                                 const vm_intrinsics *intr, const vm_pose *pose, const vm_frame_config *cfg,
                                 int64_t frame_index, bool new_epoch) {
  if (!e->S.halo_exchange) return set_err(VM_ERR_INPUT, "engine not created in halo-exchange mode");
  if (cfg->strategy < 0 || cfg->strategy > 2) return set_err(VM_ERR_VALUE, "unknown strategy %d", cfg->strategy);
  if (cfg->trunc < e->S.cube_size) return set_err(VM_ERR_VALUE, "truncation band must be at least one cube");
  TRY(settle_all(e));
  e->part_active = false;
  const double *dd;
  TRY(stage_depth(e, depth, h, w, depth_on_device, &dd));
  fill_frame_host(e, dd, h, w, intr, pose);
  FrameDev &F = *e->h_frame;
  F.trunc = cfg->trunc;
  F.max_range = cfg->max_range;
  F.epsilon = cfg->epsilon;
  F.weight_cap = cfg->weight_cap;
  F.refine = cfg->refine;
  F.frustum_only = cfg->frustum_only;
  if (new_epoch) F.epoch = ++e->epoch;
  F.frame = (int32_t)frame_index;
  F.scope_mode = 0;
  F.strategy = cfg->strategy;
  TRY(ensure_partition_bufs(e, cfg->strategy));
  F.consume_fb = 0;   // (settle_all applied the pending records)
  F.snap = nullptr;
  F.reset_after = 0;
  F.pub_src = nullptr; F.pub_dst = nullptr; F.pub_seq = nullptr;
  F.self_dst = nullptr; F.self_seq = nullptr;
  F.ghost_recv = nullptr;
  F.ghost_max = 0;
  F.ghost_nranks = 0;
  F.row0 = F.row1 = 0;
  F.key_out = nullptr;
  F.key_count = nullptr;
  F.key_cap = 0;
  TRY(ensure_rays(e, h, w));
  F.nsteps_fixed = fixed_nsteps(e, cfg->trunc);
  F.band_step = F.nsteps_fixed > 1 ? 2.0 / (double)(F.nsteps_fixed - 1) : 0.0;
  F.block_gc_age = cfg->block_gc_age > 0 ? cfg->block_gc_age : 0;
  return VM_OK;
}

// collect (pixels, or the all-gathered key lists) + integrate owned blocks +
// pack the boundary blocks for the exchange
static int partition_frame_begin(vm_engine *e, const uint64_t *keys, int64_t n_keys, uint8_t *send,
                                 int64_t send_cap, int64_t *n_send, int64_t *n_owned_collected) {
  FrameDev &F = *e->h_frame;
  if (keys) {   // (the key pass left the frame's collect counters: clear the rest only)
    const size_t off = offsetof(Counters, nslab);
    CK(cudaMemsetAsync((char *)e->S.ctr + off, 0, sizeof(Counters) - off, e->stream));
  } else {
    TRY(reset_call_counters(e));
  }
  e->ctr_clean = false;
  e->restore_calls = false;
  cudaStream_t st = e->stream;
  e->frame_launches = 4;
  if (keys) {
    const int g = std::max(1, std::min(grid_threads(e, n_keys, 256), e->sm_count * 8));
    k_collect_keys_apply<<<g, 256, 0, st>>>(e->S, F, (const unsigned long long *)keys, (int)n_keys);
  } else {
    if (F.nsteps_fixed <= 0) {
      k_depth_stats<<<grid_blocks(e), 256, 0, st>>>(e->S, F);
      e->frame_launches++;
    }
    launch_pdl(k_collect, e->grid_collect, kCollectThreads, st, e->S, F);
  }
  launch_pdl(k_fuse_blocks, e->grid_fuse, kFB, st, e->S, F, (const int32_t *)e->S.scope,
             (const int32_t *)&e->S.ctr->ncollected, 0, (int)(F_INIT | F_INTEGRATE), 0);
  launch_pdl(k_pack_boundary, e->grid_fuse, kFB, st, e->S, F, send, (int)std::min<int64_t>(send_cap, INT32_MAX));
  TRY(check_launch());
  for (int guard = 0; guard < 64; guard++) {
    TRY(read_counters(e));
    TRY(error_from_counters(e));
    if (!e->h_ctr->need) break;
    TRY(grow_blocks(e, e->h_ctr->nblocks));
    CK(cudaMemsetAsync(&e->S.ctr->need, 0, sizeof(int32_t), st));
    e->last_resumes++;
    k_fuse_blocks<<<e->grid_fuse, kFB, 0, st>>>(e->S, F, (const int32_t *)e->S.scope,
                                                (const int32_t *)&e->S.ctr->ncollected, 0, (int)(F_INIT | F_INTEGRATE), 0);
    k_pack_boundary<<<e->grid_fuse, kFB, 0, st>>>(e->S, F, send, (int)std::min<int64_t>(send_cap, INT32_MAX));
    e->frame_launches += 2;
    TRY(check_launch());
  }
  *n_send = e->h_ctr->nsend;
  *n_owned_collected = e->h_ctr->ncollected;
  e->part_nc_own = e->h_ctr->ncollected;
  e->part_frame = F.frame;
  e->part_active = true;
  return VM_OK;
}

int vm_partition_frame_begin(vm_engine *e, const double *depth, int32_t h, int32_t w, int32_t depth_on_device,
                             const vm_intrinsics *intr, const vm_pose *pose, const vm_frame_config *cfg,
                             int64_t frame_index, uint8_t *send, int64_t send_cap, int64_t *n_send,
                             int64_t *n_owned_collected) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !intr || !pose || !cfg || !n_send || !n_owned_collected) return set_err(VM_ERR_INPUT, "null argument");
  NvtxRange nvtx_("vm_partition_frame_begin");
  TRY(partition_frame_setup(e, depth, h, w, depth_on_device, intr, pose, cfg, frame_index, true));
  return partition_frame_begin(e, nullptr, 0, send, send_cap, n_send, n_owned_collected);
}

int vm_partition_collect_keys(vm_engine *e, const double *depth, int32_t h, int32_t w, int32_t depth_on_device,
                              const vm_intrinsics *intr, const vm_pose *pose, const vm_frame_config *cfg,
                              int64_t frame_index, int32_t row0, int32_t row1, uint64_t *keys_dev, int64_t cap,
                              int64_t *n_keys) {
  if (e) e->ov_ready = false;
  if (!e || !intr || !pose || !cfg || !keys_dev || !n_keys) return set_err(VM_ERR_INPUT, "null argument");
  if (row0 < 0 || row1 < row0 || row0 % 8) return set_err(VM_ERR_VALUE, "row slice must start at a multiple of 8");
  NvtxRange nvtx_("vm_partition_collect_keys");
  TRY(partition_frame_setup(e, depth, h, w, depth_on_device, intr, pose, cfg, frame_index, true));
  FrameDev &F = *e->h_frame;
  TRY(reset_call_counters(e));
  e->ctr_clean = false;
  e->restore_calls = false;
  int32_t *d_count;
  TRY(scratch(e, 16, (void **)&d_count));
  CK(cudaMemsetAsync(d_count, 0, sizeof(int32_t), e->stream));
  FrameDev Fk = F;
  Fk.row0 = row0;
  Fk.row1 = row1;
  Fk.key_out = (unsigned long long *)keys_dev;
  Fk.key_count = d_count;
  Fk.key_cap = (int32_t)std::min<int64_t>(cap, INT32_MAX);
  if (row1 > row0) {   // (an empty slice only sets the frame up)
    if (F.nsteps_fixed <= 0) k_depth_stats<<<grid_blocks(e), 256, 0, e->stream>>>(e->S, F);   // (whole image)
    launch_pdl(k_collect, e->grid_collect, kCollectThreads, e->stream, e->S, Fk);
    TRY(check_launch());
  }
  int32_t cnt = 0;
  TRY(copy_sync(e, &cnt, d_count, sizeof cnt, cudaMemcpyDeviceToHost));
  TRY(read_counters(e));
  TRY(error_from_counters(e));
  if (cnt > Fk.key_cap) return set_err(VM_ERR_CAPACITY, "key list needs %d entries (capacity %d)", cnt, Fk.key_cap);
  *n_keys = cnt;
  return VM_OK;
}

int vm_partition_frame_begin_keys(vm_engine *e, const uint64_t *keys_dev, int64_t n_keys, uint8_t *send,
                                  int64_t send_cap, int64_t *n_send, int64_t *n_owned_collected) {
  if (e) e->ov_ready = false;
  if (!e || (!keys_dev && n_keys) || !n_send || !n_owned_collected) return set_err(VM_ERR_INPUT, "null argument");
  NvtxRange nvtx_("vm_partition_frame_begin_keys");
  static const uint64_t none = 0;
  return partition_frame_begin(e, keys_dev ? keys_dev : &none, n_keys, send, send_cap, n_send, n_owned_collected);
}

int vm_partition_repack(vm_engine *e, uint8_t *send, int64_t send_cap, int64_t *n_send) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !n_send) return set_err(VM_ERR_INPUT, "null argument");
  if (!e->part_active) return set_err(VM_ERR_INPUT, "no partition frame begun");
  CK(cudaMemsetAsync(&e->S.ctr->nsend, 0, sizeof(int32_t), e->stream));
  k_pack_boundary<<<e->grid_fuse, kFB, 0, e->stream>>>(e->S, *e->h_frame, send,
                                                       (int)std::min<int64_t>(send_cap, INT32_MAX));
  e->frame_launches++;
  TRY(check_launch());
  TRY(read_counters(e));
  *n_send = e->h_ctr->nsend;
  return VM_OK;
}

// Second half: adopt the margin records, then scope + meshing as in a fused
// frame (k_retype_place, k_gc_normals with the counter commit).
int vm_partition_frame_finish(vm_engine *e, const uint8_t *recv, const int32_t *counts, int32_t nranks,
                              int64_t max_count, vm_stats *out) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !counts || (max_count > 0 && !recv)) return set_err(VM_ERR_INPUT, "null argument");
  if (!e->part_active) return set_err(VM_ERR_INPUT, "no partition frame begun");
  if (nranks != e->S.nranks || nranks > kMaxRanks) return set_err(VM_ERR_INPUT, "rank count mismatch");
  NvtxRange nvtx_("vm_partition_frame_finish");
  e->part_active = false;
  cudaStream_t st = e->stream;
  int64_t total = 0;
  for (int q = 0; q < nranks; q++) {
    if (counts[q] < 0 || counts[q] > max_count) return set_err(VM_ERR_INPUT, "bad record count");
    if (q != e->S.rank) total += counts[q];
  }
  // every received record may become a new block: size the heap for all of
  // them now, so the rest of the frame never stops for growth
  const int64_t need = (int64_t)e->h_ctr->nblocks + total;
  if (need > e->S.block_cap) TRY(grow_blocks(e, std::min<int64_t>(need, e->S.max_blocks)));
  CK(cudaMemcpyAsync(e->d_ghost_counts, counts, sizeof(int32_t) * nranks, cudaMemcpyHostToDevice, st));
  FrameDev &F = *e->h_frame;
  F.ghost_recv = recv;
  F.ghost_max = (int32_t)max_count;
  F.ghost_nranks = nranks;
  const DevState &S = e->S;
  const long long nrec = (long long)nranks * max_count;
  k_unpack_ghosts<<<grid_threads(e, std::max<long long>(nrec, 1), 128), 128, 0, st>>>(S, F);
  launch_pdl(k_fuse_blocks, e->grid_fuse, kFB, st, S, F, (const int32_t *)S.scope, (const int32_t *)&S.ctr->ncollected,
             0, (int)(F_INIT | F_GHOST), (int)e->part_nc_own);
  launch_pdl(k_fuse_blocks, e->grid_fuse, kFB, st, S, F, (const int32_t *)S.scope, (const int32_t *)&S.ctr->ncollected,
             0, (int)F_SCOPE, 0);
  launch_retype(e, true, F);
  launch_gc(e, true, S.halo, &S.ctr->nhalo, 0,
            (int)(G_GC | G_NORMALS | G_COMMIT | G_REQUIRE_ITEMS | G_SHARDED) | gc_strategy_flag(F));
  e->frame_launches += 4 + meshing_launches(F);
  TRY(check_launch());
  TRY(read_counters(e));
  TRY(error_from_counters(e));
  for (int guard = 0; e->h_ctr->need && e->h_ctr->need_stage == 1 && guard < 8; guard++) {
    TRY(grow_records(e, record_bound(e)));   // vertex records: resume at k_retype_place
    TRY(clear_need(e));
    TRY(enqueue_meshing(e));
    e->frame_launches += 1 + meshing_launches(F);
    TRY(read_counters(e));
    TRY(error_from_counters(e));
  }
  if (e->h_ctr->need) return set_err(VM_ERR_CUDA, "halo exchange: block heap not pre-sized");
  e->ev_rec[e->ev == e->evs[1]] = false;
  fill_stats(e, e->part_frame, out ? out : &e->settled);
  if (out) out->kernel_launches = e->frame_launches;
  F.ghost_recv = nullptr;
  return VM_OK;
}

// Distributed compaction, per rank: sort the owned blocks, count their
// vertices / triangles and slot occupancy (k_compact_count over the owned list).
int vm_partition_compact_begin(vm_engine *e, int64_t *n_owned) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !n_owned) return set_err(VM_ERR_INPUT, "null argument");
  NvtxRange nvtx_("vm_partition_compact_begin");
  TRY(settle_all(e));
  TRY(read_counters(e));
  free_pcompact(e);
  auto &p = e->pc;
  const int nb = e->h_ctr->nblocks;
  const int nown = (int)(e->S.nranks > 1 ? e->h_ctr->nblocks_owned : nb);
  p.nb = nb;
  p.nown = nown;
  *n_owned = nown;
  if (nb == 0) return VM_OK;
  cudaStream_t st = e->stream;
  CK(cudaMalloc(&p.keys_in, 8ull * nb));
  CK(cudaMalloc(&p.keys_out, 8ull * nb));
  CK(cudaMalloc(&p.vals, 4ull * nb));
  CK(cudaMalloc(&p.order, 4ull * nb));
  CK(cudaMalloc(&p.vcnt, 4ull * (nb + 1)));
  CK(cudaMalloc(&p.tcnt, 4ull * (nb + 1)));
  CK(cudaMalloc(&p.occ_bits, 4ull * 48 * nb));
  CK(cudaMalloc(&p.occ_pre, 2ull * 48 * nb));
  k_owned_block_keys<<<grid_threads(e, nb, 256), 256, 0, st>>>(e->S, nb, p.keys_in, p.vals);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, p.keys_in, p.keys_out, p.vals, p.order, nb, 0, 64, st);
  CK(cudaMalloc(&p.tmp, tmp_bytes + 16));
  cub::DeviceRadixSort::SortPairs(p.tmp, tmp_bytes, p.keys_in, p.keys_out, p.vals, p.order, nb, 0, 64, st);
  if (nown) k_compact_count<<<grid_blocks(e), kThreadsCube, 0, st>>>(e->S, p.order, nown, p.vcnt, p.tcnt, p.occ_bits, p.occ_pre);
  TRY(check_launch());
  CK(cudaStreamSynchronize(st));
  return VM_OK;
}

// the owned blocks' occupancy words in sorted order (k_compact_count wrote
// them by block index)
__global__ static void k_gather_occ(const int32_t *order, int n, const uint32_t *occ_by_blk, uint32_t *out) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)n * 48;
       q += (long long)gridDim.x * blockDim.x)
    out[q] = occ_by_blk[(size_t)order[q / 48] * 48 + q % 48];
}

int vm_partition_compact_meta(vm_engine *e, uint64_t *keys, int32_t *vcnt, int32_t *tcnt, uint32_t *occ) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  auto &p = e->pc;
  if (p.nown == 0) return VM_OK;
  if (keys) TRY(copy_sync(e, keys, p.keys_out, 8ull * p.nown, cudaMemcpyDeviceToHost));
  if (vcnt) TRY(copy_sync(e, vcnt, p.vcnt, 4ull * p.nown, cudaMemcpyDeviceToHost));
  if (tcnt) TRY(copy_sync(e, tcnt, p.tcnt, 4ull * p.nown, cudaMemcpyDeviceToHost));
  if (occ) {
    uint32_t *tmp;
    CK(cudaMalloc(&tmp, 4ull * 48 * p.nown));
    k_gather_occ<<<grid_threads(e, (long long)p.nown * 48, 256), 256, 0, e->stream>>>(p.order, p.nown, p.occ_bits, tmp);
    TRY(check_launch());
    const int rc = copy_sync(e, occ, tmp, 4ull * 48 * p.nown, cudaMemcpyDeviceToHost);
    cudaFree(tmp);
    TRY(rc);
  }
  return VM_OK;
}

__global__ static void k_pbase(const int32_t *order, int n, const int32_t *my_global, const int64_t *vbase,
                               int32_t *vbase_by_blk) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    vbase_by_blk[order[i]] = (int32_t)vbase[my_global[i]];
}

int vm_partition_compact_fill(vm_engine *e, const uint64_t *gkeys, const int64_t *vbase, const int64_t *tbase,
                              const uint32_t *gocc, const int32_t *gocc_pre, int64_t n_global,
                              const int32_t *my_global, int64_t current_frame, double *pos, double *nrm,
                              int64_t *ages, int32_t *idx) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e) return set_err(VM_ERR_INPUT, "null engine");
  NvtxRange nvtx_("vm_partition_compact_fill");
  auto &p = e->pc;
  if (p.nown == 0 || n_global == 0) return VM_OK;
  if (!gkeys || !vbase || !tbase || !gocc || !gocc_pre || !my_global) return set_err(VM_ERR_INPUT, "null argument");
  cudaStream_t st = e->stream;
  const size_t ng = (size_t)n_global;
  char *buf;
  const size_t o_keys = 0, o_vb = o_keys + 8 * ng, o_tb = o_vb + 8 * ng, o_occ = o_tb + 8 * ng,
               o_pre = o_occ + 4 * 48 * ng, o_my = o_pre + 4 * 48 * ng, o_vbb = o_my + 4 * (size_t)p.nown,
               total = o_vbb + 4 * (size_t)p.nb + 64;
  CK(cudaMalloc(&buf, total));
  CK(cudaMemcpyAsync(buf + o_keys, gkeys, 8 * ng, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(buf + o_vb, vbase, 8 * ng, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(buf + o_tb, tbase, 8 * ng, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(buf + o_occ, gocc, 4 * 48 * ng, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(buf + o_pre, gocc_pre, 4 * 48 * ng, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(buf + o_my, my_global, 4 * (size_t)p.nown, cudaMemcpyHostToDevice, st));
  int32_t *vbb = (int32_t *)(buf + o_vbb);
  k_pbase<<<grid_threads(e, p.nown, 256), 256, 0, st>>>(p.order, p.nown, (const int32_t *)(buf + o_my),
                                                        (const int64_t *)(buf + o_vb), vbb);
  TRY(reset_call_counters(e));
  k_compact_vertices<<<grid_blocks(e), kThreadsCube, 0, st>>>(e->S, p.order, p.nown, p.occ_bits, p.occ_pre, vbb, pos,
                                                              nrm, (long long *)ages, (long long)current_frame,
                                                              nullptr);
  k_pcompact_triangles<<<grid_blocks(e), kThreadsCube, 0, st>>>(
      e->S, p.order, p.nown, (const int32_t *)(buf + o_my), (const unsigned long long *)(buf + o_keys),
      (int)n_global, (const int64_t *)(buf + o_vb), (const int64_t *)(buf + o_tb), (const uint32_t *)(buf + o_occ),
      (const int32_t *)(buf + o_pre), idx);
  const int lrc = check_launch();
  CK(cudaStreamSynchronize(st));
  cudaFree(buf);
  TRY(lrc);
  TRY(read_counters(e));
  return error_from_counters(e);
}

// Engine.audit (engine.py:187-230).  With slot-resident vertices and
// type-derived triangles, a reference-count mismatch shows up as a referenced
// but empty slot and a zero-ref live vertex as an occupied but unreferenced
// slot; conservation compares the pool counters with full recounts.
int vm_audit(vm_engine *e, vm_audit_report *out) {
  if (e) e->ov_ready = false;   // (frame overlap: only a frame right behind a frame)
  if (!e || !out) return set_err(VM_ERR_INPUT, "null argument");
  TRY(settle_all(e));
  TRY(read_counters(e));
  const Counters c = *e->h_ctr;
  unsigned long long *sums;
  CK(cudaMalloc(&sums, 64));
  CK(cudaMemsetAsync(sums, 0, 64, e->stream));
  if (c.nblocks) {
    k_audit<<<grid_threads(e, (long long)c.nblocks * kEV, 256), 256, 0, e->stream>>>(e->S, c.nblocks, sums);
    TRY(check_launch());
  }
  int32_t *claims = nullptr;   // vertex-record ownership: one holder per record handed out
  if (c.a_hw > 0) {
    CK(cudaMalloc(&claims, (size_t)c.a_hw * sizeof(int32_t)));
    CK(cudaMemsetAsync(claims, 0, (size_t)c.a_hw * sizeof(int32_t), e->stream));
    k_audit_records<<<grid_threads(e, std::max<long long>((long long)c.nblocks * kEV, 2LL * e->S.rec_chunk_ctas), 256),
                      256, 0, e->stream>>>(e->S, c.nblocks, c.a_hw, claims, sums + 4);
    TRY(check_launch());
  }
  unsigned long long h[8];
  CK(cudaMemcpyAsync(h, sums, 64, cudaMemcpyDeviceToHost, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  cudaFree(sums);
  if (claims) cudaFree(claims);
  out->vertices_live = c.v_live;
  out->triangles_live = c.t_live;
  out->refcount_mismatches = (int64_t)h[1];
  out->duplicate_handles = (int64_t)h[4];   // (a vertex is its slot; its record has one holder)
  out->zero_ref_live = (int64_t)h[2];
  out->conservation_ok = ((int64_t)h[0] == c.v_live) && ((int64_t)h[3] == c.t_live) &&
                         (c.v_count >= c.v_live) && (c.t_count >= c.t_live);
  return VM_OK;
}

}  // extern "C"
