// vm_kernels.cuh -- the per-frame kernels of the B200 mesh-generation path.
//
// Frame = 5 kernels on one stream, no host sync inside a frame:
//   k_depth_stats   valid-pixel count + max ray norm              (fusion.py:81-94)
//   k_collect       ray-band block collection + hash insert       (fusion.py:95-106, store.py:296-320)
//   k_fuse_blocks   init new blocks + neighbour links, TSDF
//                   integration, scope slabs + halo marking       (store.py:70-81, fusion.py:138-168,
//                                                                  mesher.py:499-543)
//   k_retype_place  cube typing (+ Hamming refinement), implicit
//                   retriangulation (triangle/ref-count deltas),
//                   claim-based vertex placement into edge slots  (mesher.py:111-257, :283-326,
//                                                                  refine.py:98-135)
//   k_gc_normals    refcount==0 vertex recycling, gradient normals
//                   with the face-normal fallback, counter commit (mesher.py:333-486)
// Kernels after k_collect return at once if the block-heap guard tripped
// (ctr->need) or an error was raised; the host grows the heap and resumes.
#pragma once
#include <cuda_pipeline.h>

#include "vm_device.cuh"

namespace vm {

constexpr int kThreadsCube = 512;   // one thread per cube of a block

enum { F_INIT = 1, F_INTEGRATE = 2, F_SCOPE = 4, F_HALO = 8, F_GHOST = 16 };
// halo-exchange record: coordinate, then the block's 512 tsdf and 512 weights
constexpr size_t kGhostRec = 16 + 8 * 512 + 4 * 512;
enum { G_GC = 1, G_NORMALS = 2, G_COMMIT = 4, G_REQUIRE_ITEMS = 8, G_SHARDED = 16,
       G_PARTITION = 32,     // G_PARTITION: requests are k_place_parity's bytes (S.vreq)
       G_OVERLAP = 64 };     // frame path: save + clear the collect counters, then let the next frame's
                             // k_collect launch (cudaTriggerProgrammaticLaunchCompletion)

// error and need are adjacent: one 8-byte load
__device__ __forceinline__ bool halted(const DevState &S) {
  const int2 v = __ldcg(reinterpret_cast<const int2 *>(&S.ctr->error));
  return (v.x | v.y) != 0;
}


// warp-aggregated append of `cnt` entries to a shared-memory list; returns
// this lane's first index
__device__ __forceinline__ int smem_append(int cnt, int *s_count) {
  const int lane = threadIdx.x & 31;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int base = 0;
  if (lane == 31 && total) base = atomicAdd(s_count, total);
  base = __shfl_sync(0xffffffffu, base, 31);
  return base + incl - cnt;
}

// ------------------------------------------------------------ shared helpers
// Per-call counters a kernel needs before its loop, read by ONE thread and
// broadcast through shared memory (every CTA reading them from every warp
// serialises thousands of requests on one L2 line).  v[0] = halted, v[1..3]
// kernel-specific.  Ends with a barrier.
// (null pointers read as 0).  sv[4] = the CTA's first list entry, prefetched
// in the same round trip when `first` is non-null.  (The MC edge masks are
// computed from the type bits, edge_mask_of, and the triangle counts read
// through the read-only cache where a cube changed: no per-CTA table staging.)
// The counters are read through the L1 / read-only path (__ldg): none of the
// fields read here changes while the kernel runs, and a grid's CTAs on one SM
// then share one L2 request instead of each queueing on the same line (2048
// CTAs x 4 requests took ~2.5 us, trace v8).
__device__ __forceinline__ void read_prologue(const DevState &S, int *sv, const int32_t *a, const int32_t *b,
                                              const int32_t *c, const int32_t *first = nullptr) {
  if (threadIdx.x == 0) {
    const int2 h = __ldg(reinterpret_cast<const int2 *>(&S.ctr->error));
    const int va = a ? __ldg(a) : 0, vb = b ? __ldg(b) : 0, vc = c ? __ldg(c) : 0;
    const int vf = first ? __ldcg(first) : -1;
    sv[0] = (h.x | h.y) != 0;
    sv[1] = va; sv[2] = vb; sv[3] = vc; sv[4] = vf;
  }
  __syncthreads();
}

// cp.async global -> shared of 4 / 8 bytes, zero-filled when `valid` is false
// (no register staging: the loads stay in flight while the warp goes on)
__device__ __forceinline__ void cp_async4(void *dst, const void *src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 4 : 0));
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ int ld_acquire(const int32_t *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Frame overlap: the CTA waits until the previous frame's k_gc_normals has
// committed (its epoch in *S.gc_done; every commit writes it, halted or not)
__device__ __forceinline__ void wait_prev_gc(const DevState &S, const FrameDev &F) {
  if (F.wait_epoch <= 0) return;
  if (threadIdx.x == 0)
    while (ld_acquire(S.gc_done) < F.wait_epoch) __nanosleep(200);
  __syncthreads();
}

// Publish the previous frame's counter snapshot to the host (k_collect, one CTA)
__device__ __forceinline__ void publish_snapshot(const FrameDev &F) {
  constexpr int kWords = (int)(sizeof(Counters) / 4);
  const uint32_t *src = reinterpret_cast<const uint32_t *>(F.pub_src);
  uint32_t *dst = reinterpret_cast<uint32_t *>(F.pub_dst);
  for (int q = threadIdx.x; q < kWords; q += blockDim.x) dst[q] = __ldcg(src + q);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long *>(F.pub_seq) = F.pub_id;
  }
}

// The frame's host copy has landed (copy-stream flag, FrameDev::in_flag): one
// thread polls, the CTA waits
__device__ __forceinline__ void wait_input_flag(const DevState &S, const FrameDev &F) {
  if (!F.in_flag) return;
  if (threadIdx.x == 0) {
    const unsigned long long t0 = gtimer();
    for (;;) {
      unsigned long long v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(F.in_flag) : "memory");
      if (v >= F.in_id) break;
      if (gtimer() - t0 > 2000000000ull) {   // (2 s: the copy failed -- raise, never hang)
        set_error(S, ERR_CONSISTENCY, 60);
        break;
      }
      __nanosleep(256);
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------ depth stats
__device__ __forceinline__ void wait_input_flag(const DevState &S, const FrameDev &F);

__global__ void __launch_bounds__(256) k_depth_stats(DevState S, const FrameDev F) {
  // PDL: wait for the previous kernel -- except behind the previous frame's
  // k_gc_normals (F.overlap): this pass reads only the frame's depth (after
  // its host copy, when there is one) and writes collect counters the gc
  // cleared before it let this frame launch
  if (!F.overlap) cudaGridDependencySynchronize();
  wait_input_flag(S, F);
  if (blockIdx.x == 0 && threadIdx.x == 0) S.ctr->t_start_ns = gtimer();
  __shared__ double smax[8];
  __shared__ int scnt[8];
  const long long npix = (long long)F.h * F.w;
  double best = -1.0;
  int cnt = 0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
       p += (long long)gridDim.x * blockDim.x) {
    double d;
    if (F.raw) {   // raw u16 frame: convert exactly as read_depth and keep the f64 depth
      d = (double)F.raw[p] / F.depth_scale;
      F.depth_out[p] = d;
    } else {
      d = F.depth[p];
    }
    if (d > 0 && d <= F.max_range) {
      const int v = (int)(p / F.w), u = (int)(p - (long long)v * F.w);
      const double rx = ((double)u - F.cx) / F.fx, ry = ((double)v - F.cy) / F.fy;
      best = fmax(best, sqrt(__dadd_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)), 1.0)));
      cnt++;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  cnt = warp_sum(cnt);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) { smax[wid] = best; scnt[wid] = cnt; }
  if (F.raw) __threadfence();   // (the f64 depth written here is read by an overlapped k_collect)
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) { best = fmax(best, smax[w]); cnt += scnt[w]; }
    if (cnt) {
      atomicAdd(&S.ctr->nvalid, cnt);
      atomicMax(&S.ctr->maxnorm_bits, (unsigned long long)__double_as_longlong(best));
    }
    __threadfence();
    atomicAdd(&S.ctr->ds_done, 1);   // (an overlapped k_collect counts the CTAs done)
  }
}

// ------------------------------------------------------------ norm bounds
// min / max ray norm over every pixel of an (h, w) image (positive doubles
// order as their bit patterns).  The band step count is monotone in the max
// norm over the VALID pixels, which lies between the two, so when both bounds
// give the same count the frame needs no depth reduction (fusion.py:88-94).
// Also fills the per-column / per-row ray tables (fusion.py:29-33: (u - cx) / fx,
// (v - cy) / fy), so the per-pixel passes do not divide.
__global__ void k_norm_bounds(const FrameDev F, unsigned long long *out, double *rays) {
  const long long npix = (long long)F.h * F.w;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < F.w + F.h; q += gridDim.x * blockDim.x)
    rays[q] = q < F.w ? ((double)q - F.cx) / F.fx : ((double)(q - F.w) - F.cy) / F.fy;
  unsigned long long lo = ~0ull, hi = 0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
       p += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(p / F.w), u = (int)(p - (long long)v * F.w);
    const double rx = ((double)u - F.cx) / F.fx, ry = ((double)v - F.cy) / F.fy;
    const unsigned long long b = (unsigned long long)__double_as_longlong(
        sqrt(__dadd_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)), 1.0)));
    lo = b < lo ? b : lo;
    hi = b > hi ? b : hi;
  }
  atomicMin(out, lo);
  atomicMax(out + 1, hi);
}

// ------------------------------------------------------------ face-normal fallback
// edge index, in the neighbour cube owner - du*e_u - dw*e_w, of the edge slot
// owned along `axis` (u, w the other two axes)
// (register-only: [axis][du*2+dw] packed 4 bits each -- per-thread axes would
// make a constant-bank table read serialise)
__device__ __forceinline__ int cube_edge_of_slot(int axis, int du, int dw) {
  constexpr unsigned long long kTab = 0x0ull | 4ull << 4 | 2ull << 8 | 6ull << 12 | 3ull << 16 | 7ull << 20 |
                                      1ull << 24 | 5ull << 28 | 8ull << 32 | 11ull << 36 | 9ull << 40 | 10ull << 44;
  return (int)((kTab >> (4 * (axis * 4 + du * 2 + dw))) & 15ull);
}

// position q of the 9^3 type tile over cube locals -1..7 -> neighbour
// direction and source cube (index arithmetic, no table load on the chain)
__device__ __forceinline__ void type_tile_src(int q, int &dir, int &src) {
  const int a = q / 81, r = q - a * 81, bb = r / 9, cc = r - bb * 9;
  const int lx = a - 1, ly = bb - 1, lz = cc - 1;
  dir = nbr_dir(lx < 0 ? -1 : 0, ly < 0 ? -1 : 0, lz < 0 ? -1 : 0);
  src = (lx & 7) * 64 + (ly & 7) * 8 + (lz & 7);
}

// edge e -> owner-cube offset (x | y<<1 | z<<2) | axis << 3, 5 bits per edge (mc_tables.py:44-64)
__host__ __device__ constexpr unsigned long long edge_own_axis(int e) {
  constexpr int own[12] = {0, 1, 2, 0, 4, 5, 6, 4, 0, 1, 3, 2};
  constexpr int axis[12] = {0, 1, 0, 1, 0, 1, 0, 1, 2, 2, 2, 2};
  return (unsigned long long)(own[e] | axis[e] << 3);
}
constexpr unsigned long long kEdgeOwnAxis =
    edge_own_axis(0) | edge_own_axis(1) << 5 | edge_own_axis(2) << 10 | edge_own_axis(3) << 15 |
    edge_own_axis(4) << 20 | edge_own_axis(5) << 25 | edge_own_axis(6) << 30 | edge_own_axis(7) << 35 |
    edge_own_axis(8) << 40 | edge_own_axis(9) << 45 | edge_own_axis(10) << 50 | edge_own_axis(11) << 55;

// The 4 cubes around the edge slot (slot_ci, axis): candidate j = (du, dw) =
// (j >> 1, j & 1) sits at -du along u and -dw along w (u, w = the other two
// axes), i.e. at cube locals (l0, l1, l2) in [-1, 7]^3.
__device__ __forceinline__ void slot_cube(int slot_ci, int axis, int j, int &l0, int &l1, int &l2) {
  const int du = j >> 1, dw = j & 1;
  l0 = (slot_ci >> 6) - (axis == 0 ? 0 : du);
  l1 = ((slot_ci >> 3) & 7) - (axis == 0 ? du : 0) - (axis == 2 ? dw : 0);
  l2 = (slot_ci & 7) - (axis == 2 ? 0 : dw);
}

// Face-normal fallback for one vertex, computed by one warp (mesher.py:456-486).
// `types4` holds the types of the 4 cubes around the slot (byte j = candidate
// j), `cand` flags the candidates whose triangles count (edge in the cube's
// mask, cube inside a halo block of this call); lanes 0..26 hold the block's
// neighbour row in `nbr_lane`.  Lane l handles (incident cube j = l / 5,
// triangle slot s = l % 5); the contributions are then summed by lane 0 in the
// reference's order: vertex position k major, then halo blocks in sorted order,
// then cube, then triangle slot -- bit-identical to np.add.at's.
__device__ __forceinline__ void fallback_normal_warp(const double *__restrict__ vparam, double cube_size,
                                                     int nbr_lane, uint32_t types4, uint32_t cand, int4 bc,
                                                     int slot_ci, int axis, double *dst) {
  const int lane = threadIdx.x & 31;
  // the vertex's current normal ("never set" test) is requested first
  const double o0 = lane == 0 ? dst[0] : 0.0, o1 = lane == 0 ? dst[1] : 0.0, o2 = lane == 0 ? dst[2] : 0.0;
  // lane l: candidate cube j = l / 5, triangle slot s = l % 5
  const int j = lane / 5, s = lane % 5;
  const int jj = j < 4 ? j : 0;
  int m0, m1, m2;
  slot_cube(slot_ci, axis, jj, m0, m1, m2);
  const int tt = (types4 >> (8 * jj)) & 0xFF;
  const int e = cube_edge_of_slot(axis, jj >> 1, jj & 1);
  // rank of the candidate cube by (sorted block, cube) key among the valid ones
  int jrank = 0;
  {
    auto key = [&](int q) {
      int a0, a1, a2;
      slot_cube(slot_ci, axis, q, a0, a1, a2);
      const int dx = a0 < 0 ? -1 : 0, dy = a1 < 0 ? -1 : 0, dz = a2 < 0 ? -1 : 0;
      return (((dx + 1) * 4 + (dy + 1) * 2 + (dz + 1)) << 9) | ((a0 & 7) * 64 + (a1 & 7) * 8 + (a2 & 7));
    };
    const int mine = key(jj);
#pragma unroll
    for (int q = 0; q < 4; q++) jrank += ((cand >> q) & 1) && key(q) < mine;
  }
  const bool my_valid = j < 4 && ((cand >> jj) & 1) && s < c_tri_count[tt];
  const unsigned long long packed = c_tri_packed[tt];
  int kpos = -1;
  if (my_valid) {
#pragma unroll
    for (int q = 0; q < 3; q++)
      if ((int)((packed >> (4 * (3 * s + q))) & 0xF) == e) kpos = q;
  }
  // owner block of each of the triangle's 3 vertices (shuffled from the row)
  int obq[3], oxq[3], oyq[3], ozq[3], axq[3];
#pragma unroll
  for (int q = 0; q < 3; q++) {
    const int eq = (int)((packed >> (4 * (3 * s + q))) & 0xF);
    const int oa = (int)((kEdgeOwnAxis >> (5 * eq)) & 31);   // owner offset | axis << 3
    const int own = oa & 7;
    axq[q] = oa >> 3;
    oxq[q] = m0 + (own & 1); oyq[q] = m1 + ((own >> 1) & 1); ozq[q] = m2 + ((own >> 2) & 1);
    const int dir = nbr_dir(oxq[q] < 0 ? -1 : oxq[q] >> 3, oyq[q] < 0 ? -1 : oyq[q] >> 3,
                            ozq[q] < 0 ? -1 : ozq[q] >> 3);
    obq[q] = __shfl_sync(0xffffffffu, nbr_lane, dir);
  }
  double fn[3] = {0.0, 0.0, 0.0};
  if (kpos >= 0) {
    double p[3][3];
#pragma unroll
    for (int q = 0; q < 3; q++) {
      const int ox = oxq[q], oy = oyq[q], oz = ozq[q], ax = axq[q];
      const double pa = vparam[(size_t)obq[q] * kEV + ((ox & 7) * 64 + (oy & 7) * 8 + (oz & 7)) * 3 + ax];
      const double gx = __dmul_rn((double)(bc.x * kB + ox), cube_size);
      const double gy = __dmul_rn((double)(bc.y * kB + oy), cube_size);
      const double gz = __dmul_rn((double)(bc.z * kB + oz), cube_size);
      p[q][0] = ax == 0 ? pa : gx;
      p[q][1] = ax == 1 ? pa : gy;
      p[q][2] = ax == 2 ? pa : gz;
    }
    const double a[3] = {p[1][0] - p[0][0], p[1][1] - p[0][1], p[1][2] - p[0][2]};
    const double bb[3] = {p[2][0] - p[0][0], p[2][1] - p[0][1], p[2][2] - p[0][2]};
    fn[0] = __dmul_rn(a[1], bb[2]) - __dmul_rn(a[2], bb[1]);
    fn[1] = __dmul_rn(a[2], bb[0]) - __dmul_rn(a[0], bb[2]);
    fn[2] = __dmul_rn(a[0], bb[1]) - __dmul_rn(a[1], bb[0]);
  }
  // ordered accumulation: k major, then cube rank, then triangle slot.  The
  // pending lanes' keys are distinct and < 60: their ranks come from one
  // 64-bit presence mask, then the contributions are added in rank order
  const bool pend = kpos >= 0;
  const int mykey = pend ? (kpos * 4 + jrank) * 5 + s : 0;
  const unsigned klo = __reduce_or_sync(0xffffffffu, pend && mykey < 32 ? 1u << mykey : 0u);
  const unsigned khi = __reduce_or_sync(0xffffffffu, pend && mykey >= 32 ? 1u << (mykey - 32) : 0u);
  const int myrank = !pend ? -1
                     : mykey < 32 ? __popc(klo & ((1u << mykey) - 1u))
                                  : __popc(klo) + __popc(khi & ((1u << (mykey - 32)) - 1u));
  double acc[3] = {0.0, 0.0, 0.0};
  const int npend = __popc(klo) + __popc(khi);
  for (int it = 0; it < npend; it++) {
    const int bl = __ffs(__ballot_sync(0xffffffffu, myrank == it)) - 1;
    acc[0] = __dadd_rn(acc[0], __shfl_sync(0xffffffffu, fn[0], bl));
    acc[1] = __dadd_rn(acc[1], __shfl_sync(0xffffffffu, fn[1], bl));
    acc[2] = __dadd_rn(acc[2], __shfl_sync(0xffffffffu, fn[2], bl));
  }
  if (lane == 0) {
    const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(acc[0], acc[0]), __dmul_rn(acc[1], acc[1])),
                                      __dmul_rn(acc[2], acc[2])));
    if (nrm > 1e-20) {
      dst[0] = (-1.0 * acc[0]) / nrm;
      dst[1] = (-1.0 * acc[1]) / nrm;
      dst[2] = (-1.0 * acc[2]) / nrm;
    } else if (o0 == 0.0 && o1 == 0.0 && o2 == 0.0) {
      dst[2] = 1.0;
    }
  }
}

// (the rare inline path of k_gc_normals: out of line, off its register budget)
__device__ __noinline__ void fallback_normal_inline(const double *vparam, double cube_size, int nbr_lane,
                                                    uint32_t types4, uint32_t cand, int4 bc, int slot_ci, int axis,
                                                    double *dst) {
  fallback_normal_warp(vparam, cube_size, nbr_lane, types4, cand, bc, slot_ci, axis, dst);
}

struct FallbackArgs {   // what the consumer touches (passed by value: no DevState copy in local memory)
  Counters *ctr;
  const int4 *fallback;
  const int32_t *nbr;
  const int4 *bcoord;
  const double *vparam;
  VertexRec *vrec;
  double cube_size;
};

__device__ __noinline__ void consume_fallback(const FallbackArgs S, int f);

// Apply fallback records [0, n), one warp per record: warp `first` of
// `nwarps` takes record `first`, and when there are more records than warps
// (C5: ~7.6 k records for ~1.1 k warps) the warps that finish first take the
// rest one at a time from a counter (*next, requested while the current
// record is processed) -- the spare CTAs are dispatched last and a few at a
// time under the previous frame's gc, so a static share would leave the last
// ones with the longest chains.
__device__ __noinline__ void consume_fallbacks(const FallbackArgs S, int n, int first, int nwarps, int32_t *next) {
  const int lane = threadIdx.x & 31;
  int f = first;
  while (f < n) {
    int fn = n;
    if (n > nwarps && lane == 0) fn = nwarps + atomicAdd(next, 1);
    consume_fallback(S, f);
    f = __shfl_sync(0xffffffffu, fn, 0);
  }
}

// one record (its warp)
__device__ __noinline__ void consume_fallback(const FallbackArgs S, int f) {
  const int lane = threadIdx.x & 31;
  {
    // record: block, slot | candidate mask << 11, the 4 cube types, the vertex record
    const int4 rec = __ldcg(S.fallback + f);
    const int b = rec.x, sl = rec.y & 2047;
    const int nbr_lane = lane < 27 ? (lane == 13 ? b : __ldcg(S.nbr + (size_t)b * 27 + lane)) : -1;
    const int4 bc = __ldcg(S.bcoord + b);
    fallback_normal_warp(S.vparam, S.cube_size, nbr_lane, (uint32_t)rec.z, (uint32_t)rec.y >> 11, bc, sl / 3,
                         sl % 3, S.vrec[rec.w].nrm);
  }
}

// Top up k_gc_normals' per-CTA vertex-record ranges (kept >= kRecChunk, a run
// of 2 kRecChunk appended when short): one thread per gc CTA index, run by the
// next frame's k_collect off its critical path, so the gc never waits for the
// record counter in the common case.
__device__ __noinline__ void top_up_record_ranges(long long *ranges, int nctas, int64_t *a_hw, int first,
                                                  int stride) {
  for (int c = first; c < nctas; c += stride) {
    long long *rr = ranges + 4 * c;
    const longlong2 r0 = *reinterpret_cast<const longlong2 *>(rr), r1 = *reinterpret_cast<const longlong2 *>(rr + 2);
    long long a0 = r0.x, e0 = r0.y;
    if ((e0 - a0) + (r1.y - r1.x) >= kRecChunk) continue;
    const long long nb = (long long)atomicAdd(reinterpret_cast<unsigned long long *>(a_hw),
                                              (unsigned long long)(2 * kRecChunk));
    if (e0 <= a0) { a0 = r1.x; e0 = r1.y; }   // (range 1 moves up; both short cannot happen: range 1 is
                                               //  consumed only after range 0)
    *reinterpret_cast<longlong2 *>(rr) = make_longlong2(a0, e0);
    *reinterpret_cast<longlong2 *>(rr + 2) = make_longlong2(nb, nb + 2 * kRecChunk);
  }
}

// ------------------------------------------------------------ collect
// fusion.py:95-106 + store.py:296-320.  A CTA covers a 64x8-pixel region (two
// pixels per thread, coalesced rows).  The band samples' block keys are first
// merged inside each warp (__match_any_sync), then in a CTA-local shared-memory
// set; after one barrier the region's DISTINCT blocks are probed / inserted in
// the global table in parallel, one thread each -- one hash round trip per
// block and region instead of one per sample step and warp.
constexpr int kCollectThreads = 256;
constexpr int kRegionW = 64, kRegionH = 8;
constexpr int kCSet = 1024;   // CTA-local key set (open addressing)
constexpr int kCOver = 256;   // keys that found no free set slot within 32 probes
constexpr unsigned long long kNoKey = ~0ull;

__device__ __forceinline__ unsigned cset_hash(unsigned long long k) {
  const unsigned x = (unsigned)(k ^ (k >> 21) ^ (k >> 42));
  return (x * 2654435761u) >> (32 - 10);
}

// probe / insert one block; returns its index if this call collects it now
// (first to stamp it this call), else -1
__device__ __forceinline__ int collect_block(const DevState &S, const FrameDev &F, int x, int y, int z) {
  HashRef r = hash_find_ref(S, x, y, z);
  bool created = false;
  if (r.idx == -1) r = hash_insert_collect(S, x, y, z, F.epoch, r.free_slot, &created);
  else if (r.idx == -2)   // a key whose allocation failed (table full): the reference raises again
    set_error(S, ERR_CAPACITY, S.max_blocks, S.table_size, 1, F.epoch);
  if (created) {
    S.stamp_collect[r.idx] = F.epoch;
    return r.idx;
  }
  if (r.idx >= 0 && r.stamp != F.epoch && atomicExch(r.stamp_ptr, F.epoch) != F.epoch) {
    S.stamp_collect[r.idx] = F.epoch;
    return r.idx;
  }
  return -1;
}

__global__ void __launch_bounds__(kCollectThreads, 5) k_collect(DevState S, const FrameDev F) {
  // PDL: wait for the previous kernel -- except behind the previous frame's
  // k_gc_normals (F.overlap): nothing below reads or writes what that kernel
  // does, save the parts that first wait for its commit (wait_prev_gc)
  if (!F.overlap) cudaGridDependencySynchronize();
  trace_at(S, TK_COLLECT, 0);
  trace_span(S, 0, F.frame, false);
  Counters *ctr = S.ctr;
  if (blockIdx.x == 0 && threadIdx.x == 0 && F.nsteps_fixed > 0) {   // (not when it stops at the guard)
    const int2 h = __ldcg(reinterpret_cast<const int2 *>(&ctr->error));
    if (!(h.x != 0 || (h.y != 0 && h.y != F.epoch))) ctr->t_start_ns = gtimer();
  }
  if (F.pub_src && blockIdx.x == gridDim.x - 1) {   // (the last CTA to be dispatched)
    wait_prev_gc(S, F);
    publish_snapshot(F);
  }
  int nsteps = F.nsteps_fixed;
  if (nsteps <= 0 && F.ds_wait > 0) {   // (overlapped: no grid-dependency wait covers k_depth_stats)
    if (threadIdx.x == 0)
      while (ld_acquire(&ctr->ds_done) < F.ds_wait) __nanosleep(128);
    __syncthreads();
  }
  if (nsteps <= 0 && ld_vol(&ctr->nvalid) == 0) {
    nsteps = 0;   // (no valid pixel: no band samples; the spare CTAs' work still runs)
  } else if (nsteps <= 0) {
    const double maxnorm = __longlong_as_double((long long)ld_vol(&ctr->maxnorm_bits));
    const double half_block = S.extent * 0.5;
    const double band = __dmul_rn(__dmul_rn(2.0, F.trunc), maxnorm);
    nsteps = (int)ceil(band / half_block) + 1;
    if (nsteps < 2) nsteps = 2;
  }
  const double step = F.nsteps_fixed > 0 ? F.band_step : 2.0 / (double)(nsteps - 1);
  const bool multi = S.nranks > 1 && F.key_out == nullptr;   // (a key list keeps every block)
  trace_at(S, TK_COLLECT, 1);
  __shared__ unsigned long long s_key[kCSet];
  __shared__ uint16_t s_list[kCSet];
  __shared__ unsigned long long s_over[kCOver];
  __shared__ int s_out[kCSet + kCOver];
  __shared__ int s_n, s_nover, s_valid, s_nout, s_base, s_stop;
  const int t = threadIdx.x, lane = t & 31;
  const int rx = (F.w + kRegionW - 1) / kRegionW;
  // (the row slice of a sharded band walk: region rows [ry_begin, ry_begin + ry))
  const int ry_begin = F.row1 > 0 ? F.row0 / kRegionH : 0;
  const int ry = (F.row1 > 0 ? (min(F.row1, F.h) + kRegionH - 1) / kRegionH : (F.h + kRegionH - 1) / kRegionH) - ry_begin;
  const bool emit = F.key_out != nullptr;   // list the keys, do not collect
  // Guard (error / heap exhausted): a frame queued behind one that stopped
  // must not write anything -- the host resumes the stopped frame and launches
  // this one again.  Read here, checked before the first write (the load's
  // latency hides behind the first region's sampling).
  // The heap flag counts only when an earlier frame set it: a sibling CTA of
  // this k_collect may set it mid-kernel (the frame then resumes after
  // k_collect, whose results must be complete).
  int stop = 0;
  if (t == 0) {
    const int2 h = __ldcg(reinterpret_cast<const int2 *>(&ctr->error));
    stop = h.x != 0 || (h.y != 0 && h.y != F.epoch);
  }
  // The previous frame's face-normal fallback records (k_gc_normals) are
  // applied here, by the CTAs that have no pixel region (else by every CTA
  // after its regions): nothing in this kernel reads or writes what they use
  // (types, vertex coordinates, neighbour rows) and the idle warps absorb them.
  const int nreg = rx * ry, wpc = kCollectThreads / 32;
  const bool spare = (int)gridDim.x > nreg;
  if (spare && (int)blockIdx.x >= nreg) {
    if (t == 0) s_stop = stop;
    __syncthreads();
    if (s_stop) return;
  }
  if (spare && (int)blockIdx.x >= nreg) wait_prev_gc(S, F);
  if (spare && (int)blockIdx.x >= nreg)
    top_up_record_ranges(S.rec_chunk, S.rec_chunk_ctas, &ctr->a_hw, (blockIdx.x - nreg) * kCollectThreads + t,
                         ((int)gridDim.x - nreg) * kCollectThreads);
  if (F.consume_fb && spare && (int)blockIdx.x >= nreg) {
    const int nfb = min(ld_vol(&ctr->fb_pending), S.fb_cap);   // (records past the ring were applied inline)
    consume_fallbacks(FallbackArgs{S.ctr, S.fallback, S.nbr, S.bcoord, S.vparam, S.vrec, S.cube_size}, nfb,
                      (blockIdx.x - nreg) * wpc + (t >> 5), ((int)gridDim.x - nreg) * wpc, &ctr->fb_next);
  }
  int nvalid = 0, nth = 0;
  if (t == 0) s_valid = 0;
  if ((int)blockIdx.x < nreg) wait_input_flag(S, F);   // the frame's host copy has landed
  for (int reg = blockIdx.x; reg < rx * ry; reg += gridDim.x, nth++) {
    trace_item(S, TK_COLLECT, nth, 0);
    for (int q = t; q < kCSet; q += kCollectThreads) s_key[q] = kNoKey;
    if (t == 0) { s_n = 0; s_nover = 0; }
    __syncthreads();
    const int ryl = reg / rx, rx0 = reg - ryl * rx, ry0 = ry_begin + ryl;
    const int u = rx0 * kRegionW + (t & (kRegionW - 1));
    for (int pass = 0; pass < 2; pass++) {   // pass 1 only if the key set overflowed
    const bool direct = pass == 1;
    if (direct) {
      if (s_nover <= kCOver) break;   // (uniform: read after the barrier below)
      __syncthreads();
    }
    const double rxn = u < F.w ? __ldg(S.rays + u) : 0.0;
    double d[2];
    bool valid[2];
#pragma unroll
    for (int k = 0; k < 2; k++) {   // both depth loads in flight together
      const int v = ry0 * kRegionH + (t >> 6) + 4 * k;
      const long long idx = (long long)v * F.w + u;
      if (F.raw) {   // raw u16 frame: convert exactly as read_depth and keep the f64 depth
        d[k] = (u < F.w && v < F.h) ? (double)F.raw[idx] / F.depth_scale : 0.0;
        if (u < F.w && v < F.h) F.depth_out[idx] = d[k];
      } else {
        d[k] = (u < F.w && v < F.h) ? F.depth[idx] : 0.0;
      }
    }
#pragma unroll
    for (int k = 0; k < 2; k++) {
      const int v = ry0 * kRegionH + (t >> 6) + 4 * k;
      valid[k] = u < F.w && v < F.h && d[k] > 0 && d[k] <= F.max_range;
      double qs[3] = {0, 0, 0};
      if (valid[k]) {
        nvalid++;
        const double ryn = __ldg(S.rays + F.w + v);
        const double pc[3] = {__dmul_rn(rxn, d[k]), __dmul_rn(ryn, d[k]), __dmul_rn(1.0, d[k])};
        for (int j = 0; j < 3; j++) qs[j] = matvec_row(pc, F.R, j);   // pts_cam @ R.T
      }
      if (!__any_sync(0xffffffffu, valid[k])) continue;
      const double delta = valid[k] ? F.trunc / d[k] : 0.0;
      for (int i = 0; i < nsteps; i++) {
        unsigned long long key = kNoKey;
        int c[3] = {0, 0, 0};
        double pw[3];
        bool near = false;   // a coordinate within 1e-7 blocks of a block face: divide exactly
        if (valid[k]) {
          const double sv = (i == nsteps - 1) ? 1.0 : __dadd_rn(__dmul_rn((double)i, step), -1.0);
          const double f = __dadd_rn(1.0, __dmul_rn(sv, delta));
#pragma unroll
          for (int j = 0; j < 3; j++) {
            pw[j] = __dadd_rn(F.t[j], __dmul_rn(qs[j], f));
            c[j] = floor_div_fast(pw[j], S.inv_extent, near);
          }
        }
        // (warp-uniform branch: the correctly rounded divisions run only in the
        // rare warps that need them instead of predicated in every sample)
        if (__any_sync(0xffffffffu, near) && near)
#pragma unroll
          for (int j = 0; j < 3; j++) c[j] = (int)floor(pw[j] / S.extent);
        if (valid[k] && (!multi || block_relevant(S, c[0], c[1], c[2])))
          key = (unsigned long long)pack_coord(c[0], c[1], c[2]);
        if (!__any_sync(0xffffffffu, key != kNoKey)) continue;
        const unsigned grp = __match_any_sync(0xffffffffu, key);
        if (direct) {   // (rare) the set overflowed: probe the table directly
          if (key != kNoKey && lane == __ffs(grp) - 1) {
            if (emit) {
              const int at = atomicAdd(F.key_count, 1);
              if (at < F.key_cap) F.key_out[at] = key;
            } else {
              const int got = collect_block(S, F, c[0], c[1], c[2]);
              if (got >= 0) S.scope[atomicAdd(&ctr->ncollected, 1)] = got;
            }
          }
          continue;
        }
        if (key != kNoKey && lane == __ffs(grp) - 1) {
          // CTA-local set: first inserter lists the key
          unsigned h = cset_hash(key);
          bool placed = false;
          for (int probe = 0; probe < 32 && !placed; probe++, h = (h + 1) & (kCSet - 1)) {
            // (a plain read first: most probes meet the key already listed)
            unsigned long long old = *reinterpret_cast<volatile unsigned long long *>(&s_key[h]);
            if (old == kNoKey) old = atomicCAS(&s_key[h], kNoKey, key);
            if (old == kNoKey) s_list[atomicAdd(&s_n, 1)] = (uint16_t)h;
            placed = old == kNoKey || old == key;
          }
          if (!placed) {   // set crowded: the overflow list, or (full) a direct pass
            const int o = atomicAdd(&s_nover, 1);
            if (o < kCOver) s_over[o] = key;
          }
        }
      }
    }
    trace_item(S, TK_COLLECT, nth, 1);
    if (t == 0) s_stop = stop;
    __syncthreads();
    if (s_stop) return;   // (uniform; before any table write)
    trace_item(S, TK_COLLECT, nth, 2);
    // the region's distinct blocks, one thread each (+ keys that found the set
    // crowded); the newly collected ones are appended with one atomic per CTA
    const int nk = s_n, no = min(s_nover, kCOver);
    if (emit) {   // sharded band walk: list the region's distinct keys (one atomic per CTA)
      if (t == 0) s_base = atomicAdd(F.key_count, nk + no);
      __syncthreads();
      for (int q = t; q < nk + no; q += kCollectThreads)
        if (s_base + q < F.key_cap) F.key_out[s_base + q] = q < nk ? s_key[s_list[q]] : s_over[q - nk];
      __syncthreads();
      if (pass == 0) continue;
      break;
    }
    if (t == 0) s_nout = 0;
    __syncthreads();
    for (int q0 = 0; q0 < nk + no; q0 += kCollectThreads) {
      const int q = q0 + t;
      int got = -1;
      if (q < nk + no) {
        const unsigned long long key = q < nk ? s_key[s_list[q]] : s_over[q - nk];
        const long long off = 1LL << 20;
        const int x = (int)((long long)(key >> 42) - off),
                  y = (int)((long long)((key >> 21) & 0x1FFFFF) - off), z = (int)((long long)(key & 0x1FFFFF) - off);
        got = collect_block(S, F, x, y, z);
      }
      const int pos = smem_append(got >= 0, &s_nout);
      if (got >= 0) s_out[pos] = got;
    }
    __syncthreads();
    if (t == 0 && s_nout) s_base = atomicAdd(&ctr->ncollected, s_nout);
    __syncthreads();
    for (int q = t; q < s_nout; q += kCollectThreads) S.scope[s_base + q] = s_out[q];
    __syncthreads();
    if (pass == 0) continue;
    }   // pass
    __syncthreads();   // the set is reset for the next region
    trace_item(S, TK_COLLECT, nth, 3);
  }
  if (!spare) wait_prev_gc(S, F);
  if (!spare)
    top_up_record_ranges(S.rec_chunk, S.rec_chunk_ctas, &ctr->a_hw, blockIdx.x * kCollectThreads + t,
                         (int)gridDim.x * kCollectThreads);
  if (F.consume_fb && !spare) {
    const int nfb = min(ld_vol(&ctr->fb_pending), S.fb_cap);   // (records past the ring were applied inline)
    consume_fallbacks(FallbackArgs{S.ctr, S.fallback, S.nbr, S.bcoord, S.vparam, S.vrec, S.cube_size}, nfb,
                      blockIdx.x * wpc + (t >> 5), (int)gridDim.x * wpc, &ctr->fb_next);
  }

  if (F.nsteps_fixed > 0) {   // valid-pixel count (k_depth_stats did not run): one atomic per CTA
    nvalid = __reduce_add_sync(0xffffffffu, (unsigned)nvalid);
    if (lane == 0 && nvalid) atomicAdd(&s_valid, nvalid);
    __syncthreads();
    if (t == 0 && s_valid) atomicAdd(&ctr->nvalid, s_valid);
  }
  if (blockIdx.x == 0 && t == 0) ctr->nsteps = nsteps;
  trace_count(S, TK_COLLECT, nth);
  trace_span(S, 0, F.frame, true);
  trace_at(S, TK_COLLECT, 31);
}

// Sharded band walk (spatial partition): collect this rank's relevant blocks
// from the union of the ranks' key lists (k_collect with F.key_out), one key
// per thread; a block listed by several ranks / regions is collected once
// (collect_block's stamp exchange).  Appends to the scope list like k_collect.
__global__ void __launch_bounds__(256) k_collect_keys_apply(DevState S, const FrameDev F,
                                                            const unsigned long long *__restrict__ keys, int n) {
  cudaGridDependencySynchronize();
  if (halted(S)) return;
  const int lane = threadIdx.x & 31;
  for (int i0 = blockIdx.x * blockDim.x; i0 < n; i0 += gridDim.x * blockDim.x) {
    const int i = i0 + threadIdx.x;
    int got = -1;
    if (i < n) {
      const unsigned long long key = __ldg(keys + i);
      const long long off = 1LL << 20;
      const int x = (int)((long long)(key >> 42) - off), y = (int)((long long)((key >> 21) & 0x1FFFFF) - off),
                z = (int)((long long)(key & 0x1FFFFF) - off);
      // (a word that is not a packed coordinate -- the empty-slot key, say -- is never probed)
      if (!(key >> 63) && block_relevant(S, x, y, z)) got = collect_block(S, F, x, y, z);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, got >= 0);
    if (!bal) continue;
    int base = 0;
    if (lane == __ffs(bal) - 1) base = atomicAdd(&S.ctr->ncollected, __popc(bal));
    base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
    if (got >= 0) S.scope[base + __popc(bal & ((1u << lane) - 1))] = got;
  }
}

// ------------------------------------------------------------ explicit lists
__global__ void k_insert_coords(DevState S, const int3 *__restrict__ coords, int n,
                                int32_t *__restrict__ out, int epoch) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int3 c = coords[i];
    int idx = hash_find(S, c.x, c.y, c.z);
    if (idx == -1) idx = hash_insert(S, c.x, c.y, c.z, epoch);
    out[i] = idx;
  }
}

__global__ void k_lookup_coords(DevState S, const int3 *__restrict__ coords, int n,
                                int32_t *__restrict__ out, int32_t *stamp, int32_t epoch) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int3 c = coords[i];
    const int idx = hash_find(S, c.x, c.y, c.z);
    out[i] = idx;
    if (stamp && idx >= 0) stamp[idx] = epoch;
  }
}

// ------------------------------------------------------------ block init
// Block.empty (store.py:70-81) + 26-neighbour links.  One CTA per block.
__device__ __forceinline__ void init_block(const DevState &S, int b, int t) {
  S.tsdf[(size_t)b * kNC + t] = 0.0;
  S.weight[(size_t)b * kNC + t] = 0;
  S.tp[(size_t)b * kNC + t] = 0;
  S.tc[(size_t)b * kNC + t] = 0;
  // (the slots' vertex records stay: a reused block index keeps its handles)
  if (t < kEV / 32) {
    S.vocc[(size_t)b * (kEV / 32) + t] = 0u;
    S.vclaim[(size_t)b * (kEV / 32) + t] = 0u;
  }
}

__global__ void __launch_bounds__(kThreadsCube) k_init_blocks(DevState S, int epoch) {
  if (halted(S)) return;
  // the blocks allocated by this call (stamp_new == epoch), phase API only
  const int nb_all = ld_vol(&S.ctr->nblocks);
  for (int b = blockIdx.x; b < nb_all; b += gridDim.x) {
    if (__ldcg(S.stamp_new + b) != epoch) continue;
    init_block(S, b, threadIdx.x);
    if (threadIdx.x < kNC / 32) S.vmask[(size_t)b * (kNC / 32) + threadIdx.x] = 0u;
    if (threadIdx.x < 27) {
      const int t = threadIdx.x;
      const int4 c = S.bcoord[b];
      const int y = (t == 13) ? b : hash_find(S, c.x + t / 9 - 1, c.y + (t / 3) % 3 - 1, c.z + t % 3 - 1);
      S.nbr[(size_t)b * 27 + t] = y;
      if (y >= 0 && t != 13) S.nbr[(size_t)y * 27 + (26 - t)] = b;
    }
  }
}

// ------------------------------------------------------------ fuse blocks
// One CTA per collected block, one thread per corner:
//  F_INIT      blocks allocated this call are initialised and linked;
//  F_INTEGRATE TSDF running average (fusion.py:138-168);
//  F_SCOPE     minus-slab scope marking (mesher.py:499-527)
//  F_HALO      27-neighbour halo marking (mesher.py:530-543; in fuse_frame
//              the halo is marked by k_retype_place instead)
//              (mesher.py:499-543), with hash lookups (links of blocks
//              created in this launch are still being written).
constexpr int kFB = 128;   // threads per CTA of k_fuse_blocks (4 corners each)

// F_GHOST (halo exchange): items [base, n) are margin blocks received from
// their owners; their samples are copied from the records instead of integrated.
__global__ void __launch_bounds__(kFB, 6) k_fuse_blocks(DevState S, const FrameDev F,
                                                     const int32_t *__restrict__ list,
                                                     const int32_t *__restrict__ count_ptr,
                                                     int count_const, int flags, int base = 0) {
  cudaGridDependencySynchronize();   // PDL: wait for the previous kernel of the frame
  trace_at(S, TK_FUSE, 0);
  trace_span(S, 1, F.frame, false);
  __shared__ int s_pro[5];
  const int list_cap = count_ptr ? S.max_blocks : count_const;
  read_prologue(S, s_pro, count_ptr, nullptr, nullptr,
                base + (int)blockIdx.x < list_cap ? list + base + blockIdx.x : nullptr);
  if (s_pro[0]) return;
  const int n = count_ptr ? s_pro[1] : count_const;
  if (F.consume_fb && blockIdx.x == 0 && threadIdx.x == 0) S.ctr->fb_pending = 0;   // (k_collect applied them)
  trace_at(S, TK_FUSE, 1);
  int nth = 0;
  const int t = threadIdx.x;
  // neighbour probe of this thread: 7 lanes of each warp, directions 0..26
  const int pl = t & 31, pdir = (t >> 5) * 7 + pl;
  const bool prober = pl < 7 && pdir < 27;
  // the item list entry of the CTA's next item is requested one item ahead
  int b_next = (base + (int)blockIdx.x < n) ? s_pro[4] : -1;
  if (b_next == -1 && base + (int)blockIdx.x < n) b_next = __ldcg(list + base + blockIdx.x);
  for (int i = base + blockIdx.x; i < n; i += gridDim.x, nth++) {
    trace_item(S, TK_FUSE, nth, 0);
    const int b = b_next;
    b_next = i + (int)gridDim.x < n ? __ldcg(list + i + gridDim.x) : -1;
    if (b < 0) continue;
    const int4 c = __ldcg(S.bcoord + b);
    const bool fresh = (flags & F_INIT) && __ldcg(S.stamp_new + b) == F.epoch;
    if ((flags & (F_INTEGRATE | F_GHOST)) && threadIdx.x == 0) S.last_frame[b] = F.frame;   // (block GC)
    // fusion.py:138-168, four corners per thread.  The old state of the corners
    // is requested first, so its round trip overlaps the projections and the
    // depth gathers.
    double t_old[kNC / kFB], zc[kNC / kFB], meas[kNC / kFB];
    int w_old[kNC / kFB];
    bool ok[kNC / kFB];
    if (flags & F_INTEGRATE) {
#pragma unroll
      for (int j = 0; j < kNC / kFB; j++) {
        // (requested before `fresh` is known: a new block's storage is read and
        // ignored, so the loads need not wait for its stamp)
        const size_t q = (size_t)b * kNC + t + j * kFB;
        const double tv = S.tsdf[q];
        const int wv = S.weight[q];
        t_old[j] = fresh ? 0.0 : tv;
        w_old[j] = fresh ? 0 : wv;
      }
      const double bx = __dmul_rn((double)c.x, S.extent), by = __dmul_rn((double)c.y, S.extent),
                   bz = __dmul_rn((double)c.z, S.extent);
#pragma unroll
      for (int j = 0; j < kNC / kFB; j++) {
        const int ci = t + j * kFB;
        double a[3];
        a[0] = __dadd_rn(bx, __dmul_rn((double)(ci >> 6), S.cube_size)) - F.t[0];
        a[1] = __dadd_rn(by, __dmul_rn((double)((ci >> 3) & 7), S.cube_size)) - F.t[1];
        a[2] = __dadd_rn(bz, __dmul_rn((double)(ci & 7), S.cube_size)) - F.t[2];
        const double z = matvec_col(a, F.R, 2);
        zc[j] = z;
        ok[j] = false;
        meas[j] = 0.0;
        if (!(z > 0)) continue;
        const double x = matvec_col(a, F.R, 0), y = matvec_col(a, F.R, 1);
        const double u = rint(__dadd_rn(__dmul_rn(F.fx, x) / z, F.cx));
        const double v = rint(__dadd_rn(__dmul_rn(F.fy, y) / z, F.cy));
        if (!(u >= 0 && u < (double)F.w && v >= 0 && v < (double)F.h)) continue;
        ok[j] = true;
        meas[j] = F.depth[(long long)v * F.w + (long long)u];
      }
    }
    if (fresh)
#pragma unroll
      for (int j = 0; j < kNC / kFB; j++) init_block(S, b, t + j * kFB);
    const int dx = pdir / 9 - 1, dy = (pdir / 3) % 3 - 1, dz = pdir % 3 - 1;
    const bool minus = dx <= 0 && dy <= 0 && dz <= 0 && pdir != 13;
    // probes: all 27 to link a new block or to mark the halo (F_HALO); else
    // only the 7 minus directions (slab scope items)
    if (prober && ((fresh && (flags & F_INIT)) || (flags & F_HALO) || ((flags & F_SCOPE) && minus))) {
      int nb = b, nb_collected = 1;
      if (pdir != 13) {
        if (fresh) {   // its links are built here, from the table
          const HashRef r = hash_find_ref(S, c.x + dx, c.y + dy, c.z + dz);
          nb = r.idx;
          nb_collected = r.stamp == F.epoch;
        } else {
          // an older block's row is complete except for neighbours created in
          // this call, which are collected and mark themselves
          nb = __ldcg(S.nbr + (size_t)b * 27 + pdir);
          nb_collected = nb >= 0 && __ldcg(S.stamp_collect + nb) == F.epoch;
        }
      }
      if (fresh) {
        S.nbr[(size_t)b * 27 + pdir] = nb;
        if (nb >= 0 && pdir != 13) S.nbr[(size_t)nb * 27 + (26 - pdir)] = b;
      }
      if ((flags & F_HALO) && nb >= 0) {
        if (ld_vol(S.stamp_halo + nb) != F.epoch && atomicExch(S.stamp_halo + nb, F.epoch) != F.epoch)
          S.halo[atomicAdd(&S.ctr->nhalo, 1)] = nb;
      }
      // minus neighbour n = c - o, o in {0,1}^3 \ 0, not itself collected
      if ((flags & F_SCOPE) && nb >= 0 && minus && !nb_collected) {
        const int o = (-dx) * 4 + (-dy) * 2 + (-dz);
        const unsigned sh = 8 * (nb & 3);
        const unsigned old = atomicOr((unsigned *)(S.slab_bits + (nb & ~3)), (1u << (o - 1)) << sh);
        if (((old >> sh) & 0xFF) == 0) S.scope[n + atomicAdd(&S.ctr->nslab, 1)] = nb;   // (n = collected)
      }
    }
    if (flags & F_GHOST) {   // the owner's samples, as integrated there (bit-identical)
      const uint8_t *rec = F.ghost_recv + (size_t)__ldcg(S.ghost_src + i) * kGhostRec;
      const double *gt = reinterpret_cast<const double *>(rec + 16);
      const int32_t *gw = reinterpret_cast<const int32_t *>(rec + 16 + 8 * kNC);
#pragma unroll
      for (int j = 0; j < kNC / kFB; j++) {
        const int ci = t + j * kFB;
        const double tv = __ldcg(gt + ci);
        const int32_t wv = __ldcg(gw + ci);
        S.tsdf[(size_t)b * kNC + ci] = tv;
        S.weight[(size_t)b * kNC + ci] = wv;
        const unsigned vb = __ballot_sync(0xffffffffu, wv > 0);
        if ((threadIdx.x & 31) == 0) S.vmask[(size_t)b * (kNC / 32) + (ci >> 5)] = vb;
      }
      continue;
    }
    if (!(flags & F_INTEGRATE)) continue;
#pragma unroll
    for (int j = 0; j < kNC / kFB; j++) {
      bool upd = ok[j] && meas[j] > 0 && meas[j] <= F.max_range && meas[j] - zc[j] >= -F.trunc;
      // validity bitmap: a warp's 32 lanes hold 32 consecutive corners (one word)
      const unsigned vb = __ballot_sync(0xffffffffu, upd && (fresh || w_old[j] == 0));
      if ((threadIdx.x & 31) == 0) {
        uint32_t *wp = S.vmask + (size_t)b * (kNC / 32) + ((t + j * kFB) >> 5);
        if (fresh) *wp = vb;                 // (a new block's words are written whole)
        else if (vb) atomicOr(wp, vb);
      }
      if (!upd) continue;
      const double m = meas[j];
      const double sdf = m - zc[j];
      double dn = sdf / F.trunc;
      dn = dn < -1.0 ? -1.0 : (dn > 1.0 ? 1.0 : dn);
      const size_t q = (size_t)b * kNC + t + j * kFB;
      const double wo = (double)w_old[j];
      S.tsdf[q] = __dadd_rn(__dmul_rn(wo, t_old[j]), dn) / __dadd_rn(wo, 1.0);
      const long long nw = (long long)w_old[j] + 1;
      S.weight[q] = (int)(nw < F.weight_cap ? nw : F.weight_cap);
    }
    trace_item(S, TK_FUSE, nth, 3);
  }
  trace_count(S, TK_FUSE, nth);
  trace_span(S, 1, F.frame, true);
  trace_at(S, TK_FUSE, 31);
}

// halo of an explicit scope (extract_frame default, mesher.py:627-633)
__global__ void k_halo_from_items(DevState S, const FrameDev F) {
  if (halted(S)) return;
  const int epoch = F.epoch;
  const int ni = ld_vol(&S.ctr->nexplicit);
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < (long long)ni * 27;
       t += (long long)gridDim.x * blockDim.x) {
    const int c = S.scope[t / 27];
    if (c < 0) continue;
    const int n = S.nbr[(size_t)c * 27 + (int)(t % 27)];
    if (n < 0) continue;
    if (ld_vol(S.stamp_halo + n) != epoch && atomicExch(S.stamp_halo + n, epoch) != epoch)
      S.halo[atomicAdd(&S.ctr->nhalo, 1)] = n;
  }
}

__global__ void k_clear_slabs(DevState S, int nc, int ns) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x)
    S.slab_bits[S.scope[nc + i]] = 0;
}

// ------------------------------------------------------------ retype + place
// Per-item "resolved" record: the item's block, neighbour row and selection mode
struct Resolved {
  int4 coord;
  int nbr[27];
  int b, mode, slab, item;   // mode: -1 past the end, 0 skip, 1 full, 2 slab bits, 3 explicit mask
  int owned;                 // counters only accumulate over blocks this rank owns
};

// registers warp 0 carries while the loads of a future item are in flight
struct ResolveRegs {
  int v;       // lanes 0..26: neighbour row entry; lane 27: slab bits
  int4 coord;  // lane 28
};

__device__ __forceinline__ ResolveRegs resolve_load(const DevState &S, const FrameDev &F, int b, int item,
                                                    int nc) {
  const int lane = threadIdx.x & 31;
  ResolveRegs r;
  r.v = -1;
  r.coord = make_int4(0, 0, 0, 0);
  if (b >= 0) {
    if (lane < 27) r.v = lane == 13 ? b : __ldcg(S.nbr + (size_t)b * 27 + lane);
    else if (lane == 27) r.v = (F.scope_mode == 0 && item >= nc) ? __ldcg(S.slab_bits + b) : 0;
    else if (lane == 28) r.coord = __ldcg(S.bcoord + b);
  }
  return r;
}

__device__ __forceinline__ void resolve_store(const DevState &S, const FrameDev &F, const ResolveRegs &r,
                                              int b, int item, int n, int nc, Resolved &R) {
  const int lane = threadIdx.x & 31;
  if (lane < 27) R.nbr[lane] = r.v;
  const int slab = __shfl_sync(0xffffffffu, r.v, 27);
  int4 c;
  c.x = __shfl_sync(0xffffffffu, r.coord.x, 28);
  c.y = __shfl_sync(0xffffffffu, r.coord.y, 28);
  c.z = __shfl_sync(0xffffffffu, r.coord.z, 28);
  c.w = 0;
  if (lane == 27) {
    int mode;
    if (item >= n) mode = -1;
    else if (b < 0) mode = 0;
    else if (F.scope_mode == 1) mode = 3;
    else if (item < nc) mode = 1;
    else { mode = 2; S.slab_bits[b] = 0; }   // slab consumed: clear for the next frame
    if (mode > 0 && F.frustum_only && !block_in_frustum_dev(c, F, S.extent)) mode = 0;
    R.mode = mode;
    R.b = b;
    R.slab = slab;
    R.item = item;
    R.coord = c;
    R.owned = (b >= 0 && S.nranks > 1) ? __ldcg(S.bowned + b) : 1;
  }
}

constexpr int kNT = 64;   // threads per CTA of k_retype_place (one tile column each)
constexpr int kTileSlots = 729 * 3;   // edge slots owned by the 9^3 tile points (3 axes each)


// position q < 217 of the (B+1)^3 tile's plus layer (points with a coordinate
// == 8): tile point, neighbour direction and source sample (mesher.py:75-96)
__device__ __forceinline__ void ext_src(int q, int &p, int &dir, int &src) {
  int x, y, z;
  if (q < 64) { x = 8; y = q >> 3; z = q & 7; }
  else if (q < 128) { x = (q - 64) >> 3; y = 8; z = q & 7; }
  else if (q < 192) { x = (q - 128) >> 3; y = q & 7; z = 8; }
  else if (q < 200) { x = 8; y = 8; z = q - 192; }
  else if (q < 208) { x = 8; y = q - 200; z = 8; }
  else if (q < 216) { x = q - 208; y = 8; z = 8; }
  else { x = 8; y = 8; z = 8; }
  p = (x * 9 + y) * 9 + z;
  dir = ((x >> 3) + 1) * 9 + ((y >> 3) + 1) * 3 + ((z >> 3) + 1);
  src = (x & 7) * 64 + (y & 7) * 8 + (z & 7);
}

// Corner bytes of the 4 cubes z0..z0+3 of a column, bit plane starting at bit
// `sh` of the 4 column words of the (x, y) footprint: byte j holds cube
// z0 + j's 8 corner bits in CORNER_OFFSETS order (mc_tables.py:31-34:
// (0,0,0) (1,0,0) (1,1,0) (0,1,0), then the same at z + 1).  spread4 moves
// 4 bits to the low bit of 4 bytes (one multiply, no carries).
// position of the k-th (0-based) set bit of m (k < popc(m)), branch-free
__device__ __forceinline__ int select_bit(uint32_t m, int k) {
  int p = 0, c;
  c = __popc(m & 0xFFFFu);         if (k >= c) { k -= c; p = 16; }
  c = __popc((m >> p) & 0xFFu);    if (k >= c) { k -= c; p += 8; }
  c = __popc((m >> p) & 0xFu);     if (k >= c) { k -= c; p += 4; }
  c = __popc((m >> p) & 0x3u);     if (k >= c) { k -= c; p += 2; }
  c = (int)((m >> p) & 1u);        if (k >= c) p += 1;
  return p;
}

// bit z (z < 9) -> bit 3 z
__device__ __forceinline__ uint32_t part1by2_9(uint32_t x) {
  x &= 0x1FFu;
  x = (x | (x << 16)) & 0x030000FFu;
  x = (x | (x << 8)) & 0x0300F00Fu;
  x = (x | (x << 4)) & 0x030C30C3u;
  return (x | (x << 2)) & 0x09249249u;
}
__device__ __forceinline__ uint32_t spread4(uint32_t v) { return ((v & 0xFu) * 0x00204081u) & 0x01010101u; }
__device__ __forceinline__ uint32_t corner_bytes4(const uint32_t (&w)[4], int sh) {
  uint32_t r = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) r |= (spread4(w[k] >> sh) << k) | (spread4(w[k] >> (sh + 1)) << (k + 4));
  return r;
}

// One CTA of 128 threads per scope item (persistent over the item list).
//  * stage: the block's tsdf/weight/types and the plus layer of its 7 plus
//    neighbours (mesher.py:75-96); the corner predicates (tsdf < 0, weight > 0,
//    |tsdf| < eps) are packed with warp ballots into one 27-bit word per tile
//    column (x, y) -- bit z, 9 + z, 18 + z;
//  * typing (+ Hamming refinement), one thread per 4-cube run of a column:
//    8 corner bits from 4 column words (mesher.py:111-134, refine.py:98-135);
//    a cube whose type changed is retriangulated implicitly (its triangles
//    become TRI_TABLE[type_curr], mesher.py:283-326) and contributes the
//    triangle / irregular-count deltas;
//  * placement (mesher.py:178-257): the requested edge slots are deduplicated
//    in a shared-memory bitmap (all requesters of a slot write identical bits),
//    then each is claimed (atomicCAS on its birth word -- exactly one
//    allocation per edge) and its coordinate written.
__global__ void __launch_bounds__(kNT, 18) k_retype_place(DevState S, const FrameDev F) {
  cudaGridDependencySynchronize();   // PDL: wait for the previous kernel of the frame
  trace_at(S, TK_RETYPE, 0);
  trace_span(S, 2, F.frame, false);
  // Prologue, one thread, every load in one round trip: the halt flags, the
  // item counts, the CTA's first scope entry, and the vertex-record capacity
  // check -- this frame can give at most kRecsPerItem records per scope item
  // (and never more than the stored blocks have slots).  Every CTA reads the
  // same counters and takes the same decision; on a shortfall the frame stops
  // here and the host grows the record arena and resumes it at this kernel
  // (need_stage 1) -- before anything is written.
  __shared__ int s_pro[5];
  __shared__ int s_halt;
  if (threadIdx.x == 0) {
    // (4 requests on the counter block's lines: every CTA of the grid makes them)
    // (through L1, see read_prologue: nothing read here changes during the kernel --
    // a CTA that raises need below makes every CTA take the same decision)
    const Counters *c = S.ctr;
    const int4 hd = __ldg(reinterpret_cast<const int4 *>(c));             // nblocks, ovf, error, need
    const int4 cw = __ldg(reinterpret_cast<const int4 *>(&c->nvalid));    // nvalid, nsteps, ncollected, nnew
    const int4 it = __ldg(reinterpret_cast<const int4 *>(&c->nslab));     // nslab, nexplicit, nitems_live, nhalo
    const int first = (int)blockIdx.x < S.max_blocks ? __ldcg(S.scope + blockIdx.x) : -1;
    const long long hw = (long long)__ldg(reinterpret_cast<const unsigned long long *>(&c->a_hw));
    const int nbl = hd.x, nc0 = cw.z, ns0 = it.x, ne0 = it.y;
    int halt = (hd.z | hd.w) != 0;
    s_pro[0] = halt; s_pro[1] = nc0; s_pro[2] = ns0; s_pro[3] = ne0; s_pro[4] = first;
    if (!halt) {
      const long long items = F.scope_mode != 0 ? ne0 : (long long)nc0 + ns0;
      const long long bound = min(kRecsPerItem * items, (long long)kEV * nbl);
      if (hw + bound + 4 * kRecChunk * S.rec_chunk_ctas > S.vrec_cap) {   // (+ the gc CTAs' record ranges)
        halt = 1;
        S.ctr->need_stage = 1;
        atomicExch(&S.ctr->need, F.epoch);
      }
    }
    s_halt = halt;
  }
  __syncthreads();
  if (s_halt) return;
  // meshing starts here: every k_fuse_blocks CTA has completed (engine.py:127-156's split)
  if (blockIdx.x == 0 && threadIdx.x == 0) S.ctr->t_mesh_ns = gtimer();
  const int nc = s_pro[1];
  const int n = F.scope_mode != 0 ? s_pro[3] : nc + s_pro[2];
  trace_at(S, TK_RETYPE, 1);
  int nth = 0;
  __shared__ double tile[729];
  __shared__ uint32_t s_col[81];    // tile column x*9+y: sign bits 0..7, valid 9..16, small 18..25
  __shared__ uint8_t s_top[81];     // its z = 8 point: bit 0 sign, 2 small
  // typing inputs, reused by the placement as per-warp slot lists
  __shared__ union __align__(16) {
    struct {
      uint32_t vm8[8 * 16];   // weight > 0 bitmaps: block + 7 plus-neighbours
      uint8_t tc[kNC], tp[kNC];
    } ty;
  } U;
  uint32_t *const s_vm8 = U.ty.vm8;
  uint8_t *const s_tc = U.ty.tc, *const s_tp = U.ty.tp;
  __shared__ uint32_t s_claim[3 * 81];   // requested slots: [axis][tile column], bit = owner z
  __shared__ uint32_t s_mcol[81];        // placement: a column's requested slots (bit 3 z + axis)
  __shared__ int s_pre[82];              //   and the exclusive prefix of their counts
  __shared__ Resolved R;
  const int t = threadIdx.x, lane = t & 31;
  const double l = S.cube_size;
  const int do_refine = F.refine;
  const double eps = F.epsilon;
  const bool part = F.strategy == 2;   // placement by k_place_parity: record the selection instead
  int placements = 0, active = 0, changed = 0, t_rel = 0, t_new = 0, irr = 0, refined = 0, live = 0;
  for (int i = blockIdx.x; i < n; i += gridDim.x, nth++) {
    trace_item(S, TK_RETYPE, nth, 0);
    if (t < 32) {
      const int b = i == (int)blockIdx.x && s_pro[4] != -1 ? s_pro[4] : __ldcg(S.scope + i);
      const ResolveRegs rr = resolve_load(S, F, b, i, nc);
      resolve_store(S, F, rr, b, i, n, nc, R);
    }
    for (int q = t; q < 3 * 81; q += kNT) s_claim[q] = 0;
    __syncthreads();
    trace_item(S, TK_RETYPE, nth, 1);
    const int mode = R.mode;
    // fused_halo (mesher.py:530-543): a collected item marks its 27-neighbourhood
    // (frustum-culled ones too).  The exchanges are issued after the tile loads
    // below and their results consumed only at the end of the item, where the
    // first markers are appended to the halo list with one atomic per warp (a
    // single hot counter: an append on the critical path queued behind every
    // other CTA's)
    const bool halo_item = F.scope_mode == 0 && i < nc && R.b >= 0 && t < 27;
    int h_nb = -1, h_old = F.epoch;
    auto mark_halo = [&]() {
      if (!halo_item) return;
      h_nb = R.nbr[t];
      if (h_nb >= 0) h_old = atomicExch(S.stamp_halo + h_nb, F.epoch);
    };
    auto append_halo = [&]() {
      if (t >= 32) return;
      const bool nw = h_nb >= 0 && h_old != F.epoch;
      const unsigned bal = __ballot_sync(0xffffffffu, nw);
      if (!bal) return;
      const int cnt = __popc(bal), r = __popc(bal & ((1u << t) - 1));
      const int k = blockIdx.x & (kHaloShards - 1);
      int base = 0;
      if (t == 0) base = atomicAdd(&S.ctr->nhalo_sh[k], cnt);
      base = __shfl_sync(0xffffffffu, base, 0);
      const int room = max(0, S.halo_sh_cap - base);
      int obase = 0;
      if (room < cnt) {   // (uniform) the shard is full: the rest go to the general list
        if (t == 0) obase = atomicAdd(&S.ctr->nhalo, cnt - room);
        obase = __shfl_sync(0xffffffffu, obase, 0);
      }
      if (nw) {
        if (r < room) S.halo_sh[(size_t)k * S.halo_sh_cap + base + r] = h_nb;
        else S.halo[obase + r - room] = h_nb;
      }
    };
    if (mode <= 0) {
      if (part) S.psel[(size_t)i * 64 + t] = 0;
      mark_halo();
      append_halo();
      __syncthreads();
      continue;
    }
    const int b = R.b;
    const int own = R.owned;
    if (t == 0) live++;
    {
      // batched gathers: all loads in flight before any shared-memory store
      constexpr int kOwn = kNC / kNT, kExt = (217 + kNT - 1) / kNT;
      double ov[kOwn], xv[kExt];
      int xp[kExt];
      uint4 tcv = make_uint4(0, 0, 0, 0);
      if (t < 32) {   // weight > 0 bitmaps of the block and its 7 plus-neighbours (o = dx*4+dy*2+dz)
        const int o = t >> 2;
        const int nb = R.nbr[nbr_dir(o >> 2, (o >> 1) & 1, o & 1)];
        cp_async16(&s_vm8[t * 4], S.vmask + (size_t)(nb >= 0 ? nb : 0) * (kNC / 32) + (t & 3) * 4, nb >= 0);
      }
#pragma unroll
      for (int j = 0; j < kOwn; j++) ov[j] = S.tsdf[(size_t)b * kNC + t + j * kNT];
      tcv = t < 32 ? reinterpret_cast<const uint4 *>(S.tc + (size_t)b * kNC)[t]
                   : reinterpret_cast<const uint4 *>(S.tp + (size_t)b * kNC)[t - 32];
#pragma unroll
      for (int j = 0; j < kExt; j++) {
        const int q = t + j * kNT;
        xv[j] = 0.0;
        xp[j] = -1;
        if (q < 217) {
          int dir, src;
          ext_src(q, xp[j], dir, src);
          const int nb = R.nbr[dir];
          if (nb >= 0) xv[j] = S.tsdf[(size_t)nb * kNC + src];
        }
      }
      mark_halo();
      // own samples: lanes 8g..8g+7 hold z = 0..7 of one column
      const int g8 = (lane >> 3) * 8;
#pragma unroll
      for (int j = 0; j < kOwn; j++) {
        const int c = t + j * kNT;
        const int col = (c >> 6) * 9 + ((c >> 3) & 7);
        tile[col * 9 + (c & 7)] = ov[j];
        const unsigned bs = __ballot_sync(0xffffffffu, ov[j] < 0.0);
        const unsigned bm = __ballot_sync(0xffffffffu, fabs(ov[j]) < eps);
        if ((lane & 7) == 0) s_col[col] = ((bs >> g8) & 0xFFu) | (((bm >> g8) & 0xFFu) << 18);
      }
      reinterpret_cast<uint4 *>(t < 32 ? s_tc : s_tp)[t & 31] = tcv;
      cp_async_wait_all();
      // plus layer: q < 128 are the x = 8 and y = 8 faces (z = 0..7 runs of a
      // column), q = 192..199 the column (8, 8); the rest are z = 8 points
#pragma unroll
      for (int j = 0; j < kExt; j++) {
        const int q = t + j * kNT;
        const bool run = q < 128 || (q >= 192 && q < 200);
        const unsigned bs = __ballot_sync(0xffffffffu, xv[j] < 0.0);
        const unsigned bm = __ballot_sync(0xffffffffu, fabs(xv[j]) < eps);
        if (xp[j] >= 0) {
          tile[xp[j]] = xv[j];
          const int col = xp[j] / 9;
          if (run) {
            if ((lane & 7) == 0) s_col[col] = ((bs >> g8) & 0xFFu) | (((bm >> g8) & 0xFFu) << 18);
          } else {
            s_top[col] = (uint8_t)((xv[j] < 0.0) | ((fabs(xv[j]) < eps) << 2));
          }
        }
      }
    }
    __syncthreads();
    trace_item(S, TK_RETYPE, nth, 2);
    // typing: thread t -> tile column (x, y) = (t >> 3, t & 7), its 8 cubes.
    // The corner bytes of 4 cubes at a time are formed bit-sliced: byte j of a
    // plane word holds the 8 corner bits of cube z0 + j.
    {
      const int x = t >> 3, y = t & 7;
      uint32_t w[4];
      const int cols[4] = {x * 9 + y, (x + 1) * 9 + y, (x + 1) * 9 + y + 1, x * 9 + y + 1};
      const int cx[4] = {x, x + 1, x + 1, x}, cy[4] = {y, y, y + 1, y + 1};
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const uint32_t tp8 = s_top[cols[k]];
        // weight > 0 of the column's 9 points from the bitmaps: z = 0..7 are one
        // byte of block (X>>3, Y>>3, 0), z = 8 one bit of block (X>>3, Y>>3, 1)
        const int ob = ((cx[k] >> 3) << 2) | ((cy[k] >> 3) << 1);
        const int c0 = (cx[k] & 7) * 64 + (cy[k] & 7) * 8;
        const uint32_t val9 = ((s_vm8[ob * 16 + (c0 >> 5)] >> (c0 & 31)) & 0xFFu) |
                              (((s_vm8[(ob | 1) * 16 + (c0 >> 5)] >> (c0 & 31)) & 1u) << 8);
        w[k] = s_col[cols[k]] | ((tp8 & 1u) << 8) | (val9 << 9) | (((tp8 >> 2) & 1u) << 26);
      }
      uint32_t cxa = 0, cxb = 0, cya = 0, cyb = 0, cza = 0, czb = 0, czc = 0, czd = 0;
      if (!do_refine) {
        // Without refinement a cube's type is its corner signs and its edge
        // mask their sign changes (edge_mask_of), so the column's 8 cubes are
        // typed word-parallel: bit z of every word below is cube z (or owner
        // height z).  Selected cubes (scope rule, all 8 weights > 0):
        uint32_t sel;
        if (mode == 1) {
          sel = 0xFFu;
        } else if (mode == 2) {
          const int sb = ((x == 7) << 2) | ((y == 7) << 1);
          sel = ((R.slab & c_slab_sel[sb]) ? 0x7Fu : 0u) | ((R.slab & c_slab_sel[sb | 1]) ? 0x80u : 0u);
        } else {
          const int c0 = (x * 8 + y) * 8;
          sel = (S.item_mask[(size_t)R.item * 16 + (c0 >> 5)] >> (c0 & 31)) & 0xFFu;
        }
        const uint32_t vall = ((w[0] & w[1] & w[2] & w[3]) >> 9) & 0x1FFu;   // points z with 4 weights > 0
        sel &= vall & (vall >> 1);
        if (part) S.psel[(size_t)i * 64 + t] = (uint8_t)sel;
        const uint32_t sg0 = w[0] & 0x1FFu, sg1 = w[1] & 0x1FFu, sg2 = w[2] & 0x1FFu, sg3 = w[3] & 0x1FFu;
        // sign changes along the cube edges (mc_tables.py:44-64): e0/e4 between
        // corners 0-1 at z / z + 1, e1/e5 1-2, e2/e6 3-2, e3/e7 0-3, e8..e11 the
        // verticals of corners 0..3
        const uint32_t d01 = sg0 ^ sg1, d12 = sg1 ^ sg2, d32 = sg3 ^ sg2, d03 = sg0 ^ sg3;
        const uint32_t z0m = (sg0 ^ (sg0 >> 1)) & 0xFFu, z1m = (sg1 ^ (sg1 >> 1)) & 0xFFu,
                       z2m = (sg2 ^ (sg2 >> 1)) & 0xFFu, z3m = (sg3 ^ (sg3 >> 1)) & 0xFFu;
        const uint32_t sel2 = sel | (sel << 1);   // owner heights of the e0..e7 slots: z and z + 1
        cxa = d01 & sel2;   // e0, e4: (x, y)
        cxb = d32 & sel2;   // e2, e6: (x, y+1)
        cya = d12 & sel2;   // e1, e5: (x+1, y)
        cyb = d03 & sel2;   // e3, e7: (x, y)
        cza = z0m & sel;    // e8: (x, y)
        czb = z1m & sel;    // e9: (x+1, y)
        czc = z2m & sel;    // e10: (x+1, y+1)
        czd = z3m & sel;    // e11: (x, y+1)
        if (own) {
          const uint32_t hz = d01 | d12 | d32 | d03;
          const uint32_t nonuni = (hz | (hz >> 1) | z0m | z1m | z2m | z3m) & 0xFFu;   // type not 0 / 0xFF
          active += __popc(nonuni & sel);
          placements += __popc(d01 & sel) + __popc(d01 & (sel << 1)) + __popc(d32 & sel) +
                        __popc(d32 & (sel << 1)) + __popc(d12 & sel) + __popc(d12 & (sel << 1)) +
                        __popc(d03 & sel) + __popc(d03 & (sel << 1)) + __popc(cza) + __popc(czb) +
                        __popc(czc) + __popc(czd);
        }
#pragma unroll
        for (int half = 0; half < 2; half++) {
          const int z0 = 4 * half;
          const uint32_t tcw = corner_bytes4(w, z0);   // the 4 cubes' new types
          const uint32_t m = spread4(sel >> z0) * 0xFFu;
          const int c0 = (x * 8 + y) * 8 + z0;
          const uint32_t old_tc = reinterpret_cast<const uint32_t *>(s_tc)[c0 >> 2];
          const uint32_t old_tp = reinterpret_cast<const uint32_t *>(s_tp)[c0 >> 2];
          const uint32_t new_tp = (old_tp & ~m) | (old_tc & m), new_tc = (old_tc & ~m) | (tcw & m);
          if (own)   // changed cubes (type_curr != type_prev): their triangle deltas
            for (uint32_t ch = __vcmpne4(tcw, old_tc) & m; ch;) {
              const int sh = (__ffs(ch) - 1) & ~7;
              ch &= ~(0xFFu << sh);
              const unsigned tp = (old_tc >> sh) & 0xFFu, tc = (tcw >> sh) & 0xFFu;
              changed++;
              const int nold = __ldg(g_tri_count + tp), nnew = __ldg(g_tri_count + tc);
              t_rel += nold;
              t_new += nnew;
              irr += (nnew > 0 && !is_regular_type(tc)) - (nold > 0 && !is_regular_type(tp));
            }
          if (new_tc != old_tc || new_tp != old_tp) {   // 4 cubes per 32-bit store
            const size_t q4 = ((size_t)b * kNC + c0) >> 2;
            reinterpret_cast<uint32_t *>(S.tp)[q4] = new_tp;
            reinterpret_cast<uint32_t *>(S.tc)[q4] = new_tc;
          }
        }
      } else {
      uint32_t selb = 0;   // (partition: the column's selected cubes)
#pragma unroll
      for (int half = 0; half < 2; half++) {
        const int z0 = 4 * half;
        const uint32_t sgn = corner_bytes4(w, z0), val = corner_bytes4(w, 9 + z0);
        const uint32_t sml = do_refine ? corner_bytes4(w, 18 + z0) : 0u;
        const int c0 = (x * 8 + y) * 8 + z0;
        const uint32_t old_tc = reinterpret_cast<const uint32_t *>(s_tc)[c0 >> 2];
        const uint32_t old_tp = reinterpret_cast<const uint32_t *>(s_tp)[c0 >> 2];
        uint32_t new_tc = old_tc, new_tp = old_tp;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          const int z = z0 + k;
          const int c = c0 + k;
          bool sel;
          if (mode == 1) sel = true;
          else if (mode == 2) sel = (R.slab & c_slab_sel[((x == 7) << 2) | ((y == 7) << 1) | (z == 7)]) != 0;
          else sel = (S.item_mask[(size_t)R.item * 16 + (c >> 5)] >> (c & 31)) & 1;
          sel = sel && ((val >> (8 * k)) & 0xFFu) == 0xFFu;   // all 8 weights > 0
          if (!sel) continue;
          selb |= 1u << z;
          const unsigned bits = (sgn >> (8 * k)) & 0xFFu;
          const unsigned tp = (old_tc >> (8 * k)) & 0xFFu;
          unsigned tc = bits;
          if (do_refine) {
            bool ch;
            tc = refine_type(bits, tp, (sml >> (8 * k)) & 0xFFu, &ch);
            refined += ch && own;
          }
          new_tp = (new_tp & ~(0xFFu << (8 * k))) | (tp << (8 * k));
          new_tc = (new_tc & ~(0xFFu << (8 * k))) | (tc << (8 * k));
          if (tc != tp && own) {
            changed++;
            const int nold = __ldg(g_tri_count + tp), nnew = __ldg(g_tri_count + tc);
            t_rel += nold;
            t_new += nnew;
            irr += (nnew > 0 && !is_regular_type(tc)) - (nold > 0 && !is_regular_type(tp));
          }
          const unsigned mask = edge_mask_of(tc);
          if (mask && own) {
            active++;
            placements += __popc(mask);
          }
          // request the mask edges' slots: per axis, the owner point's column
          // word (bit = owner z), edge geometry of mc_tables.py:44-64
          const unsigned b0 = 1u << z, b1 = 2u << z;
          cxa |= (mask & 1u ? b0 : 0u) | (mask & 16u ? b1 : 0u);            // e0, e4: (x, y)
          cxb |= (mask & 4u ? b0 : 0u) | (mask & 64u ? b1 : 0u);            // e2, e6: (x, y+1)
          cya |= (mask & 2u ? b0 : 0u) | (mask & 32u ? b1 : 0u);            // e1, e5: (x+1, y)
          cyb |= (mask & 8u ? b0 : 0u) | (mask & 128u ? b1 : 0u);           // e3, e7: (x, y)
          cza |= mask & 256u ? b0 : 0u;                                      // e8: (x, y)
          czb |= mask & 512u ? b0 : 0u;                                      // e9: (x+1, y)
          czc |= mask & 1024u ? b0 : 0u;                                     // e10: (x+1, y+1)
          czd |= mask & 2048u ? b0 : 0u;                                     // e11: (x, y+1)
        }
        if (new_tc != old_tc || new_tp != old_tp) {   // 4 cubes per 32-bit store
          const size_t q4 = ((size_t)b * kNC + c0) >> 2;
          reinterpret_cast<uint32_t *>(S.tp)[q4] = new_tp;
          reinterpret_cast<uint32_t *>(S.tc)[q4] = new_tc;
        }
      }
      if (part) S.psel[(size_t)i * 64 + t] = (uint8_t)selb;
      }
      if (part) cxa = cxb = cya = cyb = cza = czb = czc = czd = 0u;   // (no claims)
      // one shared-memory OR per (axis, column) word this thread touched
      if (cxa) atomicOr(&s_claim[0 * 81 + cols[0]], cxa);
      if (cxb) atomicOr(&s_claim[0 * 81 + cols[3]], cxb);
      if (cya) atomicOr(&s_claim[1 * 81 + cols[1]], cya);
      if (cyb) atomicOr(&s_claim[1 * 81 + cols[0]], cyb);
      if (cza) atomicOr(&s_claim[2 * 81 + cols[0]], cza);
      if (czb) atomicOr(&s_claim[2 * 81 + cols[1]], czb);
      if (czc) atomicOr(&s_claim[2 * 81 + cols[2]], czc);
      if (czd) atomicOr(&s_claim[2 * 81 + cols[3]], czd);
    }
    __syncthreads();
    trace_item(S, TK_RETYPE, nth, 3);
    // placement (mesher.py:216-235).  Claims, one tile column per lane: its 3
    // claim words interleave into a 27-bit mask, bit 3 z + axis = the slot
    // (z, axis) of the column's owner cubes -- consecutive slot indices of the
    // owner block (C-order cubes, 3 slots each), so the column's requests are
    // <= 3 OR reductions into the owner blocks' claim bitmaps (k_gc_normals
    // turns first requests into allocations).  Coordinates: the item's
    // requested slots in column order are split into 64 equal runs, one per
    // thread (both warps get the same share whatever the surface's position
    // in the block); every requester of a slot writes the same bits.
    if (!part) {
      const int wq = t >> 5;
#pragma unroll
      for (int round = 0; round < 2; round++) {
        // warp 0: columns 0..31, 64..72; warp 1: 32..63, 73..80
        const int col = round == 0 ? wq * 32 + lane : 64 + wq * 9 + lane;
        if (round == 1 && lane >= 9 - wq) continue;
        uint32_t m = part1by2_9(s_claim[col]) | (part1by2_9(s_claim[81 + col]) << 1) |
                     (part1by2_9(s_claim[162 + col]) << 2);
        if (m) {
          const int ox = col / 9, oy = col - 9 * ox;
          const int sA = ((ox & 7) * 64 + (oy & 7) * 8) * 3;   // slot of (owner cube z = 0, axis 0)
          const int A = R.nbr[nbr_dir(ox >> 3, oy >> 3, 0)], B = R.nbr[nbr_dir(ox >> 3, oy >> 3, 1)];
          const uint32_t mA = m & 0xFFFFFFu, mB = m >> 24;
          const int off = sA & 31;
          if (mA) {
            if (A >= 0) {
              uint32_t *wp = S.vclaim + (size_t)A * (kEV / 32) + (sA >> 5);
              atomicOr(wp, mA << off);
              if (off > 8) atomicOr(wp + 1, mA >> (32 - off));
            } else {
              set_error(S, ERR_CONSISTENCY, 10, R.coord.x * kB + ox, R.coord.y * kB + oy,
                        R.coord.z * kB + (__ffs(mA) - 1) / 3);
              m &= ~0xFFFFFFu;
            }
          }
          if (mB) {
            if (B >= 0) atomicOr(S.vclaim + (size_t)B * (kEV / 32) + (sA >> 5), mB << off);
            else {
              set_error(S, ERR_CONSISTENCY, 10, R.coord.x * kB + ox, R.coord.y * kB + oy, R.coord.z * kB + 8);
              m &= 0xFFFFFFu;
            }
          }
        }
        s_mcol[col] = m;
      }
      __syncthreads();
      if (t < 32) {   // exclusive prefix of the 81 columns' counts (3 columns per lane)
        const int c0 = 3 * lane;
        const int n0 = lane < 27 ? __popc(s_mcol[c0]) : 0, n1 = lane < 27 ? __popc(s_mcol[c0 + 1]) : 0,
                  n2 = lane < 27 ? __popc(s_mcol[c0 + 2]) : 0;
        int incl = n0 + n1 + n2;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += u;
        }
        const int excl = incl - n0 - n1 - n2;
        if (lane < 27) {
          s_pre[c0] = excl;
          s_pre[c0 + 1] = excl + n0;
          s_pre[c0 + 2] = excl + n0 + n1;
        }
        if (lane == 31) s_pre[81] = incl;
      }
      __syncthreads();
      const int total = s_pre[81];
      const int per = (total + kNT - 1) / kNT;
      int e = t * per;
      const int e_end = min(total, e + per);
      if (e < e_end) {
        int c = 0;   // the column holding entry e: the last one with s_pre[c] <= e
#pragma unroll
        for (int step = 64; step > 0; step >>= 1)
          if (c + step < 81 && s_pre[c + step] <= e) c += step;
        uint32_t m = s_mcol[c];
        for (int k = e - s_pre[c]; k > 0; k--) m &= m - 1;   // (skip the column's first entries)
        for (; e < e_end; e++) {
          while (!m) m = s_mcol[++c];
          const int bit = __ffs(m) - 1;
          m &= m - 1;
          const int z = bit / 3, axis = bit - 3 * z;
          const int cx = c / 9, cy = c - 9 * cx;
          const int owner = R.nbr[nbr_dir(cx >> 3, cy >> 3, z >> 3)];
          const size_t slot = (size_t)owner * kEV + ((cx & 7) * 64 + (cy & 7) * 8 + (z & 7)) * 3 + axis;
          // start corner = the owner point; end corner one step along the axis
          const int pt = c * 9 + z;
          const double d0 = tile[pt], d1 = tile[pt + (axis == 0 ? 81 : axis == 1 ? 9 : 1)];
          const double param = (d0 == d1) ? 0.5 : d0 / (d0 - d1);
          const int ga = axis == 0 ? R.coord.x * kB + cx : axis == 1 ? R.coord.y * kB + cy : R.coord.z * kB + z;
          S.vparam[slot] = __dadd_rn(__dmul_rn((double)ga, l), __dmul_rn(param, l));
        }
      }
    }
    trace_at(S, TK_RETYPE, 30);
    append_halo();
    if (t == 32) trace_at_any(S, TK_RETYPE, 29);
    __syncthreads();   // R, tile and the placement list are rewritten by the next item
  }
  {
    trace_count(S, TK_RETYPE, nth);
    trace_at(S, TK_RETYPE, 28);
    const int vals[7] = {placements, active, changed, t_rel, t_new, irr, refined};
    int64_t *const dst[7] = {&S.ctr->placements, &S.ctr->active, &S.ctr->changed,
                             &S.ctr->t_released, &S.ctr->t_allocated, &S.ctr->irr_delta, &S.ctr->refined};
    warp_add_counters<7>(vals, dst);
  }
  if (t == 0 && live) S.ctr->nitems_live = 1;   // (a flag: some item was live this call)
  trace_span(S, 2, F.frame, true);
  trace_at(S, TK_RETYPE, 31);
}
constexpr size_t kRetypeSmem = 0;

// Strategy "partition" (mesher.py:250-254, 606-614): vertex placement in eight
// passes, one per 2x2x2 parity class of the cubes (one launch each, so the
// passes are separated by grid-wide completion).  Inside a pass no two cubes
// share an edge slot (cubes of one class are >= 2 apart along some axis, and
// the 4 cubes around an edge all differ in parity), so every request and
// coordinate is a PLAIN store: a request byte per slot (no atomic on a shared
// bitmap word, whose 32 slots span cubes of one class) and the slot's
// coordinate along its axis.  k_gc_normals (G_PARTITION) then reads the bytes
// as the claim bitmap.  Results are identical to the claim strategy's.
// One CTA of 64 threads per scope item: thread t = one of the item's 64 cubes
// of the class -- tile column (2 (t >> 4 & 3) + px, 2 (t >> 2 & 3) + py),
// z = 2 (t & 3) + pz.
__global__ void __launch_bounds__(kNT) k_place_parity(DevState S, const FrameDev F, int parity) {
  cudaGridDependencySynchronize();   // PDL: the previous pass (or the retype) has completed
  __shared__ int s_pro[5];
  read_prologue(S, s_pro, &S.ctr->ncollected, &S.ctr->nslab, &S.ctr->nexplicit, nullptr);
  if (s_pro[0]) return;
  const int nc = s_pro[1];
  const int n = F.scope_mode != 0 ? s_pro[3] : nc + s_pro[2];
  __shared__ int s_row[27];
  __shared__ int4 s_coord;
  const int t = threadIdx.x;
  const int x = 2 * ((t >> 4) & 3) + (parity & 1), y = 2 * ((t >> 2) & 3) + ((parity >> 1) & 1),
            z = 2 * (t & 3) + ((parity >> 2) & 1);
  const int c = (x * 8 + y) * 8 + z;
  const double l = S.cube_size;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int b = __ldcg(S.scope + i);
    if (b < 0) continue;   // (uniform)
    if (t < 27) s_row[t] = t == 13 ? b : __ldcg(S.nbr + (size_t)b * 27 + t);
    if (t == 27) s_coord = __ldcg(S.bcoord + b);
    const bool sel = (__ldcg(S.psel + (size_t)i * 64 + x * 8 + y) >> z) & 1u;
    const unsigned mask = sel ? edge_mask_of(__ldcg(S.tc + (size_t)b * kNC + c)) : 0u;
    __syncthreads();
    const int4 bc = s_coord;
    for (unsigned m = mask; m; m &= m - 1) {
      const int e = __ffs(m) - 1;
      const int oa = (int)((kEdgeOwnAxis >> (5 * e)) & 31);   // owner offset | axis << 3
      const int axis = oa >> 3;
      const int ox = x + (oa & 1), oy = y + ((oa >> 1) & 1), oz = z + ((oa >> 2) & 1);
      const int ob = s_row[nbr_dir(ox >> 3, oy >> 3, oz >> 3)];
      if (ob < 0) {   // mesher.py:200-203
        set_error(S, ERR_CONSISTENCY, 10, bc.x * kB + ox, bc.y * kB + oy, bc.z * kB + oz);
        continue;
      }
      const size_t slot = (size_t)ob * kEV + ((ox & 7) * 64 + (oy & 7) * 8 + (oz & 7)) * 3 + axis;
      // start corner = the owner point, end corner one step along the axis
      const int ex = ox + (axis == 0), ey = oy + (axis == 1), ez = oz + (axis == 2);
      const int eb = s_row[nbr_dir(ex >> 3, ey >> 3, ez >> 3)];
      const double d0 = S.tsdf[(size_t)ob * kNC + (ox & 7) * 64 + (oy & 7) * 8 + (oz & 7)];
      const double d1 = eb >= 0 ? S.tsdf[(size_t)eb * kNC + (ex & 7) * 64 + (ey & 7) * 8 + (ez & 7)] : 0.0;
      const double param = (d0 == d1) ? 0.5 : d0 / (d0 - d1);
      const int ga = axis == 0 ? bc.x * kB + ox : axis == 1 ? bc.y * kB + oy : bc.z * kB + oz;
      S.vreq[slot] = 1;
      S.vparam[slot] = __dadd_rn(__dmul_rn((double)ga, l), __dmul_rn(param, l));
    }
    __syncthreads();   // s_row is rewritten by the next item
  }
}

// the 32 request bytes of one slot word as bits (strategy "partition")
__device__ __forceinline__ uint32_t pack_requests(const uint8_t *p) {
  const uint4 a = __ldcg(reinterpret_cast<const uint4 *>(p)), b = __ldcg(reinterpret_cast<const uint4 *>(p + 16));
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  uint32_t r = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) {   // byte j of word k -> bit 4 k + j
    const uint32_t v = w[k];
    r |= (((v & 0xFFu) != 0) | (((v >> 8) & 0xFFu) != 0) << 1 | (((v >> 16) & 0xFFu) != 0) << 2 |
          ((v >> 24) != 0) << 3) << (4 * k);
  }
  return r;
}
__device__ __forceinline__ void clear_requests(uint8_t *p) {
  reinterpret_cast<uint4 *>(p)[0] = make_uint4(0, 0, 0, 0);
  reinterpret_cast<uint4 *>(p)[1] = make_uint4(0, 0, 0, 0);
}


// ------------------------------------------------------------ GC + normals
constexpr int kGT = 128;  // threads per CTA of k_gc_normals (warps 0..kGW-1 stage a halo block each)
// type tile over cube locals -1..7: 81 columns (lx, ly) of 16 bytes, z = 0..7
// at bytes 0..7 and z = -1 at byte 15 (the -z neighbour's z = 7, fetched as
// the aligned word of its z = 4..7 into bytes 12..15)
__device__ __forceinline__ int tt_idx(int lx, int ly, int lz) { return ((lx + 1) * 9 + (ly + 1)) * 16 + (lz & 15); }


// weight > 0 of the sample at block-local corner (lx, ly, lz) in [-1, 9]^3,
// from the 27 neighbours' staged validity bitmaps
__device__ __forceinline__ bool sample_valid(const uint32_t *s_vm, int lx, int ly, int lz) {
  const int c = (lx & 7) * 64 + (ly & 7) * 8 + (lz & 7);
  return (s_vm[nbr_dir(lx >> 3, ly >> 3, lz >> 3) * 16 + (c >> 5)] >> (c & 31)) & 1u;
}

// tsdf / weight sample at block-local corner (lx, ly, lz) in [-1, 9]^3
__device__ __forceinline__ size_t sample_index(const int *s_nbr, int lx, int ly, int lz) {
  const int nb = s_nbr[nbr_dir(lx >> 3, ly >> 3, lz >> 3)];
  return nb < 0 ? ~(size_t)0 : (size_t)nb * kNC + ((lx & 7) * 64 + (ly & 7) * 8 + (lz & 7));
}

// End of k_gc_normals, every CTA (halted ones included).  G_COMMIT: the last
// CTA to arrive folds the call's deltas into the pool counters (not for a
// halted frame: it is resumed and committed then); then, when F.snap is set,
// copies the counter block there (device memory; the next frame's k_collect
// publishes it to the host) and with F.reset_after clears the per-call
// counters for the next frame -- so consecutive frames need no stream
// operation between their kernels.
__device__ __forceinline__ void gc_commit(const DevState &S, const FrameDev &F, int mode, bool halted,
                                          Counters &s_c /* shared scratch: the last CTA's copy of the counter block */) {
  __shared__ int s_last;
  Counters *ctr = S.ctr;
  if (threadIdx.x == 0) {
    int last = 0;
    if (mode & G_COMMIT) {
      __threadfence();
      last = atomicAdd(&ctr->done_gc, 1) == (int)gridDim.x - 1;
    }
    s_last = last;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // one round trip: the whole block, a word per thread (every other CTA has
  // arrived, so nothing changes it meanwhile)
  constexpr int kWords = (int)(sizeof(Counters) / 4);
  {
    const volatile uint32_t *src = reinterpret_cast<const volatile uint32_t *>(ctr);
    uint32_t *sw = reinterpret_cast<uint32_t *>(&s_c);
    for (int q = threadIdx.x; q < kWords; q += blockDim.x) sw[q] = src[q];
  }
  __syncthreads();
  // `halted` is this frame's own state, read in the prologue: with frame
  // overlap the next frame's k_collect may have raised need / error since
  if (threadIdx.x == 0) {
    Counters &c = s_c;
    if ((mode & G_OVERLAP) && !halted) {   // the snapshot shows this frame's collect counters and block counts
      c.nvalid = c.sv_nvalid; c.nsteps = c.sv_nsteps; c.ncollected = c.sv_ncollected; c.nnew = c.sv_nnew;
      c.maxnorm_bits = c.sv_maxnorm_bits; c.t_start_ns = c.sv_t_start_ns;
      c.nblocks = c.sv_nblocks; c.nfree = c.sv_nfree; c.nblocks_owned = c.sv_nblocks_owned;
      c.error = 0; c.need = 0;
      c.err_info[0] = c.err_info[1] = c.err_info[2] = c.err_info[3] = 0;
    }
    if (!halted) {   // the fold, mirrored into the global block (persistent fields only)
      const long long allocs_all = c.v_allocs, fr = c.v_frees;
      const long long peak = c.v_live + allocs_all;     // all allocations precede all frees
      if (S.max_vertices > 0 && peak > S.max_vertices) {
        set_error(S, ERR_CAPACITY, peak, S.max_vertices, 3);
        if (c.error == 0) {
          c.error = ERR_CAPACITY;
          c.err_info[0] = peak; c.err_info[1] = S.max_vertices; c.err_info[2] = 3; c.err_info[3] = 0;
        }
      }
      if (peak > c.v_count) c.v_count = peak;
      c.v_live = peak - fr;
      c.v_recycled += fr;
      c.v_events += allocs_all;
      c.t_live += c.t_allocated - c.t_released;
      c.t_recycled += c.t_released;
      if (c.t_live > c.t_count) c.t_count = c.t_live;
      c.irregular += c.irr_delta;
      ctr->v_count = c.v_count; ctr->v_live = c.v_live; ctr->v_recycled = c.v_recycled;
      ctr->v_events = c.v_events; ctr->t_live = c.t_live; ctr->t_recycled = c.t_recycled;
      ctr->t_count = c.t_count; ctr->irregular = c.irregular;
    }
    c.done_gc = 0;
    ctr->done_gc = 0;
    c.t_end_ns = gtimer();
    ctr->t_end_ns = c.t_end_ns;   // (resumed frames and the phase API read the global block)
  }
  if (F.snap) {
  __syncthreads();
  {
    // (with G_OVERLAP the collect counters were cleared at the kernel's start)
    const int reset_from = (int)((mode & G_OVERLAP) ? offsetof(Counters, nslab) : offsetof(Counters, nvalid)) / 4;
    // (halted: nothing is cleared -- see below)
    const uint32_t *sw = reinterpret_cast<const uint32_t *>(&s_c);
    uint32_t *dst = reinterpret_cast<uint32_t *>(F.snap);
    for (int q = threadIdx.x; q < kWords; q += blockDim.x) {
      dst[q] = sw[q];
      if (F.reset_after && !halted && q >= reset_from) reinterpret_cast<uint32_t *>(ctr)[q] = 0u;
    }
  }
  if (F.self_dst && threadIdx.x < 32) {   // publish to the host now (the next frame's k_collect waits on a copy)
    const uint4 *sv = reinterpret_cast<const uint4 *>(&s_c);
    uint4 *hd = reinterpret_cast<uint4 *>(F.self_dst);
    for (int q = threadIdx.x; q < (int)(sizeof(Counters) / 16); q += 32) hd[q] = sv[q];
    __syncwarp();
    if (threadIdx.x == 0) {
      __threadfence_system();
      *reinterpret_cast<volatile unsigned long long *>(F.self_seq) = F.self_id;
    }
  }
  }
  // the commit is complete: a next frame's k_collect waiting on it may go on
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(S.gc_done), "r"(F.epoch) : "memory");
  }
}


// per-item shared state of k_gc_normals (one warp stages and collects each)
struct GcItem {
  Resolved R;
  uint32_t occ[kEV / 32];               // slot occupancy bits
  uint32_t cl[kEV / 32];                // this frame's placement requests
  uint32_t rb[kEV / 32];                // the slot has a vertex record
  __align__(16) uint32_t vm[27 * 16];   // weight > 0 bitmaps of the 27 neighbours
  __align__(16) uint8_t tt[81 * 16];    // type_curr over cube locals -1..7 (tt_idx)
  uint8_t inhalo[28];                   // neighbour is a halo block of this call
};
// entry of the CTA's union slot lists: item k (of kGW) << 11 | slot (< kEV = 1536)
__device__ __forceinline__ uint16_t gc_entry(int k, int sl) { return (uint16_t)((k << 11) | sl); }

// kGW warps per CTA, kGW halo blocks per CTA at a time: each warp resolves
// and stages its own block (cp.async: occupancy and request bits, the 9^3 type
// tile, the 27 neighbours' weight bitmaps); requests, GC, normals and the
// fallback records then run over the union of the kGW blocks' slots with the
// whole CTA, so a block with many vertices shares the work with lighter ones.
//  * requests (k_retype_place) of empty slots become allocations: birth =
//    frame, normal 0 (store.py:145-162);
//  * G_GC clears every occupied slot that no cube references any more (the
//    reference's refcount == 0 recycling, mesher.py:333-356: the 4 cubes
//    around the edge from the type tile), word-parallel over the bitmap;
//  * G_NORMALS: central-difference normals from each vertex's 12-sample
//    stencil (mesher.py:369-439), tsdf gathered directly, "observed" from the
//    bitmaps; stencil failures are recorded with their 4 cube types and
//    candidate mask for the face-normal fallback (mesher.py:456-486), applied
//    by the next frame's k_collect (or k_flush_fallbacks).
// G_COMMIT: the last CTA folds the per-call deltas into the pool counters.
constexpr int kGW = 4;
constexpr int kGWarps = kGT / 32;   // (the CTA's warps: all share the slot work)
constexpr int kGV = 1;   // surviving vertices per thread per normals pass

__global__ void __launch_bounds__(kGT, 8) k_gc_normals(DevState S, const FrameDev F,
                                                   const int32_t *__restrict__ list,
                                                   const int32_t *__restrict__ count_ptr,
                                                   int count_const, int mode) {
  cudaGridDependencySynchronize();   // PDL: wait for the previous kernel of the frame
  trace_at(S, TK_GC, 0);
  trace_span(S, 3, F.frame, false);
  Counters *ctr = S.ctr;
  __shared__ int s_pro[5];
  __shared__ int s_shp[kHaloShards + 1];   // G_SHARDED: prefix of the shard fills
  // the CTA's slot list (gc_entry): occupied slots, compacted in place to the
  // surviving ones, then the failed-gradient ones, then the records applied
  // inline -- each pass reads a chunk, syncs, and only then appends (an append
  // never passes the entries read so far), so one list serves all four and the
  // CTA fits 8 per SM
  __shared__ __align__(16) uint16_t s_la[kGW * kEV];
  static_assert(sizeof(s_la) >= sizeof(Counters), "gc_commit's scratch");
  const bool sharded = (mode & G_SHARDED) != 0;
  // prologue: warp 0 issues every load at once (halt flags and counts on
  // lane 0, the halo shard fills on all lanes), one round trip
  if (threadIdx.x < 32) {
    int4 hd = make_int4(0, 0, 0, 0), it = make_int4(0, 0, 0, 0);
    int vb = 0;
    if (threadIdx.x == 0) {
      // (through L1, see read_prologue; the next frame's k_collect, which may
      // raise need / error, launches only after every CTA has passed here)
      hd = __ldg(reinterpret_cast<const int4 *>(ctr));                  // nblocks, ovf, error, need
      if (mode & G_REQUIRE_ITEMS) it = __ldg(reinterpret_cast<const int4 *>(&ctr->nslab));   // .z nitems_live
      vb = count_ptr ? __ldg(count_ptr) : 0;
    }
    const int2 h = make_int2(hd.z, hd.w);
    const int va = it.z;
    int c = sharded ? min(__ldg(ctr->nhalo_sh + threadIdx.x), S.halo_sh_cap) : 0;
    if (threadIdx.x == 0) {
      s_pro[0] = (h.x | h.y) != 0;
      s_pro[1] = va; s_pro[2] = vb; s_pro[3] = 0; s_pro[4] = -1;
    }
    if (sharded) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, c, o);
        if ((int)threadIdx.x >= o) c += u;
      }
      s_shp[threadIdx.x + 1] = c;
      if (threadIdx.x == 0) s_shp[0] = 0;
    }
  }
  __syncthreads();
  if (mode & G_OVERLAP) {
    // the frame's collect counters and block counts are saved for the commit's
    // snapshot and the collect counters cleared -- then the next frame's
    // k_collect may launch: once every CTA of this grid has triggered.  (A
    // halted frame keeps them: the host resumes it from them; the next
    // frame's k_collect stops at its guard and writes none of them.)
    if (blockIdx.x == 0 && !s_pro[0]) {
      if (threadIdx.x == 0) {
        const int4 a = __ldcg(reinterpret_cast<const int4 *>(&ctr->nvalid));          // nvalid, nsteps, ncollected, nnew
        const ulonglong2 m = __ldcg(reinterpret_cast<const ulonglong2 *>(&ctr->maxnorm_bits));   // maxnorm, t_start
        const int nb = __ldcg(&ctr->nblocks), nf = __ldcg(&ctr->nfree);
        const long long no = (long long)__ldcg(reinterpret_cast<const unsigned long long *>(&ctr->nblocks_owned));
        *reinterpret_cast<int4 *>(&ctr->sv_nvalid) = a;
        *reinterpret_cast<ulonglong2 *>(&ctr->sv_maxnorm_bits) = m;
        ctr->sv_nblocks = nb; ctr->sv_nfree = nf; ctr->sv_nblocks_owned = no;
        *reinterpret_cast<int4 *>(&ctr->nvalid) = make_int4(0, 0, 0, 0);
        *reinterpret_cast<ulonglong2 *>(&ctr->maxnorm_bits) = make_ulonglong2(0ull, 0ull);
        *reinterpret_cast<int4 *>(&ctr->fb_next) = make_int4(0, 0, 0, 0);
        __threadfence();
      }
      __syncthreads();
    }
    cudaTriggerProgrammaticLaunchCompletion();
  }
  if (s_pro[0]) {   // halted frame: no work, but the commit still publishes
    gc_commit(S, F, mode, true, *reinterpret_cast<Counters *>(s_la));
    return;
  }
  const int live_items = (mode & G_REQUIRE_ITEMS) ? s_pro[1] : 1;
  const int nsh = sharded ? s_shp[kHaloShards] : 0;
  const int n = live_items > 0 ? nsh + (count_ptr ? s_pro[2] : count_const) : 0;
  __shared__ long long s_rr[4];   // this CTA's free vertex records: ranges [s_rr[0], s_rr[1]), [s_rr[2], s_rr[3])
  // a round's records: j < s_asg[1] -> s_asg[0] + j; j < s_asg3[0] -> s_asg[2] + j - s_asg[1];
  // else s_asg3[1] + j - s_asg3[0]
  __shared__ long long s_asg[3], s_asg3[2];
  __shared__ int s_rr_dirty;
  if (threadIdx.x == 0) s_rr_dirty = 0;
  // this CTA's free vertex records (two ranges kept between calls), staged
  // asynchronously; topped up at the CTA's end when short
  long long *const rec_ranges = S.rec_chunk + 4 * (blockIdx.x % S.rec_chunk_ctas);
  if (threadIdx.x == 0 && n > 0) {
    cp_async16(&s_rr[0], rec_ranges, true);
    cp_async16(&s_rr[2], rec_ranges + 2, true);
  }
  __shared__ GcItem G[kGW];
  __shared__ int s_nocc, s_nv, s_nfb, s_nin;
  __shared__ int red[4 * kGWarps];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  GcItem &I = G[w < kGW ? w : 0];   // (warps past kGW stage nothing)
  const bool normals = (mode & G_NORMALS) != 0;
  FrameDev Fr = F;
  Fr.scope_mode = 1;   // resolve as explicit items: no slab bits
  Fr.frustum_only = 0;
  int frees = 0, computed = 0, fallbacks = 0, allocs = 0;
  trace_at(S, TK_GC, 1);
  const int per_round = (int)gridDim.x * kGW;
  int nth = 0;
  for (int base = 0; base < n; base += per_round, nth++) {
    trace_item(S, TK_GC, nth, 0);
    // (the kGW blocks of a CTA are a grid apart in the list: neighbouring list
    // entries are neighbouring blocks of similar surface density)
    const int i = base + w * (int)gridDim.x + blockIdx.x;
    if (w < kGW) {
      int bi = -1;
      if (i < nsh) {   // shard k holds flat items [s_shp[k], s_shp[k + 1])
        int k = 0;
#pragma unroll
        for (int step = kHaloShards / 2; step > 0; step >>= 1)
          if (s_shp[k + step] <= i) k += step;
        bi = __ldcg(S.halo_sh + (size_t)k * S.halo_sh_cap + (i - s_shp[k]));
      } else if (i < n) {
        bi = __ldcg(list + (i - nsh));
      }
      const ResolveRegs rr = resolve_load(S, Fr, bi, i, 0);
      resolve_store(S, Fr, rr, bi, i, n, 0, I.R);
    }
    if (t == 0) { s_nocc = 0; s_nv = 0; s_nfb = 0; s_nin = 0; }
    __syncwarp();
    const bool live = w < kGW && I.R.mode > 0;
    const int b = I.R.b;
    if (live) {
      // stage occupancy + requests, types and halo flags (all copies in flight)
      for (int q = lane; q < kEV / 32; q += 32) {
        cp_async4(&I.occ[q], S.vocc + (size_t)b * (kEV / 32) + q, true);
        cp_async4(&I.rb[q], S.vrb + (size_t)b * (kEV / 32) + q, true);
        if (mode & G_PARTITION) I.cl[q] = pack_requests(S.vreq + (size_t)b * kEV + q * 32);
        else cp_async4(&I.cl[q], S.vclaim + (size_t)b * (kEV / 32) + q, true);
      }
      for (int q = lane; q < 2 * 81; q += 32) {   // per column: the z = 0..7 run, then z = -1
        const int col = q >> 1, lx = col / 9 - 1, ly = col % 9 - 1;
        const int dx = lx < 0 ? -1 : 0, dy = ly < 0 ? -1 : 0;
        const size_t row = (size_t)((lx & 7) * 64 + (ly & 7) * 8);
        if ((q & 1) == 0) {
          const int nb = I.R.nbr[nbr_dir(dx, dy, 0)];
          cp_async8(&I.tt[col * 16], S.tc + (size_t)(nb >= 0 ? nb : 0) * kNC + row, nb >= 0);
        } else {
          const int nb = I.R.nbr[nbr_dir(dx, dy, -1)];
          cp_async4(&I.tt[col * 16 + 12], S.tc + (size_t)(nb >= 0 ? nb : 0) * kNC + row + 4, nb >= 0);
        }
      }
      if (normals)   // weight > 0 bitmaps of the 27 neighbours (16 words each, 4 x 16 B)
        for (int q = lane; q < 27 * 4; q += 32) {
          const int nb = I.R.nbr[q >> 2];
          cp_async16(&I.vm[q * 4], S.vmask + (size_t)(nb >= 0 ? nb : 0) * (kNC / 32) + (q & 3) * 4, nb >= 0);
        }
      int hv = 0;
      if (normals && lane < 27) {
        const int nb = I.R.nbr[lane];
        hv = nb >= 0 && __ldcg(S.stamp_halo + nb) == F.epoch;
      }
      if (lane < 27) I.inhalo[lane] = (uint8_t)hv;
      cp_async_wait_all();
      __syncwarp();
      trace_item(S, TK_GC, nth, 2);
    }
    __syncthreads();   // every block staged
    trace_sub(S, TK_GC, nth, 2);
    // requests, over the kGW blocks' bitmap words: a requested empty slot is
    // allocated (birth = frame, normal 0); every occupied slot is listed
    constexpr int kReqRounds = (kGW * (kEV / 32) + kGT - 1) / kGT;
    uint32_t rec_new[kReqRounds];   // allocated slots that have no vertex record yet
    int n_rec = 0;
#pragma unroll
    for (int r = 0; r < kReqRounds; r++) {
      const int wi = t + r * kGT;
      const int k = wi / (kEV / 32), wd = wi - k * (kEV / 32);
      uint32_t word = 0;
      rec_new[r] = 0;
      if (wi < kGW * (kEV / 32) && G[k].R.mode > 0) {
        GcItem &J = G[k];
        const size_t bk = (size_t)J.R.b;
        const uint32_t claim = J.cl[wd], fresh = claim & ~J.occ[wd];
        rec_new[r] = fresh & ~J.rb[wd];   // first occupation: a record is handed out below
        n_rec += __popc(rec_new[r]);
        // Birth and zero normal go into the slot's record: with the normals
        // pass they are written there (it reads every surviving slot's record
        // handle anyway, and writes every surviving vertex's normal -- zero
        // first where its stencil fails, for the fallback's "never set" test)
        if (!normals)
          for (uint32_t m = fresh & J.rb[wd]; m; m &= m - 1) {
            VertexRec &vr = S.vrec[S.vh[bk * kEV + wd * 32 + __ffs(m) - 1]];
            vr.birth = F.frame;
            vr.nrm[0] = 0.0; vr.nrm[1] = 0.0; vr.nrm[2] = 0.0;
          }
        allocs += J.R.owned * __popc(fresh);   // counted by the slot's owning rank
        if (claim) {
          if (mode & G_PARTITION) clear_requests(S.vreq + bk * kEV + wd * 32);
          else S.vclaim[bk * (kEV / 32) + wd] = 0u;
        }
        word = J.occ[wd] | claim;
        J.occ[wd] = word;
        J.cl[wd] = fresh;   // (the allocations of this call, for the normals pass)
      }
      int pos = smem_append(__popc(word), &s_nocc);
      for (uint32_t m = word; m; m &= m - 1) s_la[pos++] = gc_entry(k, wd * 32 + __ffs(m) - 1);
    }
    // vertex records for first-time slots, from this CTA's chunk (capacity was
    // checked by k_retype_place's prologue)
    if (__syncthreads_or(n_rec)) {
      int incl = n_rec;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (lane == 31) red[w] = incl;
      __syncthreads();
      if (t == 0) {
        int acc = 0;
        for (int q = 0; q < kGWarps; q++) { const int c = red[q]; red[q] = acc; acc += c; }
        cp_async_wait_all();   // (s_rr)
        long long a0 = s_rr[0], e0 = s_rr[1], a1 = s_rr[2], e1 = s_rr[3];
        if ((e0 - a0) + (e1 - a1) < acc) {   // more than the CTA holds: merge its ranges' use with a new run
          // (range 0 is used first: move range 1 behind it only when range 0 is empty)
          if (e0 <= a0) { a0 = a1; e0 = e1; a1 = e1 = 0; }
          const long long short_by = acc - (e0 - a0) - (e1 - a1);
          const long long want = (short_by + 2 * kRecChunk - 1) / kRecChunk * kRecChunk;
          const long long nb =
              (long long)atomicAdd(reinterpret_cast<unsigned long long *>(&ctr->a_hw), (unsigned long long)want);
          if (e1 > a1) {   // both ranges in use: they are consumed whole, the new run follows range 1
            s_asg[0] = a0; s_asg[1] = e0 - a0; s_asg[2] = a1;
            s_asg3[0] = (e0 - a0) + (e1 - a1); s_asg3[1] = nb;
            a0 = nb + short_by; e0 = nb + want; a1 = e1 = 0;
          } else {
            s_asg[0] = a0; s_asg[1] = e0 - a0; s_asg[2] = nb;
            s_asg3[0] = 1LL << 62;
            a0 = nb + short_by; e0 = nb + want; a1 = e1 = 0;
          }
        } else {
          s_asg[0] = a0; s_asg[1] = e0 - a0; s_asg[2] = a1;   // range 0 first, then range 1
          s_asg3[0] = 1LL << 62;
          // consume acc records; the rest stays for later rounds and calls
          if (acc <= e0 - a0) {
            a0 += acc;
          } else {
            a1 += acc - (e0 - a0);
            a0 = a1; e0 = e1; a1 = e1 = 0;
          }
        }
        s_rr[0] = a0; s_rr[1] = e0; s_rr[2] = a1; s_rr[3] = e1;
        s_rr_dirty = 1;
      }
      __syncthreads();
      const long long r_cur = s_asg[0], r_rem = s_asg[1], r_new = s_asg[2], r_lim = s_asg3[0], r_ext = s_asg3[1];
      long long j = red[w] + incl - n_rec;   // this thread's first record, as an index into the CTA's run
#pragma unroll
      for (int r = 0; r < kReqRounds; r++) {
        if (!rec_new[r]) continue;
        const int wi = t + r * kGT;
        const int k = wi / (kEV / 32), wd = wi - k * (kEV / 32);
        GcItem &J = G[k];
        J.rb[wd] |= rec_new[r];   // (this thread's word only)
        for (uint32_t m = rec_new[r]; m; m &= m - 1, j++) {
          const long long h = j < r_rem ? r_cur + j : j < r_lim ? r_new + (j - r_rem) : r_ext + (j - r_lim);
          S.vh[(size_t)J.R.b * kEV + wd * 32 + __ffs(m) - 1] = (int32_t)h;
          if (!normals) {
            S.vrec[h].birth = F.frame;
            S.vrec[h].nrm[0] = 0.0; S.vrec[h].nrm[1] = 0.0; S.vrec[h].nrm[2] = 0.0;
          }
        }
        S.vrb[(size_t)J.R.b * (kEV / 32) + wd] = J.rb[wd];
      }
      __syncthreads();   // (the handles are read by the normals pass; red is reused)
    }
    trace_sub(S, TK_GC, nth, 3);
    // GC over the occupied list: a slot survives iff a cube around its edge
    // still has the edge in its mask (the 4 cubes at -du along u, -dw along w;
    // u, w = the two axes other than the slot's)
    const int nocc = s_nocc;
    for (int p0 = 0; p0 < nocc; p0 += kGT) {
      const int p = p0 + t;
      bool keep = false;
      uint16_t e = 0;
      if (p < nocc) {
        e = s_la[p];
        keep = true;
        if (mode & G_GC) {
          GcItem &J = G[e >> 11];
          const int sl = e & 2047, c = sl / 3, axis = sl - 3 * c;
          // (no short-circuit: the 4 type and mask lookups issue together)
          unsigned ty[4], ref = 0;
#pragma unroll
          for (int q = 0; q < 4; q++) {
            int l0, l1, l2;
            slot_cube(c, axis, q, l0, l1, l2);
            ty[q] = J.tt[tt_idx(l0, l1, l2)];
          }
#pragma unroll
          for (int q = 0; q < 4; q++) ref |= edge_mask_of(ty[q]) >> cube_edge_of_slot(axis, q >> 1, q & 1);
          if (!(ref & 1u)) {
            keep = false;   // (the slot keeps its vertex record for a later occupation)
            atomicAnd(&J.occ[sl >> 5], ~(1u << (sl & 31)));
            frees += J.R.owned;
          }
        }
      }
      if (normals) {
        __syncthreads();   // (the chunk is read: appends stay below it)
        const int pos = smem_append(keep ? 1 : 0, &s_nv);
        if (keep) s_la[pos] = e;
      }
    }
    __syncthreads();
    for (int wi = t; wi < kGW * (kEV / 32); wi += kGT) {   // occupancy after requests + frees
      const int k = wi / (kEV / 32), wd = wi - k * (kEV / 32);
      if (G[k].R.mode > 0) S.vocc[(size_t)G[k].R.b * (kEV / 32) + wd] = G[k].occ[wd];
    }
    trace_sub(S, TK_GC, nth, 0);
    if (normals) {
      // the surviving vertices, whole CTA, two per thread per pass (their 24
      // tsdf loads in flight together)
      const int nv = s_nv;
      for (int p0 = 0; p0 < nv; p0 += kGV * kGT) {
        double v[kGV][12];
        int slv[kGV], itv[kGV], hv[kGV];
        bool val[kGV];
#pragma unroll
        for (int u = 0; u < kGV; u++) {
          const int p = p0 + u * kGT + t;
          const uint16_t e = p < nv ? s_la[p] : (uint16_t)0;
          const int k = e >> 11;
          itv[u] = k;
          slv[u] = p < nv ? (e & 2047) : -1;
          const GcItem &J = G[k];
          const int bj = J.R.b;
          const int sl = slv[u] < 0 ? 0 : slv[u];
          const int ci = sl / 3, axis = sl - 3 * ci;
          const int x0 = ci >> 6, y0 = (ci >> 3) & 7, z0 = ci & 7;
          const int x1 = x0 + (axis == 0), y1 = y0 + (axis == 1), z1 = z0 + (axis == 2);
          // the 12 stencil samples c0 +- e_d, c1 +- e_d (c1 = c0 + e_axis), absent
          // neighbours read a dummy in-bounds sample; weight > 0 from the staged
          // bitmaps (absent = 0)
          const size_t dummy = (size_t)(bj < 0 ? 0 : bj) * kNC;
          hv[u] = slv[u] >= 0 ? S.vh[(size_t)bj * kEV + sl] : 0;   // the vertex record (requested with the samples)
          bool ok = slv[u] >= 0;
#pragma unroll
          for (int d = 0; d < 3; d++) {
            const int dx = d == 0, dy = d == 1, dz = d == 2;
            const size_t a = sample_index(J.R.nbr, x0 + dx, y0 + dy, z0 + dz);
            const size_t bq = sample_index(J.R.nbr, x0 - dx, y0 - dy, z0 - dz);
            const size_t cq = sample_index(J.R.nbr, x1 + dx, y1 + dy, z1 + dz);
            const size_t dq = sample_index(J.R.nbr, x1 - dx, y1 - dy, z1 - dz);
            v[u][4 * d + 0] = S.tsdf[a == ~(size_t)0 ? dummy : a];     // c0 + e_d
            v[u][4 * d + 1] = S.tsdf[bq == ~(size_t)0 ? dummy : bq];   // c0 - e_d
            v[u][4 * d + 2] = S.tsdf[cq == ~(size_t)0 ? dummy : cq];   // c1 + e_d
            v[u][4 * d + 3] = S.tsdf[dq == ~(size_t)0 ? dummy : dq];   // c1 - e_d
            ok = ok & sample_valid(J.vm, x0 + dx, y0 + dy, z0 + dz) & sample_valid(J.vm, x0 - dx, y0 - dy, z0 - dz) &
                 sample_valid(J.vm, x1 + dx, y1 + dy, z1 + dz) & sample_valid(J.vm, x1 - dx, y1 - dy, z1 - dz);
          }
          val[u] = ok;
        }
        __syncthreads();   // (the chunk's entries are read: failure appends stay below them)
#pragma unroll
        for (int u = 0; u < kGV; u++) {
          if (slv[u] < 0) continue;
          const GcItem &J = G[itv[u]];
          const int sl = slv[u];
          const int axis = sl - 3 * (sl / 3);
          computed += J.R.owned;
          const double d0 = axis == 0 ? v[u][3] : axis == 1 ? v[u][7] : v[u][11];   // samples at c0 and c1
          const double d1 = axis == 0 ? v[u][0] : axis == 1 ? v[u][4] : v[u][8];
          const double denom = d0 - d1;
          const double param = (denom != 0) ? d0 / denom : 0.5;
          double g[3];
          const double wa = 1.0 - param;
#pragma unroll
          for (int d = 0; d < 3; d++)
            g[d] = __dadd_rn(__dmul_rn(wa, v[u][4 * d] - v[u][4 * d + 1]),
                             __dmul_rn(param, v[u][4 * d + 2] - v[u][4 * d + 3]));
          const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(g[0], g[0]), __dmul_rn(g[1], g[1])),
                                            __dmul_rn(g[2], g[2])));
          const bool fresh = (J.cl[sl >> 5] >> (sl & 31)) & 1u;   // allocated by this call
          if (fresh) S.vrec[hv[u]].birth = F.frame;
          if (val[u] && nrm > 1e-12) {
            double *dst = S.vrec[hv[u]].nrm;
            dst[0] = g[0] / nrm; dst[1] = g[1] / nrm; dst[2] = g[2] / nrm;
          } else {
            if (fresh) {   // its normal starts at zero
              double *dst = S.vrec[hv[u]].nrm;
              dst[0] = 0.0; dst[1] = 0.0; dst[2] = 0.0;
            }
            fallbacks += J.R.owned;
            s_la[atomicAdd(&s_nfb, 1)] = gc_entry(itv[u], sl);
          }
        }
      }
      __syncthreads();
      trace_sub(S, TK_GC, nth, 1);
      // face-normal fallback records: the failed slots with their 4 cube types
      // and candidate mask (staged tile, row, halo flags).  The record list is
      // a bounded ring (fb_cap); records past it are applied right here, one
      // warp each -- everything a fallback reads (types, vertex coordinates,
      // neighbour rows, the vertex's own normal just written) is final once
      // the frame's k_retype_place has completed.
      auto fb_record = [&](uint16_t e, uint32_t &types4, uint32_t &cand) {
        const GcItem &J = G[e >> 11];
        const int sl = e & 2047;
        const int ci = sl / 3, axis = sl - 3 * ci;
        types4 = 0;
        cand = 0;
#pragma unroll
        for (int q = 0; q < 4; q++) {
          int l0, l1, l2;
          slot_cube(ci, axis, q, l0, l1, l2);
          const uint32_t ty = J.tt[tt_idx(l0, l1, l2)];
          const int dir = nbr_dir(l0 < 0 ? -1 : 0, l1 < 0 ? -1 : 0, l2 < 0 ? -1 : 0);
          types4 |= ty << (8 * q);
          if (((edge_mask_of(ty) >> cube_edge_of_slot(axis, q >> 1, q & 1)) & 1) && J.R.nbr[dir] >= 0 &&
              J.inhalo[dir])
            cand |= 1u << q;
        }
      };
      const int nfb = s_nfb;
      for (int p0 = 0; p0 < nfb; p0 += kGT) {   // (warp-uniform: one ring slot reservation per warp)
        const int p = p0 + t;
        const bool has = p < nfb;
        const uint16_t e = has ? s_la[p] : (uint16_t)0;
        __syncthreads();   // (the chunk is read: inline appends stay below it)
        const int bb = G[e >> 11].R.b, sl = e & 2047;
        const int h = has ? S.vh[(size_t)bb * kEV + sl] : 0;   // (requested before the reservation)
        const unsigned bal = __ballot_sync(0xffffffffu, has);
        if (!bal) continue;
        int at = 0;
        if (lane == __ffs(bal) - 1) at = atomicAdd(&ctr->fb_pending, __popc(bal));
        at = __shfl_sync(0xffffffffu, at, __ffs(bal) - 1) + __popc(bal & ((1u << lane) - 1));
        if (!has) continue;
        uint32_t types4, cand;
        fb_record(e, types4, cand);
        if (at < S.fb_cap) S.fallback[at] = make_int4(bb, sl | (int)(cand << 11), (int)types4, h);
        else s_la[atomicAdd(&s_nin, 1)] = e;
      }
      __syncthreads();
      for (int q = w; q < s_nin; q += kGWarps) {   // ring full: inline, one warp per record
        const uint16_t e = s_la[q];
        const GcItem &J = G[e >> 11];
        const int sl = e & 2047;
        uint32_t types4, cand;
        fb_record(e, types4, cand);
        fallback_normal_inline(S.vparam, S.cube_size, lane < 27 ? J.R.nbr[lane] : -1, types4, cand, J.R.coord,
                             sl / 3, sl % 3, S.vrec[S.vh[(size_t)J.R.b * kEV + sl]].nrm);
      }
    }
    trace_item(S, TK_GC, nth, 3);
    __syncthreads();   // the items' shared state is rewritten by the next round
  }
  if (threadIdx.x == 0 && s_rr_dirty) {   // the ranges' rest (the next frame's k_collect tops them up)
    *reinterpret_cast<longlong2 *>(rec_ranges) = make_longlong2(s_rr[0], s_rr[1]);
    *reinterpret_cast<longlong2 *>(rec_ranges + 2) = make_longlong2(s_rr[2], s_rr[3]);
  }
  trace_count(S, TK_GC, nth);
  trace_at(S, TK_GC, 28);
  {
    // warp sums, then thread 0 adds all four: its own fence in gc_commit then
    // orders them before its arrival count (the fold reads v_frees / v_allocs)
    const int vals[4] = {frees, computed, fallbacks, allocs};
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int v = (int)__reduce_add_sync(0xffffffffu, (unsigned)vals[k]);
      if (lane == 0) red[w * 4 + k] = v;
    }
    __syncthreads();
    if (t == 0) {
      int64_t *const dst[4] = {&ctr->v_frees, &ctr->normals, &ctr->fallbacks, &ctr->v_allocs};
#pragma unroll
      for (int k = 0; k < 4; k++) {
        long long r = 0;
#pragma unroll
        for (int q = 0; q < kGWarps; q++) r += red[q * 4 + k];
        if (r) atomicAdd((unsigned long long *)dst[k], (unsigned long long)r);
      }
    }
  }
  gc_commit(S, F, mode, false, *reinterpret_cast<Counters *>(s_la));   // (the lists are spent)
  trace_span(S, 3, F.frame, true);
  trace_at(S, TK_GC, 31);
}
constexpr size_t kGcSmem = 0;


// ------------------------------------------------------------ block GC
// Opt-in block eviction (north star item 5; the reference never frees a
// block, store.py:14, so this is off in parity mode).  A block is evicted when
// it was last collected at least `age` frames ago and holds nothing: no
// occupied edge slot, no pending request and no observed sample (every
// weight 0; weights never decrease).  Every cube with a corner in it is then
// undefined and every normal stencil touching it unobserved, exactly as for
// an absent block, so the mesh is unchanged -- only blocks_active differs.
// (A free-space block -- tsdf +1 with weight > 0 -- is kept: a neighbour's
// boundary cube can be defined through its samples.)
// Its hash entry keeps the key with value kEvicted (a re-observation
// allocates a fresh block there), its neighbours' rows are unlinked and its
// index goes to the free list, which allocations pop first.  One warp per
// block; runs before a frame's k_collect.
__global__ void __launch_bounds__(256) k_block_gc(DevState S, int frame, int age) {
  const int lane = threadIdx.x & 31;
  const int nb = ld_vol(&S.ctr->nblocks);
  const int warps = (int)(gridDim.x * blockDim.x) >> 5;
  long long evicted = 0;
  for (int b = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); b < nb; b += warps) {
    const int4 c = S.bcoord[b];
    if (c.w != 0 || S.last_frame[b] > frame - age) continue;   // (dead, or seen recently)
    bool busy = false;
    for (int q = lane; q < kEV / 32; q += 32)
      busy |= (S.vocc[(size_t)b * (kEV / 32) + q] | S.vclaim[(size_t)b * (kEV / 32) + q]) != 0u;
    if (lane < kNC / 32) busy |= S.vmask[(size_t)b * (kNC / 32) + lane] != 0u;   // a sample with weight > 0
    if (__any_sync(0xffffffffu, busy)) continue;
    // unlink: neighbours forget the block, its own row is cleared
    if (lane < 27 && lane != 13) {
      const int n = S.nbr[(size_t)b * 27 + lane];
      if (n >= 0) S.nbr[(size_t)n * 27 + (26 - lane)] = -1;
    }
    if (lane < 27) S.nbr[(size_t)b * 27 + lane] = -1;
    if (lane == 0) {
      // the hash entry keeps its key, value kEvicted
      const long long key = pack_coord(c.x, c.y, c.z);
      const unsigned bk = bucket_of(S, key);
      HashSlot *kb = S.slots + (size_t)bk * kSlotsPerBucket;
      bool done = false;
      for (int i = 0; i < kSlotsPerBucket && !done; i++)
        if (kb[i].key == key) { kb[i].val = kEvicted; done = true; }
      for (int e = S.ovf_head[bk]; e >= 0 && !done; e = S.ovf_next[e])
        if (S.ovf_key[e] == key) { S.ovf_val[e] = kEvicted; done = true; }
      S.bcoord[b] = make_int4(c.x, c.y, c.z, 1);   // dead
      S.free_list[atomicAdd(&S.ctr->nfree, 1)] = b;
      if (S.nranks > 1 && S.bowned[b]) atomicAdd((unsigned long long *)&S.ctr->nblocks_owned, ~0ull);
      evicted++;
    }
  }
  evicted = warp_sum(evicted);
  if (lane == 0 && evicted) atomicAdd((unsigned long long *)&S.ctr->evicted_total, (unsigned long long)evicted);
}

// ------------------------------------------------------------ full scans
__global__ void k_irregular_full(DevState S, int nblocks, unsigned long long *out) {
  long long cnt = 0;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)nblocks * kNC;
       q += (long long)gridDim.x * blockDim.x) {
    const unsigned tc = S.tc[q];
    cnt += c_tri_count[tc] > 0 && !is_regular_type(tc) && (S.nranks <= 1 || S.bowned[q / kNC]);
  }
  cnt = warp_sum(cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, (unsigned long long)cnt);
}

// reference count of one slot = incidences of its edge in the triangles of
// the (up to 4) cubes around it; returns -1 cubes outside existing blocks as 0
__device__ int slot_refcount(const DevState &S, int b, int slot) {
  const int ci = slot / 3, axis = slot % 3;
  const int x = ci >> 6, y = (ci >> 3) & 7, z = ci & 7;
  const int u = axis == 0 ? 1 : 0, w = axis == 2 ? 1 : 2;
  int cnt = 0;
  for (int du = 0; du < 2; du++)
    for (int dw = 0; dw < 2; dw++) {
      int l[3] = {x, y, z};
      l[u] -= du;
      l[w] -= dw;
      const int dir = nbr_dir(l[0] < 0 ? -1 : 0, l[1] < 0 ? -1 : 0, l[2] < 0 ? -1 : 0);
      const int nb = (dir == 13) ? b : S.nbr[(size_t)b * 27 + dir];
      if (nb < 0) continue;
      const unsigned tt = S.tc[(size_t)nb * kNC + ((l[0] & 7) * 64 + (l[1] & 7) * 8 + (l[2] & 7))];
      const int e = cube_edge_of_slot(axis, du, dw);
      const unsigned long long packed = c_tri_packed[tt];
      for (int q = 0; q < 3 * c_tri_count[tt]; q++) cnt += (int)((packed >> (4 * q)) & 0xF) == e;
    }
  return cnt;
}

// audit (engine.py:187-230): occupancy vs references over every slot.
// sums: [0] occupied slots, [1] referenced-but-empty slots (missing vertex),
// [2] occupied-but-unreferenced slots, [3] triangles (sum TRI_COUNT)
__global__ void k_audit(DevState S, int nblocks, unsigned long long *sums) {
  long long occ = 0, missing = 0, zero = 0, tris = 0;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)nblocks * kEV;
       q += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(q / kEV), slot = (int)(q % kEV);
    const bool o = (S.vocc[q >> 5] >> (q & 31)) & 1u;
    const bool r = slot_refcount(S, b, slot) > 0;
    occ += o;
    missing += r && !o;
    zero += o && !r;
    if (slot % 3 == 0) tris += c_tri_count[S.tc[(size_t)b * kNC + slot / 3]];
  }
  occ = warp_sum(occ); missing = warp_sum(missing); zero = warp_sum(zero); tris = warp_sum(tris);
  if ((threadIdx.x & 31) == 0) {
    if (occ) atomicAdd(sums + 0, (unsigned long long)occ);
    if (missing) atomicAdd(sums + 1, (unsigned long long)missing);
    if (zero) atomicAdd(sums + 2, (unsigned long long)zero);
    if (tris) atomicAdd(sums + 3, (unsigned long long)tris);
  }
}

// Vertex-record ownership (audit): every record handed out (< a_hw) belongs
// to at most one holder -- a slot with its has-record bit, or a gc CTA's free
// range.  claims[h] counts the holders; every claim past the first, and every
// record-holding slot whose handle lies outside [0, a_hw), is counted in
// out[0] (the report's duplicate_handles).
__global__ void k_audit_records(DevState S, int nblocks, long long a_hw, int32_t *claims, unsigned long long *out) {
  long long dup = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)nblocks * kEV; q += stride) {
    if (!((S.vrb[q >> 5] >> (q & 31)) & 1u)) continue;
    const long long h = S.vh[q];
    if (h < 0 || h >= a_hw) { dup++; continue; }
    dup += atomicAdd(claims + h, 1) > 0;
  }
  // the gc CTAs' free ranges [s_rr[0], s_rr[1]), [s_rr[2], s_rr[3])
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < 2LL * S.rec_chunk_ctas; c += stride) {
    const long long a = S.rec_chunk[2 * c], e = S.rec_chunk[2 * c + 1];
    for (long long h = a; h < e; h++) {
      if (h < 0 || h >= a_hw) { dup++; continue; }
      dup += atomicAdd(claims + h, 1) > 0;
    }
  }
  dup = warp_sum(dup);
  if ((threadIdx.x & 31) == 0 && dup) atomicAdd(out, (unsigned long long)dup);
}

__global__ void k_refine_eval(const uint8_t *tc, const uint8_t *tp, const double *corners, int n,
                              double eps, int32_t *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned cur = tc[i], prev = tp[i];
    unsigned small = 0;
    for (int k = 0; k < 8; k++) small |= (fabs(corners[(size_t)i * 8 + k]) < eps ? 1u : 0u) << k;
    if (__popc((cur ^ prev) & 0xFF) > 3) { out[i] = -1; continue; }
    bool ch;
    const unsigned r = refine_type(cur, prev, small, &ch);
    bool hit = false;   // detect_disturbance returns None when nothing qualifies
    for (int j = 0; j < 6; j++) {
      const unsigned diff = (cur ^ c_regular[j]) & 0xFF;
      if (__popc(diff) <= 3 && !(diff & ~small)) hit = true;
    }
    out[i] = hit ? (int)r : -1;
  }
}

__global__ void k_frustum_eval(DevState S, const FrameDev F, const int3 *coords, int n,
                               uint8_t *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int3 c = coords[i];
    out[i] = block_in_frustum_dev(make_int4(c.x, c.y, c.z, 0), F, S.extent);
  }
}

__global__ void k_scatter_samples(DevState S, const int32_t *idx, int n, const double *tsdf,
                                  const int32_t *weight) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)n * kNC;
       q += (long long)gridDim.x * blockDim.x) {
    const int b = idx[q / kNC];
    if (b < 0) continue;
    const size_t dst = (size_t)b * kNC + (q % kNC);
    if (tsdf) S.tsdf[dst] = tsdf[q];
    if (weight) S.weight[dst] = weight[q];
  }
}

// apply pending face-normal fallback records (before the engine state is read
// or changed outside fuse_frame)
__global__ void __launch_bounds__(128) k_flush_fallbacks(DevState S) {
  const int n = min(ld_vol(&S.ctr->fb_pending), S.fb_cap);
  const FallbackArgs A{S.ctr, S.fallback, S.nbr, S.bcoord, S.vparam, S.vrec, S.cube_size};
  for (int f = blockIdx.x * 4 + (threadIdx.x >> 5); f < n; f += (int)gridDim.x * 4) consume_fallback(A, f);
}

// phase API (mesher.extract_frame with an arbitrary halo): apply every pending
// placement request of every block (in fuse_frame k_gc_normals does it for the
// halo, which holds every block a scope cube can request a slot of)
__global__ void k_apply_claims(DevState S, int nblocks, int frame, int from_bytes) {
  long long allocs = 0;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)nblocks * (kEV / 32);
       q += (long long)gridDim.x * blockDim.x) {
    uint32_t claim = S.vclaim[q];
    if (from_bytes) {   // strategy "partition": k_place_parity's request bytes
      claim |= pack_requests(S.vreq + (size_t)q * 32);
      if (claim) clear_requests(S.vreq + (size_t)q * 32);
    }
    if (!claim) continue;
    const uint32_t old = S.vocc[q], fresh = claim & ~old;
    const long long b = q / (kEV / 32);
    for (uint32_t m = fresh; m; m &= m - 1) {
      const size_t sl = (size_t)q * 32 + __ffs(m) - 1;
      int h = S.vh[sl];
      if (h < 0) {   // (first occupation: a new record; the caller's retype checked the capacity)
        h = (int)atomicAdd((unsigned long long *)&S.ctr->a_hw, 1ull);
        S.vh[sl] = h;
        atomicOr(S.vrb + (sl >> 5), 1u << (sl & 31));
      }
      S.vrec[h].birth = frame;
      S.vrec[h].nrm[0] = 0.0; S.vrec[h].nrm[1] = 0.0; S.vrec[h].nrm[2] = 0.0;
    }
    if (S.nranks <= 1 || S.bowned[b]) allocs += __popc(fresh);
    S.vocc[q] = old | claim;
    S.vclaim[q] = 0u;
  }
  allocs = warp_sum(allocs);
  if ((threadIdx.x & 31) == 0 && allocs) atomicAdd((unsigned long long *)&S.ctr->v_allocs, (unsigned long long)allocs);
}

// per-slot views of the vertex records of listed blocks (export): birth (-1
// empty) and normal (0 when empty)
__global__ void k_gather_slots(DevState S, const int32_t *idx, int n, int32_t *birth, double *normal) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)n * kEV;
       q += (long long)gridDim.x * blockDim.x) {
    const size_t sq = (size_t)idx[q / kEV] * kEV + (size_t)(q % kEV);
    const bool occ = (S.vocc[sq >> 5] >> (sq & 31)) & 1u;
    const int h = occ ? S.vh[sq] : -1;
    if (birth) birth[q] = h >= 0 ? S.vrec[h].birth : -1;
    if (normal)
      for (int d = 0; d < 3; d++) normal[3 * q + d] = h >= 0 ? S.vrec[h].nrm[d] : 0.0;
  }
}

// ... and back (import): every slot with birth >= 0 gets a record (the host
// sized the arena and writes the occupancy bits)
__global__ void k_scatter_slots(DevState S, const int32_t *idx, int n, const int32_t *birth, const double *normal) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)n * kEV;
       q += (long long)gridDim.x * blockDim.x) {
    if (birth[q] < 0) continue;
    const size_t sq = (size_t)idx[q / kEV] * kEV + (size_t)(q % kEV);
    int h = S.vh[sq];
    if (h < 0) {
      h = (int)atomicAdd((unsigned long long *)&S.ctr->a_hw, 1ull);
      S.vh[sq] = h;
      atomicOr(S.vrb + (sq >> 5), 1u << (sq & 31));
    }
    S.vrec[h].birth = birth[q];
    for (int d = 0; d < 3; d++) S.vrec[h].nrm[d] = normal ? normal[3 * q + d] : 0.0;
  }
}

// validity bitmap of listed blocks from their weights (after host writes)
__global__ void k_rebuild_vmask(DevState S, const int32_t *idx, int n) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)n * (kNC / 32);
       q += (long long)gridDim.x * blockDim.x) {
    const int b = idx[q / (kNC / 32)];
    if (b < 0) continue;
    const int w = (int)(q % (kNC / 32));
    uint32_t bits = 0;
    for (int k = 0; k < 32; k++) bits |= (S.weight[(size_t)b * kNC + w * 32 + k] > 0 ? 1u : 0u) << k;
    S.vmask[(size_t)b * (kNC / 32) + w] = bits;
  }
}

// ------------------------------------------------------------ compaction
// store.py:388-425: blocks in sorted-coordinate order, vertices in (x,y,z,axis)
// slot order, triangles in (x,y,z,slot) order, dense remap of handles.
__global__ void k_block_keys(DevState S, int nblocks, unsigned long long *keys, int32_t *vals) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nblocks; i += gridDim.x * blockDim.x) {
    const int4 c = S.bcoord[i];
    keys[i] = c.w ? ~0ull : (unsigned long long)pack_coord(c.x, c.y, c.z);   // (evicted blocks last)
    vals[i] = i;
  }
}

// per sorted block: occupied slots, triangles; also the 1536-bit occupancy
// mask and per-32-slot prefix counts used for O(1) slot -> dense index
__global__ void __launch_bounds__(kThreadsCube) k_compact_count(DevState S, const int32_t *order, int nblocks,
                                                                int32_t *vcnt, int32_t *tcnt,
                                                                uint32_t *occ_bits, uint16_t *occ_pre) {
  __shared__ long long red[32];
  __shared__ int wc[48];
  for (int i = blockIdx.x; i < nblocks; i += gridDim.x) {
    const int b = order[i];
    const int t = threadIdx.x;
    if (t < 48) {   // the occupancy words as they are
      const uint32_t ball = S.vocc[(size_t)b * 48 + t];
      occ_bits[(size_t)b * 48 + t] = ball;
      wc[t] = __popc(ball);
    }
    __syncthreads();
    if (t == 0) {
      int acc = 0;
      for (int w = 0; w < 48; w++) { occ_pre[(size_t)b * 48 + w] = (uint16_t)acc; acc += wc[w]; }
      vcnt[i] = acc;
    }
    const long long nt = block_sum(c_tri_count[S.tc[(size_t)b * kNC + t]], red);
    if (t == 0) tcnt[i] = (int)nt;
    __syncthreads();
  }
}

__global__ void k_block_base(const int32_t *order, const int32_t *vbase, int nblocks, int32_t *vbase_by_blk) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nblocks; i += gridDim.x * blockDim.x)
    vbase_by_blk[order[i]] = vbase[i];
}

__device__ __forceinline__ int slot_index(const uint32_t *occ_bits, const uint16_t *occ_pre,
                                          const int32_t *vbase_by_blk, int b, int s) {
  const int w = s >> 5;
  return vbase_by_blk[b] + occ_pre[(size_t)b * 48 + w] +
         __popc(occ_bits[(size_t)b * 48 + w] & ((1u << (s & 31)) - 1));
}

__global__ void __launch_bounds__(kThreadsCube) k_compact_vertices(DevState S, const int32_t *order, int nblocks,
                                                                   const uint32_t *occ_bits, const uint16_t *occ_pre,
                                                                   const int32_t *vbase_by_blk, double *pos,
                                                                   double *nrm, long long *ages, long long frame,
                                                                   int32_t *ev_handles) {
  for (int i = blockIdx.x; i < nblocks; i += gridDim.x) {
    const int b = order[i];
    for (int s = threadIdx.x; s < kEV; s += blockDim.x) {
      const size_t q = (size_t)b * kEV + s;
      int o = -1;
      if ((occ_bits[(size_t)b * 48 + (s >> 5)] >> (s & 31)) & 1u) {
        const VertexRec &vr = S.vrec[S.vh[q]];
        o = slot_index(occ_bits, occ_pre, vbase_by_blk, b, s);
        slot_position(S, b, s, pos + 3 * (size_t)o);
        for (int d = 0; d < 3; d++) nrm[3 * (size_t)o + d] = vr.nrm[d];
        ages[o] = frame - (long long)vr.birth;
      }
      if (ev_handles) ev_handles[q] = o;
    }
  }
}

__device__ __forceinline__ int block_rank(int v, int *sh, int *tot) {
  // block-wide exclusive scan of small ints (blockDim = 512)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  __syncthreads();
  if (lane == 31) sh[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int w = 0; w < nw; w++) { const int c = sh[w]; sh[w] = acc; acc += c; }
    sh[32] = acc;
  }
  __syncthreads();
  *tot = sh[32];
  return sh[wid] + incl - v;
}

__global__ void __launch_bounds__(kThreadsCube) k_compact_triangles(DevState S, const int32_t *order, int nblocks,
                                                                    const int32_t *tbase, const uint32_t *occ_bits,
                                                                    const uint16_t *occ_pre,
                                                                    const int32_t *vbase_by_blk, int32_t *idx,
                                                                    int32_t *tri_handles) {
  __shared__ int sh[33];
  for (int i = blockIdx.x; i < nblocks; i += gridDim.x) {
    const int b = order[i];
    const int t = threadIdx.x;
    const int x = t >> 6, y = (t >> 3) & 7, z = t & 7;
    const unsigned tt = S.tc[(size_t)b * kNC + t];
    const int ntri = c_tri_count[tt];
    int tot;
    const int r = block_rank(ntri, sh, &tot);
    const unsigned long long packed = c_tri_packed[tt];
    for (int j = 0; j < ntri; j++) {
      const int o = tbase[i] + r + j;
      for (int k = 0; k < 3; k++) {
        const int e = (int)((packed >> (4 * (3 * j + k))) & 0xF);
        const int own = c_e_own[e];
        const int ox = x + (own & 1), oy = y + ((own >> 1) & 1), oz = z + ((own >> 2) & 1);
        const int dir = nbr_dir(ox >> 3, oy >> 3, oz >> 3);
        const int ob = (dir == 13) ? b : S.nbr[(size_t)b * 27 + dir];
        const int s = ((ox & 7) * 64 + (oy & 7) * 8 + (oz & 7)) * 3 + c_e_axis[e];
        int m = -1;
        if (ob >= 0 && ((S.vocc[(size_t)ob * 48 + (s >> 5)] >> (s & 31)) & 1u))
          m = slot_index(occ_bits, occ_pre, vbase_by_blk, ob, s);
        else set_error(S, ERR_CONSISTENCY, 40, b);
        idx[3 * (size_t)o + k] = m;
      }
    }
    if (tri_handles)
      for (int j = 0; j < 5; j++) tri_handles[((size_t)b * kNC + t) * 5 + j] = j < ntri ? tbase[i] + r + j : -1;
    __syncthreads();
  }
}

// snapshot helper: per-slot reference counts (VertexPool.refcount view)
__global__ void k_slot_refcounts(DevState S, int nblocks, const int32_t *ev_handles, int32_t *refcount) {
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)nblocks * kEV;
       q += (long long)gridDim.x * blockDim.x) {
    const int h = ev_handles[q];
    if (h >= 0) refcount[h] = slot_refcount(S, (int)(q / kEV), (int)(q % kEV));
  }
}

}  // namespace vm
