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

enum { F_INIT = 1, F_INTEGRATE = 2, F_SCOPE = 4 };
enum { G_GC = 1, G_NORMALS = 2, G_COMMIT = 4, G_REQUIRE_ITEMS = 8 };

// error and need are adjacent: one 8-byte load
__device__ __forceinline__ bool halted(const DevState &S) {
  const int2 v = __ldcg(reinterpret_cast<const int2 *>(&S.ctr->error));
  return (v.x | v.y) != 0;
}

__device__ __forceinline__ int list_count(const int32_t *count_ptr, int count_const) {
  return count_ptr ? ld_vol(count_ptr) : count_const;
}

// ------------------------------------------------------------ depth stats
__global__ void __launch_bounds__(256) k_depth_stats(DevState S, const FrameDev F) {
  cudaGridDependencySynchronize();   // PDL: wait for the previous kernel of the frame
  __shared__ double smax[8];
  __shared__ int scnt[8];
  const long long npix = (long long)F.h * F.w;
  double best = -1.0;
  int cnt = 0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
       p += (long long)gridDim.x * blockDim.x) {
    const double d = F.depth[p];
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
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) { best = fmax(best, smax[w]); cnt += scnt[w]; }
    if (cnt) {
      atomicAdd(&S.ctr->nvalid, cnt);
      atomicMax(&S.ctr->maxnorm_bits, (unsigned long long)__double_as_longlong(best));
    }
  }
}

// ------------------------------------------------------------ norm bounds
// min / max ray norm over every pixel of an (h, w) image (positive doubles
// order as their bit patterns).  The band step count is monotone in the max
// norm over the VALID pixels, which lies between the two, so when both bounds
// give the same count the frame needs no depth reduction (fusion.py:88-94).
__global__ void k_norm_bounds(const FrameDev F, unsigned long long *out) {
  const long long npix = (long long)F.h * F.w;
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

// ------------------------------------------------------------ collect
// One thread per pixel looping over the nsteps band samples.  Samples of a
// warp falling in the same block are merged with __match_any_sync, so one
// lane per distinct block probes the hash table.  A warp covers an 8x4 pixel
// tile (blocks project to compact image regions, so fewer distinct blocks per
// warp than a 32-pixel row).
__global__ void __launch_bounds__(256) k_collect(DevState S, const FrameDev F) {
  cudaGridDependencySynchronize();   // PDL: wait for the previous kernel of the frame
  Counters *ctr = S.ctr;
  int nsteps = F.nsteps_fixed;
  if (nsteps <= 0) {
    if (ld_vol(&ctr->nvalid) == 0) return;
    const double maxnorm = __longlong_as_double((long long)ld_vol(&ctr->maxnorm_bits));
    const double half_block = S.extent * 0.5;
    const double band = __dmul_rn(__dmul_rn(2.0, F.trunc), maxnorm);
    nsteps = (int)ceil(band / half_block) + 1;
    if (nsteps < 2) nsteps = 2;
  }
  const double step = 2.0 / (double)(nsteps - 1);
  const int lane = threadIdx.x & 31;
  // warp tiles of 8x4 pixels, row-major over the tile grid
  const int tiles_x = (F.w + 7) >> 3, tiles_y = (F.h + 3) >> 2;
  const long long ntiles = (long long)tiles_x * tiles_y;
  const long long wstride = (long long)gridDim.x * (blockDim.x >> 5);
  int nvalid = 0;
  for (long long tile = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); tile < ntiles;
       tile += wstride) {
    const int ty = (int)(tile / tiles_x), tx = (int)(tile - (long long)ty * tiles_x);
    const int u = tx * 8 + (lane & 7), v = ty * 4 + (lane >> 3);
    double d = 0.0, qs[3] = {0, 0, 0};
    bool valid = false;
    if (u < F.w && v < F.h) {
      d = F.depth[(long long)v * F.w + u];
      valid = d > 0 && d <= F.max_range;
    }
    if (valid) {
      nvalid++;
      const double rx = ((double)u - F.cx) / F.fx, ry = ((double)v - F.cy) / F.fy;
      const double pc[3] = {__dmul_rn(rx, d), __dmul_rn(ry, d), __dmul_rn(1.0, d)};
      for (int j = 0; j < 3; j++) qs[j] = matvec_row(pc, F.R, j);   // pts_cam @ R.T
    }
    if (!__any_sync(0xffffffffu, valid)) continue;
    const double delta = valid ? F.trunc / d : 0.0;
    for (int i = 0; i < nsteps; i++) {
      long long key = kEmptyKey;
      int c[3] = {0, 0, 0};
      if (valid) {
        const double s = (i == nsteps - 1) ? 1.0 : __dadd_rn(__dmul_rn((double)i, step), -1.0);
        const double f = __dadd_rn(1.0, __dmul_rn(s, delta));
        for (int j = 0; j < 3; j++)
          c[j] = (int)floor(__dadd_rn(F.t[j], __dmul_rn(qs[j], f)) / S.extent);
        if (block_relevant(S, c[0], c[1], c[2])) key = pack_coord(c[0], c[1], c[2]);
      }
      const unsigned grp = __match_any_sync(0xffffffffu, key);
      if (key != kEmptyKey && lane == __ffs(grp) - 1) {
        HashRef r = hash_find_ref(S, c[0], c[1], c[2]);
        if (r.idx == -1) r = hash_insert_ref(S, c[0], c[1], c[2], F.epoch);
        if (r.idx >= 0 && r.stamp != F.epoch && atomicExch(r.stamp_ptr, F.epoch) != F.epoch)
          S.scope[atomicAdd(&ctr->ncollected, 1)] = r.idx;
      }
    }
  }
  if (F.nsteps_fixed > 0) {   // valid-pixel count (k_depth_stats did not run): one atomic per CTA
    __shared__ int s_valid;
    if (threadIdx.x == 0) s_valid = 0;
    __syncthreads();
    nvalid = warp_sum(nvalid);
    if (lane == 0 && nvalid) atomicAdd(&s_valid, nvalid);
    __syncthreads();
    if (threadIdx.x == 0 && s_valid) atomicAdd(&ctr->nvalid, s_valid);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->nsteps = nsteps;
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
  int32_t *vb = S.vbirth + (size_t)b * kEV;
  vb[t] = -1;
  vb[t + kNC] = -1;
  vb[t + 2 * kNC] = -1;
}

__global__ void __launch_bounds__(kThreadsCube) k_init_blocks(DevState S) {
  if (halted(S)) return;
  const int nnew = ld_vol(&S.ctr->nnew);
  for (int i = blockIdx.x; i < nnew; i += gridDim.x) {
    const int b = S.newlist[i];
    init_block(S, b, threadIdx.x);
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
//  F_SCOPE     27-neighbour halo marking and minus-slab scope marking
//              (mesher.py:499-543), with hash lookups (links of blocks
//              created in this launch are still being written).
constexpr int kFB = 128;   // threads per CTA of k_fuse_blocks (4 corners each)

__global__ void __launch_bounds__(kFB, 6) k_fuse_blocks(DevState S, const FrameDev F,
                                                     const int32_t *__restrict__ list,
                                                     const int32_t *__restrict__ count_ptr,
                                                     int count_const, int flags) {
  cudaGridDependencySynchronize();   // PDL: wait for the previous kernel of the frame
  const bool stop = halted(S);
  const int n = list_count(count_ptr, count_const);   // issued together with the halt check
  if (stop) return;
  const int t = threadIdx.x;
  // neighbour probe of this thread: 7 lanes of each warp, directions 0..26
  const int pl = t & 31, pdir = (t >> 5) * 7 + pl;
  const bool prober = pl < 7 && pdir < 27;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int b = __ldcg(list + i);
    if (b < 0) continue;
    const int4 c = __ldcg(S.bcoord + b);
    const bool fresh = (flags & F_INIT) && __ldcg(S.stamp_new + b) == F.epoch;
    // fusion.py:138-168, four corners per thread.  The old state of the corners
    // is requested first, so its round trip overlaps the projections and the
    // depth gathers.
    double t_old[kNC / kFB], zc[kNC / kFB], meas[kNC / kFB];
    int w_old[kNC / kFB];
    bool ok[kNC / kFB];
    if (flags & F_INTEGRATE) {
#pragma unroll
      for (int j = 0; j < kNC / kFB; j++) {
        const size_t q = (size_t)b * kNC + t + j * kFB;
        t_old[j] = fresh ? 0.0 : S.tsdf[q];
        w_old[j] = fresh ? 0 : S.weight[q];
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
    if ((flags & (F_SCOPE | F_INIT)) && prober) {
      const int dx = pdir / 9 - 1, dy = (pdir / 3) % 3 - 1, dz = pdir % 3 - 1;
      int nb = b, nb_collected = 1;
      if (pdir != 13) {
        const HashRef r = hash_find_ref(S, c.x + dx, c.y + dy, c.z + dz);
        nb = r.idx;
        nb_collected = r.stamp == F.epoch;
      }
      if (fresh) {
        S.nbr[(size_t)b * 27 + pdir] = nb;
        if (nb >= 0 && pdir != 13) S.nbr[(size_t)nb * 27 + (26 - pdir)] = b;
      }
      if ((flags & F_SCOPE) && nb >= 0) {
        if (ld_vol(S.stamp_halo + nb) != F.epoch && atomicExch(S.stamp_halo + nb, F.epoch) != F.epoch)
          S.halo[atomicAdd(&S.ctr->nhalo, 1)] = nb;
        // minus neighbour n = c - o, o in {0,1}^3 \ 0, not itself collected
        if (dx <= 0 && dy <= 0 && dz <= 0 && pdir != 13 && !nb_collected) {
          const int o = (-dx) * 4 + (-dy) * 2 + (-dz);
          const unsigned sh = 8 * (nb & 3);
          const unsigned old = atomicOr((unsigned *)(S.slab_bits + (nb & ~3)), (1u << (o - 1)) << sh);
          if (((old >> sh) & 0xFF) == 0)
            S.scope[ld_vol(&S.ctr->ncollected) + atomicAdd(&S.ctr->nslab, 1)] = nb;
        }
      }
    }
    if (!(flags & F_INTEGRATE)) continue;
#pragma unroll
    for (int j = 0; j < kNC / kFB; j++) {
      if (!ok[j]) continue;
      const double m = meas[j];
      if (!(m > 0 && m <= F.max_range)) continue;
      const double sdf = m - zc[j];
      if (!(sdf >= -F.trunc)) continue;
      double dn = sdf / F.trunc;
      dn = dn < -1.0 ? -1.0 : (dn > 1.0 ? 1.0 : dn);
      const size_t q = (size_t)b * kNC + t + j * kFB;
      const double wo = (double)w_old[j];
      S.tsdf[q] = __dadd_rn(__dmul_rn(wo, t_old[j]), dn) / __dadd_rn(wo, 1.0);
      const long long nw = (long long)w_old[j] + 1;
      S.weight[q] = (int)(nw < F.weight_cap ? nw : F.weight_cap);
    }
  }
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

// ------------------------------------------------------------ tile loaders
// the block's 27-neighbour row, cached in shared memory (one round trip)
__device__ __forceinline__ void load_nbr_row(const DevState &S, int b, int *s_nbr) {
  if (threadIdx.x < 27) s_nbr[threadIdx.x] = threadIdx.x == 13 ? b : S.nbr[(size_t)b * 27 + threadIdx.x];
}

// (B+1)^3 tile of a block plus its 7 plus-neighbours (mesher.py:75-96):
// tsdf and the "weight > 0" flag.
__device__ __forceinline__ void load_ext_tile(const DevState &S, int b, const int *s_nbr, double *tile,
                                              uint8_t *tw) {
  const int t = threadIdx.x;
  {
    const int x = t >> 6, y = (t >> 3) & 7, z = t & 7;
    const size_t q = (size_t)b * kNC + t;
    tile[(x * 9 + y) * 9 + z] = S.tsdf[q];
    tw[(x * 9 + y) * 9 + z] = S.weight[q] > 0;
  }
  if (t < 217) {
    int x, y, z;   // the 217 tile positions with max(x, y, z) == 8
    if (t < 64) { x = 8; y = t >> 3; z = t & 7; }
    else if (t < 128) { x = (t - 64) >> 3; y = 8; z = t & 7; }
    else if (t < 192) { x = (t - 128) >> 3; y = t & 7; z = 8; }
    else if (t < 200) { x = 8; y = 8; z = t - 192; }
    else if (t < 208) { x = 8; y = t - 200; z = 8; }
    else if (t < 216) { x = t - 208; y = 8; z = 8; }
    else { x = 8; y = 8; z = 8; }
    const int nb = s_nbr[nbr_dir(x >> 3, y >> 3, z >> 3)];
    double v = 0.0;
    uint8_t w = 0;
    if (nb >= 0) {
      const size_t q = (size_t)nb * kNC + ((x & 7) * 64 + (y & 7) * 8 + (z & 7));
      v = S.tsdf[q];
      w = S.weight[q] > 0;
    }
    tile[(x * 9 + y) * 9 + z] = v;
    tw[(x * 9 + y) * 9 + z] = w;
  }
}

__device__ __forceinline__ int item_count(const DevState &S, const FrameDev &F) {
  if (F.scope_mode != 0) return __ldcg(&S.ctr->nexplicit);
  const int2 v = __ldcg(reinterpret_cast<const int2 *>(&S.ctr->ncollected));   // ncollected, nnew
  return v.x + __ldcg(&S.ctr->nslab);
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

// ------------------------------------------------------------ retype + place
// One CTA per scope item (persistent over the item list), one thread per cube
// for typing.  Software-pipelined: while block i is typed and placed, the
// neighbour row and the 9^3 tsdf/weight tile + type row of the CTA's next
// block stream into the other shared-memory buffer with cp.async (LDGSTS).
// Typing and refinement as the reference; a cube whose type changed is
// retriangulated implicitly (its triangles become TRI_TABLE[type_curr]) and
// contributes the triangle / irregular-count deltas.  The (active cube, mask
// edge) placements are compacted in shared memory and spread over the CTA:
// each claims its edge slot (atomicCAS on the slot's birth word -- exactly one
// allocation per edge) and writes the interpolated coordinate; all requesters
// produce identical bits (mesher.py:216-235).
constexpr int kMaxPlace = kNC * 12;

// Tile-source tables (filled by vm_create): for every staged tile position,
// the neighbour direction (0..26) and the source cube index in that block,
// so the loaders do no div/mod index arithmetic.
__device__ uint32_t g_ext_tab[217];   // 9^3 tile position | dir << 10 | src << 15 (positions with a coord == 8)
__device__ uint16_t g_sten_tab[1331]; // dir << 9 | src, 11^3 stencil over locals -1..9
__device__ uint16_t g_type_tab[729];  // dir << 9 | src, 9^3 type tile over locals -1..7

// Per-item "resolved" record (three in flight: computing, staged, resolving)
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
  const int lane = threadIdx.x;
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
  const int lane = threadIdx.x;
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

constexpr int kNT = 128;   // threads per CTA of the per-block meshing kernels (4 cubes each)

// One CTA of 128 threads per scope item (persistent over the item list).
// Small CTAs keep ~8 blocks in flight per SM so their serial phases (resolve,
// staging, typing, placement) overlap across blocks.  Typing and refinement
// as the reference; a cube whose type changed is retriangulated implicitly
// (its triangles become TRI_TABLE[type_curr]) and contributes the triangle /
// irregular-count deltas.  The (active cube, mask edge) placements are
// compacted in shared memory and spread over the CTA: each claims its edge
// slot (atomicCAS on the slot's birth word -- exactly one allocation per
// edge) and writes the interpolated coordinate; all requesters produce
// identical bits (mesher.py:216-235).
__global__ void __launch_bounds__(kNT, 8) k_retype_place(DevState S, const FrameDev F) {
  cudaGridDependencySynchronize();   // PDL: wait for the previous kernel of the frame
  if (halted(S)) return;
  __shared__ double tile[729];
  __shared__ uint8_t tw[729];
  __shared__ __align__(16) uint8_t s_tc[kNC];
  __shared__ uint16_t s_place[kMaxPlace];
  __shared__ Resolved R;
  __shared__ long long red8[8 * 32];
  __shared__ int s_nplace;
  const int n = item_count(S, F);
  const int nc = __ldcg(&S.ctr->ncollected);
  const int t = threadIdx.x;
  const double l = S.cube_size;
  const int frame = F.frame;
  const int do_refine = F.refine;
  const double eps = F.epsilon;
  long long allocs = 0, placements = 0, active = 0, changed = 0, t_rel = 0, t_new = 0, irr = 0,
            refined = 0, live = 0;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    if (t < 32) {
      const int b = __ldcg(S.scope + i);
      const ResolveRegs rr = resolve_load(S, F, b, i, nc);
      resolve_store(S, F, rr, b, i, n, nc, R);
    }
    if (t == 0) s_nplace = 0;
    __syncthreads();
    const int mode = R.mode;
    if (mode <= 0) {
      __syncthreads();
      continue;
    }
    const int b = R.b;
    const int own = R.owned;
    if (t == 0) live++;
    // stage the (B+1)^3 tile (mesher.py:75-96) and the current types
    {
      // batched gathers: all loads in flight before any shared-memory store
      double ov[kNC / kNT], xv[2];
      int ow[kNC / kNT], xw[2], xp[2];
      uint4 tcv = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < kNC / kNT; j++) {
        ov[j] = S.tsdf[(size_t)b * kNC + t + j * kNT];
        ow[j] = S.weight[(size_t)b * kNC + t + j * kNT];
      }
      if (t < 32) tcv = reinterpret_cast<const uint4 *>(S.tc + (size_t)b * kNC)[t];
#pragma unroll
      for (int j = 0; j < 2; j++) {
        const int q = t + j * kNT;
        xv[j] = 0.0;
        xw[j] = 0;
        xp[j] = -1;
        if (q < 217) {
          const uint32_t e = __ldg(&g_ext_tab[q]);
          const int nb = R.nbr[(e >> 10) & 31];
          xp[j] = e & 1023;
          if (nb >= 0) {
            const size_t src = (size_t)nb * kNC + (e >> 15);
            xv[j] = S.tsdf[src];
            xw[j] = S.weight[src];
          }
        }
      }
#pragma unroll
      for (int j = 0; j < kNC / kNT; j++) {
        const int c = t + j * kNT;
        const int p = ((c >> 6) * 9 + ((c >> 3) & 7)) * 9 + (c & 7);
        tile[p] = ov[j];
        tw[p] = ow[j] > 0;
      }
      if (t < 32) reinterpret_cast<uint4 *>(s_tc)[t] = tcv;
#pragma unroll
      for (int j = 0; j < 2; j++)
        if (xp[j] >= 0) {
          tile[xp[j]] = xv[j];
          tw[xp[j]] = xw[j] > 0;
        }
    }
    __syncthreads();
#pragma unroll 1
    for (int j = 0; j < kNC / kNT; j++) {
      const int c = t + j * kNT;
      const int x = c >> 6, y = (c >> 3) & 7, z = c & 7;
      bool sel;
      if (mode == 1) sel = true;
      else if (mode == 2) sel = (R.slab & c_slab_sel[((x == 7) << 2) | ((y == 7) << 1) | (z == 7)]) != 0;
      else sel = (S.item_mask[(size_t)R.item * 16 + (c >> 5)] >> (c & 31)) & 1;
      unsigned bits = 0, small = 0;
      const int base = (x * 9 + y) * 9 + z;
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const int o = c_corner[k];
        const int e = base + (o & 1) * 81 + ((o >> 1) & 1) * 9 + ((o >> 2) & 1);
        const double cv = tile[e];
        sel = sel && tw[e];
        bits |= (cv < 0.0 ? 1u : 0u) << k;
        small |= (fabs(cv) < eps ? 1u : 0u) << k;
      }
      unsigned mask = 0;
      if (sel) {
        const unsigned tp = s_tc[c];
        unsigned tc = bits;
        if (do_refine) {
          bool ch;
          tc = refine_type(bits, tp, small, &ch);
          refined += ch && own;
        }
        const size_t q = (size_t)b * kNC + c;
        S.tp[q] = (uint8_t)tp;
        S.tc[q] = (uint8_t)tc;
        if (tc != tp && own) {
          changed++;
          const int nold = c_tri_count[tp], nnew = c_tri_count[tc];
          t_rel += nold;
          t_new += nnew;
          irr += (nnew > 0 && !is_regular_type(tc)) - (nold > 0 && !is_regular_type(tp));
        }
        mask = c_edge_mask[tc];
        if (mask && own) {
          active++;
          placements += __popc(mask);
        }
      }
      int pos = smem_append(__popc(mask), &s_nplace);
      while (mask) {
        const int e = __ffs(mask) - 1;
        mask &= mask - 1;
        s_place[pos++] = (uint16_t)((c << 4) | e);
      }
    }
    __syncthreads();
    const int np = s_nplace;
    for (int p = t; p < np; p += kNT) {
      const int ent = s_place[p];
      const int ci = ent >> 4, e = ent & 15;
      const int own = c_e_own[e], axis = c_e_axis[e];
      const int ox = (ci >> 6) + (own & 1), oy = ((ci >> 3) & 7) + ((own >> 1) & 1), oz = (ci & 7) + ((own >> 2) & 1);
      const int owner = R.nbr[nbr_dir(ox >> 3, oy >> 3, oz >> 3)];
      if (owner < 0) {
        set_error(S, ERR_CONSISTENCY, 10, R.coord.x * kB + (ci >> 6), R.coord.y * kB + ((ci >> 3) & 7),
                  R.coord.z * kB + (ci & 7));
        continue;
      }
      const size_t slot = (size_t)owner * kEV + (((ox & 7) * 64 + (oy & 7) * 8 + (oz & 7)) * 3 + axis);
      // start corner = owner cube origin; end corner one step along the axis
      const int p0 = (ox * 9 + oy) * 9 + oz;
      const double d0 = tile[p0];
      const double d1 = tile[p0 + (axis == 0 ? 81 : axis == 1 ? 9 : 1)];
      const double param = (d0 == d1) ? 0.5 : d0 / (d0 - d1);
      const int ga = (axis == 0 ? R.coord.x * kB + ox : axis == 1 ? R.coord.y * kB + oy : R.coord.z * kB + oz);
      S.vparam[slot] = __dadd_rn(__dmul_rn((double)ga, l), __dmul_rn(param, l));
      if (atomicCAS(S.vbirth + slot, -1, frame) == -1) {
        allocs += (S.nranks <= 1 || S.bowned[owner]);   // counted by the slot's owning rank
        S.vnrm[3 * slot] = 0.0; S.vnrm[3 * slot + 1] = 0.0; S.vnrm[3 * slot + 2] = 0.0;
      }
    }
    __syncthreads();   // R, tile and the placement list are rewritten by the next item
  }
  {
    long long vals[8] = {allocs, placements, active, changed, t_rel, t_new, irr, refined};
    int64_t *const dst[8] = {&S.ctr->v_allocs, &S.ctr->placements, &S.ctr->active, &S.ctr->changed,
                             &S.ctr->t_released, &S.ctr->t_allocated, &S.ctr->irr_delta, &S.ctr->refined};
    block_add_counters<8>(vals, red8, dst);
  }
  if (t == 0 && live) atomicAdd(&S.ctr->nitems_live, (int)live);
}
constexpr size_t kRetypeSmem = 0;



// ------------------------------------------------------------ GC + normals
// edge index, in the neighbour cube owner - du*e_u - dw*e_w, of the edge slot
// owned along `axis` (u, w the other two axes)
__device__ __forceinline__ int cube_edge_of_slot(int axis, int du, int dw) {
  const int u = axis == 0 ? 1 : 0, w = axis == 2 ? 1 : 2;
  const int own = (du << u) | (dw << w);
  return c_edge_of[axis][own];
}

// type of the cube at local (l0, l1, l2) in [-1, 7]^3 from the staged words
// (each word is the aligned 4 bytes of tc holding the cube's type)
__device__ __forceinline__ int staged_type(const uint32_t *ttw, int l0, int l1, int l2) {
  return (ttw[((l0 + 1) * 9 + (l1 + 1)) * 9 + (l2 + 1)] >> (8 * (l2 & 3))) & 0xFF;
}

// Face-normal fallback for one vertex, computed by one warp (mesher.py:459-486).
// Lane l handles candidate (incident cube j = l / 5, triangle slot s = l % 5);
// the contributions are then summed by lane 0 in the reference's order:
// vertex position k major, then halo blocks in sorted order, then cube, then
// triangle slot -- so the result is bit-identical to np.add.at's.
__device__ void fallback_normal_warp(const DevState &S, const uint8_t *ttile, const int *s_nbr, int4 bc,
                                     int slot_ci, int axis, int epoch, double *dst) {
  const int lane = threadIdx.x & 31;
  const int lx = slot_ci >> 6, ly = (slot_ci >> 3) & 7, lz = slot_ci & 7;
  const int u = axis == 0 ? 1 : 0, w = axis == 2 ? 1 : 2;
  // cube candidates j = 0..3: (du, dw) = (j >> 1, j & 1)
  int cj = -1, ckey = 0x7fffffff, ctt = 0, ce = 0;
  int cl[3] = {0, 0, 0};
  if (lane < 4) {
    const int du = lane >> 1, dw = lane & 1;
    int l[3] = {lx, ly, lz};
    l[u] -= du;
    l[w] -= dw;
    const int tt = ttile[((l[0] + 1) * 9 + (l[1] + 1)) * 9 + (l[2] + 1)];
    const int e = cube_edge_of_slot(axis, du, dw);
    const int dx = l[0] < 0 ? -1 : 0, dy = l[1] < 0 ? -1 : 0, dz = l[2] < 0 ? -1 : 0;
    const int nb = s_nbr[nbr_dir(dx, dy, dz)];
    if (((c_edge_mask[tt] >> e) & 1) && nb >= 0 && ld_vol(S.stamp_halo + nb) == epoch) {
      cj = lane;
      ckey = (((dx + 1) * 4 + (dy + 1) * 2 + (dz + 1)) << 9) | ((l[0] & 7) * 64 + (l[1] & 7) * 8 + (l[2] & 7));
      ctt = tt;
      ce = e;
      cl[0] = l[0]; cl[1] = l[1]; cl[2] = l[2];
    }
  }
  // rank of each cube candidate by (sorted block, cube) key
  int rank = 0;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const int kj = __shfl_sync(0xffffffffu, ckey, j);
    rank += (kj < ckey);
  }
  // lane l: candidate cube j = l / 5, triangle slot s = l % 5
  const int j = lane / 5, s = lane % 5;
  const int jj = j < 4 ? j : 0;
  const int my_valid = __shfl_sync(0xffffffffu, cj, jj) >= 0 && j < 4;
  const int tt = __shfl_sync(0xffffffffu, ctt, jj);
  const int e = __shfl_sync(0xffffffffu, ce, jj);
  const int jrank = __shfl_sync(0xffffffffu, rank, jj);
  const int c0 = __shfl_sync(0xffffffffu, cl[0], jj), c1 = __shfl_sync(0xffffffffu, cl[1], jj),
            c2 = __shfl_sync(0xffffffffu, cl[2], jj);
  int kpos = -1;
  double fn[3] = {0.0, 0.0, 0.0};
  if (my_valid && s < c_tri_count[tt]) {
    const unsigned long long packed = c_tri_packed[tt];
    for (int q = 0; q < 3; q++)
      if ((int)((packed >> (4 * (3 * s + q))) & 0xF) == e) kpos = q;
    if (kpos >= 0) {
      double p[3][3];
      for (int q = 0; q < 3; q++) {
        const int eq = (int)((packed >> (4 * (3 * s + q))) & 0xF);
        const int own = c_e_own[eq], ax = c_e_axis[eq];
        const int ox = c0 + (own & 1), oy = c1 + ((own >> 1) & 1), oz = c2 + ((own >> 2) & 1);
        const int ob = s_nbr[nbr_dir(ox < 0 ? -1 : ox >> 3, oy < 0 ? -1 : oy >> 3, oz < 0 ? -1 : oz >> 3)];
        const int g[3] = {bc.x * kB + ox, bc.y * kB + oy, bc.z * kB + oz};
        for (int d = 0; d < 3; d++) p[q][d] = __dmul_rn((double)g[d], S.cube_size);
        p[q][ax] = S.vparam[(size_t)ob * kEV + ((ox & 7) * 64 + (oy & 7) * 8 + (oz & 7)) * 3 + ax];
      }
      const double a[3] = {p[1][0] - p[0][0], p[1][1] - p[0][1], p[1][2] - p[0][2]};
      const double bb[3] = {p[2][0] - p[0][0], p[2][1] - p[0][1], p[2][2] - p[0][2]};
      fn[0] = __dmul_rn(a[1], bb[2]) - __dmul_rn(a[2], bb[1]);
      fn[1] = __dmul_rn(a[2], bb[0]) - __dmul_rn(a[0], bb[2]);
      fn[2] = __dmul_rn(a[0], bb[1]) - __dmul_rn(a[1], bb[0]);
    }
  }
  // ordered accumulation: k major, then cube rank, then triangle slot
  int mykey = kpos >= 0 ? (kpos * 4 + jrank) * 5 + s : (1 << 20);
  double acc[3] = {0.0, 0.0, 0.0};
  const int npend = __popc(__ballot_sync(0xffffffffu, kpos >= 0));
  for (int it = 0; it < npend; it++) {
    int best = mykey, bl = lane;   // pending lane with the smallest key
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int ok = __shfl_xor_sync(0xffffffffu, best, o), ol = __shfl_xor_sync(0xffffffffu, bl, o);
      if (ok < best || (ok == best && ol < bl)) { best = ok; bl = ol; }
    }
    acc[0] = __dadd_rn(acc[0], __shfl_sync(0xffffffffu, fn[0], bl));
    acc[1] = __dadd_rn(acc[1], __shfl_sync(0xffffffffu, fn[1], bl));
    acc[2] = __dadd_rn(acc[2], __shfl_sync(0xffffffffu, fn[2], bl));
    if (lane == bl) mykey = 1 << 20;
  }
  if (lane == 0) {
    const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(acc[0], acc[0]), __dmul_rn(acc[1], acc[1])),
                                      __dmul_rn(acc[2], acc[2])));
    if (nrm > 1e-20) {
      dst[0] = (-1.0 * acc[0]) / nrm;
      dst[1] = (-1.0 * acc[1]) / nrm;
      dst[2] = (-1.0 * acc[2]) / nrm;
    } else if (dst[0] == 0.0 && dst[1] == 0.0 && dst[2] == 0.0) {
      dst[2] = 1.0;
    }
  }
}

// Face-normal fallback worklist consumer: one warp per vertex; stages the
// vertex's block neighbour row and the 9^3 type tile entries it needs through
// shared memory, then runs the ordered warp accumulation.
constexpr int kFT = 128;
__global__ void __launch_bounds__(kFT) k_fallback(DevState S, const FrameDev F) {
  cudaGridDependencySynchronize();   // PDL: wait for the previous kernel of the frame
  if (halted(S)) return;
  __shared__ int s_nbr[kFT / 32][27];
  __shared__ uint8_t s_tt[kFT / 32][729];
  __shared__ int4 s_coord[kFT / 32];
  const int n = __ldcg(&S.ctr->nfallback);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int f = blockIdx.x * (kFT / 32) + w; f < n; f += gridDim.x * (kFT / 32)) {
    const int2 rec = S.fallback[f];
    const int b = rec.x, sl = rec.y;
    if (lane < 27) s_nbr[w][lane] = lane == 13 ? b : __ldcg(S.nbr + (size_t)b * 27 + lane);
    if (lane == 27) s_coord[w] = __ldcg(S.bcoord + b);
    __syncwarp();
    // only the types of the <= 4 cubes around the slot are read: stage those
    const int ci = sl / 3, axis = sl % 3;
    const int u = axis == 0 ? 1 : 0, ww = axis == 2 ? 1 : 2;
    if (lane < 4) {
      int l[3] = {ci >> 6, (ci >> 3) & 7, ci & 7};
      l[u] -= lane >> 1;
      l[ww] -= lane & 1;
      const int nb = s_nbr[w][nbr_dir(l[0] >> 3, l[1] >> 3, l[2] >> 3)];
      s_tt[w][((l[0] + 1) * 9 + (l[1] + 1)) * 9 + (l[2] + 1)] =
          nb >= 0 ? S.tc[(size_t)nb * kNC + ((l[0] & 7) * 64 + (l[1] & 7) * 8 + (l[2] & 7))] : 0;
    }
    __syncwarp();
    fallback_normal_warp(S, s_tt[w], s_nbr[w], s_coord[w], ci, axis, F.epoch, S.vnrm + 3 * ((size_t)b * kEV + sl));
    __syncwarp();
  }
}

constexpr int kGT = 64;   // threads per CTA of k_gc_normals

// tsdf / weight sample at block-local corner (lx, ly, lz) in [-1, 9]^3
__device__ __forceinline__ size_t sample_index(const int *s_nbr, int lx, int ly, int lz) {
  const int nb = s_nbr[nbr_dir(lx >> 3, ly >> 3, lz >> 3)];
  return nb < 0 ? ~(size_t)0 : (size_t)nb * kNC + ((lx & 7) * 64 + (ly & 7) * 8 + (lz & 7));
}

// One CTA of 64 threads per listed (halo) block; small shared footprint so
// every halo block of a frame is resident at once.  G_GC clears every
// occupied slot that no cube references any more (the reference's refcount ==
// 0 recycling: the 4 cubes around the edge are read from a staged 9^3 type
// tile); the surviving vertices are compacted and G_NORMALS gathers each
// vertex's 12-point stencil directly (mesher.py:400-439), the face-normal
// fallback one warp per vertex.  G_COMMIT: the last CTA folds the per-call
// deltas into the pool counters.
__global__ void __launch_bounds__(kGT, 16) k_gc_normals(DevState S, const FrameDev F,
                                                    const int32_t *__restrict__ list,
                                                    const int32_t *__restrict__ count_ptr,
                                                    int count_const, int mode) {
  cudaGridDependencySynchronize();   // PDL: wait for the previous kernel of the frame
  if (halted(S)) return;
  Counters *ctr = S.ctr;
  const bool run = !(mode & G_REQUIRE_ITEMS) || __ldcg(&ctr->nitems_live) > 0;
  __shared__ uint8_t tt[729];        // type_curr over cube locals -1..7
  __shared__ uint32_t occ[kEV / 32]; // slot occupancy bits
  __shared__ uint16_t s_vlist[kEV];
  __shared__ Resolved R;
  __shared__ int s_nv;
  __shared__ long long red[3 * 32];
  const int n = run ? (count_ptr ? __ldcg(count_ptr) : count_const) : 0;
  const int t = threadIdx.x, lane = t & 31;
  FrameDev Fr = F;
  Fr.scope_mode = 1;   // resolve as explicit items: no slab bits
  Fr.frustum_only = 0;
  long long frees = 0, computed = 0, fallbacks = 0;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    if (t < 32) {
      const int b = __ldcg(list + i);
      const ResolveRegs rr = resolve_load(S, Fr, b, i, 0);
      resolve_store(S, Fr, rr, b, i, n, 0, R);
    }
    if (t == 0) s_nv = 0;
    __syncthreads();
    if (R.mode <= 0) {
      __syncthreads();
      continue;
    }
    const int b = R.b;
    // stage slot occupancy and the type tile (batched: all loads in flight)
#pragma unroll
    for (int j0 = 0; j0 < kEV / kGT; j0 += 8) {
      int bv[8];
#pragma unroll
      for (int j = 0; j < 8; j++) bv[j] = S.vbirth[(size_t)b * kEV + (j0 + j) * kGT + t];
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const unsigned ball = __ballot_sync(0xffffffffu, bv[j] >= 0);
        if (lane == 0) occ[((j0 + j) * kGT + t) >> 5] = ball;
      }
    }
    {
      constexpr int kT = (729 + kGT - 1) / kGT;   // 12
      uint8_t tv[kT];
#pragma unroll
      for (int j = 0; j < kT; j++) {
        const int q = t + j * kGT;
        tv[j] = 0;
        if (q < 729) {
          const int e = __ldg(&g_type_tab[q]);
          const int nb = R.nbr[e >> 9];
          if (nb >= 0) tv[j] = S.tc[(size_t)nb * kNC + (e & 511)];
        }
      }
#pragma unroll
      for (int j = 0; j < kT; j++)
        if (t + j * kGT < 729) tt[t + j * kGT] = tv[j];
    }
    __syncthreads();
    // GC: a slot survives iff a cube around its edge still has the edge in its mask
#pragma unroll 1
    for (int j = 0; j < kNC / kGT; j++) {
      const int c = t + j * kGT;
      const int x = c >> 6, y = (c >> 3) & 7, z = c & 7;
      int keep = 0;
      unsigned keep_axes = 0;
#pragma unroll
      for (int axis = 0; axis < 3; axis++) {
        const int sl = c * 3 + axis;
        if (!((occ[sl >> 5] >> (sl & 31)) & 1)) continue;
        if (mode & G_GC) {
          // the 4 cubes around the edge: offsets -du along u, -dw along w
          // (u, w = the two axes other than `axis`); tile strides 81, 9, 1
          const int su = axis == 0 ? 9 : 81, sw = axis == 2 ? 9 : 1;
          const int p0 = ((x + 1) * 9 + (y + 1)) * 9 + (z + 1);
          bool ref = false;
#pragma unroll
          for (int j = 0; j < 4; j++) {
            const int du = j >> 1, dw = j & 1;
            ref = ref || ((c_edge_mask[tt[p0 - du * su - dw * sw]] >> cube_edge_of_slot(axis, du, dw)) & 1);
          }
          if (!ref) {
            S.vbirth[(size_t)b * kEV + sl] = -1;
            frees += R.owned;
            continue;
          }
        }
        keep++;
        keep_axes |= 1u << axis;
      }
      if (mode & G_NORMALS) {
        int pos = smem_append(keep, &s_nv);
        for (int axis = 0; axis < 3; axis++)
          if ((keep_axes >> axis) & 1) s_vlist[pos++] = (uint16_t)(c * 3 + axis);
      }
    }
    if (mode & G_NORMALS) {
      __syncthreads();
      const int nv = s_nv;
      for (int p = t; p < nv; p += kGT) {
        const int sl = s_vlist[p];
        const int ci = sl / 3, axis = sl - 3 * (sl / 3);
        computed += R.owned;
        const int x0 = ci >> 6, y0 = (ci >> 3) & 7, z0 = ci & 7;
        const int x1 = x0 + (axis == 0), y1 = y0 + (axis == 1), z1 = z0 + (axis == 2);
        // the 12 stencil points: c0 +- e_d, c1 +- e_d (c0 + e_axis = c1, c1 - e_axis = c0);
        // all 24 loads are issued before any is used (absent neighbours read a
        // dummy in-bounds sample and are masked out)
        double v0p[3], v0m[3], v1p[3], v1m[3];
        int w0p[3], w0m[3], w1p[3], w1m[3];
        bool inb = true;
        const size_t dummy = (size_t)b * kNC;
#pragma unroll
        for (int d = 0; d < 3; d++) {
          const int dx = d == 0, dy = d == 1, dz = d == 2;
          size_t a = sample_index(R.nbr, x0 + dx, y0 + dy, z0 + dz);
          size_t bq = sample_index(R.nbr, x0 - dx, y0 - dy, z0 - dz);
          size_t cq = sample_index(R.nbr, x1 + dx, y1 + dy, z1 + dz);
          size_t dq = sample_index(R.nbr, x1 - dx, y1 - dy, z1 - dz);
          inb = inb && a != ~(size_t)0 && bq != ~(size_t)0 && cq != ~(size_t)0 && dq != ~(size_t)0;
          a = a == ~(size_t)0 ? dummy : a;
          bq = bq == ~(size_t)0 ? dummy : bq;
          cq = cq == ~(size_t)0 ? dummy : cq;
          dq = dq == ~(size_t)0 ? dummy : dq;
          v0p[d] = S.tsdf[a]; v0m[d] = S.tsdf[bq]; v1p[d] = S.tsdf[cq]; v1m[d] = S.tsdf[dq];
          w0p[d] = S.weight[a]; w0m[d] = S.weight[bq]; w1p[d] = S.weight[cq]; w1m[d] = S.weight[dq];
        }
        bool valid = inb;   // (an invalid stencil's gradient is never used)
#pragma unroll
        for (int d = 0; d < 3; d++) valid = valid && w0p[d] > 0 && w0m[d] > 0 && w1p[d] > 0 && w1m[d] > 0;
        const double d0 = axis == 0 ? v1m[0] : axis == 1 ? v1m[1] : v1m[2];   // samples at c0 and c1
        const double d1 = axis == 0 ? v0p[0] : axis == 1 ? v0p[1] : v0p[2];
        const double denom = d0 - d1;
        const double param = (denom != 0) ? d0 / denom : 0.5;
        double g[3];
        const double wa = 1.0 - param;
#pragma unroll
        for (int d = 0; d < 3; d++)
          g[d] = __dadd_rn(__dmul_rn(wa, v0p[d] - v0m[d]), __dmul_rn(param, v1p[d] - v1m[d]));
        const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(g[0], g[0]), __dmul_rn(g[1], g[1])),
                                          __dmul_rn(g[2], g[2])));
        if (valid && nrm > 1e-12) {
          double *dst = S.vnrm + 3 * ((size_t)b * kEV + sl);
          dst[0] = g[0] / nrm; dst[1] = g[1] / nrm; dst[2] = g[2] / nrm;
        } else {
          fallbacks += R.owned;   // face-normal fallback: deferred to k_fallback (global worklist)
          S.fallback[atomicAdd(&ctr->nfallback, 1)] = make_int2(b, sl);
        }
      }
    }
    __syncthreads();   // R and the tiles are rewritten by the next item
  }
  {
    long long vals[3] = {frees, computed, fallbacks};
    int64_t *const dst[3] = {&ctr->v_frees, &ctr->normals, &ctr->fallbacks};
    block_add_counters<3>(vals, red, dst);
  }
  if (t == 0 && (mode & G_COMMIT)) {
    __threadfence();
    if (atomicAdd(&ctr->done_gc, 1) == (int)gridDim.x - 1) {
      __threadfence();
      const long long allocs = ld_vol(&ctr->v_allocs), fr = ld_vol(&ctr->v_frees);
      const long long peak = ctr->v_live + allocs;     // all allocations precede all frees
      if (S.max_vertices > 0 && peak > S.max_vertices)
        set_error(S, ERR_CAPACITY, peak, S.max_vertices, 3);
      if (peak > ctr->v_count) ctr->v_count = peak;
      ctr->v_live = peak - fr;
      ctr->v_recycled += fr;
      ctr->v_events += allocs;
      const long long rel = ld_vol(&ctr->t_released), nw = ld_vol(&ctr->t_allocated);
      ctr->t_live += nw - rel;
      ctr->t_recycled += rel;
      if (ctr->t_live > ctr->t_count) ctr->t_count = ctr->t_live;
      ctr->irregular += ld_vol(&ctr->irr_delta);
      ctr->done_gc = 0;
    }
  }
}
constexpr size_t kGcSmem = 0;




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
    const bool o = S.vbirth[q] >= 0;
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

// ------------------------------------------------------------ compaction
// store.py:388-425: blocks in sorted-coordinate order, vertices in (x,y,z,axis)
// slot order, triangles in (x,y,z,slot) order, dense remap of handles.
__global__ void k_block_keys(DevState S, int nblocks, unsigned long long *keys, int32_t *vals) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nblocks; i += gridDim.x * blockDim.x) {
    const int4 c = S.bcoord[i];
    keys[i] = (unsigned long long)pack_coord(c.x, c.y, c.z);
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
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    for (int r = 0; r < 3; r++) {
      const int s = r * kThreadsCube + t;
      const unsigned ball = __ballot_sync(0xffffffffu, S.vbirth[(size_t)b * kEV + s] >= 0);
      if (lane == 0) { occ_bits[(size_t)b * 48 + r * 16 + wid] = ball; wc[r * 16 + wid] = __popc(ball); }
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
      const int birth = S.vbirth[q];
      int o = -1;
      if (birth >= 0) {
        o = slot_index(occ_bits, occ_pre, vbase_by_blk, b, s);
        slot_position(S, b, s, pos + 3 * (size_t)o);
        for (int d = 0; d < 3; d++) nrm[3 * (size_t)o + d] = S.vnrm[3 * q + d];
        ages[o] = frame - (long long)birth;
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
        if (ob >= 0 && S.vbirth[(size_t)ob * kEV + s] >= 0) m = slot_index(occ_bits, occ_pre, vbase_by_blk, ob, s);
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
