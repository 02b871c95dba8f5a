// vm_kernels.cuh -- the per-frame kernels of the B200 mesh-generation path.
//
// Frame pipeline (one CUDA stream, no host sync inside a frame):
//   k_depth_stats  valid-pixel count + max ray norm           (fusion.py:81-94)
//   k_collect      ray-band block collection + hash insert    (fusion.py:95-106, store.py:296-320)
//   k_init_blocks  zero-init new blocks + neighbour links     (store.py:70-81)
//   k_integrate    TSDF running average                       (fusion.py:138-168)
//   k_scope_halo   minus-slab scope + 27-neighbour halo       (mesher.py:499-543)
//   k_retype       cube typing (+ Hamming refinement)         (mesher.py:111-134, refine.py:98-135)
//   k_place        claim-based edge-vertex placement          (mesher.py:178-257)
//   k_tri_release  free triangles of changed cubes            (mesher.py:296-307)
//   k_tri_alloc    emit triangles of changed cubes            (mesher.py:308-320)
//   k_gc           refcount==0 vertex recycling               (mesher.py:333-356)
//   k_normals      blended central-difference gradients       (mesher.py:400-439)
//   k_fallback     face-normal fallback, reference order      (mesher.py:442-486)
// Every kernel after k_collect returns immediately when a capacity guard
// tripped (ctr->need) or an error was raised, so the host can grow an arena
// and resume the frame at the failed segment.
#pragma once
#include "vm_device.cuh"

namespace vm {

constexpr int kThreadsCube = 512;   // one thread per cube of a block

__device__ __forceinline__ bool halted(const DevState &S) {
  return ld_vol(&S.ctr->need) != 0 || ld_vol(&S.ctr->error) != 0;
}

// ------------------------------------------------------------ depth stats
__global__ void k_depth_stats(DevState S, const FrameDev *__restrict__ Fp) {
  const FrameDev &F = *Fp;
  const long long npix = (long long)F.h * F.w;
  long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  double best = -1.0;
  int cnt = 0;
  for (; p < npix; p += (long long)gridDim.x * blockDim.x) {
    double d = F.depth[p];
    if (d > 0 && d <= F.max_range) {
      int v = (int)(p / F.w), u = (int)(p - (long long)v * F.w);
      double rx = ((double)u - F.cx) / F.fx, ry = ((double)v - F.cy) / F.fy;
      double n = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)), 1.0));
      best = fmax(best, n);
      cnt++;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  cnt = warp_sum(cnt);
  if ((threadIdx.x & 31) == 0 && cnt) {
    atomicAdd(&S.ctr->nvalid, cnt);
    atomicMax(&S.ctr->maxnorm_bits, (unsigned long long)__double_as_longlong(best));
  }
}

// ------------------------------------------------------------ collect
// One thread per pixel, looping over the nsteps band samples.  Samples of a
// warp that fall in the same block are merged with __match_any_sync, so only
// one lane per distinct block probes the hash table.
__global__ void k_collect(DevState S, const FrameDev *__restrict__ Fp) {
  const FrameDev &F = *Fp;
  Counters *ctr = S.ctr;
  if (ld_vol(&ctr->nvalid) == 0) return;
  const double maxnorm = __longlong_as_double((long long)ld_vol(&ctr->maxnorm_bits));
  const double half_block = S.extent * 0.5;
  const double band = __dmul_rn(__dmul_rn(2.0, F.trunc), maxnorm);
  int nsteps = (int)ceil(band / half_block) + 1;
  if (nsteps < 2) nsteps = 2;
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->nsteps = nsteps;
  const double step = 2.0 / (double)(nsteps - 1);
  const long long npix = (long long)F.h * F.w;
  const int lane = threadIdx.x & 31;
  const long long wstride = (long long)gridDim.x * blockDim.x;
  for (long long base = (long long)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < npix;
       base += wstride) {
    const long long p = base + lane;
    double d = 0.0, qs[3] = {0, 0, 0};
    bool valid = false;
    if (p < npix) {
      d = F.depth[p];
      valid = d > 0 && d <= F.max_range;
    }
    if (valid) {
      int v = (int)(p / F.w), u = (int)(p - (long long)v * F.w);
      double rx = ((double)u - F.cx) / F.fx, ry = ((double)v - F.cy) / F.fy;
      double pc[3] = {__dmul_rn(rx, d), __dmul_rn(ry, d), __dmul_rn(1.0, d)};
      for (int j = 0; j < 3; j++) qs[j] = matvec_row(pc, F.R, j);   // pts_cam @ R.T
    }
    const double delta = valid ? F.trunc / d : 0.0;
    for (int i = 0; i < nsteps; i++) {
      long long key = kEmptyKey;
      int c[3] = {0, 0, 0};
      if (valid) {
        const double s = (i == nsteps - 1) ? 1.0 : __dadd_rn(__dmul_rn((double)i, step), -1.0);
        const double f = __dadd_rn(1.0, __dmul_rn(s, delta));
        for (int j = 0; j < 3; j++)
          c[j] = (int)floor(__dadd_rn(F.t[j], __dmul_rn(qs[j], f)) / S.extent);
        key = pack_coord(c[0], c[1], c[2]);
      }
      const unsigned grp = __match_any_sync(0xffffffffu, key);
      if (key != kEmptyKey && lane == __ffs(grp) - 1) {
        int idx = hash_find(S, c[0], c[1], c[2]);
        if (idx == -1) idx = hash_insert(S, c[0], c[1], c[2]);
        if (idx >= 0 && ld_vol(S.stamp_collect + idx) != F.epoch &&
            atomicExch(S.stamp_collect + idx, F.epoch) != F.epoch)
          S.scope[atomicAdd(&ctr->ncollected, 1)] = idx;
      }
    }
  }
}

// ------------------------------------------------------------ insert list
// explicit coordinates (vm_set_blocks): insert, return indices
__global__ void k_insert_coords(DevState S, const int3 *__restrict__ coords, int n,
                                int32_t *__restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int3 c = coords[i];
    int idx = hash_find(S, c.x, c.y, c.z);
    if (idx == -1) idx = hash_insert(S, c.x, c.y, c.z);
    out[i] = idx;
  }
}

// map coordinates to block indices (absent -> -1); optionally stamp them
__global__ void k_lookup_coords(DevState S, const int3 *__restrict__ coords, int n,
                                int32_t *__restrict__ out, int32_t *stamp, int32_t epoch) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int3 c = coords[i];
    int idx = hash_find(S, c.x, c.y, c.z);
    out[i] = idx;
    if (stamp && idx >= 0) stamp[idx] = epoch;
  }
}

// ------------------------------------------------------------ init blocks
// Block.empty (store.py:70-81) for every block allocated this call, plus the
// 26-neighbour links used by all later kernels for O(1) neighbour access.
__global__ void __launch_bounds__(256) k_init_blocks(DevState S) {
  if (halted(S)) return;
  const int nnew = ld_vol(&S.ctr->nnew);
  for (int i = blockIdx.x; i < nnew; i += gridDim.x) {
    const int b = S.newlist[i];
    const int t = threadIdx.x;
    double2 *ts = reinterpret_cast<double2 *>(S.tsdf + (size_t)b * kNC);
    int4 *wt = reinterpret_cast<int4 *>(S.weight + (size_t)b * kNC);
    ts[t] = make_double2(0.0, 0.0);                                   // 256 x 16 B
    if (t < 128) wt[t] = make_int4(0, 0, 0, 0);                        // 128 x 16 B
    if (t < 32) {
      reinterpret_cast<int4 *>(S.tp + (size_t)b * kNC)[t] = make_int4(0, 0, 0, 0);
      reinterpret_cast<int4 *>(S.tc + (size_t)b * kNC)[t] = make_int4(0, 0, 0, 0);
    }
    int4 *ev = reinterpret_cast<int4 *>(S.ev + (size_t)b * kEV);        // 384 x 16 B
    for (int q = t; q < kEV / 4; q += blockDim.x) ev[q] = make_int4(-1, -1, -1, -1);
    int4 *tr = reinterpret_cast<int4 *>(S.tri + (size_t)b * kTS);       // 640 x 16 B
    for (int q = t; q < kTS / 4; q += blockDim.x) tr[q] = make_int4(-1, -1, -1, -1);
    if (t < 27) {
      const int4 c = S.bcoord[b];
      const int dx = t / 9 - 1, dy = (t / 3) % 3 - 1, dz = t % 3 - 1;
      int y = (t == 13) ? b : hash_find(S, c.x + dx, c.y + dy, c.z + dz);
      S.nbr[(size_t)b * 27 + t] = y;
      if (y >= 0 && t != 13) S.nbr[(size_t)y * 27 + (26 - t)] = b;
    }
  }
}

// ------------------------------------------------------------ integrate
// One CTA per block, one thread per corner (coalesced tsdf/weight rows).
__global__ void __launch_bounds__(kThreadsCube) k_integrate(DevState S,
                                                            const FrameDev *__restrict__ Fp,
                                                            const int32_t *__restrict__ list,
                                                            const int32_t *__restrict__ count_ptr,
                                                            int count_const) {
  if (halted(S)) return;
  __shared__ FrameDev F;
  if (threadIdx.x == 0) F = *Fp;
  __syncthreads();
  const int n = count_ptr ? ld_vol(count_ptr) : count_const;
  const int ci = threadIdx.x;
  const int lx = ci >> 6, ly = (ci >> 3) & 7, lz = ci & 7;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int b = list[i];
    if (b < 0) continue;
    const int4 c = S.bcoord[b];
    double a[3];
    a[0] = __dadd_rn(__dmul_rn((double)c.x, S.extent), __dmul_rn((double)lx, S.cube_size)) - F.t[0];
    a[1] = __dadd_rn(__dmul_rn((double)c.y, S.extent), __dmul_rn((double)ly, S.cube_size)) - F.t[1];
    a[2] = __dadd_rn(__dmul_rn((double)c.z, S.extent), __dmul_rn((double)lz, S.cube_size)) - F.t[2];
    const double z = matvec_col(a, F.R, 2);
    if (!(z > 0)) continue;
    const double x = matvec_col(a, F.R, 0), y = matvec_col(a, F.R, 1);
    const double u = rint(__dadd_rn(__dmul_rn(F.fx, x) / z, F.cx));
    const double v = rint(__dadd_rn(__dmul_rn(F.fy, y) / z, F.cy));
    if (!(u >= 0 && u < (double)F.w && v >= 0 && v < (double)F.h)) continue;
    const double meas = F.depth[(long long)v * F.w + (long long)u];
    if (!(meas > 0 && meas <= F.max_range)) continue;
    const double sdf = meas - z;
    if (!(sdf >= -F.trunc)) continue;
    double dn = sdf / F.trunc;
    dn = dn < -1.0 ? -1.0 : (dn > 1.0 ? 1.0 : dn);
    const size_t q = (size_t)b * kNC + ci;
    const int w_old = S.weight[q];
    const double wo = (double)w_old;
    S.tsdf[q] = __dadd_rn(__dmul_rn(wo, S.tsdf[q]), dn) / __dadd_rn(wo, 1.0);
    const long long nw = (long long)w_old + 1;
    S.weight[q] = (int)(nw < F.weight_cap ? nw : F.weight_cap);
  }
}

// ------------------------------------------------------------ scope + halo
// thread per (collected block, neighbour offset)
__global__ void k_scope_halo(DevState S, const FrameDev *__restrict__ Fp) {
  if (halted(S)) return;
  const int epoch = Fp->epoch;
  const int nc = ld_vol(&S.ctr->ncollected);
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < (long long)nc * 27;
       t += (long long)gridDim.x * blockDim.x) {
    const int item = (int)(t / 27), d = (int)(t % 27);
    const int c = S.scope[item];
    const int n = S.nbr[(size_t)c * 27 + d];
    if (n < 0) continue;
    if (ld_vol(S.stamp_halo + n) != epoch && atomicExch(S.stamp_halo + n, epoch) != epoch)
      S.halo[atomicAdd(&S.ctr->nhalo, 1)] = n;
    const int dx = d / 9 - 1, dy = (d / 3) % 3 - 1, dz = d % 3 - 1;
    if (dx > 0 || dy > 0 || dz > 0 || d == 13) continue;     // minus offsets only
    if (ld_vol(S.stamp_collect + n) == epoch) continue;        // fully in scope
    const int o = (-dx) * 4 + (-dy) * 2 + (-dz);               // n = c - o
    const unsigned old = atomicOr((unsigned *)(S.slab_bits + (n & ~3)), (1u << (o - 1)) << (8 * (n & 3)));
    if (((old >> (8 * (n & 3))) & 0xFF) == 0)
      S.scope[nc + atomicAdd(&S.ctr->nslab, 1)] = n;
  }
}

// halo of an explicit scope (extract_frame default, mesher.py:627-633)
__global__ void k_halo_from_items(DevState S, const FrameDev *__restrict__ Fp) {
  if (halted(S)) return;
  const int epoch = Fp->epoch;
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

// ------------------------------------------------------------ tile loaders
// (B+1)^3 tile of a block plus its 7 plus-neighbours (mesher.py:75-96)
__device__ __forceinline__ void load_ext_tile(const DevState &S, int b, double *tile,
                                              uint8_t *tw, bool want_w) {
  const int t = threadIdx.x;
  {
    const int x = t >> 6, y = (t >> 3) & 7, z = t & 7;
    const size_t q = (size_t)b * kNC + t;
    tile[(x * 9 + y) * 9 + z] = S.tsdf[q];
    if (want_w) tw[(x * 9 + y) * 9 + z] = S.weight[q] > 0;
  }
  if (t < 217) {
    // enumerate tile positions with max(x, y, z) == 8
    int x, y, z;
    if (t < 64) { x = 8; y = t >> 3; z = t & 7; }                 // x face
    else if (t < 128) { x = (t - 64) >> 3; y = 8; z = t & 7; }    // y face
    else if (t < 192) { x = (t - 128) >> 3; y = t & 7; z = 8; }   // z face
    else if (t < 200) { x = 8; y = 8; z = t - 192; }              // xy edge
    else if (t < 208) { x = 8; y = t - 200; z = 8; }              // xz edge
    else if (t < 216) { x = t - 208; y = 8; z = 8; }              // yz edge
    else { x = 8; y = 8; z = 8; }                                  // corner
    const int dir = nbr_dir(x >> 3, y >> 3, z >> 3);
    const int nb = S.nbr[(size_t)b * 27 + dir];
    double v = 0.0;
    uint8_t w = 0;
    if (nb >= 0) {
      const size_t q = (size_t)nb * kNC + ((x & 7) * 64 + (y & 7) * 8 + (z & 7));
      v = S.tsdf[q];
      if (want_w) w = S.weight[q] > 0;
    }
    tile[(x * 9 + y) * 9 + z] = v;
    if (want_w) tw[(x * 9 + y) * 9 + z] = w;
  }
}

__device__ __forceinline__ int item_count(const DevState &S, const FrameDev &F) {
  return F.scope_mode == 0 ? ld_vol(&S.ctr->ncollected) + ld_vol(&S.ctr->nslab)
                           : ld_vol(&S.ctr->nexplicit);
}

// ------------------------------------------------------------ retype (+refine)
__global__ void __launch_bounds__(kThreadsCube) k_retype(DevState S, const FrameDev *__restrict__ Fp) {
  if (halted(S)) return;
  __shared__ double tile[729];
  __shared__ uint8_t tw[729];
  __shared__ long long red[32];
  __shared__ int s_mask_mode;  // 0 none selected, 1 full, 2 slab bits, 3 explicit
  __shared__ int s_slab;
  const FrameDev &F = *Fp;
  const int n = item_count(S, F);
  const int nc = ld_vol(&S.ctr->ncollected);
  const int t = threadIdx.x;
  long long v_bound = 0, t_bound = 0, active = 0, changed = 0, refined = 0, live = 0;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int b = S.scope[i];
    if (t == 0) {
      int mode;
      if (b < 0) mode = 0;
      else if (F.scope_mode == 1) mode = 3;
      else if (i < nc) mode = 1;
      else { mode = 2; s_slab = S.slab_bits[b]; S.slab_bits[b] = 0; }
      if (mode && F.frustum_only && !block_in_frustum_dev(S.bcoord[b], F, S.extent)) mode = 0;
      s_mask_mode = mode;
      if (mode) live++;
    }
    __syncthreads();
    const int mode = s_mask_mode;
    if (mode == 0) {
      if (t < 16) S.item_sel[(size_t)i * 16 + t] = 0;
      __syncthreads();
      continue;
    }
    load_ext_tile(S, b, tile, tw, true);
    __syncthreads();
    const int x = t >> 6, y = (t >> 3) & 7, z = t & 7;
    bool sel;
    if (mode == 1) sel = true;
    else if (mode == 2) sel = (s_slab & c_slab_sel[((x == 7) << 2) | ((y == 7) << 1) | (z == 7)]) != 0;
    else sel = (S.item_mask[(size_t)i * 16 + (t >> 5)] >> (t & 31)) & 1;
    double corner[8];
    unsigned bits = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const int o = c_corner[k];
      const int e = ((x + (o & 1)) * 9 + (y + ((o >> 1) & 1))) * 9 + (z + ((o >> 2) & 1));
      corner[k] = tile[e];
      sel = sel && tw[e];
      bits |= (corner[k] < 0.0 ? 1u : 0u) << k;
    }
    if (sel) {
      const size_t q = (size_t)b * kNC + t;
      const unsigned tp = S.tc[q];
      unsigned tc = bits;
      if (F.refine) {
        bool ch;
        tc = refine_type(bits, tp, corner, F.epsilon, &ch);
        refined += ch;
      }
      S.tp[q] = (uint8_t)tp;
      S.tc[q] = (uint8_t)tc;
      const unsigned m = c_edge_mask[tc];
      if (m) { active++; v_bound += __popc(m); }
      if (tc != tp) { changed++; t_bound += 5; }
    }
    const unsigned ball = __ballot_sync(0xffffffffu, sel);
    if ((t & 31) == 0) S.item_sel[(size_t)i * 16 + (t >> 5)] = ball;
    __syncthreads();
  }
  long long r;
  r = block_sum(v_bound, red); if (t == 0 && r) atomicAdd((unsigned long long *)&S.ctr->v_bound, (unsigned long long)r);
  r = block_sum(t_bound, red); if (t == 0 && r) atomicAdd((unsigned long long *)&S.ctr->t_bound, (unsigned long long)r);
  r = block_sum(active, red); if (t == 0 && r) atomicAdd((unsigned long long *)&S.ctr->active_cubes, (unsigned long long)r);
  r = block_sum(changed, red); if (t == 0 && r) atomicAdd((unsigned long long *)&S.ctr->changed_cubes, (unsigned long long)r);
  r = block_sum(refined, red); if (t == 0 && r) atomicAdd((unsigned long long *)&S.ctr->refined, (unsigned long long)r);
  if (t == 0 && live) atomicAdd(&S.ctr->nitems_live, (int)live);
}

// ------------------------------------------------------------ placement
// Edge-owned vertices (mesher.py:178-235): each active cube visits its mask
// edges; the owner slot is claimed with atomicCAS (-1 -> -2), the winner takes
// a ticket (free-stack pop or arena bump), initialises the record and
// publishes the handle.  Every requester that sees a published handle
// rewrites the same position bits (d0, d1 are the oriented edge endpoint
// samples), so no requester waits on another.
// parity >= 0: the partition strategy's lock-free pass (mesher.py:250-254).
__device__ __forceinline__ int take_vertex(const DevState &S, int ticket, int F0, int C0, int frame) {
  int h;
  if (ticket < F0) h = S.vfree[F0 - 1 - ticket];
  else {
    h = C0 + (ticket - F0);
    if (S.max_vertices > 0 && (long long)h >= S.max_vertices) {
      set_error(S, ERR_CAPACITY, h, S.max_vertices, 3);
      return -1;
    }
  }
  S.valive[h] = 1;
  S.vref[h] = 0;
  S.vbirth[h] = frame;
  S.vnrm[3 * (size_t)h] = 0.0; S.vnrm[3 * (size_t)h + 1] = 0.0; S.vnrm[3 * (size_t)h + 2] = 0.0;
  return h;
}

__global__ void __launch_bounds__(kThreadsCube) k_place(DevState S, const FrameDev *__restrict__ Fp,
                                                        int parity, int last_pass) {
  if (halted(S)) return;
  Counters *ctr = S.ctr;
  const int F0 = ld_vol(&ctr->v_free), C0 = ld_vol(&ctr->v_count);
  {
    // capacity guard: reserve bound = sum of popcount(edge masks) (mesher.py:579-589)
    long long bound = ld_vol(&ctr->v_bound);
    long long need = bound - F0;
    if (need > 0 && (long long)C0 + need > (long long)S.v_cap) {
      if (threadIdx.x == 0) atomicOr(&ctr->need, NEED_VERTS);
      return;
    }
  }
  __shared__ double tile[729];
  __shared__ long long red[32];
  const FrameDev &F = *Fp;
  const int n = item_count(S, F);
  const int t = threadIdx.x;
  const int x = t >> 6, y = (t >> 3) & 7, z = t & 7;
  const double l = S.cube_size;
  long long placements = 0;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int b = S.scope[i];
    const uint32_t selw = (b >= 0) ? S.item_sel[(size_t)i * 16 + (t >> 5)] : 0u;
    if (__syncthreads_or(selw != 0) == 0) continue;
    load_ext_tile(S, b, tile, nullptr, false);
    __syncthreads();
    const bool sel = (selw >> (t & 31)) & 1;
    const unsigned tc = sel ? S.tc[(size_t)b * kNC + t] : 0u;
    unsigned mask = c_edge_mask[tc];
    if (parity >= 0 && (((x & 1) | ((y & 1) << 1) | ((z & 1) << 2)) != parity)) mask = 0;
    if (mask) {
      const int4 bc = S.bcoord[b];
      const int gx = bc.x * kB + x, gy = bc.y * kB + y, gz = bc.z * kB + z;
      placements += __popc(mask);
      while (mask) {
        const int e = __ffs(mask) - 1;
        mask &= mask - 1;
        const int own = c_e_own[e], axis = c_e_axis[e];
        const int ox = x + (own & 1), oy = y + ((own >> 1) & 1), oz = z + ((own >> 2) & 1);
        const int dir = nbr_dir(ox >> 3, oy >> 3, oz >> 3);
        const int owner = (dir == 13) ? b : S.nbr[(size_t)b * 27 + dir];
        if (owner < 0) {
          set_error(S, ERR_CONSISTENCY, 10, gx, gy, gz);
          continue;
        }
        int32_t *slot = S.ev + (size_t)owner * kEV + (((ox & 7) * 64 + (oy & 7) * 8 + (oz & 7)) * 3 + axis);
        int h = ld_vol(slot);
        if (h == -1) {
          if (parity >= 0) {
            const int ticket = atomicAdd(&ctr->v_tickets, 1);
            h = take_vertex(S, ticket, F0, C0, F.frame);
            *slot = h;
          } else {
            const int old = atomicCAS(slot, -1, -2);
            if (old == -1) {
              const int ticket = atomicAdd(&ctr->v_tickets, 1);
              h = take_vertex(S, ticket, F0, C0, F.frame);
              __threadfence();
              atomicExch(slot, h);
            } else {
              h = old;   // -2: the winner writes the position
            }
          }
        }
        if (h < 0) continue;
        const int sc = c_corner[c_e_start[e]], ec = c_corner[c_e_end[e]];
        const int sx = sc & 1, sy = (sc >> 1) & 1, sz = (sc >> 2) & 1;
        const double d0 = tile[((x + sx) * 9 + (y + sy)) * 9 + (z + sz)];
        const double d1 = tile[((x + (ec & 1)) * 9 + (y + ((ec >> 1) & 1))) * 9 + (z + ((ec >> 2) & 1))];
        const double param = (d0 == d1) ? 0.5 : d0 / (d0 - d1);
        double p[3] = {__dmul_rn((double)(gx + sx), l), __dmul_rn((double)(gy + sy), l),
                       __dmul_rn((double)(gz + sz), l)};
        p[axis] = __dadd_rn(p[axis], __dmul_rn(param, l));
        double *dst = S.vpos + 3 * (size_t)h;
        dst[0] = p[0]; dst[1] = p[1]; dst[2] = p[2];
      }
    }
    __syncthreads();
  }
  long long r = block_sum(placements, red);
  if (t == 0) {
    if (r) atomicAdd((unsigned long long *)&ctr->edge_placements, (unsigned long long)r);
    if (last_pass) {
      __threadfence();
      if (atomicAdd(&ctr->done_place, 1) == (int)gridDim.x - 1) {
        // last CTA: commit the tickets to the arena counters
        const int tickets = ld_vol(&ctr->v_tickets);
        const int used = tickets < F0 ? tickets : F0;
        ctr->v_free = F0 - used;
        ctr->v_count = C0 + (tickets - used);
        ctr->v_events += tickets;
        ctr->done_place = 0;
      }
    }
  }
}

// ------------------------------------------------------------ triangulation
// Changed cubes release their old triangles (decref x3, push to the free
// stack) ...
__global__ void __launch_bounds__(kThreadsCube) k_tri_release(DevState S, const FrameDev *__restrict__ Fp) {
  if (halted(S)) return;
  __shared__ long long red[32];
  const FrameDev &F = *Fp;
  const int n = item_count(S, F);
  const int t = threadIdx.x;
  const int lane = t & 31;
  long long released = 0, irr = 0;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int b = S.scope[i];
    const uint32_t selw = (b >= 0) ? S.item_sel[(size_t)i * 16 + (t >> 5)] : 0u;
    if (selw == 0) continue;   // warp-uniform
    const bool sel = (selw >> lane) & 1;
    const size_t q = (size_t)b * kNC + t;
    const unsigned tc = sel ? S.tc[q] : 0u, tp = sel ? S.tp[q] : 0u;
    const bool changed = sel && tc != tp;
    int mine[5];
    int cnt = 0;
    if (changed) {
      int32_t *slots = S.tri + (size_t)b * kTS + t * 5;
      for (int s = 0; s < 5; s++) {
        const int th = slots[s];
        if (th < 0) continue;
        mine[cnt++] = th;
        slots[s] = -1;
        for (int k = 0; k < 3; k++) {
          const int v = S.tverts[3 * (size_t)th + k];
          if (atomicSub(S.vref + v, 1) <= 0) set_error(S, ERR_CONSISTENCY, 20, v);
        }
        if (!S.talive[th]) set_error(S, ERR_CONSISTENCY, 21, th);
        S.talive[th] = 0;
      }
      if (cnt && !is_regular_type(tp)) irr--;
    }
    // warp-aggregated push onto the triangle free stack
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int base = 0;
    if (lane == 31 && total) base = atomicAdd(&S.ctr->t_free, total);
    base = __shfl_sync(0xffffffffu, base, 31);
    for (int k = 0; k < cnt; k++) S.tfree[base + incl - cnt + k] = mine[k];
    released += cnt;
  }
  long long r = block_sum(released, red);
  if (t == 0 && r) {
    atomicAdd((unsigned long long *)&S.ctr->t_released, (unsigned long long)r);
    atomicAdd((unsigned long long *)&S.ctr->t_recycled, (unsigned long long)r);
  }
  r = block_sum(irr, red);
  if (t == 0 && r) atomicAdd((unsigned long long *)&S.ctr->irregular, (unsigned long long)r);
}

// ... then emit TRI_TABLE[type] (incref x3) via tickets on the free stack/arena.
__global__ void __launch_bounds__(kThreadsCube) k_tri_alloc(DevState S, const FrameDev *__restrict__ Fp) {
  if (halted(S)) return;
  Counters *ctr = S.ctr;
  const int F0 = ld_vol(&ctr->t_free), C0 = ld_vol(&ctr->t_count);
  {
    long long bound = ld_vol(&ctr->t_bound);
    long long need = bound - F0;
    if (need > 0 && (long long)C0 + need > (long long)S.t_cap) {
      if (threadIdx.x == 0) atomicOr(&ctr->need, NEED_TRIS);
      return;
    }
  }
  __shared__ long long red[32];
  const FrameDev &F = *Fp;
  const int n = item_count(S, F);
  const int t = threadIdx.x;
  const int lane = t & 31;
  const int x = t >> 6, y = (t >> 3) & 7, z = t & 7;
  long long allocated = 0, irr = 0;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int b = S.scope[i];
    const uint32_t selw = (b >= 0) ? S.item_sel[(size_t)i * 16 + (t >> 5)] : 0u;
    if (selw == 0) continue;   // warp-uniform
    const bool sel = (selw >> lane) & 1;
    const size_t q = (size_t)b * kNC + t;
    const unsigned tc = sel ? S.tc[q] : 0u, tp = sel ? S.tp[q] : 0u;
    const int ntri = (sel && tc != tp) ? c_tri_count[tc] : 0;
    int incl = ntri;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int base = 0;
    if (lane == 31 && total) base = atomicAdd(&ctr->t_tickets, total);
    base = __shfl_sync(0xffffffffu, base, 31);
    if (ntri) {
      const unsigned long long packed = c_tri_packed[tc];
      int32_t *slots = S.tri + (size_t)b * kTS + t * 5;
      int ticket = base + incl - ntri;
      for (int j = 0; j < ntri; j++, ticket++) {
        int hv[3];
        bool ok = true;
        for (int k = 0; k < 3; k++) {
          const int e = (int)((packed >> (4 * (3 * j + k))) & 0xF);
          const int own = c_e_own[e];
          const int ox = x + (own & 1), oy = y + ((own >> 1) & 1), oz = z + ((own >> 2) & 1);
          const int dir = nbr_dir(ox >> 3, oy >> 3, oz >> 3);
          const int owner = (dir == 13) ? b : S.nbr[(size_t)b * 27 + dir];
          hv[k] = owner < 0 ? -1
                            : S.ev[(size_t)owner * kEV + (((ox & 7) * 64 + (oy & 7) * 8 + (oz & 7)) * 3 + c_e_axis[e])];
          if (hv[k] < 0) {
            const int4 bc = S.bcoord[b];
            set_error(S, ERR_CONSISTENCY, owner < 0 ? 11 : 12, bc.x * kB + x, bc.y * kB + y, bc.z * kB + z);
            ok = false;
          }
        }
        if (!ok) break;
        const int th = ticket < F0 ? S.tfree[F0 - 1 - ticket] : C0 + (ticket - F0);
        S.tverts[3 * (size_t)th] = hv[0];
        S.tverts[3 * (size_t)th + 1] = hv[1];
        S.tverts[3 * (size_t)th + 2] = hv[2];
        S.talive[th] = 1;
        slots[j] = th;
        atomicAdd(S.vref + hv[0], 1);
        atomicAdd(S.vref + hv[1], 1);
        atomicAdd(S.vref + hv[2], 1);
      }
      allocated += ntri;
      if (!is_regular_type(tc)) irr++;
    }
  }
  long long r = block_sum(allocated, red);
  if (t == 0 && r) atomicAdd((unsigned long long *)&ctr->t_allocated, (unsigned long long)r);
  r = block_sum(irr, red);
  if (t == 0) {
    if (r) atomicAdd((unsigned long long *)&ctr->irregular, (unsigned long long)r);
    __threadfence();
    if (atomicAdd(&ctr->done_tri, 1) == (int)gridDim.x - 1) {
      const int tickets = ld_vol(&ctr->t_tickets);
      const int used = tickets < F0 ? tickets : F0;
      ctr->t_free = F0 - used;
      ctr->t_count = C0 + (tickets - used);
      ctr->done_tri = 0;
    }
  }
}

// ------------------------------------------------------------ vertex GC
__device__ __forceinline__ int list_count(const int32_t *count_ptr, int count_const) {
  return count_ptr ? ld_vol(count_ptr) : count_const;
}

__global__ void __launch_bounds__(kThreadsCube) k_gc(DevState S, const int32_t *__restrict__ list,
                                                     const int32_t *__restrict__ count_ptr,
                                                     int count_const, int require_items) {
  if (halted(S)) return;
  if (require_items && ld_vol(&S.ctr->nitems_live) == 0) return;
  __shared__ long long red[32];
  const int n = list_count(count_ptr, count_const);
  const int t = threadIdx.x, lane = t & 31;
  long long freed = 0;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int b = list[i];
    if (b < 0) continue;
    for (int r = 0; r < 3; r++) {
      const int s = r * kThreadsCube + t;
      int32_t *slot = S.ev + (size_t)b * kEV + s;
      const int h = *slot;
      const bool dead = h >= 0 && S.vref[h] == 0;
      const unsigned ball = __ballot_sync(0xffffffffu, dead);
      if (!ball) continue;
      int base = 0;
      if (lane == 0) base = atomicAdd(&S.ctr->v_free, __popc(ball));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (dead) {
        *slot = -1;
        if (!S.valive[h]) set_error(S, ERR_CONSISTENCY, 30, h);
        S.valive[h] = 0;
        S.vfree[base + __popc(ball & ((1u << lane) - 1))] = h;
      }
      freed += dead;
    }
  }
  long long r = block_sum(freed, red);
  if (t == 0 && r) {
    atomicAdd((unsigned long long *)&S.ctr->v_freed, (unsigned long long)r);
    atomicAdd((unsigned long long *)&S.ctr->v_recycled, (unsigned long long)r);
  }
}

// ------------------------------------------------------------ normals
// 11^3 stencil tile over locals -1..9 (mesher.py:369-397)
__global__ void __launch_bounds__(kThreadsCube) k_normals(DevState S, const int32_t *__restrict__ list,
                                                          const int32_t *__restrict__ count_ptr,
                                                          int count_const, int require_items) {
  if (halted(S)) return;
  if (require_items && ld_vol(&S.ctr->nitems_live) == 0) return;
  __shared__ double st[1331];
  __shared__ uint8_t sw[1331];
  __shared__ long long red[32];
  const int n = list_count(count_ptr, count_const);
  const int t = threadIdx.x, lane = t & 31;
  long long computed = 0;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int b = list[i];
    if (b < 0) continue;
    for (int q = t; q < 1331; q += kThreadsCube) {
      const int X = q / 121, Y = (q / 11) % 11, Z = q % 11;
      const int lx = X - 1, ly = Y - 1, lz = Z - 1;
      const int dir = nbr_dir(lx >> 3, ly >> 3, lz >> 3);
      const int nb = (dir == 13) ? b : S.nbr[(size_t)b * 27 + dir];
      double v = 0.0;
      uint8_t w = 0;
      if (nb >= 0) {
        const size_t src = (size_t)nb * kNC + ((lx & 7) * 64 + (ly & 7) * 8 + (lz & 7));
        v = S.tsdf[src];
        w = S.weight[src] > 0;
      }
      st[q] = v;
      sw[q] = w;
    }
    __syncthreads();
    const int x = t >> 6, y = (t >> 3) & 7, z = t & 7;
    for (int axis = 0; axis < 3; axis++) {
      const int h = S.ev[(size_t)b * kEV + t * 3 + axis];
      bool fb = false;
      if (h >= 0) {
        computed++;
        int c0[3] = {x + 1, y + 1, z + 1};
        int c1[3] = {x + 1, y + 1, z + 1};
        c1[axis]++;
        const double d0 = st[(c0[0] * 11 + c0[1]) * 11 + c0[2]];
        const double d1 = st[(c1[0] * 11 + c1[1]) * 11 + c1[2]];
        const double denom = d0 - d1;
        const double param = (denom != 0) ? d0 / denom : 0.5;
        double g0[3], g1[3];
        bool valid = true;
#pragma unroll
        for (int d = 0; d < 3; d++) {
          int pp[3] = {c0[0], c0[1], c0[2]}, mm[3] = {c0[0], c0[1], c0[2]};
          pp[d]++; mm[d]--;
          const int ip = (pp[0] * 11 + pp[1]) * 11 + pp[2], im = (mm[0] * 11 + mm[1]) * 11 + mm[2];
          g0[d] = st[ip] - st[im];
          valid = valid && sw[ip] && sw[im];
        }
#pragma unroll
        for (int d = 0; d < 3; d++) {
          int pp[3] = {c1[0], c1[1], c1[2]}, mm[3] = {c1[0], c1[1], c1[2]};
          pp[d]++; mm[d]--;
          const int ip = (pp[0] * 11 + pp[1]) * 11 + pp[2], im = (mm[0] * 11 + mm[1]) * 11 + mm[2];
          g1[d] = st[ip] - st[im];
          valid = valid && sw[ip] && sw[im];
        }
        double g[3];
        const double wa = 1.0 - param;
#pragma unroll
        for (int d = 0; d < 3; d++) g[d] = __dadd_rn(__dmul_rn(wa, g0[d]), __dmul_rn(param, g1[d]));
        const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(g[0], g[0]), __dmul_rn(g[1], g[1])),
                                          __dmul_rn(g[2], g[2])));
        if (valid && nrm > 1e-12) {
          double *dst = S.vnrm + 3 * (size_t)h;
          dst[0] = g[0] / nrm; dst[1] = g[1] / nrm; dst[2] = g[2] / nrm;
        } else {
          fb = true;
        }
      }
      const unsigned ball = __ballot_sync(0xffffffffu, fb);
      if (ball) {
        int base = 0;
        if (lane == 0) base = atomicAdd(&S.ctr->nfallback, __popc(ball));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (fb) {
          FallbackRec rec;
          rec.h = h; rec.blk = b; rec.slot = t * 3 + axis;
          S.fallback[base + __popc(ball & ((1u << lane) - 1))] = rec;
        }
      }
    }
    __syncthreads();
  }
  long long r = block_sum(computed, red);
  if (t == 0 && r) atomicAdd((unsigned long long *)&S.ctr->normals, (unsigned long long)r);
}

// Face-normal fallback, one thread per fallback vertex.  Accumulates the face
// normals of incident triangles stored in halo blocks in exactly the
// reference order (np.add.at: vertex position k major, then halo blocks in
// sorted order, then flat slot order; mesher.py:466-477), so the result is
// deterministic and bit-identical to the reference.
__global__ void k_fallback(DevState S, const FrameDev *__restrict__ Fp, int require_items) {
  if (halted(S)) return;
  if (require_items && ld_vol(&S.ctr->nitems_live) == 0) return;
  const int epoch = Fp->epoch;
  const int n = ld_vol(&S.ctr->nfallback);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const FallbackRec rec = S.fallback[i];
    const int v = rec.h, ob = rec.blk, ci = rec.slot / 3, axis = rec.slot % 3;
    const int lx = ci >> 6, ly = (ci >> 3) & 7, lz = ci & 7;
    // the (up to) 4 cubes sharing this edge: owner cube minus offsets in the
    // two axes orthogonal to the edge
    const int a1 = axis == 0 ? 1 : 0, a2 = axis == 2 ? 1 : 2;
    int cb[4], cc[4], key[4];
    int m = 0;
    for (int u = 0; u < 2; u++)
      for (int w = 0; w < 2; w++) {
        int l[3] = {lx, ly, lz};
        l[a1] -= u;
        l[a2] -= w;
        const int dx = l[0] < 0 ? -1 : 0, dy = l[1] < 0 ? -1 : 0, dz = l[2] < 0 ? -1 : 0;
        const int dir = nbr_dir(dx, dy, dz);
        const int nb = (dir == 13) ? ob : S.nbr[(size_t)ob * 27 + dir];
        if (nb < 0 || ld_vol(S.stamp_halo + nb) != epoch) continue;
        const int cidx = ((l[0] & 7) * 64 + (l[1] & 7) * 8 + (l[2] & 7));
        // sort key: block coordinate (offset in {-1,0}^3, lexicographic), then cube
        const int k = (((dx + 1) * 4 + (dy + 1) * 2 + (dz + 1)) << 9) | cidx;
        int j = m++;
        while (j > 0 && key[j - 1] > k) { key[j] = key[j - 1]; cb[j] = cb[j - 1]; cc[j] = cc[j - 1]; j--; }
        key[j] = k; cb[j] = nb; cc[j] = cidx;
      }
    double acc[3] = {0.0, 0.0, 0.0};
    for (int k = 0; k < 3; k++)
      for (int j = 0; j < m; j++)
        for (int s = 0; s < 5; s++) {
          const int th = S.tri[(size_t)cb[j] * kTS + cc[j] * 5 + s];
          if (th < 0 || S.tverts[3 * (size_t)th + k] != v) continue;
          const double *p0 = S.vpos + 3 * (size_t)S.tverts[3 * (size_t)th];
          const double *p1 = S.vpos + 3 * (size_t)S.tverts[3 * (size_t)th + 1];
          const double *p2 = S.vpos + 3 * (size_t)S.tverts[3 * (size_t)th + 2];
          const double a[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
          const double bb[3] = {p2[0] - p0[0], p2[1] - p0[1], p2[2] - p0[2]};
          acc[0] = __dadd_rn(acc[0], __dmul_rn(a[1], bb[2]) - __dmul_rn(a[2], bb[1]));
          acc[1] = __dadd_rn(acc[1], __dmul_rn(a[2], bb[0]) - __dmul_rn(a[0], bb[2]));
          acc[2] = __dadd_rn(acc[2], __dmul_rn(a[0], bb[1]) - __dmul_rn(a[1], bb[0]));
        }
    const double nrm = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(acc[0], acc[0]), __dmul_rn(acc[1], acc[1])),
                                      __dmul_rn(acc[2], acc[2])));
    double *dst = S.vnrm + 3 * (size_t)v;
    if (nrm > 1e-20) {
      dst[0] = (-1.0 * acc[0]) / nrm;
      dst[1] = (-1.0 * acc[1]) / nrm;
      dst[2] = (-1.0 * acc[2]) / nrm;
    } else if (dst[0] == 0.0 && dst[1] == 0.0 && dst[2] == 0.0) {
      dst[2] = 1.0;
    }
  }
}

// ------------------------------------------------------------ audit etc.
// full-scan irregular count (engine.py:169-176)
__global__ void k_irregular_full(DevState S, int nblocks, unsigned long long *out) {
  long long cnt = 0;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)nblocks * kNC;
       q += (long long)gridDim.x * blockDim.x) {
    const int32_t *s = S.tri + q * 5;
    bool has = s[0] >= 0 || s[1] >= 0 || s[2] >= 0 || s[3] >= 0 || s[4] >= 0;
    cnt += has && !is_regular_type(S.tc[q]);
  }
  cnt = warp_sum(cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, (unsigned long long)cnt);
}

// audit pass 1 over all blocks: incident-triangle tally, slot occupancy
__global__ void k_audit_blocks(DevState S, int nblocks, int32_t *tally, int32_t *seen,
                               unsigned long long *sums) {
  long long rows = 0, handles = 0, dup = 0;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < (long long)nblocks * kNC;
       q += (long long)gridDim.x * blockDim.x) {
    for (int s = 0; s < 5; s++) {
      const int th = S.tri[q * 5 + s];
      if (th < 0) continue;
      rows++;
      for (int k = 0; k < 3; k++) atomicAdd(tally + S.tverts[3 * (size_t)th + k], 1);
    }
    for (int a = 0; a < 3; a++) {
      const int h = S.ev[q * 3 + a];
      if (h < 0) continue;
      handles++;
      if (atomicAdd(seen + h, 1) > 0) dup++;
    }
  }
  rows = warp_sum(rows); handles = warp_sum(handles); dup = warp_sum(dup);
  if ((threadIdx.x & 31) == 0) {
    if (rows) atomicAdd(sums + 0, (unsigned long long)rows);
    if (handles) atomicAdd(sums + 1, (unsigned long long)handles);
    if (dup) atomicAdd(sums + 2, (unsigned long long)dup);
  }
}

// audit pass 2 over the arenas
__global__ void k_audit_pools(DevState S, int vcount, int tcount, const int32_t *tally,
                              unsigned long long *sums) {
  long long mism = 0, zero = 0, alive = 0, talive = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < vcount || i < tcount; i += gridDim.x * blockDim.x) {
    if (i < vcount) {
      mism += tally[i] != S.vref[i];
      zero += S.valive[i] && S.vref[i] == 0;
      alive += S.valive[i];
    }
    if (i < tcount) talive += S.talive[i];
  }
  mism = warp_sum(mism); zero = warp_sum(zero); alive = warp_sum(alive); talive = warp_sum(talive);
  if ((threadIdx.x & 31) == 0) {
    if (mism) atomicAdd(sums + 3, (unsigned long long)mism);
    if (zero) atomicAdd(sums + 4, (unsigned long long)zero);
    if (alive) atomicAdd(sums + 5, (unsigned long long)alive);
    if (talive) atomicAdd(sums + 6, (unsigned long long)talive);
  }
}

// refine evaluation for arbitrary (t_curr, t_prev, corners) -- exhaustive KAT
__global__ void k_refine_eval(const uint8_t *tc, const uint8_t *tp, const double *corners, int n,
                              double eps, int32_t *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double c[8];
    for (int k = 0; k < 8; k++) c[k] = corners[(size_t)i * 8 + k];
    const unsigned cur = tc[i], prev = tp[i];
    // detect_disturbance semantics: None unless a regular type was selected
    bool ch;
    if (__popc((cur ^ prev) & 0xFF) > 3) { out[i] = -1; continue; }
    unsigned r = refine_type(cur, prev, c, eps, &ch);
    // refine_type returns cur when nothing qualified; distinguish "hit with
    // cur already regular" from "no hit"
    bool hit = false;
    for (int j = 0; j < 6; j++) {
      unsigned diff = (cur ^ c_regular[j]) & 0xFF;
      if (__popc(diff) > 3) continue;
      bool ok = true;
      for (int k = 0; k < 8; k++)
        if (((diff >> k) & 1) && !(fabs(c[k]) < eps)) ok = false;
      if (ok) hit = true;
    }
    out[i] = hit ? (int)r : -1;
  }
}

__global__ void k_frustum_eval(DevState S, const FrameDev *__restrict__ Fp, const int3 *coords, int n,
                               uint8_t *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int3 c = coords[i];
    out[i] = block_in_frustum_dev(make_int4(c.x, c.y, c.z, 0), *Fp, S.extent);
  }
}

// scatter uploaded samples into blocks (vm_set_blocks)
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
// (store.py:388-425) sorted block order -> per-block counts -> scan -> fill
__global__ void k_block_keys(DevState S, int nblocks, unsigned long long *keys, int32_t *vals) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nblocks; i += gridDim.x * blockDim.x) {
    int4 c = S.bcoord[i];
    keys[i] = (unsigned long long)pack_coord(c.x, c.y, c.z);
    vals[i] = i;
  }
}

__global__ void __launch_bounds__(kThreadsCube) k_compact_count(DevState S, const int32_t *order, int nblocks,
                                                                int32_t *vcnt, int32_t *tcnt) {
  __shared__ long long red[32];
  for (int i = blockIdx.x; i < nblocks; i += gridDim.x) {
    const int b = order[i];
    long long v = 0, tt = 0;
    for (int s = threadIdx.x; s < kEV; s += blockDim.x) v += S.ev[(size_t)b * kEV + s] >= 0;
    for (int s = threadIdx.x; s < kTS; s += blockDim.x) tt += S.tri[(size_t)b * kTS + s] >= 0;
    long long rv = block_sum(v, red);
    if (threadIdx.x == 0) vcnt[i] = (int)rv;
    long long rt = block_sum(tt, red);
    if (threadIdx.x == 0) tcnt[i] = (int)rt;
  }
}

// block-wide exclusive scan of 0/1 flags; returns the flag's rank, total in *tot
__device__ __forceinline__ int block_rank(bool flag, int *sh, int *tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned ball = __ballot_sync(0xffffffffu, flag);
  __syncthreads();
  if (lane == 0) sh[wid] = __popc(ball);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int w = 0; w < nw; w++) { int c = sh[w]; sh[w] = acc; acc += c; }
    sh[32] = acc;
  }
  __syncthreads();
  *tot = sh[32];
  return sh[wid] + __popc(ball & ((1u << lane) - 1));
}

__global__ void __launch_bounds__(kThreadsCube) k_compact_vertices(DevState S, const int32_t *order, int nblocks,
                                                                   const int32_t *vbase, int32_t *remap,
                                                                   double *pos, double *nrm, long long *ages,
                                                                   long long frame) {
  __shared__ int sh[33];
  for (int i = blockIdx.x; i < nblocks; i += gridDim.x) {
    const int b = order[i];
    int base = vbase[i];
    for (int s0 = 0; s0 < kEV; s0 += blockDim.x) {
      const int s = s0 + threadIdx.x;
      const int h = S.ev[(size_t)b * kEV + s];
      int tot;
      const int r = block_rank(h >= 0, sh, &tot);
      if (h >= 0) {
        const int o = base + r;
        remap[h] = o;
        for (int d = 0; d < 3; d++) {
          pos[3 * (size_t)o + d] = S.vpos[3 * (size_t)h + d];
          nrm[3 * (size_t)o + d] = S.vnrm[3 * (size_t)h + d];
        }
        ages[o] = frame - (long long)S.vbirth[h];
      }
      base += tot;
    }
  }
}

__global__ void __launch_bounds__(kThreadsCube) k_compact_triangles(DevState S, const int32_t *order, int nblocks,
                                                                    const int32_t *tbase, const int32_t *remap,
                                                                    int32_t *idx) {
  __shared__ int sh[33];
  for (int i = blockIdx.x; i < nblocks; i += gridDim.x) {
    const int b = order[i];
    int base = tbase[i];
    for (int s0 = 0; s0 < kTS; s0 += blockDim.x) {
      const int s = s0 + threadIdx.x;
      const int th = S.tri[(size_t)b * kTS + s];
      int tot;
      const int r = block_rank(th >= 0, sh, &tot);
      if (th >= 0) {
        const int o = base + r;
        for (int k = 0; k < 3; k++) {
          const int m = remap[S.tverts[3 * (size_t)th + k]];
          if (m < 0) set_error(S, ERR_CONSISTENCY, 40, th);
          idx[3 * (size_t)o + k] = m;
        }
      }
      base += tot;
    }
  }
}

}  // namespace vm
