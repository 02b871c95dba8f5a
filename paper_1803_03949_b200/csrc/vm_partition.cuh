// vm_partition.cuh -- kernels of the spatially partitioned reconstruction
// (DESIGN.md section 6): the halo exchange of boundary blocks
// before meshing, and the per-rank half of the distributed compaction.
//
// Ownership: blocks belong to hashed tiles of 2^tile_shift blocks per axis
// (tile_owner); a rank meshes its owned blocks plus a 1-block margin, so all
// of its owned results (types, vertex slots, GC decisions, normals) are exact.
// In halo-exchange mode (DevState::halo_exchange) the margin blocks' samples
// are not integrated by the rank itself: every owner packs its collected
// boundary blocks (k_pack_boundary), the ranks all-gather the records (NCCL
// on the GPU box, gloo in the CPU tests) and each rank adopts the ones in its
// margin as collected "ghost" blocks (k_unpack_ghosts + k_fuse_blocks
// F_GHOST) -- the owner's integration, bit for bit.
#pragma once
#include "vm_kernels.cuh"

namespace vm {

// Pack the collected owned blocks that lie in another rank's margin:
// coordinate, 512 tsdf, 512 weights (kGhostRec bytes).  One CTA per block,
// after k_fuse_blocks integrated them.  Records past `cap` are counted, not
// written (the host grows the buffer and packs again).
__global__ void __launch_bounds__(kFB) k_pack_boundary(DevState S, const FrameDev F, uint8_t *__restrict__ send,
                                                      int cap) {
  cudaGridDependencySynchronize();
  __shared__ int s_pro[5];
  __shared__ int s_pos;
  read_prologue(S, s_pro, &S.ctr->ncollected, nullptr, nullptr, nullptr);
  if (s_pro[0]) return;
  const int n = s_pro[1];
  const int t = threadIdx.x;
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    const int b = __ldcg(S.scope + i);
    const int4 c = __ldcg(S.bcoord + b);
    if (!block_on_boundary(S, c.x, c.y, c.z)) continue;   // (uniform over the CTA)
    if (t == 0) s_pos = atomicAdd(&S.ctr->nsend, 1);
    __syncthreads();
    const int pos = s_pos;
    __syncthreads();   // (s_pos is rewritten by the next item)
    if (pos >= cap) continue;
    uint8_t *rec = send + (size_t)pos * kGhostRec;
    if (t == 0) *reinterpret_cast<int4 *>(rec) = make_int4(c.x, c.y, c.z, 0);
    const double2 *ts = reinterpret_cast<const double2 *>(S.tsdf + (size_t)b * kNC);
    double2 *td = reinterpret_cast<double2 *>(rec + 16);
#pragma unroll
    for (int j = 0; j < kNC / 2 / kFB; j++) td[t + j * kFB] = __ldcg(ts + t + j * kFB);
    const int4 *ws = reinterpret_cast<const int4 *>(S.weight + (size_t)b * kNC);
    reinterpret_cast<int4 *>(rec + 16 + 8 * kNC)[t] = __ldcg(ws + t);
  }
}

// Adopt the received records that lie in this rank's margin: find or
// allocate the block, mark it collected this call and append it to the scope
// list (its record index in ghost_src at the same position).  The host sized
// the block heap for every received record beforehand, so no frame resumes.
__global__ void k_unpack_ghosts(DevState S, const FrameDev F) {
  if (halted(S)) return;
  const int total = F.ghost_nranks * F.ghost_max;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < total; r += gridDim.x * blockDim.x) {
    const int q = r / F.ghost_max, k = r - q * F.ghost_max;
    if (q == S.rank || k >= __ldg(S.ghost_counts + q)) continue;
    const int4 c = *reinterpret_cast<const int4 *>(F.ghost_recv + (size_t)r * kGhostRec);
    if (!block_in_margin(S, c.x, c.y, c.z)) continue;
    HashRef h = hash_find_ref(S, c.x, c.y, c.z);
    if (h.idx == -1) h = hash_insert_ref(S, c.x, c.y, c.z, F.epoch);
    if (h.idx == -2) set_error(S, ERR_CAPACITY, S.max_blocks, S.table_size, 1, F.epoch);
    if (h.idx >= 0 && h.stamp != F.epoch && atomicExch(h.stamp_ptr, F.epoch) != F.epoch) {
      S.stamp_collect[h.idx] = F.epoch;
      const int pos = atomicAdd(&S.ctr->ncollected, 1);
      S.scope[pos] = h.idx;
      S.ghost_src[pos] = r;
    }
  }
}

// ---------------------------------------------------------------- compaction
// Sort keys of this rank's OWNED blocks (others sort to the end).
__global__ void k_owned_block_keys(DevState S, int nblocks, unsigned long long *keys, int32_t *vals) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nblocks; i += gridDim.x * blockDim.x) {
    const int4 c = S.bcoord[i];
    const bool own = (S.nranks <= 1 || S.bowned[i]) && c.w == 0;
    keys[i] = own ? (unsigned long long)pack_coord(c.x, c.y, c.z) : ~0ull;
    vals[i] = i;
  }
}

// binary search of a packed block key in the globally sorted key list
__device__ __forceinline__ int find_key(const unsigned long long *__restrict__ keys, int n, unsigned long long k) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(keys + mid) < k) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && __ldg(keys + lo) == k) ? lo : -1;
}

// Triangles of this rank's owned blocks at their GLOBAL positions
// (store.py:396-406): a vertex owned by block g (any rank's) is
// vbase[g] + (occupied slots of g before it), from the gathered occupancy of
// every rank's owned blocks -- never from a local margin replica, whose
// occupancy may lack slots only cubes outside this rank's margin reference.
__global__ void __launch_bounds__(kThreadsCube) k_pcompact_triangles(
    DevState S, const int32_t *order, int nown, const int32_t *__restrict__ my_global,
    const unsigned long long *__restrict__ gkeys, int nglobal, const int64_t *__restrict__ vbase,
    const int64_t *__restrict__ tbase, const uint32_t *__restrict__ gocc, const int32_t *__restrict__ gocc_pre,
    int32_t *idx) {
  __shared__ int sh[33];
  for (int i = blockIdx.x; i < nown; i += gridDim.x) {
    const int b = order[i];
    const int gi = my_global[i];
    const int4 bc = S.bcoord[b];
    const int t = threadIdx.x;
    const int x = t >> 6, y = (t >> 3) & 7, z = t & 7;
    const unsigned tt = S.tc[(size_t)b * kNC + t];
    const int ntri = c_tri_count[tt];
    int tot;
    const int r = block_rank(ntri, sh, &tot);
    const unsigned long long packed = c_tri_packed[tt];
    for (int j = 0; j < ntri; j++) {
      const long long o = tbase[gi] + r + j;
      for (int k = 0; k < 3; k++) {
        const int e = (int)((packed >> (4 * (3 * j + k))) & 0xF);
        const int own = c_e_own[e];
        const int ox = x + (own & 1), oy = y + ((own >> 1) & 1), oz = z + ((own >> 2) & 1);
        const int gb = (ox | oy | oz) >> 3 ? find_key(gkeys, nglobal, (unsigned long long)pack_coord(
                                                  bc.x + (ox >> 3), bc.y + (oy >> 3), bc.z + (oz >> 3)))
                                           : gi;
        const int s = ((ox & 7) * 64 + (oy & 7) * 8 + (oz & 7)) * 3 + c_e_axis[e];
        int m = -1;
        if (gb >= 0) {
          const uint32_t w = __ldg(gocc + (size_t)gb * 48 + (s >> 5));
          if ((w >> (s & 31)) & 1u)
            m = (int)(vbase[gb] + __ldg(gocc_pre + (size_t)gb * 48 + (s >> 5)) + __popc(w & ((1u << (s & 31)) - 1)));
        }
        if (m < 0) set_error(S, ERR_CONSISTENCY, 40, b);
        idx[3 * (size_t)o + k] = m;
      }
    }
    __syncthreads();
  }
}

}  // namespace vm
