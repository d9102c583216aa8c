// Device-side state of the BFS driver (drivers.cu) shared with the fused
// level-sweep kernel (bmv_stream.cu).
#pragma once

#include "b2sr_internal.cuh"

namespace b2sr {

constexpr uint32_t PUSH_CH = 1024;  // tiles per push work entry (hub rows split)

struct BfsCounters {
    int any;
    uint32_t list_n;                     // push work entries
    unsigned long long frontier_tiles;   // tiles of a in frontier tile rows
    unsigned long long removed_tiles;    // tiles of at rows whose keep word became zero
    unsigned long long frontier_vertices;
};

// Direction of one level, chosen on the device from the previous level's counters.
enum BfsMode : int { BFS_NONE = 0, BFS_PUSH = 1, BFS_PULL = 2, BFS_PULL_ACTIVE = 3 };

struct BfsCtl {
    int mode;
    int done;
    uint32_t list_n;       // push entries of this level (copied from cnt)
    uint32_t active_n;     // active loads of this level
    unsigned long long unvisited;
    long long sweeps;
    uint32_t blocks_done;  // last-block detection in the update kernel
    int sparse;            // pull over a sparse frontier: fetch tile bytes lazily
    BfsCounters cnt;       // written by the level's update, consumed by the next plan
};

// One level's outcome as the host sees it (mapped host memory ring).
// One 8-byte word (a single store from the device, a single load on the host:
// no system-scope fence between fields): level | done << 32 | sweeps << 33.
struct BfsSnap {
    unsigned long long w;
};
__host__ __device__ inline unsigned long long bfs_snap_pack(uint32_t level, int done, long long sweeps) {
    return (unsigned long long)level | ((unsigned long long)(done ? 1 : 0) << 32) |
           ((unsigned long long)(sweeps & 0x7FFFFFFFll) << 33);
}
inline void bfs_snap_read(const volatile BfsSnap *s, uint32_t *level, int *done, long long *sweeps) {
    const unsigned long long w = s->w;
    *level = (uint32_t)w;
    *done = (int)((w >> 32) & 1u);
    *sweeps = (long long)(w >> 33);
}

// One fused level (bmv_stream.cu): push levels scatter the OR of the frontier
// bit-rows of every listed chunk of a into next (visited != null: bits of
// visited vertices dropped first; the update masks them either way); pull
// levels stream at.
// Row blocks (multi-GPU): push reads the frontier words of a's rows at
// `pfrontier` (the global frontier shifted to the block) and scatters into
// the global-length `pnext`; pull writes the block's rows at `next`.  NULL:
// pfrontier = frontier, pnext = next (one GPU).
void launch_bfs_level(b2sr_matrix *at, const b2sr_matrix *a, BfsCtl *ctl, const uint2 *push_list,
                      const uint32_t *active_list, const void *hx, size_t hb, const void *frontier, void *next,
                      const void *visited, cudaStream_t s, const void *pfrontier = nullptr, void *pnext = nullptr,
                      bool pdl = false);
// Top-down level of the push-only BFS (no transpose; d = 4, 8): the listed
// chunks of a, bits of visited vertices dropped before the scatter.
void launch_bfs_push_level(const b2sr_matrix *a, const BfsCtl *ctl, const uint2 *push_list, const void *frontier,
                           const void *visited, void *next, cudaStream_t s, bool pdl = false);

}  // namespace b2sr
