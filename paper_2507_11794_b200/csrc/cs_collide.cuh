// cs_collide.cuh -- broad-phase grid and narrow-phase argument blocks.
#pragma once
#include "cs_common.cuh"
#include "cs_kernels.cuh"
#include <math.h>

namespace cs {

// Uniform grid over the obstacle's bounding box.  cell_of() is monotone in x
// (RN subtract, RN multiply, floor, clamp), so a box [lo, hi] covers exactly
// the cells cell_of(lo) .. cell_of(hi) and every point inside it maps into
// that range -- the property the conservative candidate search relies on.
struct GridDesc {
    float origin[3];
    float lo[3], hi[3];   // union of the triangle boxes
    float inv_cell, cell;
    int dims[3];

    __host__ __device__ __forceinline__ int cell_of(float x, int axis) const {
#ifdef __CUDA_ARCH__
        const float f = floorf(__fmul_rn(__fsub_rn(x, origin[axis]), inv_cell));
#else
        const float f = floorf((x - origin[axis]) * inv_cell);
#endif
        if (!(f >= 0.f)) return 0;
        if (f >= (float)(dims[axis] - 1)) return dims[axis] - 1;
        return (int)f;
    }
    __host__ __device__ __forceinline__ void cell_range(const float *l, const float *h, int *a,
                                                        int *b) const {
        for (int d = 0; d < 3; ++d) {
            a[d] = cell_of(l[d], d);
            b[d] = cell_of(h[d], d);
        }
    }
    __host__ __device__ __forceinline__ bool overlaps(const float *l, const float *h) const {
        return (l[0] <= hi[0]) & (h[0] >= lo[0]) & (l[1] <= hi[1]) & (h[1] >= lo[1]) &
               (l[2] <= hi[2]) & (h[2] >= lo[2]);
    }
    __host__ __device__ __forceinline__ uint32_t key(int x, int y, int z) const {
        return (uint32_t)(((int64_t)z * dims[1] + y) * dims[0] + x);
    }
};

struct BroadPhase {
    GridDesc grid{};
    int64_t num_cells = 0;
    int64_t num_refs = 0;
    int64_t num_tris = 0;            // obstacle triangles
    uint32_t *cell_begin = nullptr;  // per cell: first index into cell_tris
    uint32_t *cell_end = nullptr;
    uint32_t *cell_keys = nullptr;   // sorted (cell key) per reference
    uint32_t *cell_tris = nullptr;   // triangle id per reference
    float *tri_box = nullptr;        // per triangle: lo xyz, hi xyz (kernels.py:62-66)
    float4 *edge_box = nullptr;      // per triangle: its 3 edges' padded boxes (kernels.py:55-59),
                                     // lo xyz hi xyz per edge, 18 floats in 5 float4`s
    // batched narrow phase: (begin, end) per cell in one 8-byte word, and per
    // sorted reference its triangle's box with the triangle id in lo.w --
    // one 32-byte load per candidate instead of ctri -> tri_box
    uint2 *cell_be = nullptr;
    float4 *ref_box = nullptr;
    bool packed_cells = false;       // every grid axis <= 1024 cells (10-bit packing)
    int warp_per_query = 3;          // narrow phase: one fused candidate enumeration per
                                     // cloth triangle for both passes (3, default),
                                     // 32-query batches per warp and pass (2), warp per
                                     // query (1) or thread per query (0)
    uint8_t *tri_own = nullptr;      // mode 3: per cloth triangle, the unique edges it owns
                                     // (bit k: nodes k, k+1 mod 3; each edge owned once)
};

struct CollideArgs {
    const float *pos;       // current state base (planes x y z vx vy vz)
    int64_t plane;
    int32_t *acc;           // 3 planes, i32 fixed point (responseAccumulator)
    int32_t *count;         // 1 plane (responseCount)
    uint32_t *touched;      // nodes whose count went 0 -> 1 this frame
    uint32_t *touched_n;
    uint32_t *blocks_done;            // k_respond's last-block counter (self-resetting)
    unsigned long long *frame_hits;
    unsigned long long *frame_responded;
    unsigned long long *hit_counter;  // cumulative hitCounter
    unsigned long long *frame_counter;
    unsigned long long *ring;         // per-frame (hits, responded), ring_size frames
    int ring_size;
    uint32_t *clog;                   // optional contact log: (storage node, triangle)
    uint32_t *clog_n;
    uint32_t clog_cap;
    float eps, margin, pad, scale_f;
    double scale_d;
    // row bands: only nodes with storage index in [own_lo, own_hi) receive
    // contacts, and a hit counts only when its primitive's minimum node is
    // owned -- the union over bands equals one engine
    int64_t own_lo, own_hi;
};

// RAII device scratch for construction-time helpers
struct DeviceScratch {
    void *p = nullptr;
    size_t n = 0;
    void *get(size_t bytes) {
        if (bytes > n) {
            if (p) cudaFree(p);
            cudaMalloc(&p, bytes);
            n = bytes;
        }
        return p;
    }
    ~DeviceScratch() {
        if (p) cudaFree(p);
    }
};

void scan_exclusive(const uint32_t *in, uint32_t *out, int64_t n, DeviceScratch &scratch,
                    cudaStream_t st);
void radix_sort_pairs(uint32_t *keys, uint32_t *vals, uint32_t *tmp_keys, uint32_t *tmp_vals,
                      int64_t n, int key_bits, DeviceScratch &scratch, cudaStream_t st);
int build_broadphase(BroadPhase &bp, const float *d_corners, int64_t nt, const float *h_corners,
                     float cell_size, cudaStream_t st);
void free_broadphase(BroadPhase &bp);
void launch_detect(const CollideArgs &A, const BroadPhase &bp, const float *corners,
                   const float *normals, const int32_t *edges, int64_t ne, const int32_t *tris,
                   int64_t nc, cudaStream_t st);
void launch_respond(const CollideArgs &A, float *state, const uint32_t *pinbits,
                    const float *inv_mass, int average, int64_t max_nodes, int num_sms,
                    bool end_of_frame, cudaStream_t st);
void launch_respond_end(const CollideArgs &A, bool end_of_frame, cudaStream_t st);
void launch_rebuild_touched(const CollideArgs &A, int64_t rows, int64_t nx, int64_t pitch,
                            cudaStream_t st);

}  // namespace cs
