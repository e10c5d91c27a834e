// cs_collide.cu -- cloth vs static triangle mesh: uniform-grid broad phase
// (built on device once per obstacle), the two narrow-phase passes and the
// respond pass.
//
// Reference semantics (all bit-exact):
//   narrow-phase predicate  gpu/kernels.py:136-168 (_segment_triangle_f32),
//                           collision.py:96-146
//   pass A (cloth edges)    gpu/kernels.py:186-237, detect_cloth_edges.wgsl
//   pass B (obstacle edges) gpu/kernels.py:240-290, detect_obstacle_edges.wgsl
//   accumulation            gpu/kernels.py:171-183 (i32 fixed point, atomics)
//   respond                 gpu/kernels.py:293-311, respond.wgsl
//   box prefilter           gpu/kernels.py:55-78 (BOX_PAD = 1e-5)
//
// The reference tests every (edge, triangle) pair and rejects most with a
// padded axis-aligned box test before the Moller-Trumbore algebra.  Here the
// candidate pairs come from a static uniform grid over the obstacle
// triangles; each candidate then runs the reference's exact box test and
// predicate, so the hit set equals the reference's (its own tests assert that
// prefilter == brute force, test_gpu_engine.py:267-307).  A pair seen from
// several cells is processed only in the cell holding the minimum corner of
// the two boxes' intersection, so every pair is tested exactly once.
//
// Broad-phase build (construction time; the obstacle is static):
//   1. per triangle: count covered cells            (k_tri_cell_count)
//   2. block-wide warp-shuffle exclusive scan        (scan_exclusive)
//   3. emit (cell key, triangle id) pairs            (k_tri_cell_emit)
//   4. LSD radix sort of the keys, 8 bits per pass   (radix_sort_pairs)
//   5. cell [begin, end) by adjacent difference      (k_cell_ranges)
#include "cs_collide.cuh"

namespace cs {

// ============================================================================
// scans and radix sort
// ============================================================================
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Exclusive scan of a u32 array in one kernel with chained per-block
// reductions (three phases: block sums, scan of block sums, block scan).
constexpr int SCAN_BLOCK = 1024;
constexpr int SCAN_ITEMS = 4;  // per thread
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_ITEMS;

__device__ uint32_t block_excl_scan(uint32_t v, uint32_t *total) {
    __shared__ uint32_t warp_sums[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t inc = warp_incl_scan(v);
    if (lane == 31) warp_sums[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        uint32_t w = lane < nw ? warp_sums[lane] : 0u;
        w = warp_incl_scan(w);
        if (lane < nw) warp_sums[lane] = w;
    }
    __syncthreads();
    const uint32_t base = wid ? warp_sums[wid - 1] : 0u;
    if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
    __syncthreads();
    return base + inc - v;
}

__global__ void k_scan_tiles(const uint32_t *in, uint32_t *out, int64_t n, uint32_t *tile_sums) {
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    uint32_t v[SCAN_ITEMS], s = 0;
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) {
        v[q] = (base + q < n) ? in[base + q] : 0u;
        s += v[q];
    }
    uint32_t total;
    uint32_t pre = block_excl_scan(s, &total);
#pragma unroll
    for (int q = 0; q < SCAN_ITEMS; ++q) {
        if (base + q < n) out[base + q] = pre;
        pre += v[q];
    }
    if (threadIdx.x == 0 && tile_sums) tile_sums[blockIdx.x] = total;
}

__global__ void k_add_tile_offsets(uint32_t *out, int64_t n, const uint32_t *tile_offsets) {
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    const uint32_t add = tile_offsets[blockIdx.x];
    for (int64_t q = threadIdx.x; q < SCAN_TILE; q += blockDim.x)
        if (base + q < n) out[base + q] += add;
}

// out[i] = sum(in[0..i)), recursive over tiles; returns the total via *d_total
// (device scalar) when given.
void scan_exclusive(const uint32_t *in, uint32_t *out, int64_t n, DeviceScratch &scratch,
                    cudaStream_t st) {
    if (n <= 0) return;
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (tiles == 1) {
        k_scan_tiles<<<1, SCAN_BLOCK, 0, st>>>(in, out, n, nullptr);
        return;
    }
    uint32_t *sums = (uint32_t *)scratch.get(tiles * sizeof(uint32_t) * 2 + 256);
    uint32_t *offs = sums + tiles;
    k_scan_tiles<<<(unsigned)tiles, SCAN_BLOCK, 0, st>>>(in, out, n, sums);
    DeviceScratch inner;
    scan_exclusive(sums, offs, tiles, inner, st);
    k_add_tile_offsets<<<(unsigned)tiles, SCAN_BLOCK, 0, st>>>(out, n, offs);
    cudaStreamSynchronize(st);  // `inner` is released on return
}

// ---- LSD radix sort of (key, value) u32 pairs, 8-bit digits -----------------------
constexpr int RS_BLOCK = 256;
constexpr int RS_CHUNK = 4096;  // items per block

__global__ void k_radix_hist(const uint32_t *keys, int64_t n, int shift, uint32_t *hist,
                             int nblocks) {
    __shared__ uint32_t h[256];
    for (int d = threadIdx.x; d < 256; d += blockDim.x) h[d] = 0;
    __syncthreads();
    const int64_t lo = (int64_t)blockIdx.x * RS_CHUNK;
    const int64_t hi = min(lo + RS_CHUNK, n);
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
        atomicAdd(&h[(keys[i] >> shift) & 255u], 1u);
    __syncthreads();
    // digit-major so one exclusive scan yields every (digit, block) offset
    for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[(int64_t)d * nblocks + blockIdx.x] = h[d];
}

// Stable scatter: items of a chunk are ranked in order, 256 at a time; lanes
// with equal digits are ranked with __match_any_sync.
__global__ void k_radix_scatter(const uint32_t *keys, const uint32_t *vals, uint32_t *okeys,
                                uint32_t *ovals, int64_t n, int shift, const uint32_t *offsets,
                                int nblocks) {
    __shared__ uint32_t base[256];
    __shared__ uint32_t wcount[RS_BLOCK / 32][256];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int d = threadIdx.x; d < 256; d += blockDim.x) base[d] = offsets[(int64_t)d * nblocks + blockIdx.x];
    const int64_t lo = (int64_t)blockIdx.x * RS_CHUNK;
    const int64_t hi = min(lo + RS_CHUNK, n);
    for (int64_t t0 = lo; t0 < hi; t0 += RS_BLOCK) {
        for (int q = threadIdx.x; q < (RS_BLOCK / 32) * 256; q += blockDim.x) (&wcount[0][0])[q] = 0;
        __syncthreads();
        const int64_t i = t0 + threadIdx.x;
        const bool valid = i < hi;
        const uint32_t k = valid ? keys[i] : 0u;
        const uint32_t d = valid ? ((k >> shift) & 255u) : 256u;  // 256 never matches a real digit
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
        if (valid && rank == 0) wcount[wid][d] = __popc(peers);
        __syncthreads();
        // exclusive prefix over warps for this thread's digit
        uint32_t before = 0;
        if (valid)
            for (int w = 0; w < wid; ++w) before += wcount[w][d];
        if (valid) {
            const uint32_t pos = base[d] + before + rank;
            okeys[pos] = k;
            ovals[pos] = vals[i];
        }
        __syncthreads();
        // advance per-digit bases by this sub-tile's counts
        for (int dd = threadIdx.x; dd < 256; dd += blockDim.x) {
            uint32_t c = 0;
            for (int w = 0; w < RS_BLOCK / 32; ++w) c += wcount[w][dd];
            base[dd] += c;
        }
        __syncthreads();
    }
}

void radix_sort_pairs(uint32_t *keys, uint32_t *vals, uint32_t *tmp_keys, uint32_t *tmp_vals,
                      int64_t n, int key_bits, DeviceScratch &scratch, cudaStream_t st) {
    if (n <= 1) return;
    const int nblocks = (int)((n + RS_CHUNK - 1) / RS_CHUNK);
    uint32_t *hist = (uint32_t *)scratch.get((size_t)256 * nblocks * sizeof(uint32_t) * 2 + 256);
    uint32_t *offs = hist + (size_t)256 * nblocks;
    uint32_t *ka = keys, *va = vals, *kb = tmp_keys, *vb = tmp_vals;
    int passes = (key_bits + 7) / 8;
    if (passes < 1) passes = 1;
    for (int pass = 0; pass < passes; ++pass) {
        const int shift = pass * 8;
        k_radix_hist<<<nblocks, RS_BLOCK, 0, st>>>(ka, n, shift, hist, nblocks);
        DeviceScratch s2;
        scan_exclusive(hist, offs, (int64_t)256 * nblocks, s2, st);
        k_radix_scatter<<<nblocks, RS_BLOCK, 0, st>>>(ka, va, kb, vb, n, shift, offs, nblocks);
        cudaStreamSynchronize(st);
        uint32_t *t = ka; ka = kb; kb = t;
        t = va; va = vb; vb = t;
    }
    if (ka != keys) {
        cudaMemcpyAsync(keys, ka, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(vals, va, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
    }
}

// ============================================================================
// broad-phase build
// ============================================================================
__device__ __forceinline__ void tri_box(const float *c, float *lo, float *hi) {
    // kernels.py:62-66 triangle_boxes (unpadded)
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        lo[d] = fminf(fminf(c[d], c[3 + d]), c[6 + d]);
        hi[d] = fmaxf(fmaxf(c[d], c[3 + d]), c[6 + d]);
    }
}

__global__ void k_tri_cell_count(const GridDesc g, int64_t nt, const float *__restrict__ corners,
                                 uint32_t *__restrict__ counts) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    float lo[3], hi[3];
    tri_box(corners + 9 * t, lo, hi);
    int a[3], b[3];
    g.cell_range(lo, hi, a, b);
    counts[t] = (uint32_t)((b[0] - a[0] + 1) * (b[1] - a[1] + 1) * (b[2] - a[2] + 1));
}

__global__ void k_tri_cell_emit(const GridDesc g, int64_t nt, const float *__restrict__ corners,
                                const uint32_t *__restrict__ offsets, uint32_t *__restrict__ keys,
                                uint32_t *__restrict__ vals) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    float lo[3], hi[3];
    tri_box(corners + 9 * t, lo, hi);
    int a[3], b[3];
    g.cell_range(lo, hi, a, b);
    uint32_t o = offsets[t];
    for (int z = a[2]; z <= b[2]; ++z)
        for (int y = a[1]; y <= b[1]; ++y)
            for (int x = a[0]; x <= b[0]; ++x) {
                keys[o] = g.key(x, y, z);
                vals[o] = (uint32_t)t;
                ++o;
            }
}

__global__ void k_cell_ranges(const uint32_t *__restrict__ keys, int64_t n,
                              uint32_t *__restrict__ cell_begin, uint32_t *__restrict__ cell_end) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = keys[i];
    if (i == 0 || keys[i - 1] != k) cell_begin[k] = (uint32_t)i;
    if (i == n - 1 || keys[i + 1] != k) cell_end[k] = (uint32_t)(i + 1);
}

static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

void launch_tri_boxes(int64_t nt, const float *corners, float *box, cudaStream_t st);
void launch_edge_boxes(int64_t nt, const float *corners, float4 *box, cudaStream_t st);
// per obstacle triangle, its 3 edges' boxes padded by BOX_PAD (kernels.py:55-59:
// lo = min(st, en) - pad, hi = max(st, en) + pad, f32, pad fixed at 1e-5 as
// CollideArgs::pad), 18 floats in 5 float4 (the fused narrow phase's pass B)
__global__ void k_edge_boxes(int64_t nt, const float *__restrict__ corners,
                             float4 *__restrict__ box, float pad) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const float *c = corners + 9 * t;
    float f[20];
#pragma unroll
    for (int slot = 0; slot < 3; ++slot) {
        const float *st = c + 3 * slot;
        const float *en = c + 3 * (slot == 2 ? 0 : slot + 1);
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            f[6 * slot + d] = __fsub_rn(fminf(st[d], en[d]), pad);
            f[6 * slot + 3 + d] = __fadd_rn(fmaxf(st[d], en[d]), pad);
        }
    }
    f[18] = f[19] = 0.f;
#pragma unroll
    for (int q = 0; q < 5; ++q) box[5 * t + q] = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
}
void launch_edge_boxes(int64_t nt, const float *corners, float4 *box, cudaStream_t st) {
    if (nt > 0) k_edge_boxes<<<nblk(nt, 256), 256, 0, st>>>(nt, corners, box, 1e-5f);
}

__global__ void k_pack_cells(int64_t n, const uint32_t *__restrict__ beg,
                             const uint32_t *__restrict__ end, uint2 *__restrict__ be) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) be[i] = make_uint2(beg[i], end[i]);
}

// per sorted reference: its triangle's box, the triangle id (lo.w) and the
// grid cell of the box's minimum corner packed 10:10:10 (hi.w) -- the dedup
// test then needs no cell_of per candidate, because cell_of is monotone:
// cell_of(max(q_lo, t_lo)) == max(cell_of(q_lo), cell_of(t_lo)).
__global__ void k_ref_boxes(const GridDesc g, int64_t n, const uint32_t *__restrict__ tris,
                            const float *__restrict__ tbox, float4 *__restrict__ out) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t t = tris[r];
    const float *b = tbox + 6 * (int64_t)t;
    const uint32_t cell = (uint32_t)g.cell_of(b[0], 0) | ((uint32_t)g.cell_of(b[1], 1) << 10) |
                          ((uint32_t)g.cell_of(b[2], 2) << 20);
    out[2 * r] = make_float4(b[0], b[1], b[2], __uint_as_float(t));
    out[2 * r + 1] = make_float4(b[3], b[4], b[5], __uint_as_float(cell));
}

int build_broadphase(BroadPhase &bp, const float *d_corners, int64_t nt, const float *h_corners,
                     float cell_size, cudaStream_t st) {
    // grid over the obstacle's bounding box (host: static data, computed once)
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    double mean_ext = 0.0;
    for (int64_t t = 0; t < nt; ++t) {
        float a[3], b[3];
        for (int d = 0; d < 3; ++d) {
            const float *c = h_corners + 9 * t;
            a[d] = fminf(fminf(c[d], c[3 + d]), c[6 + d]);
            b[d] = fmaxf(fmaxf(c[d], c[3 + d]), c[6 + d]);
            lo[d] = fminf(lo[d], a[d]);
            hi[d] = fmaxf(hi[d], b[d]);
        }
        mean_ext += fmax(fmax(b[0] - a[0], b[1] - a[1]), b[2] - a[2]);
    }
    mean_ext /= (double)(nt > 0 ? nt : 1);
    // cells about one triangle box across: C3 sweep (tools/c3_cells.py) put
    // the optimum near 1x the mean extent (2x was 40% slower)
    float cs_ = cell_size > 0.f ? cell_size : (float)(1.0 * mean_ext);
    if (!(cs_ > 0.f)) cs_ = 1.0f;
    int dims[3];
    for (;;) {
        int64_t total = 1;
        for (int d = 0; d < 3; ++d) {
            dims[d] = (int)ceil((double)(hi[d] - lo[d]) / cs_) + 1;
            if (dims[d] < 1) dims[d] = 1;
            total *= dims[d];
        }
        if (total <= (int64_t)1 << 24) break;  // keys stay within 24 bits
        cs_ *= 1.25f;
    }
    GridDesc &g = bp.grid;
    for (int d = 0; d < 3; ++d) {
        g.origin[d] = lo[d];
        g.dims[d] = dims[d];
        g.lo[d] = lo[d];
        g.hi[d] = hi[d];
    }
    g.inv_cell = 1.0f / cs_;
    g.cell = cs_;
    bp.num_cells = (int64_t)dims[0] * dims[1] * dims[2];
    bp.num_tris = nt;

    uint32_t *counts, *offsets;
    cudaMalloc(&counts, (nt + 1) * sizeof(uint32_t));
    cudaMalloc(&offsets, (nt + 1) * sizeof(uint32_t));
    cudaMemsetAsync(counts, 0, (nt + 1) * sizeof(uint32_t), st);
    k_tri_cell_count<<<nblk(nt, 256), 256, 0, st>>>(g, nt, d_corners, counts);
    DeviceScratch scratch;
    scan_exclusive(counts, offsets, nt + 1, scratch, st);
    uint32_t total = 0;
    cudaMemcpyAsync(&total, offsets + nt, sizeof(uint32_t), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    bp.num_refs = total;
    uint32_t *keys, *vals, *tk, *tv;
    cudaMalloc(&keys, (total + 1) * sizeof(uint32_t));
    cudaMalloc(&vals, (total + 1) * sizeof(uint32_t));
    cudaMalloc(&tk, (total + 1) * sizeof(uint32_t));
    cudaMalloc(&tv, (total + 1) * sizeof(uint32_t));
    k_tri_cell_emit<<<nblk(nt, 256), 256, 0, st>>>(g, nt, d_corners, offsets, keys, vals);
    int bits = 1;
    while (((int64_t)1 << bits) < bp.num_cells) ++bits;
    radix_sort_pairs(keys, vals, tk, tv, total, bits, scratch, st);
    cudaMalloc(&bp.cell_begin, bp.num_cells * sizeof(uint32_t));
    cudaMalloc(&bp.cell_end, bp.num_cells * sizeof(uint32_t));
    cudaMemsetAsync(bp.cell_begin, 0, bp.num_cells * sizeof(uint32_t), st);
    cudaMemsetAsync(bp.cell_end, 0, bp.num_cells * sizeof(uint32_t), st);
    k_cell_ranges<<<nblk(total, 256), 256, 0, st>>>(keys, total, bp.cell_begin, bp.cell_end);
    bp.cell_keys = keys;  // sorted keys (kept for the bit-exact assignment test)
    bp.cell_tris = vals;
    cudaStreamSynchronize(st);
    cudaFree(counts);
    cudaFree(offsets);
    cudaFree(tk);
    cudaMalloc(&bp.tri_box, 6 * (nt > 0 ? nt : 1) * sizeof(float));
    launch_tri_boxes(nt, d_corners, bp.tri_box, st);
    cudaMalloc(&bp.edge_box, 5 * (nt > 0 ? nt : 1) * sizeof(float4));
    launch_edge_boxes(nt, d_corners, bp.edge_box, st);
    cudaMalloc(&bp.cell_be, bp.num_cells * sizeof(uint2));
    cudaMalloc(&bp.ref_box, 2 * (total + 1) * sizeof(float4));
    k_pack_cells<<<nblk(bp.num_cells, 256), 256, 0, st>>>(bp.num_cells, bp.cell_begin, bp.cell_end,
                                                          bp.cell_be);
    if (total > 0)
        k_ref_boxes<<<nblk(total, 256), 256, 0, st>>>(g, total, bp.cell_tris, bp.tri_box, bp.ref_box);
    bp.packed_cells = dims[0] <= 1024 && dims[1] <= 1024 && dims[2] <= 1024;
    cudaFree(tv);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

void free_broadphase(BroadPhase &bp) {
    cudaFree(bp.tri_own);
    cudaFree(bp.edge_box);
    cudaFree(bp.cell_be);
    cudaFree(bp.ref_box);
    cudaFree(bp.cell_begin);
    cudaFree(bp.cell_end);
    cudaFree(bp.cell_keys);
    cudaFree(bp.cell_tris);
    cudaFree(bp.tri_box);
    bp = BroadPhase();
}

// ============================================================================
// narrow phase
// ============================================================================

// _segment_triangle_f32 (kernels.py:136-168) with numpy's exact operation order
__device__ __forceinline__ bool seg_tri(const float *st, const float *en, const float *v0,
                                        const float *v1, const float *v2, float eps, float *pt) {
    const float d0 = fsub(en[0], st[0]), d1 = fsub(en[1], st[1]), d2 = fsub(en[2], st[2]);
    const float d_len = fsqrt(dot3x(d0, d1, d2, d0, d1, d2));
    if (!(d_len > eps)) return false;
    float r0, r1, r2;  // d / |d|: IEEE quotients, one shared reciprocal (div3)
    div3<true>(d0, d1, d2, d_len, r0, r1, r2);
    const float e10 = fsub(v1[0], v0[0]), e11 = fsub(v1[1], v0[1]), e12 = fsub(v1[2], v0[2]);
    const float e20 = fsub(v2[0], v0[0]), e21 = fsub(v2[1], v0[1]), e22 = fsub(v2[2], v0[2]);
    const float h0 = fsub(fmul(r1, e22), fmul(r2, e21));
    const float h1 = fsub(fmul(r2, e20), fmul(r0, e22));
    const float h2 = fsub(fmul(r0, e21), fmul(r1, e20));
    const float a = dot3x(e10, e11, e12, h0, h1, h2);
    if (!(fabsf(a) >= eps)) return false;
    const float f = fdiv(1.0f, a);
    const float s0 = fsub(st[0], v0[0]), s1 = fsub(st[1], v0[1]), s2 = fsub(st[2], v0[2]);
    const float u = fmul(f, dot3x(s0, s1, s2, h0, h1, h2));
    if (!((u >= 0.f) & (u <= 1.f))) return false;
    const float q0 = fsub(fmul(s1, e12), fmul(s2, e11));
    const float q1 = fsub(fmul(s2, e10), fmul(s0, e12));
    const float q2 = fsub(fmul(s0, e11), fmul(s1, e10));
    const float v = fmul(f, dot3x(r0, r1, r2, q0, q1, q2));
    if (!((v >= 0.f) & (fadd(u, v) <= 1.f))) return false;
    const float t = fmul(f, dot3x(e20, e21, e22, q0, q1, q2));
    if (!((t > eps) & (t < d_len))) return false;
    pt[0] = fadd(st[0], fmul(t, r0));
    pt[1] = fadd(st[1], fmul(t, r1));
    pt[2] = fadd(st[2], fmul(t, r2));
    return true;
}

// np.maximum (NaN propagating)
__device__ __forceinline__ float np_max(float a, float b) {
    if (a != a || b != b) return __int_as_float(0x7fc00000);
    return a >= b ? a : b;
}

// _accumulate_hits (kernels.py:171-183) for one node; returns true when the
// node's count went 0 -> 1 (it joins the touched list).
__device__ __forceinline__ void accumulate(const CollideArgs &A, int64_t g, const float *p,
                                           const float *hit, const float *on, uint32_t tri) {
    if (g < A.own_lo || g >= A.own_hi) return;  // another band's node
    if (A.clog) {  // optional (node, triangle) contact log for the parity tests
        const uint32_t slot = atomicAdd(A.clog_n, 1u);
        if (slot < A.clog_cap) {
            A.clog[2 * slot] = (uint32_t)g;
            A.clog[2 * slot + 1] = tri;
        }
    }
    const float depth0 = -dot3x(fsub(p[0], hit[0]), fsub(p[1], hit[1]), fsub(p[2], hit[2]), on[0],
                                on[1], on[2]);
    const float depth = np_max(depth0, 0.f);
    const float sc = fadd(depth, A.margin);
    atomicAdd(A.acc + g, encode_fixed(fmul(on[0], sc), A.scale_f));
    atomicAdd(A.acc + A.plane + g, encode_fixed(fmul(on[1], sc), A.scale_f));
    atomicAdd(A.acc + 2 * A.plane + g, encode_fixed(fmul(on[2], sc), A.scale_f));
    const int old = atomicAdd(A.count + g, 1);
    if (old == 0) {
        const uint32_t slot = atomicAdd(A.touched_n, 1u);
        A.touched[slot] = (uint32_t)g;
    }
}

__device__ __forceinline__ uint32_t owned_hit(const CollideArgs &A, int64_t min_node) {
    return (min_node >= A.own_lo) & (min_node < A.own_hi);
}

__device__ __forceinline__ void load_pos(const CollideArgs &A, int64_t g, float *p) {
    p[0] = A.pos[g];
    p[1] = A.pos[A.plane + g];
    p[2] = A.pos[2 * A.plane + g];
}

__device__ __forceinline__ bool box_overlap(const float *la, const float *ha, const float *lb,
                                            const float *hb) {
    return (la[0] <= hb[0]) & (lb[0] <= ha[0]) & (la[1] <= hb[1]) & (lb[1] <= ha[1]) &
           (la[2] <= hb[2]) & (lb[2] <= ha[2]);
}

// warp-aggregated counter increment; every lane of the warp calls it (the
// callers have no early returns), so one atomic per warp suffices
__device__ __forceinline__ void count_hits(unsigned long long *ctr, uint32_t n) {
    const uint32_t v = __reduce_add_sync(0xffffffffu, n);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(ctr, (unsigned long long)v);
}

// Pass A: one thread per unique cloth edge, candidates from the grid.
__global__ void __launch_bounds__(256)
k_detect_cloth_edges(const CollideArgs A, const GridDesc g, const uint32_t *__restrict__ cbeg,
                     const uint32_t *__restrict__ cend, const uint32_t *__restrict__ ctri,
                     const float *__restrict__ corners, const float *__restrict__ normals,
                     const int32_t *__restrict__ edges, int64_t ne) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    uint32_t hits = 0;
    if (e < ne) {
        const int64_t ga = edges[2 * e], gb = edges[2 * e + 1];
        float st[3], en[3], lo[3], hi[3];
        load_pos(A, ga, st);
        load_pos(A, gb, en);
#pragma unroll
        for (int d = 0; d < 3; ++d) {  // kernels.py:55-59 segment_boxes
            lo[d] = fsub(fminf(st[d], en[d]), A.pad);
            hi[d] = fadd(fmaxf(st[d], en[d]), A.pad);
        }
        if (g.overlaps(lo, hi)) {
            int a[3], b[3];
            g.cell_range(lo, hi, a, b);
            for (int z = a[2]; z <= b[2]; ++z)
                for (int y = a[1]; y <= b[1]; ++y)
                    for (int x = a[0]; x <= b[0]; ++x) {
                        const uint32_t key = g.key(x, y, z);
                        const uint32_t c1 = cend[key];
                        for (uint32_t q = cbeg[key]; q < c1; ++q) {
                            const uint32_t t = ctri[q];
                            const float *c = corners + 9 * (int64_t)t;
                            float tlo[3], thi[3];
                            tri_box(c, tlo, thi);
                            if (!box_overlap(lo, hi, tlo, thi)) continue;
                            // dedup: min corner of the intersection lies in this cell
                            const float m[3] = {fmaxf(lo[0], tlo[0]), fmaxf(lo[1], tlo[1]),
                                                fmaxf(lo[2], tlo[2])};
                            if (g.cell_of(m[0], 0) != x || g.cell_of(m[1], 1) != y ||
                                g.cell_of(m[2], 2) != z)
                                continue;
                            float pt[3];
                            if (!seg_tri(st, en, c, c + 3, c + 6, A.eps, pt)) continue;
                            hits += owned_hit(A, ga < gb ? ga : gb);
                            const float *nrm = normals + 3 * (int64_t)t;
                            const float sa = dot3x(fsub(st[0], pt[0]), fsub(st[1], pt[1]),
                                                   fsub(st[2], pt[2]), nrm[0], nrm[1], nrm[2]);
                            const float sb = dot3x(fsub(en[0], pt[0]), fsub(en[1], pt[1]),
                                                   fsub(en[2], pt[2]), nrm[0], nrm[1], nrm[2]);
                            const float sign = np_max(sa, sb) >= 0.f ? 1.f : -1.f;
                            const float on[3] = {fmul(nrm[0], sign), fmul(nrm[1], sign),
                                                 fmul(nrm[2], sign)};
                            accumulate(A, ga, st, pt, on, t);
                            accumulate(A, gb, en, pt, on, t);
                        }
                    }
        }
    }
    count_hits(A.frame_hits, hits);
}

// Pass B: one thread per cloth triangle; candidates are obstacle triangles
// whose box meets the cloth box padded by 2*pad (a superset of the
// reference's padded-edge-box test, which is then applied exactly per edge).
__global__ void __launch_bounds__(256)
k_detect_obstacle_edges(const CollideArgs A, const GridDesc g, const uint32_t *__restrict__ cbeg,
                        const uint32_t *__restrict__ cend, const uint32_t *__restrict__ ctri,
                        const float *__restrict__ corners, const float *__restrict__ normals,
                        const int32_t *__restrict__ tris, int64_t nc) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    uint32_t hits = 0;
    if (c < nc) {
        const int64_t n0 = tris[3 * c], n1 = tris[3 * c + 1], n2 = tris[3 * c + 2];
        float v0[3], v1[3], v2[3];
        load_pos(A, n0, v0);
        load_pos(A, n1, v1);
        load_pos(A, n2, v2);
        float clo[3], chi[3], qlo[3], qhi[3];
        const float pad2 = 2.0f * A.pad;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            clo[d] = fminf(fminf(v0[d], v1[d]), v2[d]);
            chi[d] = fmaxf(fmaxf(v0[d], v1[d]), v2[d]);
            qlo[d] = clo[d] - pad2;
            qhi[d] = chi[d] + pad2;
        }
        if (g.overlaps(qlo, qhi)) {
            int a[3], b[3];
            g.cell_range(qlo, qhi, a, b);
            for (int z = a[2]; z <= b[2]; ++z)
                for (int y = a[1]; y <= b[1]; ++y)
                    for (int x = a[0]; x <= b[0]; ++x) {
                        const uint32_t key = g.key(x, y, z);
                        const uint32_t c1 = cend[key];
                        for (uint32_t q = cbeg[key]; q < c1; ++q) {
                            const uint32_t t = ctri[q];
                            const float *cr = corners + 9 * (int64_t)t;
                            float tlo[3], thi[3];
                            tri_box(cr, tlo, thi);
                            if (!box_overlap(qlo, qhi, tlo, thi)) continue;
                            const float m[3] = {fmaxf(qlo[0], tlo[0]), fmaxf(qlo[1], tlo[1]),
                                                fmaxf(qlo[2], tlo[2])};
                            if (g.cell_of(m[0], 0) != x || g.cell_of(m[1], 1) != y ||
                                g.cell_of(m[2], 2) != z)
                                continue;
                            const float *nrm = normals + 3 * (int64_t)t;
                            for (int slot = 0; slot < 3; ++slot) {
                                const float *st = cr + 3 * slot;
                                const float *en = cr + 3 * ((slot + 1) % 3);
                                float elo[3], ehi[3];
#pragma unroll
                                for (int d = 0; d < 3; ++d) {
                                    elo[d] = fsub(fminf(st[d], en[d]), A.pad);
                                    ehi[d] = fadd(fmaxf(st[d], en[d]), A.pad);
                                }
                                if (!box_overlap(elo, ehi, clo, chi)) continue;
                                float pt[3];
                                if (!seg_tri(st, en, v0, v1, v2, A.eps, pt)) continue;
                                hits += owned_hit(A, min(n0, min(n1, n2)));
                                const float t0 = dot3x(fsub(v0[0], pt[0]), fsub(v0[1], pt[1]),
                                                       fsub(v0[2], pt[2]), nrm[0], nrm[1], nrm[2]);
                                const float t1 = dot3x(fsub(v1[0], pt[0]), fsub(v1[1], pt[1]),
                                                       fsub(v1[2], pt[2]), nrm[0], nrm[1], nrm[2]);
                                const float t2 = dot3x(fsub(v2[0], pt[0]), fsub(v2[1], pt[1]),
                                                       fsub(v2[2], pt[2]), nrm[0], nrm[1], nrm[2]);
                                const float total = fadd(fadd(t0, t1), t2);
                                const float sign = total >= 0.f ? 1.f : -1.f;
                                const float on[3] = {fmul(nrm[0], sign), fmul(nrm[1], sign),
                                                     fmul(nrm[2], sign)};
                                accumulate(A, n0, v0, pt, on, t);
                                accumulate(A, n1, v1, pt, on, t);
                                accumulate(A, n2, v2, pt, on, t);
                            }
                        }
                    }
        }
    }
    count_hits(A.frame_hits, hits);
}

// Respond (kernels.py:293-311) over the touched list only: every node with a
// nonzero count is on the list exactly once.  Flip-and-halve the velocity,
// add the decoded (optionally averaged) offset, clear the accumulators.
__device__ __forceinline__ void respond_end(const CollideArgs &A, int end_of_frame);

__global__ void __launch_bounds__(256)
k_respond(const CollideArgs A, float *__restrict__ pos, const uint32_t *__restrict__ pinbits,
          const float *__restrict__ inv_mass, int average, int end_of_frame) {
    const uint32_t n = *A.touched_n;
    // blocks past the touched list have no item in the grid-stride loop and
    // leave at once: only the `busy` ones take part in the last-block
    // protocol below (block 0 always, so an empty frame is still closed).
    // C3 touches ~15K of 100K nodes: 60 of the 391 blocks do the fence +
    // counter atomic instead of all of them.
    const uint32_t need = (n + blockDim.x - 1) / blockDim.x;
    const uint32_t busy = need < gridDim.x ? (need ? need : 1u) : gridDim.x;
    if (blockIdx.x >= busy) return;
    uint32_t moved = 0;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
        const int64_t g = A.touched[q];
        // every load of the node issued at once (one dependent round trip
        // after the touched list instead of two)
        const int cnt = A.count[g];
        const bool pinned = inv_mass ? !(inv_mass[g] > 0.f) : ((pinbits[g >> 5] >> (g & 31)) & 1u);
        int32_t raw[3];
        float x[3], v[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            raw[d] = A.acc[d * A.plane + g];
            x[d] = pos[d * A.plane + g];
            v[d] = pos[(3 + d) * A.plane + g];
        }
        if (cnt > 0 && !pinned) {
            ++moved;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                float dv = decode_fixed(raw[d], A.scale_d);
                if (average) dv = fdiv(dv, (float)cnt);
                pos[(3 + d) * A.plane + g] = fmul(v[d], -0.5f);
                pos[d * A.plane + g] = fadd(x[d], dv);
            }
        }
        A.acc[g] = 0;
        A.acc[A.plane + g] = 0;
        A.acc[2 * A.plane + g] = 0;
        A.count[g] = 0;
    }
    count_hits(A.frame_responded, moved);
    // the last block to finish closes the frame (no separate launch)
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(A.blocks_done, 1u) == busy - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        *A.blocks_done = 0;
        respond_end(A, end_of_frame);
    }
}

// After the respond pass: clear the touched list; at the end of a frame also
// fold the frame's hits into the cumulative hitCounter and record
// (hits, responded) in the per-frame ring that StepResult reads lazily.
__device__ __forceinline__ void respond_end(const CollideArgs &A, int end_of_frame) {
    *A.touched_n = 0;
    if (end_of_frame) {
        const unsigned long long f = *A.frame_counter;
        const unsigned long long hits = atomicAdd(A.frame_hits, 0ull);
        const unsigned long long resp = atomicAdd(A.frame_responded, 0ull);
        *A.hit_counter += hits;
        A.ring[2 * (f % A.ring_size)] = hits;
        A.ring[2 * (f % A.ring_size) + 1] = resp;
        *A.frame_counter = f + 1;
    }
}

__global__ void k_respond_end(const CollideArgs A, int end_of_frame) { respond_end(A, end_of_frame); }

// Rebuild the touched list from the count buffer (after host writes).
__global__ void k_rebuild_touched(const CollideArgs A, int64_t n_rows, int64_t nx, int64_t pitch) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n_rows * nx) return;
    const int64_t g = (v / nx) * pitch + (v % nx);
    if (A.count[g] != 0) {
        const uint32_t slot = atomicAdd(A.touched_n, 1u);
        A.touched[slot] = (uint32_t)g;
    }
}

// ---------------------------------------------------------------------------
// Warp-per-query narrow phase ("one warp per cell-candidate batch").  A warp
// takes one query (cloth edge for pass A, cloth triangle for pass B); its
// lanes read up to 32 of the query's grid cells at a time, a warp-shuffle
// inclusive scan flattens the cells' candidate lists, and every lane takes
// candidates t = lane, lane+32, ... (owner cell found by a 5-step shuffle
// binary search).  Divergence between queries with few and many candidates
// -- the cost of the thread-per-query kernels above -- disappears; queries
// whose box misses the obstacle leave after one test.  Same box test, dedup
// rule, predicate and accumulation as the thread-per-query kernels.
// ---------------------------------------------------------------------------
template <int PASS>  // 0: cloth edges vs obstacle triangles, 1: obstacle edges vs cloth triangles
__global__ void __launch_bounds__(256)
k_detect_warp(const CollideArgs A, const GridDesc g, const uint32_t *__restrict__ cbeg,
              const uint32_t *__restrict__ cend, const uint32_t *__restrict__ ctri,
              const float *__restrict__ tbox, const float *__restrict__ corners,
              const float *__restrict__ normals, const int32_t *__restrict__ items, int64_t nq) {
    const int lane = threadIdx.x & 31;
    const int64_t q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    uint32_t hits = 0;
    if (q < nq) {  // warp-uniform
        float v[3][3];
        int64_t nid[3];
        const int nv = PASS == 0 ? 2 : 3;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (k < nv) {
                nid[k] = items[nv * q + k];
                load_pos(A, nid[k], v[k]);
            }
        }
        float lo[3], hi[3], clo[3], chi[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            if (PASS == 0) {  // kernels.py:55-59: padded segment box
                lo[d] = fsub(fminf(v[0][d], v[1][d]), A.pad);
                hi[d] = fadd(fmaxf(v[0][d], v[1][d]), A.pad);
            } else {          // cloth triangle box, queried padded by 2*pad
                clo[d] = fminf(fminf(v[0][d], v[1][d]), v[2][d]);
                chi[d] = fmaxf(fmaxf(v[0][d], v[1][d]), v[2][d]);
                lo[d] = clo[d] - 2.0f * A.pad;
                hi[d] = chi[d] + 2.0f * A.pad;
            }
        }
        if (g.overlaps(lo, hi)) {
            int a[3], b[3];
            g.cell_range(lo, hi, a, b);
            const int ex = b[0] - a[0] + 1, ey = b[1] - a[1] + 1, ez = b[2] - a[2] + 1;
            const int ncell = ex * ey * ez;
            for (int c0 = 0; c0 < ncell; c0 += 32) {
                const int c = c0 + lane;
                int cx = 0, cy = 0, cz = 0;
                uint32_t beg = 0, cnt = 0;
                if (c < ncell) {
                    cx = a[0] + c % ex;
                    cy = a[1] + (c / ex) % ey;
                    cz = a[2] + c / (ex * ey);
                    const uint32_t key = g.key(cx, cy, cz);
                    beg = cbeg[key];
                    cnt = cend[key] - beg;
                }
                const uint32_t incl = warp_incl_scan(cnt);
                const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
                for (uint32_t t0 = 0; t0 < total; t0 += 32) {
                    const uint32_t t = t0 + lane;
                    // owner lane: smallest L with incl[L] > t
                    int o = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const uint32_t probe = __shfl_sync(0xffffffffu, incl, o + step - 1);
                        if (probe <= t) o += step;
                    }
                    const uint32_t ob = __shfl_sync(0xffffffffu, beg, o);
                    const uint32_t oi = __shfl_sync(0xffffffffu, incl, o);
                    const uint32_t oc = __shfl_sync(0xffffffffu, cnt, o);
                    const int ox = __shfl_sync(0xffffffffu, cx, o);
                    const int oy = __shfl_sync(0xffffffffu, cy, o);
                    const int oz = __shfl_sync(0xffffffffu, cz, o);
                    if (t >= total) continue;
                    const uint32_t tri = ctri[ob + (t - (oi - oc))];
                    const float *tb = tbox + 6 * (int64_t)tri;
                    const float tlo[3] = {tb[0], tb[1], tb[2]}, thi[3] = {tb[3], tb[4], tb[5]};
                    if (!box_overlap(lo, hi, tlo, thi)) continue;
                    // dedup: the minimum corner of the intersection lies in this cell
                    if (g.cell_of(fmaxf(lo[0], tlo[0]), 0) != ox || g.cell_of(fmaxf(lo[1], tlo[1]), 1) != oy ||
                        g.cell_of(fmaxf(lo[2], tlo[2]), 2) != oz)
                        continue;
                    const float *cr = corners + 9 * (int64_t)tri;
                    const float *nrm = normals + 3 * (int64_t)tri;
                    if (PASS == 0) {
                        float pt[3];
                        if (!seg_tri(v[0], v[1], cr, cr + 3, cr + 6, A.eps, pt)) continue;
                        hits += owned_hit(A, nid[0] < nid[1] ? nid[0] : nid[1]);
                        const float sa = dot3x(fsub(v[0][0], pt[0]), fsub(v[0][1], pt[1]),
                                               fsub(v[0][2], pt[2]), nrm[0], nrm[1], nrm[2]);
                        const float sb = dot3x(fsub(v[1][0], pt[0]), fsub(v[1][1], pt[1]),
                                               fsub(v[1][2], pt[2]), nrm[0], nrm[1], nrm[2]);
                        const float sign = np_max(sa, sb) >= 0.f ? 1.f : -1.f;
                        const float on[3] = {fmul(nrm[0], sign), fmul(nrm[1], sign), fmul(nrm[2], sign)};
                        accumulate(A, nid[0], v[0], pt, on, tri);
                        accumulate(A, nid[1], v[1], pt, on, tri);
                    } else {
                        for (int slot = 0; slot < 3; ++slot) {
                            const float *st = cr + 3 * slot;
                            const float *en = cr + 3 * ((slot + 1) % 3);
                            float elo[3], ehi[3];
#pragma unroll
                            for (int d = 0; d < 3; ++d) {
                                elo[d] = fsub(fminf(st[d], en[d]), A.pad);
                                ehi[d] = fadd(fmaxf(st[d], en[d]), A.pad);
                            }
                            if (!box_overlap(elo, ehi, clo, chi)) continue;
                            float pt[3];
                            if (!seg_tri(st, en, v[0], v[1], v[2], A.eps, pt)) continue;
                            hits += owned_hit(A, min(nid[0], min(nid[1], nid[2])));
                            const float t0s = dot3x(fsub(v[0][0], pt[0]), fsub(v[0][1], pt[1]),
                                                    fsub(v[0][2], pt[2]), nrm[0], nrm[1], nrm[2]);
                            const float t1s = dot3x(fsub(v[1][0], pt[0]), fsub(v[1][1], pt[1]),
                                                    fsub(v[1][2], pt[2]), nrm[0], nrm[1], nrm[2]);
                            const float t2s = dot3x(fsub(v[2][0], pt[0]), fsub(v[2][1], pt[1]),
                                                    fsub(v[2][2], pt[2]), nrm[0], nrm[1], nrm[2]);
                            const float sign = fadd(fadd(t0s, t1s), t2s) >= 0.f ? 1.f : -1.f;
                            const float on[3] = {fmul(nrm[0], sign), fmul(nrm[1], sign), fmul(nrm[2], sign)};
                            accumulate(A, nid[0], v[0], pt, on, tri);
                            accumulate(A, nid[1], v[1], pt, on, tri);
                            accumulate(A, nid[2], v[2], pt, on, tri);
                        }
                    }
                }
            }
        }
    }
    count_hits(A.frame_hits, hits);
}

// ---------------------------------------------------------------------------
// Batched narrow phase (default): a warp takes 32 QUERIES, one per lane, and
// flattens all of their (query, grid cell) pairs and then all of those
// cells' candidate triangles across the 32 lanes -- "one warp per
// cell-candidate batch".  The warp-per-query kernel above leaves most lanes
// idle (a draped cloth edge meets ~5-20 candidates); here every lane of
// every inner iteration tests a real (query, candidate) pair, and the
// queries' geometry sits in shared memory where any lane can read it.  Same
// box test, dedup rule, predicate, accumulation and hit ownership as the
// other two mappings, so the hit set and the integer accumulators are
// identical.
// ---------------------------------------------------------------------------
#ifndef CS_DETECT_BATCH_WARPS
#define CS_DETECT_BATCH_WARPS 4
#endif
constexpr int BATCH_WARPS = CS_DETECT_BATCH_WARPS;  // warps per narrow-phase block
#ifndef CS_DETECT_WPSM
#define CS_DETECT_WPSM 80  // target warps per SM when choosing queries per warp
#endif
#ifndef CS_DETECT_STRIDED
#define CS_DETECT_STRIDED 1
#endif
#ifndef CS_DETECT_MINB
#define CS_DETECT_MINB 8  // <= 64 registers, 32 resident warps per SM (strided queries: C3 frame -3%)
#endif
struct QuerySlot {
    float v[3][3];
    float lo[3], hi[3];   // query box (PASS 0: padded segment box; PASS 1: tri box +- 2 pad)
    float clo[3], chi[3]; // PASS 1: unpadded cloth triangle box
    int64_t nid[3];
    int a[3], ex, ey;     // first cell and extents of the cell range
};

__device__ __forceinline__ int warp_owner(uint32_t incl, uint32_t t) {
    // smallest lane L with incl[L] > t (incl non-decreasing across lanes)
    int o = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1) {
        const uint32_t probe = __shfl_sync(0xffffffffu, incl, o + step - 1);
        if (probe <= t) o += step;
    }
    return o;
}

// One narrow-phase item: query slot `qs` of this warp against obstacle
// triangle `tri` (PASS 1: its edge `slot`).  Returns the hits it owns.
template <int PASS>
__device__ __forceinline__ uint32_t narrow_item(const CollideArgs &A, const QuerySlot &Q,
                                                uint32_t tri, int slot,
                                                const float *__restrict__ corners,
                                                const float *__restrict__ normals) {
    const float *cr = corners + 9 * (int64_t)tri;
    const float *nrm = normals + 3 * (int64_t)tri;
    float v[3][3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int d = 0; d < 3; ++d) v[k][d] = Q.v[k][d];
    float pt[3];
    if (PASS == 0) {
        if (!seg_tri(v[0], v[1], cr, cr + 3, cr + 6, A.eps, pt)) return 0;
        const float sa = dot3x(fsub(v[0][0], pt[0]), fsub(v[0][1], pt[1]), fsub(v[0][2], pt[2]),
                               nrm[0], nrm[1], nrm[2]);
        const float sb = dot3x(fsub(v[1][0], pt[0]), fsub(v[1][1], pt[1]), fsub(v[1][2], pt[2]),
                               nrm[0], nrm[1], nrm[2]);
        const float sign = np_max(sa, sb) >= 0.f ? 1.f : -1.f;
        const float on[3] = {fmul(nrm[0], sign), fmul(nrm[1], sign), fmul(nrm[2], sign)};
        accumulate(A, Q.nid[0], v[0], pt, on, tri);
        accumulate(A, Q.nid[1], v[1], pt, on, tri);
        return owned_hit(A, Q.nid[0] < Q.nid[1] ? Q.nid[0] : Q.nid[1]);
    } else {
        const float *st = cr + 3 * slot;
        const float *en = cr + 3 * (slot == 2 ? 0 : slot + 1);
        if (!seg_tri(st, en, v[0], v[1], v[2], A.eps, pt)) return 0;
        const float t0s = dot3x(fsub(v[0][0], pt[0]), fsub(v[0][1], pt[1]), fsub(v[0][2], pt[2]),
                                nrm[0], nrm[1], nrm[2]);
        const float t1s = dot3x(fsub(v[1][0], pt[0]), fsub(v[1][1], pt[1]), fsub(v[1][2], pt[2]),
                                nrm[0], nrm[1], nrm[2]);
        const float t2s = dot3x(fsub(v[2][0], pt[0]), fsub(v[2][1], pt[1]), fsub(v[2][2], pt[2]),
                                nrm[0], nrm[1], nrm[2]);
        const float sign = fadd(fadd(t0s, t1s), t2s) >= 0.f ? 1.f : -1.f;
        const float on[3] = {fmul(nrm[0], sign), fmul(nrm[1], sign), fmul(nrm[2], sign)};
        accumulate(A, Q.nid[0], v[0], pt, on, tri);
        accumulate(A, Q.nid[1], v[1], pt, on, tri);
        accumulate(A, Q.nid[2], v[2], pt, on, tri);
        return owned_hit(A, min(Q.nid[0], min(Q.nid[1], Q.nid[2])));
    }
}

constexpr int QCAP = 128;  // per-warp item queue: < 32 left + 32 lanes x 3 slots

struct BatchShared {
    QuerySlot slots[BATCH_WARPS][32];
    // items that survived the box / dedup (/ edge box) filters wait here until
    // a full warp's worth can run the predicate with every lane active
    uint32_t qtri[BATCH_WARPS][QCAP];
    uint8_t qmeta[BATCH_WARPS][QCAP];  // query slot << 2 | edge slot
};

template <int PASS, bool PACKED>
__device__ __forceinline__ void detect_batch(BatchShared &S, int64_t blk, const CollideArgs &A,
                                             const GridDesc &g, const uint2 *__restrict__ cbe,
                                             const float4 *__restrict__ rbox,
                                             const float *__restrict__ corners,
                                             const float *__restrict__ normals,
                                             const int32_t *__restrict__ items, int64_t nq, int qb) {
    auto &slots = S.slots;
    auto &qtri = S.qtri;
    auto &qmeta = S.qmeta;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    // qb queries per warp (lanes >= qb hold none): 32 when queries are
    // plentiful, fewer so that small clouds still spread over every SM
#if CS_DETECT_STRIDED
    // query = lane * warps + warp: a warp's queries sit nw apart in index
    // (and so in space), so the warps drawn from a dense contact region no
    // longer carry all of its candidates (the frame's tail)
    const int64_t nw = (nq + qb - 1) / qb;
    const int64_t wi = blk * BATCH_WARPS + w;
    const int64_t q = wi < nw ? (int64_t)lane * nw + wi : nq;  // padding warps: none
#else
    const int64_t q = (blk * BATCH_WARPS + w) * qb + lane;
#endif
    QuerySlot &my = slots[w][lane];
    const int nv = PASS == 0 ? 2 : 3;
    uint32_t ncell = 0;
    if (lane < qb && q < nq) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (k < nv) {
                my.nid[k] = items[nv * q + k];
                load_pos(A, my.nid[k], my.v[k]);
            }
        }
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            if (PASS == 0) {  // kernels.py:55-59: padded segment box
                my.lo[d] = fsub(fminf(my.v[0][d], my.v[1][d]), A.pad);
                my.hi[d] = fadd(fmaxf(my.v[0][d], my.v[1][d]), A.pad);
            } else {          // cloth triangle box, queried padded by 2*pad
                my.clo[d] = fminf(fminf(my.v[0][d], my.v[1][d]), my.v[2][d]);
                my.chi[d] = fmaxf(fmaxf(my.v[0][d], my.v[1][d]), my.v[2][d]);
                my.lo[d] = my.clo[d] - 2.0f * A.pad;
                my.hi[d] = my.chi[d] + 2.0f * A.pad;
            }
        }
        if (g.overlaps(my.lo, my.hi)) {
            int a[3], b[3];
            g.cell_range(my.lo, my.hi, a, b);
            my.a[0] = a[0];
            my.a[1] = a[1];
            my.a[2] = a[2];
            my.ex = b[0] - a[0] + 1;
            my.ey = b[1] - a[1] + 1;
            ncell = (uint32_t)(my.ex * my.ey * (b[2] - a[2] + 1));
        }
    }
    __syncwarp();
    uint32_t hits = 0;
    int qn = 0;  // queued items (warp-uniform)
    auto drain = [&](int keep) {  // run the predicate on full warps of queued items
        while (qn > keep) {
            // a FULL warp of items while more than `keep` wait (the excess
            // alone would run the predicate on a few lanes: ncu saw 5-17
            // active lanes per predicate instruction)
            const int take = qn < 32 ? qn : 32;
            __syncwarp();
            if (lane < take) {
                const int k = qn - take + lane;
                const uint8_t meta = qmeta[w][k];
                hits += narrow_item<PASS>(A, slots[w][meta >> 2], qtri[w][k], meta & 3, corners,
                                          normals);
            }
            qn -= take;
            __syncwarp();
        }
    };
    auto push = [&](bool want, uint32_t tri, int qs, int slot) {
        const uint32_t m = __ballot_sync(0xffffffffu, want);
        if (want) {
            const int k = qn + __popc(m & lt_mask);
            qtri[w][k] = tri;
            qmeta[w][k] = (uint8_t)((qs << 2) | slot);
        }
        qn += __popc(m);
    };
    const uint32_t cincl = warp_incl_scan(ncell);
    const uint32_t ctotal = __shfl_sync(0xffffffffu, cincl, 31);
    for (uint32_t c0 = 0; c0 < ctotal; c0 += 32) {
        // this lane's (query, cell) pair; what a candidate lane needs of its
        // owner cell goes out in three shuffles: `rb` (the cell's first
        // reference minus its first flattened index: ref = rb + t), the cell
        // coordinates packed 10:10:10 (every axis <= 1024 cells: PACKED) or
        // its key, and the query slot
        const uint32_t c = c0 + lane;
        int oq = 0;
        uint32_t cell = 0, beg = 0, cnt = 0;
        {
            const int o = warp_owner(cincl, c);
            const uint32_t oincl = __shfl_sync(0xffffffffu, cincl, o);
            const uint32_t on = __shfl_sync(0xffffffffu, ncell, o);
            if (c < ctotal) {
                const QuerySlot &Q = slots[w][o];
                const int local = (int)(c - (oincl - on));
                const int cx = Q.a[0] + local % Q.ex;
                const int cy = Q.a[1] + (local / Q.ex) % Q.ey;
                const int cz = Q.a[2] + local / (Q.ex * Q.ey);
                const uint32_t key = g.key(cx, cy, cz);
                const uint2 r = cbe[key];
                beg = r.x;
                cnt = r.y - r.x;
                oq = o;
                cell = PACKED ? (uint32_t)cx | ((uint32_t)cy << 10) | ((uint32_t)cz << 20) : key;
            }
        }
        const uint32_t incl = warp_incl_scan(cnt);
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t rbase = beg - (incl - cnt);
        for (uint32_t t0 = 0; t0 < total; t0 += 32) {
            const uint32_t t = t0 + lane;
            const int o = warp_owner(incl, t);
            const uint32_t orb = __shfl_sync(0xffffffffu, rbase, o);
            const uint32_t ocell = __shfl_sync(0xffffffffu, cell, o);
            const int qq = __shfl_sync(0xffffffffu, oq, o);
            bool ok = t < total;
            uint32_t tri = 0;
            if (ok) {
                const QuerySlot &Q = slots[w][qq];
                const uint32_t ref = orb + t;
                const float4 b0 = rbox[2 * (int64_t)ref], b1 = rbox[2 * (int64_t)ref + 1];
                tri = __float_as_uint(b0.w);
                const float tlo[3] = {b0.x, b0.y, b0.z}, thi[3] = {b1.x, b1.y, b1.z};
                // box test, then dedup: the minimum corner of the intersection
                // lies in this cell
                if (PACKED) {
                    const uint32_t tc = __float_as_uint(b1.w);
                    ok = box_overlap(Q.lo, Q.hi, tlo, thi) &&
                         (uint32_t)max(Q.a[0], (int)(tc & 1023u)) == (ocell & 1023u) &&
                         (uint32_t)max(Q.a[1], (int)((tc >> 10) & 1023u)) == ((ocell >> 10) & 1023u) &&
                         (uint32_t)max(Q.a[2], (int)(tc >> 20)) == (ocell >> 20);
                } else {
                    const int ox = (int)(ocell % (uint32_t)g.dims[0]);
                    const int oy = (int)((ocell / (uint32_t)g.dims[0]) % (uint32_t)g.dims[1]);
                    const int oz = (int)(ocell / ((uint32_t)g.dims[0] * (uint32_t)g.dims[1]));
                    ok = box_overlap(Q.lo, Q.hi, tlo, thi) &&
                         g.cell_of(fmaxf(Q.lo[0], tlo[0]), 0) == ox &&
                         g.cell_of(fmaxf(Q.lo[1], tlo[1]), 1) == oy &&
                         g.cell_of(fmaxf(Q.lo[2], tlo[2]), 2) == oz;
                }
            }
            if (PASS == 0) {
                push(ok, tri, qq, 0);
            } else {
                const float *cr = corners + 9 * (int64_t)tri;
#pragma unroll
                for (int slot = 0; slot < 3; ++slot) {  // obstacle edge 3t+slot
                    bool e_ok = ok;
                    if (e_ok) {
                        const QuerySlot &Q = slots[w][qq];
                        const float *st = cr + 3 * slot;
                        const float *en = cr + 3 * (slot == 2 ? 0 : slot + 1);
                        float elo[3], ehi[3];
#pragma unroll
                        for (int d = 0; d < 3; ++d) {
                            elo[d] = fsub(fminf(st[d], en[d]), A.pad);
                            ehi[d] = fadd(fmaxf(st[d], en[d]), A.pad);
                        }
                        e_ok = box_overlap(elo, ehi, Q.clo, Q.chi);
                    }
                    push(e_ok, tri, qq, slot);
                }
            }
            drain(31);
        }
    }
    drain(0);
    count_hits(A.frame_hits, hits);
}

// ---------------------------------------------------------------------------
// Fused narrow phase (default, narrow="tri"): ONE candidate enumeration per
// cloth triangle serves both reference passes.  The batched mapping above
// enumerates grid candidates twice -- once per cloth edge (pass A) and once
// per cloth triangle (pass B) -- although a cloth edge's padded box lies
// inside its triangle's box padded by 2 pad.  Here every unique cloth edge
// is owned by the lowest-index triangle containing it (tri_own: 3 bits per
// triangle, built with the engine), and each surviving (cloth triangle,
// obstacle triangle) candidate is expanded into
//   * pass A items: each owned edge, oriented (lower node, higher node) as in
//     unique_edges, whose padded box meets the obstacle triangle's box
//     (kernels.py:55-78) -- the reference's own prefilter, exactly;
//   * pass B items: each obstacle edge 3t+slot whose padded box meets the
//     cloth triangle's box.
// The candidate superset is the same as pass B's (the triangle query box),
// so every pair the reference's prefilter keeps is tested exactly once; the
// predicate, offsets, accumulation and hit ownership are those of the
// other mappings (hits and integer accumulators identical).
// ---------------------------------------------------------------------------
struct TriSlot {
    float v[3][3];
    float lo[3], hi[3];    // query box: cloth triangle box +- 2 pad
    float clo[3], chi[3];  // unpadded cloth triangle box (pass B's edge-box test)
    int64_t nid[3];
    int a[3], ex, ey;      // first cell and extents of the cell range
    uint32_t own;          // owned-edge mask (edge k = nodes k, k+1 mod 3)
};

constexpr int QCAP_T = 224;  // < 32 left + 32 lanes x 6 items

struct TriShared {
    TriSlot slots[BATCH_WARPS][32];
    // queued item: obstacle triangle | query slot << 27 | kind << 24 (kind
    // 0-2: the query's edge k, 3-5: obstacle edge slot) -- launch_detect
    // keeps obstacles under 2^24 triangles on this path
    uint32_t qitem[BATCH_WARPS][QCAP_T];
};

// one item: pass A (kind 0-2, the query's edge `kind`) or pass B (kind 3-5,
// obstacle edge slot kind-3) of query Q against obstacle triangle `tri`
__device__ __forceinline__ uint32_t tri_item(const CollideArgs &A, const TriSlot &Q, uint32_t tri,
                                             int kind, const float *__restrict__ corners,
                                             const float *__restrict__ normals) {
    const float *cr = corners + 9 * (int64_t)tri;
    const float *nrm = normals + 3 * (int64_t)tri;
    float pt[3];
    if (kind < 3) {
        const int k1 = kind == 2 ? 0 : kind + 1;
        const bool lo_first = Q.nid[kind] < Q.nid[k1];
        const int ia = lo_first ? kind : k1, ib = lo_first ? k1 : kind;
        float st[3], en[3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            st[d] = Q.v[ia][d];
            en[d] = Q.v[ib][d];
        }
        if (!seg_tri(st, en, cr, cr + 3, cr + 6, A.eps, pt)) return 0;
        const float sa = dot3x(fsub(st[0], pt[0]), fsub(st[1], pt[1]), fsub(st[2], pt[2]), nrm[0],
                               nrm[1], nrm[2]);
        const float sb = dot3x(fsub(en[0], pt[0]), fsub(en[1], pt[1]), fsub(en[2], pt[2]), nrm[0],
                               nrm[1], nrm[2]);
        const float sign = np_max(sa, sb) >= 0.f ? 1.f : -1.f;
        const float on[3] = {fmul(nrm[0], sign), fmul(nrm[1], sign), fmul(nrm[2], sign)};
        accumulate(A, Q.nid[ia], st, pt, on, tri);
        accumulate(A, Q.nid[ib], en, pt, on, tri);
        return owned_hit(A, Q.nid[ia]);
    }
    const int slot = kind - 3;
    const float *st = cr + 3 * slot;
    const float *en = cr + 3 * (slot == 2 ? 0 : slot + 1);
    float v[3][3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int d = 0; d < 3; ++d) v[k][d] = Q.v[k][d];
    if (!seg_tri(st, en, v[0], v[1], v[2], A.eps, pt)) return 0;
    const float t0s = dot3x(fsub(v[0][0], pt[0]), fsub(v[0][1], pt[1]), fsub(v[0][2], pt[2]), nrm[0],
                            nrm[1], nrm[2]);
    const float t1s = dot3x(fsub(v[1][0], pt[0]), fsub(v[1][1], pt[1]), fsub(v[1][2], pt[2]), nrm[0],
                            nrm[1], nrm[2]);
    const float t2s = dot3x(fsub(v[2][0], pt[0]), fsub(v[2][1], pt[1]), fsub(v[2][2], pt[2]), nrm[0],
                            nrm[1], nrm[2]);
    const float sign = fadd(fadd(t0s, t1s), t2s) >= 0.f ? 1.f : -1.f;
    const float on[3] = {fmul(nrm[0], sign), fmul(nrm[1], sign), fmul(nrm[2], sign)};
    accumulate(A, Q.nid[0], v[0], pt, on, tri);
    accumulate(A, Q.nid[1], v[1], pt, on, tri);
    accumulate(A, Q.nid[2], v[2], pt, on, tri);
    return owned_hit(A, min(Q.nid[0], min(Q.nid[1], Q.nid[2])));
}

template <bool PACKED>
__device__ __forceinline__ void detect_tri(TriShared &S, int64_t blk, const CollideArgs &A,
                                           const GridDesc &g, const uint2 *__restrict__ cbe,
                                           const float4 *__restrict__ rbox,
                                           const float *__restrict__ corners,
                                           const float *__restrict__ normals,
                                           const int32_t *__restrict__ tris,
                                           const uint8_t *__restrict__ tri_own,
                                           const float4 *__restrict__ ebox, int64_t nq, int qb) {
    auto &slots = S.slots;
    auto &qitem = S.qitem;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // strided queries (as detect_batch): query = lane * warps + warp
    const int64_t nw = (nq + qb - 1) / qb;
    const int64_t wi = blk * BATCH_WARPS + w;
    const int64_t q = wi < nw ? (int64_t)lane * nw + wi : nq;
    TriSlot &my = slots[w][lane];
    uint32_t ncell = 0;
    if (lane < qb && q < nq) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            my.nid[k] = tris[3 * q + k];
            load_pos(A, my.nid[k], my.v[k]);
        }
        my.own = tri_own[q];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            my.clo[d] = fminf(fminf(my.v[0][d], my.v[1][d]), my.v[2][d]);
            my.chi[d] = fmaxf(fmaxf(my.v[0][d], my.v[1][d]), my.v[2][d]);
            my.lo[d] = my.clo[d] - 2.0f * A.pad;
            my.hi[d] = my.chi[d] + 2.0f * A.pad;
        }
        if (g.overlaps(my.lo, my.hi)) {
            int a[3], b[3];
            g.cell_range(my.lo, my.hi, a, b);
            my.a[0] = a[0];
            my.a[1] = a[1];
            my.a[2] = a[2];
            my.ex = b[0] - a[0] + 1;
            my.ey = b[1] - a[1] + 1;
            ncell = (uint32_t)(my.ex * my.ey * (b[2] - a[2] + 1));
        }
    }
    __syncwarp();
    uint32_t hits = 0;
    int qn = 0;  // queued items (warp-uniform)
    auto drain = [&](int keep) {  // run the predicate on full warps of queued items
        while (qn > keep) {
            // a FULL warp of items while more than `keep` wait (the excess
            // alone would run the predicate on a few lanes: ncu saw 5-17
            // active lanes per predicate instruction)
            const int take = qn < 32 ? qn : 32;
            __syncwarp();
            if (lane < take) {
                const uint32_t it = qitem[w][qn - take + lane];
                hits += tri_item(A, slots[w][it >> 27], it & 0xffffffu, (int)((it >> 24) & 7u),
                                 corners, normals);
            }
            qn -= take;
            __syncwarp();
        }
    };
    // queue every item of this lane's candidate at once: bit k of `items`
    // = kind k (0-2 pass A edges, 3-5 pass B edge slots); one warp scan
    // places them
    auto push6 = [&](uint32_t items, uint32_t tri, int qs) {
        const uint32_t n = __popc(items);
        const uint32_t incl = warp_incl_scan(n);
        int k = qn + (int)(incl - n);
        const uint32_t head = tri | ((uint32_t)qs << 27);
        while (items) {
            const int kind = __ffs(items) - 1;
            items &= items - 1u;
            qitem[w][k++] = head | ((uint32_t)kind << 24);
        }
        qn += (int)__shfl_sync(0xffffffffu, incl, 31);
    };
    const uint32_t cincl = warp_incl_scan(ncell);
    const uint32_t ctotal = __shfl_sync(0xffffffffu, cincl, 31);
    for (uint32_t c0 = 0; c0 < ctotal; c0 += 32) {
        const uint32_t c = c0 + lane;
        int oq = 0;
        uint32_t cell = 0, beg = 0, cnt = 0;
        {
            const int o = warp_owner(cincl, c);
            const uint32_t oincl = __shfl_sync(0xffffffffu, cincl, o);
            const uint32_t on = __shfl_sync(0xffffffffu, ncell, o);
            if (c < ctotal) {
                const TriSlot &Q = slots[w][o];
                const int local = (int)(c - (oincl - on));
                const int cx = Q.a[0] + local % Q.ex;
                const int cy = Q.a[1] + (local / Q.ex) % Q.ey;
                const int cz = Q.a[2] + local / (Q.ex * Q.ey);
                const uint32_t key = g.key(cx, cy, cz);
                const uint2 r = cbe[key];
                beg = r.x;
                cnt = r.y - r.x;
                oq = o;
                cell = PACKED ? (uint32_t)cx | ((uint32_t)cy << 10) | ((uint32_t)cz << 20) : key;
            }
        }
        const uint32_t incl = warp_incl_scan(cnt);
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t rbase = beg - (incl - cnt);
        for (uint32_t t0 = 0; t0 < total; t0 += 32) {
            const uint32_t t = t0 + lane;
            const int o = warp_owner(incl, t);
            const uint32_t orb = __shfl_sync(0xffffffffu, rbase, o);
            const uint32_t ocell = __shfl_sync(0xffffffffu, cell, o);
            const int qq = __shfl_sync(0xffffffffu, oq, o);
            bool ok = t < total;
            uint32_t tri = 0;
            float tlo[3] = {0.f, 0.f, 0.f}, thi[3] = {0.f, 0.f, 0.f};
            if (ok) {
                const TriSlot &Q = slots[w][qq];
                const uint32_t ref = orb + t;
                const float4 b0 = rbox[2 * (int64_t)ref], b1 = rbox[2 * (int64_t)ref + 1];
                tri = __float_as_uint(b0.w);
                tlo[0] = b0.x; tlo[1] = b0.y; tlo[2] = b0.z;
                thi[0] = b1.x; thi[1] = b1.y; thi[2] = b1.z;
                if (PACKED) {
                    const uint32_t tc = __float_as_uint(b1.w);
                    ok = box_overlap(Q.lo, Q.hi, tlo, thi) &&
                         (uint32_t)max(Q.a[0], (int)(tc & 1023u)) == (ocell & 1023u) &&
                         (uint32_t)max(Q.a[1], (int)((tc >> 10) & 1023u)) == ((ocell >> 10) & 1023u) &&
                         (uint32_t)max(Q.a[2], (int)(tc >> 20)) == (ocell >> 20);
                } else {
                    const int ox = (int)(ocell % (uint32_t)g.dims[0]);
                    const int oy = (int)((ocell / (uint32_t)g.dims[0]) % (uint32_t)g.dims[1]);
                    const int oz = (int)(ocell / ((uint32_t)g.dims[0] * (uint32_t)g.dims[1]));
                    ok = box_overlap(Q.lo, Q.hi, tlo, thi) &&
                         g.cell_of(fmaxf(Q.lo[0], tlo[0]), 0) == ox &&
                         g.cell_of(fmaxf(Q.lo[1], tlo[1]), 1) == oy &&
                         g.cell_of(fmaxf(Q.lo[2], tlo[2]), 2) == oz;
                }
            }
            uint32_t items = 0;
            if (ok) {
                const TriSlot &Q = slots[w][qq];
                // pass A: the query's owned edges whose padded box meets the
                // obstacle triangle's box (kernels.py:55-78)
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    if ((Q.own >> k) & 1u) {
                        const int k1 = k == 2 ? 0 : k + 1;
                        float elo[3], ehi[3];
#pragma unroll
                        for (int d = 0; d < 3; ++d) {
                            elo[d] = fsub(fminf(Q.v[k][d], Q.v[k1][d]), A.pad);
                            ehi[d] = fadd(fmaxf(Q.v[k][d], Q.v[k1][d]), A.pad);
                        }
                        if (box_overlap(elo, ehi, tlo, thi)) items |= 1u << k;
                    }
                }
                // pass B: obstacle edges 3t+slot whose padded box (precomputed,
                // the same f32 operations) meets the cloth triangle's box
                const float4 *eb = ebox + 5 * (int64_t)tri;
                const float4 e0 = eb[0], e1 = eb[1], e2 = eb[2], e3 = eb[3], e4 = eb[4];
                const float b0lo[3] = {e0.x, e0.y, e0.z}, b0hi[3] = {e0.w, e1.x, e1.y};
                const float b1lo[3] = {e1.z, e1.w, e2.x}, b1hi[3] = {e2.y, e2.z, e2.w};
                const float b2lo[3] = {e3.x, e3.y, e3.z}, b2hi[3] = {e3.w, e4.x, e4.y};
                if (box_overlap(b0lo, b0hi, Q.clo, Q.chi)) items |= 8u;
                if (box_overlap(b1lo, b1hi, Q.clo, Q.chi)) items |= 16u;
                if (box_overlap(b2lo, b2hi, Q.clo, Q.chi)) items |= 32u;
            }
            push6(items, tri, qq);
            drain(31);
        }
    }
    drain(0);
    count_hits(A.frame_hits, hits);
}

__global__ void __launch_bounds__(32 * BATCH_WARPS, CS_DETECT_MINB)
k_detect_tri(const CollideArgs A, const GridDesc g, const uint2 *__restrict__ cbe,
             const float4 *__restrict__ rbox, const float *__restrict__ corners,
             const float *__restrict__ normals, const int32_t *__restrict__ tris,
             const uint8_t *__restrict__ tri_own, const float4 *__restrict__ ebox, int64_t nc,
             int qb, int packed) {
    __shared__ TriShared S;
    if (packed)
        detect_tri<true>(S, blockIdx.x, A, g, cbe, rbox, corners, normals, tris, tri_own, ebox, nc,
                         qb);
    else
        detect_tri<false>(S, blockIdx.x, A, g, cbe, rbox, corners, normals, tris, tri_own, ebox,
                          nc, qb);
}

// Both passes in ONE launch: blocks [0, blocks_a) take cloth edges (pass A),
// the rest cloth triangles (pass B) -- no dependency between them, one
// launch latency instead of two.
__global__ void __launch_bounds__(32 * BATCH_WARPS, CS_DETECT_MINB)
k_detect_batch(const CollideArgs A, const GridDesc g, const uint2 *__restrict__ cbe,
               const float4 *__restrict__ rbox, const float *__restrict__ corners,
               const float *__restrict__ normals, const int32_t *__restrict__ edges, int64_t ne,
               int qb_a, int64_t blocks_a, const int32_t *__restrict__ tris, int64_t nc, int qb_b,
               int packed) {
    __shared__ BatchShared S;
    if ((int64_t)blockIdx.x < blocks_a) {
        if (packed)
            detect_batch<0, true>(S, blockIdx.x, A, g, cbe, rbox, corners, normals, edges, ne, qb_a);
        else
            detect_batch<0, false>(S, blockIdx.x, A, g, cbe, rbox, corners, normals, edges, ne, qb_a);
    } else {
        if (packed)
            detect_batch<1, true>(S, blockIdx.x - blocks_a, A, g, cbe, rbox, corners, normals, tris,
                                  nc, qb_b);
        else
            detect_batch<1, false>(S, blockIdx.x - blocks_a, A, g, cbe, rbox, corners, normals, tris,
                                   nc, qb_b);
    }
}

__global__ void k_tri_boxes(int64_t nt, const float *__restrict__ corners, float *__restrict__ box) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nt) return;
    float lo[3], hi[3];
    tri_box(corners + 9 * t, lo, hi);
    for (int d = 0; d < 3; ++d) {
        box[6 * t + d] = lo[d];
        box[6 * t + 3 + d] = hi[d];
    }
}

void launch_tri_boxes(int64_t nt, const float *corners, float *box, cudaStream_t st) {
    if (nt > 0) k_tri_boxes<<<nblk(nt, 256), 256, 0, st>>>(nt, corners, box);
}

void launch_detect(const CollideArgs &A, const BroadPhase &bp, const float *corners,
                   const float *normals, const int32_t *edges, int64_t ne, const int32_t *tris,
                   int64_t nc, cudaStream_t st) {
    if (bp.warp_per_query == 3 && bp.tri_own && bp.num_tris < (1 << 24)) {
        int qb = 32;
        while (qb > 1 && nc / qb < (int64_t)148 * CS_DETECT_WPSM) qb >>= 1;
        const int64_t blocks = nc > 0 ? nblk((nc + qb - 1) / qb, BATCH_WARPS) : 0;
        if (blocks > 0)
            k_detect_tri<<<(unsigned)blocks, 32 * BATCH_WARPS, 0, st>>>(
                A, bp.grid, bp.cell_be, bp.ref_box, corners, normals, tris, bp.tri_own, bp.edge_box,
                nc, qb, bp.packed_cells ? 1 : 0);
        return;
    }
    if (bp.warp_per_query >= 2) {
        // queries per warp: the largest power of two <= 32 that still leaves
        // >= CS_DETECT_WPSM warps per SM (148 SMs).  With contiguous batches
        // the frame's time was the tail of the warps whose queries sat in the
        // densest contact region, and smaller batches in more warps shortened
        // it (C3, 8 queries per warp at 160: 153 -> 138 us).  Strided batches
        // (CS_DETECT_STRIDED) spread that region over every warp, so fewer,
        // fuller warps win: C3 16 queries per warp at 80, frame 139 -> 116 us
        // (tools/ab_c3.sh); one query per warp for small clouds (C4)
        auto qb_for = [](int64_t nq) {
            int qb = 32;
            while (qb > 1 && nq / qb < (int64_t)148 * CS_DETECT_WPSM) qb >>= 1;
            return qb;
        };
        const int qa = qb_for(ne), qc = qb_for(nc);
        const int64_t ba = ne > 0 ? nblk((ne + qa - 1) / qa, BATCH_WARPS) : 0;
        const int64_t bc = nc > 0 ? nblk((nc + qc - 1) / qc, BATCH_WARPS) : 0;
        if (ba + bc > 0)
            k_detect_batch<<<(unsigned)(ba + bc), 32 * BATCH_WARPS, 0, st>>>(
                A, bp.grid, bp.cell_be, bp.ref_box, corners, normals, edges, ne, qa, ba, tris, nc,
                qc, bp.packed_cells ? 1 : 0);
        return;
    }
    if (bp.warp_per_query) {
        if (ne > 0)
            k_detect_warp<0><<<nblk(ne * 32, 256), 256, 0, st>>>(A, bp.grid, bp.cell_begin, bp.cell_end,
                                                                 bp.cell_tris, bp.tri_box, corners,
                                                                 normals, edges, ne);
        if (nc > 0)
            k_detect_warp<1><<<nblk(nc * 32, 256), 256, 0, st>>>(A, bp.grid, bp.cell_begin, bp.cell_end,
                                                                 bp.cell_tris, bp.tri_box, corners,
                                                                 normals, tris, nc);
        return;
    }
    if (ne > 0)
        k_detect_cloth_edges<<<nblk(ne, 256), 256, 0, st>>>(A, bp.grid, bp.cell_begin, bp.cell_end,
                                                             bp.cell_tris, corners, normals, edges, ne);
    if (nc > 0)
        k_detect_obstacle_edges<<<nblk(nc, 256), 256, 0, st>>>(A, bp.grid, bp.cell_begin,
                                                                bp.cell_end, bp.cell_tris, corners,
                                                                normals, tris, nc);
}

void launch_respond(const CollideArgs &A, float *state, const uint32_t *pinbits,
                    const float *inv_mass, int average, int64_t max_nodes, int num_sms,
                    bool end_of_frame, cudaStream_t st) {
    int64_t blocks = (max_nodes + 255) / 256;
    const int64_t cap = (int64_t)num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    k_respond<<<(unsigned)blocks, 256, 0, st>>>(A, state, pinbits, inv_mass, average,
                                                 end_of_frame ? 1 : 0);
}

void launch_respond_end(const CollideArgs &A, bool end_of_frame, cudaStream_t st) {
    k_respond_end<<<1, 1, 0, st>>>(A, end_of_frame ? 1 : 0);
}

void launch_rebuild_touched(const CollideArgs &A, int64_t rows, int64_t nx, int64_t pitch,
                            cudaStream_t st) {
    cudaMemsetAsync(A.touched_n, 0, sizeof(uint32_t), st);
    const int64_t n = rows * nx;
    if (n > 0) k_rebuild_touched<<<nblk(n, 256), 256, 0, st>>>(A, rows, nx, pitch);
}

}  // namespace cs
