// cs_snapshot.cu -- the reference's orthographic depth-shaded PNG snapshot
// (clothsim/io.py:187-287, snapshot_png / _rasterize) rendered on the device,
// so a frame of a large cloth is pictured without reading its positions back.
//
// The reference paints triangles one by one into a float64 z-buffer; a pixel
// takes the NEAREST depth (strict greater-than: on ties the earlier triangle
// keeps it; cloth triangles precede obstacle triangles).  Here every
// triangle is one thread and the z-buffer is resolved in two passes over the
// same arithmetic:
//   1. k_snap_depth : atomicMax of the order-preserving u64 key of zpix;
//   2. k_snap_owner : among the triangles whose zpix equals the pixel's
//                     maximum, atomicMin of the triangle index -- the
//                     earliest one, which is the reference's owner;
//   3. k_snap_zrange: min / max depth over covered pixels;
//   4. k_snap_shade : 0.25 + 0.75 (z - zmin) / zspan times the material tint,
//                     clipped, x255, round-half-even (numpy .round()).
// All float64 arithmetic uses the _rn intrinsics in numpy's operation order
// (no FMA contraction), so the pixels are bit-identical to the reference's.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

namespace cs {

namespace {

// order-preserving map f64 -> u64 (larger double <=> larger key); key 0 is
// below every finite value and stands for the reference's -inf background
__device__ __forceinline__ uint64_t okey(double d) {
    d = __dadd_rn(d, 0.0);  // -0.0 -> +0.0: numpy's > treats them as equal
    const uint64_t b = (uint64_t)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double unkey(uint64_t k) {
    const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double d;
    memcpy(&d, &b, sizeof d);
    return d;
}

struct View {
    double lo_u, lo_v, scale;
    int au, av, ad;
    int width, height;
};

struct Tri2 {
    double x[3], y[3], z[3];
};

__device__ __forceinline__ Tri2 project(const double *verts, const int32_t *tri, const View &v) {
    Tri2 t;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double *p = verts + 3 * (int64_t)tri[k];
        // px = (p_u - lo_u) * scale ; py = (H - 1) - (p_v - lo_v) * scale
        t.x[k] = __dmul_rn(__dsub_rn(p[v.au], v.lo_u), v.scale);
        t.y[k] = __dsub_rn((double)(v.height - 1), __dmul_rn(__dsub_rn(p[v.av], v.lo_v), v.scale));
        t.z[k] = p[v.ad];
    }
    return t;
}

// Walk the covered pixels of triangle t exactly like _rasterize (io.py:195-222)
// and call f(pixel, zpix) for every inside pixel.
template <typename F>
__device__ __forceinline__ void raster(const Tri2 &t, const View &v, F f) {
    const double mnx = fmin(fmin(t.x[0], t.x[1]), t.x[2]), mxx = fmax(fmax(t.x[0], t.x[1]), t.x[2]);
    const double mny = fmin(fmin(t.y[0], t.y[1]), t.y[2]), mxy = fmax(fmax(t.y[0], t.y[1]), t.y[2]);
    // xmin = max(int(floor(min)), 0) ... ymax = min(int(ceil(max)), H - 1)
    const double fx0 = floor(mnx), fx1 = ceil(mxx), fy0 = floor(mny), fy1 = ceil(mxy);
    const int xmin = fx0 > 0.0 ? (fx0 < 1e9 ? (int)fx0 : 1000000000) : 0;
    const int ymin = fy0 > 0.0 ? (fy0 < 1e9 ? (int)fy0 : 1000000000) : 0;
    const int xmax = fx1 < (double)(v.width - 1) ? (fx1 > -1e9 ? (int)fx1 : -1000000000) : v.width - 1;
    const int ymax = fy1 < (double)(v.height - 1) ? (fy1 > -1e9 ? (int)fy1 : -1000000000) : v.height - 1;
    if (xmin > xmax || ymin > ymax) return;
    const double x0 = t.x[0], y0 = t.y[0], x1 = t.x[1], y1 = t.y[1], x2 = t.x[2], y2 = t.y[2];
    const double a = __dsub_rn(y1, y2), b = __dsub_rn(x2, x1);   // (y1-y2), (x2-x1)
    const double c = __dsub_rn(y2, y0), e = __dsub_rn(x0, x2);   // (y2-y0), (x0-x2)
    const double denom = __dadd_rn(__dmul_rn(a, e), __dmul_rn(b, __dsub_rn(y0, y2)));
    if (fabs(denom) < 1e-12) return;
    for (int py = ymin; py <= ymax; ++py) {
        const double gy = __dadd_rn((double)py, 0.5);
        const double dy = __dsub_rn(gy, y2);
        for (int px = xmin; px <= xmax; ++px) {
            const double gx = __dadd_rn((double)px, 0.5);
            const double dx = __dsub_rn(gx, x2);
            const double w0 = __ddiv_rn(__dadd_rn(__dmul_rn(a, dx), __dmul_rn(b, dy)), denom);
            const double w1 = __ddiv_rn(__dadd_rn(__dmul_rn(c, dx), __dmul_rn(e, dy)), denom);
            const double w2 = __dsub_rn(__dsub_rn(1.0, w0), w1);
            if ((w0 >= 0.0) & (w1 >= 0.0) & (w2 >= 0.0)) {
                const double z = __dadd_rn(__dadd_rn(__dmul_rn(w0, t.z[0]), __dmul_rn(w1, t.z[1])),
                                           __dmul_rn(w2, t.z[2]));
                f((int64_t)py * v.width + px, z);
            }
        }
    }
}

__global__ void k_snap_depth(const double *verts, const int32_t *tris, int64_t nt, View v,
                             unsigned long long *depth) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nt) return;
    const Tri2 t = project(verts, tris + 3 * i, v);
    raster(t, v, [&](int64_t pix, double z) { atomicMax(depth + pix, (unsigned long long)okey(z)); });
}

__global__ void k_snap_owner(const double *verts, const int32_t *tris, int64_t nt, View v,
                             const unsigned long long *depth, unsigned long long *owner) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nt) return;
    const Tri2 t = project(verts, tris + 3 * i, v);
    raster(t, v, [&](int64_t pix, double z) {
        if ((unsigned long long)okey(z) == depth[pix]) atomicMin(owner + pix, (unsigned long long)i);
    });
}

__global__ void k_snap_zrange(const unsigned long long *depth, const unsigned long long *owner,
                              int64_t npix, unsigned long long *zr) {
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        if (owner[p] != ~0ull) {
            lo = min(lo, depth[p]);
            hi = max(hi, depth[p]);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(zr, lo);
        atomicMax(zr + 1, hi);
    }
}

__global__ void k_snap_shade(const unsigned long long *depth, const unsigned long long *owner,
                             int64_t npix, int64_t n_cloth, const unsigned long long *zr,
                             uint8_t *rgb) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= npix) return;
    const unsigned long long ow = owner[p];
    uint8_t out[3] = {0, 0, 0};
    if (ow != ~0ull) {
        // io.py:_CLOTH_TINT / _OBSTACLE_TINT
        const double tint_c[3] = {0.92, 0.92, 0.98}, tint_o[3] = {0.45, 0.62, 0.85};
        const double *tint = ow < (unsigned long long)n_cloth ? tint_c : tint_o;
        const double zmin = unkey(zr[0]), zmax = unkey(zr[1]);
        const double zspan = fmax(__dsub_rn(zmax, zmin), 1e-12);
        const double shade =
            __dadd_rn(0.25, __ddiv_rn(__dmul_rn(0.75, __dsub_rn(unkey(depth[p]), zmin)), zspan));
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double c = fmin(fmax(__dmul_rn(shade, tint[k]), 0.0), 1.0);
            out[k] = (uint8_t)rint(__dmul_rn(c, 255.0));
        }
    }
    rgb[3 * p] = out[0];
    rgb[3 * p + 1] = out[1];
    rgb[3 * p + 2] = out[2];
}

}  // namespace

// bounds of (n,3) f64 vertices: out[0..2] = min, out[3..5] = max (as keys)
__global__ void k_snap_bounds(const double *verts, int64_t n, unsigned long long *out) {
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const unsigned long long k = okey(verts[3 * i + d]);
            lo[d] = min(lo[d], k);
            hi[d] = max(hi[d], k);
        }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            lo[d] = min(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
            hi[d] = max(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(out + d, lo[d]);
            atomicMax(out + 3 + d, hi[d]);
        }
    }
}

cudaError_t snapshot_bounds(const double *verts, int64_t n, double out[6], cudaStream_t st) {
    unsigned long long *d = nullptr;
    cudaError_t e = cudaMallocAsync(&d, 6 * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    const unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
    cudaMemcpyAsync(d, init, sizeof(init), cudaMemcpyHostToDevice, st);
    const int64_t blocks = n > 0 ? ((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184) : 1;
    k_snap_bounds<<<(unsigned)blocks, 256, 0, st>>>(verts, n, d);
    unsigned long long h[6];
    cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(d, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    for (int k = 0; k < 6; ++k) out[k] = unkey(h[k]);
    return cudaGetLastError();
}

cudaError_t snapshot_render(const double *verts, const int32_t *tris, int64_t nt, int64_t n_cloth,
                            const double view[3], const int32_t axes[3], int width, int height,
                            uint8_t *rgb, void *scratch, cudaStream_t st) {
    View v{view[0], view[1], view[2], axes[0], axes[1], axes[2], width, height};
    const int64_t npix = (int64_t)width * height;
    unsigned long long *depth = (unsigned long long *)scratch;
    unsigned long long *owner = depth + npix;
    unsigned long long *zr = owner + npix;
    cudaMemsetAsync(depth, 0, npix * sizeof(unsigned long long), st);       // -inf
    cudaMemsetAsync(owner, 0xff, npix * sizeof(unsigned long long), st);    // no triangle
    const unsigned long long zinit[2] = {~0ull, 0ull};
    cudaMemcpyAsync(zr, zinit, sizeof(zinit), cudaMemcpyHostToDevice, st);
    if (nt > 0) {
        const unsigned tb = (unsigned)((nt + 127) / 128);
        k_snap_depth<<<tb, 128, 0, st>>>(verts, tris, nt, v, depth);
        k_snap_owner<<<tb, 128, 0, st>>>(verts, tris, nt, v, depth, owner);
    }
    const unsigned pb = (unsigned)((npix + 255) / 256);
    k_snap_zrange<<<pb < 296 ? pb : 296, 256, 0, st>>>(depth, owner, npix, zr);
    k_snap_shade<<<pb, 256, 0, st>>>(depth, owner, npix, n_cloth, zr, rgb);
    // the zinit staging buffer is a host stack array: finish before returning
    cudaError_t e = cudaStreamSynchronize(st);
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace cs
