// cs_gridgen.cu -- generate_cloth_grid (mesh.py:223-317) on the device.
//
// The reference builds a cloth in Python loops (3.8 s at 800^2, ~100 s at
// 4096^2), and even a vectorised host build spends
// seconds materialising 100M springs that the stencil engine never reads.
// Here a grid engine is created from the grid's parameters alone
// (cs_create_grid): node positions, pins, the uniform inverse mass and the
// six spring families' rest lengths come from kernels over the nodes /
// springs of the local rows, in the reference's float64 arithmetic:
//
//   x_i = i * (width / (nx - 1)), the last one = width  (np.linspace)
//   z_j = j * (height / (ny - 1)), the last one = height
//   rest = sqrt((dx*dx + dy*dy) + dz*dz)                 (np.linalg.norm)
//
// and, on request, the whole topology of the local sheet in the reference's
// order (cs_grid_topology: springs, kinds, rest lengths, triangles,
// positions) -- bit-identical to mesh.py's arrays (tests/test_gpu_gridgen.py).
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstring>

namespace cs {

namespace {

// np.linspace(0.0, stop, n)[k] (numpy: arange(n) * (stop / (n - 1)) + 0.0,
// last element = stop)
__device__ __forceinline__ double lin(int k, int n, double stop) {
    if (k == n - 1) return stop;
    return __dadd_rn(__dmul_rn((double)k, __ddiv_rn(stop, (double)(n - 1))), 0.0);
}

// |p_b - p_a| of two generation-plane nodes (x, 0, z): ((dx^2 + 0^2) + dz^2)
__device__ __forceinline__ double rest_len(double xa, double za, double xb, double zb) {
    const double dx = __dsub_rn(xb, xa), dz = __dsub_rn(zb, za), dy = __dsub_rn(0.0, 0.0);
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

// ordered-int keys of non-negative floats (rest lengths are >= 0); reduced
// across the warp first (one atomic pair per warp and family: per-thread
// atomics on the 12 words took 0.5 ms at 4096^2); `has` = this lane has a
// spring of the family (the call is warp-uniform)
__device__ __forceinline__ void minmax(unsigned *mm, int fam, float v, bool has) {
    const unsigned k = __float_as_uint(v);
    const unsigned lo = __reduce_min_sync(0xffffffffu, has ? k : 0xffffffffu);
    const unsigned hi = __reduce_max_sync(0xffffffffu, has ? k : 0u);
    if ((threadIdx.x & 31) == 0 && lo != 0xffffffffu) {
        atomicMin(mm + 2 * fam, lo);
        atomicMax(mm + 2 * fam + 1, hi);
    }
}

// Positions (f32 planes x y z at pitch layout) of local rows [0, rows) =
// global rows [row0, row0 + rows); orientation 1 = the hanging scene's
// rotation (x, 0, z) -> (x, -z, 0) (scenes.py _rotate_xz_to_xy).
__global__ void k_grid_positions(int nx, int ny, int row0, int rows, double width, double height,
                                 int orient, int64_t pitch, int64_t plane, float *__restrict__ st,
                                 double *__restrict__ pos64) {
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= (int64_t)nx * rows) return;
    const int i = (int)(n % nx), lj = (int)(n / nx), j = row0 + lj;
    const double x = lin(i, nx, width), z = lin(j, ny, height);
    double p[3] = {x, 0.0, z};
    if (orient == 1) {  // rotated[:, 1] = -positions[:, 2], rotated[:, 2] = 0
        p[1] = -z;
        p[2] = 0.0;
    }
    if (st) {
        const int64_t g = (int64_t)lj * pitch + i;
        st[g] = (float)p[0];
        st[plane + g] = (float)p[1];
        st[2 * plane + g] = (float)p[2];
    }
    if (pos64) {
        pos64[3 * n] = p[0];
        pos64[3 * n + 1] = p[1];
        pos64[3 * n + 2] = p[2];
    }
}

// Per spring family of the local sheet (its springs between local rows),
// min and max of f32(rest): +i, +j, shear (1,1), shear (-1,1), bend +2i,
// bend +2j.  One thread per local node.
__global__ void k_grid_rest_minmax(int nx, int ny, int row0, int rows, double width,
                                   double height, unsigned *__restrict__ mm) {
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool v = n < (int64_t)nx * rows;  // every lane stays for the warp reductions
    const int i = v ? (int)(n % nx) : 0, lj = v ? (int)(n / nx) : 0, j = row0 + lj;
    const double x0 = lin(i, nx, width), z0 = lin(j, ny, height);
    const bool i1 = v && i + 1 < nx, j1 = v && lj + 1 < rows, i2 = v && i + 2 < nx,
               j2 = v && lj + 2 < rows;
    const double x1 = i1 ? lin(i + 1, nx, width) : 0.0, z1 = j1 ? lin(j + 1, ny, height) : 0.0;
    minmax(mm, 0, i1 ? (float)rest_len(x0, z0, x1, z0) : 0.f, i1);
    minmax(mm, 1, j1 ? (float)rest_len(x0, z0, x0, z1) : 0.f, j1);
    minmax(mm, 2, (i1 && j1) ? (float)rest_len(x0, z0, x1, z1) : 0.f, i1 && j1);  // (i,j)->(i+1,j+1)
    minmax(mm, 3, (i1 && j1) ? (float)rest_len(x1, z0, x0, z1) : 0.f, i1 && j1);  // (i+1,j)->(i,j+1)
    minmax(mm, 4, i2 ? (float)rest_len(x0, z0, lin(i + 2, nx, width), z0) : 0.f, i2);
    minmax(mm, 5, j2 ? (float)rest_len(x0, z0, x0, lin(j + 2, ny, height)) : 0.f, j2);
}

// generate_cloth_grid's spring / triangle arrays of the local sheet (nx x
// rows nodes, local indices), in its order: per node (row-major) structural
// +i then +j; per cell the two shears; per node bend +2i then +2j; per cell
// triangles (v00, v01, v10), (v10, v01, v11).  One thread per local node;
// each computes its springs' closed-form positions in the arrays.
__global__ void k_grid_topology(int nx, int ny, int row0, int rows, double width, double height,
                                int32_t *__restrict__ springs, int32_t *__restrict__ kinds,
                                double *__restrict__ rest, int32_t *__restrict__ tris) {
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= (int64_t)nx * rows) return;
    const int i = (int)(n % nx), lj = (int)(n / nx), j = row0 + lj;
    const int64_t X = nx, R = rows;
    const double x0 = lin(i, nx, width), z0 = lin(j, ny, height);
    const bool i1 = i + 1 < nx, j1 = lj + 1 < rows, i2 = i + 2 < nx, j2 = lj + 2 < rows;
    const double x1 = i1 ? lin(i + 1, nx, width) : 0.0, z1 = j1 ? lin(j + 1, ny, height) : 0.0;
    auto put = [&](int64_t s, int64_t a, int64_t b, int kind, double r) {
        if (springs) {
            springs[2 * s] = (int32_t)a;
            springs[2 * s + 1] = (int32_t)b;
        }
        if (kinds) kinds[s] = kind;
        if (rest) rest[s] = r;
    };
    // structural: rows above hold 2X-1 each; this row's nodes before hold
    // 1 + j1 each
    int64_t s = (int64_t)lj * (2 * X - 1) + (int64_t)i * (1 + (j1 ? 1 : 0));
    if (i1) put(s++, n, n + 1, 0, rest_len(x0, z0, x1, z0));
    if (j1) put(s++, n, n + X, 0, rest_len(x0, z0, x0, z1));
    const int64_t n_st = X * (R - 1) + R * (X - 1);
    if (i1 && j1) {  // shear of cell (i, lj)
        const int64_t c = (int64_t)lj * (X - 1) + i;
        put(n_st + 2 * c, n, n + X + 1, 1, rest_len(x0, z0, x1, z1));
        put(n_st + 2 * c + 1, n + 1, n + X, 1, rest_len(x1, z0, x0, z1));
        if (tris) {
            int32_t *t = tris + 6 * c;
            t[0] = (int32_t)n; t[1] = (int32_t)(n + X); t[2] = (int32_t)(n + 1);
            t[3] = (int32_t)(n + 1); t[4] = (int32_t)(n + X); t[5] = (int32_t)(n + X + 1);
        }
    }
    const int64_t n_sh = 2 * (X - 1) * (R - 1);
    // bend: rows lj' < lj hold (X-2)+ + (lj'+2 < R ? X : 0) each; this row's
    // nodes before hold (i'+2 < X) + j2 each
    const int64_t m = X > 2 ? X - 2 : 0;
    const int64_t full = lj < R - 2 ? lj : (R - 2 > 0 ? R - 2 : 0);
    int64_t b = n_st + n_sh + full * (m + X) + (int64_t)(lj - full) * m +
                (i < m ? i : m) + (int64_t)i * (j2 ? 1 : 0);
    if (i2) put(b++, n, n + 2, 2, rest_len(x0, z0, lin(i + 2, nx, width), z0));
    if (j2) put(b++, n, n + 2 * X, 2, rest_len(x0, z0, x0, lin(j + 2, ny, height)));
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace

cudaError_t grid_positions(int nx, int ny, int row0, int rows, double width, double height,
                           int orient, int64_t pitch, int64_t plane, float *state, double *pos64,
                           cudaStream_t st) {
    k_grid_positions<<<nblk((int64_t)nx * rows), 256, 0, st>>>(nx, ny, row0, rows, width, height,
                                                               orient, pitch, plane, state, pos64);
    return cudaGetLastError();
}

// rest6[q]: the family's single f32 rest length; false when a family holds
// two different f32 values (then the stencil does not apply)
cudaError_t grid_rest6(int nx, int ny, int row0, int rows, double width, double height,
                       float rest6[6], bool *uniform, cudaStream_t st) {
    unsigned *mm = nullptr;
    cudaError_t e = cudaMalloc(&mm, 12 * sizeof(unsigned));
    if (e != cudaSuccess) return e;
    unsigned init[12];
    for (int q = 0; q < 6; ++q) {
        init[2 * q] = 0xffffffffu;
        init[2 * q + 1] = 0u;
    }
    cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, st);
    k_grid_rest_minmax<<<nblk((int64_t)nx * rows), 256, 0, st>>>(nx, ny, row0, rows, width, height,
                                                                 mm);
    unsigned out[12];
    cudaMemcpyAsync(out, mm, sizeof out, cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    cudaFree(mm);
    if (e != cudaSuccess) return e;
    *uniform = true;
    for (int q = 0; q < 6; ++q) {
        if (out[2 * q] == 0xffffffffu) {  // no spring of this family (a 2-wide sheet)
            rest6[q] = 0.f;
            continue;
        }
        if (out[2 * q] != out[2 * q + 1]) *uniform = false;
        unsigned u = out[2 * q];
        float f;
        memcpy(&f, &u, 4);
        rest6[q] = f;
    }
    return cudaGetLastError();
}

cudaError_t grid_topology(int nx, int ny, int row0, int rows, double width, double height,
                          int32_t *springs, int32_t *kinds, double *rest, int32_t *tris,
                          double *pos64, cudaStream_t st) {
    k_grid_topology<<<nblk((int64_t)nx * rows), 256, 0, st>>>(nx, ny, row0, rows, width, height,
                                                              springs, kinds, rest, tris);
    if (pos64)
        k_grid_positions<<<nblk((int64_t)nx * rows), 256, 0, st>>>(
            nx, ny, row0, rows, width, height, 0, 0, 0, nullptr, pos64);
    return cudaGetLastError();
}

}  // namespace cs
