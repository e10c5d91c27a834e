// cs_grid.cu -- regular-grid stencil kernels: fused spring force + integrate,
// the i32 force debug pass, and vertex normals.
//
// Reference semantics: gpu/kernels.py:86-133 (spring_force + integrate) and
// :314-339 (normal_update); spring topology and order from
// mesh.generate_cloth_grid (mesh.py:274-305).
//
// Data layout in HBM: one state buffer = six f32 planes x, y, z, vx, vy, vz,
// each `pitch * ny` elements with row j at offset j*pitch (pitch = nx rounded
// up to 32, so every warp-row is one 128-B line).  Two state buffers
// ping-pong: the step reads `src` and writes `dst`, so "previousPositions"
// costs no traffic.  Pins are a bitmask (1 bit per node); free nodes share one
// inverse mass.  Algorithmic traffic of the fused step: 24 B read + 24 B
// written per node.
//
// Per node the 12 incident springs are summed in ascending spring-id order of
// the reference's spring table, so the stencil path and the generic CSR path
// give bit-identical results.  Because RN subtraction is sign-symmetric, a
// spring evaluated from either endpoint yields exactly the negated force of
// the other endpoint (the reference's action/reaction), in both arithmetic
// modes.
#include "cs_common.cuh"
#include "cs_kernels.cuh"

namespace cs {

constexpr int TX = 32;     // tile width  (one warp per row)
constexpr int TY = 16;     // tile height (each thread computes 2 rows)
constexpr int BY = 8;      // block rows
constexpr int H = 2;       // stencil radius (bend springs reach +-2)
constexpr int SW = TX + 2 * H;   // 36
constexpr int SH = TY + 2 * H;   // 20

struct NbrSpec {
    int di, dj, kind, rest;
};
// ascending spring id for node (i,j): see mesh.py:274-289
__constant__ NbrSpec c_nbr[12] = {
    {0, -1, 0, 1}, {-1, 0, 0, 0}, {1, 0, 0, 0}, {0, 1, 0, 1},
    {-1, -1, 1, 2}, {1, -1, 1, 3}, {-1, 1, 1, 3}, {1, 1, 1, 2},
    {0, -2, 2, 5}, {-2, 0, 2, 4}, {2, 0, 2, 4}, {0, 2, 2, 5},
};

// Fused spring-force + integrate over one 32x16 tile.
//   FIXED = true : reference-engine arithmetic (i32 accumulation).
//   FORCES_ONLY  : write the i32 spring forces (read_forces_raw) and stop.
template <bool FIXED, bool FORCES_ONLY>
__global__ void __launch_bounds__(TX * BY)
k_grid_step(const StepParams p, const float *__restrict__ src, float *__restrict__ dst,
            const uint32_t *__restrict__ pinbits, const float *__restrict__ ext,
            int32_t *__restrict__ forces_out) {
    __shared__ float s[6][SH][SW];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const int tid = ty * TX + tx;

    // stage the tile plus a 2-node halo of all six planes
    for (int idx = tid; idx < SH * SW; idx += TX * BY) {
        const int r = idx / SW, c = idx - r * SW;
        const int gi = x0 - H + c, gj = y0 - H + r;
        const bool in = (gi >= 0) & (gi < p.nx) & (gj >= 0) & (gj < p.ny);
        const int64_t g = (int64_t)gj * p.pitch + gi;
#pragma unroll
        for (int q = 0; q < 6; ++q) s[q][r][c] = in ? __ldg(src + q * p.plane + g) : 0.0f;
    }
    __syncthreads();

    const int i = x0 + tx;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        const int ly = ty + half * BY;
        const int j = y0 + ly;
        if (i >= p.nx || j >= p.ny) continue;
        const int sr = ly + H, sc = tx + H;
        const float px = s[0][sr][sc], py = s[1][sr][sc], pz = s[2][sr][sc];
        const float vx = s[3][sr][sc], vy = s[4][sr][sc], vz = s[5][sr][sc];
        const int64_t g = (int64_t)j * p.pitch + i;

        float fx = 0.f, fy = 0.f, fz = 0.f;
        uint32_t ix = 0, iy = 0, iz = 0;  // i32 sums mod 2^32
#pragma unroll
        for (int n = 0; n < 12; ++n) {
            const int di = c_nbr[n].di, dj = c_nbr[n].dj;
            const int ni = i + di, nj = j + dj;
            if (ni < 0 || ni >= p.nx || nj < 0 || nj >= p.ny) continue;
            const float k = c_nbr[n].kind == 0 ? p.k_struct : (c_nbr[n].kind == 1 ? p.k_shear : p.k_bend);
            const float rest = p.rest[c_nbr[n].rest];
            const int qr = sr + dj, qc = sc + di;
            const float dx = s[0][qr][qc] - px, dy = s[1][qr][qc] - py, dz = s[2][qr][qc] - pz;
            const float ux = s[3][qr][qc] - vx, uy = s[4][qr][qc] - vy, uz = s[5][qr][qc] - vz;
            if (FIXED) {
                int32_t ex, ey, ez;
                spring_fixed(dx, dy, dz, ux, uy, uz, k, rest, p.damping, p.scale_f, ex, ey, ez);
                ix += (uint32_t)ex; iy += (uint32_t)ey; iz += (uint32_t)ez;
            } else {
                spring_fast(dx, dy, dz, ux, uy, uz, k, rest, p.damping, fx, fy, fz);
            }
        }
        if (FORCES_ONLY) {
            forces_out[g] = (int32_t)ix;
            forces_out[p.plane + g] = (int32_t)iy;
            forces_out[2 * p.plane + g] = (int32_t)iz;
            continue;
        }
        const bool pinned = (pinbits[g >> 5] >> (g & 31)) & 1u;
        float nx_ = px, ny_ = py, nz_ = pz, nvx = vx, nvy = vy, nvz = vz;
        if (!pinned) {
            float ax, ay, az;
            const float ex = ext ? ext[g] : 0.f, ey = ext ? ext[p.plane + g] : 0.f,
                        ez = ext ? ext[2 * p.plane + g] : 0.f;
            if (FIXED) {
                // kernels.py:126-133: accel = F*inv_m + g + ext (f32, no FMA)
                ax = fadd(fadd(fmul(decode_fixed((int32_t)ix, p.scale_d), p.inv_mass), p.gx), ex);
                ay = fadd(fadd(fmul(decode_fixed((int32_t)iy, p.scale_d), p.inv_mass), p.gy), ey);
                az = fadd(fadd(fmul(decode_fixed((int32_t)iz, p.scale_d), p.inv_mass), p.gz), ez);
                integrate_exact(p.explicit_euler, p.dt, ax, ay, az, nx_, ny_, nz_, nvx, nvy, nvz);
            } else {
                ax = fmaf(fx, p.inv_mass, p.gx) + ex;
                ay = fmaf(fy, p.inv_mass, p.gy) + ey;
                az = fmaf(fz, p.inv_mass, p.gz) + ez;
                integrate_fast(p.explicit_euler, p.dt, ax, ay, az, nx_, ny_, nz_, nvx, nvy, nvz);
            }
        }
        dst[g] = nx_;
        dst[p.plane + g] = ny_;
        dst[2 * p.plane + g] = nz_;
        dst[3 * p.plane + g] = nvx;
        dst[4 * p.plane + g] = nvy;
        dst[5 * p.plane + g] = nvz;
    }
}

// ---------------------------------------------------------------------------
// Vertex normals (kernels.py:314-339) on the grid triangulation
// (mesh.py:296-305): cell (ci,cj) has T0 = (v00, v01, v10) and
// T1 = (v10, v01, v11).  Each face normal is computed once per tile into
// shared memory and every node gathers its <= 6 incident faces in ascending
// triangle id, summed like np.add.reduceat: first + ((0 + g1) + g2 ...).
// ---------------------------------------------------------------------------
constexpr int NTX = 32, NTY = 8;

template <bool EXACT>
__global__ void __launch_bounds__(NTX * NTY)
k_grid_normals(const StepParams p, const float *__restrict__ state, float *__restrict__ nrm) {
    __shared__ float sp[3][NTY + 2][NTX + 2];
    __shared__ float sf[2][3][NTY + 1][NTX + 1];
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * NTX + tx;
    const int x0 = blockIdx.x * NTX, y0 = blockIdx.y * NTY;
    for (int idx = tid; idx < (NTY + 2) * (NTX + 2); idx += NTX * NTY) {
        const int r = idx / (NTX + 2), c = idx - r * (NTX + 2);
        const int gi = x0 - 1 + c, gj = y0 - 1 + r;
        const bool in = (gi >= 0) & (gi < p.nx) & (gj >= 0) & (gj < p.ny);
        const int64_t g = (int64_t)gj * p.pitch + gi;
#pragma unroll
        for (int q = 0; q < 3; ++q) sp[q][r][c] = in ? __ldg(state + q * p.plane + g) : 0.f;
    }
    __syncthreads();
    // faces of cells (x0-1 .. x0+NTX-1) x (y0-1 .. y0+NTY-1)
    for (int idx = tid; idx < (NTY + 1) * (NTX + 1); idx += NTX * NTY) {
        const int r = idx / (NTX + 1), c = idx - r * (NTX + 1);
        // cell (ci,cj) = (x0-1+c, y0-1+r); its v00 sits at sp[.][r][c]
        float p00[3], p10[3], p01[3], p11[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            p00[q] = sp[q][r][c];
            p10[q] = sp[q][r][c + 1];
            p01[q] = sp[q][r + 1][c];
            p11[q] = sp[q][r + 1][c + 1];
        }
        float f0[3], f1[3];
        face_normal<EXACT>(p00, p01, p10, f0);
        face_normal<EXACT>(p10, p01, p11, f1);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            sf[0][q][r][c] = f0[q];
            sf[1][q][r][c] = f1[q];
        }
    }
    __syncthreads();
    const int i = x0 + tx, j = y0 + ty;
    if (i >= p.nx || j >= p.ny) return;
    // incident (cell dx, cell dy, which) in ascending triangle id
    const int cdx[6] = {-1, 0, 0, -1, -1, 0};
    const int cdy[6] = {-1, -1, -1, 0, 0, 0};
    const int wh[6] = {1, 0, 1, 0, 1, 0};
    float s0 = 0.f, s1 = 0.f, s2 = 0.f;   // first face
    float r0 = 0.f, r1 = 0.f, r2 = 0.f;   // pairwise_sum of the rest
    int cnt = 0;
#pragma unroll
    for (int t = 0; t < 6; ++t) {
        const int ci = i + cdx[t], cj = j + cdy[t];
        if (ci < 0 || ci >= p.nx - 1 || cj < 0 || cj >= p.ny - 1) continue;
        const int r = ty + 1 + cdy[t], c = tx + 1 + cdx[t];
        const float a = sf[wh[t]][0][r][c], b = sf[wh[t]][1][r][c], d = sf[wh[t]][2][r][c];
        if (cnt == 0) {
            s0 = a; s1 = b; s2 = d;
        } else {
            r0 = fadd(r0, a); r1 = fadd(r1, b); r2 = fadd(r2, d);
        }
        ++cnt;
    }
    if (cnt > 1) { s0 = fadd(s0, r0); s1 = fadd(s1, r1); s2 = fadd(s2, r2); }
    float o[3];
    normalize_or_up<EXACT>(s0, s1, s2, o);
    const int64_t g = (int64_t)j * p.pitch + i;
    nrm[g] = o[0];
    nrm[p.plane + g] = o[1];
    nrm[2 * p.plane + g] = o[2];
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
void launch_grid_step(const StepParams &p, bool fixed, const float *src, float *dst,
                      const uint32_t *pinbits, const float *ext, cudaStream_t st) {
    dim3 grid((p.nx + TX - 1) / TX, (p.ny + TY - 1) / TY), block(TX, BY);
    if (fixed)
        k_grid_step<true, false><<<grid, block, 0, st>>>(p, src, dst, pinbits, ext, nullptr);
    else
        k_grid_step<false, false><<<grid, block, 0, st>>>(p, src, dst, pinbits, ext, nullptr);
}

void launch_grid_forces(const StepParams &p, const float *src, int32_t *forces, cudaStream_t st) {
    dim3 grid((p.nx + TX - 1) / TX, (p.ny + TY - 1) / TY), block(TX, BY);
    k_grid_step<true, true><<<grid, block, 0, st>>>(p, src, nullptr, nullptr, nullptr, forces);
}

void launch_grid_normals(const StepParams &p, bool exact, const float *state, float *nrm,
                         cudaStream_t st) {
    dim3 grid((p.nx + NTX - 1) / NTX, (p.ny + NTY - 1) / NTY), block(NTX, NTY);
    if (exact)
        k_grid_normals<true><<<grid, block, 0, st>>>(p, state, nrm);
    else
        k_grid_normals<false><<<grid, block, 0, st>>>(p, state, nrm);
}

}  // namespace cs
