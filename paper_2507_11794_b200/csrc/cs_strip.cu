// cs_strip.cu -- the scalar warp-strip grid kernel: fused spring force +
// integrate (+ the previous frame's vertex normals), one warp per 28-column
// x 64-row strip, no shared memory, no block barriers.  It serves the
// reference-exact fixed-point mode and Engine(kernel="strip"); the fast
// default is its paired-column successor in cs_pair3.cu.
//
// Reference semantics: gpu/kernels.py:86-133 (spring_force + integrate) and
// :314-339 (normal_update) on the grid topology of mesh.py:274-305.
//
// Why this shape.  The first stencil kernel (cs_grid.cu: smem tile, every
// node evaluating its 12 springs) measured 89% issue-active / 19% DRAM on
// ncu at 4096^2 -- instruction bound at ~460 instr/node.  Here:
//   * each lane owns one column; the warp walks down its strip keeping rows
//     j, j+1, j+2 of (x, y, z, vx, vy, vz) in registers (sliding window),
//     loading row j+3 one iteration ahead;
//   * each node evaluates only its 6 FORWARD springs (+i, +2i, +j, +2j and
//     the two cell diagonals it starts) -- every spring exactly once;
//   * reactions go to the partner as the exact negation (RN is sign
//     symmetric): same-row partners through __shfl_up, next-row partners
//     through per-lane pending accumulators (pend1, pend2), the diagonal ones
//     shifted one lane through __shfl;
//   * lanes 0-1 and 30-31 are the +-2 column halo; lanes 2..29 store.
// The sum order is fixed by the program, so results are deterministic; in
// fixed-point mode the i32 sums are order independent and therefore
// bit-identical to the reference engine's atomics.
//
// Normals: while the window holds the (old) positions, each lane also forms
// the two faces of its cell and the node normal of the OLD state -- i.e. the
// previous frame's normal_update, fused into this frame's pass (24 B/node of
// traffic saved).  The engine marks normals stale after a frame and runs the
// stand-alone normals kernel only when someone reads them.
//
// Traffic per node: 24 B read (pos+vel), 24 B written (pos+vel), 12 B
// normals written = 60 B for a full frame.
#include "cs_common.cuh"
#include "cs_kernels.cuh"

namespace cs {

constexpr int SW = 32;       // columns per warp (lanes)
constexpr int SO = 28;       // output columns per warp
constexpr int SH_MAX = 64;   // output rows per warp (fewer when the grid is small)
constexpr int SWPB = 4;      // warps per block

struct N6 {
    float x, y, z, vx, vy, vz;
};

__device__ __forceinline__ N6 shdn(const N6 &a, int d) {
    N6 r;
    r.x = __shfl_down_sync(0xffffffffu, a.x, d);
    r.y = __shfl_down_sync(0xffffffffu, a.y, d);
    r.z = __shfl_down_sync(0xffffffffu, a.z, d);
    r.vx = __shfl_down_sync(0xffffffffu, a.vx, d);
    r.vy = __shfl_down_sync(0xffffffffu, a.vy, d);
    r.vz = __shfl_down_sync(0xffffffffu, a.vz, d);
    return r;
}
__device__ __forceinline__ N6 shup(const N6 &a, int d) {
    N6 r;
    r.x = __shfl_up_sync(0xffffffffu, a.x, d);
    r.y = __shfl_up_sync(0xffffffffu, a.y, d);
    r.z = __shfl_up_sync(0xffffffffu, a.z, d);
    r.vx = __shfl_up_sync(0xffffffffu, a.vx, d);
    r.vy = __shfl_up_sync(0xffffffffu, a.vy, d);
    r.vz = __shfl_up_sync(0xffffffffu, a.vz, d);
    return r;
}

template <typename T>
struct V3 {
    T x, y, z;
};

template <typename T>
__device__ __forceinline__ V3<T> v3up(const V3<T> &a, int d) {
    return {__shfl_up_sync(0xffffffffu, a.x, d), __shfl_up_sync(0xffffffffu, a.y, d),
            __shfl_up_sync(0xffffffffu, a.z, d)};
}
template <typename T>
__device__ __forceinline__ V3<T> v3dn(const V3<T> &a, int d) {
    return {__shfl_down_sync(0xffffffffu, a.x, d), __shfl_down_sync(0xffffffffu, a.y, d),
            __shfl_down_sync(0xffffffffu, a.z, d)};
}

// accumulator type: float (fast gather) or u32 (i32 fixed point, wrapping)
template <bool FIXED>
struct Acc;
template <>
struct Acc<false> {
    using T = float;
};
template <>
struct Acc<true> {
    using T = uint32_t;
};

// Force on `a` from the spring (a -> b); zero when the spring does not exist.
template <bool FIXED>
__device__ __forceinline__ V3<typename Acc<FIXED>::T> fwd(const N6 &a, const N6 &b, float k,
                                                          float rest, float c, float scale_f,
                                                          bool ok) {
    const float dx = b.x - a.x, dy = b.y - a.y, dz = b.z - a.z;
    const float ux = b.vx - a.vx, uy = b.vy - a.vy, uz = b.vz - a.vz;
    if constexpr (FIXED) {
        int32_t ex, ey, ez;
        spring_fixed(dx, dy, dz, ux, uy, uz, k, rest, c, scale_f, ex, ey, ez);
        if (!ok) ex = ey = ez = 0;
        return {(uint32_t)ex, (uint32_t)ey, (uint32_t)ez};
    } else {
        const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
        const float inv = rsqrtf(fmaxf(d2, 1e-30f));
        // one Newton step on the residual makes |d| (nearly) correctly
        // rounded, so a spring at rest sees exactly zero stretch
        const float l0 = d2 * inv;
        const float len = fmaf(fmaf(-l0, l0, d2), 0.5f * inv, l0);
        const float rel = fmaf(ux, dx, fmaf(uy, dy, uz * dz)) * inv;
        float sc = fmaf(k, len - rest, c * rel) * inv;
        sc = (ok && d2 >= 1e-24f) ? sc : 0.f;  // solver.py:111-113 skips length < 1e-12
        return {sc * dx, sc * dy, sc * dz};
    }
}

template <typename T>
__device__ __forceinline__ void addv(V3<T> &a, const V3<T> &b) {
    a.x += b.x; a.y += b.y; a.z += b.z;
}
template <typename T>
__device__ __forceinline__ void subv(V3<T> &a, const V3<T> &b) {
    a.x -= b.x; a.y -= b.y; a.z -= b.z;
}

__device__ __forceinline__ N6 load6(const StepParams &p, const float *__restrict__ src, int i,
                                    int j) {
    N6 r = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (i >= 0 && i < p.nx && j >= 0 && j < p.ny) {
        const int64_t g = (int64_t)j * p.pitch + i;
        r.x = __ldg(src + g);
        r.y = __ldg(src + p.plane + g);
        r.z = __ldg(src + 2 * p.plane + g);
        r.vx = __ldg(src + 3 * p.plane + g);
        r.vy = __ldg(src + 4 * p.plane + g);
        r.vz = __ldg(src + 5 * p.plane + g);
    }
    return r;
}

// face normal of (p0, p1, p2) from N6 positions
template <bool EXACT>
__device__ __forceinline__ V3<float> face6(const N6 &a, const N6 &b, const N6 &c, bool ok) {
    const float p0[3] = {a.x, a.y, a.z}, p1[3] = {b.x, b.y, b.z}, p2[3] = {c.x, c.y, c.z};
    float o[3];
    face_normal<EXACT>(p0, p1, p2, o);
    if (!ok) o[0] = o[1] = o[2] = 0.f;
    return {o[0], o[1], o[2]};
}

template <bool FIXED, bool NORMALS>
__global__ void __launch_bounds__(SW *SWPB)
k_strip_step(const StepParams p, const float *__restrict__ src, float *__restrict__ dst,
             const uint32_t *__restrict__ pinbits, const float *__restrict__ ext,
             float *__restrict__ nrm) {
    using T = typename Acc<FIXED>::T;
    const int lane = threadIdx.x & 31;
    const int warp = blockIdx.x * SWPB + (threadIdx.x >> 5);
    const int strips_x = (p.nx + SO - 1) / SO;
    const int sx = warp % strips_x, sy = warp / strips_x;
    const int y0 = p.row_lo + sy * p.strip_h;
    if (y0 >= p.row_hi) return;  // whole warp exits together
    const int y1 = min(y0 + p.strip_h, p.row_hi);
    const int i = sx * SO - 2 + lane;
    const bool col_ok = (i >= 0) & (i < p.nx);
    const bool out_lane = (lane >= 2) & (lane < 30) & col_ok;
    const float ks = p.k_struct, kh = p.k_shear, kb = p.k_bend, c = p.damping;

    N6 A = load6(p, src, i, y0 - 2);
    N6 B = load6(p, src, i, y0 - 1);
    N6 C = load6(p, src, i, y0);
    N6 D = load6(p, src, i, y0 + 1);  // prefetched one row ahead
    V3<T> pend0 = {0, 0, 0}, pend1 = {0, 0, 0}, pend2 = {0, 0, 0};
    V3<float> pT0 = {0.f, 0.f, 0.f}, pT1 = {0.f, 0.f, 0.f};  // faces of cell (i, j-1)
    bool pT0ok = false, pT1ok = false;

    for (int j = y0 - 2; j < y1; ++j) {
        // A = row j, B = row j+1, C = row j+2 (D = row j+3 in flight)
        const N6 E = load6(p, src, i, j + 4);
        const N6 A1 = shdn(A, 1), A2 = shdn(A, 2), B1d = shdn(B, 1), B1u = shup(B, 1);
        const bool src_ok = col_ok & (j >= 0) & (j < p.ny);
        const bool r1 = j + 1 < p.ny, r2 = j + 2 < p.ny;
        const bool ip1 = i + 1 < p.nx, ip2 = i + 2 < p.nx, im1 = i >= 1;
        // the six forward springs of node (i, j), each evaluated once
        const V3<T> fsi = fwd<FIXED>(A, A1, ks, p.rest[0], c, p.scale_f, src_ok & ip1);
        const V3<T> fsj = fwd<FIXED>(A, B, ks, p.rest[1], c, p.scale_f, src_ok & r1);
        const V3<T> fh1 = fwd<FIXED>(A, B1d, kh, p.rest[2], c, p.scale_f, src_ok & ip1 & r1);
        const V3<T> fh2 = fwd<FIXED>(A, B1u, kh, p.rest[3], c, p.scale_f, src_ok & im1 & r1);
        const V3<T> fbi = fwd<FIXED>(A, A2, kb, p.rest[4], c, p.scale_f, src_ok & ip2);
        const V3<T> fbj = fwd<FIXED>(A, C, kb, p.rest[5], c, p.scale_f, src_ok & r2);
        // reactions of same-row springs started by lanes -1 and -2
        const V3<T> rsi = v3up(fsi, 1), rbi = v3up(fbi, 2);
        V3<T> F = pend0;
        addv(F, fsi); addv(F, fsj); addv(F, fh1); addv(F, fh2); addv(F, fbi); addv(F, fbj);
        subv(F, rsi); subv(F, rbi);
        // reactions owed to rows j+1 and j+2
        subv(pend1, fsj);
        subv(pend1, v3up(fh1, 1));
        subv(pend1, v3dn(fh2, 1));
        subv(pend2, fbj);

        V3<float> T0 = {0.f, 0.f, 0.f}, T1 = {0.f, 0.f, 0.f};
        bool T0ok = false, T1ok = false;
        if (NORMALS) {
            // cell (i, j): T0 = (v00, v01, v10), T1 = (v10, v01, v11)
            const bool cell = col_ok & ip1 & (j >= 0) & r1;
            T0 = face6<FIXED>(A, B, A1, cell);
            T1 = face6<FIXED>(A1, B, B1d, cell);
            T0ok = T1ok = cell;
        }
        if (NORMALS) {
            // node normal of the OLD state: faces of cells (i-1,j-1).T1,
            // (i,j-1).T0, (i,j-1).T1, (i-1,j).T0, (i-1,j).T1, (i,j).T0 in
            // ascending triangle id (engine.py:232-242)
            const V3<float> q0 = v3up(pT1, 1), q3 = v3up(T0, 1), q4 = v3up(T1, 1);
            const bool q0ok = __shfl_up_sync(0xffffffffu, pT1ok, 1) & im1;
            const bool q3ok = __shfl_up_sync(0xffffffffu, T0ok, 1) & im1;
            const bool q4ok = __shfl_up_sync(0xffffffffu, T1ok, 1) & im1;
            if (j >= y0 && out_lane) {
                const V3<float> f[6] = {q0, pT0, pT1, q3, q4, T0};
                const bool fok[6] = {q0ok, pT0ok, pT1ok, q3ok, q4ok, T0ok};
                float s0 = 0.f, s1 = 0.f, s2 = 0.f, r0 = 0.f, rr1 = 0.f, rr2 = 0.f;
                int cnt = 0;
#pragma unroll
                for (int t = 0; t < 6; ++t) {
                    if (!fok[t]) continue;
                    if (FIXED) {  // np.add.reduceat: first + ((0 + g1) + g2 ...)
                        if (cnt == 0) { s0 = f[t].x; s1 = f[t].y; s2 = f[t].z; }
                        else { r0 = fadd(r0, f[t].x); rr1 = fadd(rr1, f[t].y); rr2 = fadd(rr2, f[t].z); }
                    } else {
                        s0 += f[t].x; s1 += f[t].y; s2 += f[t].z;
                    }
                    ++cnt;
                }
                if (FIXED && cnt > 1) { s0 = fadd(s0, r0); s1 = fadd(s1, rr1); s2 = fadd(s2, rr2); }
                float o[3];
                normalize_or_up<FIXED>(s0, s1, s2, o);
                const int64_t g = (int64_t)j * p.pitch + i;
                nrm[g] = o[0];
                nrm[p.plane + g] = o[1];
                nrm[2 * p.plane + g] = o[2];
            }
            pT0 = T0; pT1 = T1; pT0ok = T0ok; pT1ok = T1ok;
        }

        if (j >= y0 && out_lane) {
            const int64_t g = (int64_t)j * p.pitch + i;
            const bool pinned = (__ldg(pinbits + (g >> 5)) >> (g & 31)) & 1u;
            float x = A.x, y = A.y, z = A.z, vx = A.vx, vy = A.vy, vz = A.vz;
            if (!pinned) {
                const float ex = ext ? ext[g] : 0.f, ey = ext ? ext[p.plane + g] : 0.f,
                            ez = ext ? ext[2 * p.plane + g] : 0.f;
                if (FIXED) {
                    const float ax = fadd(fadd(fmul(decode_fixed((int32_t)F.x, p.scale_d), p.inv_mass), p.gx), ex);
                    const float ay = fadd(fadd(fmul(decode_fixed((int32_t)F.y, p.scale_d), p.inv_mass), p.gy), ey);
                    const float az = fadd(fadd(fmul(decode_fixed((int32_t)F.z, p.scale_d), p.inv_mass), p.gz), ez);
                    integrate_exact(p.explicit_euler, p.dt, ax, ay, az, x, y, z, vx, vy, vz);
                } else {
                    const float ax = fmaf((float)F.x, p.inv_mass, p.gx) + ex;
                    const float ay = fmaf((float)F.y, p.inv_mass, p.gy) + ey;
                    const float az = fmaf((float)F.z, p.inv_mass, p.gz) + ez;
                    integrate_fast(p.explicit_euler, p.dt, ax, ay, az, x, y, z, vx, vy, vz);
                }
            }
            dst[g] = x;
            dst[p.plane + g] = y;
            dst[2 * p.plane + g] = z;
            dst[3 * p.plane + g] = vx;
            dst[4 * p.plane + g] = vy;
            dst[5 * p.plane + g] = vz;
        }
        // slide the window
        A = B; B = C; C = D; D = E;
        pend0 = pend1; pend1 = pend2; pend2 = {0, 0, 0};
    }
}

void launch_strip_step(const StepParams &p, bool fixed, bool normals, const float *src,
                       float *dst, const uint32_t *pinbits, const float *ext, float *nrm,
                       cudaStream_t st, bool packed, const HaloDst *halo) {
    if (packed) {  // paired-column f32x2 kernel (fast or reference-exact): cs_pair3.cu
        launch_pair3_step(p, normals, src, dst, pinbits, ext, nrm, st, halo, fixed);
        return;
    }
    // Tall strips amortise the 2-row vertical halo; small grids get shorter
    // strips so that >= ~16 warps per SM (148 SMs) are resident.
    const int sxn = (p.nx + SO - 1) / SO;
    const dim3 block(SW * SWPB);
    int sh = SH_MAX;
    const int rows = p.row_hi - p.row_lo;
    while (sh > 8 && (int64_t)sxn * ((rows + sh - 1) / sh) < 148 * 16) sh /= 2;
    StepParams q = p;
    q.strip_h = sh;
    const int64_t strips = (int64_t)sxn * ((rows + sh - 1) / sh);
    if (strips <= 0) return;
    const unsigned blocks = (unsigned)((strips + SWPB - 1) / SWPB);
    if (fixed) {
        if (normals) k_strip_step<true, true><<<blocks, block, 0, st>>>(q, src, dst, pinbits, ext, nrm);
        else k_strip_step<true, false><<<blocks, block, 0, st>>>(q, src, dst, pinbits, ext, nrm);
    } else {
        if (normals) k_strip_step<false, true><<<blocks, block, 0, st>>>(q, src, dst, pinbits, ext, nrm);
        else k_strip_step<false, false><<<blocks, block, 0, st>>>(q, src, dst, pinbits, ext, nrm);
    }
}

}  // namespace cs
