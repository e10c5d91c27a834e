// cs_csr.cu -- generic per-node CSR gather (arbitrary spring tables), the
// float64 solver-exact path, CSR vertex normals, and the respond pass.
//
// CSR layout (built at construction from the reference spring table,
// engine.py:204-213): for node n, entries off[n] .. off[n+1]-1 hold
// (neighbour, kind, rest) of every spring touching n, in ascending spring
// id -- exactly the order in which the reference solver's scatter loop
// (solver.py:104-129) adds contributions into node n, so the float64 path
// reproduces solver.step bit for bit.  State planes are `N` elements long
// (pitch = N, one "row").
#include "cs_common.cuh"
#include "cs_kernels.cuh"

namespace cs {


// ---- float32 (fast gather or reference-engine fixed point) --------------------
template <bool FIXED, bool FORCES_ONLY>
__global__ void __launch_bounds__(256)
k_csr_step(const CsrParams p, const float *__restrict__ src, float *__restrict__ dst,
           const int64_t *__restrict__ off, const int32_t *__restrict__ nbr,
           const uint8_t *__restrict__ kind, const float *__restrict__ rest,
           const float *__restrict__ inv_mass, const float *__restrict__ ext,
           int32_t *__restrict__ forces_out) {
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= p.n) return;
    const int64_t P = p.plane;
    const float px = src[n], py = src[P + n], pz = src[2 * P + n];
    const float vx = src[3 * P + n], vy = src[4 * P + n], vz = src[5 * P + n];
    float fx = 0.f, fy = 0.f, fz = 0.f;
    uint32_t ix = 0, iy = 0, iz = 0;
    for (int64_t e = off[n]; e < off[n + 1]; ++e) {
        const int64_t m = nbr[e];
        const float k = p.k[kind[e]];
        const float dx = src[m] - px, dy = src[P + m] - py, dz = src[2 * P + m] - pz;
        const float ux = src[3 * P + m] - vx, uy = src[4 * P + m] - vy, uz = src[5 * P + m] - vz;
        if (FIXED) {
            int32_t ex, ey, ez;
            spring_fixed(dx, dy, dz, ux, uy, uz, k, rest[e], p.damping, p.scale_f, ex, ey, ez);
            ix += (uint32_t)ex; iy += (uint32_t)ey; iz += (uint32_t)ez;
        } else {
            spring_fast(dx, dy, dz, ux, uy, uz, k, rest[e], p.damping, fx, fy, fz);
        }
    }
    if (FORCES_ONLY) {
        forces_out[n] = (int32_t)ix;
        forces_out[P + n] = (int32_t)iy;
        forces_out[2 * P + n] = (int32_t)iz;
        return;
    }
    const float im = inv_mass[n];
    float x = px, y = py, z = pz, ux = vx, uy = vy, uz = vz;
    if (im > 0.f) {
        const float ex = ext ? ext[n] : 0.f, ey = ext ? ext[P + n] : 0.f, ez = ext ? ext[2 * P + n] : 0.f;
        if (FIXED) {
            const float ax = fadd(fadd(fmul(decode_fixed((int32_t)ix, p.scale_d), im), p.gx), ex);
            const float ay = fadd(fadd(fmul(decode_fixed((int32_t)iy, p.scale_d), im), p.gy), ey);
            const float az = fadd(fadd(fmul(decode_fixed((int32_t)iz, p.scale_d), im), p.gz), ez);
            integrate_exact(p.explicit_euler, p.dt, ax, ay, az, x, y, z, ux, uy, uz);
        } else {
            const float ax = fmaf(fx, im, p.gx) + ex, ay = fmaf(fy, im, p.gy) + ey,
                        az = fmaf(fz, im, p.gz) + ez;
            integrate_fast(p.explicit_euler, p.dt, ax, ay, az, x, y, z, ux, uy, uz);
        }
    }
    dst[n] = x; dst[P + n] = y; dst[2 * P + n] = z;
    dst[3 * P + n] = ux; dst[4 * P + n] = uy; dst[5 * P + n] = uz;
}

// ---- float64, solver-exact (solver.py:86-172) --------------------------------------
__global__ void __launch_bounds__(256)
k_csr_step_f64(const CsrParams p, const double *__restrict__ src, double *__restrict__ dst,
               const int64_t *__restrict__ off, const int32_t *__restrict__ nbr,
               const uint8_t *__restrict__ kind, const double *__restrict__ rest,
               const double *__restrict__ mass, const uint8_t *__restrict__ pinned,
               const double *__restrict__ ext) {
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= p.n) return;
    const int64_t P = p.plane;
    const double px = src[n], py = src[P + n], pz = src[2 * P + n];
    const double vx = src[3 * P + n], vy = src[4 * P + n], vz = src[5 * P + n];
    double fx = 0.0, fy = 0.0, fz = 0.0;
    for (int64_t e = off[n]; e < off[n + 1]; ++e) {
        const int64_t m = nbr[e];
        double gx, gy, gz;
        if (spring_f64(__dsub_rn(src[m], px), __dsub_rn(src[P + m], py), __dsub_rn(src[2 * P + m], pz),
                       __dsub_rn(src[3 * P + m], vx), __dsub_rn(src[4 * P + m], vy),
                       __dsub_rn(src[5 * P + m], vz), p.k_d[kind[e]], rest[e], p.damping_d, gx,
                       gy, gz)) {
            fx = __dadd_rn(fx, gx); fy = __dadd_rn(fy, gy); fz = __dadd_rn(fz, gz);
        }
    }
    const double m = mass[n];
    // forces += m*g ; forces += m*ext (solver.py:136-138)
    fx = __dadd_rn(fx, __dmul_rn(m, p.g_d[0]));
    fy = __dadd_rn(fy, __dmul_rn(m, p.g_d[1]));
    fz = __dadd_rn(fz, __dmul_rn(m, p.g_d[2]));
    if (ext) {
        fx = __dadd_rn(fx, __dmul_rn(m, ext[n]));
        fy = __dadd_rn(fy, __dmul_rn(m, ext[P + n]));
        fz = __dadd_rn(fz, __dmul_rn(m, ext[2 * P + n]));
    }
    double x = px, y = py, z = pz, ux = vx, uy = vy, uz = vz;
    if (pinned[n]) {
        ux = uy = uz = 0.0;  // solver.py:170
    } else {
        const double dt = p.dt_d;
        const double ax = __ddiv_rn(fx, m), ay = __ddiv_rn(fy, m), az = __ddiv_rn(fz, m);
        if (p.explicit_euler) {
            x = __dadd_rn(x, __dmul_rn(ux, dt)); y = __dadd_rn(y, __dmul_rn(uy, dt));
            z = __dadd_rn(z, __dmul_rn(uz, dt));
            ux = __dadd_rn(ux, __dmul_rn(ax, dt)); uy = __dadd_rn(uy, __dmul_rn(ay, dt));
            uz = __dadd_rn(uz, __dmul_rn(az, dt));
        } else {
            ux = __dadd_rn(ux, __dmul_rn(ax, dt)); uy = __dadd_rn(uy, __dmul_rn(ay, dt));
            uz = __dadd_rn(uz, __dmul_rn(az, dt));
            x = __dadd_rn(x, __dmul_rn(ux, dt)); y = __dadd_rn(y, __dmul_rn(uy, dt));
            z = __dadd_rn(z, __dmul_rn(uz, dt));
        }
    }
    dst[n] = x; dst[P + n] = y; dst[2 * P + n] = z;
    dst[3 * P + n] = ux; dst[4 * P + n] = uy; dst[5 * P + n] = uz;
}

// ---- normals over an arbitrary triangulation ---------------------------------------
// pass 1: one unit face normal per triangle (f32 planes of length C)
template <bool EXACT>
__global__ void k_face_normals(int64_t nc, int64_t P, const float *__restrict__ pos,
                               const int32_t *__restrict__ tris, float *__restrict__ face) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nc) return;
    float q[3][3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int64_t v = tris[3 * t + c];
        q[c][0] = pos[v]; q[c][1] = pos[P + v]; q[c][2] = pos[2 * P + v];
    }
    float o[3];
    face_normal<EXACT>(q[0], q[1], q[2], o);
    face[t] = o[0]; face[nc + t] = o[1]; face[2 * nc + t] = o[2];
}

// pass 2: per node, first + pairwise_sum(rest) over the ascending incidence
// list (np.add.reduceat, kernels.py:329-332), then normalise.
template <bool EXACT>
__global__ void k_gather_normals(int64_t n, int64_t P, int64_t nc, const float *__restrict__ face,
                                 const int64_t *__restrict__ off, const int32_t *__restrict__ inc,
                                 float *__restrict__ out) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    float s[3] = {0.f, 0.f, 0.f};
    const int64_t lo = off[v], hi = off[v + 1];
    if (hi > lo) {
        const int64_t t0 = inc[lo];
        s[0] = face[t0]; s[1] = face[nc + t0]; s[2] = face[2 * nc + t0];
        const int64_t m = hi - lo - 1;
        float r[3] = {0.f, 0.f, 0.f};
        if (m < 8) {
            for (int64_t q = lo + 1; q < hi; ++q) {
                const int64_t t = inc[q];
                r[0] = fadd(r[0], face[t]); r[1] = fadd(r[1], face[nc + t]);
                r[2] = fadd(r[2], face[2 * nc + t]);
            }
        } else {
            // numpy pairwise_sum, 8 <= m <= 128 (larger degrees recurse in numpy;
            // meshes here never reach that)
            for (int d = 0; d < 3; ++d) {
                float acc[8];
                for (int j = 0; j < 8; ++j) acc[j] = face[d * nc + inc[lo + 1 + j]];
                int64_t i = 8;
                for (; i < m - (m % 8); i += 8)
                    for (int j = 0; j < 8; ++j) acc[j] = fadd(acc[j], face[d * nc + inc[lo + 1 + i + j]]);
                float res = fadd(fadd(fadd(acc[0], acc[1]), fadd(acc[2], acc[3])),
                                 fadd(fadd(acc[4], acc[5]), fadd(acc[6], acc[7])));
                for (; i < m; ++i) res = fadd(res, face[d * nc + inc[lo + 1 + i]]);
                r[d] = res;
            }
        }
        if (m > 0) { s[0] = fadd(s[0], r[0]); s[1] = fadd(s[1], r[1]); s[2] = fadd(s[2], r[2]); }
    }
    float o[3];
    normalize_or_up<EXACT>(s[0], s[1], s[2], o);
    out[v] = o[0]; out[P + v] = o[1]; out[2 * P + v] = o[2];
}

// float64 normals, mesh.compute_vertex_normals (mesh.py:404-434): np.add.at
// per corner => per node the incident faces in (corner, triangle) order,
// summed sequentially from 0.
__global__ void k_face_normals_f64(int64_t nc, int64_t P, const double *__restrict__ pos,
                                   const int32_t *__restrict__ tris, double *__restrict__ face) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nc) return;
    double q[3][3];
    for (int c = 0; c < 3; ++c) {
        const int64_t v = tris[3 * t + c];
        q[c][0] = pos[v]; q[c][1] = pos[P + v]; q[c][2] = pos[2 * P + v];
    }
    const double a0 = __dsub_rn(q[1][0], q[0][0]), a1 = __dsub_rn(q[1][1], q[0][1]),
                 a2 = __dsub_rn(q[1][2], q[0][2]);
    const double b0 = __dsub_rn(q[2][0], q[0][0]), b1 = __dsub_rn(q[2][1], q[0][1]),
                 b2 = __dsub_rn(q[2][2], q[0][2]);
    const double f0 = __dsub_rn(__dmul_rn(a1, b2), __dmul_rn(a2, b1));
    const double f1 = __dsub_rn(__dmul_rn(a2, b0), __dmul_rn(a0, b2));
    const double f2 = __dsub_rn(__dmul_rn(a0, b1), __dmul_rn(a1, b0));
    const double len = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(f0, f0), __dmul_rn(f1, f1)), __dmul_rn(f2, f2)));
    double o0 = 0.0, o1 = 0.0, o2 = 0.0;  // zero-area faces contribute nothing
    if (len > 1e-30) { o0 = __ddiv_rn(f0, len); o1 = __ddiv_rn(f1, len); o2 = __ddiv_rn(f2, len); }
    face[t] = o0; face[nc + t] = o1; face[2 * nc + t] = o2;
}

__global__ void k_gather_normals_f64(int64_t n, int64_t P, int64_t nc,
                                     const double *__restrict__ face,
                                     const int64_t *__restrict__ off,
                                     const int32_t *__restrict__ inc, double *__restrict__ out) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int64_t q = off[v]; q < off[v + 1]; ++q) {
        const int64_t t = inc[q];
        s0 = __dadd_rn(s0, face[t]); s1 = __dadd_rn(s1, face[nc + t]); s2 = __dadd_rn(s2, face[2 * nc + t]);
    }
    const double len = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(s0, s0), __dmul_rn(s1, s1)), __dmul_rn(s2, s2)));
    if (len > 1e-30) {
        out[v] = __ddiv_rn(s0, len); out[P + v] = __ddiv_rn(s1, len); out[2 * P + v] = __ddiv_rn(s2, len);
    } else {
        out[v] = 0.0; out[P + v] = 1.0; out[2 * P + v] = 0.0;
    }
}

// ---- launchers ------------------------------------------------------------------------
static inline unsigned nblk(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

void launch_csr_step(const CsrParams &p, bool fixed, const float *src, float *dst,
                     const int64_t *off, const int32_t *nbr, const uint8_t *kind,
                     const float *rest, const float *im, const float *ext, cudaStream_t st) {
    if (fixed)
        k_csr_step<true, false><<<nblk(p.n, 256), 256, 0, st>>>(p, src, dst, off, nbr, kind, rest, im, ext, nullptr);
    else
        k_csr_step<false, false><<<nblk(p.n, 256), 256, 0, st>>>(p, src, dst, off, nbr, kind, rest, im, ext, nullptr);
}

void launch_csr_forces(const CsrParams &p, const float *src, const int64_t *off,
                       const int32_t *nbr, const uint8_t *kind, const float *rest,
                       int32_t *forces, cudaStream_t st) {
    k_csr_step<true, true><<<nblk(p.n, 256), 256, 0, st>>>(p, src, nullptr, off, nbr, kind, rest,
                                                          nullptr, nullptr, forces);
}

void launch_csr_step_f64(const CsrParams &p, const double *src, double *dst, const int64_t *off,
                         const int32_t *nbr, const uint8_t *kind, const double *rest,
                         const double *mass, const uint8_t *pinned, const double *ext,
                         cudaStream_t st) {
    k_csr_step_f64<<<nblk(p.n, 256), 256, 0, st>>>(p, src, dst, off, nbr, kind, rest, mass, pinned, ext);
}

void launch_csr_normals(int64_t n, int64_t P, int64_t nc, bool exact, const float *pos,
                        const int32_t *tris, float *face, const int64_t *off, const int32_t *inc,
                        float *out, cudaStream_t st) {
    if (exact) {
        k_face_normals<true><<<nblk(nc, 256), 256, 0, st>>>(nc, P, pos, tris, face);
        k_gather_normals<true><<<nblk(n, 256), 256, 0, st>>>(n, P, nc, face, off, inc, out);
    } else {
        k_face_normals<false><<<nblk(nc, 256), 256, 0, st>>>(nc, P, pos, tris, face);
        k_gather_normals<false><<<nblk(n, 256), 256, 0, st>>>(n, P, nc, face, off, inc, out);
    }
}

void launch_csr_normals_f64(int64_t n, int64_t P, int64_t nc, const double *pos,
                            const int32_t *tris, double *face, const int64_t *off,
                            const int32_t *inc, double *out, cudaStream_t st) {
    k_face_normals_f64<<<nblk(nc, 256), 256, 0, st>>>(nc, P, pos, tris, face);
    k_gather_normals_f64<<<nblk(n, 256), 256, 0, st>>>(n, P, nc, face, off, inc, out);
}

}  // namespace cs
