// cs_kernels.cuh -- per-spring / per-face device math shared by the stencil
// and CSR kernels.  See cs_common.cuh for the two arithmetic modes.
#pragma once
#include "cs_common.cuh"

namespace cs {

// Reference-engine spring force seen from one endpoint (kernels.py:86-110):
// d = p_other - p_self, u = v_other - v_self.  Returns the encoded i32 force.
__device__ __forceinline__ void spring_fixed(float dx, float dy, float dz, float ux, float uy,
                                             float uz, float k, float rest, float c,
                                             float scale_f, int32_t &ex, int32_t &ey,
                                             int32_t &ez) {
    const float len = fsqrt(dot3x(dx, dy, dz, dx, dy, dz));
    const bool ok = len > 1e-12f;
    const float safe = ok ? len : 1.0f;
    const float ax = fdiv(dx, safe), ay = fdiv(dy, safe), az = fdiv(dz, safe);
    const float rel = dot3x(ux, uy, uz, ax, ay, az);
    float mag = fadd(fmul(k, fsub(len, rest)), fmul(c, rel));
    if (!ok) mag = 0.0f;
    ex = encode_fixed(fmul(mag, ax), scale_f);
    ey = encode_fixed(fmul(mag, ay), scale_f);
    ez = encode_fixed(fmul(mag, az), scale_f);
}

// Fast f32 spring force (Hooke + axial damping, solver.py:72-83), one
// reciprocal square root; springs shorter than 1e-12 are skipped
// (solver.py:111-113).
__device__ __forceinline__ void spring_fast(float dx, float dy, float dz, float ux, float uy,
                                            float uz, float k, float rest, float c, float &fx,
                                            float &fy, float &fz) {
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    if (d2 >= 1e-24f) {
        const float inv = rsqrtf(d2);
        const float l0 = d2 * inv;
        const float len = fmaf(fmaf(-l0, l0, d2), 0.5f * inv, l0);  // Newton-refined |d|
        const float rel = fmaf(ux, dx, fmaf(uy, dy, uz * dz)) * inv;
        const float sc = fmaf(k, len - rest, c * rel) * inv;
        fx = fmaf(sc, dx, fx);
        fy = fmaf(sc, dy, fy);
        fz = fmaf(sc, dz, fz);
    }
}

// Float64 spring force with the reference solver's exact operation order
// (solver.py:104-129); returns the force on `self` (the reference's +g for
// endpoint a, and exactly -g for endpoint b by RN sign symmetry).
__device__ __forceinline__ bool spring_f64(double dx, double dy, double dz, double ux,
                                           double uy, double uz, double k, double rest,
                                           double c, double &gx, double &gy, double &gz) {
    const double length =
        __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    if (length < 1e-12) return false;
    const double ax = __ddiv_rn(dx, length), ay = __ddiv_rn(dy, length), az = __ddiv_rn(dz, length);
    const double rel =
        __dadd_rn(__dadd_rn(__dmul_rn(ux, ax), __dmul_rn(uy, ay)), __dmul_rn(uz, az));
    const double mag = __dadd_rn(__dmul_rn(k, __dsub_rn(length, rest)), __dmul_rn(c, rel));
    gx = __dmul_rn(mag, ax);
    gy = __dmul_rn(mag, ay);
    gz = __dmul_rn(mag, az);
    return true;
}

__device__ __forceinline__ void integrate_exact(int explicit_euler, float dt, float ax, float ay,
                                                float az, float &x, float &y, float &z,
                                                float &vx, float &vy, float &vz) {
    if (explicit_euler) {
        x = fadd(x, fmul(vx, dt)); y = fadd(y, fmul(vy, dt)); z = fadd(z, fmul(vz, dt));
        vx = fadd(vx, fmul(ax, dt)); vy = fadd(vy, fmul(ay, dt)); vz = fadd(vz, fmul(az, dt));
    } else {
        vx = fadd(vx, fmul(ax, dt)); vy = fadd(vy, fmul(ay, dt)); vz = fadd(vz, fmul(az, dt));
        x = fadd(x, fmul(vx, dt)); y = fadd(y, fmul(vy, dt)); z = fadd(z, fmul(vz, dt));
    }
}

__device__ __forceinline__ void integrate_fast(int explicit_euler, float dt, float ax, float ay,
                                               float az, float &x, float &y, float &z, float &vx,
                                               float &vy, float &vz) {
    if (explicit_euler) {
        x = fmaf(vx, dt, x); y = fmaf(vy, dt, y); z = fmaf(vz, dt, z);
        vx = fmaf(ax, dt, vx); vy = fmaf(ay, dt, vy); vz = fmaf(az, dt, vz);
    } else {
        vx = fmaf(ax, dt, vx); vy = fmaf(ay, dt, vy); vz = fmaf(az, dt, vz);
        x = fmaf(vx, dt, x); y = fmaf(vy, dt, y); z = fmaf(vz, dt, z);
    }
}

// Unit face normal of (p0, p1, p2), np.cross order; zero for degenerate faces
// (kernels.py:318-323: norm > 1e-20).
template <bool EXACT>
__device__ __forceinline__ void face_normal(const float *p0, const float *p1, const float *p2,
                                            float *out) {
    if (EXACT) {
        const float a0 = fsub(p1[0], p0[0]), a1 = fsub(p1[1], p0[1]), a2 = fsub(p1[2], p0[2]);
        const float b0 = fsub(p2[0], p0[0]), b1 = fsub(p2[1], p0[1]), b2 = fsub(p2[2], p0[2]);
        const float f0 = fsub(fmul(a1, b2), fmul(a2, b1));
        const float f1 = fsub(fmul(a2, b0), fmul(a0, b2));
        const float f2 = fsub(fmul(a0, b1), fmul(a1, b0));
        const float nrm = fsqrt(dot3x(f0, f1, f2, f0, f1, f2));
        if (nrm > 1e-20f) {
            out[0] = fdiv(f0, nrm); out[1] = fdiv(f1, nrm); out[2] = fdiv(f2, nrm);
        } else {
            out[0] = out[1] = out[2] = 0.f;
        }
    } else {
        const float a0 = p1[0] - p0[0], a1 = p1[1] - p0[1], a2 = p1[2] - p0[2];
        const float b0 = p2[0] - p0[0], b1 = p2[1] - p0[1], b2 = p2[2] - p0[2];
        const float f0 = a1 * b2 - a2 * b1;
        const float f1 = a2 * b0 - a0 * b2;
        const float f2 = a0 * b1 - a1 * b0;
        const float d2 = fmaf(f0, f0, fmaf(f1, f1, f2 * f2));
        if (d2 > 1e-40f) {
            const float inv = rsqrtf(d2);
            out[0] = f0 * inv; out[1] = f1 * inv; out[2] = f2 * inv;
        } else {
            out[0] = out[1] = out[2] = 0.f;
        }
    }
}

// Normalise a normal sum; +y fallback for vanishing sums (kernels.py:333-338).
template <bool EXACT>
__device__ __forceinline__ void normalize_or_up(float s0, float s1, float s2, float *o) {
    if (EXACT) {
        const float len = fsqrt(dot3x(s0, s1, s2, s0, s1, s2));
        if (len > 1e-20f) {
            o[0] = fdiv(s0, len); o[1] = fdiv(s1, len); o[2] = fdiv(s2, len);
            return;
        }
    } else {
        const float d2 = fmaf(s0, s0, fmaf(s1, s1, s2 * s2));
        if (d2 > 1e-40f) {
            const float inv = rsqrtf(d2);
            o[0] = s0 * inv; o[1] = s1 * inv; o[2] = s2 * inv;
            return;
        }
    }
    o[0] = 0.f; o[1] = 1.f; o[2] = 0.f;
}

// ---- CSR (generic) path parameters -----------------------------------------------
struct CsrParams {
    int64_t n;
    int64_t plane;
    float dt, gx, gy, gz, damping, scale_f;
    float k[3];
    double scale_d;
    double dt_d, g_d[3], k_d[3], damping_d;
    int explicit_euler;
};
void launch_csr_step(const CsrParams &p, bool fixed, const float *src, float *dst,
                     const int64_t *off, const int32_t *nbr, const uint8_t *kind,
                     const float *rest, const float *im, const float *ext, cudaStream_t st);
void launch_csr_forces(const CsrParams &p, const float *src, const int64_t *off,
                       const int32_t *nbr, const uint8_t *kind, const float *rest,
                       int32_t *forces, cudaStream_t st);
void launch_csr_step_f64(const CsrParams &p, const double *src, double *dst, const int64_t *off,
                         const int32_t *nbr, const uint8_t *kind, const double *rest,
                         const double *mass, const uint8_t *pinned, const double *ext,
                         cudaStream_t st);
void launch_csr_normals(int64_t n, int64_t P, int64_t nc, bool exact, const float *pos,
                        const int32_t *tris, float *face, const int64_t *off, const int32_t *inc,
                        float *out, cudaStream_t st);
void launch_csr_normals_f64(int64_t n, int64_t P, int64_t nc, const double *pos,
                            const int32_t *tris, double *face, const int64_t *off,
                            const int32_t *inc, double *out, cudaStream_t st);

// ---- launchers (defined in the .cu files) -------------------------------------
void launch_grid_step(const StepParams &p, bool fixed, const float *src, float *dst,
                      const uint32_t *pinbits, const float *ext, cudaStream_t st);
// A row band's neighbour planes (x y z vx vy vz of the neighbour's
// destination state buffer), each pre-shifted by (dst_row0 - src_row0) rows
// so that the LOCAL element offset of a boundary node addresses its halo
// copy on the neighbour (NVLink peer memory, or the same device in tests).
struct HaloDst {
    float *up[6];
    float *dn[6];
    // the in-kernel seam handshake (k_pair3; null = the stream waits /
    // signals around the kernel instead): this band's flag words -- [0] /
    // [1] passes the upper / lower neighbour completed (written by them),
    // [2] / [5] passes whose upper / lower seam this band completed (device
    // counters, so the frame is graph-capturable), [3] / [6] seam warps done
    // in the running launch, [4] error word -- and the neighbours' words
    // this band writes
    uint32_t *flags = nullptr;
    uint32_t *to_up = nullptr, *to_dn = nullptr;
};
void launch_strip_step(const StepParams &p, bool fixed, bool normals, const float *src,
                       float *dst, const uint32_t *pinbits, const float *ext, float *nrm,
                       cudaStream_t st, bool packed = false, const HaloDst *halo = nullptr);
void launch_pair3_step(const StepParams &p, bool normals, const float *src, float *dst,
                       const uint32_t *pinbits, const float *ext, float *nrm, cudaStream_t st,
                       const HaloDst *halo = nullptr, bool exact = false);
// copy rows [r0, r1) of the six planes of `src` to the (pre-shifted) planes `to`
void launch_push_rows(const float *src, int64_t plane, int pitch, int r0, int r1,
                      float *const to[6], cudaStream_t st);
void launch_pair_normals(const StepParams &p, const float *state, float *nrm, cudaStream_t st);
// reference-exact normals (kernels.py:314-339) in the same paired strip layout
void launch_pair_normals_exact(const StepParams &p, const float *state, float *nrm,
                               cudaStream_t st);
int pair3_rows(const StepParams &p);
void launch_pair3_forces(const StepParams &p, const float *src, const uint32_t *pinbits,
                         int32_t *forces, cudaStream_t st);
void launch_grid_forces(const StepParams &p, const float *src, int32_t *forces, cudaStream_t st);
void launch_grid_normals(const StepParams &p, bool exact, const float *state, float *nrm,
                         cudaStream_t st);

}  // namespace cs
