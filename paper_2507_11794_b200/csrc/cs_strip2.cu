// cs_strip2.cu -- packed fast-mode grid kernel (the production path).
//
// Same algorithm as k_strip_step in cs_strip.cu (warp per column strip,
// sliding register window, six forward springs per node, reactions through
// shuffles / pending accumulators, the previous frame's normals fused in),
// but every lane advances TWO strips at once -- rows [y0, y0+h) in .x and
// [y0+h, y0+2h) in .y of float2 registers -- so the spring, normal and
// integrate arithmetic issues on Blackwell's paired fp32 pipes (FADD2 /
// FMUL2 / FFMA2, two results per instruction).  Shuffles, loads and stores
// stay per element.  Addresses are 32-bit element offsets from per-plane base
// pointers held in uniform registers.
//
// Reference semantics: gpu/kernels.py:86-133 and :314-339 on the topology of
// mesh.py:274-305; fast-mode tolerances.
#include "cs_common.cuh"
#include "cs_kernels.cuh"

namespace cs {

namespace {
constexpr int SW = 32;    // lanes = columns loaded
constexpr int SO = 28;    // columns stored (lanes 2..29)
constexpr int WPB = 4;    // warps per block

struct Planes {
    const float *s[6];    // source x y z vx vy vz
    float *d[6];          // destination
    float *n[3];          // normals
    const float *e[3];    // external acceleration (or null)
};

__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 sp2(float s) { return make_float2(s, s); }
// a - b with one rounding
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __ffma2_rn(b, sp2(-1.f), a); }

struct P6 {
    float2 x, y, z, vx, vy, vz;
};
struct Q3 {
    float2 x, y, z;
};

__device__ __forceinline__ float2 sdn(float2 v, int d) {
    return make_float2(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d));
}
__device__ __forceinline__ float2 sup(float2 v, int d) {
    return make_float2(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d));
}
__device__ __forceinline__ P6 pdn(const P6 &a, int d) {
    return {sdn(a.x, d), sdn(a.y, d), sdn(a.z, d), sdn(a.vx, d), sdn(a.vy, d), sdn(a.vz, d)};
}
__device__ __forceinline__ P6 pup(const P6 &a, int d) {
    return {sup(a.x, d), sup(a.y, d), sup(a.z, d), sup(a.vx, d), sup(a.vy, d), sup(a.vz, d)};
}
__device__ __forceinline__ Q3 qup(const Q3 &a, int d) { return {sup(a.x, d), sup(a.y, d), sup(a.z, d)}; }
__device__ __forceinline__ Q3 qdn(const Q3 &a, int d) { return {sdn(a.x, d), sdn(a.y, d), sdn(a.z, d)}; }
__device__ __forceinline__ void qadd(Q3 &a, const Q3 &b) {
    a.x = add2(a.x, b.x); a.y = add2(a.y, b.y); a.z = add2(a.z, b.z);
}
__device__ __forceinline__ void qsub(Q3 &a, const Q3 &b) {
    a.x = sub2(a.x, b.x); a.y = sub2(a.y, b.y); a.z = sub2(a.z, b.z);
}

// rows at element offsets oa / ob (valid flags va / vb) of the six planes
__device__ __forceinline__ void load_pair(const Planes &P, uint32_t oa, uint32_t ob, bool va,
                                          bool vb, P6 &r) {
    float a[6], b[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        a[q] = va ? __ldg(P.s[q] + oa) : 0.f;
        b[q] = vb ? __ldg(P.s[q] + ob) : 0.f;
    }
    r = {make_float2(a[0], b[0]), make_float2(a[1], b[1]), make_float2(a[2], b[2]),
         make_float2(a[3], b[3]), make_float2(a[4], b[4]), make_float2(a[5], b[5])};
}

// force on `a` from spring (a -> b) for both elements; `mask` is 1 where the
// spring exists.  Springs shorter than 1e-12 contribute nothing
// (solver.py:111-113): their inverse length is forced to 0.
__device__ __forceinline__ Q3 fwd2(const P6 &a, const P6 &b, float2 k, float2 rest, float2 c,
                                   float2 mask) {
    const float2 dx = sub2(b.x, a.x), dy = sub2(b.y, a.y), dz = sub2(b.z, a.z);
    const float2 ux = sub2(b.vx, a.vx), uy = sub2(b.vy, a.vy), uz = sub2(b.vz, a.vz);
    const float2 d2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
    float2 inv = make_float2(d2.x >= 1e-24f ? rsqrtf(d2.x) : 0.f, d2.y >= 1e-24f ? rsqrtf(d2.y) : 0.f);
    inv = mul2(inv, mask);
    // one Newton step on the residual: |d| nearly correctly rounded
    const float2 l0 = mul2(d2, inv);
    const float2 len = fma2(fma2(mul2(l0, sp2(-1.f)), l0, d2), mul2(inv, sp2(0.5f)), l0);
    const float2 rel = mul2(fma2(ux, dx, fma2(uy, dy, mul2(uz, dz))), inv);
    const float2 sc = mul2(fma2(k, sub2(len, rest), mul2(c, rel)), inv);
    return {mul2(sc, dx), mul2(sc, dy), mul2(sc, dz)};
}

// unit normal of face (p0, p1, p2) for both elements, zero where mask is 0
__device__ __forceinline__ Q3 face2(const P6 &p0, const P6 &p1, const P6 &p2, float2 mask) {
    const float2 ax = sub2(p1.x, p0.x), ay = sub2(p1.y, p0.y), az = sub2(p1.z, p0.z);
    const float2 bx = sub2(p2.x, p0.x), by = sub2(p2.y, p0.y), bz = sub2(p2.z, p0.z);
    const float2 fx = fma2(ay, bz, mul2(mul2(az, by), sp2(-1.f)));
    const float2 fy = fma2(az, bx, mul2(mul2(ax, bz), sp2(-1.f)));
    const float2 fz = fma2(ax, by, mul2(mul2(ay, bx), sp2(-1.f)));
    const float2 d2 = fma2(fx, fx, fma2(fy, fy, mul2(fz, fz)));
    float2 inv = make_float2(d2.x > 1e-40f ? rsqrtf(d2.x) : 0.f, d2.y > 1e-40f ? rsqrtf(d2.y) : 0.f);
    inv = mul2(inv, mask);
    return {mul2(fx, inv), mul2(fy, inv), mul2(fz, inv)};
}

__device__ __forceinline__ float okf(bool b) { return b ? 1.f : 0.f; }

template <bool NORMALS, bool EXT>
__global__ void __launch_bounds__(SW *WPB)
k_strip2(const StepParams p, const Planes P, const uint32_t *__restrict__ pinbits) {
    const int lane = threadIdx.x & 31;
    const int warp = blockIdx.x * WPB + (threadIdx.x >> 5);
    const int strips_x = (p.nx + SO - 1) / SO;
    const int sx = warp % strips_x, spair = warp / strips_x;
    const int h = p.strip_h;
    const int ya = 2 * spair * h, yb = ya + h;
    if (ya >= p.ny) return;  // warp-uniform exit
    const int yae = min(ya + h, p.ny), ybe = min(yb + h, p.ny);
    const int i = sx * SO - 2 + lane;
    const bool col_ok = (i >= 0) & (i < p.nx);
    const bool out_lane = (lane >= 2) & (lane < 30) & col_ok;
    const float cm = okf(col_ok), m_ip1 = okf(col_ok & (i + 1 < p.nx));
    const float m_ip2 = okf(col_ok & (i + 2 < p.nx)), m_im1 = okf(col_ok & (i >= 1));
    const float2 ks = sp2(p.k_struct), kh = sp2(p.k_shear), kb = sp2(p.k_bend), c = sp2(p.damping);
    const float2 r0 = sp2(p.rest[0]), r1 = sp2(p.rest[1]), r2 = sp2(p.rest[2]);
    const float2 r3 = sp2(p.rest[3]), r4 = sp2(p.rest[4]), r5 = sp2(p.rest[5]);
    const uint32_t pitch = (uint32_t)p.pitch, hp = (uint32_t)h * pitch;
    const uint32_t ci = (uint32_t)(col_ok ? i : 0);

    auto rowv = [&](int j) { return col_ok & (j >= 0) & (j < p.ny); };
    auto off = [&](int j) { return (uint32_t)(j >= 0 ? j : 0) * pitch + ci; };

    P6 A, B, C, D;
    load_pair(P, off(ya - 2), off(yb - 2), rowv(ya - 2), rowv(yb - 2), A);
    load_pair(P, off(ya - 1), off(yb - 1), rowv(ya - 1), rowv(yb - 1), B);
    load_pair(P, off(ya), off(yb), rowv(ya), rowv(yb), C);
    Q3 pend0 = {sp2(0.f), sp2(0.f), sp2(0.f)}, pend1 = pend0, pend2 = pend0;
    Q3 pT0 = pend0, pT1 = pend0;  // faces of cell (i, j-1)
    P6 A1 = pdn(A, 1);

    for (int t = -2; t < h; ++t) {
        const int ja = ya + t, jb = yb + t;
        load_pair(P, off(ja + 3), off(jb + 3), rowv(ja + 3), rowv(jb + 3), D);
        const P6 A2 = pdn(A, 2), B1d = pdn(B, 1), B1u = pup(B, 1);
        // row existence (warp-uniform) times column existence (per lane)
        const float2 rs = make_float2(okf((ja >= 0) & (ja < p.ny)), okf((jb >= 0) & (jb < p.ny)));
        const float2 rs1 = make_float2(okf(ja + 1 < p.ny), okf(jb + 1 < p.ny));
        const float2 rs2 = make_float2(okf(ja + 2 < p.ny), okf(jb + 2 < p.ny));
        const float2 rr1 = mul2(rs, rs1);
        const Q3 fsi = fwd2(A, A1, ks, r0, c, mul2(rs, sp2(m_ip1)));
        const Q3 fsj = fwd2(A, B, ks, r1, c, mul2(rr1, sp2(cm)));
        const Q3 fh1 = fwd2(A, B1d, kh, r2, c, mul2(rr1, sp2(m_ip1)));
        const Q3 fh2 = fwd2(A, B1u, kh, r3, c, mul2(rr1, sp2(m_im1)));
        const Q3 fbi = fwd2(A, A2, kb, r4, c, mul2(rs, sp2(m_ip2)));
        const Q3 fbj = fwd2(A, C, kb, r5, c, mul2(mul2(rs, rs2), sp2(cm)));
        Q3 F = pend0;
        qadd(F, fsi); qadd(F, fsj); qadd(F, fh1); qadd(F, fh2); qadd(F, fbi); qadd(F, fbj);
        qsub(F, qup(fsi, 1));
        qsub(F, qup(fbi, 2));
        qsub(pend1, fsj);
        qsub(pend1, qup(fh1, 1));
        qsub(pend1, qdn(fh2, 1));
        qsub(pend2, fbj);

        const uint32_t oa = off(ja), ob = off(jb);
        const bool sa = out_lane & (t >= 0) & (ja < yae), sb = out_lane & (t >= 0) & (jb < ybe);
        if (NORMALS) {
            // cell (i, j): T0 = (v00, v01, v10), T1 = (v10, v01, v11)
            const float2 mc = mul2(rr1, sp2(m_ip1));
            const Q3 T0 = face2(A, B, A1, mc);
            const Q3 T1 = face2(A1, B, B1d, mc);
            // node normal of the OLD state: faces of (i-1,j-1).T1, (i,j-1).T0,
            // (i,j-1).T1, (i-1,j).T0, (i-1,j).T1, (i,j).T0 (absent cells are 0)
            Q3 s = qup(pT1, 1);
            qadd(s, pT0);
            qadd(s, pT1);
            qadd(s, qup(T0, 1));
            qadd(s, qup(T1, 1));
            qadd(s, T0);
            const float2 n2 = fma2(s.x, s.x, fma2(s.y, s.y, mul2(s.z, s.z)));
            if (sa) {
                const bool up = !(n2.x > 1e-40f);  // +y fallback (kernels.py:333-338)
                const float iv = up ? 0.f : rsqrtf(n2.x);
                P.n[0][oa] = s.x.x * iv;
                P.n[1][oa] = up ? 1.f : s.y.x * iv;
                P.n[2][oa] = s.z.x * iv;
            }
            if (sb) {
                const bool up = !(n2.y > 1e-40f);
                const float iv = up ? 0.f : rsqrtf(n2.y);
                P.n[0][ob] = s.x.y * iv;
                P.n[1][ob] = up ? 1.f : s.y.y * iv;
                P.n[2][ob] = s.z.y * iv;
            }
            pT0 = T0;
            pT1 = T1;
        }

        // integrate: a = F * inv_m + g (+ ext), semi-implicit unless flagged
        const float2 im = sp2(p.inv_mass), dt = sp2(p.dt);
        float2 ax = fma2(F.x, im, sp2(p.gx)), ay = fma2(F.y, im, sp2(p.gy)), az = fma2(F.z, im, sp2(p.gz));
        if (EXT) {
            const bool la = rowv(ja), lb = rowv(jb);
            ax = add2(ax, make_float2(la ? P.e[0][oa] : 0.f, lb ? P.e[0][ob] : 0.f));
            ay = add2(ay, make_float2(la ? P.e[1][oa] : 0.f, lb ? P.e[1][ob] : 0.f));
            az = add2(az, make_float2(la ? P.e[2][oa] : 0.f, lb ? P.e[2][ob] : 0.f));
        }
        float2 x = A.x, y = A.y, z = A.z, vx = A.vx, vy = A.vy, vz = A.vz;
        if (p.explicit_euler) {
            x = fma2(vx, dt, x); y = fma2(vy, dt, y); z = fma2(vz, dt, z);
            vx = fma2(ax, dt, vx); vy = fma2(ay, dt, vy); vz = fma2(az, dt, vz);
        } else {
            vx = fma2(ax, dt, vx); vy = fma2(ay, dt, vy); vz = fma2(az, dt, vz);
            x = fma2(vx, dt, x); y = fma2(vy, dt, y); z = fma2(vz, dt, z);
        }
        if (sa) {
            const bool pin = (__ldg(pinbits + (oa >> 5)) >> (oa & 31)) & 1u;
            P.d[0][oa] = pin ? A.x.x : x.x;
            P.d[1][oa] = pin ? A.y.x : y.x;
            P.d[2][oa] = pin ? A.z.x : z.x;
            P.d[3][oa] = pin ? A.vx.x : vx.x;
            P.d[4][oa] = pin ? A.vy.x : vy.x;
            P.d[5][oa] = pin ? A.vz.x : vz.x;
        }
        if (sb) {
            const bool pin = (__ldg(pinbits + (ob >> 5)) >> (ob & 31)) & 1u;
            P.d[0][ob] = pin ? A.x.y : x.y;
            P.d[1][ob] = pin ? A.y.y : y.y;
            P.d[2][ob] = pin ? A.z.y : z.y;
            P.d[3][ob] = pin ? A.vx.y : vx.y;
            P.d[4][ob] = pin ? A.vy.y : vy.y;
            P.d[5][ob] = pin ? A.vz.y : vz.y;
        }
        // slide: row j+1 becomes current; its one-lane shift is B1d
        A = B; B = C; C = D; A1 = B1d;
        pend0 = pend1; pend1 = pend2; pend2 = {sp2(0.f), sp2(0.f), sp2(0.f)};
    }
}
}  // namespace

int strip2_rows(const StepParams &p) {
    // tall strips amortise the 2-row vertical halo; small grids get shorter
    // strips so that enough warps are resident (148 SMs)
    static int forced = -1;
    if (forced < 0) {
        const char *e = getenv("CS_STRIP_ROWS");
        forced = e ? atoi(e) : 0;
    }
    if (forced > 0) return forced;
    const int sxn = (p.nx + SO - 1) / SO;
    int sh = 64;
    while (sh > 8 && (int64_t)sxn * ((p.ny + 2 * sh - 1) / (2 * sh)) < 148 * 12) sh /= 2;
    return sh;
}

void launch_strip2_step(const StepParams &p, bool normals, const float *src, float *dst,
                        const uint32_t *pinbits, const float *ext, float *nrm, cudaStream_t st) {
    StepParams q = p;
    q.strip_h = strip2_rows(p);
    Planes P;
    for (int k = 0; k < 6; ++k) {
        P.s[k] = src + k * p.plane;
        P.d[k] = dst + k * p.plane;
    }
    for (int k = 0; k < 3; ++k) {
        P.n[k] = nrm + k * p.plane;
        P.e[k] = ext ? ext + k * p.plane : nullptr;
    }
    const int sxn = (p.nx + SO - 1) / SO;
    const int64_t warps = (int64_t)sxn * ((p.ny + 2 * q.strip_h - 1) / (2 * q.strip_h));
    const unsigned blocks = (unsigned)((warps + WPB - 1) / WPB);
    const dim3 block(SW * WPB);
    if (normals) {
        if (ext) k_strip2<true, true><<<blocks, block, 0, st>>>(q, P, pinbits);
        else k_strip2<true, false><<<blocks, block, 0, st>>>(q, P, pinbits);
    } else {
        if (ext) k_strip2<false, true><<<blocks, block, 0, st>>>(q, P, pinbits);
        else k_strip2<false, false><<<blocks, block, 0, st>>>(q, P, pinbits);
    }
}

}  // namespace cs
