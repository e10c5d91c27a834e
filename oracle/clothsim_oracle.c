/*
 * clothsim_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference cloth step (arxiv 2507.11794, Python
 * package `clothsim` under /root/reference/pkg/src).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the checker or the timed CPU baseline.
 * The product path (paper_2507_11794_b200) never links or calls it.
 *
 * Two restatements live here:
 *
 *   or_sol_*  float64 serial solver: clothsim/solver.py and collision.py.
 *             Compiled with -ffp-contract=off so every operation rounds like
 *             the Python float arithmetic it restates (bit-exact, pinned by
 *             tests/golden fixtures generated from the reference).
 *
 *   or_eng_*  float32 "GPU engine" semantics: clothsim/gpu/kernels.py and
 *             fixedpoint.py -- per-spring f32 force, i32 fixed-point
 *             accumulation (scale 2^16, RNE, saturating), f32 integrate,
 *             f32 Moller-Trumbore with numpy's operation order, fixed-point
 *             response accumulation, CSR normals.  Bit-exact vs the numpy
 *             twins (pinned by golden fixtures).
 *
 * numpy operation order that matters for bit-exactness (verified with the
 * reference's numpy 2.3): einsum("ij,ij->i") sums ((p0+p1)+p2) in f32;
 * np.cross computes a1*b2-a2*b1, a2*b0-a0*b2, a0*b1-a1*b0; sqrt and divide
 * are correctly rounded.
 *
 * Multithreading (OpenMP) is used only where the result is provably
 * order-independent (integer accumulation) or where contacts are replayed in
 * the serial order, so nthreads never changes a single bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_EXPORT __attribute__((visibility("default")))

typedef int64_t i64;
typedef int32_t i32;

static int g_threads = 1;

OR_EXPORT void or_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
OR_EXPORT int or_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ======================================================================= */
/* float64 solver: clothsim/solver.py                                       */
/* ======================================================================= */

/* solver.accumulate_forces (solver.py:86-139): Python loop over springs in
 * table order, then + m*g, + m*ext, pinned rows zeroed.  Serial when
 * g_threads == 1; the threaded variant is a node gather with the same
 * per-node add sequence, so both are bit-exact. */
OR_EXPORT i64 or_sol_forces(i64 n, i64 ns, const i32 *sidx, const double *rest,
                            const i32 *kinds, const double *k3, double c,
                            const double *pos, const double *vel,
                            const double *mass, const uint8_t *pinned,
                            const double *g, const double *ext, double *f) {
    i64 degenerate = 0;
    int nt = g_threads;
    if (nt <= 1) {
        for (i64 i = 0; i < 3 * n; ++i) f[i] = 0.0;
        for (i64 s = 0; s < ns; ++s) {
            i64 a = sidx[2 * s], b = sidx[2 * s + 1];
            const double *pa = pos + 3 * a, *pb = pos + 3 * b;
            double dx = pb[0] - pa[0], dy = pb[1] - pa[1], dz = pb[2] - pa[2];
            double length = sqrt(dx * dx + dy * dy + dz * dz);
            if (length < 1e-12) { degenerate++; continue; }
            double ux = dx / length, uy = dy / length, uz = dz / length;
            const double *va = vel + 3 * a, *vb = vel + 3 * b;
            double rel = (vb[0] - va[0]) * ux + (vb[1] - va[1]) * uy + (vb[2] - va[2]) * uz;
            double mag = k3[kinds[s]] * (length - rest[s]) + c * rel;
            double gx = mag * ux, gy = mag * uy, gz = mag * uz;
            f[3 * a] += gx; f[3 * a + 1] += gy; f[3 * a + 2] += gz;
            f[3 * b] -= gx; f[3 * b + 1] -= gy; f[3 * b + 2] -= gz;
        }
    } else {
        /* Threaded variant: node gather over a CSR of incident springs sorted
         * by spring id.  Each node then receives exactly the serial loop's
         * sequence of adds (0 + g_s1 - g_s2 ...), so the result is
         * bit-identical to the serial scatter for any thread count. */
        /* the incidence CSR depends only on the spring table: cache it */
        static const i32 *c_sidx = NULL;
        static i64 c_ns = -1, c_n = -1, c_sig = 0;
        static i64 *off = NULL, *ent = NULL;
        i64 sig = ns > 0 ? ((i64)sidx[0] * 31 + sidx[2 * ns - 1]) * 131 + sidx[ns] : 0;
        if (c_sidx != sidx || c_ns != ns || c_n != n || c_sig != sig) {
            free(off);
            free(ent);
            off = (i64 *)calloc(n + 1, sizeof(i64));
            ent = (i64 *)malloc(sizeof(i64) * 2 * (ns > 0 ? ns : 1));
            for (i64 s = 0; s < ns; ++s) { off[sidx[2 * s] + 1]++; off[sidx[2 * s + 1] + 1]++; }
            for (i64 i = 0; i < n; ++i) off[i + 1] += off[i];
            i64 *fill = (i64 *)malloc(sizeof(i64) * (n > 0 ? n : 1));
            memcpy(fill, off, sizeof(i64) * n);
            for (i64 s = 0; s < ns; ++s) { ent[fill[sidx[2 * s]]++] = s; ent[fill[sidx[2 * s + 1]]++] = s; }
            free(fill);
            c_sidx = sidx; c_ns = ns; c_n = n; c_sig = sig;
        }
        i64 degs = 0;
#pragma omp parallel for num_threads(nt) schedule(static) reduction(+ : degs)
        for (i64 v = 0; v < n; ++v) {
            double fx = 0.0, fy = 0.0, fz = 0.0;
            for (i64 q = off[v]; q < off[v + 1]; ++q) {
                i64 s = ent[q];
                i64 a = sidx[2 * s], b = sidx[2 * s + 1];
                const double *pa = pos + 3 * a, *pb = pos + 3 * b;
                double dx = pb[0] - pa[0], dy = pb[1] - pa[1], dz = pb[2] - pa[2];
                double length = sqrt(dx * dx + dy * dy + dz * dz);
                if (length < 1e-12) { if (v == a) degs++; continue; }
                double ux = dx / length, uy = dy / length, uz = dz / length;
                const double *va = vel + 3 * a, *vb = vel + 3 * b;
                double rel = (vb[0] - va[0]) * ux + (vb[1] - va[1]) * uy + (vb[2] - va[2]) * uz;
                double mag = k3[kinds[s]] * (length - rest[s]) + c * rel;
                double gx = mag * ux, gy = mag * uy, gz = mag * uz;
                if (v == a) { fx += gx; fy += gy; fz += gz; }
                else { fx -= gx; fy -= gy; fz -= gz; }
            }
            f[3 * v] = fx; f[3 * v + 1] = fy; f[3 * v + 2] = fz;
        }
        degenerate = degs;
    }
    /* forces += masses[:, None] * gravity; forces += masses * ext; pinned = 0 */
    for (i64 i = 0; i < n; ++i) {
        for (int d = 0; d < 3; ++d) f[3 * i + d] = f[3 * i + d] + mass[i] * g[d];
        if (ext)
            for (int d = 0; d < 3; ++d) f[3 * i + d] = f[3 * i + d] + mass[i] * ext[3 * i + d];
        if (pinned[i]) f[3 * i] = f[3 * i + 1] = f[3 * i + 2] = 0.0;
    }
    return degenerate;
}

/* solver.integrate (solver.py:157-172).  Returns the first non-finite node
 * (solver._check_finite, :175-182) or -1. */
OR_EXPORT i64 or_sol_integrate(i64 n, double *pos, double *prev, double *vel,
                               const double *f, const double *mass,
                               const uint8_t *pinned, double dt, int explicit_euler) {
    memcpy(prev, pos, sizeof(double) * 3 * n);
    for (i64 i = 0; i < n; ++i) {
        if (pinned[i]) {
            vel[3 * i] = vel[3 * i + 1] = vel[3 * i + 2] = 0.0;
            continue;
        }
        double m = mass[i];
        for (int d = 0; d < 3; ++d) {
            if (explicit_euler) {
                pos[3 * i + d] += vel[3 * i + d] * dt;
                vel[3 * i + d] += f[3 * i + d] / m * dt;
            } else {
                vel[3 * i + d] += f[3 * i + d] / m * dt;
                pos[3 * i + d] += vel[3 * i + d] * dt;
            }
        }
    }
    for (i64 i = 0; i < n; ++i)
        for (int d = 0; d < 3; ++d)
            if (!isfinite(pos[3 * i + d]) || !isfinite(vel[3 * i + d])) return i;
    return -1;
}

/* collision.edge_triangle_intersect (collision.py:96-146), float64. */
static int sol_mt(const double *s, const double *e, const double *v0, const double *v1,
                  const double *v2, double eps, double *point) {
    double sx = s[0], sy = s[1], sz = s[2];
    double dx = e[0] - sx, dy = e[1] - sy, dz = e[2] - sz;
    double d_len = sqrt(dx * dx + dy * dy + dz * dz);
    if (d_len <= eps) return 0;
    double rx = dx / d_len, ry = dy / d_len, rz = dz / d_len;
    double ax0 = v0[0], ay0 = v0[1], az0 = v0[2];
    double e1x = v1[0] - ax0, e1y = v1[1] - ay0, e1z = v1[2] - az0;
    double e2x = v2[0] - ax0, e2y = v2[1] - ay0, e2z = v2[2] - az0;
    double hx = ry * e2z - rz * e2y;
    double hy = rz * e2x - rx * e2z;
    double hz = rx * e2y - ry * e2x;
    double a = e1x * hx + e1y * hy + e1z * hz;
    if (-eps < a && a < eps) return 0;
    double f = 1.0 / a;
    double px = sx - ax0, py = sy - ay0, pz = sz - az0;
    double u = f * (px * hx + py * hy + pz * hz);
    if (u < 0.0 || u > 1.0) return 0;
    double qx = py * e1z - pz * e1y;
    double qy = pz * e1x - px * e1z;
    double qz = px * e1y - py * e1x;
    double v = f * (rx * qx + ry * qy + rz * qz);
    if (v < 0.0 || u + v > 1.0) return 0;
    double t = f * (e2x * qx + e2y * qy + e2z * qz);
    if (t <= eps || t >= d_len) return 0;
    point[0] = sx + t * rx; point[1] = sy + t * ry; point[2] = sz + t * rz;
    return 1;
}

static double plane_side(const double *p, const double *o, const double *n) {
    return (p[0] - o[0]) * n[0] + (p[1] - o[1]) * n[1] + (p[2] - o[2]) * n[2];
}

/* collision._offsets_for_hit (collision.py:149-171) */
static void sol_offset(const double *p, const double *hit, const double *fn, double sign,
                       double margin, double *out) {
    double nx = fn[0] * sign, ny = fn[1] * sign, nz = fn[2] * sign;
    double depth = -((p[0] - hit[0]) * nx + (p[1] - hit[1]) * ny + (p[2] - hit[2]) * nz);
    if (depth < 0.0) depth = 0.0;
    double scale = depth + margin;
    out[0] = nx * scale; out[1] = ny * scale; out[2] = nz * scale;
}

typedef struct { i64 node, tri; double off[3]; } sol_contact;
typedef struct { sol_contact *v; i64 n, cap; i64 hits; } sol_list;

static void list_push(sol_list *l, i64 node, i64 tri, const double *off) {
    if (l->n == l->cap) {
        l->cap = l->cap ? 2 * l->cap : 64;
        l->v = (sol_contact *)realloc(l->v, sizeof(sol_contact) * l->cap);
    }
    l->v[l->n].node = node;
    l->v[l->n].tri = tri;
    memcpy(l->v[l->n].off, off, sizeof(double) * 3);
    l->n++;
}

/* optional (node, obstacle triangle) log of the contacts of or_sol_detect,
 * in the solver's order (collision.py:218-240 Contact.nodes per hit) */
static i32 *g_clog = NULL;
static i64 g_clog_cap = 0, g_clog_n = 0;
OR_EXPORT void or_sol_contact_log(i32 *buf, i64 cap) {
    g_clog = buf;
    g_clog_cap = cap;
    g_clog_n = 0;
}
OR_EXPORT i64 or_sol_contact_count(void) { return g_clog_n; }
static void clog_push(i64 node, i64 tri) {
    if (g_clog && g_clog_n < g_clog_cap) {
        g_clog[2 * g_clog_n] = (i32)node;
        g_clog[2 * g_clog_n + 1] = (i32)tri;
    }
    g_clog_n++;
}

/* collision.detect_all (collision.py:243-315): every unique cloth edge vs
 * every obstacle triangle, then every obstacle edge (3t+slot) vs every cloth
 * triangle.  Contacts are applied to acc/count in exactly the serial order
 * (chunks are replayed in order), so the f64 sums are bit-identical to the
 * Python loop for any thread count.  Returns the hit count. */
OR_EXPORT i64 or_sol_detect(i64 n, const double *pos, i64 ne, const i32 *edges, i64 nc,
                            const i32 *ctris, i64 nt, const double *overt, const i32 *otris,
                            const double *onorm, double eps, double margin, double *acc,
                            i64 *count) {
    int nth = g_threads;
    i64 hits = 0;
    g_clog_n = 0;
    for (i64 i = 0; i < 3 * n; ++i) acc[i] = 0.0;
    for (i64 i = 0; i < n; ++i) count[i] = 0;
    /* pass A: cloth edges vs obstacle triangles */
    {
        int chunks = nth;
        sol_list *lists = (sol_list *)calloc(chunks, sizeof(sol_list));
#pragma omp parallel for num_threads(nth) schedule(static, 1)
        for (int ch = 0; ch < chunks; ++ch) {
            i64 lo = ne * ch / chunks, hi = ne * (ch + 1) / chunks;
            sol_list *L = &lists[ch];
            for (i64 e = lo; e < hi; ++e) {
                const double *pa = pos + 3 * (i64)edges[2 * e], *pb = pos + 3 * (i64)edges[2 * e + 1];
                for (i64 t = 0; t < nt; ++t) {
                    const i32 *tri = otris + 3 * t;
                    double hit[3];
                    if (!sol_mt(pa, pb, overt + 3 * (i64)tri[0], overt + 3 * (i64)tri[1],
                                overt + 3 * (i64)tri[2], eps, hit))
                        continue;
                    const double *fn = onorm + 3 * t;
                    double sa = plane_side(pa, hit, fn), sb = plane_side(pb, hit, fn);
                    double mx = (sb > sa) ? sb : sa; /* python max(a, b) */
                    double sign = mx >= 0.0 ? 1.0 : -1.0;
                    double off[3];
                    L->hits++;
                    sol_offset(pa, hit, fn, sign, margin, off);
                    list_push(L, edges[2 * e], t, off);
                    sol_offset(pb, hit, fn, sign, margin, off);
                    list_push(L, edges[2 * e + 1], t, off);
                }
            }
        }
        for (int ch = 0; ch < chunks; ++ch) {
            sol_list *L = &lists[ch];
            for (i64 q = 0; q < L->n; ++q) {
                i64 nd = L->v[q].node;
                for (int d = 0; d < 3; ++d) acc[3 * nd + d] += L->v[q].off[d];
                count[nd] += 1;
                clog_push(nd, L->v[q].tri);
            }
            hits += L->hits;
            free(L->v);
        }
        free(lists);
    }
    /* pass B: obstacle triangle edges vs cloth triangles */
    {
        int chunks = nth;
        sol_list *lists = (sol_list *)calloc(chunks, sizeof(sol_list));
#pragma omp parallel for num_threads(nth) schedule(static, 1)
        for (int ch = 0; ch < chunks; ++ch) {
            i64 lo = nt * ch / chunks, hi = nt * (ch + 1) / chunks;
            sol_list *L = &lists[ch];
            for (i64 t = lo; t < hi; ++t) {
                const i32 *tri = otris + 3 * t;
                const double *fn = onorm + 3 * t;
                for (int slot = 0; slot < 3; ++slot) {
                    const double *ea = overt + 3 * (i64)tri[slot];
                    const double *eb = overt + 3 * (i64)tri[(slot + 1) % 3];
                    for (i64 c = 0; c < nc; ++c) {
                        const i32 *ct = ctris + 3 * c;
                        const double *c0 = pos + 3 * (i64)ct[0], *c1 = pos + 3 * (i64)ct[1],
                                     *c2 = pos + 3 * (i64)ct[2];
                        double hit[3];
                        if (!sol_mt(ea, eb, c0, c1, c2, eps, hit)) continue;
                        /* sum(generator) starts from int 0 */
                        double total = 0.0;
                        total = total + plane_side(c0, hit, fn);
                        total = total + plane_side(c1, hit, fn);
                        total = total + plane_side(c2, hit, fn);
                        double sign = total >= 0.0 ? 1.0 : -1.0;
                        double off[3];
                        L->hits++;
                        sol_offset(c0, hit, fn, sign, margin, off);
                        list_push(L, ct[0], t, off);
                        sol_offset(c1, hit, fn, sign, margin, off);
                        list_push(L, ct[1], t, off);
                        sol_offset(c2, hit, fn, sign, margin, off);
                        list_push(L, ct[2], t, off);
                    }
                }
            }
        }
        for (int ch = 0; ch < chunks; ++ch) {
            sol_list *L = &lists[ch];
            for (i64 q = 0; q < L->n; ++q) {
                i64 nd = L->v[q].node;
                for (int d = 0; d < 3; ++d) acc[3 * nd + d] += L->v[q].off[d];
                count[nd] += 1;
                clog_push(nd, L->v[q].tri);
            }
            hits += L->hits;
            free(L->v);
        }
        free(lists);
    }
    return hits;
}

/* collision.apply_collision_response (collision.py:318-346) */
OR_EXPORT i64 or_sol_respond(i64 n, double *pos, double *vel, double *acc, i64 *count,
                             const uint8_t *pinned, int average) {
    i64 responded = 0;
    for (i64 i = 0; i < n; ++i) {
        if (count[i] > 0 && !(pinned && pinned[i])) {
            for (int d = 0; d < 3; ++d) {
                vel[3 * i + d] *= -0.5;
                double off = acc[3 * i + d];
                if (average) off = off / (double)count[i];
                pos[3 * i + d] += off;
            }
            responded++;
        }
    }
    memset(acc, 0, sizeof(double) * 3 * n);
    memset(count, 0, sizeof(i64) * n);
    return responded;
}

/* mesh.compute_face_normals (mesh.py:390-401) */
OR_EXPORT void or_sol_face_normals(i64 nt, const double *v, const i32 *tris, double *out) {
    for (i64 t = 0; t < nt; ++t) {
        const double *a = v + 3 * (i64)tris[3 * t], *b = v + 3 * (i64)tris[3 * t + 1],
                     *c = v + 3 * (i64)tris[3 * t + 2];
        double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
        double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
        double nx = e1[1] * e2[2] - e1[2] * e2[1];
        double ny = e1[2] * e2[0] - e1[0] * e2[2];
        double nz = e1[0] * e2[1] - e1[1] * e2[0];
        double len = sqrt(nx * nx + ny * ny + nz * nz);
        if (len > 1e-30) {
            out[3 * t] = nx / len; out[3 * t + 1] = ny / len; out[3 * t + 2] = nz / len;
        } else {
            out[3 * t] = 0.0; out[3 * t + 1] = 1.0; out[3 * t + 2] = 0.0;
        }
    }
}

/* mesh.compute_vertex_normals (mesh.py:404-434): face normals, zero-area
 * faces dropped, np.add.at per corner (corner 0 over all faces, then 1, 2). */
OR_EXPORT void or_sol_vertex_normals(i64 n, i64 nt, const i32 *tris, const double *pos,
                                     double *out) {
    double *fn = (double *)malloc(sizeof(double) * 3 * nt);
    or_sol_face_normals(nt, pos, tris, fn);
    double *accum = (double *)calloc(3 * n, sizeof(double));
    for (i64 t = 0; t < nt; ++t) {
        const double *a = pos + 3 * (i64)tris[3 * t], *b = pos + 3 * (i64)tris[3 * t + 1],
                     *c = pos + 3 * (i64)tris[3 * t + 2];
        double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
        double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
        double nx = e1[1] * e2[2] - e1[2] * e2[1];
        double ny = e1[2] * e2[0] - e1[0] * e2[2];
        double nz = e1[0] * e2[1] - e1[1] * e2[0];
        double area2 = sqrt(nx * nx + ny * ny + nz * nz);
        if (!(area2 > 1e-30)) fn[3 * t] = fn[3 * t + 1] = fn[3 * t + 2] = 0.0;
    }
    for (int corner = 0; corner < 3; ++corner)
        for (i64 t = 0; t < nt; ++t) {
            i64 v = tris[3 * t + corner];
            for (int d = 0; d < 3; ++d) accum[3 * v + d] += fn[3 * t + d];
        }
    for (i64 i = 0; i < n; ++i) {
        double x = accum[3 * i], y = accum[3 * i + 1], z = accum[3 * i + 2];
        double len = sqrt(x * x + y * y + z * z);
        if (len > 1e-30) {
            out[3 * i] = x / len; out[3 * i + 1] = y / len; out[3 * i + 2] = z / len;
        } else {
            out[3 * i] = 0.0; out[3 * i + 1] = 1.0; out[3 * i + 2] = 0.0;
        }
    }
    free(fn);
    free(accum);
}

/* ======================================================================= */
/* float32 engine semantics: clothsim/gpu/kernels.py + fixedpoint.py        */
/* ======================================================================= */

#define FIXED_SAT 2147483520.0

/* fixedpoint.encode_values (fixedpoint.py:28-41), float32=True */
static inline i32 enc(float x, float scale_f) {
    float prod = x * scale_f;
    double r = (double)rintf(prod);
    if (isnan(r)) return 0; /* numpy: nan -> int64 min -> int32 0 */
    if (r > FIXED_SAT) r = FIXED_SAT;
    if (r < -FIXED_SAT) r = -FIXED_SAT;
    return (i32)(i64)r;
}
/* fixedpoint.decode_values (fixedpoint.py:44-47), float32=True */
static inline float dec(i32 raw, double scale) { return (float)((double)raw / scale); }
static inline void wrap_add(i32 *p, i32 v) { *p = (i32)((uint32_t)*p + (uint32_t)v); }

OR_EXPORT i32 or_encode(float x, float scale_f) { return enc(x, scale_f); }
OR_EXPORT float or_decode(i32 raw, double scale) { return dec(raw, scale); }

static inline float dot3f(const float *a, const float *b) {
    float p0 = a[0] * b[0], p1 = a[1] * b[1], p2 = a[2] * b[2];
    return (p0 + p1) + p2;
}

/* kernel_spring_force (kernels.py:86-110): per spring, encode once, add to a
 * and the negated integer to b.  Integer adds => order independent. */
OR_EXPORT void or_eng_spring_force(i64 n, i64 ns, const i32 *sidx, const float *rest,
                                   const float *stiff, const float *damp, const float *pos,
                                   const float *vel, float scale_f, i32 *forces) {
    memset(forces, 0, sizeof(i32) * 3 * n);
    for (i64 s = 0; s < ns; ++s) {
        i64 a = sidx[2 * s], b = sidx[2 * s + 1];
        float delta[3], dv[3], axis[3];
        for (int d = 0; d < 3; ++d) delta[d] = pos[3 * b + d] - pos[3 * a + d];
        float length = sqrtf(dot3f(delta, delta));
        int ok = length > 1e-12f;
        float safe = ok ? length : 1.0f;
        for (int d = 0; d < 3; ++d) axis[d] = delta[d] / safe;
        for (int d = 0; d < 3; ++d) dv[d] = vel[3 * b + d] - vel[3 * a + d];
        float rel = dot3f(dv, axis);
        float mag = stiff[s] * (length - rest[s]) + damp[s] * rel;
        if (!ok) mag = 0.0f;
        for (int d = 0; d < 3; ++d) {
            i32 e = enc(mag * axis[d], scale_f);
            wrap_add(&forces[3 * a + d], e);
            wrap_add(&forces[3 * b + d], (i32)(0u - (uint32_t)e));
        }
    }
}

/* kernel_integrate (kernels.py:113-133) */
OR_EXPORT void or_eng_integrate(i64 n, float *pos, float *prev, float *vel, const i32 *forces,
                                const float *inv_mass, const float *ext, const float *g, float dt,
                                double scale, int explicit_euler) {
    memcpy(prev, pos, sizeof(float) * 3 * n);
    for (i64 i = 0; i < n; ++i) {
        if (!(inv_mass[i] > 0.0f)) continue;
        for (int d = 0; d < 3; ++d) {
            float F = dec(forces[3 * i + d], scale);
            float a = F * inv_mass[i] + g[d];
            a = a + (ext ? ext[3 * i + d] : 0.0f);
            if (explicit_euler) {
                pos[3 * i + d] += vel[3 * i + d] * dt;
                vel[3 * i + d] += a * dt;
            } else {
                vel[3 * i + d] += a * dt;
                pos[3 * i + d] += vel[3 * i + d] * dt;
            }
        }
    }
}

/* _segment_triangle_f32 (kernels.py:136-168), numpy operation order. */
static int eng_mt(const float *st, const float *en, const float *v0, const float *v1,
                  const float *v2, float eps, float *point) {
    float d[3] = {en[0] - st[0], en[1] - st[1], en[2] - st[2]};
    float d_len = sqrtf(dot3f(d, d));
    int valid = d_len > eps;
    float safe = valid ? d_len : 1.0f;
    float r[3] = {d[0] / safe, d[1] / safe, d[2] / safe};
    float e1[3] = {v1[0] - v0[0], v1[1] - v0[1], v1[2] - v0[2]};
    float e2[3] = {v2[0] - v0[0], v2[1] - v0[1], v2[2] - v0[2]};
    float h[3] = {r[1] * e2[2] - r[2] * e2[1], r[2] * e2[0] - r[0] * e2[2],
                  r[0] * e2[1] - r[1] * e2[0]};
    float a = dot3f(e1, h);
    valid = valid && (fabsf(a) >= eps);
    float safe_a = valid ? a : 1.0f;
    float f = 1.0f / safe_a;
    float s[3] = {st[0] - v0[0], st[1] - v0[1], st[2] - v0[2]};
    float u = f * dot3f(s, h);
    valid = valid && (u >= 0.0f) && (u <= 1.0f);
    float q[3] = {s[1] * e1[2] - s[2] * e1[1], s[2] * e1[0] - s[0] * e1[2],
                  s[0] * e1[1] - s[1] * e1[0]};
    float v = f * dot3f(r, q);
    valid = valid && (v >= 0.0f) && (u + v <= 1.0f);
    float t = f * dot3f(e2, q);
    valid = valid && (t > eps) && (t < d_len);
    if (valid) {
        point[0] = st[0] + t * r[0];
        point[1] = st[1] + t * r[1];
        point[2] = st[2] + t * r[2];
    }
    return valid;
}

OR_EXPORT int or_eng_segment_triangle(const float *st, const float *en, const float *v0,
                                      const float *v1, const float *v2, float eps, float *point) {
    return eng_mt(st, en, v0, v1, v2, eps, point);
}

/* np.maximum semantics (NaN propagates) */
static inline float np_maxf(float a, float b) {
    if (isnan(a) || isnan(b)) return NAN;
    return a >= b ? a : b;
}

/* _accumulate_hits (kernels.py:171-183) for one node */
static inline void eng_accumulate(i64 node, const float *p, const float *hit, const float *on,
                                  float margin, float scale_f, i32 *acc, i32 *count) {
    float dd[3] = {p[0] - hit[0], p[1] - hit[1], p[2] - hit[2]};
    float depth = -dot3f(dd, on);
    depth = np_maxf(depth, 0.0f);
    float sc = depth + margin;
    uint32_t *uacc = (uint32_t *)acc, *ucnt = (uint32_t *)count;
    for (int d = 0; d < 3; ++d) {
        uint32_t e = (uint32_t)enc(on[d] * sc, scale_f);
#pragma omp atomic
        uacc[3 * node + d] += e; /* mod 2^32: the reference's wrapping i32 atomics */
    }
#pragma omp atomic
    ucnt[node] += 1u;
}

/* padded/unpadded box overlap of kernels.py:55-78 */
static inline int box_overlap(const float *lo_a, const float *hi_a, const float *lo_b,
                              const float *hi_b) {
    return lo_a[0] <= hi_b[0] && lo_b[0] <= hi_a[0] && lo_a[1] <= hi_b[1] &&
           lo_b[1] <= hi_a[1] && lo_a[2] <= hi_b[2] && lo_b[2] <= hi_a[2];
}

/* kernel_detect_cloth_edges (kernels.py:186-237).  prefilter=1 applies the
 * reference's padded-box rejection (BOX_PAD, kernels.py:48); prefilter=0 is
 * the unfiltered WGSL semantics.  Returns the hit count. */
OR_EXPORT i64 or_eng_detect_cloth_edges(i64 ne, const i32 *edges, const float *pos, i64 nt,
                                        const float *corners /*T*9*/, const float *normals,
                                        float eps, float margin, float scale_f, float pad,
                                        int prefilter, i32 *acc, i32 *count) {
    float *tlo = (float *)malloc(sizeof(float) * 3 * nt), *thi = (float *)malloc(sizeof(float) * 3 * nt);
    for (i64 t = 0; t < nt; ++t)
        for (int d = 0; d < 3; ++d) {
            float a = corners[9 * t + d], b = corners[9 * t + 3 + d], c = corners[9 * t + 6 + d];
            float lo = fminf(fminf(a, b), c), hi = fmaxf(fmaxf(a, b), c);
            tlo[3 * t + d] = lo; thi[3 * t + d] = hi;
        }
    i64 hits = 0;
#pragma omp parallel for num_threads(g_threads) schedule(dynamic, 64) reduction(+ : hits)
    for (i64 e = 0; e < ne; ++e) {
        i64 na = edges[2 * e], nb = edges[2 * e + 1];
        const float *st = pos + 3 * na, *en = pos + 3 * nb;
        float lo[3], hi[3];
        for (int d = 0; d < 3; ++d) {
            lo[d] = fminf(st[d], en[d]) - pad;
            hi[d] = fmaxf(st[d], en[d]) + pad;
        }
        for (i64 t = 0; t < nt; ++t) {
            if (prefilter && !box_overlap(lo, hi, tlo + 3 * t, thi + 3 * t)) continue;
            float pt[3];
            const float *c = corners + 9 * t;
            if (!eng_mt(st, en, c, c + 3, c + 6, eps, pt)) continue;
            hits++;
            const float *nrm = normals + 3 * t;
            float da[3] = {st[0] - pt[0], st[1] - pt[1], st[2] - pt[2]};
            float db[3] = {en[0] - pt[0], en[1] - pt[1], en[2] - pt[2]};
            float side_a = dot3f(da, nrm), side_b = dot3f(db, nrm);
            float sign = np_maxf(side_a, side_b) >= 0.0f ? 1.0f : -1.0f;
            float on[3] = {nrm[0] * sign, nrm[1] * sign, nrm[2] * sign};
            eng_accumulate(na, st, pt, on, margin, scale_f, acc, count);
            eng_accumulate(nb, en, pt, on, margin, scale_f, acc, count);
        }
    }
    free(tlo);
    free(thi);
    return hits;
}

/* kernel_detect_obstacle_edges (kernels.py:240-290) */
OR_EXPORT i64 or_eng_detect_obstacle_edges(i64 nt, const float *corners, const float *normals,
                                           i64 nc, const i32 *ctris, const float *pos, float eps,
                                           float margin, float scale_f, float pad, int prefilter,
                                           i32 *acc, i32 *count) {
    float *clo = (float *)malloc(sizeof(float) * 3 * nc), *chi = (float *)malloc(sizeof(float) * 3 * nc);
    for (i64 c = 0; c < nc; ++c)
        for (int d = 0; d < 3; ++d) {
            float a = pos[3 * (i64)ctris[3 * c] + d], b = pos[3 * (i64)ctris[3 * c + 1] + d],
                  cc = pos[3 * (i64)ctris[3 * c + 2] + d];
            clo[3 * c + d] = fminf(fminf(a, b), cc);
            chi[3 * c + d] = fmaxf(fmaxf(a, b), cc);
        }
    i64 hits = 0;
#pragma omp parallel for num_threads(g_threads) schedule(dynamic, 16) reduction(+ : hits)
    for (i64 e = 0; e < 3 * nt; ++e) {
        i64 t = e / 3;
        int slot = (int)(e % 3);
        const float *st = corners + 9 * t + 3 * slot;
        const float *en = corners + 9 * t + 3 * ((slot + 1) % 3);
        float lo[3], hi[3];
        for (int d = 0; d < 3; ++d) {
            lo[d] = fminf(st[d], en[d]) - pad;
            hi[d] = fmaxf(st[d], en[d]) + pad;
        }
        const float *nrm = normals + 3 * t;
        for (i64 c = 0; c < nc; ++c) {
            if (prefilter && !box_overlap(lo, hi, clo + 3 * c, chi + 3 * c)) continue;
            const i32 *ct = ctris + 3 * c;
            const float *v0 = pos + 3 * (i64)ct[0], *v1 = pos + 3 * (i64)ct[1], *v2 = pos + 3 * (i64)ct[2];
            float pt[3];
            if (!eng_mt(st, en, v0, v1, v2, eps, pt)) continue;
            hits++;
            float d0[3] = {v0[0] - pt[0], v0[1] - pt[1], v0[2] - pt[2]};
            float d1[3] = {v1[0] - pt[0], v1[1] - pt[1], v1[2] - pt[2]};
            float d2[3] = {v2[0] - pt[0], v2[1] - pt[1], v2[2] - pt[2]};
            float total = (dot3f(d0, nrm) + dot3f(d1, nrm)) + dot3f(d2, nrm);
            float sign = total >= 0.0f ? 1.0f : -1.0f;
            float on[3] = {nrm[0] * sign, nrm[1] * sign, nrm[2] * sign};
            eng_accumulate(ct[0], v0, pt, on, margin, scale_f, acc, count);
            eng_accumulate(ct[1], v1, pt, on, margin, scale_f, acc, count);
            eng_accumulate(ct[2], v2, pt, on, margin, scale_f, acc, count);
        }
    }
    free(clo);
    free(chi);
    return hits;
}

/* kernel_respond (kernels.py:293-311) */
OR_EXPORT i64 or_eng_respond(i64 n, float *pos, float *vel, i32 *acc, i32 *count,
                             const float *inv_mass, double scale, int average) {
    i64 responded = 0;
    for (i64 i = 0; i < n; ++i) {
        if (count[i] > 0 && inv_mass[i] > 0.0f) {
            responded++;
            for (int d = 0; d < 3; ++d) {
                float dv = dec(acc[3 * i + d], scale);
                if (average) dv = dv / (float)count[i];
                vel[3 * i + d] *= -0.5f;
                pos[3 * i + d] += dv;
            }
        }
    }
    memset(acc, 0, sizeof(i32) * 3 * n);
    memset(count, 0, sizeof(i32) * n);
    return responded;
}

/* numpy's float32 pairwise summation (numpy/_core/src/umath/loops_utils.h
 * pairwise_sum), the inner loop of add.reduce / add.reduceat. */
static float np_pairwise_sum(const float *a, i64 n) {
    if (n < 8) {
        float res = 0.0f;
        for (i64 i = 0; i < n; ++i) res += a[i];
        return res;
    } else if (n <= 128) {
        float r[8];
        i64 i;
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    } else {
        i64 n2 = n / 2;
        n2 -= n2 % 8;
        return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
    }
}

/* kernel_normal_update (kernels.py:314-339) with the CSR incidence of
 * engine.py:232-242 (ascending triangle order per node). */
OR_EXPORT void or_eng_normals(i64 n, i64 nc, const i32 *tris, const float *pos,
                              const i64 *inc_off, const i64 *inc_tri, float *out) {
    float *face = (float *)malloc(sizeof(float) * 3 * nc);
    for (i64 t = 0; t < nc; ++t) {
        const float *p0 = pos + 3 * (i64)tris[3 * t], *p1 = pos + 3 * (i64)tris[3 * t + 1],
                    *p2 = pos + 3 * (i64)tris[3 * t + 2];
        float a[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
        float b[3] = {p2[0] - p0[0], p2[1] - p0[1], p2[2] - p0[2]};
        float f[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
        float nrm = sqrtf(dot3f(f, f));
        int ok = nrm > 1e-20f;
        float sn = ok ? nrm : 1.0f;
        for (int d = 0; d < 3; ++d) face[3 * t + d] = ok ? f[d] / sn : 0.0f;
    }
    for (i64 i = 0; i < n; ++i) {
        float s[3] = {0.0f, 0.0f, 0.0f};
        i64 lo = inc_off[i], hi = inc_off[i + 1];
        if (hi > lo) {
            /* np.add.reduceat on axis 0: out = first + pairwise_sum(rest) */
            float buf[4096];
            i64 m = hi - lo - 1;
            for (int d = 0; d < 3; ++d) {
                i64 mm = m < 4096 ? m : 4096;
                for (i64 q = 0; q < mm; ++q) buf[q] = face[3 * inc_tri[lo + 1 + q] + d];
                s[d] = face[3 * inc_tri[lo] + d] + np_pairwise_sum(buf, mm);
            }
        }
        float len = sqrtf(dot3f(s, s));
        if (len > 1e-20f) {
            float sl = len;
            for (int d = 0; d < 3; ++d) out[3 * i + d] = s[d] / sl;
        } else {
            out[3 * i] = 0.0f; out[3 * i + 1] = 1.0f; out[3 * i + 2] = 0.0f;
        }
    }
    free(face);
}
