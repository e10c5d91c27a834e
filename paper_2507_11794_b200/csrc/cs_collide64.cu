// cs_collide64.cu -- float64 collision, bit-identical to the reference
// solver's detect_all + apply_collision_response (collision.py:243-346).
//
// The solver tests every cloth edge against every obstacle triangle, then
// every obstacle edge (3t+slot) against every cloth triangle, in float64, and
// adds each contact's offset into acc[node] in that serial order.  Here:
//   * candidates come from the (float32) uniform grid of the obstacle, queried
//     with boxes rounded OUTWARD from the float64 geometry plus the 1e-5 pad,
//     so every pair the exact predicate could accept is tested (the grid only
//     prunes) and the dedup rule still visits each pair once;
//   * the predicate, plane sides and offsets follow collision.py's float64
//     operation order (no FMA contraction: __dmul_rn / __dadd_rn);
//   * every contact is emitted with its serial-order key, the contacts are
//     sorted by (node, key) with three stable radix passes, and one thread per
//     node sums its offsets sequentially in key order -- the same float64
//     additions, in the same order, as the Python loop.
#include "cs_collide.cuh"
#include "cs_collide64.cuh"

namespace cs {

namespace {

__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// collision.edge_triangle_intersect (collision.py:96-146), its float64 operation order
__device__ bool mt64(const double *s, const double *e, const double *v0, const double *v1,
                     const double *v2, double eps, double *point) {
    const double dx = dsub(e[0], s[0]), dy = dsub(e[1], s[1]), dz = dsub(e[2], s[2]);
    const double d_len = __dsqrt_rn(dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz)));
    if (d_len <= eps) return false;
    const double rx = __ddiv_rn(dx, d_len), ry = __ddiv_rn(dy, d_len), rz = __ddiv_rn(dz, d_len);
    const double e1x = dsub(v1[0], v0[0]), e1y = dsub(v1[1], v0[1]), e1z = dsub(v1[2], v0[2]);
    const double e2x = dsub(v2[0], v0[0]), e2y = dsub(v2[1], v0[1]), e2z = dsub(v2[2], v0[2]);
    const double hx = dsub(dmul(ry, e2z), dmul(rz, e2y));
    const double hy = dsub(dmul(rz, e2x), dmul(rx, e2z));
    const double hz = dsub(dmul(rx, e2y), dmul(ry, e2x));
    const double a = dadd(dadd(dmul(e1x, hx), dmul(e1y, hy)), dmul(e1z, hz));
    if (-eps < a && a < eps) return false;
    const double f = __ddiv_rn(1.0, a);
    const double px = dsub(s[0], v0[0]), py = dsub(s[1], v0[1]), pz = dsub(s[2], v0[2]);
    const double u = dmul(f, dadd(dadd(dmul(px, hx), dmul(py, hy)), dmul(pz, hz)));
    if (u < 0.0 || u > 1.0) return false;
    const double qx = dsub(dmul(py, e1z), dmul(pz, e1y));
    const double qy = dsub(dmul(pz, e1x), dmul(px, e1z));
    const double qz = dsub(dmul(px, e1y), dmul(py, e1x));
    const double v = dmul(f, dadd(dadd(dmul(rx, qx), dmul(ry, qy)), dmul(rz, qz)));
    if (v < 0.0 || dadd(u, v) > 1.0) return false;
    const double t = dmul(f, dadd(dadd(dmul(e2x, qx), dmul(e2y, qy)), dmul(e2z, qz)));
    if (t <= eps || t >= d_len) return false;
    point[0] = dadd(s[0], dmul(t, rx));
    point[1] = dadd(s[1], dmul(t, ry));
    point[2] = dadd(s[2], dmul(t, rz));
    return true;
}

__device__ __forceinline__ double side64(const double *p, const double *o, const double *n) {
    return dadd(dadd(dmul(dsub(p[0], o[0]), n[0]), dmul(dsub(p[1], o[1]), n[1])),
                dmul(dsub(p[2], o[2]), n[2]));
}

// collision._offsets_for_hit (collision.py:149-171)
__device__ __forceinline__ void offset64(const double *p, const double *hit, const double *fn,
                                         double sign, double margin, double *out) {
    const double n[3] = {dmul(fn[0], sign), dmul(fn[1], sign), dmul(fn[2], sign)};
    double depth = -side64(p, hit, n);
    if (depth < 0.0) depth = 0.0;
    const double scale = dadd(depth, margin);
    out[0] = dmul(n[0], scale);
    out[1] = dmul(n[1], scale);
    out[2] = dmul(n[2], scale);
}

__device__ __forceinline__ void emit(const Detect64Args &D, uint32_t node, uint32_t tri,
                                     uint64_t key, const double *off) {
    if (D.clog) {
        const uint32_t slot = atomicAdd(D.clog_n, 1u);
        if (slot < D.clog_cap) {
            D.clog[2 * slot] = node;
            D.clog[2 * slot + 1] = tri;
        }
    }
    const uint32_t k = atomicAdd(D.count, 1u);
    if (k >= D.cap) return;  // overflow: the host grows the buffers and re-runs
    D.node[k] = node;
    D.klo[k] = (uint32_t)key;
    D.khi[k] = (uint32_t)(key >> 32);
    D.off[3 * k] = off[0];
    D.off[3 * k + 1] = off[1];
    D.off[3 * k + 2] = off[2];
}

__device__ __forceinline__ void load64(const Detect64Args &D, int64_t n, double *p) {
    p[0] = D.pos[n];
    p[1] = D.pos[D.plane + n];
    p[2] = D.pos[2 * D.plane + n];
}

__device__ __forceinline__ bool box_hit(const float *la, const float *ha, const float *lb,
                                        const float *hb) {
    return (la[0] <= hb[0]) & (lb[0] <= ha[0]) & (la[1] <= hb[1]) & (lb[1] <= ha[1]) &
           (la[2] <= hb[2]) & (lb[2] <= ha[2]);
}

// float32 box that contains the float64 points, widened by `pad`
__device__ __forceinline__ void outward_box(const double *const *pts, int n, float pad, float *lo,
                                            float *hi) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double mn = pts[0][d], mx = pts[0][d];
        for (int k = 1; k < n; ++k) {
            mn = fmin(mn, pts[k][d]);
            mx = fmax(mx, pts[k][d]);
        }
        lo[d] = __fsub_rd(__double2float_rd(mn), pad);
        hi[d] = __fadd_ru(__double2float_ru(mx), pad);
    }
}

template <int PASS>
__global__ void __launch_bounds__(128)
k_detect64(const Detect64Args D, const GridDesc g, const uint32_t *__restrict__ cbeg,
           const uint32_t *__restrict__ cend, const uint32_t *__restrict__ ctri,
           const float *__restrict__ tbox, const int32_t *__restrict__ items, int64_t nq,
           unsigned long long *frame_hits) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const int nv = PASS == 0 ? 2 : 3;
    double v[3][3];
    int64_t nid[3];
    for (int k = 0; k < nv; ++k) {
        nid[k] = items[nv * q + k];
        load64(D, nid[k], v[k]);
    }
    const double *pts[3] = {v[0], v[1], v[2]};
    float lo[3], hi[3];
    outward_box(pts, nv, PASS == 0 ? D.pad : 2.0f * D.pad, lo, hi);
    if (!g.overlaps(lo, hi)) return;
    int a[3], b[3];
    g.cell_range(lo, hi, a, b);
    unsigned long long hits = 0;
    for (int z = a[2]; z <= b[2]; ++z)
        for (int y = a[1]; y <= b[1]; ++y)
            for (int x = a[0]; x <= b[0]; ++x) {
                const uint32_t key = g.key(x, y, z);
                const uint32_t c1 = cend[key];
                for (uint32_t r = cbeg[key]; r < c1; ++r) {
                    const uint32_t t = ctri[r];
                    const float *tb = tbox + 6 * (int64_t)t;
                    const float tlo[3] = {tb[0], tb[1], tb[2]}, thi[3] = {tb[3], tb[4], tb[5]};
                    if (!box_hit(lo, hi, tlo, thi)) continue;
                    if (g.cell_of(fmaxf(lo[0], tlo[0]), 0) != x ||
                        g.cell_of(fmaxf(lo[1], tlo[1]), 1) != y ||
                        g.cell_of(fmaxf(lo[2], tlo[2]), 2) != z)
                        continue;  // dedup: counted in the cell of the intersection's min corner
                    const double *cr = D.corners + 9 * (int64_t)t;
                    const double *fn = D.normals + 3 * (int64_t)t;
                    if (PASS == 0) {
                        double hit[3];
                        if (!mt64(v[0], v[1], cr, cr + 3, cr + 6, D.eps, hit)) continue;
                        const double sa = side64(v[0], hit, fn), sb = side64(v[1], hit, fn);
                        const double mx = sb > sa ? sb : sa;  // python max(a, b)
                        const double sign = mx >= 0.0 ? 1.0 : -1.0;
                        ++hits;
                        const uint64_t base = ((uint64_t)q * (uint64_t)D.nt + t) * 2u;
                        double off[3];
                        offset64(v[0], hit, fn, sign, D.margin, off);
                        emit(D, (uint32_t)nid[0], t, base, off);
                        offset64(v[1], hit, fn, sign, D.margin, off);
                        emit(D, (uint32_t)nid[1], t, base + 1, off);
                    } else {
                        for (int slot = 0; slot < 3; ++slot) {
                            const double *ea = cr + 3 * slot;
                            const double *eb = cr + 3 * (slot == 2 ? 0 : slot + 1);
                            double hit[3];
                            if (!mt64(ea, eb, v[0], v[1], v[2], D.eps, hit)) continue;
                            // sum(generator) starts from int 0
                            double total = 0.0;
                            total = dadd(total, side64(v[0], hit, fn));
                            total = dadd(total, side64(v[1], hit, fn));
                            total = dadd(total, side64(v[2], hit, fn));
                            const double sign = total >= 0.0 ? 1.0 : -1.0;
                            ++hits;
                            const uint64_t base =
                                (1ull << 63) |
                                ((((uint64_t)t * 3u + slot) * (uint64_t)D.nc + (uint64_t)q) * 4u);
                            double off[3];
                            for (int k = 0; k < 3; ++k) {
                                offset64(v[k], hit, fn, sign, D.margin, off);
                                emit(D, (uint32_t)nid[k], t, base + k, off);
                            }
                        }
                    }
                }
            }
    if (hits) atomicAdd(frame_hits, hits);
}

__global__ void k_iota(uint32_t n, uint32_t *idx) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) idx[i] = i;
}

__global__ void k_gather_key(uint32_t n, const uint32_t *__restrict__ src,
                             const uint32_t *__restrict__ idx, uint32_t *__restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = src[idx[i]];
}

// one thread per node segment of the (node, key)-sorted contacts:
// acc = ((0 + o_1) + o_2) + ..., then apply_collision_response (collision.py:318-346)
__global__ void k_respond64(uint32_t n, const uint32_t *__restrict__ snode,
                            const uint32_t *__restrict__ idx, const double *__restrict__ off,
                            double *__restrict__ state, int64_t plane,
                            const uint8_t *__restrict__ pinned, int average,
                            unsigned long long *frame_responded) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (i > 0 && snode[i] == snode[i - 1])) return;
    const uint32_t node = snode[i];
    double acc[3] = {0.0, 0.0, 0.0};
    int64_t cnt = 0;
    for (uint32_t j = i; j < n && snode[j] == node; ++j) {
        const uint32_t c = idx[j];
        acc[0] = dadd(acc[0], off[3 * c]);
        acc[1] = dadd(acc[1], off[3 * c + 1]);
        acc[2] = dadd(acc[2], off[3 * c + 2]);
        ++cnt;
    }
    if (pinned && pinned[node]) return;
    for (int d = 0; d < 3; ++d) {
        double *vel = state + (3 + d) * plane + node;
        double *pos = state + d * plane + node;
        *vel = dmul(*vel, -0.5);
        double o = acc[d];
        if (average) o = __ddiv_rn(o, (double)cnt);
        *pos = dadd(*pos, o);
    }
    atomicAdd(frame_responded, 1ull);
}

inline unsigned blocks_for(int64_t n, int b) { return (unsigned)((n + b - 1) / b); }

}  // namespace

int Contacts64::reserve(int64_t want) {
    if (want <= cap) return 0;
    release();
    cap = want;
    cudaError_t e = cudaSuccess;
    e = e ? e : cudaMalloc(&node, cap * sizeof(uint32_t));
    e = e ? e : cudaMalloc(&klo, cap * sizeof(uint32_t));
    e = e ? e : cudaMalloc(&khi, cap * sizeof(uint32_t));
    e = e ? e : cudaMalloc(&off, 3 * cap * sizeof(double));
    for (int k = 0; k < 4; ++k) e = e ? e : cudaMalloc(&sort[k], cap * sizeof(uint32_t));
    if (!count) e = e ? e : cudaMalloc(&count, sizeof(uint32_t));
    return e == cudaSuccess ? 0 : -1;
}

void Contacts64::release() {
    cudaFree(node);
    cudaFree(klo);
    cudaFree(khi);
    cudaFree(off);
    for (int k = 0; k < 4; ++k) cudaFree(sort[k]), sort[k] = nullptr;
    node = klo = khi = nullptr;
    off = nullptr;
    cap = 0;
}

void launch_detect64(Contacts64 &C, const Detect64Args &D0, const BroadPhase &bp,
                     const int32_t *edges, int64_t ne, const int32_t *tris, int64_t nc,
                     unsigned long long *frame_hits, cudaStream_t st) {
    Detect64Args D = D0;
    D.node = C.node;
    D.klo = C.klo;
    D.khi = C.khi;
    D.off = C.off;
    D.count = C.count;
    D.cap = (uint32_t)C.cap;
    cudaMemsetAsync(C.count, 0, sizeof(uint32_t), st);
    if (ne > 0)
        k_detect64<0><<<blocks_for(ne, 128), 128, 0, st>>>(D, bp.grid, bp.cell_begin, bp.cell_end,
                                                            bp.cell_tris, bp.tri_box, edges, ne,
                                                            frame_hits);
    if (nc > 0)
        k_detect64<1><<<blocks_for(nc, 128), 128, 0, st>>>(D, bp.grid, bp.cell_begin, bp.cell_end,
                                                            bp.cell_tris, bp.tri_box, tris, nc,
                                                            frame_hits);
}

void launch_respond64(Contacts64 &C, uint32_t n, int node_bits, double *state, int64_t plane,
                      const uint8_t *pinned, int average, unsigned long long *frame_responded,
                      cudaStream_t st) {
    if (n == 0) return;
    DeviceScratch scratch;
    uint32_t *keys = C.sort[0], *idx = C.sort[1], *tk = C.sort[2], *tv = C.sort[3];
    // stable LSD: key low word, key high word, node -> order by (node, key)
    k_iota<<<blocks_for(n, 256), 256, 0, st>>>(n, idx);
    cudaMemcpyAsync(keys, C.klo, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
    radix_sort_pairs(keys, idx, tk, tv, n, 32, scratch, st);
    k_gather_key<<<blocks_for(n, 256), 256, 0, st>>>(n, C.khi, idx, keys);
    radix_sort_pairs(keys, idx, tk, tv, n, 32, scratch, st);
    k_gather_key<<<blocks_for(n, 256), 256, 0, st>>>(n, C.node, idx, keys);
    radix_sort_pairs(keys, idx, tk, tv, n, node_bits, scratch, st);
    k_respond64<<<blocks_for(n, 256), 256, 0, st>>>(n, keys, idx, C.off, state, plane, pinned,
                                                    average, frame_responded);
    cudaStreamSynchronize(st);  // the scratch is released on return
}

}  // namespace cs
