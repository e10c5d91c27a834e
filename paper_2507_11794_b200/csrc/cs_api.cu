// cs_api.cu -- the C ABI (include/clothsim_b200.h): engine construction,
// frame sequencing and CUDA-graph replay, host <-> device transfers.
//
// Mirrors gpu/engine.py:108-394 (Engine): construction bakes the cloth and
// obstacle into device buffers (engine.py:193-244), a frame submits
//   [spring_force+integrate] x substeps -> detect A -> detect B -> respond
//   -> normals                                           (engine.py:304-344)
// and readbacks return copies in the reference's (N,3) layouts.
#include <cuda.h>
#include <cuda_runtime.h>
#include <climits>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/clothsim_b200.h"
#include "cs_collide.cuh"
#include "cs_collide64.cuh"
#include "cs_common.cuh"
#include "cs_kernels.cuh"


using namespace cs;

namespace cs {  // cs_gridgen.cu
cudaError_t grid_positions(int nx, int ny, int row0, int rows, double width, double height,
                           int orient, int64_t pitch, int64_t plane, float *state, double *pos64,
                           cudaStream_t st);
cudaError_t grid_rest6(int nx, int ny, int row0, int rows, double width, double height,
                       float rest6[6], bool *uniform, cudaStream_t st);
cudaError_t grid_topology(int nx, int ny, int row0, int rows, double width, double height,
                          int32_t *springs, int32_t *kinds, double *rest, int32_t *tris,
                          double *pos64, cudaStream_t st);
}  // namespace cs

// a grid engine generated on the device (cs_create_grid): the global grid,
// the local rows, the uniform inverse mass and the pinned global rows
struct GridGen {
    int nx, ny, row0;
    double width, height;
    int orient;
    float inv_mass;
    std::vector<int> pinned_rows;
};

static thread_local std::string g_err;

static int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CK(call)                                                                      \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess)                                                        \
            return fail(CS_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <typename T>
static cudaError_t dalloc(T **p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    return cudaMalloc((void **)p, count * sizeof(T));
}

struct cs_engine {
    uint32_t flags = 0;
    bool grid = false, fixed = false, fp64 = false, use_graph = true;
    int64_t N = 0, nx = 0, rows = 0, pitch = 0, plane = 0;
    cudaStream_t st = nullptr;
    bool own_stream = false;
    int num_sms = 148;
    int device = 0;  // the CUDA device the engine's buffers live on
    int substeps = 1;
    bool average = true;

    void *state[2] = {nullptr, nullptr};
    int cur = 0;
    size_t esz = 4;
    void *normals = nullptr;
    uint32_t *pinbits = nullptr;
    float *inv_mass = nullptr;     // CSR f32 path
    double *mass64 = nullptr;      // f64 path
    uint8_t *pinned8 = nullptr;
    void *ext = nullptr;
    bool has_ext = false;
    int32_t *forces_raw = nullptr;
    bool forces_valid = false;

    int64_t *csr_off = nullptr;
    int32_t *csr_nbr = nullptr;
    uint8_t *csr_kind = nullptr;
    float *csr_rest = nullptr;
    double *csr_rest64 = nullptr;
    int64_t *inc_off = nullptr;
    int32_t *inc_tri = nullptr;
    void *face = nullptr;
    int32_t *tris_g = nullptr;     // triangles in storage indices
    int32_t *edges_g = nullptr;
    int64_t nc = 0, ne = 0, nt = 0;

    bool has_obstacle = false;
    bool strip = true;          // grid path uses the warp-strip kernel (cs_strip.cu)
    // The strip kernel can compute the previous frame's normals in the same
    // pass (fused: one launch per frame, 60 B/node) or a stand-alone normals
    // kernel can follow it (split: 72 B/node).  Measured on B200 with
    // k_pair3: fused 24.6 vs split 26.6 us at C2 (640K nodes) and 297.5 vs
    // 315.5 us at C5 (16.8M) -- fused is the default at every size;
    // CS_FLAG_SPLIT_NORMALS forces the split pair (k_pair3 + k_pair_normals).
    bool fuse_normals() const {
        if (!(grid && strip)) return false;
        if (flags & CS_FLAG_SPLIT_NORMALS) return false;
        // the reference-exact paired kernel integrates only: its frame runs
        // the exact normals kernel after it (fused into the step kernel the
        // exact normals made the C2 frame slower, 59.8 vs 55.9 us)
        if (fixed && (flags & CS_FLAG_PAIRED)) return false;
        return true;
    }
    // The exact paired frame's normals kernel (split, see above) computes the
    // normals of the frame's starting state on a forked stream, concurrently
    // with the force pass that reads the same state: both kernels are
    // latency-bound with issue slots to spare.  The buffer then trails by one
    // frame like the fused one (refreshed when read).  CS_NRM_OVERLAP=0
    // restores the serial order.
    bool lag_normals() const {
        if (fuse_normals() || banded || !(grid && strip && fixed && (flags & CS_FLAG_PAIRED)))
            return false;
        static int on = -1;  // read once
        if (on < 0) {
            const char *e = getenv("CS_NRM_OVERLAP");
            on = !(e && e[0] == '0');
        }
        return on != 0;
    }
    bool normals_lagged() const { return fuse_normals() || lag_normals(); }
    cudaStream_t nrm_st = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_nrm = nullptr;
    bool normals_stale = false; // normals buffer holds the previous frame's (fused)
    float *corners = nullptr, *onormals = nullptr;
    BroadPhase bp;
    // float64 solver-exact collision (cs_collide64.cu)
    double *corners64 = nullptr, *onormals64 = nullptr;
    double eps64 = 1e-6, margin64 = 1e-3;
    Contacts64 c64;
    uint32_t c64_n = 0;
    int32_t *acc = nullptr, *count = nullptr;
    uint32_t *touched = nullptr, *touched_n = nullptr, *respond_done = nullptr;
    // [frame_hits, frame_responded, hit_counter, frame_counter, ring (2 x kRing)]
    unsigned long long *stats = nullptr;
    static constexpr int kRing = 4096;
    float eps = 1e-6f, margin = 1e-3f;

    void *stage = nullptr;
    size_t stage_bytes = 0;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    // graphs of graph_frames frames (CS_GRAPH_FRAMES, even), per start parity
    cudaGraphExec_t graphG[2] = {nullptr, nullptr};
    // optional contact log (cs_contact_log / cs_read_contacts)
    uint32_t *clog = nullptr, *clog_n = nullptr;
    int64_t clog_cap = 0;
    // cs_record: copy stream, per-parity events and device staging
    cudaStream_t copy_st = nullptr;
    cudaEvent_t ev_frame[2] = {nullptr, nullptr}, ev_moved[2] = {nullptr, nullptr};
    // cross-stream ordering of device-pointer transfers (cs_read_device /
    // cs_write_device / cs_set_stream)
    cudaEvent_t ev_join = nullptr;
    float *rec_stage[2] = {nullptr, nullptr};
    int64_t frames = 0;
    // row band (cs_set_halo_peers): neighbours' buffers + per-pass handshake
    struct Link {
        bool on = false;
        void *state[2] = {nullptr, nullptr};
        int64_t plane = 0, src_row0 = 0, dst_row0 = 0, rows = 0;
        uint32_t *remote_flag = nullptr;
    };
    bool banded = false;
    Link up, dn;
    // flag words: [0] passes the upper neighbour finished, [1] the lower one's
    // (written by them); the in-kernel handshake's [2] / [5] passes whose
    // upper / lower seam this band finished, [3] / [6] seam warps done in the
    // running launch, [4] its error word (HaloDst::flags)
    uint32_t *hflags = nullptr;
    uint32_t passes = 0;         // force passes this engine issued
    // Fast collision-free bands with fused normals do the seam handshake
    // inside k_pair3 (seam warps wait, the last block signals): frames are
    // graph-captured like a single engine's.  Otherwise (fixed arithmetic,
    // split normals, obstacles, CS_FLAG_MEMOP_SEAM) the stream waits on /
    // writes the flag words around each pass.
    bool seam_in_kernel() const {
        return banded && grid && strip && (flags & CS_FLAG_PAIRED) && !fixed && !has_obstacle &&
               fuse_normals() && !(flags & CS_FLAG_MEMOP_SEAM);
    }
    StepParams sp{};
    CsrParams cp{};

    int64_t gidx(int64_t n) const { return grid ? (n / nx) * pitch + (n % nx) : n; }
    CollideArgs cargs() const {
        CollideArgs A;
        A.pos = (const float *)state[cur];
        A.plane = plane;
        A.acc = acc;
        A.count = count;
        A.touched = touched;
        A.touched_n = touched_n;
        A.blocks_done = respond_done;
        A.frame_hits = stats;
        A.frame_responded = stats + 1;
        A.hit_counter = stats + 2;
        A.frame_counter = stats + 3;
        A.ring = stats + 4;
        A.ring_size = kRing;
        A.clog = clog;
        A.clog_n = clog_n;
        A.clog_cap = (uint32_t)clog_cap;
        A.eps = eps;
        A.margin = margin;
        A.pad = 1e-5f;  // kernels.py:48 BOX_PAD
        A.scale_f = sp.scale_f;
        A.scale_d = sp.scale_d;
        A.own_lo = banded ? (int64_t)sp.row_lo * pitch : 0;
        A.own_hi = banded ? (int64_t)sp.row_hi * pitch : INT64_MAX;
        return A;
    }
    int kernels_per_frame() const {
        int k = substeps;  // one fused force+integrate launch per substep
        // detect: both passes in one launch (fused or batched narrow phase)
        // or two; respond closes the frame in its last block
        if (has_obstacle) k += (bp.warp_per_query >= 2 ? 1 : 2) + 1;
        if (!fuse_normals()) k += grid ? 1 : 2;  // normals (else fused into the strip kernel)
        return k;
    }
};

// ---------------------------------------------------------------------------
// layout transposes: host AoS (N,3) <-> device SoA planes (pitch layout)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_aos_to_planes(int64_t N, int64_t nx, int64_t pitch, int64_t plane, int comps,
                                const T *__restrict__ aos, T *__restrict__ planes) {
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int64_t g = (n / nx) * pitch + (n % nx);
    for (int c = 0; c < comps; ++c) planes[c * plane + g] = aos[n * comps + c];
}
template <typename T>
__global__ void k_planes_to_aos(int64_t N, int64_t nx, int64_t pitch, int64_t plane, int comps,
                                const T *__restrict__ planes, T *__restrict__ aos) {
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int64_t g = (n / nx) * pitch + (n % nx);
    for (int c = 0; c < comps; ++c) aos[n * comps + c] = planes[c * plane + g];
}
// positions (3 planes, f32 or f64) -> device f64 (N,3): the snapshot's input
template <typename T>
__global__ void k_planes_to_aos64(int64_t N, int64_t nx, int64_t pitch, int64_t plane,
                                  const T *__restrict__ planes, double *__restrict__ aos) {
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int64_t g = (n / nx) * pitch + (n % nx);
    for (int c = 0; c < 3; ++c) aos[n * 3 + c] = (double)planes[c * plane + g];
}
// planes (pitch layout) <-> (N, comps) AoS with a type conversion: the
// device-pointer transfers (a float64 engine's f32 views, f32 -> f64 writes)
template <typename Ti, typename To>
__global__ void k_planes_to_aos_cvt(int64_t N, int64_t nx, int64_t pitch, int64_t plane, int comps,
                                    const Ti *__restrict__ planes, To *__restrict__ aos) {
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int64_t g = (n / nx) * pitch + (n % nx);
    for (int c = 0; c < comps; ++c) aos[n * comps + c] = (To)planes[c * plane + g];
}
template <typename Ti, typename To>
__global__ void k_aos_to_planes_cvt(int64_t N, int64_t nx, int64_t pitch, int64_t plane, int comps,
                                    const Ti *__restrict__ aos, To *__restrict__ planes) {
    const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int64_t g = (n / nx) * pitch + (n % nx);
    for (int c = 0; c < comps; ++c) planes[c * plane + g] = (To)aos[n * comps + c];
}
__global__ void k_f64_to_f32(int64_t n, const double *a, float *b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = (float)a[i];
}
__global__ void k_f32_to_f64(int64_t n, const float *a, double *b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = (double)a[i];
}
static inline unsigned nb(int64_t n) { return (unsigned)((n + 255) / 256); }

static int ensure_stage(cs_engine *h, size_t bytes) {
    if (bytes > h->stage_bytes) {
        if (h->stage) cudaFree(h->stage);
        CK(cudaMalloc(&h->stage, bytes));
        h->stage_bytes = bytes;
    }
    return 0;
}

// upload host AoS into planes (T = float / double / int32)
template <typename T>
static int upload_planes(cs_engine *h, const T *host, T *planes, int comps) {
    const size_t bytes = (size_t)h->N * comps * sizeof(T);
    if (int r = ensure_stage(h, bytes)) return r;
    CK(cudaMemcpyAsync(h->stage, host, bytes, cudaMemcpyHostToDevice, h->st));
    const int64_t nxx = h->grid ? h->nx : h->N;
    k_aos_to_planes<T><<<nb(h->N), 256, 0, h->st>>>(h->N, nxx, h->pitch, h->plane, comps,
                                                    (const T *)h->stage, planes);
    CK(cudaGetLastError());
    return 0;
}
template <typename T>
static int download_planes(cs_engine *h, const T *planes, T *host, int comps) {
    const size_t bytes = (size_t)h->N * comps * sizeof(T);
    if (int r = ensure_stage(h, bytes)) return r;
    const int64_t nxx = h->grid ? h->nx : h->N;
    k_planes_to_aos<T><<<nb(h->N), 256, 0, h->st>>>(h->N, nxx, h->pitch, h->plane, comps, planes,
                                                    (T *)h->stage);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(host, h->stage, bytes, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    return 0;
}

static void drop_graphs(cs_engine *h) {
    for (int i = 0; i < 2; ++i) {
        if (h->graph[i]) {
            cudaGraphExecDestroy(h->graph[i]);
            h->graph[i] = nullptr;
        }
        if (h->graphG[i]) {
            cudaGraphExecDestroy(h->graphG[i]);
            h->graphG[i] = nullptr;
        }
    }
}

// frames per captured graph for runs of many frames (CS_GRAPH_FRAMES, an
// even count so a graph returns to its starting state buffer; 1 = one frame
// per graph).  Inside a graph consecutive step kernels overlap launch and
// drain (programmatic dependent launch, CS_PDL in cs_pair3.cu): 8-way band
// of C5, linked, 34.9 -> 33.8 us per frame with 8 frames per graph; C2 and
// C5 unchanged (tools/ab_pdl.sh)
static int graph_frames() {
    static int g = -1;
    if (g < 0) {
        const char *e = getenv("CS_GRAPH_FRAMES");
        g = e ? atoi(e) : 8;
        if (g > 1 && (g & 1)) ++g;
        if (g < 1) g = 1;
    }
    return g;
}

// ---------------------------------------------------------------------------
// passes
// ---------------------------------------------------------------------------
static HaloDst halo_dst(const cs_engine *h, int dst);

static void pass_force_integrate(cs_engine *h, bool fuse_normals = false) {
    for (int s = 0; s < h->substeps; ++s) {
        const int src = h->cur, dst = 1 - h->cur;
        if (h->seam_in_kernel()) {  // a row band: peer stores + seam handshake in the kernel
            const HaloDst hd = halo_dst(h, dst);
            launch_strip_step(h->sp, false, fuse_normals && s == 0, (const float *)h->state[src],
                              (float *)h->state[dst], h->pinbits,
                              h->has_ext ? (const float *)h->ext : nullptr, (float *)h->normals,
                              h->st, true, &hd);
            h->cur = dst;
            continue;
        }
        if (h->fp64) {
            launch_csr_step_f64(h->cp, (const double *)h->state[src], (double *)h->state[dst],
                                h->csr_off, h->csr_nbr, h->csr_kind, h->csr_rest64, h->mass64,
                                h->pinned8, h->has_ext ? (const double *)h->ext : nullptr, h->st);
        } else if (h->grid && h->strip) {
            // normals of the frame's starting state ride along in the first substep
            launch_strip_step(h->sp, h->fixed, fuse_normals && s == 0, (const float *)h->state[src],
                              (float *)h->state[dst], h->pinbits,
                              h->has_ext ? (const float *)h->ext : nullptr, (float *)h->normals, h->st,
                              (h->flags & CS_FLAG_PAIRED) != 0);
        } else if (h->grid) {
            launch_grid_step(h->sp, h->fixed, (const float *)h->state[src], (float *)h->state[dst],
                             h->pinbits, h->has_ext ? (const float *)h->ext : nullptr, h->st);
        } else {
            launch_csr_step(h->cp, h->fixed, (const float *)h->state[src], (float *)h->state[dst],
                            h->csr_off, h->csr_nbr, h->csr_kind, h->csr_rest, h->inv_mass,
                            h->has_ext ? (const float *)h->ext : nullptr, h->st);
        }
        h->cur = dst;
    }
    h->forces_valid = true;
}

static Detect64Args detect64_args(const cs_engine *h) {
    Detect64Args D{};
    D.pos = (const double *)h->state[h->cur];
    D.plane = h->plane;
    D.corners = h->corners64;
    D.normals = h->onormals64;
    D.nt = h->nt;
    D.nc = h->nc;
    D.eps = h->eps64;
    D.margin = h->margin64;
    D.pad = 1e-5f;
    D.clog = h->clog;
    D.clog_n = h->clog_n;
    D.clog_cap = (uint32_t)h->clog_cap;
    return D;
}

static void pass_detect(cs_engine *h) {
    cudaMemsetAsync(h->stats, 0, 2 * sizeof(unsigned long long), h->st);
    if (h->clog) cudaMemsetAsync(h->clog_n, 0, sizeof(uint32_t), h->st);
    if (!h->has_obstacle) return;
    if (h->fp64) {
        // the float64 path synchronises: its contact count sizes the sort,
        // and an overflowing pass is re-run with larger buffers
        for (;;) {
            if (h->clog) cudaMemsetAsync(h->clog_n, 0, sizeof(uint32_t), h->st);
            launch_detect64(h->c64, detect64_args(h), h->bp, h->edges_g, h->ne, h->tris_g, h->nc,
                            h->stats, h->st);
            cudaMemcpyAsync(&h->c64_n, h->c64.count, sizeof(uint32_t), cudaMemcpyDeviceToHost, h->st);
            cudaStreamSynchronize(h->st);
            if (h->c64_n <= h->c64.cap) break;
            h->c64.reserve(2 * (int64_t)h->c64_n);
            cudaMemsetAsync(h->stats, 0, 2 * sizeof(unsigned long long), h->st);
        }
        return;
    }
    launch_detect(h->cargs(), h->bp, h->corners, h->onormals, h->edges_g, h->ne, h->tris_g, h->nc,
                  h->st);
}

static void pass_respond(cs_engine *h) {
    if (!h->has_obstacle) return;
    if (h->fp64) {
        int bits = 1;
        while (((int64_t)1 << bits) < h->N) ++bits;
        launch_respond64(h->c64, h->c64_n, bits, (double *)h->state[h->cur], h->plane, h->pinned8,
                         h->average ? 1 : 0, h->stats + 1, h->st);
        h->c64_n = 0;
        launch_respond_end(h->cargs(), true, h->st);
        return;
    }
    launch_respond(h->cargs(), (float *)h->state[h->cur], h->grid ? h->pinbits : nullptr,
                   h->grid ? nullptr : h->inv_mass, h->average ? 1 : 0, h->N, h->num_sms,
                   /*end_of_frame=*/true, h->st);
}

static void pass_normals(cs_engine *h, cudaStream_t st = nullptr) {
    if (st) {  // the exact paired kernel on a forked stream (cs_engine::lag_normals)
        launch_pair_normals_exact(h->sp, (const float *)h->state[h->cur], (float *)h->normals, st);
        return;
    }
    if (h->fp64) {
        launch_csr_normals_f64(h->N, h->plane, h->nc, (const double *)h->state[h->cur], h->tris_g,
                               (double *)h->face, h->inc_off, h->inc_tri, (double *)h->normals, h->st);
    } else if (h->grid && h->strip && (h->flags & CS_FLAG_PAIRED)) {
        if (h->fixed)
            launch_pair_normals_exact(h->sp, (const float *)h->state[h->cur], (float *)h->normals, h->st);
        else
            launch_pair_normals(h->sp, (const float *)h->state[h->cur], (float *)h->normals, h->st);
    } else if (h->grid) {
        launch_grid_normals(h->sp, h->fixed, (const float *)h->state[h->cur], (float *)h->normals, h->st);
    } else {
        launch_csr_normals(h->N, h->plane, h->nc, h->fixed, (const float *)h->state[h->cur],
                           h->tris_g, (float *)h->face, h->inc_off, h->inc_tri, (float *)h->normals,
                           h->st);
    }
}

// One frame (engine.py:304-344).  On the strip path the normal_update of
// frame t runs inside frame t+1's force pass; the buffer is marked stale and
// refreshed by a stand-alone normals launch only when it is read.
static void launch_frame(cs_engine *h) {
    // The fast mode fuses the normals into the step kernel.  A side-stream
    // variant (the starting state's normals beside a force-only step) lost:
    // 319.6 vs 321.6 us at 4096^2, where both kernels fill the SMs, and
    // 22.6 vs 20.5 us at C2; on an 8-way band the pieces alone are 26.7 +
    // 13.3 us against 33.4 us fused (tools/band_split.py).  The exact mode,
    // whose normals are a separate kernel anyway, does run them beside the
    // force pass (lag_normals: C2 52.1 -> 51.4 us, C5 813 -> 739 us).
    const bool fuse = h->fuse_normals(), lag = h->lag_normals();
    if (lag) {  // the starting state's normals, beside the force pass
        cudaEventRecord(h->ev_fork, h->st);
        cudaStreamWaitEvent(h->nrm_st, h->ev_fork, 0);
        pass_normals(h, h->nrm_st);
        cudaEventRecord(h->ev_nrm, h->nrm_st);
    }
    pass_force_integrate(h, fuse);
    if (h->has_obstacle) {
        pass_detect(h);
        pass_respond(h);
    }
    if (lag)
        cudaStreamWaitEvent(h->st, h->ev_nrm, 0);
    else if (!fuse)
        pass_normals(h);
    h->normals_stale = fuse || lag;
}

// ---------------------------------------------------------------------------
// row bands (BASELINE config 5): one engine per GPU holds its owned rows plus
// a 2-row halo on each side.  The step kernel itself stores each boundary row
// into the neighbour's halo (peer memory over NVLink: cudaIpc handles across
// processes, plain pointers within one); a stream-ordered handshake replaces
// the exchange step -- before force pass t an engine's stream waits until
// each neighbour has finished pass t-1 (so the halo it reads is complete and
// the buffer the neighbour writes is no longer being read), and after the
// pass it bumps its pass count in each neighbour's flag word.  No host
// synchronisation, no NCCL call and no packing kernel on the data path.
// ---------------------------------------------------------------------------
typedef CUresult (*PfnValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PfnValue32 g_wait32 = nullptr, g_write32 = nullptr;
// CU_STREAM_WAIT_VALUE_FLUSH where the device supports it: remote (peer)
// writes that reached this GPU before the flag are visible to the work the
// wait releases -- the neighbour's halo stores, for the next pass
static unsigned g_wait_flush = 0;
typedef CUresult (*PfnDevAttr)(int *, CUdevice_attribute, CUdevice);

static int load_memops() {
    if (g_wait32 && g_write32) return 0;
    cudaDriverEntryPointQueryResult q1 = cudaDriverEntryPointSymbolNotFound, q2 = q1;
    CK(cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", (void **)&g_wait32, 12000,
                                        cudaEnableDefault, &q1));
    CK(cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", (void **)&g_write32, 12000,
                                        cudaEnableDefault, &q2));
    if (q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess || !g_wait32 ||
        !g_write32) {
        g_wait32 = g_write32 = nullptr;
        return fail(CS_E_CUDA, "the driver does not provide cuStreamWaitValue32/cuStreamWriteValue32");
    }
    PfnDevAttr attr = nullptr;
    cudaDriverEntryPointQueryResult q3 = cudaDriverEntryPointSymbolNotFound;
    int dev = 0, flush = 0;
    if (cudaGetDriverEntryPointByVersion("cuDeviceGetAttribute", (void **)&attr, 12000,
                                         cudaEnableDefault, &q3) == cudaSuccess &&
        q3 == cudaDriverEntryPointSuccess && attr && cudaGetDevice(&dev) == cudaSuccess &&
        attr(&flush, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, (CUdevice)dev) == CUDA_SUCCESS &&
        flush)
        g_wait_flush = CU_STREAM_WAIT_VALUE_FLUSH;
    return 0;
}

#define CU(call)                                                                         \
    do {                                                                                 \
        CUresult r_ = (call);                                                            \
        if (r_ != CUDA_SUCCESS)                                                          \
            return fail(CS_E_CUDA, std::string(#call) + ": CUresult " + std::to_string((int)r_)); \
    } while (0)

static int halo_wait(cs_engine *h) {
    if (h->up.on)
        CU(g_wait32((CUstream)h->st, (CUdeviceptr)(h->hflags + 0), h->passes,
                    CU_STREAM_WAIT_VALUE_GEQ | g_wait_flush));
    if (h->dn.on)
        CU(g_wait32((CUstream)h->st, (CUdeviceptr)(h->hflags + 1), h->passes,
                    CU_STREAM_WAIT_VALUE_GEQ | g_wait_flush));
    return 0;
}

static int halo_signal(cs_engine *h) {
    ++h->passes;  // the default write orders the pass's (peer) stores before the flag
    if (h->up.on)
        CU(g_write32((CUstream)h->st, (CUdeviceptr)h->up.remote_flag, h->passes, CU_STREAM_WRITE_VALUE_DEFAULT));
    if (h->dn.on)
        CU(g_write32((CUstream)h->st, (CUdeviceptr)h->dn.remote_flag, h->passes, CU_STREAM_WRITE_VALUE_DEFAULT));
    return 0;
}

// neighbour planes of buffer `dst`, shifted so that local offsets address them
static HaloDst halo_dst(const cs_engine *h, int dst) {
    HaloDst d{};
    auto fill = [&](const cs_engine::Link &L, float **out) {
        for (int q = 0; q < 6; ++q) {
            if (!L.on) {
                out[q] = nullptr;
                continue;
            }
            const int64_t elems = q * L.plane + (L.dst_row0 - L.src_row0) * h->pitch;
            out[q] = (float *)((intptr_t)L.state[dst] + (intptr_t)(elems * 4));
        }
    };
    fill(h->up, d.up);
    fill(h->dn, d.dn);
    if (h->seam_in_kernel()) {
        d.flags = h->hflags;
        d.to_up = h->up.on ? h->up.remote_flag : nullptr;
        d.to_dn = h->dn.on ? h->dn.remote_flag : nullptr;
    }
    return d;
}

// the in-kernel handshake gave up waiting for a neighbour (error word)
static int seam_check(cs_engine *h) {
    if (!h->seam_in_kernel()) return 0;
    uint32_t e = 0;
    CK(cudaMemcpyAsync(&e, h->hflags + 4, sizeof(e), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (e) return fail(CS_E_CUDA, "row-band seam handshake timed out (a neighbour band stopped stepping)");
    return 0;
}

static int banded_frame(cs_engine *h) {
    const bool fuse = h->fuse_normals();
    const bool packed = (h->flags & CS_FLAG_PAIRED) != 0;
    const bool fused_push = packed;  // k_pair3 (fast or exact) stores into the peers itself
    for (int s = 0; s < h->substeps; ++s) {
        if (int r = halo_wait(h)) return r;
        if (s == 0 && !fuse) pass_normals(h);  // the frame's starting state, halo complete
        const int src = h->cur, dst = 1 - h->cur;
        const HaloDst hd = halo_dst(h, dst);
        launch_strip_step(h->sp, h->fixed, fuse && s == 0, (const float *)h->state[src],
                          (float *)h->state[dst], h->pinbits,
                          h->has_ext ? (const float *)h->ext : nullptr, (float *)h->normals, h->st,
                          packed, fused_push ? &hd : nullptr);
        if (!fused_push) {
            if (h->up.on)
                launch_push_rows((const float *)h->state[dst], h->plane, (int)h->pitch,
                                 (int)h->up.src_row0, (int)(h->up.src_row0 + h->up.rows), hd.up, h->st);
            if (h->dn.on)
                launch_push_rows((const float *)h->state[dst], h->plane, (int)h->pitch,
                                 (int)h->dn.src_row0, (int)(h->dn.src_row0 + h->dn.rows), hd.dn, h->st);
        }
        CK(cudaGetLastError());
        h->cur = dst;
        if (int r = halo_signal(h)) return r;
    }
    if (h->has_obstacle) {
        // Detection needs the neighbours' post-step boundary rows (the halo
        // now holds them), and the respond pass changes owned nodes after
        // they were sent -- so: wait, detect, signal "detect done", respond,
        // wait until the neighbours finished detecting (they read the halo
        // we are about to overwrite), push the post-respond boundary rows,
        // signal.  Each band accumulates only into its owned nodes and
        // counts only the hits of primitives whose minimum node it owns.
        if (int r = halo_wait(h)) return r;
        pass_detect(h);
        if (int r = halo_signal(h)) return r;
        pass_respond(h);
        if (int r = halo_wait(h)) return r;
        const HaloDst hd = halo_dst(h, h->cur);
        if (h->up.on)
            launch_push_rows((const float *)h->state[h->cur], h->plane, (int)h->pitch,
                             (int)h->up.src_row0, (int)(h->up.src_row0 + h->up.rows), hd.up, h->st);
        if (h->dn.on)
            launch_push_rows((const float *)h->state[h->cur], h->plane, (int)h->pitch,
                             (int)h->dn.src_row0, (int)(h->dn.src_row0 + h->dn.rows), hd.dn, h->st);
        CK(cudaGetLastError());
        if (int r = halo_signal(h)) return r;
    }
    h->forces_valid = true;
    h->normals_stale = true;  // normals trail by one frame; refreshed when read
    return 0;
}

static void flush_normals(cs_engine *h) {
    if (h->normals_stale) {
        if (h->banded) halo_wait(h);  // the neighbours' last pass completes our halo
        pass_normals(h);
        h->normals_stale = false;
    }
}

// ---------------------------------------------------------------------------
// construction
// ---------------------------------------------------------------------------
extern "C" int cs_abi_version(void) { return CS_ABI_VERSION; }
extern "C" const char *cs_last_error(void) { return g_err.c_str(); }

__global__ void k_fill_inv_mass(int64_t rows, int64_t nx, int64_t pitch, float im,
                                const uint32_t *__restrict__ pinbits, float *__restrict__ out) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= rows * nx) return;
    const int64_t g = (v / nx) * pitch + (v % nx);
    out[g] = ((pinbits[g >> 5] >> (g & 31)) & 1u) ? 0.f : im;
}

static int build(cs_engine *h, const cs_desc *d, const GridGen *gen = nullptr) {
    const int64_t N = d->num_nodes;
    h->flags = d->flags;
    h->fixed = (d->flags & CS_FLAG_FIXED_POINT) != 0;
    h->fp64 = (d->flags & CS_FLAG_FP64) != 0;
    h->use_graph = (d->flags & CS_FLAG_NO_GRAPH) == 0;
    h->average = (d->flags & CS_FLAG_AVERAGE_RESPONSE) != 0;
    h->substeps = d->substeps < 1 ? 1 : d->substeps;
    h->N = N;
    if (h->fp64 && h->fixed) return fail(CS_E_INVALID, "CS_FLAG_FP64 and CS_FLAG_FIXED_POINT are exclusive");
    if (h->fp64 && d->num_obstacle_tris > 0 && (!d->obstacle_corners64 || !d->obstacle_normals64))
        return fail(CS_E_INVALID, "float64 engines with an obstacle need obstacle_corners64/normals64");
    if (h->fp64 && (!d->masses64 || !d->pinned || !d->spring_rest64))
        return fail(CS_E_INVALID, "float64 engines need masses64, pinned and spring_rest64");

    // uniform inverse mass among free nodes => grid stencil eligible
    float im_free = gen ? gen->inv_mass : 0.f;
    bool uniform = true;
    for (int64_t i = 0; !gen && i < N; ++i) {
        const float v = d->inv_mass[i];
        if (v > 0.f) {
            if (im_free == 0.f) im_free = v;
            else if (v != im_free) { uniform = false; break; }
        }
    }
    h->strip = !(d->flags & CS_FLAG_TILE_KERNEL);
    h->grid = d->nx >= 2 && d->ny >= 2 && (int64_t)d->nx * d->ny == N && !h->fp64 && uniform &&
              !(d->flags & CS_FLAG_FORCE_CSR);
    h->esz = h->fp64 ? 8 : 4;
    if (h->grid) {
        h->nx = d->nx;
        h->rows = d->ny;
        h->pitch = (d->nx + 31) / 32 * 32;
        h->plane = h->pitch * h->rows;
    } else {
        h->nx = N;
        h->rows = 1;
        h->pitch = N;
        h->plane = N;
    }
    const int64_t P = h->plane;

    int dev = 0;
    CK(cudaGetDevice(&dev));
    h->device = dev;
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (d->stream) {
        h->st = (cudaStream_t)d->stream;
    } else {
        CK(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
        h->own_stream = true;
    }

    // ---- parameters (engine.py:246-285) ----
    StepParams &sp = h->sp;
    sp.nx = (int)h->nx;
    sp.ny = (int)h->rows;
    sp.pitch = (int)h->pitch;
    sp.plane = P;
    sp.dt = (float)d->dt;
    sp.gx = (float)d->gravity[0];
    sp.gy = (float)d->gravity[1];
    sp.gz = (float)d->gravity[2];
    sp.k_struct = (float)d->stiffness[0];
    sp.k_shear = (float)d->stiffness[1];
    sp.k_bend = (float)d->stiffness[2];
    sp.damping = (float)d->damping;
    for (int q = 0; q < 6; ++q) {
        sp.rest[q] = d->grid_rest[q];
        const double kq = q < 2 ? sp.k_struct : (q < 4 ? sp.k_shear : sp.k_bend);
        sp.nkr2[q] = (float)(-kq * (double)sp.rest[q] * (double)sp.rest[q]);
    }
    sp.inv_mass = im_free;
    sp.scale_f = (float)d->fixed_point_scale;
    sp.scale_d = (double)d->fixed_point_scale;
    sp.inv_scale_pow2 = 0.f;
    if (d->fixed_point_scale > 0 && (d->fixed_point_scale & (d->fixed_point_scale - 1)) == 0)
        sp.inv_scale_pow2 = (float)(1.0 / (double)d->fixed_point_scale);
    sp.explicit_euler = (d->flags & CS_FLAG_EXPLICIT_EULER) ? 1 : 0;
    sp.row_lo = 0;
    sp.row_hi = sp.ny;
    sp.halo_up_hi = INT_MIN;
    sp.halo_dn_lo = INT_MAX;
    CsrParams &cp = h->cp;
    cp.n = N;
    cp.plane = P;
    cp.dt = sp.dt;
    cp.gx = sp.gx; cp.gy = sp.gy; cp.gz = sp.gz;
    cp.damping = sp.damping;
    cp.scale_f = sp.scale_f;
    cp.scale_d = sp.scale_d;
    cp.k[0] = sp.k_struct; cp.k[1] = sp.k_shear; cp.k[2] = sp.k_bend;
    cp.dt_d = d->dt;
    for (int q = 0; q < 3; ++q) {
        cp.g_d[q] = d->gravity[q];
        cp.k_d[q] = d->stiffness[q];
    }
    cp.damping_d = d->damping;
    cp.explicit_euler = sp.explicit_euler;
    h->eps = d->epsilon_mt;
    h->margin = d->response_margin;

    // ---- state (ping-pong SoA planes) ----
    for (int b = 0; b < 2; ++b) {
        CK(cudaMalloc(&h->state[b], 6 * P * h->esz));
        CK(cudaMemsetAsync(h->state[b], 0, 6 * P * h->esz, h->st));
    }
    CK(cudaMalloc(&h->normals, 3 * P * h->esz));
    CK(cudaMemsetAsync(h->normals, 0, 3 * P * h->esz, h->st));
    if (h->fp64) {
        if (d->positions64) {
            if (int r = upload_planes<double>(h, d->positions64, (double *)h->state[0], 3)) return r;
        } else {
            if (int r = upload_planes<float>(h, d->positions, (float *)h->state[1], 3)) return r;
            k_f32_to_f64<<<nb(3 * P), 256, 0, h->st>>>(3 * P, (const float *)h->state[1], (double *)h->state[0]);
        }
    } else if (gen) {
        CK(grid_positions(gen->nx, gen->ny, gen->row0, (int)h->rows, gen->width, gen->height,
                          gen->orient, h->pitch, P, (float *)h->state[0], nullptr, h->st));
    } else {
        if (int r = upload_planes<float>(h, d->positions, (float *)h->state[0], 3)) return r;
    }
    CK(cudaMemcpyAsync(h->state[1], h->state[0], 6 * P * h->esz, cudaMemcpyDeviceToDevice, h->st));

    // ---- masses / pins ----
    if (h->grid) {
        const int64_t words = (P + 31) / 32;
        std::vector<uint32_t> bits(words, 0u);
        if (gen) {  // whole pinned rows (mesh.py:260-263)
            for (int j : gen->pinned_rows) {
                const int64_t lj = j - gen->row0;
                if (lj < 0 || lj >= h->rows) continue;
                for (int64_t i = 0; i < h->nx; ++i) {
                    const int64_t g = lj * h->pitch + i;
                    bits[g >> 5] |= 1u << (g & 31);
                }
            }
        } else {
            for (int64_t n = 0; n < N; ++n)
                if (!(d->inv_mass[n] > 0.f)) {
                    const int64_t g = h->gidx(n);
                    bits[g >> 5] |= 1u << (g & 31);
                }
        }
        CK(dalloc(&h->pinbits, words));
        CK(cudaMemcpyAsync(h->pinbits, bits.data(), words * 4, cudaMemcpyHostToDevice, h->st));
        CK(cudaStreamSynchronize(h->st));  // `bits` goes out of scope
    }
    CK(dalloc(&h->inv_mass, P));  // storage layout (the respond pass reads it too)
    CK(cudaMemsetAsync(h->inv_mass, 0, P * 4, h->st));
    if (gen) {
        k_fill_inv_mass<<<nb(N), 256, 0, h->st>>>(h->rows, h->nx, h->pitch, gen->inv_mass, h->pinbits,
                                                  h->inv_mass);
        CK(cudaGetLastError());
    } else if (int r = upload_planes<float>(h, d->inv_mass, h->inv_mass, 1)) {
        return r;
    }
    if (h->fp64) {
        CK(dalloc(&h->mass64, N));
        CK(dalloc(&h->pinned8, N));
        CK(cudaMemcpyAsync(h->mass64, d->masses64, N * 8, cudaMemcpyHostToDevice, h->st));
        CK(cudaMemcpyAsync(h->pinned8, d->pinned, N, cudaMemcpyHostToDevice, h->st));
    }

    // ---- spring CSR (generic / f64 paths): ascending spring id per node ----
    if (!h->grid) {
        const int64_t S = d->num_springs;
        std::vector<int64_t> off(N + 1, 0);
        for (int64_t s = 0; s < S; ++s) {
            const int32_t a = d->springs[2 * s], b = d->springs[2 * s + 1];
            if (a < 0 || a >= N || b < 0 || b >= N) return fail(CS_E_INVALID, "spring endpoint out of range");
            off[a + 1]++;
            off[b + 1]++;
        }
        for (int64_t i = 0; i < N; ++i) off[i + 1] += off[i];
        std::vector<int64_t> fill(off.begin(), off.end() - 1);
        std::vector<int32_t> nbr(2 * S);
        std::vector<uint8_t> kind(2 * S);
        std::vector<float> rest(2 * S);
        std::vector<double> rest64(h->fp64 ? 2 * S : 0);
        for (int64_t s = 0; s < S; ++s) {  // s ascending => each list sorted by spring id
            const int32_t a = d->springs[2 * s], b = d->springs[2 * s + 1];
            const int k = d->spring_kinds[s];
            if (k < 0 || k > 2) return fail(CS_E_INVALID, "spring kind must be 0, 1 or 2");
            int64_t ea = fill[a]++, eb = fill[b]++;
            nbr[ea] = b; nbr[eb] = a;
            kind[ea] = kind[eb] = (uint8_t)k;
            rest[ea] = rest[eb] = d->spring_rest[s];
            if (h->fp64) rest64[ea] = rest64[eb] = d->spring_rest64[s];
        }
        CK(dalloc(&h->csr_off, N + 1));
        CK(dalloc(&h->csr_nbr, 2 * S));
        CK(dalloc(&h->csr_kind, 2 * S));
        CK(dalloc(&h->csr_rest, 2 * S));
        CK(cudaMemcpy(h->csr_off, off.data(), (N + 1) * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->csr_nbr, nbr.data(), 2 * S * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->csr_kind, kind.data(), 2 * S, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->csr_rest, rest.data(), 2 * S * 4, cudaMemcpyHostToDevice));
        if (h->fp64) {
            CK(dalloc(&h->csr_rest64, 2 * S));
            CK(cudaMemcpy(h->csr_rest64, rest64.data(), 2 * S * 8, cudaMemcpyHostToDevice));
        }
    }

    // ---- triangles, incidence CSR, edges ----
    h->nc = d->num_tris;
    h->ne = d->num_edges;
    if (!gen) {  // a generated grid needs no triangle table (no obstacle, stencil normals)
        const int64_t C = h->nc;
        std::vector<int32_t> tg(3 * C);
        for (int64_t i = 0; i < 3 * C; ++i) {
            const int32_t v = d->tris[i];
            if (v < 0 || v >= N) return fail(CS_E_INVALID, "triangle vertex out of range");
            tg[i] = (int32_t)h->gidx(v);
        }
        CK(dalloc(&h->tris_g, 3 * C));
        CK(cudaMemcpy(h->tris_g, tg.data(), 3 * C * 4, cudaMemcpyHostToDevice));
        if (!h->grid) {
            // engine.py:232-242: ascending triangle order per node; the f64
            // path uses np.add.at's (corner, triangle) order (mesh.py:425-427)
            std::vector<int64_t> off(N + 1, 0);
            for (int64_t i = 0; i < 3 * C; ++i) off[d->tris[i] + 1]++;
            for (int64_t i = 0; i < N; ++i) off[i + 1] += off[i];
            std::vector<int64_t> fill(off.begin(), off.end() - 1);
            std::vector<int32_t> inc(3 * C);
            if (h->fp64) {
                for (int c = 0; c < 3; ++c)
                    for (int64_t t = 0; t < C; ++t) inc[fill[d->tris[3 * t + c]]++] = (int32_t)t;
            } else {
                for (int64_t t = 0; t < C; ++t)
                    for (int c = 0; c < 3; ++c) {
                        const int32_t v = d->tris[3 * t + c];
                        // a triangle listing a vertex twice appears twice, like reduceat
                        inc[fill[v]++] = (int32_t)t;
                    }
            }
            CK(dalloc(&h->inc_off, N + 1));
            CK(dalloc(&h->inc_tri, 3 * C));
            CK(cudaMemcpy(h->inc_off, off.data(), (N + 1) * 8, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(h->inc_tri, inc.data(), 3 * C * 4, cudaMemcpyHostToDevice));
            CK(cudaMalloc(&h->face, 3 * (C > 0 ? C : 1) * h->esz));
        }
        if (h->ne > 0) {
            std::vector<int32_t> eg(2 * h->ne);
            for (int64_t i = 0; i < 2 * h->ne; ++i) {
                const int32_t v = d->edges[i];
                if (v < 0 || v >= N) return fail(CS_E_INVALID, "edge vertex out of range");
                eg[i] = (int32_t)h->gidx(v);
            }
            CK(dalloc(&h->edges_g, 2 * h->ne));
            CK(cudaMemcpy(h->edges_g, eg.data(), 2 * h->ne * 4, cudaMemcpyHostToDevice));
        }
    }

    // ---- collision buffers + broad phase (engine.py:218-230) ----
    CK(dalloc(&h->stats, 4 + 2 * cs_engine::kRing));
    CK(cudaMemsetAsync(h->stats, 0, (4 + 2 * cs_engine::kRing) * sizeof(unsigned long long), h->st));
    CK(dalloc(&h->acc, 3 * P));
    CK(dalloc(&h->count, P));
    CK(dalloc(&h->touched, P));
    CK(dalloc(&h->touched_n, 1));
    CK(dalloc(&h->respond_done, 1));
    CK(cudaMemsetAsync(h->respond_done, 0, 4, h->st));
    CK(cudaMemsetAsync(h->acc, 0, 3 * P * 4, h->st));
    CK(cudaMemsetAsync(h->count, 0, P * 4, h->st));
    CK(cudaMemsetAsync(h->touched_n, 0, 4, h->st));
    h->nt = d->num_obstacle_tris;
    h->has_obstacle = h->nt > 0;
    if (h->has_obstacle) {
        CK(dalloc(&h->corners, 9 * h->nt));
        CK(dalloc(&h->onormals, 3 * h->nt));
        CK(cudaMemcpy(h->corners, d->obstacle_corners, 9 * h->nt * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->onormals, d->obstacle_normals, 3 * h->nt * 4, cudaMemcpyHostToDevice));
        if (build_broadphase(h->bp, h->corners, h->nt, d->obstacle_corners, d->cell_size, h->st))
            return fail(CS_E_CUDA, std::string("broad-phase build failed: ") +
                                       cudaGetErrorString(cudaGetLastError()));
        h->bp.warp_per_query = (d->flags & CS_FLAG_THREAD_NARROW) ? 0
                               : (d->flags & CS_FLAG_WARP_NARROW)  ? 1
                               : (d->flags & CS_FLAG_SPLIT_NARROW) ? 2 : 3;
        if (h->bp.warp_per_query == 3 && h->nc > 0) {
            // every unique cloth edge owned by the lowest-index triangle that
            // contains it: bit k of tri_own[t] = edge (tris[t][k], tris[t][k+1 mod 3])
            const int64_t C = h->nc;
            std::vector<uint8_t> own(C, 0);
            if (h->grid) {  // generate_cloth_grid's order (mesh.py:296-305), closed form
                const int64_t nx = h->nx, cw = nx - 1;
                for (int64_t t = 0; t < C; ++t) {
                    const int64_t cell = t >> 1, i = cell % cw, j = cell / cw;
                    own[t] = (t & 1) ? (uint8_t)6u  // T1 (v10, v01, v11): top and right edges
                                     : (uint8_t)(2u | (i == 0 ? 1u : 0u) | (j == 0 ? 4u : 0u));
                }
            } else {
                std::vector<std::pair<uint64_t, int64_t>> e(3 * C);
                for (int64_t t = 0; t < C; ++t)
                    for (int k = 0; k < 3; ++k) {
                        const uint32_t a = (uint32_t)d->tris[3 * t + k];
                        const uint32_t b = (uint32_t)d->tris[3 * t + (k + 1) % 3];
                        const uint64_t key = ((uint64_t)std::min(a, b) << 32) | std::max(a, b);
                        e[3 * t + k] = {key, 3 * t + k};
                    }
                std::sort(e.begin(), e.end());
                for (size_t i = 0; i < e.size(); ++i)
                    if (i == 0 || e[i].first != e[i - 1].first)
                        own[e[i].second / 3] |= (uint8_t)(1u << (e[i].second % 3));
            }
            CK(dalloc(&h->bp.tri_own, C));
            CK(cudaMemcpy(h->bp.tri_own, own.data(), C, cudaMemcpyHostToDevice));
        }
        if (h->fp64) {
            CK(dalloc(&h->corners64, 9 * h->nt));
            CK(dalloc(&h->onormals64, 3 * h->nt));
            CK(cudaMemcpy(h->corners64, d->obstacle_corners64, 9 * h->nt * 8, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(h->onormals64, d->obstacle_normals64, 3 * h->nt * 8, cudaMemcpyHostToDevice));
            h->eps64 = d->epsilon_mt64;
            h->margin64 = d->response_margin64;
            if (h->c64.reserve(std::max<int64_t>(4096, 4 * N)))
                return fail(CS_E_CAPACITY, "float64 contact buffers");
            h->use_graph = false;  // the float64 collision passes synchronise
        }
    }
    CK(cudaStreamSynchronize(h->st));
    CK(cudaGetLastError());
    return 0;
}

extern "C" int cs_destroy(cs_engine *h) {
    if (!h) return 0;
    // every stream that may still touch the engine's buffers, before freeing
    if (h->st) cudaStreamSynchronize(h->st);
    if (h->nrm_st) cudaStreamSynchronize(h->nrm_st);
    if (h->copy_st) cudaStreamSynchronize(h->copy_st);
    drop_graphs(h);
    void *ptrs[] = {h->state[0], h->state[1], h->normals, h->pinbits, h->inv_mass, h->mass64,
                    h->pinned8, h->ext, h->forces_raw, h->csr_off, h->csr_nbr, h->csr_kind,
                    h->csr_rest, h->csr_rest64, h->inc_off, h->inc_tri, h->face, h->tris_g,
                    h->edges_g, h->corners, h->onormals, h->acc, h->count, h->touched,
                    h->touched_n, h->stats, h->stage, h->hflags, h->corners64, h->onormals64,
                    h->respond_done};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    if (h->has_obstacle) free_broadphase(h->bp);
    h->c64.release();
    if (h->c64.count) cudaFree(h->c64.count);
    if (h->own_stream && h->st) cudaStreamDestroy(h->st);
    if (h->copy_st) {
        cudaStreamSynchronize(h->copy_st);
        cudaStreamDestroy(h->copy_st);
    }
    if (h->nrm_st) {
        cudaStreamSynchronize(h->nrm_st);
        cudaStreamDestroy(h->nrm_st);
    }
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ev_nrm) cudaEventDestroy(h->ev_nrm);
    if (h->clog) cudaFree(h->clog);
    if (h->clog_n) cudaFree(h->clog_n);
    if (h->ev_join) cudaEventDestroy(h->ev_join);
    for (int i = 0; i < 2; ++i) {
        if (h->ev_frame[i]) cudaEventDestroy(h->ev_frame[i]);
        if (h->ev_moved[i]) cudaEventDestroy(h->ev_moved[i]);
        if (h->rec_stage[i]) cudaFree(h->rec_stage[i]);
    }
    delete h;
    return 0;
}

extern "C" int cs_create(const cs_desc *d, cs_engine **out) {
    if (!d || !out) return fail(CS_E_INVALID, "null argument");
    *out = nullptr;
    if (d->abi_version != CS_ABI_VERSION) return fail(CS_E_INVALID, "ABI version mismatch");
    if (d->num_nodes < 1 || !d->positions || !d->inv_mass)
        return fail(CS_E_INVALID, "num_nodes, positions and inv_mass are required");
    if (d->num_obstacle_tris > 0 && (!d->obstacle_corners || !d->obstacle_normals))
        return fail(CS_E_INVALID, "obstacle arrays missing");
    if (d->num_nodes > ((int64_t)1 << 31) - 1) return fail(CS_E_CAPACITY, "more than 2^31-1 nodes");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(CS_E_NODEVICE, "no CUDA device is available");
    }
    cs_engine *h = new cs_engine();
    int r = build(h, d);
    if (r) {
        std::string keep = g_err;
        cudaGetLastError();
        cs_destroy(h);
        g_err = keep;
        return r;
    }
    *out = h;
    return 0;
}

// A grid engine straight from generate_cloth_grid's parameters (mesh.py:
// 223-317), every per-node / per-spring quantity generated on the device.
extern "C" int cs_create_grid(const cs_grid_desc *g, cs_engine **out) {
    if (!g || !out) return fail(CS_E_INVALID, "null argument");
    *out = nullptr;
    if (g->abi_version != CS_ABI_VERSION) return fail(CS_E_INVALID, "ABI version mismatch");
    if (g->nx < 2 || g->ny < 2) return fail(CS_E_INVALID, "grid needs at least 2 nodes per side");
    if (!(g->width > 0.0) || !(g->height > 0.0)) return fail(CS_E_INVALID, "cloth dimensions must be positive");
    if (!(g->total_mass > 0.0)) return fail(CS_E_INVALID, "total_mass must be positive");
    const int row0 = g->row_lo, rows = g->row_hi - g->row_lo;
    if (row0 < 0 || g->row_hi > g->ny || rows < 2) return fail(CS_E_INVALID, "local rows out of range");
    if (g->flags & (CS_FLAG_FP64 | CS_FLAG_FORCE_CSR))
        return fail(CS_E_INVALID, "generated grids run the float32 stencil (fast or fixed)");
    if (g->num_pinned_rows > 0 && !g->pinned_rows) return fail(CS_E_INVALID, "pinned_rows missing");
    if ((int64_t)g->nx * rows > ((int64_t)1 << 31) - 1) return fail(CS_E_CAPACITY, "more than 2^31-1 nodes");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(CS_E_NODEVICE, "no CUDA device is available");
    }
    GridGen gen;
    gen.nx = g->nx;
    gen.ny = g->ny;
    gen.row0 = row0;
    gen.width = g->width;
    gen.height = g->height;
    gen.orient = g->orientation;
    const double m = g->total_mass / ((double)g->nx * g->ny);  // mesh.py:258
    gen.inv_mass = (float)(1.0 / m);                           // engine.py:199-202
    for (int k = 0; k < g->num_pinned_rows; ++k) {
        if (g->pinned_rows[k] < 0 || g->pinned_rows[k] >= g->ny)
            return fail(CS_E_INVALID, "pinned row index out of range");
        gen.pinned_rows.push_back(g->pinned_rows[k]);
    }
    cs_desc d;
    memset(&d, 0, sizeof d);
    d.abi_version = CS_ABI_VERSION;
    d.flags = g->flags;
    d.nx = g->nx;
    d.ny = rows;
    bool uniform = true;
    const cudaError_t e = grid_rest6(g->nx, g->ny, row0, rows, g->width, g->height, d.grid_rest,
                                     &uniform, (cudaStream_t)g->stream);
    if (e != cudaSuccess) return fail(CS_E_CUDA, std::string("grid rest lengths: ") + cudaGetErrorString(e));
    if (!uniform)
        return fail(CS_E_INVALID, "a spring family of this grid has more than one float32 rest "
                                  "length; build the engine from the mesh instead");
    d.num_nodes = (int64_t)g->nx * rows;
    d.num_tris = 2 * (int64_t)(g->nx - 1) * (rows - 1);
    d.dt = g->dt;
    for (int q = 0; q < 3; ++q) {
        d.gravity[q] = g->gravity[q];
        d.stiffness[q] = g->stiffness[q];
    }
    d.damping = g->damping;
    d.epsilon_mt = g->epsilon_mt;
    d.response_margin = g->response_margin;
    d.fixed_point_scale = g->fixed_point_scale;
    d.substeps = g->substeps;
    d.stream = g->stream;
    cs_engine *h = new cs_engine();
    int r = build(h, &d, &gen);
    if (r) {
        std::string keep = g_err;
        cudaGetLastError();
        cs_destroy(h);
        g_err = keep;
        return r;
    }
    *out = h;
    return 0;
}

extern "C" int cs_grid_topology(int32_t nx, int32_t ny, int32_t row_lo, int32_t row_hi,
                                double width, double height, int32_t *springs, int32_t *kinds,
                                double *rest, int32_t *tris, double *positions, void *stream) {
    if (nx < 2 || ny < 2 || row_lo < 0 || row_hi > ny || row_hi - row_lo < 2)
        return fail(CS_E_INVALID, "bad grid / rows");
    const cudaError_t e = grid_topology(nx, ny, row_lo, row_hi - row_lo, width, height, springs,
                                        kinds, rest, tris, positions, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(CS_E_CUDA, cudaGetErrorString(e));
    return 0;
}

// ---------------------------------------------------------------------------
// stepping
// ---------------------------------------------------------------------------
extern "C" int cs_step(cs_engine *h, int32_t frames) {
    if (!h) return fail(CS_E_INVALID, "null engine");
    if (h->banded && !h->seam_in_kernel()) {  // stream handshake values change every frame: no graph
        for (int32_t f = 0; f < frames; ++f) {
            if (int r = banded_frame(h)) return r;
            h->frames++;
        }
        return 0;
    }
    if (h->lag_normals() && !h->nrm_st) {
        CK(cudaStreamCreateWithFlags(&h->nrm_st, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->ev_nrm, cudaEventDisableTiming));
    }
    const int G = graph_frames();
    for (int32_t f = 0; f < frames;) {
        int n = 1;  // frames this iteration
        if (h->use_graph) {
            const int start = h->cur;
            n = (G > 1 && frames - f >= G) ? G : 1;
            cudaGraphExec_t &ge = n > 1 ? h->graphG[start] : h->graph[start];
            if (!ge) {
                cudaGraph_t g;
                CK(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
                for (int k = 0; k < n; ++k) launch_frame(h);
                CK(cudaStreamEndCapture(h->st, &g));
                CK(cudaGraphInstantiate(&ge, g, 0));
                cudaGraphDestroy(g);
                h->cur = start;  // capture did not execute anything
            }
            CK(cudaGraphLaunch(ge, h->st));
            // replay the parity bookkeeping of the graph's frames
            if ((h->substeps * n) & 1) h->cur = 1 - start;
            h->forces_valid = true;
            h->normals_stale = h->normals_lagged();
        } else {
            launch_frame(h);
            CK(cudaGetLastError());
        }
        if (h->banded) h->passes += (uint32_t)(h->substeps * n);  // replayed in-kernel handshakes
        h->frames += n;
        f += n;
    }
    return 0;
}

// Advance `frames` frames and stream every frame's positions, (N,3) f32
// each, into host_out[frames][N][3] -- engine.py:341-343 (`readback=True`)
// for a whole run.  The device->host copy of frame f (a transpose kernel on a
// copy stream, then the DMA) overlaps the computation of frame f+1; the
// compute stream only waits for frame f's transpose (microseconds) before
// reusing its buffer.  host_out should be pinned for the DMA to be async.
extern "C" int cs_record(cs_engine *h, int32_t frames, float *host_out) {
    if (!h || !host_out) return fail(CS_E_INVALID, "null argument");
    if (h->fp64) return fail(CS_E_INVALID, "cs_record streams float32 positions");
    if (!h->copy_st) {
        CK(cudaStreamCreateWithFlags(&h->copy_st, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            CK(cudaEventCreateWithFlags(&h->ev_frame[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&h->ev_moved[i], cudaEventDisableTiming));
            CK(cudaMalloc(&h->rec_stage[i], (size_t)h->N * 3 * sizeof(float)));
        }
    }
    const int64_t nxx = h->grid ? h->nx : h->N;
    for (int32_t f = 0; f < frames; ++f) {
        const int k = f & 1;
        if (f > 0) CK(cudaStreamWaitEvent(h->st, h->ev_moved[k ^ 1], 0));  // f-1 transposed
        if (int r = cs_step(h, 1)) return r;
        // a row band's halo rows of the new state are the neighbours' peer
        // stores: wait for their pass, as cs_read does, before copying
        if (h->banded)
            if (int r = halo_wait(h)) return r;
        CK(cudaEventRecord(h->ev_frame[k], h->st));
        CK(cudaStreamWaitEvent(h->copy_st, h->ev_frame[k], 0));
        k_planes_to_aos<float><<<nb(h->N), 256, 0, h->copy_st>>>(
            h->N, nxx, h->pitch, h->plane, 3, (const float *)h->state[h->cur], h->rec_stage[k]);
        CK(cudaGetLastError());
        CK(cudaEventRecord(h->ev_moved[k], h->copy_st));
        CK(cudaMemcpyAsync(host_out + (size_t)f * h->N * 3, h->rec_stage[k],
                           (size_t)h->N * 3 * sizeof(float), cudaMemcpyDeviceToHost, h->copy_st));
    }
    CK(cudaStreamSynchronize(h->copy_st));
    CK(cudaStreamSynchronize(h->st));
    return 0;
}

// Record every (cloth node, obstacle triangle) contact of the following
// detect passes (capacity 0 switches the log off).
extern "C" int cs_contact_log(cs_engine *h, int64_t capacity) {
    if (!h || capacity < 0) return fail(CS_E_INVALID, "bad argument");
    CK(cudaStreamSynchronize(h->st));
    if (h->clog) cudaFree(h->clog);
    if (h->clog_n) cudaFree(h->clog_n);
    h->clog = nullptr;
    h->clog_n = nullptr;
    h->clog_cap = 0;
    if (capacity > 0) {
        CK(dalloc(&h->clog, 2 * capacity));
        CK(dalloc(&h->clog_n, 1));
        CK(cudaMemset(h->clog_n, 0, sizeof(uint32_t)));
        h->clog_cap = capacity;
    }
    drop_graphs(h);  // the detect kernels' arguments changed
    return 0;
}

// The last frame's contacts as (node index, triangle) int32 pairs; *n gets
// the total count (which may exceed `max` -- then the log was truncated).
extern "C" int cs_read_contacts(cs_engine *h, int32_t *out, int64_t max, int64_t *n) {
    if (!h || !n) return fail(CS_E_INVALID, "null argument");
    if (!h->clog) return fail(CS_E_INVALID, "contact log is off (cs_contact_log)");
    uint32_t cnt = 0;
    CK(cudaMemcpyAsync(&cnt, h->clog_n, sizeof(cnt), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    *n = cnt;
    const int64_t k = std::min<int64_t>(std::min<int64_t>(cnt, h->clog_cap), max);
    if (k > 0 && out) {
        std::vector<uint32_t> raw(2 * k);
        CK(cudaMemcpy(raw.data(), h->clog, 2 * k * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < k; ++i) {
            const int64_t g = raw[2 * i];
            out[2 * i] = (int32_t)(h->grid ? (g / h->pitch) * h->nx + g % h->pitch : g);
            out[2 * i + 1] = (int32_t)raw[2 * i + 1];
        }
    }
    return 0;
}

extern "C" int cs_run_pass(cs_engine *h, int32_t pass_id) {
    if (!h) return fail(CS_E_INVALID, "null engine");
    switch (pass_id) {
        case CS_PASS_FORCE_INTEGRATE: flush_normals(h); pass_force_integrate(h); break;
        case CS_PASS_DETECT: pass_detect(h); break;
        case CS_PASS_RESPOND:
            if (h->has_obstacle) pass_respond(h);
            break;
        case CS_PASS_NORMALS: pass_normals(h); h->normals_stale = false; h->frames++; break;
        default: return fail(CS_E_INVALID, "unknown pass id");
    }
    CK(cudaGetLastError());
    return 0;
}

extern "C" int cs_respond(cs_engine *h, int64_t *responded) {
    if (!h) return fail(CS_E_INVALID, "null engine");
    flush_normals(h);  // the buffer must describe the pre-respond positions
    CK(cudaMemsetAsync(h->stats + 1, 0, sizeof(unsigned long long), h->st));
    launch_respond(h->cargs(), (float *)h->state[h->cur], h->grid ? h->pinbits : nullptr,
                   h->grid ? nullptr : h->inv_mass, h->average ? 1 : 0, h->N, h->num_sms,
                   /*end_of_frame=*/false, h->st);
    CK(cudaGetLastError());
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, h->stats + 1, sizeof(v), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (responded) *responded = (int64_t)v;
    return 0;
}

extern "C" int cs_frame_stats(cs_engine *h, cs_stats *out) {
    if (!h || !out) return fail(CS_E_INVALID, "null argument");
    unsigned long long v[3] = {0, 0, 0};
    CK(cudaMemcpyAsync(v, h->stats, sizeof(v), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    out->hits = (int64_t)v[0];
    out->responded = (int64_t)v[1];
    out->hit_counter = (int64_t)v[2];
    out->frames = h->frames;
    return 0;
}

extern "C" int cs_frame_hits(cs_engine *h, int64_t frame, int64_t *hits, int64_t *responded) {
    if (!h) return fail(CS_E_INVALID, "null engine");
    if (!h->has_obstacle) {
        if (hits) *hits = 0;
        if (responded) *responded = 0;
        return 0;
    }
    unsigned long long fc = 0, v[2] = {0, 0};
    CK(cudaMemcpyAsync(&fc, h->stats + 3, sizeof(fc), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (frame < 0 || (unsigned long long)frame >= fc ||
        fc - (unsigned long long)frame > (unsigned long long)cs_engine::kRing)
        return fail(CS_E_INVALID, "frame statistics no longer available (ring of 4096 frames)");
    const int64_t slot = frame % cs_engine::kRing;
    CK(cudaMemcpy(v, h->stats + 4 + 2 * slot, sizeof(v), cudaMemcpyDeviceToHost));
    if (hits) *hits = (int64_t)v[0];
    if (responded) *responded = (int64_t)v[1];
    return 0;
}

extern "C" int cs_synchronize(cs_engine *h) {
    if (!h) return fail(CS_E_INVALID, "null engine");
    CK(cudaStreamSynchronize(h->st));
    return seam_check(h);
}

extern "C" int cs_stream(cs_engine *h, void **stream) {
    if (!h || !stream) return fail(CS_E_INVALID, "null argument");
    *stream = (void *)h->st;
    return 0;
}

// ---------------------------------------------------------------------------
// transfers
// ---------------------------------------------------------------------------
static int cs_read_impl(cs_engine *h, int32_t id, void *dst);
extern "C" int cs_read(cs_engine *h, int32_t id, void *dst) {
    if (!h || !dst) return fail(CS_E_INVALID, "null argument");
    if (int r = cs_read_impl(h, id, dst)) return r;
    return seam_check(h);
}
static int cs_read_impl(cs_engine *h, int32_t id, void *dst) {
    const int64_t P = h->plane;
    switch (id) {
        case CS_BUF_POSITIONS:
        case CS_BUF_VELOCITIES:
        case CS_BUF_PREV_POSITIONS:
        case CS_BUF_NORMALS:
        case CS_BUF_NORMALS_LAGGED: {
            if (id == CS_BUF_NORMALS) flush_normals(h);
            if (h->banded) {
                if (int r = halo_wait(h)) return r;  // halo rows of the current state landed
            }
            const void *base = (id == CS_BUF_NORMALS || id == CS_BUF_NORMALS_LAGGED) ? h->normals
                               : id == CS_BUF_PREV_POSITIONS ? h->state[1 - h->cur]
                                                             : h->state[h->cur];
            const int64_t o = id == CS_BUF_VELOCITIES ? 3 * P : 0;
            if (h->fp64) {
                float *tmp;
                CK(cudaMalloc(&tmp, 3 * P * 4));
                k_f64_to_f32<<<nb(3 * P), 256, 0, h->st>>>(3 * P, (const double *)base + o, tmp);
                int r = download_planes<float>(h, tmp, (float *)dst, 3);
                cudaFree(tmp);
                return r;
            }
            return download_planes<float>(h, (const float *)base + o, (float *)dst, 3);
        }
        case CS_BUF_POSITIONS64:
        case CS_BUF_VELOCITIES64: {
            if (!h->fp64) return fail(CS_E_INVALID, "float64 buffers need a CS_FLAG_FP64 engine");
            const int64_t o = id == CS_BUF_VELOCITIES64 ? 3 * P : 0;
            return download_planes<double>(h, (const double *)h->state[h->cur] + o, (double *)dst, 3);
        }
        case CS_BUF_FORCES_RAW: {
            if (h->fp64) return fail(CS_E_INVALID, "read_forces_raw is a float32-engine buffer");
            if (!h->forces_valid) {
                memset(dst, 0, (size_t)h->N * 3 * 4);
                return 0;
            }
            if (!h->forces_raw) CK(dalloc(&h->forces_raw, 3 * P));
            const float *prev = (const float *)h->state[1 - h->cur];
            if (h->grid && h->strip && !h->fixed && (h->flags & CS_FLAG_PAIRED))
                // the fast kernel's own forces (k_pair3 in its read-only mode)
                launch_pair3_forces(h->sp, prev, h->pinbits, h->forces_raw, h->st);
            else if (h->grid)
                launch_grid_forces(h->sp, prev, h->forces_raw, h->st);
            else
                launch_csr_forces(h->cp, prev, h->csr_off, h->csr_nbr, h->csr_kind, h->csr_rest,
                                  h->forces_raw, h->st);
            CK(cudaGetLastError());
            return download_planes<int32_t>(h, h->forces_raw, (int32_t *)dst, 3);
        }
        case CS_BUF_ACCUMULATOR:
            return download_planes<int32_t>(h, h->acc, (int32_t *)dst, 3);
        case CS_BUF_COUNTS:
            return download_planes<int32_t>(h, h->count, (int32_t *)dst, 1);
        default:
            return fail(CS_E_INVALID, "unknown buffer id");
    }
}

extern "C" int cs_write(cs_engine *h, int32_t id, const void *src) {
    if (!h) return fail(CS_E_INVALID, "null engine");
    const int64_t P = h->plane;
    switch (id) {
        case CS_BUF_POSITIONS:
        case CS_BUF_VELOCITIES: {
            if (!src) return fail(CS_E_INVALID, "null source");
            flush_normals(h);
            const int64_t o = id == CS_BUF_VELOCITIES ? 3 * P : 0;
            if (h->fp64) {
                float *tmp;
                CK(cudaMalloc(&tmp, 3 * P * 4));
                CK(cudaMemsetAsync(tmp, 0, 3 * P * 4, h->st));
                int r = upload_planes<float>(h, (const float *)src, tmp, 3);
                if (!r) k_f32_to_f64<<<nb(3 * P), 256, 0, h->st>>>(3 * P, tmp, (double *)h->state[h->cur] + o);
                CK(cudaStreamSynchronize(h->st));
                cudaFree(tmp);
                return r;
            }
            int r = upload_planes<float>(h, (const float *)src, (float *)h->state[h->cur] + o, 3);
            if (!r) CK(cudaStreamSynchronize(h->st));
            return r;
        }
        case CS_BUF_POSITIONS64:
        case CS_BUF_VELOCITIES64: {
            if (!h->fp64) return fail(CS_E_INVALID, "float64 buffers need a CS_FLAG_FP64 engine");
            const int64_t o = id == CS_BUF_VELOCITIES64 ? 3 * P : 0;
            int r = upload_planes<double>(h, (const double *)src, (double *)h->state[h->cur] + o, 3);
            if (!r) CK(cudaStreamSynchronize(h->st));
            return r;
        }
        case CS_BUF_EXT_ACCEL: {
            if (!src) {  // set_external_accel(None): zeros (engine.py:299-300)
                if (h->has_ext) {
                    CK(cudaMemsetAsync(h->ext, 0, 3 * P * h->esz, h->st));
                    CK(cudaStreamSynchronize(h->st));
                }
                return 0;
            }
            if (!h->ext) {
                CK(cudaMalloc(&h->ext, 3 * P * h->esz));
                CK(cudaMemsetAsync(h->ext, 0, 3 * P * h->esz, h->st));
                drop_graphs(h);  // kernels now read the ext planes
            }
            h->has_ext = true;
            int r;
            if (h->fp64) {
                float *tmp;
                CK(cudaMalloc(&tmp, 3 * P * 4));
                CK(cudaMemsetAsync(tmp, 0, 3 * P * 4, h->st));
                r = upload_planes<float>(h, (const float *)src, tmp, 3);
                if (!r) k_f32_to_f64<<<nb(3 * P), 256, 0, h->st>>>(3 * P, tmp, (double *)h->ext);
                CK(cudaStreamSynchronize(h->st));
                cudaFree(tmp);
            } else {
                r = upload_planes<float>(h, (const float *)src, (float *)h->ext, 3);
                if (!r) CK(cudaStreamSynchronize(h->st));
            }
            return r;
        }
        case CS_BUF_ACCUMULATOR:
        case CS_BUF_COUNTS: {
            if (!src) return fail(CS_E_INVALID, "null source");
            int r = id == CS_BUF_ACCUMULATOR ? upload_planes<int32_t>(h, (const int32_t *)src, h->acc, 3)
                                             : upload_planes<int32_t>(h, (const int32_t *)src, h->count, 1);
            if (r) return r;
            launch_rebuild_touched(h->cargs(), h->rows, h->grid ? h->nx : h->N, h->pitch, h->st);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(h->st));
            return 0;
        }
        default:
            return fail(CS_E_INVALID, "unknown or read-only buffer id");
    }
}

// ---- device-pointer transfers (PyTorch tensors: tensor.data_ptr()) ------------------
// `to` waits for everything enqueued on `from` so far
static int join(cs_engine *h, cudaStream_t from, cudaStream_t to) {
    if (from == to) return 0;
    if (!h->ev_join) CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    CK(cudaEventRecord(h->ev_join, from));
    CK(cudaStreamWaitEvent(to, h->ev_join, 0));
    return 0;
}

#ifdef CS_PAIR3_TRACE
namespace cs { int pair3_trace_read(unsigned long long *out, int n); }
// diagnostic builds only: per-warp {start, end, smid} of the last k_pair3 launch
extern "C" int cs_debug_pair3_trace(unsigned long long *out, int32_t n) {
    return cs::pair3_trace_read(out, n);
}
#endif
extern "C" int cs_device(cs_engine *h, int32_t *device) {
    if (!h || !device) return fail(CS_E_INVALID, "null argument");
    *device = h->device;
    return 0;
}

extern "C" int cs_set_stream(cs_engine *h, void *stream) {
    if (!h) return fail(CS_E_INVALID, "null engine");
    cudaStream_t s = (cudaStream_t)stream;
    if (!s) return fail(CS_E_INVALID, "pass a real CUDA stream (the legacy default stream is not one)");
    if (h->banded) return fail(CS_E_INVALID, "a linked row band keeps its stream");
    if (s == h->st) return 0;
    if (int r = join(h, h->st, s)) return r;  // the new stream continues after the old one's work
    if (h->copy_st) CK(cudaStreamSynchronize(h->copy_st));
    if (h->own_stream) {
        CK(cudaStreamSynchronize(h->st));
        CK(cudaStreamDestroy(h->st));
        h->own_stream = false;
    }
    h->st = s;  // captured graphs are stream-independent: cudaGraphLaunch takes the stream
    return 0;
}

extern "C" int cs_read_device(cs_engine *h, int32_t id, void *dst, void *stream) {
    if (!h || !dst) return fail(CS_E_INVALID, "null argument");
    cudaStream_t s = stream ? (cudaStream_t)stream : h->st;
    const int64_t P = h->plane, nxx = h->grid ? h->nx : h->N;
    const void *base = nullptr;
    int comps = 3;
    bool wide = h->fp64, i32 = false, want64 = false;
    switch (id) {
        case CS_BUF_POSITIONS: case CS_BUF_POSITIONS64: base = h->state[h->cur]; break;
        case CS_BUF_VELOCITIES: case CS_BUF_VELOCITIES64:
            base = (const char *)h->state[h->cur] + 3 * P * h->esz;
            break;
        case CS_BUF_PREV_POSITIONS: base = h->state[1 - h->cur]; break;
        case CS_BUF_NORMALS: flush_normals(h); base = h->normals; break;
        case CS_BUF_NORMALS_LAGGED: base = h->normals; break;
        case CS_BUF_ACCUMULATOR: base = h->acc; wide = false; i32 = true; break;
        case CS_BUF_COUNTS: base = h->count; wide = false; i32 = true; comps = 1; break;
        default: return fail(CS_E_INVALID, "buffer id not readable into device memory");
    }
    if (id == CS_BUF_POSITIONS64 || id == CS_BUF_VELOCITIES64) {
        if (!h->fp64) return fail(CS_E_INVALID, "float64 buffers need a CS_FLAG_FP64 engine");
        want64 = true;
    }
    if (h->banded)
        if (int r = halo_wait(h)) return r;  // halo rows of the current state landed
    if (int r = join(h, h->st, s)) return r;
    const unsigned g = nb(h->N);
    if (i32)
        k_planes_to_aos_cvt<int32_t, int32_t><<<g, 256, 0, s>>>(h->N, nxx, h->pitch, P, comps,
                                                                (const int32_t *)base, (int32_t *)dst);
    else if (wide && want64)
        k_planes_to_aos_cvt<double, double><<<g, 256, 0, s>>>(h->N, nxx, h->pitch, P, 3,
                                                              (const double *)base, (double *)dst);
    else if (wide)
        k_planes_to_aos_cvt<double, float><<<g, 256, 0, s>>>(h->N, nxx, h->pitch, P, 3,
                                                             (const double *)base, (float *)dst);
    else
        k_planes_to_aos_cvt<float, float><<<g, 256, 0, s>>>(h->N, nxx, h->pitch, P, 3,
                                                            (const float *)base, (float *)dst);
    CK(cudaGetLastError());
    return join(h, s, h->st);  // later frames may not overwrite the state under the read
}

extern "C" int cs_write_device(cs_engine *h, int32_t id, const void *src, void *stream) {
    if (!h || !src) return fail(CS_E_INVALID, "null argument");
    cudaStream_t s = stream ? (cudaStream_t)stream : h->st;
    const int64_t P = h->plane, nxx = h->grid ? h->nx : h->N;
    void *base = nullptr;
    bool src64 = false;
    switch (id) {
        case CS_BUF_POSITIONS: base = h->state[h->cur]; break;
        case CS_BUF_VELOCITIES: base = (char *)h->state[h->cur] + 3 * P * h->esz; break;
        case CS_BUF_POSITIONS64: src64 = true; base = h->state[h->cur]; break;
        case CS_BUF_VELOCITIES64: src64 = true; base = (char *)h->state[h->cur] + 3 * P * h->esz; break;
        case CS_BUF_EXT_ACCEL:
            if (!h->ext) {
                CK(cudaMalloc(&h->ext, 3 * P * h->esz));
                CK(cudaMemsetAsync(h->ext, 0, 3 * P * h->esz, h->st));
                drop_graphs(h);  // kernels now read the ext planes
            }
            h->has_ext = true;
            base = h->ext;
            break;
        default: return fail(CS_E_INVALID, "buffer id not writable from device memory");
    }
    if (src64 && !h->fp64) return fail(CS_E_INVALID, "float64 buffers need a CS_FLAG_FP64 engine");
    if (id == CS_BUF_POSITIONS || id == CS_BUF_VELOCITIES || src64) flush_normals(h);
    if (h->banded)
        if (int r = halo_wait(h)) return r;
    if (int r = join(h, h->st, s)) return r;
    const unsigned g = nb(h->N);
    if (src64)
        k_aos_to_planes_cvt<double, double><<<g, 256, 0, s>>>(h->N, nxx, h->pitch, P, 3,
                                                              (const double *)src, (double *)base);
    else if (h->fp64)
        k_aos_to_planes_cvt<float, double><<<g, 256, 0, s>>>(h->N, nxx, h->pitch, P, 3,
                                                             (const float *)src, (double *)base);
    else
        k_aos_to_planes_cvt<float, float><<<g, 256, 0, s>>>(h->N, nxx, h->pitch, P, 3,
                                                            (const float *)src, (float *)base);
    CK(cudaGetLastError());
    return join(h, s, h->st);  // the next frame reads the new state
}

extern "C" int cs_inject_response(cs_engine *h, int64_t node, const int32_t raw[3], int32_t count) {
    if (!h) return fail(CS_E_INVALID, "null engine");
    if (node < 0 || node >= h->N) return fail(CS_E_INVALID, "node index out of range");
    const int64_t g = h->gidx(node);
    for (int c = 0; c < 3; ++c)
        CK(cudaMemcpyAsync(h->acc + c * h->plane + g, raw + c, 4, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(h->count + g, &count, 4, cudaMemcpyHostToDevice, h->st));
    launch_rebuild_touched(h->cargs(), h->rows, h->grid ? h->nx : h->N, h->pitch, h->st);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(h->st));
    return 0;
}

extern "C" int cs_state_plane(cs_engine *h, int32_t which, void **ptr, int64_t *pitch) {
    if (!h || !ptr || which < 0 || which > 5) return fail(CS_E_INVALID, "bad argument");
    *ptr = (char *)h->state[h->cur] + (size_t)which * h->plane * h->esz;
    if (pitch) *pitch = h->pitch;
    return 0;
}

// ---- row bands -------------------------------------------------------------
extern "C" int cs_state_buffers(cs_engine *h, void **state0, void **state1, uint32_t **flags,
                                int64_t *plane, int64_t *pitch) {
    if (!h) return fail(CS_E_INVALID, "null engine");
    if (!h->hflags) {
        CK(dalloc(&h->hflags, 8));
        CK(cudaMemset(h->hflags, 0, 8 * sizeof(uint32_t)));
    }
    if (state0) *state0 = h->state[0];
    if (state1) *state1 = h->state[1];
    if (flags) *flags = h->hflags;
    if (plane) *plane = h->plane;
    if (pitch) *pitch = h->pitch;
    return 0;
}

extern "C" int cs_set_halo_peers(cs_engine *h, int64_t row_lo, int64_t row_hi,
                                 const cs_halo_peer *up, const cs_halo_peer *down) {
    if (!h) return fail(CS_E_INVALID, "null engine");
    if (!h->grid || !h->strip || h->fp64)
        return fail(CS_E_INVALID, "row bands need the float32 grid strip path");
    if (h->frames != 0 || h->cur != 0)
        return fail(CS_E_INVALID, "link row bands before the first frame (lockstep parity)");
    if (row_lo < 0 || row_hi > h->rows || row_lo >= row_hi)
        return fail(CS_E_INVALID, "owned rows out of range");
    if (int r = load_memops()) return r;
    if (int r = cs_state_buffers(h, nullptr, nullptr, nullptr, nullptr, nullptr)) return r;
    auto set = [&](cs_engine::Link &L, const cs_halo_peer *p) -> int {
        L = cs_engine::Link{};
        if (!p) return 0;
        if (!p->state[0] || !p->state[1] || !p->remote_flag || p->rows < 1 || p->plane < 1)
            return fail(CS_E_INVALID, "incomplete halo peer");
        if (p->src_row0 < row_lo || p->src_row0 + p->rows > row_hi)
            return fail(CS_E_INVALID, "halo rows sent must be owned rows");
        L.on = true;
        L.state[0] = p->state[0];
        L.state[1] = p->state[1];
        L.plane = p->plane;
        L.src_row0 = p->src_row0;
        L.dst_row0 = p->dst_row0;
        L.rows = p->rows;
        L.remote_flag = p->remote_flag;
        return 0;
    };
    if (int r = set(h->up, up)) return r;
    if (int r = set(h->dn, down)) return r;
    if (h->up.on && h->up.src_row0 != row_lo)
        return fail(CS_E_INVALID, "rows sent up must start at the first owned row");
    if (h->dn.on && h->dn.src_row0 + h->dn.rows != row_hi)
        return fail(CS_E_INVALID, "rows sent down must end at the last owned row");
    CK(cudaStreamSynchronize(h->st));
    h->sp.row_lo = (int)row_lo;
    h->sp.row_hi = (int)row_hi;
    h->sp.halo_up_hi = h->up.on ? (int)(h->up.src_row0 + h->up.rows) : INT_MIN;
    h->sp.halo_dn_lo = h->dn.on ? (int)h->dn.src_row0 : INT_MAX;
    h->banded = true;
    h->passes = 0;
    drop_graphs(h);  // frames now carry the peer stores (and the in-kernel handshake)
    return 0;
}

extern "C" int cs_ipc_export(void *dev_ptr, uint8_t handle[64]) {
    if (!dev_ptr || !handle) return fail(CS_E_INVALID, "null argument");
    cudaIpcMemHandle_t hd;
    CK(cudaIpcGetMemHandle(&hd, dev_ptr));
    static_assert(sizeof(hd) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle, &hd, 64);
    return 0;
}

extern "C" int cs_ipc_open(const uint8_t handle[64], void **dev_ptr) {
    if (!handle || !dev_ptr) return fail(CS_E_INVALID, "null argument");
    cudaIpcMemHandle_t hd;
    memcpy(&hd, handle, 64);
    CK(cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess));
    return 0;
}

extern "C" int cs_ipc_close(void *dev_ptr) {
    if (!dev_ptr) return fail(CS_E_INVALID, "null argument");
    CK(cudaIpcCloseMemHandle(dev_ptr));
    return 0;
}

extern "C" int cs_kernels_per_frame(cs_engine *h, int32_t *count) {
    if (!h || !count) return fail(CS_E_INVALID, "null argument");
    *count = h->kernels_per_frame();
    return 0;
}

extern "C" int cs_broadphase_stats(cs_engine *h, int64_t out[4]) {
    if (!h || !out) return fail(CS_E_INVALID, "null argument");
    out[0] = h->bp.num_cells;
    out[1] = h->bp.num_refs;
    out[2] = h->bp.grid.dims[0];
    out[3] = h->bp.grid.dims[1] * (int64_t)h->bp.grid.dims[2];
    return 0;
}

extern "C" int cs_broadphase_dump(cs_engine *h, float geometry[8], int32_t dims[3],
                                  uint32_t *ref_keys, uint32_t *ref_tris, uint32_t *cell_begin,
                                  uint32_t *cell_end) {
    if (!h) return fail(CS_E_INVALID, "null engine");
    if (!h->has_obstacle) return fail(CS_E_INVALID, "the engine has no obstacle (no broad phase)");
    const GridDesc &g = h->bp.grid;
    if (geometry) {
        for (int d = 0; d < 3; ++d) geometry[d] = g.origin[d];
        geometry[3] = g.inv_cell;
        geometry[4] = g.cell;
        geometry[5] = geometry[6] = geometry[7] = 0.f;
    }
    if (dims)
        for (int d = 0; d < 3; ++d) dims[d] = g.dims[d];
    CK(cudaStreamSynchronize(h->st));
    const size_t R = (size_t)h->bp.num_refs * sizeof(uint32_t);
    const size_t C = (size_t)h->bp.num_cells * sizeof(uint32_t);
    if (ref_keys && R) CK(cudaMemcpy(ref_keys, h->bp.cell_keys, R, cudaMemcpyDeviceToHost));
    if (ref_tris && R) CK(cudaMemcpy(ref_tris, h->bp.cell_tris, R, cudaMemcpyDeviceToHost));
    if (cell_begin && C) CK(cudaMemcpy(cell_begin, h->bp.cell_begin, C, cudaMemcpyDeviceToHost));
    if (cell_end && C) CK(cudaMemcpy(cell_end, h->bp.cell_end, C, cudaMemcpyDeviceToHost));
    return 0;
}

extern "C" int cs_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

extern "C" int cs_mem_info(int64_t *free_bytes, int64_t *total_bytes) {
    size_t f = 0, t = 0;
    CK(cudaMemGetInfo(&f, &t));
    if (free_bytes) *free_bytes = (int64_t)f;
    if (total_bytes) *total_bytes = (int64_t)t;
    return 0;
}

// ---- snapshot_png on the device (io.py:225-287), cs_snapshot.cu ----------------
namespace cs {
cudaError_t snapshot_bounds(const double *verts, int64_t n, double out[6], cudaStream_t st);
cudaError_t snapshot_render(const double *verts, const int32_t *tris, int64_t nt, int64_t n_cloth,
                            const double view[3], const int32_t axes[3], int width, int height,
                            uint8_t *rgb, void *scratch, cudaStream_t st);
}  // namespace cs

extern "C" int cs_snapshot_bounds(const double *verts, int64_t n, double out[6], void *stream) {
    if (!verts || n <= 0 || !out) return fail(CS_E_INVALID, "cs_snapshot_bounds: no vertices");
    const cudaError_t e = cs::snapshot_bounds(verts, n, out, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(CS_E_CUDA, cudaGetErrorString(e));
    return CS_OK;
}

extern "C" int cs_snapshot_render(const double *verts, const int32_t *tris, int64_t num_tris,
                                  int64_t num_cloth_tris, const double view[3],
                                  const int32_t axes[3], int32_t width, int32_t height,
                                  uint8_t *rgb, void *scratch, void *stream) {
    if (!verts || (num_tris > 0 && !tris) || !view || !axes || !rgb || !scratch)
        return fail(CS_E_INVALID, "cs_snapshot_render: null argument");
    if (width < 8 || height < 8) return fail(CS_E_INVALID, "snapshot size too small");
    for (int k = 0; k < 3; ++k)
        if (axes[k] < 0 || axes[k] > 2) return fail(CS_E_INVALID, "snapshot axes must be 0..2");
    const cudaError_t e = cs::snapshot_render(verts, tris, num_tris, num_cloth_tris, view, axes,
                                              width, height, rgb, scratch, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(CS_E_CUDA, cudaGetErrorString(e));
    return CS_OK;
}

// Current positions as device float64 (N, 3) on the engine's stream: the
// engine-side input of cs_snapshot_render (what bench.py:186 feeds
// snapshot_png from read_positions().astype(float64), without the readback).
extern "C" int cs_positions_device(cs_engine *h, double *dev_out) {
    if (!h || !dev_out) return fail(CS_E_INVALID, "null argument");
    if (h->banded) {
        if (int r = halo_wait(h)) return r;
    }
    const int64_t nxx = h->grid ? h->nx : h->N;
    if (h->fp64)
        k_planes_to_aos64<double><<<nb(h->N), 256, 0, h->st>>>(
            h->N, nxx, h->pitch, h->plane, (const double *)h->state[h->cur], dev_out);
    else
        k_planes_to_aos64<float><<<nb(h->N), 256, 0, h->st>>>(
            h->N, nxx, h->pitch, h->plane, (const float *)h->state[h->cur], dev_out);
    CK(cudaGetLastError());
    return CS_OK;
}
