/*
 * clothsim_b200.h -- C ABI of the B200-native cloth step.
 *
 * Replaces the per-frame hot path of the reference package `clothsim`
 * (arxiv 2507.11794; /root/reference/pkg/src/clothsim):
 *
 *   cs_create       <- gpu/engine.py:111-147  Engine.__init__ (+ _allocate
 *                      :151-191, _upload_static :193-244, params :246-285)
 *   cs_step         <- gpu/engine.py:304-344  Engine.step (passes of
 *                      gpu/kernels.py:81-339: zero_forces, spring_force,
 *                      integrate, detect_cloth_edges, detect_obstacle_edges,
 *                      respond, normal_update)
 *   cs_run_pass     <- the individual dispatches of engine.py:313-339
 *                      (debug snapshots, engine.py:315-337)
 *   cs_respond      <- gpu/engine.py:346-352  Engine.run_respond_pass
 *   cs_read         <- gpu/engine.py:362-378  read_positions / read_velocities /
 *                      read_normals / read_forces_raw / read_accumulator_raw /
 *                      read_counts
 *   cs_write        <- writes through Engine.buffers.pos/.vel (test hooks,
 *                      test_gpu_engine.py:99,201), set_external_accel
 *                      (engine.py:297-302), inject_response (engine.py:354-358)
 *   cs_frame_stats  <- StepResult.hits / .responded (engine.py:100-105)
 *   cs_last_error   <- the reference's exception text
 *
 * All arguments are plain pointers and sizes.  Arrays passed to cs_create,
 * cs_write and cs_read are HOST arrays (row-major (N,3) float32 etc., the
 * reference's own buffer layouts); cs_read_device / cs_write_device take
 * DEVICE pointers (a PyTorch tensor's data_ptr()) in the same layouts and a
 * stream.  The library owns the engine's own device buffers (SoA planes).
 * One handle = one CUDA stream; calls on a handle are not thread-safe, as in
 * the reference.  Every function returns 0 on success or a
 * negative CS_E* code; cs_last_error() returns the message.
 */
#ifndef CLOTHSIM_B200_H
#define CLOTHSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CS_ABI_VERSION 1

/* error codes (map to the reference's exception types) */
#define CS_OK 0
#define CS_E_INVALID (-1)      /* ValueError */
#define CS_E_CAPACITY (-2)     /* gpu/layout.py CapacityError */
#define CS_E_BUDGET (-3)       /* collision.py CollisionBudgetError */
#define CS_E_NODEVICE (-4)     /* gpu/device.py AdapterUnavailable */
#define CS_E_CUDA (-5)         /* CUDA runtime error */

/* cs_desc.flags */
#define CS_FLAG_EXPLICIT_EULER 1u   /* engine.py:45 FLAG_EXPLICIT_EULER */
#define CS_FLAG_AVERAGE_RESPONSE 2u /* engine.py:46 FLAG_AVERAGE_RESPONSE */
#define CS_FLAG_FIXED_POINT 4u      /* reference-engine arithmetic: per-spring
                                       f32 forces accumulated as i32 at
                                       fixed_point_scale (kernels.py:86-110),
                                       bit-exact with the reference engine */
#define CS_FLAG_FP64 8u             /* float64 state and arithmetic (float
                                       gather only) */
#define CS_FLAG_NO_GRAPH 16u        /* launch passes eagerly instead of
                                       replaying a captured CUDA graph */
#define CS_FLAG_FORCE_CSR 32u       /* use the generic per-node CSR gather even
                                       when the topology is a regular grid */
#define CS_FLAG_TILE_KERNEL 64u     /* grid path: the shared-memory tile kernel
                                       (every node evaluates its 12 springs)
                                       instead of the warp-strip kernel */
#define CS_FLAG_SPLIT_NORMALS 512u  /* grid path: a stand-alone normals kernel
                                       after each frame instead of fusing the
                                       previous frame's normals into the step */
#define CS_FLAG_FUSE_NORMALS 1024u  /* grid path: fuse (the default at every
                                       size; kept for explicitness) */
#define CS_FLAG_THREAD_NARROW 256u  /* collision narrow phase: one thread per
                                       query (default: batched queries per
                                       warp, flattened over cells/candidates) */
#define CS_FLAG_WARP_NARROW 2048u   /* collision narrow phase: one warp per
                                       query */
#define CS_FLAG_SPLIT_NARROW 8192u  /* collision narrow phase: 32-query batches
                                       per warp, cloth edges (pass A) and cloth
                                       triangles (pass B) enumerated separately
                                       (default: one fused enumeration per
                                       cloth triangle serves both passes) */
#define CS_FLAG_MEMOP_SEAM 4096u  /* row bands: the stream-memop seam handshake
                                       (cuStreamWaitValue32 / WriteValue32
                                       around each pass, no graph) even where
                                       the fast kernel could do it in-kernel */
#define CS_FLAG_PAIRED 128u         /* fast mode: the paired-column f32x2
                                       warp-strip kernel (cs_pair3.cu, the
                                       production path; Engine kernel="pair")
                                       instead of the scalar strip kernel */

typedef struct cs_engine cs_engine;

typedef struct cs_desc {
    int32_t abi_version;       /* = CS_ABI_VERSION */
    uint32_t flags;
    /* grid topology: nx, ny > 0 selects the regular-grid stencil path, whose
       spring/triangle/edge order must be generate_cloth_grid's
       (mesh.py:223-317); grid_rest[6] are the single f32 rest lengths of
       (structural +i, structural +j, shear (1,1), shear (-1,1), bend +2i,
       bend +2j).  nx = ny = 0 selects the generic CSR path. */
    int32_t nx, ny;
    float grid_rest[6];
    int64_t num_nodes;
    /* springs (generic path; also used to build the CSR): (S,2) i32 endpoint
       pairs, (S,) i32 kinds, (S,) f32 rest lengths -- engine.py:204-213 */
    int64_t num_springs;
    const int32_t *springs;
    const int32_t *spring_kinds;
    const float *spring_rest;
    /* render triangulation (C,3) i32 and unique edges (E,2) i32 */
    int64_t num_tris;
    const int32_t *tris;
    int64_t num_edges;
    const int32_t *edges;
    /* initial state (N,3) f32 positions (construction pose) and (N,) f32
       inverse masses (0 = pinned) -- engine.py:199-202 */
    const float *positions;
    const double *positions64; /* optional, used by CS_FLAG_FP64 */
    const float *inv_mass;
    /* float64 solver-exact path (CS_FLAG_FP64): (N,) f64 masses, (N,) u8
       pinned flags and (S,) f64 rest lengths, as in solver.py:86-172 */
    const double *masses64;
    const uint8_t *pinned;
    const double *spring_rest64;
    /* obstacle: (T,3,3) f32 corners and (T,3) f32 unit face normals
       (engine.py:218-230) */
    int64_t num_obstacle_tris;
    const float *obstacle_corners;
    const float *obstacle_normals;
    /* SimParams (mesh.py:152-204) */
    double dt;                 /* per substep: params.dt / params.substeps */
    double gravity[3];
    double stiffness[3];       /* structural, shear, bend */
    double damping;
    float epsilon_mt;
    float response_margin;
    int32_t fixed_point_scale;
    int32_t substeps;
    /* broad phase: uniform grid cell edge; <= 0 picks one automatically */
    float cell_size;
    /* CUDA stream to launch on (cudaStream_t); NULL = the library creates
       its own non-blocking stream */
    void *stream;
    /* CS_FLAG_FP64 with an obstacle: (T,3,3) f64 corners and (T,3) f64 unit
       face normals, and the float64 epsilon_mt / response_margin, for the
       solver-exact collision (collision.py:243-346) */
    const double *obstacle_corners64;
    const double *obstacle_normals64;
    double epsilon_mt64;
    double response_margin64;
} cs_desc;

typedef struct cs_stats {
    int64_t hits;          /* edge-triangle hits of the last frame */
    int64_t responded;     /* nodes moved by the last respond pass */
    int64_t frames;        /* frames stepped since creation */
    int64_t hit_counter;   /* cumulative hitCounter buffer value */
} cs_stats;

/* buffer ids for cs_read / cs_write */
#define CS_BUF_POSITIONS 0      /* f32 (N,3) (f64 with CS_FLAG_FP64 via _64) */
#define CS_BUF_VELOCITIES 1
#define CS_BUF_NORMALS 2
#define CS_BUF_PREV_POSITIONS 3
#define CS_BUF_FORCES_RAW 4     /* i32 (N,3) spring-only fixed-point forces of
                                   the last spring_force pass */
#define CS_BUF_ACCUMULATOR 5    /* i32 (N,3) responseAccumulator */
#define CS_BUF_COUNTS 6         /* i32 (N,)  responseCount */
#define CS_BUF_EXT_ACCEL 7      /* f32 (N,3) externalAccel (write only) */
#define CS_BUF_POSITIONS64 8    /* f64 (N,3) (CS_FLAG_FP64 engines) */
#define CS_BUF_VELOCITIES64 9
#define CS_BUF_NORMALS_LAGGED 10 /* f32 (N,3) the normals the last fused step
                                    kernel produced -- those of the PREVIOUS
                                    frame's final state -- without the
                                    recompute CS_BUF_NORMALS does (a renderer
                                    that accepts a one-frame lag pays nothing) */

/* passes for cs_run_pass (engine.py:313-339) */
#define CS_PASS_FORCE_INTEGRATE 0 /* zero_forces + spring_force + integrate */
#define CS_PASS_DETECT 1          /* detect_cloth_edges + detect_obstacle_edges */
#define CS_PASS_RESPOND 2
#define CS_PASS_NORMALS 3

int cs_create(const cs_desc *desc, cs_engine **out);

/* ---- generate_cloth_grid on the device (mesh.py:223-317) ----
   A stencil engine straight from the grid's parameters: positions
   (np.linspace in float64, then the scene's orientation), uniform masses
   (total_mass / (nx*ny)), whole pinned rows and the six spring families'
   rest lengths are generated by kernels -- no per-node or per-spring host
   array, so a 4096^2 cloth builds in a fraction of a second (the reference's
   Python loops take minutes).  rows [row_lo, row_hi) of the global nx x ny
   grid form the local sheet (a row band; 0, ny for the whole cloth).
   orientation: 0 = the generation plane (x, 0, z); 1 = the hanging scene's
   (x, -z, 0) (scenes.py _rotate_xz_to_xy).  Fails with CS_E_INVALID when a
   spring family's rest lengths round to two float32 values (SURVEY.md
   finding 4) -- build from the mesh then.  Fast or fixed arithmetic only. */
typedef struct cs_grid_desc {
    int32_t abi_version;       /* = CS_ABI_VERSION */
    uint32_t flags;            /* cs_desc flags (CS_FLAG_FIXED_POINT, ...) */
    int32_t nx, ny;            /* the whole grid */
    int32_t row_lo, row_hi;    /* local rows */
    double width, height, total_mass;
    int32_t orientation;
    int32_t num_pinned_rows;   /* global row indices (mesh.py:320-331) */
    const int32_t *pinned_rows;
    double dt;                 /* per substep */
    double gravity[3];
    double stiffness[3];
    double damping;
    float epsilon_mt;
    float response_margin;
    int32_t fixed_point_scale;
    int32_t substeps;
    void *stream;
} cs_grid_desc;
int cs_create_grid(const cs_grid_desc *desc, cs_engine **out);
/* generate_cloth_grid's arrays of the local sheet (local node indices,
   nx x (row_hi - row_lo) nodes, the reference's orders) into DEVICE memory:
   springs (S,2) i32, kinds (S,) i32, rest (S,) f64, triangles (C,3) i32,
   positions (N,3) f64 in the generation plane; any output may be NULL. */
int cs_grid_topology(int32_t nx, int32_t ny, int32_t row_lo, int32_t row_hi, double width,
                     double height, int32_t *springs, int32_t *kinds, double *rest,
                     int32_t *tris, double *positions, void *stream);
int cs_destroy(cs_engine *h);
/* Advance `frames` whole frames (asynchronous on the engine's stream). */
int cs_step(cs_engine *h, int32_t frames);
int cs_run_pass(cs_engine *h, int32_t pass_id);
/* Advance `frames` frames, streaming every frame's positions ((N,3) f32) into
   host_out[frames][N][3]: `step(readback=True)` (engine.py:341-343) for a
   whole run, with each frame's device->host copy overlapping the next
   frame's computation.  host_out should be page-locked. */
int cs_record(cs_engine *h, int32_t frames, float *host_out);
/* Contact log for parity checks: record every (cloth node, obstacle
   triangle) contact of subsequent detect passes (collision.py:218-240
   Contact.nodes per hit); capacity 0 turns it off.  cs_read_contacts returns
   the last frame's pairs (node index, triangle) and their total count. */
int cs_contact_log(cs_engine *h, int64_t capacity);
int cs_read_contacts(cs_engine *h, int32_t *out, int64_t max, int64_t *n);
/* Respond pass alone; writes the responded count (synchronises). */
int cs_respond(cs_engine *h, int64_t *responded);
/* Synchronise and report the last frame's hit / respond counts. */
int cs_frame_stats(cs_engine *h, cs_stats *out);
/* Hits / responded of frame `frame` (0-based), kept on device in a ring of
   the last 4096 frames so a step never has to synchronise (engine.py:100-105
   StepResult fields, resolved lazily). */
int cs_frame_hits(cs_engine *h, int64_t frame, int64_t *hits, int64_t *responded);
int cs_read(cs_engine *h, int32_t buffer_id, void *host_dst);
int cs_write(cs_engine *h, int32_t buffer_id, const void *host_src);
/* Single node accumulator write (engine.py:354-358 inject_response). */
int cs_inject_response(cs_engine *h, int64_t node, const int32_t raw[3], int32_t count);
int cs_synchronize(cs_engine *h);
/* The engine's CUDA stream (cudaStream_t), for device-side timing. */
int cs_stream(cs_engine *h, void **stream);
/* Device pointer of a state plane for halo exchange / zero-copy interop:
   which = 0..5 -> x, y, z, vx, vy, vz of the CURRENT state; returns the
   pitch (elements per grid row) through *pitch. */
int cs_state_plane(cs_engine *h, int32_t which, void **dev_ptr, int64_t *pitch);
/* ---- row bands (BASELINE config 5; no reference counterpart -- the
   reference runs one WebGPU device) ----
   One engine per GPU holds owned rows [row_lo, row_hi) of its local sheet
   plus a 2-row halo each side (bend springs reach two rows, mesh.py:284-289;
   damping reads neighbour velocities, solver.py:117-119).  A neighbour is
   described by its two state buffers and flag words (cs_state_buffers; across
   processes through cs_ipc_export / cs_ipc_open), and the step kernel stores
   my rows [src_row0, src_row0+rows) straight into its rows
   [dst_row0, dst_row0+rows) -- the halo exchange happens inside the step, as
   peer stores over NVLink -- then signals `remote_flag` (the neighbour's flag
   word 0 if I am its upper neighbour, 1 if its lower one) with the passes it
   completed.  A force pass may read its halo / overwrite the neighbour's
   only after every neighbour finished the previous pass.  Fast
   collision-free bands with fused normals do this inside the step kernel:
   only the warps of the seam chunk rows wait (spinning on the flag words),
   the launch's last block signals, and frames replay a CUDA graph like a
   single engine's.  Otherwise (CS_FLAG_MEMOP_SEAM, fixed arithmetic, split
   normals, obstacles) the stream waits on / writes the flag words around
   each pass.  Link before the first frame; every band must step in lockstep.
   With an obstacle (replicated per band) a frame has three handshakes:
   post-step rows -> detect -> "detect done" -> respond -> post-respond rows.
   Drive each band from its own CUDA context (one process per GPU): inside
   one context a stream blocked on a flag that another stream of the same
   context has not written yet can stall the whole context. */
typedef struct cs_halo_peer {
    void *state[2];        /* the neighbour's state buffers (cs_state_buffers) */
    int64_t plane;         /* the neighbour's plane stride in elements */
    int64_t src_row0;      /* first of MY local rows sent to it */
    int64_t dst_row0;      /* where that row lands in ITS local rows */
    int64_t rows;          /* rows sent (the halo depth) */
    uint32_t *remote_flag; /* its flag word for me */
} cs_halo_peer;
/* The two ping-pong state buffers (6 planes each), the two flag words
   ([0] written by the upper neighbour, [1] by the lower), plane stride and
   pitch in elements. */
int cs_state_buffers(cs_engine *h, void **state0, void **state1, uint32_t **flags,
                     int64_t *plane, int64_t *pitch);
int cs_set_halo_peers(cs_engine *h, int64_t row_lo, int64_t row_hi, const cs_halo_peer *up,
                      const cs_halo_peer *down);
/* cudaIpcGetMemHandle / cudaIpcOpenMemHandle of an engine allocation
   (a state buffer or the flag words), as 64 opaque bytes. */
int cs_ipc_export(void *dev_ptr, uint8_t handle[64]);
int cs_ipc_open(const uint8_t handle[64], void **dev_ptr);
int cs_ipc_close(void *dev_ptr);
/* Number of kernels one cs_step(h, 1) launches. */
int cs_kernels_per_frame(cs_engine *h, int32_t *count);
/* Broad-phase statistics: cells, references, last frame's candidate pairs. */
int cs_broadphase_stats(cs_engine *h, int64_t out[4]);
/* The broad-phase grid itself, for the bit-exact grid-cell assignment
   check (north star; the reference brute-forces every pair, its prefilter
   test test_gpu_engine.py:267-307 is the contract): geometry[8] = origin
   xyz, 1/cell, cell edge (f32, rest 0); dims[3] = cells per axis; the sorted
   (cell key, triangle) references, cs_broadphase_stats out[1] of each; per
   cell [begin, end) into them, out[0] of each (0, 0 for an empty cell).
   Any output may be NULL.  Synchronises. */
int cs_broadphase_dump(cs_engine *h, float geometry[8], int32_t dims[3], uint32_t *ref_keys,
                       uint32_t *ref_tris, uint32_t *cell_begin, uint32_t *cell_end);
/* Number of visible CUDA devices (0 when no driver / device): the adapter
   probe of gpu/device.py:156-172 get_adapter. */
int cs_device_count(void);
/* Free / total device memory, for the capacity check (gpu/layout.py:192-202). */
int cs_mem_info(int64_t *free_bytes, int64_t *total_bytes);
/* Orthographic depth-shaded snapshot (replaces clothsim/io.py:225-287
   snapshot_png and :187-222 _rasterize), rendered on the device.  All
   pointers are DEVICE pointers.  verts: f64 (n, 3) -- the cloth vertices,
   then the obstacle's; tris: int32 (num_tris, 3) into verts -- the cloth's
   triangles first (material 1, num_cloth_tris of them), then the obstacle's
   (material 2).  cs_snapshot_bounds returns min xyz, max xyz of verts (host
   out[6]); the caller pads them and forms view = {lo_u, lo_v, scale} exactly
   as io.py:249-258 does.  axes = {u, v, depth} coordinate indices (io.py
   _VIEW_AXES).  rgb: u8 (height, width, 3); scratch: (2*width*height + 2)
   u64.  Bit-identical pixels to the reference (float64, numpy's operation
   order, strict-greater z test with earlier-triangle ties). */
int cs_snapshot_bounds(const double *verts, int64_t n, double out[6], void *stream);
/* ---- device-pointer boundary (PyTorch tensors: tensor.data_ptr(), the
   reference's readbacks gpu/engine.py:362-378 and writes through
   Engine.buffers / set_external_accel engine.py:297-302, without a host
   copy) ----
   cs_read_device transposes buffer `id` into DEVICE memory `dev_dst` in the
   reference's (N,3) row-major layout (N for CS_BUF_COUNTS): f32 for
   POSITIONS / VELOCITIES / PREV_POSITIONS / NORMALS / NORMALS_LAGGED (a
   float64 engine converts), f64 for POSITIONS64 / VELOCITIES64, i32 for
   ACCUMULATOR / COUNTS.  cs_write_device is the inverse for POSITIONS /
   VELOCITIES (f32), POSITIONS64 / VELOCITIES64 (f64, float64 engines) and
   EXT_ACCEL (f32).  Both are enqueued on `stream` (NULL = the engine's),
   ordered after the engine's earlier work and before its later work by
   events; neither synchronises the host nor touches host memory (the
   legacy default stream is cudaStreamLegacy, (void *)1).
   cs_set_stream moves the engine to another stream for every later call
   (work already enqueued on the old stream stays ordered before it). */
int cs_read_device(cs_engine *h, int32_t buffer_id, void *dev_dst, void *stream);
int cs_write_device(cs_engine *h, int32_t buffer_id, const void *dev_src, void *stream);
int cs_set_stream(cs_engine *h, void *stream);
/* The CUDA device ordinal the engine was created on (its buffers live there;
   device pointers passed to it must too). */
int cs_device(cs_engine *h, int32_t *device);
/* The engine's current positions as DEVICE float64 (N, 3), enqueued on the
   engine's stream (cs_stream): the snapshot's cloth vertices without a
   host round trip (bench.py:186 reads them back in the reference). */
int cs_positions_device(cs_engine *h, double *dev_out);
int cs_snapshot_render(const double *verts, const int32_t *tris, int64_t num_tris,
                       int64_t num_cloth_tris, const double view[3], const int32_t axes[3],
                       int32_t width, int32_t height, uint8_t *rgb, void *scratch, void *stream);
const char *cs_last_error(void);
int cs_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CLOTHSIM_B200_H */
