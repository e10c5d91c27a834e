// cs_collide64.cuh -- float64, solver-exact collision (cs_collide64.cu).
#pragma once
#include "cs_collide.cuh"

namespace cs {

struct Detect64Args {
    const double *pos;  // float64 state planes (x y z vx vy vz), node-indexed
    int64_t plane;
    const double *corners;  // (T,3,3) float64 obstacle corners
    const double *normals;  // (T,3) float64 unit face normals
    int64_t nt, nc;
    double eps, margin;     // SimParams.epsilon_mt / response_margin as float64
    float pad;              // broad-phase pad of the float32 query boxes
    // contact output (filled by launch_detect64)
    uint32_t *node, *klo, *khi;
    double *off;
    uint32_t *count;
    uint32_t cap;
    // optional (node, obstacle triangle) contact log (cs_contact_log)
    uint32_t *clog, *clog_n;
    uint32_t clog_cap;
};

// Contact buffers: node, serial-order key (hi/lo words), offset, plus sort
// scratch; grown by the host when a detect pass overflows.
struct Contacts64 {
    uint32_t *node = nullptr, *klo = nullptr, *khi = nullptr;
    double *off = nullptr;
    uint32_t *sort[4] = {nullptr, nullptr, nullptr, nullptr};
    uint32_t *count = nullptr;
    int64_t cap = 0;
    int reserve(int64_t want);
    void release();
};

void launch_detect64(Contacts64 &C, const Detect64Args &D, const BroadPhase &bp,
                     const int32_t *edges, int64_t ne, const int32_t *tris, int64_t nc,
                     unsigned long long *frame_hits, cudaStream_t st);
// sort the n contacts by (node, key) and apply the response; synchronises
void launch_respond64(Contacts64 &C, uint32_t n, int node_bits, double *state, int64_t plane,
                      const uint8_t *pinned, int average, unsigned long long *frame_responded,
                      cudaStream_t st);

}  // namespace cs
