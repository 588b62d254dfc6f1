// gnn.cuh -- device-resident message-passing GNN (internal).
#pragma once
#include <cstdint>
#include <string>

#include "../../include/npcg.h"
#include "pattern.h"

namespace npcg {

// Offsets (in floats) of every layer inside the fp32 device weight blob,
// which follows the reference's _layer_specs order (gnn.py:130-147) with
// l = l_mp = 1: W[fan_in][fan_out] row-major, then b[fan_out].
struct LayerOff {
    int64_t w = 0, b = 0;
};

struct GnnDev {
    npcg_gnn_desc d{};
    float *w = nullptr;  // device blob
    int64_t n_floats = 0;
    LayerOff node_enc[2], edge_enc[2], edge_dec[2], node_dec[2];
    LayerOff mp_node[16][2], mp_edge[16][2];
    // north_star LayerNorm gain (w) and shift (b) per stack
    LayerOff ln_node_enc, ln_edge_enc, ln_mp_node[16], ln_mp_edge[16];
    ~GnnDev();
};

// north_star mesh inputs (device, shared by the batch); null in reference mode
struct GnnMesh {
    const double *pos = nullptr;       // [n][dim]
    const double *boundary = nullptr;  // [n]
};

// Returns "" on success.
std::string gnn_init(GnnDev &g, const npcg_gnn_desc &d, const double *weights, int64_t n_weights);

// Runs the forward pass for B systems that share pattern A and writes the
// factor values. Returns a NPCG_* code; *pivot set for NPCG_ERR_NOT_SPD.
int gnn_build(const GnnDev &g, const Pattern &A, int B, const double *A_vals, int A_batched,
              const double *rhs, double *S, double *D, double *edge_out, double *x0_out, int64_t *pivot,
              cudaStream_t stream, std::string &err, const GnnMesh *mesh = nullptr);

}  // namespace npcg
