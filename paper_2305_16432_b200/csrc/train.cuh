// train.cuh -- device training step (train.cu): loss + gradients of one
// tuple (train.py:189-205 + ad.backward) and Adam (train.py:164-185).
#pragma once
#include <cuda_runtime.h>

#include <string>

#include "../../include/npcg.h"
#include "pattern.h"

namespace npcg {

class TrainNet {
public:
    TrainNet();
    ~TrainNet();
    TrainNet(const TrainNet &) = delete;
    TrainNet &operator=(const TrainNet &) = delete;
    // weights: the reference's checkpoint layout (npcg_gnn_create). "" on success.
    std::string init(const npcg_gnn_desc &d, const double *weights, long long n_weights);
    long long n_weights() const;
    double *weights_dev() const;
    int set_weights(const double *host, int reset_moments);
    int tuple_grad(const Pattern &A, const double *A_vals, const double *node_in, const double *edge_in,
                   const double *b, const double *x, double x0_aux_weight, double *loss_host, double *grad_accum,
                   cudaStream_t st, std::string &err);
    int adam(const double *grad, double grad_scale, long long t, double lr, double b1, double b2, double eps,
             int *nonfinite, cudaStream_t st);

private:
    struct Impl;
    Impl *im;
};

}  // namespace npcg
