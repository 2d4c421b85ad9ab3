// integration/simdet_gpu.hpp -- the reference-side binding of libsdb: the
// simdet operator API (namespace simdet, /root/reference/proj/include) run on
// a B200 through the C ABI of include/sdb.h.  This is the translation unit a
// simdet maintainer adds to drop the GPU path in; every
// function keeps the reference signature, argument meaning and exception
// taxonomy (include/simdet/errors.hpp:9-40) of the function it replaces.
//
// Layout: reference Tensors are NCHW / OIHW float buffers (F16 = binary16
// values in floats, tensor.hpp:37-41); the shim stages them to device NHWC /
// KRSC (binary16 bits for F16) and back.  One libsdb context per host thread
// (the reference's one-CommGroup-per-rank rule, src/comm.cpp:242-245).
#pragma once

#include <span>
#include <utility>
#include <vector>

#include "simdet/memopt.hpp"
#include "simdet/syncbn.hpp"
#include "simdet/tensor.hpp"

struct sdb_ctx;

namespace simdet::gpu {

// this thread's libsdb context (device 0, rank 0, world 1), created on first use
sdb_ctx* context();

// simdet::conv2d (src/tensor.cpp:169-196): same ShapeErrors (conv2d_out_shape),
// output rounded to x.dtype()
Tensor conv2d(const Tensor& x, const Tensor& k, int stride, int pad);

// the Tape's conv2d backward rule (src/autograd.cpp:290-320): {dx, dk} as F32
// tensors.  dy is rounded to x.dtype() first (autograd.cpp:439).  In F16 the
// GPU finalises dx/dk in binary16 (the leaf-dtype rounding the tape applies
// to fp16 weights anyway, autograd.cpp:481), so values are binary16-valued.
std::pair<Tensor, Tensor> conv2d_backward(const Tensor& x, const Tensor& k, const Tensor& dy, int stride, int pad);

// syncbn_forward / syncbn_backward (src/syncbn.cpp:21-117) with group ==
// nullptr (plain BN).  BNStats carries count, the per-channel sums (float, as
// the reference's 2C+1 aggregation buffer) and mean/invstd.  A non-null group
// is a ContractError here: cross-GPU SyncBN runs over the ranks of a libsdb
// context created with an NCCL id (sdb_syncbn_fwd/bwd), not over a CommGroup.
std::pair<Tensor, BNStats> syncbn_forward(const Tensor& x, std::span<const float> gamma,
                                          std::span<const float> beta, float eps, CommGroup* group);
BnGrads syncbn_backward(const Tensor& dy, const Tensor& x, const BNStats& stats, std::span<const float> gamma,
                        CommGroup* group);

// iabn_forward / iabn_backward (src/memopt.cpp:226-327): NonInvertibleError
// for gamma == 0 or slope <= 0, DegenerateBatchError for N*H*W < 2; the
// backward recomputes from saved.y only
std::pair<Tensor, IabnSaved> iabn_forward(const Tensor& x, std::span<const float> gamma, std::span<const float> beta,
                                          float eps, float slope);
IabnGrads iabn_backward(const Tensor& dy, const IabnSaved& saved);

// has_nonfinite + apply_sgd of the step tail (src/trainer.cpp:78-94): in place
// on the fp32 masters and velocity, skipped (returns true) when gsum holds an
// inf/NaN; bitwise identical to the reference (explicit _rn arithmetic)
bool apply_sgd(std::span<float> w, std::span<float> v, std::span<const float> gsum, float lr, float momentum,
               double scale, int K);

}  // namespace simdet::gpu
