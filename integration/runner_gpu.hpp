// runner_gpu.hpp — the reference-side binding of the B200 path.
//
// blockgs::gpu::run_factor has exactly the signature and FactorOutcome semantics of the
// reference's run_factor (proj/include/blockgs/runner.hpp:28-29, proj/src/runner.cpp:39-67):
// distribute over `procs` ranks, run the variant, gather Q, measure LOO / residual with the
// reference's own metrics; NotSpd -> ok = false with the diagnostic; every other failure
// throws the matching blockgs error (errors.hpp:9-51).  The factorization itself runs on
// the GPU through the C ABI (include/bgs_gpu.h: bgs_factor_opts); BcgsOptions::probe is
// forwarded (RecurrenceProbe, bcgs.hpp:19-23).  A maintainer switches a caller over by
// calling gpu::run_factor instead of run_factor.
#pragma once

#include "blockgs/runner.hpp"

namespace blockgs::gpu {

FactorOutcome run_factor(VariantId v, const DenseMatrix& x, long s, int procs,
                         const BcgsOptions& opts = {});

}  // namespace blockgs::gpu
