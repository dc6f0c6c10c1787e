// sm_100a kernels of the DS-Sync step.
//
// Bandwidth-bound elementwise/reduction work: no tensor cores.  Every
// kernel streams worker rows with 128-bit vector loads/stores, one thread
// per vector, grid sized in multiples of the 148 SMs.  The reduction axis is
// the *member* axis (group size <= 8 typically) and its order is pinned by
// the reference (param.hpp:21-24): acc = x_0; acc += x_k ascending;
// acc *= 1/m.  One thread owns an element vector and folds all members in
// registers in that order, so no tree/shuffle ever re-associates the sum.
//
// All arithmetic goes through explicit round-to-nearest intrinsics
// (__fadd_rn/__dmul_rn ...), which are never contracted into FMA, matching
// the reference's SSE2 build without FMA contraction.  The
// library is also compiled with -fmad=false.
#pragma once

#include "kernel_common.cuh"
#include "kernels_problems.cuh"
#include "kernels_step.cuh"
#include "kernels_fold.cuh"
