/*
 * oracle_api.h -- TEST INFRASTRUCTURE ONLY.
 *
 * C interface of the two CPU checkers that live under oracle/:
 *   - liboracle.so  (oracle/dc_oracle.cpp): this repo's own CPU restatement of the
 *     reference algorithm for the hot path.
 *   - _ref/libdcref.so (oracle/ref_shim.cpp): the reference's own header-only C++
 *     operators compiled unchanged from /root/reference/proj/include, used to pin the
 *     restatement (and as the CPU baseline of bench.py --impl reference).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may load these.
 * The product (paper_1910_01031_b200/libdriftcast_gpu.so) never links or calls them.
 *
 * Parameter block layout is identical to dc_config in include/driftcast_gpu.h so the
 * tests can pass one ctypes struct to both.
 */
#ifndef DRIFTCAST_ORACLE_API_H
#define DRIFTCAST_ORACLE_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_params {
    int32_t nx, ny;           /* ModelGrid (grid.hpp:11-29) */
    double dx, dy;
    double g, f, h_eq;        /* PhysParams (grid.hpp:31-42) */
    double courant, limiter_theta, model_dt; /* SchemeParams (swe.hpp:16-30) */
    double q0, l0;            /* ErrorParams (stochastic.hpp:17-32) */
    int32_t c_omega;          /* CoarseGrid factor (grid.hpp:74-96) */
    int32_t c_soar;           /* fixed 2 (stochastic.hpp:20) */
    uint64_t seed;            /* experiment master seed (rng.hpp:35) */
    int32_t exact_fp;         /* ignored by the CPU checkers */
    int32_t reserved;
} orc_params;

#ifdef __cplusplus
}
#endif

#endif
