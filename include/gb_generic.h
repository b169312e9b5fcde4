/* C ABI of the generic n-ary factor path, implemented in
 * paper_2509_26581_b200/csrc/generic.cu and linked into libgb_bal.so.
 *
 * The reference's generic engine is a C++ template API: VertexDescriptor<
 * Traits> (vertex_descriptor.hpp:50-56), FactorDescriptor<Traits> with a
 * templated residual and Auto (dual-number) Jacobians
 * (factor_descriptor.hpp:139-151, :610-624), Graph and levenberg_marquardt
 * (graph.hpp:35-45, levenberg_marquardt.hpp:115-224). The device engine runs
 * host-device traits (include/gb_generic_models.hpp) with the same algorithm;
 * each entry point below builds one model's graph from flat arrays, solves it
 * on `device`, and refines the binary64 vertex arrays in place (Traits::update,
 * additive). Config, report and records are the BAL path's structs
 * (gb_bal.h: LMConfig, SolveReport, IterationRecord). Status codes as in
 * gb_bal.h; gbg_last_error() returns the message. Precision: GB_FP64 or
 * GB_FP32 (<double,double>, <float,float>). */
#ifndef GB_GENERIC_H
#define GB_GENERIC_H

#include <stdint.h>

#include "gb_bal.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* gbg_last_error(void);

/* The reference's toy (toy/circle.hpp:30-55): n 2-D points (double[2n]),
 * factor i: e = x_i^2 + y_i^2 - radius[i]^2. */
int gbg_circle_solve(int precision, uint64_t n, double* points, const double* radius, const gb_lm_config* cfg,
                     int device, gb_solve_report* report, gb_iteration_record* records, int32_t max_records);

/* EuRoC-shaped visual-inertial BA (gb_generic_models.hpp "vi"): poses
 * double[6*npose] ([angle-axis body->world | position]; pose_fixed may be
 * NULL), velocity+biases double[9*nvb], landmarks double[3*nlm]; stereo
 * factors: st_idx uint32[2*nst] (pose, landmark), st_obs double[3*nst]
 * (uL, vL, uR), cam double[5] (fx, fy, cx, cy, baseline); IMU factors:
 * imu_idx uint32[4*nimu] (pose_i, vb_i, pose_j, vb_j), imu_obs double[19*nimu]
 * (dp[3], dv[3], dR[9] row-major, dt, 3 unused), gravity double[3]. */
int gbg_vi_solve(int precision, uint64_t npose, double* poses, const uint8_t* pose_fixed, uint64_t nvb, double* vbs,
                 uint64_t nlm, double* lms, uint64_t nst, const uint32_t* st_idx, const double* st_obs,
                 const double* cam, uint64_t nimu, const uint32_t* imu_idx, const double* imu_obs,
                 const double* gravity, const gb_lm_config* cfg, int device, gb_solve_report* report,
                 gb_iteration_record* records, int32_t max_records);

#ifdef __cplusplus
}
#endif

#endif
