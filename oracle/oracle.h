/*
 * oracle.h — C interface shared by the two CPU oracles.  TEST INFRASTRUCTURE
 * ONLY: nothing in the product (paper_2204_12346_b200/) links or calls these;
 * only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * `--impl reference`) do, as the checker.
 *
 *   oracle/_ref/libsirdref.so   the reference itself (/root/reference/proj/src
 *                               compiled unmodified + ref_shim.cpp), built by
 *                               oracle/Makefile.  kind = "reference".
 *   oracle/libsirdoracle.so     sird_oracle.c, a plain-C restatement of the
 *                               reference algorithm.  kind = "port".
 *
 * Both export exactly these symbols, so a test can run the same call through
 * either library.  Status codes are the sg_status values of include/sirdgpu.h.
 * All arrays are row-major; params/positions are [beta1, beta2, t1, t2,
 * gamma, mu] (calibration.cpp:85-87); states are [S, I, R, D] per day.
 */
#ifndef SIRD_ORACLE_H
#define SIRD_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* pso.cpp:36-41 */
uint64_t oracle_mix_seed(uint64_t base, uint64_t index);
/* std::mt19937_64(seed): discard `skip` outputs, then write n raw outputs */
void oracle_mt_raw(uint64_t seed, uint64_t skip, size_t n, uint64_t* out);
/* pso.cpp:43-45 applied n times to mt19937_64(seed) */
void oracle_uniform01(uint64_t seed, size_t n, double* out);

/* integrate_euler (model.cpp:76-107); states: n_days x 4; *finite 0/1 */
int oracle_integrate(const double* params6, const double* init4, double population, int n_days, int substeps,
                     double* states, int* finite);

/* make_window_objective(...)(positions, 6, costs) (calibration.cpp:120-155) */
int oracle_eval_costs(int family, int metric, const double* infectious, const double* recovered,
                      const double* deaths, int n_days, const double* init4, double population, int substeps,
                      int n_threads, const double* positions, size_t n, double* costs);

/* optimize(config, bounds, window objective, repair) (pso.cpp:129-143).
 * Returns SG_ERR_ALL_INFEASIBLE (4) when optimize throws AllInfeasibleError;
 * history receives max_iters values in every case it gets that far. */
int oracle_fit_swarm(int family, int metric, const double* infectious, const double* recovered,
                     const double* deaths, int n_days, const double* init4, double population, int substeps,
                     int n_threads, const double* lower6, const double* upper6, uint64_t n_particles,
                     uint64_t max_iters, double inertia, double cognitive, double social, uint64_t seed,
                     int repair, double* best6, double* best_cost, double* history);

/* forecast_extension's integration (calibration.cpp:305-317) from junction4 */
int oracle_forecast(const double* params6, const double* junction4, double population, int horizon, int substeps,
                    double* states, int* finite);

#ifdef __cplusplus
}
#endif

#endif
