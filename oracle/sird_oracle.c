/*
 * sird_oracle.c — plain-C restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h): the checker the CUDA path is
 * compared against, never the product.  Parity of this file with the
 * reference itself is pinned by tests/test_oracle.py against the golden
 * vectors in tests/golden/ (generated from the reference build,
 * oracle/gen_golden.py) and, when oracle/_ref is present, call by call.
 *
 * Build with -ffp-contract=off (oracle/Makefile): every multiply and add
 * below is rounded separately, in the reference's order.  Each function
 * cites the reference lines it restates (/root/reference/proj/...).
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

enum { FAM_D = 0, FAM_IRD = 1 };
enum { M_MXSE = 0, M_MSE = 1, M_MAE = 2, M_MAPE = 3 };

/* ---- random streams ----------------------------------------------------- */

/* src/pso.cpp:36-41 — SplitMix64 finalizer of base + golden*(index+1) */
uint64_t oracle_mix_seed(uint64_t base, uint64_t index) {
    uint64_t z = base + 0x9E3779B97F4A7C15ULL * (index + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* std::mt19937_64 as specified by [rand.eng.mers] / [rand.predef]
 * (w=64, n=312, m=156, r=31, a=0xB5026F5AA96619E9, u=29, d=0x5555555555555555,
 *  s=17, b=0x71D67FFFEDA60000, t=37, c=0xFFF7EEE000000000, l=43,
 *  f=6364136223846793005); used by the reference at include/sirdfit/pso.hpp:79. */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static void mt64_twist(mt64* g) {
    for (int i = 0; i < 312; ++i) {
        const uint64_t y = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
        g->mt[i] = g->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    }
    g->idx = 0;
}

static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) mt64_twist(g);
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* src/pso.cpp:43-45 */
static double uniform01(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }

void oracle_mt_raw(uint64_t seed, uint64_t skip, size_t n, uint64_t* out) {
    mt64 g;
    mt64_seed(&g, seed);
    for (uint64_t k = 0; k < skip; ++k) (void)mt64_next(&g);
    for (size_t k = 0; k < n; ++k) out[k] = mt64_next(&g);
}

void oracle_uniform01(uint64_t seed, size_t n, double* out) {
    mt64 g;
    mt64_seed(&g, seed);
    for (size_t k = 0; k < n; ++k) out[k] = uniform01(&g);
}

/* ---- integrator ----------------------------------------------------------- */

/* src/model.cpp:55-64 */
static double beta_at(const double* p, double t) {
    if (t < p[2]) return p[0];
    if (t >= p[3]) return p[1];
    const double slope = (p[1] - p[0]) / (p[3] - p[2]);
    return p[0] + slope * (t - p[2]);
}

/* src/model.cpp:76-107 — states: n_days x 4, NaN after a blow-up */
int oracle_integrate(const double* p, const double* init, double N, int n_days, int substeps, double* states,
                     int* finite) {
    if (n_days < 1 || substeps < 1 || !(N > 0.0)) return 1; /* model.cpp:78-80 */
    for (int k = 0; k < 4 * n_days; ++k) states[k] = NAN;
    memcpy(states, init, 4 * sizeof(double));
    *finite = isfinite(init[0] + init[1] + init[2] + init[3]); /* SirdState::total, model.hpp:31 */
    if (!*finite) return 0;
    const double h = 1.0 / (double)substeps;
    double S = init[0], I = init[1], R = init[2], D = init[3];
    for (int day = 1; day < n_days; ++day) {
        for (int sub = 0; sub < substeps; ++sub) {
            const double t = (double)(day - 1) + (double)sub * h;
            /* sird_rhs, model.cpp:66-74 */
            const double inf = beta_at(p, t) / N * S * I;
            const double dS = -inf;
            const double dI = inf - p[4] * I - p[5] * I;
            const double dR = p[4] * I;
            const double dD = p[5] * I;
            S += h * dS;
            I += h * dI;
            R += h * dR;
            D += h * dD;
        }
        if (!isfinite(S) || !isfinite(I) || !isfinite(R) || !isfinite(D)) {
            *finite = 0;
            return 0;
        }
        states[4 * day + 0] = S;
        states[4 * day + 1] = I;
        states[4 * day + 2] = R;
        states[4 * day + 3] = D;
    }
    return 0;
}

/* ---- objectives --------------------------------------------------------- */

static double dmax(double a, double b) { return a < b ? b : a; } /* std::max */

/* src/objectives.cpp:15-39; stride picks one compartment of the states */
static double metric_scaled(int metric, const double* obs, const double* states, int comp, int n, double scale) {
    double acc = 0.0;
    for (int k = 0; k < n; ++k) {
        const double e = (obs[k] - states[4 * k + comp]) * scale;
        if (metric == M_MXSE) acc = dmax(acc, e * e);
        else if (metric == M_MSE) acc += e * e;
        else if (metric == M_MAE) acc += fabs(e);
    }
    if (metric == M_MSE || metric == M_MAE) acc /= (double)n;
    return acc;
}

/* src/objectives.cpp:41-55 */
static double mape(const double* obs, const double* states, int comp, int n) {
    double acc = 0.0;
    size_t kept = 0;
    for (int k = 0; k < n; ++k) {
        if (obs[k] == 0.0) continue;
        acc += fabs((obs[k] - states[4 * k + comp]) / obs[k]);
        ++kept;
    }
    if (kept == 0) return INFINITY;
    return 100.0 * acc / (double)kept;
}

/* src/objectives.cpp:61-69 */
static double compartment_cost(int metric, const double* obs, const double* states, int comp, int n) {
    if (metric == M_MAPE) return mape(obs, states, comp, n);
    double lo = obs[0], hi = obs[0]; /* std::minmax_element: first min, last max */
    for (int k = 1; k < n; ++k) {
        if (obs[k] < lo) lo = obs[k];
        if (!(obs[k] < hi)) hi = obs[k];
    }
    const double range = hi - lo;
    const double scale = range > 0.0 ? 1.0 / range : 1.0 / dmax(1.0, fabs(lo));
    return metric_scaled(metric, obs, states, comp, n, scale);
}

/* src/objectives.cpp:95-120 (observed I, R, D; states of a trajectory) */
static double objective_value(int family, int metric, const double* I, const double* R, const double* D, int n,
                              const double* states, int finite) {
    if (!finite) return INFINITY;
    if (family == FAM_D) {
        if (metric == M_MAPE) return mape(D, states, 3, n);
        return metric_scaled(metric, D, states, 3, n, 1.0);
    }
    double worst = compartment_cost(metric, I, states, 1, n);
    worst = dmax(worst, compartment_cost(metric, R, states, 2, n));
    worst = dmax(worst, compartment_cost(metric, D, states, 3, n));
    return worst;
}

/* ---- window objective (src/calibration.cpp:120-155) ----------------------- */

typedef struct {
    int family, metric, n_days, substeps;
    const double *I, *R, *D, *init;
    double N;
    const double* positions;
    double* costs;
    size_t begin, end;
} eval_job;

static void* eval_range(void* arg) {
    eval_job* j = (eval_job*)arg;
    double* states = (double*)malloc(sizeof(double) * 4 * (size_t)j->n_days);
    for (size_t k = j->begin; k < j->end; ++k) {
        int finite = 0;
        oracle_integrate(j->positions + 6 * k, j->init, j->N, j->n_days, j->substeps, states, &finite);
        j->costs[k] = objective_value(j->family, j->metric, j->I, j->R, j->D, j->n_days, states, finite);
    }
    free(states);
    return NULL;
}

/* static contiguous chunks like parallel_for (src/model.cpp:15-53); results
 * do not depend on the thread count. */
int oracle_eval_costs(int family, int metric, const double* I, const double* R, const double* D, int n_days,
                      const double* init4, double N, int substeps, int n_threads, const double* positions, size_t n,
                      double* costs) {
    if (n_days < 1 || substeps < 1 || !(N > 0.0)) return 1;
    if (n == 0) return 0;
    if (n_threads < 1) n_threads = 1;
    if ((size_t)n_threads > n) n_threads = (int)n;
    eval_job jobs[256];
    pthread_t th[256];
    if (n_threads > 256) n_threads = 256;
    const size_t chunk = (n + (size_t)n_threads - 1) / (size_t)n_threads;
    for (int w = 0; w < n_threads; ++w) {
        eval_job j = {family, metric, n_days, substeps, I, R, D, init4, N, positions, costs, 0, 0};
        j.begin = (size_t)w * chunk < n ? (size_t)w * chunk : n;
        j.end = j.begin + chunk < n ? j.begin + chunk : n;
        jobs[w] = j;
    }
    for (int w = 1; w < n_threads; ++w) pthread_create(&th[w], NULL, eval_range, &jobs[w]);
    eval_range(&jobs[0]);
    for (int w = 1; w < n_threads; ++w) pthread_join(th[w], NULL);
    return 0;
}

/* ---- particle swarm (src/pso.cpp:47-143) ---------------------------------- */

static void repair_time_order(double* x) { /* src/calibration.cpp:89-93 */
    if (x[2] > x[3]) {
        const double t = x[2];
        x[2] = x[3];
        x[3] = t;
    }
}

static double clamp(double v, double lo, double hi) { /* std::clamp */
    return v < lo ? lo : (hi < v ? hi : v);
}

int oracle_fit_swarm(int family, int metric, const double* I, const double* R, const double* D, int n_days,
                     const double* init4, double N, int substeps, int n_threads, const double* lo, const double* hi,
                     uint64_t n, uint64_t max_iters, double w, double c1, double c2, uint64_t seed, int repair,
                     double* best6, double* best_cost_out, double* history) {
    /* PsoConfig::validate / SearchBounds::validate, pso.cpp:16-34 */
    if (n == 0 || max_iters == 0 || !isfinite(w) || !isfinite(c1) || !isfinite(c2)) return 1;
    for (int d = 0; d < 6; ++d)
        if (!isfinite(lo[d]) || !isfinite(hi[d]) || lo[d] > hi[d]) return 1;
    mt64* eng = (mt64*)malloc(sizeof(mt64) * n);
    double* x = (double*)malloc(sizeof(double) * 6 * n);
    double* v = (double*)calloc(6 * n, sizeof(double));
    double* pb = (double*)malloc(sizeof(double) * 6 * n);
    double* pbc = (double*)malloc(sizeof(double) * n);
    double* cost = (double*)malloc(sizeof(double) * n);
    double gb[6] = {0, 0, 0, 0, 0, 0};
    double gbc = INFINITY;
    /* Swarm::Swarm, pso.cpp:47-75 */
    for (uint64_t i = 0; i < n; ++i) {
        mt64_seed(&eng[i], oracle_mix_seed(seed, i));
        pbc[i] = INFINITY;
        for (int d = 0; d < 6; ++d) x[6 * i + d] = lo[d] + uniform01(&eng[i]) * (hi[d] - lo[d]);
        if (repair) repair_time_order(x + 6 * i);
    }
    memcpy(pb, x, sizeof(double) * 6 * n);
    int rc = 0;
    for (uint64_t it = 0; it < max_iters; ++it) {
        /* Swarm::step, pso.cpp:77-101 */
        rc = oracle_eval_costs(family, metric, I, R, D, n_days, init4, N, substeps, n_threads, x, n, cost);
        if (rc) break;
        for (uint64_t i = 0; i < n; ++i)
            if (cost[i] < pbc[i]) {
                pbc[i] = cost[i];
                memcpy(pb + 6 * i, x + 6 * i, 6 * sizeof(double));
            }
        for (uint64_t i = 0; i < n; ++i)
            if (pbc[i] < gbc) {
                gbc = pbc[i];
                memcpy(gb, pb + 6 * i, 6 * sizeof(double));
            }
        /* Swarm::move_particles, pso.cpp:103-127 */
        const int have_best = gbc < INFINITY;
        for (uint64_t i = 0; i < n; ++i) {
            double* xi = x + 6 * i;
            double* vi = v + 6 * i;
            const double* pbi = pb + 6 * i;
            for (int d = 0; d < 6; ++d) {
                const double r1 = uniform01(&eng[i]);
                const double r2 = uniform01(&eng[i]);
                double vel = w * vi[d] + c1 * r1 * (pbi[d] - xi[d]);
                if (have_best) vel += c2 * r2 * (gb[d] - xi[d]);
                vi[d] = vel;
                xi[d] = clamp(xi[d] + vel, lo[d], hi[d]);
            }
            if (repair) repair_time_order(xi);
        }
        history[it] = gbc;
    }
    memcpy(best6, gb, sizeof gb);
    *best_cost_out = gbc;
    free(eng);
    free(x);
    free(v);
    free(pb);
    free(pbc);
    free(cost);
    if (rc) return rc;
    return gbc < INFINITY ? 0 : 4; /* optimize, pso.cpp:137-139 */
}

/* ---- forecast (src/calibration.cpp:298-322) ------------------------------- */

int oracle_forecast(const double* p, const double* junction4, double N, int horizon, int substeps, double* states,
                    int* finite) {
    const double held[6] = {p[1], p[1], 0.0, 0.0, p[4], p[5]}; /* calibration.cpp:305-312 */
    return oracle_integrate(held, junction4, N, horizon + 1, substeps, states, finite);
}
