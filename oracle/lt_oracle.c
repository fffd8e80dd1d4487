/*
 * oracle/lt_oracle.c — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain-C restatement of the reference's ∇G hot path, used only by tests/,
 * __graft_entry__.smoke() and bench.py's CPU baseline as the CHECKER of the
 * CUDA engine (never as the engine). Every function cites the reference code
 * it restates (paths relative to /root/reference/proj/include/lanetape/).
 *
 * Parity pin: tests/test_oracle.py checks this file against
 *   - the Random123 Philox KATs, uniform endpoints, AS241 points and the
 *     hand-derived draws of tests/test_rng.cpp (committed in tests/golden/),
 *   - the desk-checked Euler step of tests/test_heston.cpp:50-106,
 *   - the hand-checked two-pass case of tests/test_expectation.cpp:113-134,
 *   - and, bit for bit, the reference library itself compiled into
 *     oracle/_ref/libltref.so (oracle/ref_driver.cpp) on small configs.
 * The arithmetic below replays the reference's tape node order exactly
 * (forward: record_heston_program, heston.hpp:293-323; reverse:
 * reverse_seeded / Kernel::reverse_impl, tape.hpp:344-413,
 * kernel.hpp:212-288), so per-path outputs and adjoints are bitwise equal to
 * the reference's, and the BatchSums accumulation order
 * (expectation.hpp:109-122, 181-191, 239-244) makes the totals bitwise equal
 * as well.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/lanetape_b200.h"

/* ---- rng.hpp ---------------------------------------------------------- */

/* Philox4x32::block, rng.hpp:19-31 */
void lto_philox_block(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* uniform_from_bits, rng.hpp:38-40 */
double lto_uniform(uint32_t w0, uint32_t w1) {
    return ((w0 >> 6) * 67108864.0 + (w1 >> 6) + 0.5) * (1.0 / 4503599627370496.0);
}

/* inverse_normal_cdf (AS241 / PPND16), rng.hpp:45-85. Returns 1 on domain
 * error (the reference throws std::domain_error). */
int lto_inverse_normal_cdf(double p, double* out) {
    if (!(p > 0.0 && p < 1.0)) return 1;
    const double q = p - 0.5;
    if (fabs(q) <= 0.425) {
        const double r = 0.180625 - q * q;
        *out = q *
               (((((((2.5090809287301226727e+3 * r + 3.3430575583588128105e+4) * r +
                     6.7265770927008700853e+4) * r + 4.5921953931549871457e+4) * r +
                   1.3731693765509461125e+4) * r + 1.9715909503065514427e+3) * r +
                 1.3314166789178437745e+2) * r + 3.3871328727963666080e+0) /
               (((((((5.2264952788528545610e+3 * r + 2.8729085735721942674e+4) * r +
                     3.9307895800092710610e+4) * r + 2.1213794301586595867e+4) * r +
                   5.3941960214247511077e+3) * r + 6.8718700749205790830e+2) * r +
                 4.2313330701600911252e+1) * r + 1.0);
        return 0;
    }
    double r = q < 0.0 ? p : 1.0 - p;
    r = sqrt(-log(r));
    double value;
    if (r <= 5.0) {
        r -= 1.6;
        value = (((((((7.74545014278341407640e-4 * r + 2.27238449892691845833e-2) * r +
                      2.41780725177450611770e-1) * r + 1.27045825245236838258e+0) * r +
                    3.64784832476320460504e+0) * r + 5.76949722146069140550e+0) * r +
                  4.63033784615654529590e+0) * r + 1.42343711074968357734e+0) /
                (((((((1.05075007164441684324e-9 * r + 5.47593808499534494600e-4) * r +
                      1.51986665636164571966e-2) * r + 1.48103976427480074590e-1) * r +
                    6.89767334985100004550e-1) * r + 1.67638483018380384940e+0) * r +
                  2.05319162663775882187e+0) * r + 1.0);
    } else {
        r -= 5.0;
        value = (((((((2.01033439929228813265e-7 * r + 2.71155556874348757815e-5) * r +
                      1.24266094738807843860e-3) * r + 2.65321895265761230930e-2) * r +
                    2.96560571828504891230e-1) * r + 1.78482653991729133580e+0) * r +
                  5.46378491116411436990e+0) * r + 6.65790464350110377720e+0) /
                (((((((2.04426310338993978564e-15 * r + 1.42151175831644588870e-7) * r +
                      1.84631831751005468180e-5) * r + 7.86869131145613259100e-4) * r +
                    1.48753612908506148525e-2) * r + 1.36929880922735805310e-1) * r +
                  5.99832206555887937690e-1) * r + 1.0);
    }
    *out = q < 0.0 ? -value : value;
    return 0;
}

/* PhiloxNormalSource::fill, rng.hpp:113-127 */
void lto_fill_normals(uint64_t seed, size_t dim, int antithetic, uint64_t path, double* out) {
    const uint64_t base = antithetic ? path / 2 : path;
    const double sign = (antithetic && (path & 1u)) ? -1.0 : 1.0;
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    for (size_t pair = 0; 2 * pair < dim; ++pair) {
        const uint32_t ctr[4] = {(uint32_t)base, (uint32_t)(base >> 32), (uint32_t)pair,
                                 0x6C616E65u};
        uint32_t w[4];
        double z;
        lto_philox_block(ctr, key, w);
        lto_inverse_normal_cdf(lto_uniform(w[0], w[1]), &z);
        out[2 * pair] = sign * z;
        if (2 * pair + 1 < dim) {
            lto_inverse_normal_cdf(lto_uniform(w[2], w[3]), &z);
            out[2 * pair + 1] = sign * z;
        }
    }
}

/* ---- heston.hpp -------------------------------------------------------- */

/* floor_index, heston.hpp:72-76: largest i with nodes[i] <= x, clamped to 0 */
static size_t floor_index(const double* nodes, size_t n, double x) {
    size_t cnt = 0; /* upper_bound */
    while (cnt < n && nodes[cnt] <= x) ++cnt;
    return cnt == 0 ? 0 : cnt - 1;
}

size_t lto_heston_num_params(const ltg_heston_model* m) {
    return 5 + (size_t)m->n_t_nodes * m->n_s_nodes;
}

/* One path of the program record_heston_program records (heston.hpp:245-325)
 * replayed in node order, then its seeded reverse sweep (tape.hpp:344-413)
 * in reverse node order. x = [kappa, theta, xi, rho, v0, L row-major]
 * (pack_params, heston.hpp:212-219); z = 2*steps draws, slot 2k drives V and
 * slot 2k+1 the independent part of S (heston.hpp:301-302). y gets the m
 * payoffs; adj (may be NULL) gets the M parameter adjoints of lambda.y.
 * Returns 2 on a domain error (sqrt of a negative; the reference throws
 * EvalError), else 0. */
int lto_heston_path(const ltg_heston_model* m, const double* x, const double* z,
                    const double* lambda, double* y, double* adj) {
    const size_t steps = m->steps, cols = m->n_s_nodes;
    const double kappa = x[0], theta = x[1], xi = x[2], rho = x[3], v0 = x[4];
    const double* lev = x + 5;
    const double dt = m->dt, sqdt = sqrt(dt), mu_dt = m->mu * dt, half_dt = 0.5 * dt;
    /* rho_comp = sqrt(1 - rho*rho) * sqrt(dt)  (heston.hpp:286) */
    const double rr = rho * rho, u = 1.0 - rr;
    if (u < 0.0) return 2;
    const double sqrtu = sqrt(u), rho_comp = sqrtu * sqdt;

    /* per step pre-state and intermediates kept for the reverse sweep */
    double* S = (double*)malloc(sizeof(double) * (steps + 1));
    double* V = (double*)malloc(sizeof(double) * (steps + 1));
    double* E = (double*)malloc(sizeof(double) * steps);
    size_t* cell = (size_t*)malloc(sizeof(size_t) * steps);
    S[0] = m->s0;
    V[0] = v0;
    for (size_t k = 0; k < steps; ++k) {
        const double Vp = V[k] > 0.0 ? V[k] : 0.0;
        const size_t row = floor_index(m->t_nodes, m->n_t_nodes, (double)k * dt);
        size_t col = 0;
        for (size_t j = 1; j < cols; ++j)
            if (S[k] - m->s_nodes[j] >= 0.0) col = j; /* select_ge chain, heston.hpp:297-298 */
        cell[k] = row * cols + col;
        const double L = lev[cell[k]];
        const double sqrtV = sqrt(Vp);
        const double dWv = sqdt * z[2 * k];
        const double dWs = rho * dWv + rho_comp * z[2 * k + 1];
        const double L2 = L * L;
        const double drift = mu_dt - half_dt * (Vp * L2);
        const double diffusion = (sqrtV * L) * dWs;
        E[k] = exp(drift + diffusion);
        S[k + 1] = S[k] * E[k];
        const double mean_rev = (kappa * (theta - Vp)) * dt;
        const double vol_of_vol = (xi * sqrtV) * dWv;
        V[k + 1] = V[k] + (mean_rev + vol_of_vol);
    }
    for (uint32_t i = 0; i < m->n_instruments; ++i) {
        const double s = S[m->inst_maturity_step[i]], K = m->inst_strike[i];
        const double d = m->inst_kind[i] == LTG_PUT ? K - s : s - K;
        y[i] = d > 0.0 ? d : 0.0;
    }
    if (adj) {
        const size_t M = lto_heston_num_params(m);
        double a_kappa = 0, a_theta = 0, a_xi = 0, a_rho = 0, a_rc = 0;
        for (size_t j = 0; j < M; ++j) adj[j] = 0.0;
        double* aS = (double*)calloc(steps + 1, sizeof(double));
        /* payoff nodes come last on the tape, so they are reversed first,
         * in reverse instrument order (outputs seeded with lambda, :214-218) */
        for (size_t ii = m->n_instruments; ii-- > 0;) {
            const size_t ms = m->inst_maturity_step[ii];
            const double s = S[ms], K = m->inst_strike[ii];
            const double d = m->inst_kind[ii] == LTG_PUT ? K - s : s - K;
            const double a_sub = 0.0 + (d > 0.0 ? lambda[ii] : 0.0); /* max_zero */
            if (m->inst_kind[ii] == LTG_PUT)
                aS[ms] -= a_sub; /* sub(strike, s): arg1 -= bar */
            else
                aS[ms] += a_sub;
        }
        double aV = 0.0; /* adjoint of V_{k+1} */
        for (size_t k = steps; k-- > 0;) {
            const double Vp = V[k] > 0.0 ? V[k] : 0.0;
            const double L = lev[cell[k]];
            const double sqrtV = sqrt(Vp);
            const double dWv = sqdt * z[2 * k];
            const double tA = rho * dWv, tB = rho_comp * z[2 * k + 1];
            const double dWs = tA + tB;
            const double L2 = L * L;
            const double tE = sqrtV * L;
            const double tG = theta - Vp, tI = xi * sqrtV;
            /* V_{k+1} = add(V_k, tJ) */
            double aVk = 0.0 + aV;
            const double a_tJ = aV;
            /* tJ = add(mr, vv) */
            const double a_mr = a_tJ, a_vv = a_tJ;
            /* vv = mul(tI, dWv) */
            const double a_tI = 0.0 + a_vv * dWv;
            double a_dWv = 0.0 + a_vv * tI;
            /* tI = mul(xi, sqrtV) */
            a_xi += a_tI * sqrtV;
            double a_sqrtV = 0.0 + a_tI * xi;
            /* mr = mul(tH, c_dt) */
            const double a_tH = 0.0 + a_mr * dt;
            /* tH = mul(kappa, tG) */
            a_kappa += a_tH * tG;
            const double a_tG = 0.0 + a_tH * kappa;
            /* tG = sub(theta, Vp) */
            a_theta += a_tG;
            double a_Vp = 0.0 - a_tG;
            /* S_{k+1} = mul(S_k, E) */
            const double a_S1 = aS[k + 1];
            aS[k] += a_S1 * E[k];
            const double a_E = 0.0 + a_S1 * S[k];
            /* E = exp(tF) */
            const double a_tF = 0.0 + a_E * E[k];
            /* tF = add(drift, diffusion) */
            const double a_drift = a_tF, a_diff = a_tF;
            /* diffusion = mul(tE, dWs) */
            const double a_tE = 0.0 + a_diff * dWs;
            const double a_dWs = 0.0 + a_diff * tE;
            /* tE = mul(sqrtV, L). With one s-node L IS the parameter input
             * node and its contributions land on the parameter adjoint
             * directly; otherwise they collect on the last select node. */
            a_sqrtV += a_tE * L;
            double* aLp = cols == 1 ? &adj[5 + cell[k]] : NULL;
            double a_L = 0.0;
            if (aLp) *aLp += a_tE * sqrtV; else a_L += a_tE * sqrtV;
            /* drift = sub(c_mu_dt, tD) */
            const double a_tD = 0.0 - a_drift;
            /* tD = mul(c_half_dt, tC) */
            const double a_tC = 0.0 + a_tD * half_dt;
            /* tC = mul(Vp, L2) */
            a_Vp += a_tC * L2;
            const double a_L2 = 0.0 + a_tC * Vp;
            /* L2 = mul(L, L): both operand slots */
            if (aLp) {
                *aLp += a_L2 * L;
                *aLp += a_L2 * L;
            } else {
                a_L += a_L2 * L;
                a_L += a_L2 * L;
            }
            /* dWs = add(tA, tB) */
            const double a_tA = a_dWs, a_tB = a_dWs;
            /* tB = mul(rho_comp, z2) */
            a_rc += a_tB * z[2 * k + 1];
            /* tA = mul(rho, dWv) */
            a_rho += a_tA * dWv;
            a_dWv += a_tA * rho;
            (void)a_dWv; /* flows to the random input only */
            /* sqrtV = sqrt(Vp), derivative 0 at 0 (tape.hpp:386-390) */
            if (sqrtV > 0.0) a_Vp += a_sqrtV * 0.5 / sqrtV;
            /* select chain: the adjoint reaches the taken leverage cell only */
            if (!aLp) adj[5 + cell[k]] += a_L;
            /* Vp = max_zero(V_k) */
            if (V[k] > 0.0) aVk += a_Vp;
            aV = aVk;
        }
        /* rho_comp = mul(sqrt(sub(1, mul(rho, rho))), c_sqrt_dt) — recorded
         * before the loop, so reversed last */
        const double a_sqrtu = 0.0 + a_rc * sqdt;
        double a_u = 0.0;
        if (sqrtu > 0.0) a_u += a_sqrtu * 0.5 / sqrtu;
        const double a_rr = 0.0 - a_u;
        a_rho += a_rr * rho;
        a_rho += a_rr * rho;
        adj[0] = a_kappa;
        adj[1] = a_theta;
        adj[2] = a_xi;
        adj[3] = a_rho;
        adj[4] = aV; /* V_0 is the v0 input node */
        free(aS);
    }
    free(S);
    free(V);
    free(E);
    free(cell);
    return 0;
}

/* ---- config-4 basket (program of oracle/ref_driver.cpp record_basket) -- */

size_t lto_basket_num_params(const ltg_basket_model* m) { return m->n_assets; }

int lto_basket_path(const ltg_basket_model* m, const double* x, const double* z,
                    const double* lambda, double* y, double* adj) {
    const size_t n = m->n_assets, steps = m->steps;
    const double dt = m->dt, sqdt = sqrt(dt);
    double drift[16], vol[16];
    if (n > 16) return 1;
    for (size_t a = 0; a < n; ++a) {
        drift[a] = (m->r - 0.5 * (x[a] * x[a])) * dt;
        vol[a] = x[a] * sqdt;
    }
    double* S = (double*)malloc(sizeof(double) * (steps + 1) * n);
    double* E = (double*)malloc(sizeof(double) * steps * n);
    double* W = (double*)malloc(sizeof(double) * steps * n);
    for (size_t a = 0; a < n; ++a) S[a] = m->s0[a];
    for (size_t k = 0; k < steps; ++k) {
        const double* zk = z + k * n;
        for (size_t a = 0; a < n; ++a) {
            double w = m->chol[a * n + 0] * zk[0];
            for (size_t b = 1; b <= a; ++b) w = w + m->chol[a * n + b] * zk[b];
            W[k * n + a] = w;
            E[k * n + a] = exp(drift[a] + vol[a] * w);
            S[(k + 1) * n + a] = S[k * n + a] * E[k * n + a];
        }
    }
    for (uint32_t i = 0; i < m->n_instruments; ++i) {
        const double s = S[(size_t)m->inst_maturity_step[i] * n + m->inst_asset[i]];
        const double K = m->inst_strike[i];
        const double d = m->inst_kind[i] == LTG_PUT ? K - s : s - K;
        y[i] = d > 0.0 ? d : 0.0;
    }
    if (adj) {
        double* aS = (double*)calloc((steps + 1) * n, sizeof(double));
        double a_drift[16] = {0}, a_vol[16] = {0};
        for (size_t ii = m->n_instruments; ii-- > 0;) {
            const size_t idx = (size_t)m->inst_maturity_step[ii] * n + m->inst_asset[ii];
            const double s = S[idx], K = m->inst_strike[ii];
            const double d = m->inst_kind[ii] == LTG_PUT ? K - s : s - K;
            const double a_sub = 0.0 + (d > 0.0 ? lambda[ii] : 0.0);
            if (m->inst_kind[ii] == LTG_PUT)
                aS[idx] -= a_sub;
            else
                aS[idx] += a_sub;
        }
        for (size_t k = steps; k-- > 0;) {
            for (size_t a = n; a-- > 0;) {
                const double a_S1 = aS[(k + 1) * n + a];
                const double e = E[k * n + a];
                aS[k * n + a] += a_S1 * e;
                const double a_e = 0.0 + a_S1 * S[k * n + a];
                const double a_t2 = 0.0 + a_e * e;
                a_drift[a] += a_t2;
                a_vol[a] += a_t2 * W[k * n + a];
            }
        }
        for (size_t a = n; a-- > 0;) {
            double as = 0.0;
            as += a_vol[a] * sqdt;               /* vol = mul(sigma, c_sqdt) */
            const double a_rd = 0.0 + a_drift[a] * dt; /* drift = mul(rd, c_dt) */
            const double a_hs = 0.0 - a_rd;      /* rd = sub(c_r, hs) */
            const double a_ss = 0.0 + a_hs * 0.5; /* hs = mul(c_half, ss) */
            as += a_ss * x[a];                   /* ss = mul(sigma, sigma) */
            as += a_ss * x[a];
            adj[a] = as;
        }
        free(aS);
    }
    free(S);
    free(E);
    free(W);
    return 0;
}

/* ---- expectation.hpp ---------------------------------------------------- */

typedef int (*path_fn)(const void* model, const double* x, const double* z, const double* lambda,
                       double* y, double* adj);

static int heston_fn(const void* m, const double* x, const double* z, const double* l, double* y,
                     double* a) {
    return lto_heston_path((const ltg_heston_model*)m, x, z, l, y, a);
}
static int basket_fn(const void* m, const double* x, const double* z, const double* l, double* y,
                     double* a) {
    return lto_basket_path((const ltg_basket_model*)m, x, z, l, y, a);
}

typedef struct {
    path_fn fn;
    const void* model;
    size_t M, N, m;
} program;

static program make_program(int kind, const void* model) {
    program p;
    if (kind == 0) {
        const ltg_heston_model* h = (const ltg_heston_model*)model;
        p.fn = heston_fn;
        p.M = lto_heston_num_params(h);
        p.N = 2 * (size_t)h->steps;
        p.m = h->n_instruments;
    } else {
        const ltg_basket_model* b = (const ltg_basket_model*)model;
        p.fn = basket_fn;
        p.M = b->n_assets;
        p.N = (size_t)b->steps * b->n_assets;
        p.m = b->n_instruments;
    }
    p.model = model;
    return p;
}

/* detail::forward_pass (lambda == NULL) or detail::reverse_pass, one worker,
 * lane width c: per batch of c paths the lanes are summed in ascending order
 * and the batch partials in ascending batch order (BatchSums, :109-122). Past-
 * the-end lanes are evaluated but excluded (fill_random_lanes, :132-144).
 * kind: 0 = Heston SLV, 1 = basket. */
int lto_pass_sums(int kind, const void* model, const double* x, uint64_t seed, int antithetic,
                  int lane_width, uint64_t path_offset, uint64_t paths, const double* lambda,
                  double* sum, double* sumsq, double* adjsum) {
    const program p = make_program(kind, model);
    const size_t c = (size_t)lane_width;
    if (paths == 0 || !(c == 1 || c == 4 || c == 8)) return 1;
    double* z = (double*)malloc(sizeof(double) * p.N);
    double* y = (double*)malloc(sizeof(double) * p.m * c);
    double* a = (double*)malloc(sizeof(double) * p.M * c);
    const size_t width = lambda ? p.M : p.m;
    for (size_t k = 0; k < width; ++k) {
        if (lambda) adjsum[k] = 0.0; else { sum[k] = 0.0; sumsq[k] = 0.0; }
    }
    int rc = 0;
    const uint64_t batches = (paths + c - 1) / c;
    for (uint64_t b = 0; b < batches && rc == 0; ++b) {
        const uint64_t base = b * c;
        const uint64_t used = paths - base < c ? paths - base : c;
        for (size_t l = 0; l < used; ++l) {
            lto_fill_normals(seed, p.N, antithetic, path_offset + base + l, z);
            rc = p.fn(p.model, x, z, lambda, y + l * p.m, lambda ? a + l * p.M : NULL);
            if (rc) break;
        }
        if (!lambda) {
            for (size_t o = 0; o < p.m; ++o) {
                double s = 0.0, s2 = 0.0;
                for (size_t l = 0; l < used; ++l) {
                    const double v = y[l * p.m + o];
                    s += v;
                    s2 += v * v;
                }
                sum[o] += s;
                sumsq[o] += s2;
            }
        } else {
            for (size_t j = 0; j < p.M; ++j) {
                double s = 0.0;
                for (size_t l = 0; l < used; ++l) s += a[l * p.M + j];
                adjsum[j] += s;
            }
        }
    }
    free(z);
    free(y);
    free(a);
    return rc;
}

/* gradient_of_G, expectation.hpp:300-344 (recompute mode; store mode is
 * bitwise identical by construction, kernel.hpp:101-103) with means_from_sums
 * (:251-269). se may be NULL. */
int lto_gradient_of_G(int kind, const void* model, const double* x, const double* C,
                      uint64_t paths, uint64_t seed, int antithetic, int fresh_step2_paths,
                      int lane_width, double* G, double* means, double* lambda, double* grad,
                      double* se) {
    const program p = make_program(kind, model);
    double* sum = (double*)malloc(sizeof(double) * p.m);
    double* sumsq = (double*)malloc(sizeof(double) * p.m);
    double* tot = (double*)malloc(sizeof(double) * p.M);
    int rc = lto_pass_sums(kind, model, x, seed, antithetic, lane_width, 0, paths, NULL, sum,
                           sumsq, NULL);
    if (rc == 0) {
        const double P = (double)paths;
        *G = 0.0;
        for (size_t o = 0; o < p.m; ++o) {
            const double mean = sum[o] / P;
            means[o] = mean;
            if (se) {
                if (paths > 1) {
                    double var = (sumsq[o] - P * mean * mean) / (P - 1.0);
                    if (var < 0.0) var = 0.0;
                    se[o] = sqrt(var / P);
                } else {
                    se[o] = 0.0;
                }
            }
        }
        if (C) {
            for (size_t o = 0; o < p.m; ++o) {
                lambda[o] = means[o] - C[o];
                *G += 0.5 * lambda[o] * lambda[o];
            }
            rc = lto_pass_sums(kind, model, x, seed, antithetic, lane_width,
                               fresh_step2_paths ? paths : 0, paths, lambda, NULL, NULL, tot);
            for (size_t j = 0; j < p.M && rc == 0; ++j) grad[j] = tot[j] / P;
        }
    }
    free(sum);
    free(sumsq);
    free(tot);
    return rc;
}
