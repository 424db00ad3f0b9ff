/*
 * oracle/logistic_ref.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the reference trainer's numeric core,
 *   covault.workload.run_training   /root/reference/pkg/src/covault/workload.py:48-71
 *   covault.workload._sigmoid       /root/reference/pkg/src/covault/workload.py:44-45
 * Python floats are IEEE binary64 with one rounding per operation and no FMA, so this
 * file is compiled with -O2 -ffp-contract=off (see oracle/Makefile) and performs the
 * operations in exactly the reference order:
 *   z = bias; z += w_i * x_i (i = 0..F-1)                      workload.py:61-63
 *   delta = 0.5 * (1.0 + z / (1.0 + |z|)) - y                 workload.py:44-45, :64
 *   g_i += delta * x_i ; g_b += delta   (rows in file order)  workload.py:65-67
 *   w_i -= (lr * g_i) / n ; b -= (lr * g_b) / n               workload.py:68-70
 * Pinned by DEMO_MODEL_SHA256 (pkg/tests/test_workload.py:23) in tests/test_oracle.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <math.h>

void ref_logistic_train(const double* X, const double* y, int64_t n_rows, int64_t n_feat,
                        double lr, int64_t epochs, double* w_out, double* b_out) {
    double* w = (double*)calloc((size_t)n_feat, sizeof(double));
    double* g = (double*)calloc((size_t)n_feat, sizeof(double));
    double b = 0.0;
    double n = (double)n_rows;
    for (int64_t e = 0; e < epochs; e++) {
        for (int64_t i = 0; i < n_feat; i++) g[i] = 0.0;
        double gb = 0.0;
        for (int64_t r = 0; r < n_rows; r++) {
            const double* x = X + r * n_feat;
            double z = b;
            for (int64_t i = 0; i < n_feat; i++) { double p = w[i] * x[i]; z = z + p; }
            double t = 1.0 + fabs(z);
            double q = z / t;
            double s = 1.0 + q;
            double delta = 0.5 * s - y[r];
            for (int64_t i = 0; i < n_feat; i++) { double p = delta * x[i]; g[i] = g[i] + p; }
            gb = gb + delta;
        }
        for (int64_t i = 0; i < n_feat; i++) { double u = lr * g[i]; w[i] = w[i] - u / n; }
        { double u = lr * gb; b = b - u / n; }
    }
    for (int64_t i = 0; i < n_feat; i++) w_out[i] = w[i];
    *b_out = b;
    free(w);
    free(g);
}
