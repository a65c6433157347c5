/* Calling libb200mat.so from C, no Python: the binding a non-Python FFI (cgo,
 * JNI, N-API) would make.  Builds accu(2*A + B%C - exp(D)) as one fused
 * reduction program (include/b200mat.h bm_invocation) and C = A * B^T with
 * bm_gemm, and checks both against plain host loops.
 *
 *   gcc -O2 -std=c11 -I include examples/c_abi_example.c \
 *       -L paper_2308_03120_b200 -lb200mat -Wl,-rpath,$PWD/paper_2308_03120_b200 -lm -o build/c_abi_example
 *   ./build/c_abi_example            -> prints "c_abi_example: ok ..." and exits 0
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "b200mat.h"

#define CHECK(call)                                                                  \
    do {                                                                             \
        int rc_ = (call);                                                            \
        if (rc_ != BM_OK) {                                                          \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, bm_last_error());    \
            return 1;                                                                \
        }                                                                            \
    } while (0)

static uint64_t s_state = 12345;
static float urand(void) { /* xorshift, [0, 1) */
    s_state ^= s_state << 13; s_state ^= s_state >> 7; s_state ^= s_state << 17;
    return (float)((s_state >> 40) * (1.0 / 16777216.0));
}

static bm_view flat(void* p, int64_t n) {
    bm_view v;
    memset(&v, 0, sizeof v);
    v.base = p; v.count = n; v.stride = 1; v.rows = n; v.cols = 1; v.lda = n; v.dtype = BM_F32;
    return v;
}

int main(void) {
    if (bm_abi_version() != BM_ABI_VERSION) { fprintf(stderr, "ABI mismatch\n"); return 1; }
    CHECK(bm_init(0));
    /* ---- fused eOp + accu: 1 kernel, nothing materialised ---- */
    const int64_t n = 1 << 20;
    float* h[4];
    void* d[4];
    for (int i = 0; i < 4; ++i) {
        h[i] = (float*)malloc(n * sizeof(float));
        for (int64_t j = 0; j < n; ++j) h[i][j] = urand();
        CHECK(bm_alloc(n * (int64_t)sizeof(float), &d[i]));
        CHECK(bm_h2d(d[i], h[i], n * (int64_t)sizeof(float)));
    }
    bm_invocation inv;
    memset(&inv, 0, sizeof inv);
    inv.kind = BM_K_REDUCE;
    inv.reduce_op = BM_R_ACCU;
    inv.compute_dtype = BM_F32;
    inv.n_inputs = 4;
    for (int i = 0; i < 4; ++i) inv.inputs[i] = flat(d[i], n);
    inv.n_scalars = 1;
    inv.fscalars[0] = 2.0;
    /* post-order program: load0, *2, load1, load2, schur, plus, load3, exp, minus */
    const int32_t prog[][3] = {{BM_P_LOAD, 0, 0},  {BM_P_SCALAR, BM_S_TIMES, 0}, {BM_P_LOAD, 0, 1},
                               {BM_P_LOAD, 0, 2},  {BM_P_GLUE, BM_G_SCHUR, 0},  {BM_P_GLUE, BM_G_PLUS, 0},
                               {BM_P_LOAD, 0, 3},  {BM_P_UNARY, BM_U_EXP, -1},  {BM_P_GLUE, BM_G_MINUS, 0}};
    inv.n_prog = 9;
    memcpy(inv.prog, prog, sizeof prog);
    float got = 0.0f;
    CHECK(bm_execute_reduce(&inv, &got));
    double want = 0.0;
    for (int64_t j = 0; j < n; ++j) want += 2.0 * h[0][j] + (double)h[1][j] * h[2][j] - exp((double)h[3][j]);
    const double rel_accu = fabs(got - want) / fabs(want);

    /* ---- C = A * B^T (3xTF32 on tcgen05) ---- */
    const int64_t m = 512, nn = 384, k = 256;
    float* ha = (float*)malloc(m * k * sizeof(float));
    float* hb = (float*)malloc(nn * k * sizeof(float));
    float* hc = (float*)malloc(m * nn * sizeof(float));
    for (int64_t j = 0; j < m * k; ++j) ha[j] = urand() - 0.5f;
    for (int64_t j = 0; j < nn * k; ++j) hb[j] = urand() - 0.5f;
    void *da, *db, *dc;
    CHECK(bm_alloc(m * k * 4, &da));
    CHECK(bm_alloc(nn * k * 4, &db));
    CHECK(bm_alloc(m * nn * 4, &dc));
    CHECK(bm_h2d(da, ha, m * k * 4));
    CHECK(bm_h2d(db, hb, nn * k * 4));
    CHECK(bm_gemm(BM_F32, 0, 1, m, nn, k, da, m, db, nn, dc, m));   /* column-major, B is nn x k */
    CHECK(bm_sync());
    CHECK(bm_d2h(hc, dc, m * nn * 4));
    double err = 0.0, mx = 0.0;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < nn; ++j) {
            double s = 0.0;
            for (int64_t l = 0; l < k; ++l) s += (double)ha[i + l * m] * hb[j + l * nn];
            const double e = fabs(hc[i + j * m] - s);
            if (e > err) err = e;
            if (fabs(s) > mx) mx = fabs(s);
        }
    const double rel_gemm = err / (mx > 1.0 ? mx : 1.0);
    bm_counters c;
    CHECK(bm_get_counters(&c));
    for (int i = 0; i < 4; ++i) { bm_free(d[i]); free(h[i]); }
    bm_free(da); bm_free(db); bm_free(dc);
    free(ha); free(hb); free(hc);
    CHECK(bm_shutdown());
    const int ok = rel_accu <= 1e-5 && rel_gemm <= 1e-5;
    printf("c_abi_example: %s accu=%.9g (host f64 %.9g, rel %.2e) gemm rel %.2e launches=%lld\n", ok ? "ok" : "FAILED",
           got, want, rel_accu, rel_gemm, (long long)c.launches);
    return ok ? 0 : 1;
}
