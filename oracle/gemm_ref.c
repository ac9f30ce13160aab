/*
 * oracle/gemm_ref.c -- TEST INFRASTRUCTURE ONLY (parity oracle; never on the product path).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  It shares no code, header or constant with the CUDA path
 * (paper_2409_01075_b200/csrc, include/vx.h).
 *
 * What it computes: the plain definition of the operation the method accelerates,
 *     C = A x B,  A is M x K, B is K x N, C is M x N
 * (Sec. 4.1 "GEMM ... is mathematically defined as C = A x B";
 *  PAPER.md:866-867, Sec. 2.2: M = batch x sequence rows of A, N columns of B,
 *  K columns of A / rows of B).
 * Batched GEMM (BASELINE.json config 4) is the same definition applied per batch index b.
 *
 *     C_ref[b,i,j] = sum_{k=0}^{K-1} double(A[b,i,k]) * double(B[b,k,j])
 *
 * evaluated in IEEE binary64, one product and one add at a time, k ascending, from the
 * exact same stored input values the GPU reads (bf16 / fp16 / fp32 bit patterns are
 * widened to double exactly).  No blocking, no reordering, no BLAS.  OpenMP only
 * distributes independent output rows over threads; each element's summation order is
 * fixed, so the result is identical for any thread count.
 *
 * Build (see oracle/__init__.py):  gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC
 * -ffp-contract=off: no fused multiply-add contraction, so every product is rounded to
 * binary64 before the add, exactly as the definition above is written.
 */
#include <stdint.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* element encodings of the stored inputs */
#define ORC_BF16 0
#define ORC_FP16 1
#define ORC_FP32 2
#define ORC_FP64 3

/* layout of the stored B operand */
#define ORC_B_KN 0 /* B stored row-major K x N (the paper's B) */
#define ORC_B_NK 1 /* B stored row-major N x K (its transpose, e.g. an nn.Linear weight) */

/* bfloat16: the top 16 bits of an IEEE binary32 -> exact widening */
static double orc_bf16_to_double(uint16_t h) {
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* IEEE binary16 -> double, written out from the format definition (1 sign bit,
 * 5 exponent bits with bias 15, 10 fraction bits; subnormals, inf, nan). */
static double orc_fp16_to_double(uint16_t h) {
    int sign = (h >> 15) & 1;
    int exp = (h >> 10) & 0x1f;
    int frac = h & 0x3ff;
    double v;
    if (exp == 0) {
        v = ldexp((double)frac, -24); /* subnormal: frac * 2^-14 * 2^-10 */
    } else if (exp == 31) {
        v = frac ? NAN : INFINITY;
    } else {
        v = ldexp((double)(frac + 1024), exp - 25); /* (1 + frac/1024) * 2^(exp-15) */
    }
    return sign ? -v : v;
}

static double orc_load(const void* base, int64_t idx, int dtype) {
    switch (dtype) {
    case ORC_BF16: return orc_bf16_to_double(((const uint16_t*)base)[idx]);
    case ORC_FP16: return orc_fp16_to_double(((const uint16_t*)base)[idx]);
    case ORC_FP32: return (double)((const float*)base)[idx];
    default:       return ((const double*)base)[idx];
    }
}

/*
 * oracle_gemm: C[b, r, j] for b < batch, r < nrows (output row r is input row rows[r],
 * or row r itself when rows == NULL), j < N.
 *   A: batch x M x K, element (b,i,k) at A[b*sA + i*K + k]
 *   B: KN: element (b,k,j) at B[b*sB + k*N + j];  NK: at B[b*sB + j*K + k]
 *   C: double, element (b,r,j) at C[(b*nrows + r)*N + j]
 * Returns 0, or -1 on an invalid argument.
 */
int oracle_gemm(int64_t batch, int64_t M, int64_t N, int64_t K, int dtype, int b_layout,
                const void* A, int64_t sA, const void* B, int64_t sB,
                double* C, const int64_t* rows, int64_t nrows, int threads) {
    if (batch < 0 || M < 0 || N < 0 || K < 0 || dtype < 0 || dtype > 3) return -1;
    if (b_layout != ORC_B_KN && b_layout != ORC_B_NK) return -1;
    if (rows == NULL) nrows = M;
    for (int64_t r = 0; rows && r < nrows; ++r)
        if (rows[r] < 0 || rows[r] >= M) return -1;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
    int64_t total = batch * nrows;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t br = 0; br < total; ++br) {
        int64_t b = br / nrows, r = br % nrows;
        int64_t i = rows ? rows[r] : r;
        double* c = C + br * N;
        for (int64_t j = 0; j < N; ++j) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k) {
                double a = orc_load(A, b * sA + i * K + k, dtype);
                double bb = (b_layout == ORC_B_KN) ? orc_load(B, b * sB + k * N + j, dtype)
                                                   : orc_load(B, b * sB + j * K + k, dtype);
                double p = a * bb;
                acc = acc + p;
            }
            c[j] = acc;
        }
    }
    return 0;
}

/* number of OpenMP threads a parallel region would use (for the cpu_baseline "cores") */
int oracle_threads(int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
    int n = 1;
#pragma omp parallel
    {
#pragma omp single
        n = omp_get_num_threads();
    }
    return n;
#else
    (void)threads;
    return 1;
#endif
}
