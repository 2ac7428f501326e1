/* TEST INFRASTRUCTURE — CPU restatement (checker only; see pcot_oracle.h).
 *
 * Every routine restates the semantics the reference interpreter gives the
 * corresponding kernel spec: Executor::exec_stmt evaluates the body's parse
 * tree in IEEE double, one rounding per operation, no contraction
 * (reference core/src/exec.cpp:347-428; expression trees are left-associative
 * per expr.cpp:163-195).  Compiled with -ffp-contract=off.
 */
#include "pcot_oracle.h"

#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int g_threads = 0;

void oracle_set_threads(int n) { g_threads = n; }

int oracle_get_threads(void) {
#ifdef _OPENMP
  return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
  return 1;
#endif
}

/* reference exec.cpp:12-19 */
uint64_t oracle_fnv1a(const void* data, size_t n, uint64_t h) {
  const unsigned char* p = (const unsigned char*)data;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

static uint64_t splitmix_from(uint64_t name_hash, uint64_t flat) {
  uint64_t x = name_hash ^ (flat * 0x9E3779B97F4A7C15ULL);
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return x;
}

/* reference exec.cpp:21-28 */
double oracle_init_value(const char* name, uint64_t flat) {
  uint64_t h = oracle_fnv1a(name, strlen(name), 0xcbf29ce484222325ULL);
  return (double)(splitmix_from(h, flat) >> 11) * 0x1.0p-53;
}

/* init_value over a window [r0, r0+h) x [c0, c0+w) of a row-major grid with
 * `ncols` columns (flat = r*ncols + c), written densely to out[h*w]. */
void oracle_init_window(const char* name, uint64_t ncols, uint64_t r0, uint64_t c0, uint64_t h,
                        uint64_t w, double* out) {
  uint64_t hs = oracle_fnv1a(name, strlen(name), 0xcbf29ce484222325ULL);
  int nt = oracle_get_threads();
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t r = 0; r < (int64_t)h; ++r)
    for (uint64_t c = 0; c < w; ++c)
      out[(uint64_t)r * w + c] =
          (double)(splitmix_from(hs, (r0 + (uint64_t)r) * ncols + c0 + c) >> 11) * 0x1.0p-53;
}

void oracle_init_array(const char* name, double* out, uint64_t n) {
  uint64_t h = oracle_fnv1a(name, strlen(name), 0xcbf29ce484222325ULL);
  int nt = oracle_get_threads();
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t f = 0; f < (int64_t)n; ++f)
    out[f] = (double)(splitmix_from(h, (uint64_t)f) >> 11) * 0x1.0p-53;
}

/* 2-D 5-point ping-pong sweep.
 * jacobi2d.kernel S1 / reference heat2d.kernel:32:
 *   0.2 * ((((c + (i-1,j)) + (i+1,j)) + (i,j-1)) + (i,j+1))
 * Ring: literal 0.0 at every t (jacobi2d R0-R3), or copied forward from the
 * previous step (heat2d S2-S5, so it stays F). */
void oracle_stencil2d5(int64_t N, int64_t T, int ring_hold, const double* F, double* Out) {
  size_t n = (size_t)N * (size_t)N;
  double* a = (double*)malloc(n * sizeof(double));
  double* b = (double*)malloc(n * sizeof(double));
  int nt = oracle_get_threads();
  for (int64_t i = 0; i < N; ++i)
    for (int64_t j = 0; j < N; ++j) {
      int ring = i == 0 || j == 0 || i == N - 1 || j == N - 1;
      a[i * N + j] = ring ? (ring_hold ? F[i * N + j] : 0.0) : F[i * N + j];
    }
  memcpy(b, a, n * sizeof(double)); /* ring cells are invariant across steps */
  for (int64_t t = 1; t <= T; ++t) {
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int64_t i = 1; i < N - 1; ++i) {
      const double* r0 = a + (i - 1) * N;
      const double* r1 = a + i * N;
      const double* r2 = a + (i + 1) * N;
      double* o = b + i * N;
      for (int64_t j = 1; j < N - 1; ++j) {
        double s = r1[j] + r0[j];
        s = s + r2[j];
        s = s + r1[j - 1];
        s = s + r1[j + 1];
        o[j] = 0.2 * s;
      }
    }
    double* tmp = a;
    a = b;
    b = tmp;
  }
  memcpy(Out, a, n * sizeof(double));
  free(a);
  free(b);
}

/* 3-D 7-point ping-pong sweep; neighbour order (i-1),(i+1),(j-1),(j+1),(k-1),(k+1).
 * rule 0 (heat3d_b.kernel S1):  c + 0.125 * ((((((n1+n2)+n3)+n4)+n5)+n6) - 6.0*c)
 * rule 1 (reference heat3d.kernel:34): 0.1 * ((((((c+n1)+n2)+n3)+n4)+n5)+n6) */
void oracle_stencil3d7(int64_t N, int64_t T, int rule, int ring_hold, const double* F,
                       double* Out) {
  size_t n = (size_t)N * (size_t)N * (size_t)N;
  double* a = (double*)malloc(n * sizeof(double));
  double* b = (double*)malloc(n * sizeof(double));
  int nt = oracle_get_threads();
  const int64_t P = N * N;
  for (int64_t i = 0; i < N; ++i)
    for (int64_t j = 0; j < N; ++j)
      for (int64_t k = 0; k < N; ++k) {
        int ring = i == 0 || j == 0 || k == 0 || i == N - 1 || j == N - 1 || k == N - 1;
        int64_t f = i * P + j * N + k;
        a[f] = ring ? (ring_hold ? F[f] : 0.0) : F[f];
      }
  memcpy(b, a, n * sizeof(double));
  for (int64_t t = 1; t <= T; ++t) {
#pragma omp parallel for num_threads(nt) schedule(static)
    for (int64_t i = 1; i < N - 1; ++i)
      for (int64_t j = 1; j < N - 1; ++j) {
        const double* c = a + i * P + j * N;
        double* o = b + i * P + j * N;
        for (int64_t k = 1; k < N - 1; ++k) {
          double cc = c[k];
          double n1 = c[k - P], n2 = c[k + P], n3 = c[k - N], n4 = c[k + N];
          double n5 = c[k - 1], n6 = c[k + 1];
          double v;
          if (rule == 0) {
            double s = n1 + n2;
            s = s + n3;
            s = s + n4;
            s = s + n5;
            s = s + n6;
            double m = 6.0 * cc;
            s = s - m;
            double q = 0.125 * s;
            v = cc + q;
          } else {
            double s = cc + n1;
            s = s + n2;
            s = s + n3;
            s = s + n4;
            s = s + n5;
            s = s + n6;
            v = 0.1 * s;
          }
          o[k] = v;
        }
      }
    double* tmp = a;
    a = b;
    b = tmp;
  }
  memcpy(Out, a, n * sizeof(double));
  free(a);
  free(b);
}

/* In-place Gauss-Seidel (gs2d.kernel S1): lexicographic sweep, so the four
 * predecessors (i-1,*) and (i,j-1) already hold step-t values; 3x3 summed in
 * row-major order, then IEEE division by 9.0. Ring fixed at 0.0. */
void oracle_gs2d9(int64_t N, int64_t T, const double* F, double* Out) {
  size_t n = (size_t)N * (size_t)N;
  double* a = Out;
  for (int64_t i = 0; i < N; ++i)
    for (int64_t j = 0; j < N; ++j) {
      int ring = i == 0 || j == 0 || i == N - 1 || j == N - 1;
      a[i * N + j] = ring ? 0.0 : F[i * N + j];
    }
  (void)n;
  for (int64_t t = 1; t <= T; ++t)
    for (int64_t i = 1; i < N - 1; ++i) {
      double* r0 = a + (i - 1) * N;
      double* r1 = a + i * N;
      double* r2 = a + (i + 1) * N;
      for (int64_t j = 1; j < N - 1; ++j) {
        double s = r0[j - 1] + r0[j];
        s = s + r0[j + 1];
        s = s + r1[j - 1];
        s = s + r1[j];
        s = s + r1[j + 1];
        s = s + r2[j - 1];
        s = s + r2[j];
        s = s + r2[j + 1];
        r1[j] = s / 9.0;
      }
    }
}

/* gemm.kernel S1: C[k] = C[k-1] + ((2.0*A[i,k-1] - 1.0) * (2.0*B[k-1,j] - 1.0)),
 * k ascending, every operation rounded (no FMA).  Loop order i,k,j keeps each
 * (i,j) accumulation in k order; rows are independent so threads do not
 * change any bit. */
void oracle_gemm_rows(int64_t N, int64_t r0, int64_t r1, const double* A, const double* B,
                      double* Out) {
  int nt = oracle_get_threads();
#pragma omp parallel num_threads(nt)
  {
    double* brow = (double*)malloc((size_t)N * sizeof(double));
#pragma omp for schedule(dynamic, 1)
    for (int64_t i = r0; i < r1; ++i) {
      double* acc = Out + i * N;
      for (int64_t j = 0; j < N; ++j) acc[j] = 0.0;
      for (int64_t k = 0; k < N; ++k) {
        double av = 2.0 * A[i * N + k];
        av = av - 1.0;
        const double* b = B + k * N;
        for (int64_t j = 0; j < N; ++j) {
          double bv = 2.0 * b[j];
          bv = bv - 1.0;
          double p = av * bv;
          acc[j] = acc[j] + p;
        }
      }
    }
    free(brow);
  }
}

void oracle_gemm(int64_t N, const double* A, const double* B, double* Out) {
  oracle_gemm_rows(N, 0, N, A, B, Out);
}
