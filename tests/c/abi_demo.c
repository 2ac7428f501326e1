/* A plain-C consumer of the drop-in boundary (include/pcotgpu.h): what a
 * binding layer in the reference's toolchain would call.  Loads a kernel spec
 * file, creates an executor, runs one schedule, prints the ExecResult and the
 * first output cells.  Built and run by tests/test_boundary.py (link check on
 * CPU) and tests/test_c_abi.py (GPU run against the reference golden).
 *
 *   abi_demo <kernel file> <param values...> <scheme 0|1|2> <leaf0> */
#include <stdio.h>
#include <stdlib.h>

#include "pcotgpu.h"

static char* slurp(const char* path) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  char* s = (char*)malloc((size_t)n + 1);
  if (fread(s, 1, (size_t)n, f) != (size_t)n) n = 0;
  s[n] = 0;
  fclose(f);
  return s;
}

int main(int argc, char** argv) {
  if (argc < 5) {
    fprintf(stderr, "usage: abi_demo <kernel> <params...> <scheme> <leaf0>\n");
    return 2;
  }
  if (pcotgpu_abi_version() < 1) return 3;
  char* json = slurp(argv[1]);
  if (!json) return 4;
  const int np = argc - 4;
  int64_t params[8];
  for (int i = 0; i < np && i < 8; ++i) params[i] = atoll(argv[2 + i]);
  pcotgpu_kernel_info info;
  int st = pcotgpu_recognize(json, params, (size_t)np, &info);
  printf("recognize %d family %d\n", st, st == 0 ? info.family : -1);
  pcotgpu_handle* h = NULL;
  st = pcotgpu_create(json, params, (size_t)np, 0, &h);
  if (st != 0) {
    printf("create %d %s\n", st, pcotgpu_last_error());
    return 5;
  }
  pcotgpu_schedule s = {0};
  s.scheme = atoi(argv[argc - 2]);
  s.ndim = 1;
  s.leaf[0] = atoll(argv[argc - 1]);
  pcotgpu_result r;
  st = pcotgpu_run(h, &s, &r);
  if (st != 0) {
    printf("run %d %s\n", st, pcotgpu_last_error());
    return 6;
  }
  printf("points %llu\nreads %llu\nwrites %llu\nbt %d\nCHECKSUM %016llx\n",
         (unsigned long long)r.points, (unsigned long long)r.reads, (unsigned long long)r.writes,
         r.bt, (unsigned long long)r.checksum);
  uint64_t words = 0;
  pcotgpu_array_words(h, "Out", &words);
  double* out = (double*)malloc(words * sizeof(double));
  st = pcotgpu_read_array(h, "Out", out, words);
  printf("out0 %.17g\n", st == 0 && words ? out[0] : -1.0);
  free(out);
  pcotgpu_destroy(h);
  free(json);
  return 0;
}
