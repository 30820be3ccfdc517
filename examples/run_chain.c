/* A C host program using the loomfuse-b200 C ABI the way the reference's
 * users call the emitted function: plan a rule file, size the terminal buffers
 * from lf_plan_terminal, fill the axioms, run on host buffers, write the goals.
 *
 *   cc -O2 -I include examples/run_chain.c -L paper_1710_08774_b200 \
 *      -lloomfuse_b200 -Wl,-rpath,$PWD/paper_1710_08774_b200 -o run_chain
 *   ./run_chain spec.lf STEPS [in0.bin ... out0.bin ...]   (STEPS = 0: plan only)
 *
 * Axioms are read from / goals written to raw binary files in terminal
 * order when given (sizes from lf_plan_terminal); otherwise axioms are zero. */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "loomfuse_b200.h"

static char* slurp(const char* path, size_t* n) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  long len = ftell(f);
  fseek(f, 0, SEEK_SET);
  char* buf = (char*)malloc((size_t)len + 1);
  if (fread(buf, 1, (size_t)len, f) != (size_t)len) {
    fclose(f);
    free(buf);
    return NULL;
  }
  fclose(f);
  buf[len] = 0;
  *n = (size_t)len;
  return buf;
}

int main(int argc, char** argv) {
  if (argc < 3) {
    fprintf(stderr, "usage: %s spec.lf STEPS [terminal files...]\n", argv[0]);
    return 2;
  }
  size_t len = 0;
  char* spec = slurp(argv[1], &len);
  if (!spec) {
    fprintf(stderr, "cannot read %s\n", argv[1]);
    return 2;
  }
  lf_plan* plan = NULL;
  if (lf_plan_create(spec, len, argv[1], &plan) != LF_OK) {
    fprintf(stderr, "%s\n", lf_last_error());
    return 1;
  }
  const int nt = lf_plan_num_terminals(plan);
  printf("executor %s\n", lf_plan_executor(plan));
  void** bufs = (void**)calloc((size_t)nt, sizeof(void*));
  for (int i = 0; i < nt; ++i) {
    lf_terminal t;
    lf_plan_terminal(plan, i, &t);
    printf("%s %s %s bytes %lld extent", t.is_goal ? "goal" : "axiom", t.type, t.name, (long long)t.bytes);
    for (int d = 0; d < t.ndim; ++d) printf(" %lld", (long long)t.extent[d]);
    printf("\n");
    /* a goal given the SAME file as an axiom shares that axiom's buffer: an
     * in-place run (the spec must declare the pair in config.aliases) */
    for (int k = 0; t.is_goal && k < i && !bufs[i]; ++k)
      if (argc > 3 + i && argc > 3 + k && strcmp(argv[3 + i], argv[3 + k]) == 0) {
        bufs[i] = bufs[k];
        printf("goal %s in place on terminal %d\n", t.name, k);
      }
    if (!bufs[i]) bufs[i] = calloc(1, (size_t)(t.bytes > 0 ? t.bytes : 8));
    if (!t.is_goal && argc > 3 + i) {
      size_t n = 0;
      char* data = slurp(argv[3 + i], &n);
      if (!data || n != (size_t)t.bytes) {
        fprintf(stderr, "%s: expected %lld bytes\n", argv[3 + i], (long long)t.bytes);
        return 2;
      }
      memcpy(bufs[i], data, n);
      free(data);
    }
  }
  const int steps = atoi(argv[2]);
  if (steps > 0) {
    if (lf_run_host(plan, bufs, nt, steps) != LF_OK) {
      fprintf(stderr, "%s\n", lf_last_error());
      return 1;
    }
    for (int i = 0; i < nt; ++i) {
      lf_terminal t;
      lf_plan_terminal(plan, i, &t);
      if (!t.is_goal || argc <= 3 + i) continue;
      FILE* f = fopen(argv[3 + i], "wb");
      fwrite(bufs[i], 1, (size_t)t.bytes, f);
      fclose(f);
    }
    printf("ran %d steps\n", steps);
  }
  for (int i = 0; i < nt; ++i) {
    int shared = 0;
    for (int k = 0; k < i; ++k) shared |= bufs[k] == bufs[i];
    if (!shared) free(bufs[i]);
  }
  free(bufs);
  lf_plan_destroy(plan);
  free(spec);
  return 0;
}
