/* A plain-C host running the statistics-and-placement pass through the C ABI only
 * (include/gimbal_gpu.h): the way a non-Python, non-C++ host (cgo, JNI, a C engine) would bind it.
 * Reads host ids [T][L][k] (uint8) and candidates [C][m] (uint8) from files, counts them
 * (gimbal_stats_add_tokens from host memory, RoutingStats::add_token), builds the strong-pair set
 * (build_affinity_set), the greedy placement (greedy_place) and scores every candidate
 * (eval_cost), then writes A, E, |M|, M, greedy, D, cut, objective and the argmin to a file.
 *
 *   c_host_pass L n_e k g T C ids.bin cands.bin out.bin
 *
 * Built by paper_2602_21626_b200/shim/Makefile (gcc, C11), run by tests/test_c_host.py. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "gimbal_gpu.h"

static void die(const char* what, int st) {
  fprintf(stderr, "%s: status %d: %s\n", what, st, gimbal_last_error());
  exit(1);
}

static void* read_file(const char* path, size_t bytes) {
  FILE* f = fopen(path, "rb");
  if (!f) {
    perror(path);
    exit(1);
  }
  void* p = malloc(bytes ? bytes : 1);
  if (fread(p, 1, bytes, f) != bytes) {
    fprintf(stderr, "%s: short read\n", path);
    exit(1);
  }
  fclose(f);
  return p;
}

int main(int argc, char** argv) {
  if (argc != 10) {
    fprintf(stderr, "usage: %s L n_e k g T C ids.bin cands.bin out.bin\n", argv[0]);
    return 2;
  }
  if (gimbal_abi_version() != GIMBAL_ABI_VERSION) {
    fprintf(stderr, "ABI version %d, header %d\n", gimbal_abi_version(), GIMBAL_ABI_VERSION);
    return 1;
  }
  gimbal_topology topo;
  topo.n_layers = atoi(argv[1]);
  topo.n_experts = atoi(argv[2]);
  topo.top_k = atoi(argv[3]);
  topo.n_gpus = atoi(argv[4]);
  const int64_t T = atoll(argv[5]), C = atoll(argv[6]);
  const int64_t L = topo.n_layers, ne = topo.n_experts, m = L * ne;
  uint8_t* ids = read_file(argv[7], (size_t)(T * L * topo.top_k));
  uint8_t* cands = read_file(argv[8], (size_t)(C * m));

  int st = gimbal_topology_validate(&topo);
  if (st) die("validate", st);
  gimbal_stats_t h = NULL;
  if ((st = gimbal_stats_create(&topo, 0, &h))) die("stats_create", st);
  if ((st = gimbal_stats_add_tokens(h, ids, 1, T, GIMBAL_MEM_HOST))) die("add_tokens", st);

  uint64_t* A = malloc((size_t)m * 8);
  uint64_t* E = malloc((size_t)((L > 1 ? L - 1 : 1) * ne * ne) * 8);
  uint64_t* W = malloc((size_t)(ne * ne) * 8);
  if ((st = gimbal_stats_read(h, A, E, W, GIMBAL_MEM_HOST))) die("stats_read", st);

  int32_t* M = malloc((size_t)m * 4);
  int32_t nM = 0;
  if ((st = gimbal_affinity_set(h, 0.0, 4, (int32_t)(m / topo.n_gpus), 0, M, &nM))) die("affinity_set", st);
  int32_t* greedy = malloc((size_t)m * 4);
  if ((st = gimbal_greedy_place(h, M, nM, 0, greedy, GIMBAL_MEM_HOST, NULL))) die("greedy_place", st);

  double* D = malloc((size_t)C * 8);
  double* cut = malloc((size_t)C * 8);
  double* obj = malloc((size_t)C * 8);
  int64_t argmin = -1;
  if ((st = gimbal_eval_costs(h, cands, C, GIMBAL_MEM_HOST, 1.0, 1.0, D, cut, obj, &argmin, GIMBAL_MEM_HOST)))
    die("eval_costs", st);

  FILE* out = fopen(argv[9], "wb");
  if (!out) {
    perror(argv[9]);
    return 1;
  }
  fwrite(A, 8, (size_t)m, out);
  fwrite(E, 8, (size_t)((L - 1) * ne * ne), out);
  fwrite(&nM, 4, 1, out);
  fwrite(M, 4, (size_t)nM, out);
  fwrite(greedy, 4, (size_t)m, out);
  fwrite(D, 8, (size_t)C, out);
  fwrite(cut, 8, (size_t)C, out);
  fwrite(obj, 8, (size_t)C, out);
  fwrite(&argmin, 8, 1, out);
  fclose(out);
  gimbal_stats_destroy(h);
  printf("c_host_pass ok: T=%lld C=%lld |M|=%d argmin=%lld\n", (long long)T, (long long)C, nM, (long long)argmin);
  return 0;
}
