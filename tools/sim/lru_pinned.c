// LRU / pinned-hot simulation of the SpMM gather stream (rows in order, edges in order).
// usage: lru col.bin rowptr.bin n cap_rows pin_rows deg_rank.bin
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb"); fseek(f, 0, SEEK_END); long nnz = ftell(f) / 4; fseek(f, 0, SEEK_SET);
  int32_t* col = malloc(nnz * 4); fread(col, 4, nnz, f); fclose(f);
  int n = atoi(argv[3]); long cap = atol(argv[4]); long pin = atol(argv[5]);
  int32_t* rank = malloc((long)n * 4); f = fopen(argv[6], "rb"); fread(rank, 4, n, f); fclose(f);
  int32_t *prev = malloc((long)n * 4), *next = malloc((long)n * 4); char* in = calloc(n, 1);
  int head = -1, tail = -1; long size = 0, miss = 0, acc = 0;
  for (long e = 0; e < nnz; ++e) {
    int v = col[e]; ++acc;
    if (rank[v] < pin) continue;  // pinned: always hit
    if (in[v]) {  // move to front
      if (head != v) {
        next[prev[v]] = next[v];
        if (next[v] >= 0) prev[next[v]] = prev[v]; else tail = prev[v];
        prev[v] = -1; next[v] = head; prev[head] = v; head = v;
      }
    } else {
      ++miss;
      in[v] = 1; prev[v] = -1; next[v] = head; if (head >= 0) prev[head] = v; head = v; if (tail < 0) tail = v;
      if (++size > cap - pin) { int t = tail; tail = prev[t]; next[tail] = -1; in[t] = 0; --size; }
    }
  }
  printf("cap %ld pin %ld: miss rate %.4f\n", cap, pin, (double)miss / acc);
  return 0;
}
