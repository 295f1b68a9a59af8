// LRU replay of the SpMM's gather stream under the kernel's real schedule: work items built as
// build_work_items() does (runs of ~E edges, a row longer than E alone, rows longer than 4E
// ("hubs") first, longest first, unless nohub=1), W warps pulling items from one counter, each
// warp advancing G gathers per step, round robin.  Prints the miss rate of an LRU of `cap` rows.
// usage: lru_items col.bin rowptr.bin n cap W E G [nohub: 0 hubs first, 1 row order, 2 rows split into edge ranges of E, 3 whole-row runs + long rows cut into chunks of E in row order]
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
static int32_t *prv, *nxt;
static char* in;
static int head = -1, tail = -1;
static long size = 0, cap, miss = 0, acc = 0;
static void touch(int v) {
  ++acc;
  if (in[v]) {
    if (head != v) {
      nxt[prv[v]] = nxt[v];
      if (nxt[v] >= 0) prv[nxt[v]] = prv[v]; else tail = prv[v];
      prv[v] = -1; nxt[v] = head; prv[head] = v; head = v;
    }
  } else {
    ++miss; in[v] = 1; prv[v] = -1; nxt[v] = head;
    if (head >= 0) prv[head] = v;
    head = v;
    if (tail < 0) tail = v;
    if (++size > cap) { int t = tail; tail = prv[t]; nxt[tail] = -1; in[t] = 0; --size; }
  }
}
static int64_t* hl;
static int cmp(const void* a, const void* b) {
  int64_t x = hl[*(const long*)a], y = hl[*(const long*)b];
  if (x != y) return x > y ? -1 : 1;
  return (*(const long*)a < *(const long*)b) ? -1 : 1;
}
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb"); fseek(f, 0, SEEK_END); long nnz = ftell(f) / 4; fseek(f, 0, SEEK_SET);
  int32_t* col = malloc(nnz * 4); if (fread(col, 4, nnz, f)) {} fclose(f);
  int n = atoi(argv[3]); cap = atol(argv[4]); int W = atoi(argv[5]); long E = atol(argv[6]); int G = atoi(argv[7]);
  int nohub = argc > 8 ? atoi(argv[8]) : 0;
  int64_t* rp = malloc(((long)n + 1) * 8); f = fopen(argv[2], "rb"); if (fread(rp, 8, n + 1, f)) {} fclose(f);
  prv = malloc((long)n * 4); nxt = malloc((long)n * 4); in = calloc(n, 1);
  int64_t *rb = malloc(((long)n + 1 + nnz / (E > 0 ? E : 1)) * 8), *re = malloc(((long)n + 1 + nnz / (E > 0 ? E : 1)) * 8);  // rest items [row range)
  int64_t *hb = malloc(((long)n + 1) * 8); hl = malloc(((long)n + 1) * 8);
  long nr = 0, nh = 0; int r0 = 0; long a = 0;
  for (int r = 0; r < n; ++r) {
    long d = rp[r + 1] - rp[r];
    if (d > E) {
      if (r > r0) { rb[nr] = r0; re[nr++] = r; }
      if (nohub == 3) {  // long row split into chunks of E edges, in row order (edge ranges in rb/re)
        for (long c = rp[r]; c < rp[r + 1]; c += E) { rb[nr] = -1 - c; re[nr++] = (c + E < rp[r + 1]) ? c + E : rp[r + 1]; }
      } else if (d > 4 * E && !nohub) { hb[nh] = r; hl[nh++] = d; } else { rb[nr] = r; re[nr++] = r + 1; }
      r0 = r + 1; a = 0; continue;
    }
    a += d;
    if (a >= E) { rb[nr] = r0; re[nr++] = r + 1; r0 = r + 1; a = 0; }
  }
  if (r0 < n) { rb[nr] = r0; re[nr++] = n; }
  long* ord = malloc((nh + 1) * sizeof(long));
  for (long i = 0; i < nh; ++i) ord[i] = i;
  qsort(ord, nh, sizeof(long), cmp);
  if (nohub == 2) {  // merge-path items: fixed edge ranges of E, rows split across items
    nh = 0; nr = (nnz + E - 1) / E;
  }
  long ni = nh + nr;
  int64_t *ib = malloc(ni * 8), *ie = malloc(ni * 8);  // item edge ranges (rows are contiguous)
  for (long i = 0; i < nh; ++i) { ib[i] = rp[hb[ord[i]]]; ie[i] = rp[hb[ord[i]] + 1]; }
  for (long i = 0; i < nr; ++i) {
    if (nohub == 2) { ib[i] = i * E; ie[i] = (i + 1) * E < nnz ? (i + 1) * E : nnz; }
    else if (rb[i] < 0) { ib[nh + i] = -1 - rb[i]; ie[nh + i] = re[i]; }
    else { ib[nh + i] = rp[rb[i]]; ie[nh + i] = rp[re[i]]; }
  }
  long next = 0; int64_t *cur = malloc(W * 8), *end = malloc(W * 8); int active = 0;
  for (int w = 0; w < W; ++w) {
    if (next < ni) { cur[w] = ib[next]; end[w] = ie[next]; ++next; ++active; } else cur[w] = end[w] = 0;
  }
  while (active > 0)
    for (int w = 0; w < W; ++w) {
      if (cur[w] >= end[w]) continue;
      for (int k = 0; k < G && cur[w] < end[w]; ++k) touch(col[cur[w]++]);
      if (cur[w] >= end[w]) {
        if (next < ni) { cur[w] = ib[next]; end[w] = ie[next]; ++next; } else --active;
      }
    }
  printf("cap %ld W %d E %ld G %d nohub %d items %ld hubs %ld: miss %.4f\n", cap, W, E, G, nohub, ni, nh, (double)miss / acc);
  return 0;
}
