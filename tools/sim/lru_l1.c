// Per-SM L1 hit rate of the SpMM gathers under two ways of dealing work items to SMs.
//   mode 0: the shipped hub-first whole-row items (runs of ~E edges, rows > 4E first, longest
//           first), dealt round robin (item i -> SM i % nsm: dynamic fetch from one counter);
//   mode 1: row-order items with rows > E cut into chunks of E, each SM a contiguous slice.
// Each SM runs W streams (its warps) round robin, G gathers per stream step, through an LRU of
// `cap` rows.  usage: lru_l1 col.bin rowptr.bin n cap nsm W E G mode [sms_simulated]
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static int32_t *prv, *nxt, *stamp;
static int head = -1, tail = -1, cur_sm = 0;
static long size = 0, cap, miss = 0, acc = 0;
static char* in;
static void reset(void) { head = tail = -1; size = 0; ++cur_sm; }
static void touch(int v) {
  ++acc;
  if (in[v] && stamp[v] == cur_sm) {
    if (head != v) {
      nxt[prv[v]] = nxt[v];
      if (nxt[v] >= 0) prv[nxt[v]] = prv[v]; else tail = prv[v];
      prv[v] = -1; nxt[v] = head; prv[head] = v; head = v;
    }
  } else {
    ++miss; in[v] = 1; stamp[v] = cur_sm; prv[v] = -1; nxt[v] = head;
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
  int n = atoi(argv[3]); cap = atol(argv[4]); int nsm = atoi(argv[5]); int W = atoi(argv[6]);
  long E = atol(argv[7]); int G = atoi(argv[8]); int mode = atoi(argv[9]);
  int nsim = argc > 10 ? atoi(argv[10]) : nsm;
  int64_t* rp = malloc(((long)n + 1) * 8); f = fopen(argv[2], "rb"); if (fread(rp, 8, n + 1, f)) {} fclose(f);
  prv = malloc((long)n * 4); nxt = malloc((long)n * 4); stamp = calloc(n, 4); in = calloc(n, 1);
  long maxi = n + nnz / E + 2;
  int64_t *ib = malloc(maxi * 8), *ie = malloc(maxi * 8);
  long ni = 0;
  if (mode == 0) {
    int64_t *rb = malloc(maxi * 8), *re = malloc(maxi * 8), *hb = malloc(maxi * 8); hl = malloc(maxi * 8);
    long nr = 0, nh = 0; int r0 = 0; long a = 0;
    for (int r = 0; r < n; ++r) {
      long d = rp[r + 1] - rp[r];
      if (d > E) {
        if (r > r0) { rb[nr] = r0; re[nr++] = r; }
        if (d > 4 * E) { hb[nh] = r; hl[nh++] = d; } else { rb[nr] = r; re[nr++] = r + 1; }
        r0 = r + 1; a = 0; continue;
      }
      a += d;
      if (a >= E) { rb[nr] = r0; re[nr++] = r + 1; r0 = r + 1; a = 0; }
    }
    if (r0 < n) { rb[nr] = r0; re[nr++] = n; }
    long* ord = malloc((nh + 1) * sizeof(long));
    for (long i = 0; i < nh; ++i) ord[i] = i;
    qsort(ord, nh, sizeof(long), cmp);
    for (long i = 0; i < nh; ++i) { ib[ni] = rp[hb[ord[i]]]; ie[ni++] = rp[hb[ord[i]] + 1]; }
    for (long i = 0; i < nr; ++i) { ib[ni] = rp[rb[i]]; ie[ni++] = rp[re[i]]; }
  } else {
    int r0 = 0; long a = 0;
    for (int r = 0; r < n; ++r) {
      long d = rp[r + 1] - rp[r];
      if (d > E) {
        if (r > r0) { ib[ni] = rp[r0]; ie[ni++] = rp[r]; }
        for (int64_t c = rp[r]; c < rp[r + 1]; c += E) { ib[ni] = c; ie[ni++] = c + E < rp[r + 1] ? c + E : rp[r + 1]; }
        r0 = r + 1; a = 0; continue;
      }
      a += d;
      if (a >= E) { ib[ni] = rp[r0]; ie[ni++] = rp[r + 1]; r0 = r + 1; a = 0; }
    }
    if (r0 < n) { ib[ni] = rp[r0]; ie[ni++] = rp[n]; }
  }
  int64_t *cur = malloc(W * 8), *end = malloc(W * 8);
  long* list = malloc(ni * sizeof(long));
  for (int sm = 0; sm < nsim; ++sm) {
    int smi = (int)((long)sm * nsm / nsim);
    long nl = 0;
    if (mode == 0) { for (long i = smi; i < ni; i += nsm) list[nl++] = i; }
    else { long b = (long)smi * ni / nsm, e = (long)(smi + 1) * ni / nsm; for (long i = b; i < e; ++i) list[nl++] = i; }
    reset();
    long next = 0; int active = 0;
    for (int w = 0; w < W; ++w) {
      if (next < nl) { cur[w] = ib[list[next]]; end[w] = ie[list[next]]; ++next; ++active; } else cur[w] = end[w] = 0;
    }
    while (active > 0)
      for (int w = 0; w < W; ++w) {
        if (cur[w] >= end[w]) continue;
        for (int k = 0; k < G && cur[w] < end[w]; ++k) touch(col[cur[w]++]);
        if (cur[w] >= end[w]) {
          if (next < nl) { cur[w] = ib[list[next]]; end[w] = ie[list[next]]; ++next; } else --active;
        }
      }
  }
  printf("cap %ld nsm %d W %d E %ld G %d mode %d items %ld (%d SMs simulated): L1 hit %.4f\n", cap, nsm, W, E, G, mode, ni,
         nsim, 1.0 - (double)miss / acc);
  return 0;
}
