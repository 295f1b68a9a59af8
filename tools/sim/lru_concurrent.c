// LRU with W concurrent warps pulling items (runs of rows of ~E edges) in order, round-robin one
// group of G edges per warp per step.  usage: lru2 col.bin rowptr.bin n cap W E G
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
static int32_t *prv, *nxt; static char* in; static int head=-1, tail=-1; static long size=0, cap;
static long miss=0, acc=0;
static void touch(int v){ ++acc; if(in[v]){ if(head!=v){ nxt[prv[v]]=nxt[v]; if(nxt[v]>=0) prv[nxt[v]]=prv[v]; else tail=prv[v]; prv[v]=-1; nxt[v]=head; prv[head]=v; head=v; } }
 else { ++miss; in[v]=1; prv[v]=-1; nxt[v]=head; if(head>=0) prv[head]=v; head=v; if(tail<0) tail=v; if(++size>cap){int t=tail; tail=prv[t]; nxt[tail]=-1; in[t]=0; --size;} } }
int main(int argc,char**argv){
  FILE*f=fopen(argv[1],"rb"); fseek(f,0,SEEK_END); long nnz=ftell(f)/4; fseek(f,0,SEEK_SET);
  int32_t*col=malloc(nnz*4); if(fread(col,4,nnz,f)){} fclose(f);
  int n=atoi(argv[3]); cap=atol(argv[4]); int W=atoi(argv[5]); long E=atol(argv[6]); int G=atoi(argv[7]);
  int64_t*rp=malloc(((long)n+1)*8); f=fopen(argv[2],"rb"); if(fread(rp,8,n+1,f)){} fclose(f);
  prv=malloc((long)n*4); nxt=malloc((long)n*4); in=calloc(n,1);
  // items: runs of rows with >= E edges
  long nitems=0; int64_t* ib=malloc(((long)n+1)*8); int r0=0; long a=0; ib[0]=0;
  for(int r=0;r<n;++r){ a+=rp[r+1]-rp[r]; if(a>=E){ ib[++nitems]=rp[r+1]; a=0; r0=r+1;} }
  if(ib[nitems]<nnz) ib[++nitems]=nnz;
  long next_item=0; int64_t *cur=malloc(W*8), *end=malloc(W*8); int active=0;
  for(int w=0;w<W;++w){ if(next_item<nitems){cur[w]=ib[next_item]; end[w]=ib[next_item+1]; ++next_item; ++active;} else {cur[w]=end[w]=0;} }
  while(active>0){ for(int w=0;w<W;++w){ if(cur[w]>=end[w]) continue; for(int k=0;k<G&&cur[w]<end[w];++k) touch(col[cur[w]++]);
      if(cur[w]>=end[w]){ if(next_item<nitems){cur[w]=ib[next_item]; end[w]=ib[next_item+1]; ++next_item;} else --active; } } }
  printf("cap %ld W %d E %ld G %d: miss %.4f\n",cap,W,E,G,(double)miss/acc); return 0; }
