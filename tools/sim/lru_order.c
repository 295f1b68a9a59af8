// sequential LRU over rows in a given order file (int32 rows)
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
int main(int argc,char**argv){FILE*f=fopen(argv[1],"rb");fseek(f,0,SEEK_END);long nnz=ftell(f)/4;fseek(f,0,SEEK_SET);int32_t*col=malloc(nnz*4);if(fread(col,4,nnz,f)){}fclose(f);
int n=atoi(argv[3]);long cap=atol(argv[4]);int64_t*rp=malloc(((long)n+1)*8);f=fopen(argv[2],"rb");if(fread(rp,8,n+1,f)){}fclose(f);
int32_t*ord=malloc((long)n*4);f=fopen(argv[5],"rb");if(fread(ord,4,n,f)){}fclose(f);
int32_t*prv=malloc((long)n*4),*nx=malloc((long)n*4);char*in=calloc(n,1);int head=-1,tail=-1;long size=0,miss=0,acc=0;
for(int i=0;i<n;++i){int r=ord[i];for(int64_t e=rp[r];e<rp[r+1];++e){int v=col[e];++acc;
 if(in[v]){if(head!=v){nx[prv[v]]=nx[v];if(nx[v]>=0)prv[nx[v]]=prv[v];else tail=prv[v];prv[v]=-1;nx[v]=head;prv[head]=v;head=v;}}
 else{++miss;in[v]=1;prv[v]=-1;nx[v]=head;if(head>=0)prv[head]=v;head=v;if(tail<0)tail=v;if(++size>cap){int t=tail;tail=prv[t];nx[tail]=-1;in[t]=0;--size;}}}}
printf("miss %.4f\n",(double)miss/acc);return 0;}
