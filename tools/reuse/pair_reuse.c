/* pair_reuse.c -- analysis only (tools/reuse/run.sh): counts how often the
 * reference build re-evaluates a pair it evaluated before, with an exact set and
 * with direct-mapped memo tables of several sizes.  Built against the oracle
 * (test infrastructure) with its scan_vertex l2 call routed through hook_l2. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static float hook_l2(uint32_t a, uint32_t b, const float* data, uint32_t d);
#include "oracle_hooked.c"
/* exact set of seen pairs (open addressing), and direct-mapped caches */
static uint64_t *set; static uint64_t setcap;
static uint64_t evals, repeats, repeats_pass, pass_no;
static uint32_t *lastpass;
#define NDM 4
static uint64_t *dm[NDM]; static int dmbits[NDM]; static uint64_t dmhit[NDM];
static uint64_t mix(uint64_t z){z^=z>>33;z*=0xff51afd7ed558ccdULL;z^=z>>33;z*=0xc4ceb9fe1a85ec53ULL;z^=z>>33;return z;}
static float hook_l2(uint32_t a, uint32_t b, const float* data, uint32_t d){
  uint32_t lo=a<b?a:b, hi=a<b?b:a; uint64_t k=((uint64_t)lo<<32|hi)+1;
  ++evals;
  uint64_t h=mix(k)&(setcap-1);
  while(set[h] && set[h]!=k) h=(h+1)&(setcap-1);
  if(set[h]==k){++repeats; if(lastpass[h]==pass_no) ++repeats_pass; lastpass[h]=pass_no;}
  else {set[h]=k; lastpass[h]=pass_no;}
  for(int i=0;i<NDM;i++){uint64_t s=mix(k^0x1234567ULL)&((1ull<<dmbits[i])-1); if(dm[i][s]==k) ++dmhit[i]; else dm[i][s]=k;}
  return ro_l2_sq(data+(uint64_t)a*d, data+(uint64_t)b*d, d);
}
int dg_synth(int cfg, uint64_t seed, uint64_t row0, uint64_t nrows, float* out);
int main(int argc,char**argv){
  uint64_t n=atoll(argv[1]); int cfg=atoi(argv[2]); int dim=atoi(argv[3]);
  float* x=malloc(n*dim*4); dg_synth(cfg,cfg,0,n,x);
  setcap=1ull<<31; set=calloc(setcap,8); lastpass=calloc(setcap,4);
  int base=atoi(argv[4]);
  for(int i=0;i<NDM;i++){dmbits[i]=base+2*i; dm[i]=calloc(1ull<<dmbits[i],8);}
  ro_graph* g=ro_graph_new(n);
  if(ro_random_init(g,x,dim,20,42)) return 1;
  uint64_t c[4];
  for(uint32_t t1=1;t1<=4;t1++){ for(uint32_t t2=0;t2<15;t2++){
    uint64_t e0=evals,r0=repeats,rp0=repeats_pass,h0[NDM]; for(int i=0;i<NDM;i++)h0[i]=dmhit[i];
    ro_update_pass(g,x,dim,c); 
    printf("pass %2lu evals %9lu repeat %.3f (same pass %.3f) dm:",pass_no,evals-e0,(double)(repeats-r0)/(evals-e0+1e-9),(double)(repeats_pass-rp0)/(evals-e0+1e-9));
    for(int i=0;i<NDM;i++) printf(" 2^%d %.3f",dmbits[i],(double)(dmhit[i]-h0[i])/(evals-e0+1e-9));
    printf("\n"); fflush(stdout); pass_no++; }
    if(t1!=4) ro_add_reverse_edges(g,96,0);}
  printf("total evals %lu repeats %.4f same-pass %.4f\n",evals,(double)repeats/evals,(double)repeats_pass/evals);
  for(int i=0;i<NDM;i++) printf("dm 2^%d hit %.4f\n",dmbits[i],(double)dmhit[i]/evals);
}
