// LRU model of the gather traffic of a multi-column solve under the level order and the
// tile-blocked order of csrc/pattern.cpp (same construction, restated), on the bench pattern.
//   python tools/order_sim_gen.py            (writes /tmp/sim/xy.bin, nbr.bin: n = 1e6, m = 20)
//   g++ -O2 -o /tmp/sim/sim tools/order_sim.cpp && /tmp/sim/sim K S min_rows capacity_rows
// Prints, per direction, the gather misses of a sequential walk with `capacity_rows` rows of x
// resident (150000 rows = 60 MB at t = 50).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <vector>
using namespace std;
static uint64_t hilbert2(uint32_t x, uint32_t y, int order) {
  uint64_t d = 0;
  for (int64_t s = (int64_t)1 << (order - 1); s > 0; s >>= 1) {
    uint32_t rx = (x & s) > 0, ry = (y & s) > 0;
    d += (uint64_t)s * s * ((3 * rx) ^ ry);
    if (ry == 0) { if (rx == 1) { x = (uint32_t)(2*s-1) - x; y = (uint32_t)(2*s-1) - y; } swap(x, y); }
  }
  return d;
}
struct Lru {
  vector<int32_t> prev, next; vector<char> in; int32_t head=-1, tail=-1; int64_t cnt=0, cap;
  Lru(int64_t n, int64_t c): prev(n,-1), next(n,-1), in(n,0), cap(c) {}
  void unlink(int32_t r){ int32_t p=prev[r], q=next[r]; if(p>=0) next[p]=q; else head=q; if(q>=0) prev[q]=p; else tail=p; }
  void push(int32_t r){ prev[r]=-1; next[r]=head; if(head>=0) prev[head]=r; head=r; if(tail<0) tail=r; }
  bool access(int32_t r){ bool hit=in[r]; if(hit) unlink(r); else { in[r]=1; if(++cnt>cap){ int32_t t=tail; unlink(t); in[t]=0; --cnt; } } push(r); return hit; }
};
int main(int argc, char** argv) {
  const int64_t n = 1000000; const int m = 20;
  vector<double> xy(2*n); vector<int32_t> nbr(n*m);
  FILE* f = fopen("/tmp/sim/xy.bin","rb"); fread(xy.data(),8,2*n,f); fclose(f);
  f = fopen("/tmp/sim/nbr.bin","rb"); fread(nbr.data(),4,n*m,f); fclose(f);
  int K = atoi(argv[1]), S = atoi(argv[2]); int64_t minrows = atoll(argv[3]); int64_t cap = atoll(argv[4]);
  vector<int32_t> lev(n,0), hgt(n,0);
  for (int64_t i=0;i<n;++i){ int L=0; for(int k=0;k<m;++k){ int j=nbr[i*m+k]; if(j<0)break; L=max(L,lev[j]+1);} lev[i]=L; }
  for (int64_t i=n-1;i>=0;--i) for(int k=0;k<m;++k){ int j=nbr[i*m+k]; if(j<0)break; hgt[j]=max(hgt[j],hgt[i]+1);} 
  vector<uint64_t> key(n); for(int64_t i=0;i<n;++i) key[i]=hilbert2((uint32_t)(xy[2*i]*65535.999),(uint32_t)(xy[2*i+1]*65535.999),16);
  vector<int32_t> sperm(n), iperm(n); iota(sperm.begin(),sperm.end(),0);
  stable_sort(sperm.begin(),sperm.end(),[&](int a,int b){return key[a]<key[b];});
  for(int64_t s=0;s<n;++s) iperm[sperm[s]]=s;
  // storage-order deps
  vector<int32_t> par(n*m,-1), pc(n,0), slev(n), shgt(n);
  for(int64_t s=0;s<n;++s){ int i=sperm[s]; slev[s]=lev[i]; shgt[s]=hgt[i]; int c=0; for(int k=0;k<m;++k){int j=nbr[(int64_t)i*m+k]; if(j<0)break; par[s*m+c++]=iperm[j];} pc[s]=c; }
  vector<int32_t> tptr(n+1,0); for(int64_t s=0;s<n;++s) for(int k=0;k<pc[s];++k) tptr[par[s*m+k]+1]++;
  for(int64_t s=0;s<n;++s) tptr[s+1]+=tptr[s];
  vector<int32_t> tidx(tptr[n]); { vector<int32_t> fl(tptr.begin(),tptr.end()-1); for(int64_t s=0;s<n;++s) for(int k=0;k<pc[s];++k) tidx[fl[par[s*m+k]]++]=s; }
  int nlev=*max_element(lev.begin(),lev.end())+1, nhgt=*max_element(hgt.begin(),hgt.end())+1;
  // head
  vector<int64_t> lsize(nlev,0); for(int64_t i=0;i<n;++i) lsize[lev[i]]++;
  int Lh=0; int64_t H=0; while(Lh<nlev && H+lsize[Lh]<=3072) H+=lsize[Lh++];
  printf("nlev %d nhgt %d head L %d H %ld\n", nlev,nhgt,Lh,(long)H);
  for (int dir=0; dir<2; ++dir) {
    const vector<int32_t>& lv = dir==0? slev: shgt; int nl = dir==0? nlev: nhgt;
    auto ndeps=[&](int32_t s){ return dir==0? pc[s]: tptr[s+1]-tptr[s]; };
    auto dep=[&](int32_t s,int k){ return dir==0? par[(int64_t)s*m+k]: tidx[tptr[s]+k]; };
    vector<int64_t> sz(nl,0); vector<int32_t> rows; rows.reserve(n);
    for(int64_t s=0;s<n;++s) if(slev[s]>=Lh){ sz[lv[s]]++; }
    // level order
    vector<int32_t> lo; { vector<int64_t> ptr(nl+1,0); for(int l=0;l<nl;++l) ptr[l+1]=ptr[l]+sz[l]; lo.resize(ptr[nl]); vector<int64_t> fl(ptr.begin(),ptr.end()-1); for(int64_t s=0;s<n;++s) if(slev[s]>=Lh) lo[fl[lv[s]]++]=s; }
    // bulk range: maximal run of levels with sz>=minrows containing the largest level
    int lmax = max_element(sz.begin(),sz.end())-sz.begin(); int b0=lmax,b1=lmax+1; while(b0>0&&sz[b0-1]>=minrows)--b0; while(b1<nl&&sz[b1]>=minrows)++b1;
    int64_t brows=0; for(int l=b0;l<b1;++l) brows+=sz[l];
    printf("dir %d: levels %d bulk [%d,%d) rows %ld maxlevel %ld\n",dir,nl,b0,b1,(long)brows,(long)sz[lmax]);
    // tile order
    vector<int32_t> tile(n,0); vector<int32_t> to; to.reserve(lo.size());
    vector<uint64_t> okey(n,0);
    int64_t displaced=0;
    for (int32_t s : lo) {  // level order: deps first
      int l=lv[s]; if(l<b0||l>=b1) continue; int band=(l-b0)/K; int t=(int)((int64_t)s*S/n);
      int t0=t;
      for(int k=0;k<ndeps(s);++k){ int d=dep(s,k); int ld=lv[d]; if(slev[d]<Lh) continue; if(ld>=b0&&ld<b1&&(ld-b0)/K==band) t=max(t,tile[d]); }
      tile[s]=t; displaced += (t!=t0);
    }
    // build: levels <b0 in level order, then bulk by (band,tile,level,s), then levels>=b1
    vector<int32_t> bulk; for(int32_t s: lo){ int l=lv[s]; if(l<b0) to.push_back(s); else if(l<b1) bulk.push_back(s);} 
    stable_sort(bulk.begin(),bulk.end(),[&](int a,int b){ int ba=(lv[a]-b0)/K, bb=(lv[b]-b0)/K; if(ba!=bb) return ba<bb; if(tile[a]!=tile[b]) return tile[a]<tile[b]; if(lv[a]!=lv[b]) return lv[a]<lv[b]; return a<b;});
    for(int32_t s: bulk) to.push_back(s);
    for(int32_t s: lo) if(lv[s]>=b1) to.push_back(s);
    // validate topological
    { vector<int64_t> pos(n,-1); for(size_t p=0;p<to.size();++p) pos[to[p]]=p; int64_t bad=0; for(int32_t s: to) for(int k=0;k<ndeps(s);++k){int d=dep(s,k); if(slev[d]<Lh&&dir==0) continue; if(slev[d]<Lh) continue; if(pos[d]<0||pos[d]>=pos[s]) ++bad;} printf("  topo violations %ld  displaced %.1f%%\n",(long)bad, 100.0*displaced/max<int64_t>(1,brows)); }
    for (int which=0; which<2; ++which) {
      const vector<int32_t>& ord = which==0? lo: to;
      Lru L(n,cap); int64_t acc=0, miss=0, bacc=0, bmiss=0;
      for (int32_t s: ord) { bool inb = lv[s]>=b0&&lv[s]<b1; for(int k=0;k<ndeps(s);++k){ bool h=L.access(dep(s,k)); ++acc; miss+=!h; if(inb){++bacc; bmiss+=!h;} } L.access(s); }
      printf("  %s order: gathers %ld miss %ld (hit %.1f%%) -> DRAM %.2f GB at 400 B/row; bulk hit %.1f%%\n", which?"tile ":"level", (long)acc,(long)miss,100.0*(acc-miss)/acc, miss*400e-9, 100.0*(bacc-bmiss)/max<int64_t>(1,bacc));
    }
  }
}
