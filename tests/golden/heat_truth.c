/* Long-double serial backward-Euler solve of make_heat_problem (pde_problems.cpp:76-100) over
 * [0, 10] in `steps` uniform steps: the near-exact answer the FP64 reference and the tolerance
 * build are both measured against (tests/golden/make_heat_finals.py stores it as *_truth).
 *   gcc -O2 heat_truth.c -o heat_truth -lm && ./heat_truth 512 65536 */
#include <stdio.h>
#include <math.h>
#include <stdlib.h>
typedef long double LD;
int main(int argc,char**argv){int n=atoi(argv[1]); long steps=atol(argv[2]); LD T=10.0L;
 LD dx=1.0L/(n+1), h=T/steps; LD pi=3.14159265358979323846264338327950288L;
 LD *x=malloc(sizeof(LD)*n),*sx=malloc(sizeof(LD)*n),*cc=malloc(sizeof(LD)*n);
 for(int i=0;i<n;i++){sx[i]=sinl(pi*(i+1)*dx); x[i]=sx[i];}
 for(long k=1;k<=steps;k++){LD t=k*h; LD st=sinl(t); LD a=1+0.25L*st; LD r=h*a/(dx*dx);
  LD fa=-st, fb=a*pi*pi*cosl(t);
  for(int i=0;i<n;i++) x[i]+=h*(fa*sx[i]+fb*sx[i]);
  LD diag=1+2*r, p=diag; cc[0]=-r/p; x[0]/=p;
  for(int i=1;i<n;i++){p=diag-(-r)*cc[i-1]; cc[i]=(i<n-1)?-r/p:0; x[i]=(x[i]-(-r)*x[i-1])/p;}
  for(int i=n-2;i>=0;i--) x[i]-=cc[i]*x[i+1];
 }
 for(int i=0;i<n;i++) printf("%.21Lg\n",x[i]);
}
