// Host harness for the device eigen fragment (tests/test_spd_clamp.py): compiles the exact
// source text the code generator emits (eig_source) as plain C++ and applies the clamp to
// matrices read from stdin. Test infrastructure only.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <string>
#define __device__
#define __forceinline__ inline
static inline double sy_rcp(double x) { return 1.0 / x; }
// the device QL keeps a warp at level L while any lane still iterates there (lookahead lanes
// work on L+1 meanwhile); a single host lane emulates that with randomly busy warp-mates
static unsigned sy_host_rng = 12345u;
static inline bool sy_host_any(bool mine) {
  sy_host_rng = sy_host_rng * 1103515245u + 12345u;
  return mine || ((sy_host_rng >> 16) % 3u) == 0u;
}
#include "clamp_fragment.inc"

template <int N, bool LA>
static int run() {
  double A[N][N];
  int count = 0;
  while (true) {
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j)
        if (!(std::cin >> A[i][j])) return count;
    double d[N], e[N];
    double V[N][N];
    for (int i = 0; i < N; ++i) for (int j = 0; j < N; ++j) V[i][j] = A[i][j];
    sy_eig<N, LA>(V, d, e);
    // clamp(M) = V max(d, 0) V^T, as the fused tile kernel rebuilds it (codegen emit_spd_tail)
    for (int i = 0; i < N; ++i)
      for (int j = 0; j <= i; ++j) {
        double c = 0.0;
        for (int k = 0; k < N; ++k) c += V[i][k] * (d[k] > 0.0 ? d[k] : 0.0) * V[j][k];
        A[i][j] = c;
      }
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) std::printf("%.17g%c", i >= j ? A[i][j] : A[j][i], j + 1 == N ? '\n' : ' ');
    ++count;
  }
}

int main(int argc, char** argv) {
  // argv[2] = "la": the lookahead QL variant (sy_ql_la), else the plain one (sy_ql)
  const int n = std::atoi(argv[1]);
  const bool la = argc > 2 && std::string(argv[2]) == "la";
  switch (n) {
    case 2: la ? run<2, true>() : run<2, false>(); break;
    case 3: la ? run<3, true>() : run<3, false>(); break;
    case 4: la ? run<4, true>() : run<4, false>(); break;
    case 6: la ? run<6, true>() : run<6, false>(); break;
    case 9: la ? run<9, true>() : run<9, false>(); break;
    default: return 2;
  }
  return 0;
}
