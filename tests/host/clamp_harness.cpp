// Host harness for the device eigen fragment (tests/test_spd_clamp.py): compiles the exact
// source text the code generator emits (eig_source) as plain C++ and applies the clamp to
// matrices read from stdin. Test infrastructure only.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
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

template <int N>
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
    sy_eig<N>(V, d, e);
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
  const int n = std::atoi(argv[1]);
  switch (n) {
    case 2: run<2>(); break;
    case 3: run<3>(); break;
    case 4: run<4>(); break;
    case 6: run<6>(); break;
    case 9: run<9>(); break;
    default: return 2;
  }
  return 0;
}
