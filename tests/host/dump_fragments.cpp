// Writes the device eigen fragments as the code generator emits them (test infrastructure).
#include <cstdio>
#include "codegen.hpp"
int main() {
  std::fputs(symel_cuda::eig_source(), stdout);
  return 0;
}
