// Developer probe: emit the generated kernel for a tape file with a canned binding, so
// register use / spills can be inspected offline with `nvcc -cubin -Xptxas -v`.
// usage: codegen_probe TAPE.sytp kind(tet4|tet10|tri|flap|pair) mode(0..3) schedule fast
#include <cstdio>
#include <fstream>
#include <iostream>
#include <iterator>
#include "../paper_2303_02156_b200/csrc/codegen.hpp"
using namespace symel_cuda;
int main(int argc, char** argv) {
  std::ifstream is(argv[1], std::ios::binary);
  std::vector<std::uint8_t> blob((std::istreambuf_iterator<char>(is)), {});
  TapeIR t = parse_tape(blob.data(), blob.size());
  std::string kind = argv[2];
  KernelSpec s; s.tape = &t; s.mode = (OutMode)atoi(argv[3]); s.schedule = atoi(argv[4]); s.fast = atoi(argv[5]);
  if (argc > 6) s.threads_per_block = atoi(argv[6]);
  if (argc > 7) s.min_blocks = atoi(argv[7]);
  int nodes = kind == "tet10" ? 10 : kind == "tri" ? 3 : 4;
  s.arity = nodes; s.array_comps = {3, 3, 4, 1, 144, 12};
  for (int a = 0; a < nodes; ++a) for (int c = 0; c < 3; ++c) { s.inputs.push_back({InKind::item_comp, 0, (unsigned)a, (unsigned)c}); s.dof_slots.push_back(s.inputs.size()-1); }
  if (kind == "tet4" || kind == "tet10") {
    for (int a = 0; a < nodes; ++a) for (int c = 0; c < 3; ++c) s.inputs.push_back({InKind::item_comp, 1, (unsigned)a, (unsigned)c});
    s.inputs.push_back({InKind::param, 0, 0, 0}); s.inputs.push_back({InKind::param, 0, 0, 0});
    if (kind == "tet10") { for (int k = 0; k < 4; ++k) s.inputs.push_back({InKind::sum_comp, 0, (unsigned)k, 0});
      s.n_items = 4; s.sum_arity = 4; s.sum_items = {1/24., .58, .13, .13, 1/24., .13, .58, .13, 1/24., .13,.13,.58, 1/24.,.13,.13,.13}; }
  } else if (kind == "tri") {
    for (int c = 0; c < 4; ++c) s.inputs.push_back({InKind::elem_comp, 2, 0, (unsigned)c});
    s.inputs.push_back({InKind::elem_comp, 3, 0, 0});
    s.inputs.push_back({InKind::param, 0, 0, 0}); s.inputs.push_back({InKind::param, 0, 0, 0});
  } else if (kind == "flap") {
    for (int c = 0; c < 144; ++c) s.inputs.push_back({InKind::elem_comp, 4, 0, (unsigned)c});
    s.inputs.push_back({InKind::param, 0, 0, 0});
  } else if (kind == "pair") {
    for (int c = 0; c < 12; ++c) s.inputs.push_back({InKind::elem_comp, 5, 0, (unsigned)c});
    s.inputs.push_back({InKind::param, 0, 0, 0}); s.inputs.push_back({InKind::param, 0, 0, 0});
  }
  std::cout << emit_kernel(s);
}
