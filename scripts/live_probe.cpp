// Developer probe: max simultaneously-live doubles for a tape under a given schedule
// (outputs stored at definition). usage: live_probe TAPE.sytp schedule
#include <cstdio>
#include <fstream>
#include <iterator>
#include "../paper_2303_02156_b200/csrc/codegen.hpp"
using namespace symel_cuda;
int main(int argc, char** argv) {
  std::ifstream is(argv[1], std::ios::binary);
  std::vector<std::uint8_t> blob((std::istreambuf_iterator<char>(is)), {});
  TapeIR t = parse_tape(blob.data(), blob.size());
  auto order = schedule_instrs(t, atoi(argv[2]));
  std::uint32_t base = t.first_op_reg();
  std::vector<long> last(t.n_regs, -1), pos(t.instrs.size(), -1);
  for (size_t p = 0; p < order.size(); ++p) pos[order[p]] = p;
  for (size_t p = 0; p < order.size(); ++p) { auto& in = t.instrs[order[p]]; std::uint32_t o[3] = {in.a,in.b,in.c};
    int ar = top_arity(in.op); for (int q = 0; q < ar; ++q) last[o[q]] = std::max<long>(last[o[q]], p); }
  // live count over time (ops only; inputs assumed live throughout)
  std::vector<int> delta(order.size() + 2, 0);
  for (size_t p = 0; p < order.size(); ++p) { std::uint32_t r = base + order[p]; long l = last[r]; if (l < (long)p) l = p; delta[p]++; delta[l + 1]--; }
  int cur = 0, mx = 0; long sum = 0; for (size_t p = 0; p < order.size(); ++p) { cur += delta[p]; mx = std::max(mx, cur); sum += cur; }
  std::printf("instrs %zu scheduled %zu max_live %d mean_live %.1f\n", t.instrs.size(), order.size(), mx, double(sum)/order.size());
}
