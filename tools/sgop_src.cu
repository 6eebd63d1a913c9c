// Dump the generated SG-operator source for a tensor (offline inspection:
// compile it with nvcc -cubin -arch=sm_100a -Xptxas -v to read registers/spills).
//   tools/bin/sgop_src <n_vars> <p_in> <p_out> <out.cu>
#include <cstdio>
#include <cstdlib>

#include "../paper_2512_23027_b200/csrc/sgop.cu"

namespace sgw { std::atomic<long long> g_launches{0}; }

int main(int argc, char** argv) {
  if (argc < 5) return 1;
  const sgw::TensorHost t = sgw::triple_products(std::atoi(argv[1]), std::atoi(argv[2]), std::atoi(argv[3]));
  sgw::SgOpJit J;
  const std::string src = sgw::sgop_source(t.n_out, t.n_in, t, &J);
  FILE* f = std::fopen(argv[4], "w");
  std::fputs(src.c_str(), f);
  std::fclose(f);
  std::printf("NT=%d NIN=%d G=%d NW=%d IC=%d S=%d NCHUNK=%d CPS=%d regs=%d smem=%zu pairs=%lld coef=%lld\n", J.NT,
              J.NIN, J.G, J.NW, J.IC, J.S, J.NCHUNK, J.CPS, J.regs, J.smem, J.n_pairs, J.n_coef);
  return 0;
}
