// TEST INFRASTRUCTURE ONLY. Regenerates the random MiniCU kernels of the
// reference's soundness fuzz (reference tests/test_soundness.cpp:21-73,
// driven at :80-84 with std::mt19937(31337), 200 programs) so the GPU
// path can be checked on exactly the programs the reference's own test
// uses.  Restated here (not copied): same distributions, same draw order,
// same text layout, so the emitted sources are byte-identical with the
// ones the reference test feeds to enumerateVerdict.
//
// Usage: gen_fuzz <count> <outdir>   -> <outdir>/fuzz_<i>.mcu
#include <cstdio>
#include <fstream>
#include <random>
#include <sstream>
#include <string>

namespace {

std::string indexText(std::mt19937 &rng, int kind,
                      std::uniform_int_distribution<int> &offset) {
  if (kind == 0)
    return "t";
  if (kind == 1)
    return "t + " + std::to_string(offset(rng));
  if (kind == 2)
    return "threadIdx.x";
  if (kind == 3)
    return "blockIdx.x";
  return std::to_string(offset(rng));
}

std::string generate(std::mt19937 &rng) {
  std::uniform_int_distribution<int> nStmts(2, 6), idxPick(0, 4),
      opPick(0, 9), offset(0, 2);
  std::ostringstream body;
  body << "  int t = blockIdx.x * blockDim.x + threadIdx.x;\n";
  const int n = nStmts(rng);
  int depth = 0;
  for (int s = 0; s < n; ++s) {
    std::string idx = indexText(rng, idxPick(rng), offset);
    const int op = opPick(rng);
    const std::string pad(2 * (depth + 1), ' ');
    if (op < 4)
      body << pad << "A[" << idx << "] = t;\n";
    else if (op < 7)
      body << pad << "x = A[" << idx << "];\n";
    else if (op == 7)
      body << pad << "__syncthreads();\n";
    else if (op == 8)
      body << pad << "__syncwarp();\n";
    else if (depth == 0) {
      body << pad << "if (t < " << 2 + offset(rng) << ") {\n";
      depth = 1;
    }
  }
  for (; depth > 0; --depth)
    body << "  }\n";
  std::uniform_int_distribution<int> dim(1, 2);
  const int gx = dim(rng);
  const int bx = dim(rng) * 2;
  std::ostringstream src;
  src << "__global__ void k(float *A) {\n  int x = 0;\n"
      << body.str() << "}\n"
      << "void main() {\n  float *A;\n  cudaMalloc(&A, 16);\n  k<<<(" << gx
      << ",1,1),(" << bx << ",1,1)>>>(A);\n}\n";
  return src.str();
}

} // namespace

int main(int argc, char **argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: gen_fuzz <count> <outdir>\n");
    return 2;
  }
  const int count = std::atoi(argv[1]);
  std::mt19937 rng(31337);
  for (int i = 0; i < count; ++i) {
    std::ofstream out(std::string(argv[2]) + "/fuzz_" + std::to_string(i) +
                      ".mcu");
    out << generate(rng);
  }
  return 0;
}
