// Library pin for the oracle's Philox4x32-10: calls cuRAND's own
// curand_Philox4x32_10(uint4, uint2) (CUDA 12.9 curand_philox4x32_x.h) on the
// HOST.  Reads n records of (ctr[4], key[2]) uint32 from argv[1], writes n x 4
// uint32 outputs to argv[2].  Built and run by tests/test_oracle_rng.py only.
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>
#include <cstdint>
#include <vector>
int main(int argc, char** argv) {
  if (argc != 3) return 2;
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 3;
  std::vector<uint32_t> in;
  uint32_t w;
  while (fread(&w, 4, 1, f) == 1) in.push_back(w);
  fclose(f);
  size_t n = in.size() / 6;
  std::vector<uint32_t> out(4 * n);
  for (size_t i = 0; i < n; ++i) {
    uint4 c = make_uint4(in[6 * i], in[6 * i + 1], in[6 * i + 2], in[6 * i + 3]);
    uint2 k = make_uint2(in[6 * i + 4], in[6 * i + 5]);
    uint4 r = curand_Philox4x32_10(c, k);
    out[4 * i] = r.x; out[4 * i + 1] = r.y; out[4 * i + 2] = r.z; out[4 * i + 3] = r.w;
  }
  f = fopen(argv[2], "wb");
  fwrite(out.data(), 4, out.size(), f);
  fclose(f);
  return 0;
}
