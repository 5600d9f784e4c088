// Host packing of the occupancy upload (csrc/pack.cpp) against a scalar restatement of grid.hpp:20
// (nonzero byte = obstacle), over ragged widths and arbitrary nonzero obstacle bytes.  The ISA variant
// is chosen by AM_PACK_ISA (tests/test_pack_cpu.py runs each).
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

namespace am {
void pack_rows(const uint8_t* occ, uint32_t W, uint32_t r0, uint32_t r1, uint32_t pw, uint32_t* out);
}

int main() {
  std::mt19937 rng(7);
  long bad = 0, words = 0;
  for (uint32_t W : {1u, 2u, 31u, 32u, 33u, 63u, 64u, 65u, 95u, 96u, 97u, 127u, 128u, 129u, 1000u, 1031u, 23170u}) {
    const uint32_t H = 9, pw = (W + 31) / 32, r0 = 3;
    std::vector<uint8_t> occ((size_t)W * H + 64);  // slack: no variant may read past the last row
    for (auto& b : occ) b = rng() % 3 == 0 ? (uint8_t)(1 + rng() % 255) : 0;
    std::vector<uint32_t> out((size_t)pw * (H - r0), 0xdeadbeefu);
    am::pack_rows(occ.data(), W, r0, H, pw, out.data());
    for (uint32_t r = r0; r < H; ++r)
      for (uint32_t w = 0; w < pw; ++w, ++words) {
        uint32_t v = 0;
        for (uint32_t c = 32 * w; c < W && c < 32 * w + 32; ++c) v |= (occ[(size_t)r * W + c] != 0 ? 1u : 0u) << (c & 31);
        if (out[(size_t)(r - r0) * pw + w] != v) ++bad;
      }
  }
  std::printf("pack words %ld, mismatches %ld\n", words, bad);
  return bad != 0;
}
