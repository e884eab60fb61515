// ref_golden.cpp -- golden-vector generator compiled AGAINST the reference's
// own headers (/root/reference/proj/include/tiler/*.hpp).  The reference
// ships declarations only; the inline pieces it does define are the pins:
//   LcgStream::next            executor.hpp:73-81
//   GridLayout::plane/total    executor.hpp:27-32
//   IterationSpace::points_per_step  stencil.hpp:34-39
// Output: JSON on stdout (committed as tests/golden/ref_inline.json).
#include <cstdio>
#include <cstdint>
#include "tiler/executor.hpp"

int main() {
  std::printf("{\n  \"lcg\": {\n");
  const std::uint64_t seeds[] = {0ULL, 1ULL, 7ULL, 1806ULL, 0xDEADBEEFULL,
                                 18446744073709551615ULL};
  for (int si = 0; si < 6; ++si) {
    tiler::LcgStream s(seeds[si]);
    std::printf("    \"%llu\": [", (unsigned long long)seeds[si]);
    for (int i = 0; i < 64; ++i) {
      float v = s.next();
      std::printf("%s%.9g", i ? ", " : "", (double)v);
    }
    std::printf("]%s\n", si < 5 ? "," : "");
  }
  std::printf("  },\n  \"lcg_bits_seed7\": [");
  {
    tiler::LcgStream s(7);
    for (int i = 0; i < 16; ++i) {
      float v = s.next();
      std::uint32_t b;
      __builtin_memcpy(&b, &v, 4);
      std::printf("%s%u", i ? ", " : "", b);
    }
  }
  std::printf("],\n  \"lcg_state_after_1000_seed7\": ");
  {
    tiler::LcgStream s(7);
    for (int i = 0; i < 1000; ++i) s.next();
    std::printf("%llu", (unsigned long long)s.state);
  }
  std::printf(",\n  \"layout\": [\n");
  struct L { int n; long long D[3]; int h[3]; long long slots; };
  const L ls[] = {{1, {8, 0, 0}, {1, 0, 0}, 2},
                  {2, {1024, 1024, 0}, {1, 1, 0}, 9},
                  {3, {256, 256, 256}, {2, 2, 2}, 5},
                  {3, {512, 512, 512}, {4, 4, 4}, 3},
                  {3, {70, 28, 5}, {2, 0, 1}, 4}};
  for (int li = 0; li < 5; ++li) {
    tiler::GridLayout g;
    g.slots = ls[li].slots;
    for (int i = 0; i < ls[li].n; ++i) {
      g.interior.push_back(ls[li].D[i]);
      g.halo.push_back(ls[li].h[i]);
      g.padded.push_back(ls[li].D[i] + 2 * ls[li].h[i]);
    }
    tiler::IterationSpace sp;
    sp.extents = g.interior;
    std::printf("    {\"extents\": [");
    for (int i = 0; i < ls[li].n; ++i) std::printf("%s%lld", i ? ", " : "", ls[li].D[i]);
    std::printf("], \"halo\": [");
    for (int i = 0; i < ls[li].n; ++i) std::printf("%s%d", i ? ", " : "", ls[li].h[i]);
    std::printf("], \"slots\": %lld, \"plane\": %lld, \"total_elems\": %lld, \"points_per_step\": %lld}%s\n",
                ls[li].slots, (long long)g.plane(), (long long)g.total_elems(),
                (long long)sp.points_per_step(), li < 4 ? "," : "");
  }
  std::printf("  ]\n}\n");
  return 0;
}
