// ref_rng_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Compiles the reference's own header-only RNG (proj/include/adagio/rng.hpp,
// which needs nothing but the C++ standard library) straight from the
// read-only reference checkout and prints golden vectors as JSON.  Built by
// `make -C oracle ref` into oracle/_ref/ (git-ignored); oracle/make_golden.py
// runs it and freezes the output into tests/golden/rng_golden.json so the GPU
// box (which has no /root/reference) can still check bit-exactness.
#include "adagio/rng.hpp"

#include <cinttypes>
#include <cstdio>

int main() {
  using namespace adagio;
  const std::uint64_t seeds[] = {0ULL, 1ULL, 7ULL, 99ULL, 123ULL, 0xdeadbeefULL, ~0ULL};
  const char* purposes[] = {"jl", "spectral", "sampling", "ties", "folds", ""};
  std::printf("{\n  \"mix64\": [");
  for (int t = 0; t < 7; ++t) std::printf("%s[\"%" PRIu64 "\", \"%" PRIu64 "\"]", t ? ", " : "", seeds[t], mix64(seeds[t]));
  std::printf("],\n  \"fnv1a64\": [");
  for (int p = 0; p < 6; ++p) std::printf("%s[\"%s\", \"%" PRIu64 "\"]", p ? ", " : "", purposes[p], fnv1a64(purposes[p]));
  std::printf("],\n  \"derive_seed\": [");
  bool first = true;
  for (int t = 0; t < 7; ++t)
    for (int p = 0; p < 5; ++p) {
      std::printf("%s[\"%" PRIu64 "\", \"%s\", \"%" PRIu64 "\"]", first ? "" : ", ", seeds[t], purposes[p], derive_seed(seeds[t], purposes[p]));
      first = false;
    }
  std::printf("],\n  \"hash_position\": [");
  first = true;
  for (int t = 0; t < 4; ++t)
    for (std::uint64_t i = 0; i < 5; ++i)
      for (std::uint64_t j = 0; j < 7; j += 3) {
        std::printf("%s[\"%" PRIu64 "\", %" PRIu64 ", %" PRIu64 ", \"%" PRIu64 "\", %.1f]", first ? "" : ", ", seeds[t], i, j, hash_position(seeds[t], i, j), rademacher_sign(seeds[t], i, j));
        first = false;
      }
  std::printf("],\n  \"stream\": [");
  for (int t = 0; t < 3; ++t) {
    SeededRng rng(seeds[t + 2]);
    std::printf("%s{\"seed\": \"%" PRIu64 "\", \"u64\": [", t ? ", " : "", seeds[t + 2]);
    for (int c = 0; c < 8; ++c) std::printf("%s\"%" PRIu64 "\"", c ? ", " : "", rng.next_u64());
    std::printf("], \"below_1000\": [");
    for (int c = 0; c < 8; ++c) std::printf("%s%" PRIu64, c ? ", " : "", rng.below(1000));
    std::printf("], \"normal\": [");
    for (int c = 0; c < 9; ++c) std::printf("%s%.17g", c ? ", " : "", rng.normal());
    std::printf("]}");
  }
  std::printf("]\n}\n");
  return 0;
}
