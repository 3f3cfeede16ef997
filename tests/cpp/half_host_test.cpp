// Exhaustive check of the mirror's host-side binary16 conversions
// (samo::Half(float), float(Half); include/samo_b200/samo.hpp) against the
// oracle's restatement of half.hpp:13-71, itself pinned to the reference
// (tests/test_oracle.py): every one of the 2^32 float bit patterns and every
// one of the 65,536 halves, bit for bit (NaN payloads included).  Test
// infrastructure; built and run by tests/test_cpp_kat.py on the CPU.
#include <bit>
#include <cstdint>
#include <cstdio>

#include "samo_b200/samo.hpp"

extern "C" std::uint16_t or_float_to_half(float f);
extern "C" float or_half_to_float(std::uint16_t h);

int main() {
  unsigned long long bad = 0;
#pragma omp parallel for reduction(+ : bad) schedule(static)
  for (long long hi = 0; hi < 65536; ++hi) {
    for (std::uint32_t lo = 0; lo < 65536; ++lo) {
      const float f = std::bit_cast<float>(static_cast<std::uint32_t>(hi << 16) | lo);
      bad += samo::Half(f).bits() != or_float_to_half(f);
    }
  }
  unsigned long long bad_h = 0;
  for (std::uint32_t h = 0; h < 65536; ++h) {
    const float got = static_cast<float>(samo::Half::from_bits(static_cast<std::uint16_t>(h)));
    bad_h += std::bit_cast<std::uint32_t>(got) != std::bit_cast<std::uint32_t>(or_half_to_float(static_cast<std::uint16_t>(h)));
  }
  std::printf("float->half mismatches: %llu of 4294967296; half->float mismatches: %llu of 65536\n", bad, bad_h);
  return (bad || bad_h) ? 1 : 0;
}
