// Library pin for the oracle's Philox4x32-10: PyTorch's host-callable
// at::philox_engine (ATen/core/PhiloxRNGEngine.h).  Reads lines
// "key0 key1 c0 c1 c2 c3" (decimal) on stdin and prints the 4 output words.
// philox_engine(seed, subsequence, offset) uses key = seed and
// counter = (offset lo, offset hi, subsequence lo, subsequence hi).
#include <ATen/core/PhiloxRNGEngine.h>
#include <cstdio>
#include <cstdint>
int main() {
  unsigned long long k0, k1, c0, c1, c2, c3;
  while (std::scanf("%llu %llu %llu %llu %llu %llu", &k0, &k1, &c0, &c1, &c2, &c3) == 6) {
    uint64_t seed = (k1 << 32) | k0;
    uint64_t subseq = (c3 << 32) | c2;
    uint64_t offset = (c1 << 32) | c0;
    at::philox_engine e(seed, subseq, offset);
    uint32_t o0 = e(), o1 = e(), o2 = e(), o3 = e();
    std::printf("%u %u %u %u\n", o0, o1, o2, o3);
  }
  return 0;
}
