// Host Keccak-f[1600] timing probe: links csrc/transcript.cu compiled with different host flags (tools/probes/keccak_probe.sh).
#include <chrono>
#include <cstdint>
#include <cstdio>
namespace zkl { void keccak_f1600(uint64_t s[25]); }
int main() {
  uint64_t s[25] = {1};
  auto t0 = std::chrono::steady_clock::now();
  const int N = 200000;
  for (int i = 0; i < N; i++) zkl::keccak_f1600(s);
  auto t1 = std::chrono::steady_clock::now();
  printf("%.1f ns per keccak-f (%llx)\n", std::chrono::duration<double, std::nano>(t1 - t0).count() / N, (unsigned long long)s[0]);
}
