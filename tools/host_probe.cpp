// Host-side per-round transcript work (native SHAKE-256 transcript + field
// finishing) timed on this machine's CPU.
//   g++ -O2 -std=c++17 -I paper_2508_21393_b200/csrc -I include -x c++ \
//       paper_2508_21393_b200/csrc/transcript.cu tools/host_probe.cpp -o host_probe
#include <chrono>
#include <cstdio>
#include "transcript.cuh"
#include "hostfield.h"
using namespace zkl;
int main() {
  uint64_t st[25] = {1};
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 200000; i++) keccak_f1600(st);
  double kus = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  HostTranscript tr;
  memset(tr.state, 7, 64);
  uint8_t ev[4][32];
  for (int x = 0; x < 4; x++) for (int b = 0; b < 32; b++) ev[x][b] = (uint8_t)(x * 31 + b);
  ev[0][31] = ev[1][31] = ev[2][31] = ev[3][31] = 0x3f;
  fr_t a = Fr255::one(), b = Fr255::r2();
  t0 = std::chrono::steady_clock::now();
  const int N = 50000;
  for (int i = 0; i < N; i++) {
    for (int x = 0; x < 4; x++) a = host::Fr::mul(a, b);
    for (int x = 0; x < 4; x++) tr.append_elem("sumcheck/eval", ev[x], 32);
    uint8_t raw[64], r[32];
    tr.challenge_squeeze("sumcheck/round", 14, raw);
    reduce512_fr(raw, r);
    a = host::Fr::add(a, host::from_canon<Fr255>(r));
    tr.challenge_absorb(raw);
  }
  double rus = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 1000000; i++) a = host::Fr::mul(a, b);
  double mus = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  printf("keccak-f %.0f ns | host mul %.1f ns | full round (4 appends + challenge + drawn + 6 mul) %.2f us  [%u]\n",
         kus * 1000 / 200000, mus * 1000 / 1e6, rus / N, a.v[0] ^ tr.state[0]);
  return 0;
}
