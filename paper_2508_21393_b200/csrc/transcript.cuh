// Native Fiat-Shamir transcript, byte-identical to zklora.transcript
// (pkg/src/zklora/transcript.py:13-53):
//   record(label, data) = u16le(|label|) || label || u64le(|data|) || data
//   append:    state <- SHAKE256(state || record(label, data))[0:64]
//   challenge: raw   <- SHAKE256(state || record("challenge", label))[0:64]
//              state <- SHAKE256(state || record("drawn", raw))[0:64]
//              r = LE(raw) mod p
// ints are absorbed as their minimal little-endian encoding (>= 1 byte).
// SHAKE256 = Keccak[c=512] with rate 136 bytes and pad byte 0x1F (FIPS 202).
#pragma once
#include <stdint.h>
#include <string.h>

#include "field.cuh"

namespace zkl {

void keccak_f1600(uint64_t st[25]);
void shake256(const uint8_t* in, size_t len, uint8_t* out, size_t outlen);

struct HostTranscript {
  uint8_t state[64];

  void append(const char* label, size_t llen, const uint8_t* data, size_t dlen);
  void append_str(const char* label, const uint8_t* data, size_t dlen) {
    append(label, strlen(label), data, dlen);
  }
  // minimal little-endian encoding of a canonical element
  void append_elem(const char* label, const uint8_t* canon, int nbytes);
  void challenge_raw(const char* label, size_t llen, uint8_t raw[64]);
  // challenge_raw split in two: the 64-byte squeeze (all the next round
  // needs) and the state update by record("drawn", raw) (2 Keccak-f, off the
  // critical path: run it while the device computes).
  void challenge_squeeze(const char* label, size_t llen, uint8_t raw[64]);
  void challenge_absorb(const uint8_t raw[64]) { append("drawn", 5, raw, 64); }
};

// raw 64-byte squeeze -> canonical residue bytes (little-endian)
void reduce512_fr(const uint8_t raw[64], uint8_t out[32]);
void reduce512_m61(const uint8_t raw[64], uint8_t out[8]);

template <class F>
inline void reduce512(const uint8_t raw[64], uint8_t* out) {
  if (F::kId == 0)
    reduce512_fr(raw, out);
  else
    reduce512_m61(raw, out);
}
template <class F>
inline void challenge_canon(HostTranscript& tr, const char* label, uint8_t* out) {
  uint8_t raw[64];
  tr.challenge_raw(label, strlen(label), raw);
  reduce512<F>(raw, out);
}

}  // namespace zkl
