// Host SHAKE-256 / Keccak-f[1600] (FIPS 202) and the transcript operations.
#include "transcript.cuh"

namespace zkl {

static const uint64_t kRC[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808Aull, 0x8000000080008000ull,
    0x000000000000808Bull, 0x0000000080000001ull, 0x8000000080008081ull, 0x8000000000008009ull,
    0x000000000000008Aull, 0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000Aull,
    0x000000008000808Bull, 0x800000000000008Bull, 0x8000000000008089ull, 0x8000000000008003ull,
    0x8000000000008002ull, 0x8000000000000080ull, 0x000000000000800Aull, 0x800000008000000Aull,
    0x8000000080008081ull, 0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};

// rho offsets indexed by lane x + 5y
static const int kRho[25] = {0,  1,  62, 28, 27, 36, 44, 6,  55, 20, 3,  10, 43,
                             25, 39, 41, 45, 15, 21, 8,  18, 2,  61, 56, 14};

static inline uint64_t rotl(uint64_t v, int s) { return s ? (v << s) | (v >> (64 - s)) : v; }

// pi destination of lane i = x + 5y is y + 5 * ((2x + 3y) % 5)
static constexpr int pi_dst(int i) { return (i / 5) + 5 * ((2 * (i % 5) + 3 * (i / 5)) % 5); }

template <int I>
static inline void rho_pi(const uint64_t* a, uint64_t* b) {
  b[pi_dst(I)] = rotl(a[I], kRho[I]);
  if constexpr (I + 1 < 25) rho_pi<I + 1>(a, b);
}

void keccak_f1600(uint64_t a[25]) {
  uint64_t b[25];
  for (int round = 0; round < 24; round++) {
    const uint64_t c0 = a[0] ^ a[5] ^ a[10] ^ a[15] ^ a[20];
    const uint64_t c1 = a[1] ^ a[6] ^ a[11] ^ a[16] ^ a[21];
    const uint64_t c2 = a[2] ^ a[7] ^ a[12] ^ a[17] ^ a[22];
    const uint64_t c3 = a[3] ^ a[8] ^ a[13] ^ a[18] ^ a[23];
    const uint64_t c4 = a[4] ^ a[9] ^ a[14] ^ a[19] ^ a[24];
    const uint64_t d0 = c4 ^ rotl(c1, 1), d1 = c0 ^ rotl(c2, 1), d2 = c1 ^ rotl(c3, 1),
                   d3 = c2 ^ rotl(c4, 1), d4 = c3 ^ rotl(c0, 1);
    for (int y = 0; y < 25; y += 5) {
      a[y] ^= d0; a[y + 1] ^= d1; a[y + 2] ^= d2; a[y + 3] ^= d3; a[y + 4] ^= d4;
    }
    rho_pi<0>(a, b);
    for (int y = 0; y < 25; y += 5) {
      const uint64_t b0 = b[y], b1 = b[y + 1], b2 = b[y + 2], b3 = b[y + 3], b4 = b[y + 4];
      a[y] = b0 ^ (~b1 & b2);
      a[y + 1] = b1 ^ (~b2 & b3);
      a[y + 2] = b2 ^ (~b3 & b4);
      a[y + 3] = b3 ^ (~b4 & b0);
      a[y + 4] = b4 ^ (~b0 & b1);
    }
    a[0] ^= kRC[round];
  }
}

void shake256(const uint8_t* in, size_t len, uint8_t* out, size_t outlen) {
  const size_t rate = 136;
  uint64_t st[25] = {0};
  uint8_t* sb = reinterpret_cast<uint8_t*>(st);  // little-endian host
  while (len >= rate) {
    for (size_t i = 0; i < rate; i++) sb[i] ^= in[i];
    keccak_f1600(st);
    in += rate;
    len -= rate;
  }
  for (size_t i = 0; i < len; i++) sb[i] ^= in[i];
  sb[len] ^= 0x1F;
  sb[rate - 1] ^= 0x80;
  keccak_f1600(st);
  while (outlen) {
    size_t n = outlen < rate ? outlen : rate;
    memcpy(out, sb, n);
    out += n;
    outlen -= n;
    if (outlen) keccak_f1600(st);
  }
}

void HostTranscript::append(const char* label, size_t llen, const uint8_t* data, size_t dlen) {
  uint8_t buf[64 + 2 + 256 + 8 + 512];
  uint8_t* big = nullptr;
  size_t total = 64 + 2 + llen + 8 + dlen;
  uint8_t* p = total <= sizeof(buf) ? buf : (big = new uint8_t[total]);
  uint8_t* w = p;
  memcpy(w, state, 64); w += 64;
  w[0] = (uint8_t)llen; w[1] = (uint8_t)(llen >> 8); w += 2;
  memcpy(w, label, llen); w += llen;
  for (int i = 0; i < 8; i++) w[i] = (uint8_t)((uint64_t)dlen >> (8 * i));
  w += 8;
  memcpy(w, data, dlen);
  shake256(p, total, state, 64);
  delete[] big;
}

void HostTranscript::append_elem(const char* label, const uint8_t* canon, int nbytes) {
  int n = nbytes;
  while (n > 1 && canon[n - 1] == 0) n--;
  append(label, strlen(label), canon, (size_t)n);
}

void HostTranscript::challenge_raw(const char* label, size_t llen, uint8_t raw[64]) {
  // raw = H(state || record("challenge", label))
  uint8_t buf[64 + 2 + 9 + 8 + 256];
  uint8_t* w = buf;
  memcpy(w, state, 64); w += 64;
  w[0] = 9; w[1] = 0; w += 2;
  memcpy(w, "challenge", 9); w += 9;
  for (int i = 0; i < 8; i++) w[i] = (uint8_t)((uint64_t)llen >> (8 * i));
  w += 8;
  memcpy(w, label, llen); w += llen;
  shake256(buf, (size_t)(w - buf), raw, 64);
  append("drawn", 5, raw, 64);
}

void reduce512_fr(const uint8_t raw[64], uint8_t out[32]) {
  fr_t lo, hi;
  memcpy(&lo, raw, 32);
  memcpy(&hi, raw + 32, 32);
  for (int k = 0; k < 2; k++) {  // x < 2^256 < 3p
    if (Fr255::geq_p_portable(lo)) lo = Fr255::sub_p_portable(lo);
    if (Fr255::geq_p_portable(hi)) hi = Fr255::sub_p_portable(hi);
  }
  // hi * 2^256 mod p = mont_mul(hi, R^2)
  fr_t h = Fr255::mul_portable(hi, Fr255::r2());
  fr_t r = Fr255::add_portable(lo, h);
  memcpy(out, &r, 32);
}

void reduce512_m61(const uint8_t raw[64], uint8_t out[8]) {
  const uint64_t P = M61::P;
  unsigned __int128 acc = 0;
  for (int w = 7; w >= 0; w--) {
    uint64_t word;
    memcpy(&word, raw + 8 * w, 8);
    acc = ((acc << 64) | word) % P;
  }
  uint64_t r = (uint64_t)acc;
  memcpy(out, &r, 8);
}

}  // namespace zkl
