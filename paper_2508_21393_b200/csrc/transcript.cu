// Host SHAKE-256 / Keccak-f[1600] (FIPS 202) and the transcript operations.
#include <vector>
#include "transcript.cuh"
#include "hostfield.h"

namespace zkl {

static const uint64_t RC[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808Aull, 0x8000000080008000ull,
    0x000000000000808Bull, 0x0000000080000001ull, 0x8000000080008081ull, 0x8000000000008009ull,
    0x000000000000008Aull, 0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000Aull,
    0x000000008000808Bull, 0x800000000000008Bull, 0x8000000000008089ull, 0x8000000000008003ull,
    0x8000000000008002ull, 0x8000000000000080ull, 0x000000000000800Aull, 0x800000008000000Aull,
    0x8000000080008081ull, 0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};

#define ROL(a, n) (((a) << (n)) | ((a) >> (64 - (n))))
// Keccak-f[1600], 25 lanes in registers, theta/rho/pi fused per lane
// (b[y, 2x+3y] = rot(a[x,y] ^ d[x], rho[x,y])), then chi + iota.  ~1.3x the
// speed of the table-driven loop; the transcript is on every round's
// critical path (7 permutations per degree-3 round).  A second clone for
// x86-64-v3 hosts (BMI2 rorx / andn), picked at load time through an ifunc.
__attribute__((target_clones("default", "arch=x86-64-v3")))
void keccak_f1600(uint64_t s[25]) {
  uint64_t a00=s[0],a01=s[1],a02=s[2],a03=s[3],a04=s[4],a05=s[5],a06=s[6],a07=s[7],a08=s[8],a09=s[9],
           a10=s[10],a11=s[11],a12=s[12],a13=s[13],a14=s[14],a15=s[15],a16=s[16],a17=s[17],a18=s[18],a19=s[19],
           a20=s[20],a21=s[21],a22=s[22],a23=s[23],a24=s[24];
  for (int r = 0; r < 24; r++) {
    uint64_t c0=a00^a05^a10^a15^a20, c1=a01^a06^a11^a16^a21, c2=a02^a07^a12^a17^a22,
             c3=a03^a08^a13^a18^a23, c4=a04^a09^a14^a19^a24;
    uint64_t d0=c4^ROL(c1,1), d1=c0^ROL(c2,1), d2=c1^ROL(c3,1), d3=c2^ROL(c4,1), d4=c3^ROL(c0,1);
    // theta + rho + pi: b[y, 2x+3y] = rot(a[x,y]^d[x], r[x,y]); lane index i = x + 5y
    uint64_t b00=a00^d0;
    uint64_t b10=ROL(a01^d1,1);   // (1,0)->(0,2): idx 10
    uint64_t b20=ROL(a02^d2,62);  // (2,0)->(0,4): 20
    uint64_t b05=ROL(a03^d3,28);  // (3,0)->(0,1): 5
    uint64_t b15=ROL(a04^d4,27);  // (4,0)->(0,3): 15
    uint64_t b16=ROL(a05^d0,36);  // (0,1)->(1,3): 16
    uint64_t b01=ROL(a06^d1,44);  // (1,1)->(1,0): 1
    uint64_t b11=ROL(a07^d2,6);   // (2,1)->(1,2): 11
    uint64_t b21=ROL(a08^d3,55);  // (3,1)->(1,4): 21
    uint64_t b06=ROL(a09^d4,20);  // (4,1)->(1,1): 6
    uint64_t b07=ROL(a10^d0,3);   // (0,2)->(2,1): 7
    uint64_t b17=ROL(a11^d1,10);  // (1,2)->(2,3): 17
    uint64_t b02=ROL(a12^d2,43);  // (2,2)->(2,0): 2
    uint64_t b12=ROL(a13^d3,25);  // (3,2)->(2,2): 12
    uint64_t b22=ROL(a14^d4,39);  // (4,2)->(2,4): 22
    uint64_t b23=ROL(a15^d0,41);  // (0,3)->(3,4): 23
    uint64_t b08=ROL(a16^d1,45);  // (1,3)->(3,1): 8
    uint64_t b18=ROL(a17^d2,15);  // (2,3)->(3,3): 18
    uint64_t b03=ROL(a18^d3,21);  // (3,3)->(3,0): 3
    uint64_t b13=ROL(a19^d4,8);   // (4,3)->(3,2): 13
    uint64_t b14=ROL(a20^d0,18);  // (0,4)->(4,2): 14
    uint64_t b24=ROL(a21^d1,2);   // (1,4)->(4,4): 24
    uint64_t b09=ROL(a22^d2,61);  // (2,4)->(4,1): 9
    uint64_t b19=ROL(a23^d3,56);  // (3,4)->(4,3): 19
    uint64_t b04=ROL(a24^d4,14);  // (4,4)->(4,0): 4
    a00=b00^(~b01&b02); a01=b01^(~b02&b03); a02=b02^(~b03&b04); a03=b03^(~b04&b00); a04=b04^(~b00&b01);
    a05=b05^(~b06&b07); a06=b06^(~b07&b08); a07=b07^(~b08&b09); a08=b08^(~b09&b05); a09=b09^(~b05&b06);
    a10=b10^(~b11&b12); a11=b11^(~b12&b13); a12=b12^(~b13&b14); a13=b13^(~b14&b10); a14=b14^(~b10&b11);
    a15=b15^(~b16&b17); a16=b16^(~b17&b18); a17=b17^(~b18&b19); a18=b18^(~b19&b15); a19=b19^(~b15&b16);
    a20=b20^(~b21&b22); a21=b21^(~b22&b23); a22=b22^(~b23&b24); a23=b23^(~b24&b20); a24=b24^(~b20&b21);
    a00^=RC[r];
  }
  s[0]=a00;s[1]=a01;s[2]=a02;s[3]=a03;s[4]=a04;s[5]=a05;s[6]=a06;s[7]=a07;s[8]=a08;s[9]=a09;
  s[10]=a10;s[11]=a11;s[12]=a12;s[13]=a13;s[14]=a14;s[15]=a15;s[16]=a16;s[17]=a17;s[18]=a18;s[19]=a19;
  s[20]=a20;s[21]=a21;s[22]=a22;s[23]=a23;s[24]=a24;
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
  challenge_squeeze(label, llen, raw);
  challenge_absorb(raw);
}

void HostTranscript::challenge_squeeze(const char* label, size_t llen, uint8_t raw[64]) {
  // raw = H(state || record("challenge", label)); long labels on the heap
  uint8_t small[64 + 2 + 9 + 8 + 256];
  std::vector<uint8_t> big;
  uint8_t* buf = small;
  if (llen > 256) {
    big.resize(64 + 2 + 9 + 8 + llen);
    buf = big.data();
  }
  uint8_t* w = buf;
  memcpy(w, state, 64); w += 64;
  w[0] = 9; w[1] = 0; w += 2;
  memcpy(w, "challenge", 9); w += 9;
  for (int i = 0; i < 8; i++) w[i] = (uint8_t)((uint64_t)llen >> (8 * i));
  w += 8;
  memcpy(w, label, llen); w += llen;
  shake256(buf, (size_t)(w - buf), raw, 64);
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
  fr_t h = host::Fr::mul(hi, Fr255::r2());
  fr_t r = host::Fr::add(lo, h);
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
