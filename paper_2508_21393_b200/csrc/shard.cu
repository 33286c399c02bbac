// Multi-GPU dense sumcheck: the boolean hypercube sharded across the ranks of
// one node (BASELINE north star "partitioned across the 8
// B200s ... each round's handful of partial sums is all-reduced").
//
// Binding is MSB first (mle.py:50-56), so ranks own tables CYCLICALLY on the
// low log2(G) index bits: rank g holds entries I = i G + g.  Round j pairs I
// with I + 2^(n-1-j), which is on the same rank while 2^(n-1-j) >= G, so the
// first n - log2 G rounds move no table data at all:
//   each rank runs the round kernel on its shard (2^(n - log2 G) entries) and
//   gets its raw evaluations at x = 0..3; the ranks exchange them (a few
//   field elements per round), every rank adds the G vectors, applies the
//   post scalars, appends the same evaluations to its own transcript and
//   draws the same challenge;
// after those rounds each rank holds one entry per table (the global folded
// table's entry g); an all-gather of the k x G values lets every rank finish
// the last log2 G rounds on the host, identically.  The proof is the
// unsharded prover's, bit for bit (tests/test_shard.py, test_gpu_shard.py).
//
// The exchange is a host-side all-reduce through POSIX shared memory (ranks
// are processes of one node): each rank publishes its payload in its own
// cache-line-aligned slot with a release store of the exchange tag, then
// acquires every rank's slot for that tag.  Two slots per rank alternate by
// tag parity; a rank can only reuse a slot after every rank has published the
// next tag, i.e. after everyone has read this one.  No kernel ever waits on
// another rank (the per-round kernels are short launches; the waiting happens
// on the host between them), so ranks may even share one GPU.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "field.cuh"
#include "hostfield.h"
#include "ops.cuh"
#include "phase.cuh"
#include "transcript.cuh"

namespace zkl {

namespace {

constexpr uint64_t kShardMagic = 0x7a6b6c5348415244ull;  // "zklSHARD"
constexpr size_t kSlotPayload = 4096;
constexpr int kMaxWorld = 64;

struct alignas(64) Slot {
  std::atomic<uint64_t> tag;
  uint8_t pad[56];
  uint8_t data[kSlotPayload];
};

struct Region {
  uint64_t magic;
  uint64_t world;
  uint8_t pad[48];
  Slot slots[1];  // world x 2
};

struct ShardCtx {
  int rank = -1, world = 0;
  Region* region = nullptr;
  size_t bytes = 0;
  std::string name;
  uint64_t tag = 0;
};

ShardCtx& ctx() {
  static ShardCtx c;
  return c;
}

size_t region_bytes(int world) {
  return offsetof(Region, slots) + sizeof(Slot) * 2 * (size_t)world;
}

}  // namespace

int shard_world() { return ctx().region ? ctx().world : 1; }
int shard_rank() { return ctx().region ? ctx().rank : 0; }

// all-gather of nbytes per rank: out[g * nbytes ..] = rank g's payload
int shard_exchange(const void* mine, size_t nbytes, uint8_t* out) {
  ShardCtx& c = ctx();
  if (!c.region) {
    set_error("shard exchange: no shard context (zkl_shard_open)");
    return kErrArg;
  }
  if (nbytes > kSlotPayload) {
    set_error("shard exchange: payload %zu bytes > %zu", nbytes, kSlotPayload);
    return kErrArg;
  }
  const uint64_t t = ++c.tag;
  Slot* slots = c.region->slots;
  Slot& me = slots[2 * c.rank + (t & 1)];
  memcpy(me.data, mine, nbytes);
  me.tag.store(t, std::memory_order_release);
  const auto t0 = std::chrono::steady_clock::now();
  for (int g = 0; g < c.world; g++) {
    Slot& s = slots[2 * g + (t & 1)];
    for (uint32_t spin = 0; s.tag.load(std::memory_order_acquire) != t; spin++) {
      if ((spin & 1023) == 1023) {
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
          set_error("shard exchange: rank %d timed out waiting for rank %d (tag %llu)", c.rank,
                    g, (unsigned long long)t);
          return kErrCuda;
        }
        std::this_thread::yield();
      }
    }
    memcpy(out + (size_t)g * nbytes, s.data, nbytes);
  }
  return kOk;
}

// ---------------------------------------------------------------------------
// Sharded claim: `tables` are this rank's cyclic shard, 2^(num_vars - log2 G)
// entries each; num_vars, post_add (num_vars entries) are the global claim's.
template <class F>
int op_sumcheck_prove_sharded(void* const* tables, int k, int num_vars, const Terms<F>& tm,
                              const typename F::T* post_add, const typename F::T& post_mul,
                              uint8_t* state, uint8_t* rounds_out, uint8_t* point_out,
                              uint8_t* finals_out, cudaStream_t s) {
  using T = typename F::T;
  using H = typename host::For<F>::H;
  constexpr int nb = F::kBytes;
  const int G = shard_world();
  int lg = 0;
  while ((1 << lg) < G) lg++;
  if ((1 << lg) != G || lg > num_vars) {
    set_error("sumcheck_prove_sharded: world %d must be a power of two <= 2^num_vars", G);
    return kErrArg;
  }
  const int deg = tm.degree, nl = num_vars - lg;
  HostTranscript tr;
  memcpy(tr.state, state, 64);
  auto post = [&](int j, const T& raw) {
    const T add = post_add ? post_add[j] : F::zero();
    return H::mul(post_mul, H::add(raw, add));
  };
  auto emit = [&](int j, const T (&ev)[4]) {
    uint8_t* rj = rounds_out + (size_t)j * (deg + 1) * nb;
    for (int x = 0; x <= deg; x++) {
      host::to_canon<F>(rj + (size_t)x * nb, ev[x]);
      tr.append_elem("sumcheck/eval", rj + (size_t)x * nb, nb);
    }
    challenge_canon<F>(tr, "sumcheck/round", point_out + (size_t)j * nb);
    return host::from_canon<F>(point_out + (size_t)j * nb);
  };
  // local rounds: raw evaluations (no post scalars) summed over the ranks.
  // With the persistent engine (each rank on its own GPU) the exchange runs
  // inside run_phase's host loop while the rank's kernel waits for its
  // challenge; without it (ZKL_NO_PERSISTENT, profilers, ranks sharing a GPU)
  // every round is one fold + evaluation launch.
  std::vector<uint8_t> mine(4 * nb), all((size_t)G * 4 * nb);
  std::vector<uint8_t> fin((size_t)k * nb), allf((size_t)G * k * nb);
  Post<F> raw_post;
  raw_post.add = F::zero();
  raw_post.mul = H::one();
  uint64_t size = 1ull << nl;
  T r = F::zero();
  bool have_fin = false;
  if (nl > 0 && !no_persistent()) {
    PhaseArgs<F> a;
    a.tables = tables;
    a.k = k;
    a.num_vars = nl;
    a.tm = tm;
    a.post_add = post_add;  // global round j = local round j for the first nl rounds
    a.post_mul = post_mul;
    a.sharded = true;
    std::vector<T> lf(k);
    int rc = run_phase<F>(a, tr, rounds_out, point_out, lf.data(), s);
    if (rc) return rc;
    for (int q = 0; q < k; q++) host::to_canon<F>(fin.data() + (size_t)q * nb, lf[q]);
    r = host::from_canon<F>(point_out + (size_t)(nl - 1) * nb);
    have_fin = true;
  }
  for (int j = 0; j < nl && !have_fin; j++) {
    int rc = op_sumcheck_round<F>(tables, k, size, j > 0, r, tm, raw_post, mine.data(), s);
    if (rc) return rc;
    if (j > 0) size >>= 1;
    if ((rc = shard_exchange(mine.data(), (size_t)(deg + 1) * nb, all.data()))) return rc;
    T ev[4];
    for (int x = 0; x <= deg; x++) {
      T acc = F::zero();
      for (int g = 0; g < G; g++)
        acc = H::add(acc, host::from_canon<F>(all.data() + ((size_t)g * (deg + 1) + x) * nb));
      ev[x] = post(j, acc);
    }
    r = emit(j, ev);
  }
  // every rank's one entry per table (folded by the last local challenge)
  if (have_fin) {
  } else if (nl > 0) {
    int rc = op_sumcheck_finish<F>(tables, k, r, fin.data(), s);
    if (rc) return rc;
  } else {
    for (int q = 0; q < k; q++) {
      int rc = op_read<F>(fin.data() + (size_t)q * nb, tables[q], 1, s);
      if (rc) return rc;
    }
  }
  int rc = shard_exchange(fin.data(), (size_t)k * nb, allf.data());
  if (rc) return rc;
  // the last log2 G rounds over the gathered G-entry tables (index = rank)
  std::vector<std::vector<T>> tab(k, std::vector<T>(G));
  for (int q = 0; q < k; q++)
    for (int g = 0; g < G; g++)
      tab[q][g] = host::from_canon<F>(allf.data() + ((size_t)g * k + q) * nb);
  int m = G;
  for (int j = nl; j < num_vars; j++) {
    const int half = m / 2;
    T ev[4] = {F::zero(), F::zero(), F::zero(), F::zero()};
    for (int i = 0; i < half; i++) {
      T val[kMaxTables], dif[kMaxTables];
      for (int q = 0; q < k; q++) {
        val[q] = tab[q][i];
        dif[q] = H::sub(tab[q][i + half], tab[q][i]);
      }
      for (int x = 0; x <= deg; x++) {
        if (x)
          for (int q = 0; q < k; q++) val[q] = H::add(val[q], dif[q]);
        for (int t = 0; t < tm.nterms; t++) {
          T prod = tm.coef[t];
          for (int f = 0; f < tm.nf[t]; f++) prod = H::mul(prod, val[tm.fi[t][f]]);
          ev[x] = H::add(ev[x], prod);
        }
      }
    }
    for (int x = 0; x <= deg; x++) ev[x] = post(j, ev[x]);
    r = emit(j, ev);
    for (int q = 0; q < k; q++)
      for (int i = 0; i < half; i++)
        tab[q][i] = H::add(tab[q][i], H::mul(r, H::sub(tab[q][i + half], tab[q][i])));
    m = half;
  }
  for (int q = 0; q < k; q++) host::to_canon<F>(finals_out + (size_t)q * nb, tab[q][0]);
  memcpy(state, tr.state, 64);
  return kOk;
}

template int op_sumcheck_prove_sharded<Fr255>(void* const*, int, int, const Terms<Fr255>&,
                                              const Fr255::T*, const Fr255::T&, uint8_t*,
                                              uint8_t*, uint8_t*, uint8_t*, cudaStream_t);
template int op_sumcheck_prove_sharded<M61>(void* const*, int, int, const Terms<M61>&,
                                            const M61::T*, const M61::T&, uint8_t*, uint8_t*,
                                            uint8_t*, uint8_t*, cudaStream_t);

}  // namespace zkl

using namespace zkl;

extern "C" {

int zkl_shard_open(const char* name, int rank, int world) {
  ShardCtx& c = ctx();
  if (c.region) {
    set_error("shard_open: already open");
    return kErrArg;
  }
  if (world < 1 || world > kMaxWorld || (world & (world - 1)) || rank < 0 || rank >= world ||
      !name || !name[0] || strlen(name) > 200) {
    set_error("shard_open: bad arguments (rank %d, world %d)", rank, world);
    return kErrArg;
  }
  std::string nm = std::string("/zkl-") + name;
  const size_t bytes = region_bytes(world);
  int fd = shm_open(nm.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0) {
    set_error("shard_open: shm_open %s failed", nm.c_str());
    return kErrCuda;
  }
  struct stat st;
  if (fstat(fd, &st) == 0 && (size_t)st.st_size < bytes && ftruncate(fd, (off_t)bytes) != 0) {
    close(fd);
    set_error("shard_open: ftruncate failed");
    return kErrCuda;
  }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) {
    set_error("shard_open: mmap failed");
    return kErrCuda;
  }
  c.region = (Region*)p;
  c.bytes = bytes;
  c.rank = rank;
  c.world = world;
  c.name = nm;
  c.tag = 0;
  return kOk;
}

int zkl_shard_close(void) {
  ShardCtx& c = ctx();
  if (!c.region) return kOk;
  // a last exchange: no rank unmaps (or unlinks) while another still reads
  uint8_t one = 1;
  std::vector<uint8_t> all((size_t)c.world);
  int rc = shard_exchange(&one, 1, all.data());
  munmap(c.region, c.bytes);
  if (c.rank == 0) shm_unlink(c.name.c_str());
  c = ShardCtx();
  return rc;
}

int zkl_shard_world(void) { return shard_world(); }

int zkl_shard_exchange(const void* mine, uint64_t nbytes, void* out) {
  return shard_exchange(mine, (size_t)nbytes, (uint8_t*)out);
}

}  // extern "C"
