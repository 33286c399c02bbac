// Host API of the persistent sumcheck engine (persistent.cu), shared by the
// C-ABI entry zkl_sumcheck_prove and the native gadget drivers (zkmat.cu).
#pragma once
#include <functional>
#include <vector>

#include "ops.cuh"
#include "transcript.cuh"

namespace zkl {

enum Shape {
  kGeneric = 0, kProd2 = 1, kProd3 = 2, kSum2Prod2 = 3, kLogup = 4, kLogupTiled = 5,
  kZkMat = 6
};

template <class F>
int detect_shape(const Terms<F>& tm);

// One sumcheck (or one phase of a factored gadget) over device tables.
//   evals[x] = post_mul * (post_add[j] + sum_i combine(terms, t_x(i)))
// Tables are consumed (folded in place).  Term coefficients and the post
// scalars are applied on the host for the recognised shapes.
template <class F>
struct PhaseArgs {
  using T = typename F::T;
  void* const* tables = nullptr;
  int k = 0;
  int num_vars = 0;
  Terms<F> tm;
  const T* post_add = nullptr;  // num_vars values (storage form) or null
  T post_mul;                   // storage form
  // called once before the first round is finished on the host (e.g. to wait
  // for a device scalar or a previous phase's finals); may fill the vector
  // with post_add values and may update post_mul / tm.coef (host-applied
  // for the recognised shapes; the generic shape needs them at launch)
  std::function<int(std::vector<T>&)> prepare;
  uint32_t seq0 = 0;  // set by run_phase: mailbox sequence base of the launch
  // > 0: run only the first `rounds_limit` rounds (no finals; the caller folds
  // by the last challenge and continues with another phase).  Required for
  // the LOGUP_TILED shape, whose structure holds only while the bound
  // variables are above the tiled tables' index bits.
  int rounds_limit = 0;
  // > 0: the last `host_tail` rounds run on the host.  The cluster kernel
  // stops after round n - host_tail - 1, folds by its challenge and sends the
  // 2^host_tail-entry tables through the mailbox; the host finishes the
  // rounds (same evaluations, same transcript) and the finals, which
  // wait_phase_finals then returns.  Ignored where unsupported (grid-kernel
  // rounds, LOGUP_TILED, sharded, replays, stepwise mode).
  int host_tail = 0;
  bool host_done = false;  // set by run_phase: the finals are in fin_cache
  int forced_shape = -1;
  // LOGUP_TILED host finishing: the eq point u (num_vars, storage form) and
  // the table-side constants K3 = sum_ti B T eq_lo, SMB = sum_ti M B
  const T* lq_u = nullptr;
  T lq_k3, lq_smb;
  // one-launch-per-round mode (profilers): finals are kept here
  bool stepwise = false;
  std::vector<T> fin_cache;
  // ZKL_PROFILE_REPLAY: second run of the phase on recorded challenges
  bool replaying = false;
  const void* replay_words = nullptr;
  // multi-GPU (csrc/shard.cu): the tables are this rank's shard; every
  // round's raw sums are added across the ranks before the host finishes them
  bool sharded = false;
};

// true when the persistent (mailbox) kernels must not be used: ZKL_NO_PERSISTENT,
// CUDA_LAUNCH_BLOCKING=1, or an injected profiler / sanitizer (a replayed
// kernel would spin on a mailbox the host never answers)
bool no_persistent();

// rounds a phase leaves to the host by default (ZKL_HOST_TAIL, default 5;
// 0 = every round on the device)
int host_tail_default();

// Runs every round with the native transcript `tr` (appends each evaluation
// under "sumcheck/eval", draws "sumcheck/round").  Outputs are canonical
// little-endian: rounds (num_vars x (degree+1)), point (num_vars); finals in
// storage form (k values).  Does not synchronise the stream.  With
// finals_out == nullptr it returns right after the last challenge is sent
// (the kernel is still folding); collect the finals with wait_phase_finals.
template <class F>
int run_phase(PhaseArgs<F>& a, HostTranscript& tr, uint8_t* rounds_out, uint8_t* point_out,
              typename F::T* finals_out, cudaStream_t s);
template <class F>
int wait_phase_finals(const PhaseArgs<F>& a, typename F::T* finals_out, cudaStream_t s);

}  // namespace zkl
