// The per-rank 3D-parallel GCN engine (engine.hpp:158-259,
// trainer.hpp:478-627) on one B200. One host thread (or process) drives one
// Engine; collectives go through Comms (NCCL per-axis communicators).
#pragma once

#include <functional>
#include <map>
#include <memory>
#include <vector>

#include "comm.cuh"
#include "elementwise.cuh"
#include "layout.h"
#include "pk_common.cuh"
#include "spmm.cuh"

namespace pk {

// Row-major device matrix with a 16-byte padded leading dimension; the
// padding is zeroed once and never written, so float4 paths, Adam and the
// collectives can run over whole rows.
struct DMat {
  DevBuf<float> buf;
  i64 rows = 0, cols = 0, ld = 0;
  float* p() const { return buf.p; }
  void alloc(i64 r, i64 c, cudaStream_t st);  // zero-filled on `st`
  i64 elems() const { return rows * ld; }
};

struct AdjShard {
  int parity = 0;
  i64 r0 = 0, r1 = 0, c0 = 0, c1 = 0;
  pk_csr_owned a{}, at{};
  SpmmPlan plan_a, plan_at;
  // nnz of each forward row block, per block count (filled on first use)
  std::map<int, std::vector<u64>> block_nnz;
  const std::vector<u64>& blocks_nnz(int blocks, cudaStream_t st);
  u64 nnz_t = 0;
  ~AdjShard();
};

struct PhaseClock {
  // phases: 0 fwd spmm, 1 fwd gemm, 2 backward, 3 optimizer, 4 collectives,
  // 5 backward spmm (reported inside backward_s, as the reference times it)
  struct Mark {
    int phase;
    cudaEvent_t a, b;
  };
  std::vector<cudaEvent_t> pool;
  std::vector<Mark> marks;
  size_t used = 0;
  bool enabled = true;
  cudaEvent_t get();
  // an interval [a, b] of events recorded on any stream
  void add(int phase, cudaEvent_t a, cudaEvent_t b) { marks.push_back({phase, a, b}); }
  cudaEvent_t stamp(cudaStream_t st);
  void begin(int phase, cudaStream_t st);
  void end(cudaStream_t st);
  void collect(double out[6]);  // syncs, sums seconds per phase, resets
  void reset() {                // drop marks nobody will collect
    marks.clear();
    used = 0;
    open_phase = -1;
  }
  ~PhaseClock();
  int open_phase = -1;
  cudaEvent_t open_ev = nullptr;
};

class Engine {
 public:
  explicit Engine(const pk_engine_config& cfg);
  ~Engine();

  void comm_init(const void* uid, int world_size) { comms_.init(grid_, rank_, uid, world_size); }
  void comm_init_local(LocalCluster* cl) { comms_.init_local(grid_, rank_, cl); }
  void comm_init_solo() { comms_.init_solo(grid_, rank_); }
  // A failed rank takes its cluster down (cluster.hpp:240, 434): peers
  // blocked in (or later entering) a collective fail with ClusterAborted.
  void on_failure(const std::string& why);
  void load(const pk_dataset_view& ds, bool host);
  // adopt (optional, [6] like rv.adj): library-allocated blocks the engine
  // takes over instead of copying (entries are zeroed when taken)
  void load_rank(const pk_rank_view& rv, pk_csr_owned* adopt);
  // rank_forward_backward (trainer.hpp:478-527), enqueued without a host
  // wait: the cross-entropy sums travel to pinned host memory on the stream
  // and finish_pass() turns them into loss / accuracy (and the reference's
  // TrainingError checks) once the stream has drained.
  void forward_backward(int epoch);
  // After a stream sync: loss, accuracy, error checks of the last pass (or
  // of the pass whose sums went to `slot`).
  void finish_pass(int epoch, double* loss, double* acc, const double* slot = nullptr);
  void check_after_pass();
  void train_epochs(int first, int count, pk_epoch_metrics* out);
  void optimizer_step();
  void train_epoch(int epoch, pk_epoch_metrics* m);
  void reset_clock() { clock_.reset(); }
  // CommStats (cluster.hpp:35-65) since the load: calls and ring bytes per
  // [axis][op] (op: all_gather, all_reduce, reduce_scatter)
  void comm_stats(u64* calls9, double* bytes9) const;
  // forward_layer / backward_layer (engine.hpp:158-259) one at a time, for
  // callers that drive rank_forward_backward themselves (the C++ shim):
  // begin_pass, forward_layer(0..L-1), loss, backward_layer(L-1..0), then a
  // stream sync and finish_pass give exactly forward_backward.
  void begin_pass();
  void layer_forward(int l, bool fault) { forward_layer(l, fault); }
  void pass_loss() { loss(); }
  void layer_backward(int l) { backward_layer(l); }
  int num_layers() const { return L_; }
  Comms& comms() { return comms_; }
  bool tensor(int which, int layer, pk_tensor_view* out);
  cudaStream_t stream() const { return st_; }

 private:
  void forward_layer(int l, bool fault);
  void backward_layer(int l);
  void forward_layer_tf(int l);
  static int tf_vec();
  static bool tf_pair();
  void backward_layer_tf(int l);
  std::vector<char> tf_;  // transform-first layers (see engine.cu)
  void loss();
  // Forward row blocks of a plane's shard. The result is invariant to the
  // block count (test_engine.cpp:190-213), so `block_count = 0` is free to
  // pick for speed: one launch when no all-reduce follows, a few pipelined
  // blocks otherwise. An explicit block_count is honoured.
  int forward_blocks(i64 rows, const Layout& lay) const;
  // Row-chunked producer -> collective pipeline: produce(r0, r1) runs on the
  // compute stream, reduce(r0, r1) on the comm stream once that chunk is
  // done, so chunk c's collective overlaps chunk c+1's compute. The compute
  // stream waits for the last collective before returning. One chunk when
  // the collective's axis is a singleton (nothing moves).
  template <typename P, typename R>
  void pipelined(i64 rows, int chunks, P&& produce, R&& reduce);
  int comm_chunks(i64 rows, int axis) const;
  void on_comm(const std::function<void(cudaStream_t)>& f);
  // the same without making the compute stream wait: a later on_comm /
  // pipelined reduction's completion covers it (comm stream order)
  void on_comm_nowait(const std::function<void(cudaStream_t)>& f);
  void setup_lsa();
  static constexpr int kFuseSpmm = 1, kFuseGemm = 2;
  LsaGroup* fused(int axis, int producer) const;
  static int fused_mask();
  bool lsa_ready_ = false;

  pk_engine_config cfg_;
  Grid grid_;
  int rank_ = 0;
  Coords c_;
  int L_ = 0;
  std::vector<i64> dims_;
  std::vector<Layout> lays_;
  std::vector<Shapes> shapes_;
  cudaStream_t st_ = nullptr;
  cudaStream_t cs_ = nullptr;  // collectives (overlapped with st_)
  std::vector<cudaEvent_t> sync_ev_;
  size_t sync_used_ = 0;
  cudaEvent_t sync_event();
  Comms comms_;
  CommCounters comm_at_load_;
  // one per (plane, parity) key; keys whose block is the same range of the
  // same variant share one shard (at 1x1x1 planes 0 and 2 are both A_even)
  std::shared_ptr<AdjShard> shards_[6];
  const AdjShard& shard(const Layout& l) const;

  // parameters and optimizer state
  std::vector<DMat> w_, w_m_, w_v_, dw_;
  u64 w_step_ = 0;
  DMat f0_, f0_m_, f0_v_, df0_;
  u64 f0_step_ = 0;
  // activations and workspaces
  DMat f0g_;                           // layer-0 gathered features
  std::vector<DMat> h_, q_, fout_;     // cached H, Q and relu(Q) per layer
  std::vector<char> q_kept_;           // hidden layer's Q materialised last forward
  bool df_masked_ = false;             // df_prev_ already carries relu_backward
  std::vector<DMat> wfull_, dwp_;      // gathered W and dW partial per layer
  DMat dh_, df_, df_prev_;             // backward workspaces (max shapes)
  DMat tfbuf_;                         // transform-first: P forward, dP backward
  DMat logits_, dl_, stage_;
  i64 stage_rows_ = 0;
  DevBuf<u32> labels_;
  DevBuf<u8> mask_;
  u64 mask_count_ = 0;  // global number of masked nodes (the CE count)
  DevBuf<double> sums_;
  double* sums_host_ = nullptr;  // pinned: {loss_sum, count, correct, bad}
  double* sums_dst_ = nullptr;   // where loss() sends them (null: sums_host_)
  double* sums_ring_ = nullptr;  // train_epochs: one pinned slot per epoch
  int sums_ring_n_ = 0;
  CeWorkspace ce_ws_;
  PhaseClock clock_;
  u64 spmm_flops_ = 0, gemm_flops_ = 0;
  double spmm_bytes_ = 0, spmm_cbytes_ = 0;
  bool loaded_ = false;
  // load pieces shared by load() and load_rank()
  template <typename Mark>
  void finish_shard(std::shared_ptr<AdjShard> sh, int plane, int parity, Mark& mark);
  void set_f0(const float* src, i64 ld);
  // FAST plans hold every nonzero: free the shards' CSR columns / values
  // (8 B per nonzero for A and A^T) once the load has drained
  void drop_csr_arrays();
  void alloc_params();
  void set_labels(const u32* labels, const u8* mask, i64 lrows, u64 global_count);
};

}  // namespace pk
