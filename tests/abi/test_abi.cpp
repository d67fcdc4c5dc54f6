// C++ caller test of the drop-in boundary: the reference's own types and
// entry-point signatures (plexuskit headers, /root/reference/proj/include),
// forwarded to libplexus_b200.so by include/plexuskit_b200.hpp, checked
// against the reference's own implementations in the same process.
//
// Cases follow the reference's unit tests (known answers of
// test_kernels.cpp:12-185 and model.hpp's Adam, the engine equivalences of
// test_engine.cpp:145-171 and test_trainer.cpp:256-294) plus the C ABI's
// per-layer and RankCtx-collective entry points against the reference's
// rank_forward_backward / Cluster (cluster.hpp:265-340).
//
// Built by tests/abi/Makefile (build() runs it here, where the reference
// headers are); run on a B200 by tests/test_abi_gpu.py. Exit 0 = all pass.
#include <cmath>
#include <cstdio>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "plexuskit_b200.hpp"

using namespace plexuskit;
namespace b2 = plexuskit::b200;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      ++g_fail;                                                                  \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
    }                                                                            \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static bool same_bits(const DenseMatrix<float>& a, const DenseMatrix<float>& b) {
  return a.same_shape(b) && (a.size() == 0 || std::memcmp(a.data(), b.data(), a.size() * 4) == 0);
}

static double nrel(const DenseMatrix<float>& a, const DenseMatrix<float>& b) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const double d = static_cast<double>(a.data()[i]) - b.data()[i];
    num += d * d;
    den += static_cast<double>(b.data()[i]) * b.data()[i];
  }
  return std::sqrt(num) / (den > 0 ? std::sqrt(den) : 1.0);
}

static DenseMatrix<float> dense(std::size_t r, std::size_t c, std::vector<float> v) {
  return DenseMatrix<float>(r, c, std::move(v));
}

static DenseMatrix<float> random_dense(std::size_t r, std::size_t c, Philox& rng) {
  auto m = DenseMatrix<float>::zeros(r, c);
  for (std::size_t i = 0; i < m.size(); ++i)
    m.data()[i] = static_cast<float>(rng.uniform(-1.0, 1.0));
  return m;
}

static CsrMatrix<float> random_csr(std::size_t r, std::size_t c, double density, Philox& rng) {
  std::vector<u32> ri, ci;
  std::vector<float> v;
  for (std::size_t i = 0; i < r; ++i)
    for (std::size_t j = 0; j < c; ++j)
      if (rng.next_double() < density) {
        ri.push_back(static_cast<u32>(i));
        ci.push_back(static_cast<u32>(j));
        v.push_back(static_cast<float>(rng.uniform(-1.0, 1.0)));
      }
  return CsrMatrix<float>::from_sorted_triplets(r, c, ri, ci, v);
}

// ---------------------------------------------------------------------------

static void kernels() {
  // spmm known answers (test_kernels.cpp:12-41)
  auto eye = CsrMatrix<float>::from_sorted_triplets(3, 3, {0, 1, 2}, {0, 1, 2}, {1, 1, 1});
  auto x = dense(3, 2, {1, 2, 3, 4, 5, 6});
  CHECK(same_bits(b2::spmm(eye, x), x));
  auto swap = CsrMatrix<float>::from_sorted_triplets(2, 2, {0, 1}, {1, 0}, {1, 1});
  CHECK(same_bits(b2::spmm(swap, dense(2, 2, {1, 2, 3, 4})), dense(2, 2, {3, 4, 1, 2})));
  auto full = CsrMatrix<float>::from_sorted_triplets(2, 2, {0, 0, 1, 1}, {0, 1, 0, 1}, {1, 2, 3, 4});
  u64 flops = 0;
  b2::spmm(full, DenseMatrix<float>::zeros(2, 2), &flops);
  CHECK(flops == 16);
  auto bad = CsrMatrix<float>::from_sorted_triplets(2, 3, {0}, {2}, {5});
  CHECK(throws<ContractError>([&] { b2::spmm(bad, DenseMatrix<float>::zeros(2, 2)); }));

  // spmm / spmm_rows bitwise vs the reference on random operands
  Philox rng(11, 0);
  for (int trial = 0; trial < 8; ++trial) {
    const std::size_t m = 1 + rng.randint(300), k = 1 + rng.randint(300),
                      n = 1 + rng.randint(70);
    auto a = random_csr(m, k, 0.1, rng);
    auto f = random_dense(k, n, rng);
    CHECK(same_bits(b2::spmm(a, f), spmm(a, f)));
    const std::size_t r0 = rng.randint(m), r1 = r0 + rng.randint(m - r0 + 1);
    u64 fa = 0, fb = 0;
    CHECK(same_bits(b2::spmm_rows(a, f, r0, r1, &fa), spmm_rows(a, f, r0, r1, &fb)));
    CHECK(fa == fb);
    CHECK(same_bits(b2::transpose(a).to_dense(), a.transpose().to_dense()));
  }

  // gemm known answers (test_kernels.cpp:54-77)
  auto g = b2::gemm(dense(2, 2, {1, 2, 3, 4}), dense(2, 2, {5, 6, 7, 8}), false, false, &flops);
  CHECK(same_bits(g, dense(2, 2, {19, 22, 43, 50})));
  u64 gf = 0;
  b2::gemm(dense(2, 3, {1, 2, 3, 4, 5, 6}), DenseMatrix<float>::zeros(3, 3), false, false, &gf);
  CHECK(gf == 2 * 2 * 3 * 3);
  CHECK(throws<ContractError>([&] { b2::gemm(DenseMatrix<float>::zeros(2, 3), DenseMatrix<float>::zeros(2, 3)); }));
  for (int trial = 0; trial < 6; ++trial) {
    const std::size_t m = 1 + rng.randint(200), k = 1 + rng.randint(200), n = 1 + rng.randint(90);
    auto a = random_dense(m, k, rng), b = random_dense(k, n, rng);
    auto want = gemm(a, b);
    CHECK(same_bits(b2::gemm(a, b), want));                       // PARITY: bitwise
    CHECK(nrel(b2::gemm(a, b, false, false, nullptr, PK_MODE_FAST), want) <= 1e-5);
    CHECK(same_bits(b2::gemm(a.transposed(), b, true, false), want));  // flags == materialised
    CHECK(same_bits(b2::gemm(a, b.transposed(), false, true), want));
  }

  // relu sign cases incl. -0 and exact 0 (test_kernels.cpp:100-126)
  auto q = dense(1, 6, {-2.f, -0.f, 0.f, 1e-38f, 3.f, -1e-30f});
  auto df = dense(1, 6, {1, 2, 3, 4, 5, 6});
  CHECK(same_bits(b2::relu_forward(q), relu_forward(q)));
  CHECK(same_bits(b2::relu_backward(q, df), relu_backward(q, df)));
  auto qr = random_dense(97, 33, rng), dr = random_dense(97, 33, rng);
  CHECK(same_bits(b2::relu_forward(qr), relu_forward(qr)));
  CHECK(same_bits(b2::relu_backward(qr, dr), relu_backward(qr, dr)));

  // cross entropy: ln 2 with dlogits -+0.5 (test_kernels.cpp:128-134),
  // masked rows have zero gradient (179-185), random vs the reference
  auto ce = b2::softmax_cross_entropy_sums(dense(1, 2, {0, 0}), {0}, {1});
  CHECK(std::fabs(ce.loss_sum - std::log(2.0)) <= 1e-6);
  CHECK(ce.count == 1 && ce.correct == 1);
  CHECK(std::fabs(ce.dlogits.at(0, 0) + 0.5f) <= 1e-6f && std::fabs(ce.dlogits.at(0, 1) - 0.5f) <= 1e-6f);
  auto lg = random_dense(120, 17, rng);
  std::vector<u32> lab(120);
  std::vector<u8> msk(120);
  for (int i = 0; i < 120; ++i) lab[i] = static_cast<u32>(rng.randint(17)), msk[i] = i % 3 != 0;
  auto c1 = b2::softmax_cross_entropy_sums(lg, lab, msk);
  auto c0 = softmax_cross_entropy_sums(lg, lab, msk);
  CHECK(c1.count == c0.count && c1.correct == c0.correct);
  CHECK(std::fabs(c1.loss_sum - c0.loss_sum) <= 1e-6 * std::fabs(c0.loss_sum));
  CHECK(nrel(c1.dlogits, c0.dlogits) <= 1e-6);
  bool masked_zero = true;
  for (int i = 0; i < 120; i += 3)
    for (int j = 0; j < 17; ++j) masked_zero &= c1.dlogits.at(i, j) == 0.f;
  CHECK(masked_zero);

  // Adam: five steps bitwise vs the reference (model.hpp:88-111)
  auto p0 = random_dense(31, 9, rng);
  auto p1 = p0;
  auto s0 = AdamState<float>::like(p0), s1 = AdamState<float>::like(p1);
  AdamParams ap;
  for (int s = 0; s < 5; ++s) {
    auto gr = random_dense(31, 9, rng);
    adam_step(p0, gr, s0, ap);
    b2::adam_step(p1, gr, s1, ap);
  }
  CHECK(same_bits(p0, p1) && same_bits(s0.m, s1.m) && same_bits(s0.v, s1.v) && s1.step == 5);
}

// ---------------------------------------------------------------------------

static PreprocessedDataset<float> small_dataset() {
  RmatParams p;
  p.scale = 10;
  p.edges = 9000;
  auto ds = synth_rmat<float>(p, 12, 5, 4);
  return preprocess(ds, 4);
}

static void trainer(const PreprocessedDataset<float>& pre) {
  TrainOptions o;
  o.epochs = 4;
  o.hidden_dims = {16, 16};
  for (GridConfig grid : {GridConfig(1, 1, 1), GridConfig(2, 1, 1), GridConfig(2, 2, 2),
                          GridConfig(1, 4, 2)}) {
    auto want = train_distributed(memory_handle(pre), grid, o);
    b2::DeviceOptions eo;
    eo.mode = PK_MODE_PARITY;
    auto got = b2::train_distributed(memory_handle(pre), grid, o, {}, eo);
    double worst = 0;
    for (int e = 0; e < o.epochs; ++e)
      worst = std::max(worst, std::fabs(got.global[e].loss - want.global[e].loss) / want.global[e].loss);
    CHECK(worst <= 1e-5);
    CHECK(got.global[0].loss == want.global[0].loss ||
          std::fabs(got.global[0].loss - want.global[0].loss) <= 1e-6 * want.global[0].loss);
    for (std::size_t l = 0; l < want.weights.size(); ++l) CHECK(nrel(got.weights[l], want.weights[l]) <= 1e-4);
    CHECK(nrel(got.features, want.features) <= 1e-4);
    CHECK(got.global[0].spmm_flops == want.global[0].spmm_flops);
    CHECK(got.global[0].gemm_flops == want.global[0].gemm_flops);
    CHECK(got.global[0].allreduce_bytes == want.global[0].allreduce_bytes);
    std::printf("train_distributed grid %dx%dx%d: max loss rel %.2e\n", grid.gx(), grid.gy(),
                grid.gz(), worst);
  }
  // a failing loader on one rank: the failure surfaces, the others abort
  DatasetHandle<float> h = memory_handle(pre);
  auto inner = h.loader;
  h.loader = [inner](const GridConfig& g, Coords c, int layers) {
    if (c.x == 1) throw IoError(IoErrorCode::MissingFile, "injected: shard file missing");
    return inner(g, c, layers);
  };
  CHECK(throws<IoError>([&] { b2::train_distributed(h, GridConfig(2, 1, 1), o); }));
}

// The per-layer entry points, composed as rank_forward_backward does, equal
// the one-call pass (1x1x1, logits bit for bit in PARITY).
static void per_layer(const PreprocessedDataset<float>& pre) {
  const auto dims = model_dims(pre.feat_dim, {16, 16}, pre.num_classes);
  auto make = [&](pk_engine** e) {
    pk_engine_config cfg{};
    cfg.gx = cfg.gy = cfg.gz = 1;
    cfg.num_layers = 3;
    for (int i = 0; i < 4; ++i) cfg.dims[i] = static_cast<int64_t>(dims[i]);
    cfg.n = static_cast<int64_t>(pre.n);
    cfg.lr = 1e-2, cfg.beta1 = 0.9, cfg.beta2 = 0.999, cfg.eps = 1e-8;
    cfg.mode = PK_MODE_PARITY;
    cfg.fault_epoch = -1;
    b2::detail::rethrow(pk_engine_create(&cfg, e));
    auto t = slice_rank_tensors(pre, GridConfig(1, 1, 1), Coords{}, 3);
    std::vector<std::unique_ptr<b2::detail::DevCsr>> keep;
    pk_rank_view rv{};
    for (auto [plane, parity] : needed_adjacency_keys(3)) {
      LayerLayout lay{};
      lay.layer = plane % 2 == parity ? plane : plane + 3;
      keep.push_back(std::make_unique<b2::detail::DevCsr>(t.adj.get(lay).a));
      rv.adj[plane * 2 + parity] = keep.back()->view;
    }
    b2::detail::Dev<float> f0(t.f0.data(), t.f0.size());
    b2::detail::Dev<u32> lab(t.labels.data(), t.labels.size());
    b2::detail::Dev<u8> msk(t.mask.data(), t.mask.size());
    rv.f0 = f0.get();
    rv.f0_rows = static_cast<int64_t>(t.f0.rows());
    rv.f0_cols = rv.ld_f0 = static_cast<int64_t>(t.f0.cols());
    rv.labels = lab.get(), rv.mask = msk.get();
    rv.label_rows = static_cast<int64_t>(t.labels.size());
    b2::detail::rethrow(pk_engine_load_rank(*e, &rv));
    cudaDeviceSynchronize();
  };
  auto logits = [&](pk_engine* e) {
    pk_tensor_view v{};
    b2::detail::rethrow(pk_engine_tensor(e, PK_T_FOUT, 0, &v));
    auto out = DenseMatrix<float>::zeros(v.rows, v.cols);
    cudaMemcpy2D(out.data(), v.cols * 4, v.data, v.ld * 4, v.cols * 4, v.rows, cudaMemcpyDeviceToHost);
    return out;
  };
  pk_engine *a = nullptr, *b = nullptr;
  make(&a);
  make(&b);
  double la = 0, aa = 0, lb = 0, ab = 0;
  b2::detail::rethrow(pk_engine_forward_backward(a, 0, &la, &aa));
  b2::detail::rethrow(pk_engine_begin_pass(b));
  for (int l = 0; l < 3; ++l) b2::detail::rethrow(pk_engine_forward_layer(b, l, 0));
  b2::detail::rethrow(pk_engine_loss(b));
  for (int l = 2; l >= 0; --l) b2::detail::rethrow(pk_engine_backward_layer(b, l));
  b2::detail::rethrow(pk_engine_finish_pass(b, 0, &lb, &ab));
  CHECK(la == lb && aa == ab);
  CHECK(same_bits(logits(a), logits(b)));
  // the reference's serial pass: same logits bit for bit
  SerialTrainer<float> ser(pre, [] {
    TrainOptions o;
    o.hidden_dims = {16, 16};
    return o;
  }());
  auto pass = ser.forward_backward(0);
  CHECK(same_bits(logits(b), pass.logits));
  CHECK(std::fabs(lb - pass.loss) <= 1e-6 * pass.loss);
  pk_engine_destroy(a);
  pk_engine_destroy(b);
}

// RankCtx collectives through the C ABI on an in-process 2x2x1 cluster vs the
// reference's Cluster running the same calls (cluster.hpp:265-340).
static void collectives() {
  const GridConfig grid(2, 2, 1);
  const std::size_t rows = 37, cols = 11;
  auto local_of = [&](int r) {
    Philox rng(77, static_cast<u64>(r));
    return random_dense(rows, cols, rng);
  };
  std::vector<DenseMatrix<float>> want_ar(4), want_ag(4), want_agc(4), want_rs(4);
  Cluster ref(grid, ClusterOptions{});
  ref.run([&](RankCtx& ctx) {
    auto l = local_of(ctx.rank());
    want_ar[ctx.rank()] = ctx.all_reduce(l, Axis::X);
    want_ag[ctx.rank()] = ctx.all_gather(l, Axis::Y);
    want_agc[ctx.rank()] = ctx.all_gather(l, Axis::X, ConcatDim::Cols);
    want_rs[ctx.rank()] = ctx.reduce_scatter(l, Axis::Y);
  });
  pk_cluster* cl = nullptr;
  b2::detail::rethrow(pk_cluster_create(2, 2, 1, &cl));
  std::vector<DenseMatrix<float>> ar(4), ag(4), agc(4), rs(4);
  std::vector<std::thread> pool;
  std::mutex mu;
  std::vector<std::string> errs;
  for (int r = 0; r < 4; ++r)
    pool.emplace_back([&, r] {
      try {
        pk_engine_config cfg{};
        cfg.gx = 2, cfg.gy = 2, cfg.gz = 1, cfg.rank = r, cfg.num_layers = 1;
        cfg.dims[0] = 4, cfg.dims[1] = 3, cfg.n = 8, cfg.fault_epoch = -1;
        pk_engine* e = nullptr;
        b2::detail::rethrow(pk_engine_create(&cfg, &e));
        b2::detail::rethrow(pk_engine_comm_init_local(e, cl));
        auto l = local_of(r);
        b2::detail::Dev<float> buf(l.data(), l.size()), keep(l.data(), l.size());
        b2::detail::rethrow(pk_engine_all_reduce_f32(e, 0, buf.get(), rows, cols, cols, nullptr));
        ar[r] = b2::detail::download(buf, rows, cols);
        b2::detail::Dev<float> out(2 * rows * cols);
        b2::detail::rethrow(pk_engine_all_gather_f32(e, 1, 0, keep.get(), cols, out.get(), 2 * rows,
                                                     cols, cols, nullptr));
        ag[r] = b2::detail::download(out, 2 * rows, cols);
        b2::detail::rethrow(pk_engine_all_gather_f32(e, 0, 1, keep.get(), cols, out.get(), rows,
                                                     2 * cols, 2 * cols, nullptr));
        agc[r] = b2::detail::download(out, rows, 2 * cols);
        const int pos = r / 2;  // y coordinate
        const std::size_t own = chunk_size(rows, 2, pos);
        b2::detail::Dev<float> rbuf(l.data(), l.size()), rout(own * cols);
        b2::detail::rethrow(pk_engine_reduce_scatter_f32(e, 1, rbuf.get(), rows, cols, cols,
                                                         rout.get(), nullptr));
        rs[r] = b2::detail::download(rout, own, cols);
        cudaDeviceSynchronize();
        pk_engine_destroy(e);
      } catch (const std::exception& ex) {
        std::lock_guard<std::mutex> lk(mu);
        errs.push_back(ex.what());
      }
    });
  for (auto& t : pool) t.join();
  pk_cluster_destroy(cl);
  CHECK(errs.empty());
  for (auto& e : errs) std::fprintf(stderr, "collectives: %s\n", e.c_str());
  for (int r = 0; r < 4 && errs.empty(); ++r) {
    CHECK(same_bits(ar[r], want_ar[r]));
    CHECK(same_bits(ag[r], want_ag[r]));
    CHECK(same_bits(agc[r], want_agc[r]));
    CHECK(same_bits(rs[r], want_rs[r]));
  }
}

int main() {
  int dev = 0;
  if (cudaGetDeviceCount(&dev) != cudaSuccess || dev == 0) {
    std::fprintf(stderr, "test_abi: no CUDA device\n");
    return 2;
  }
  auto run = [](const char* name, const std::function<void()>& f) {
    const int before = g_fail;
    try {
      f();
    } catch (const std::exception& e) {
      ++g_fail;
      std::fprintf(stderr, "FAIL %s: exception %s\n", name, e.what());
    }
    std::printf("%-12s %s\n", name, g_fail == before ? "ok" : "FAILED");
  };
  run("kernels", kernels);
  const auto pre = small_dataset();
  run("per_layer", [&] { per_layer(pre); });
  run("trainer", [&] { trainer(pre); });
  run("collectives", collectives);
  std::printf("test_abi: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
