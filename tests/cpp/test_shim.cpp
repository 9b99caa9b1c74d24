// Drop-in proof: reference test bodies (proj/tests/test_plan.cpp,
// test_layout.cpp) compiled against the dfftb C++ shim (include/dfftb/dfft.hpp)
// instead of the reference headers.  `--host` runs only the plan/layout
// checks (no GPU needed); without it the single-rank execute checks run too.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>

#include "dfftb/dfft.hpp"
#include "dfftb/tensor_file.hpp"

using namespace dfftb::dfft;
using cxd = cx<double>;

static int g_fail = 0, g_pass = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (c) ++g_pass;                                                  \
    else {                                                            \
      ++g_fail;                                                       \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);       \
    }                                                                 \
  } while (0)
#define CHECK_THROWS_WITH(expr, text)                                 \
  do {                                                                \
    bool thrown_ = false;                                             \
    try {                                                             \
      (void)(expr);                                                   \
    } catch (const Error& e_) {                                       \
      thrown_ = std::string(e_.what()).find(text) != std::string::npos; \
      if (!thrown_) std::printf("  got: %s\n", e_.what());           \
    }                                                                 \
    CHECK(thrown_);                                                   \
  } while (0)

static double unit_from_hash(std::uint64_t x) {  // test_plan.cpp:19-25
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return static_cast<double>(x >> 11) * 0x1.0p-52 - 1.0;
}

static void host_tests() {
  // test_plan.cpp:136-150 — slab stage shape and SlabTooManyRanks
  auto slab = plan_slab<double>(GlobalDims{4, 4, 4}, 2, TransformKind::C2C, Direction::Forward);
  CHECK(slab.fft_stage_count() == 3);
  CHECK(slab.transpose_stage_count() == 1);
  CHECK(slab.signature() == "F2;F1;T0x;L;F0;");
  CHECK_THROWS_WITH(plan_slab<double>(GlobalDims{4, 6, 8}, 5, TransformKind::C2C, Direction::Forward),
                    "SlabTooManyRanks");
  // test_plan.cpp:172-190 — R2C hat metadata, stage counts
  auto r2c = plan_pencil<double>(GlobalDims{256, 512, 1024}, ProcessGrid{4, 2}, TransformKind::R2C,
                                 Direction::Forward);
  CHECK(r2c.output.dims == (GlobalDims{256, 512, 513}));
  CHECK(r2c.output.element == ElementKind::Complex);
  CHECK(r2c.output.all_hatted());
  for (Direction dir : {Direction::Forward, Direction::Backward}) {
    auto p = plan_pencil<double>(GlobalDims{8, 8, 8}, ProcessGrid{2, 2}, TransformKind::C2C, dir);
    CHECK(p.fft_stage_count() == 3);
    CHECK(p.transpose_stage_count() == 2);
  }
  // test_plan.cpp:192-209 — layout contract + spot index
  auto lp = plan_pencil<double>(GlobalDims{8, 4, 6}, ProcessGrid{2, 2}, TransformKind::R2C,
                                Direction::Forward);
  const std::int64_t coord[3] = {5, 1, 2};
  auto [rank, offset] = local_index(lp.output, std::span<const std::int64_t>(coord, 3));
  CHECK(rank == 1);  // grid coords (0, 1)
  CHECK(offset == (5 * 2 + 1) * 2 + (2 - 2));
  // test_plan.cpp:225-250 — general plans
  for (Direction dir : {Direction::Forward, Direction::Backward}) {
    auto g = plan_general<double>(GlobalDims{8, 8, 8}, ProcessGrid{2, 2}, TransformKind::C2C, dir);
    auto p = plan_pencil<double>(GlobalDims{8, 8, 8}, ProcessGrid{2, 2}, TransformKind::C2C, dir);
    CHECK(g.signature() == p.signature());
    CHECK(g.input == p.input);
    CHECK(g.output == p.output);
  }
  CHECK_THROWS_WITH(plan_general<double>(GlobalDims{8, 8, 8}, ProcessGrid{2}, TransformKind::C2C,
                                         Direction::Forward),
                    "GridMismatch");
  CHECK_THROWS_WITH(plan_general<double>(GlobalDims{2, 2, 2}, ProcessGrid{2, 4}, TransformKind::C2C,
                                         Direction::Forward),
                    "RankTooLow");
  // test_layout.cpp block_map examples
  auto bm = block_map(10, 4);
  CHECK(bm.counts == (std::vector<std::int64_t>{3, 3, 3, 1}));
  CHECK(bm.offsets == (std::vector<std::int64_t>{0, 3, 6, 9}));
  auto bm2 = block_map(5, 4);
  CHECK(bm2.counts == (std::vector<std::int64_t>{2, 2, 1, 0}));
  CHECK(hat_dims(GlobalDims{256, 512, 1024}, TransformKind::R2C) == (GlobalDims{256, 512, 513}));
}

static void gpu_tests() {
  LocalComm comm;
  {  // test_plan.cpp:153-170 — delta at the origin transforms to all ones (1 rank)
    auto plan = plan_pencil<double>(GlobalDims{8, 8, 8}, ProcessGrid{1, 1}, TransformKind::C2C,
                                    Direction::Forward);
    auto ctx = make_context(plan, comm);
    auto x = DistTensor<double>::zeros(plan.input, 0);
    fill_from_global(x, [](std::int64_t flat, std::span<const std::int64_t>) {
      return flat == 0 ? cxd(1, 0) : cxd(0, 0);
    });
    auto y = execute(plan, x, ctx);
    double err = 0;
    for (const auto& v : y.cplx) err = std::max(err, std::abs(v - cxd(1, 0)));
    CHECK(err < 1e-12);
    // device-resident chain: no host mirror until asked for
    ctx.mirror_to_host = false;
    auto yd = execute(plan, x, ctx);
    CHECK(yd.cplx.empty() && yd.local_size() == 512);
    auto yd2 = execute_device(plan, x, ctx);
    yd2.to_host();
    CHECK(yd2.cplx.size() == 512 && yd2.cplx[17] == y.cplx[17]);
  }
  {  // test_plan.cpp:367-390 — R2C/C2R round trip is the identity
    const GlobalDims dims{8, 8, 8};
    auto fwd = plan_pencil<double>(dims, ProcessGrid{1, 1}, TransformKind::R2C, Direction::Forward);
    auto bwd = plan_pencil<double>(dims, ProcessGrid{1, 1}, TransformKind::C2R, Direction::Backward);
    auto ctx = make_context(fwd, comm);
    auto x = DistTensor<double>::zeros(fwd.input, 0);
    fill_from_global(x, [](std::int64_t flat, std::span<const std::int64_t>) {
      return cxd(unit_from_hash(3 * flat + 1), 0.0);
    });
    auto back = execute_r2c_c2r_roundtrip(fwd, bwd, x, ctx);
    double num = 0, den = 0;
    for (std::size_t i = 0; i < back.real.size(); ++i) {
      num += (back.real[i] - x.real[i]) * (back.real[i] - x.real[i]);
      den += x.real[i] * x.real[i];
    }
    CHECK(std::sqrt(num / den) < 1e-12);
  }
  {  // test_plan.cpp:392-408 — corrupted spectrum fails the Hermitian check
    auto bwd = plan_pencil<double>(GlobalDims{4, 4, 4}, ProcessGrid{1, 1}, TransformKind::C2R,
                                   Direction::Backward);
    auto ctx = make_context(bwd, comm);
    auto spec = DistTensor<double>::zeros(bwd.input, 0);
    spec.cplx[0] = cxd(1.0, 0.7);
    spec.from_host();
    CHECK_THROWS_WITH(execute(bwd, spec, ctx), "NonHermitian");
  }
  {  // test_plan.cpp:307-321 — wrong input layout is rejected
    auto plan = plan_pencil<double>(GlobalDims{4, 4, 4}, ProcessGrid{1, 1}, TransformKind::C2C,
                                    Direction::Forward);
    auto ctx = make_context(plan, comm);
    auto x = DistTensor<double>::zeros(plan.output, 0);
    CHECK_THROWS_WITH(execute(plan, x, ctx), "LayoutMismatch");
  }
  {  // test_plan.cpp:323-341 — finiteness validation is opt-in
    PlanOptions options;
    options.validate_finite = true;
    auto plan = plan_pencil<double>(GlobalDims{2, 2, 2}, ProcessGrid{1, 1}, TransformKind::C2C,
                                    Direction::Forward, options);
    auto ctx = make_context(plan, comm);
    auto x = DistTensor<double>::zeros(plan.input, 0);
    x.cplx[3] = cxd(std::nan(""), 0.0);
    x.from_host();
    CHECK_THROWS_WITH(execute(plan, x, ctx), "non-finite");
  }
  {  // test_plan.cpp:465-483 — single precision plan within tolerance
    auto plan = plan_general<float>(GlobalDims{4, 4, 4}, ProcessGrid{1, 1}, TransformKind::C2C,
                                    Direction::Forward);
    auto ctx = make_context(plan, comm);
    auto x = DistTensor<float>::zeros(plan.input, 0);
    fill_from_global(x, [](std::int64_t flat, std::span<const std::int64_t>) {
      return cx<float>(static_cast<float>(unit_from_hash(flat)), 0.0f);
    });
    auto y = execute(plan, x, ctx);
    // direct 3-D DFT in double
    double num = 0, den = 0;
    for (int k0 = 0; k0 < 4; ++k0)
      for (int k1 = 0; k1 < 4; ++k1)
        for (int k2 = 0; k2 < 4; ++k2) {
          cxd acc(0, 0);
          for (int j = 0; j < 64; ++j) {
            const int j0 = j / 16, j1 = (j / 4) % 4, j2 = j % 4;
            const double ph = -2.0 * M_PI * (k0 * j0 + k1 * j1 + k2 * j2) / 4.0;
            acc += cxd(static_cast<float>(unit_from_hash(j)), 0.0) * std::polar(1.0, ph);
          }
          const cxd got(y.cplx[(k0 * 4 + k1) * 4 + k2]);
          num += std::norm(got - acc);
          den += std::norm(acc);
        }
    CHECK(std::sqrt(num / den) < 1e-4);
  }
}

// spectral.hpp mirror (test_spectral.cpp:79-100, 274-292): d/dz sin(2z) =
// 2 cos(2z) for real and complex fields; div(grad f) == lap f; inverse
// Laplacian round trip; NonZeroMean
static void spectral_tests() {
  LocalComm comm;
  const GlobalDims dims{8, 8, 16};
  auto c = make_spectral_context<double>(comm, dims, ProcessGrid{1, 1});
  CHECK(c.k_c2c.axis_k[0].size() == 8 && c.k_r2c.axis_k[2].size() == 9);
  CHECK(c.k_c2c.axis_k_deriv[2][8] == 0.0);  // Nyquist zeroed for derivatives
  const double tp = 2.0 * M_PI;
  auto field = [&](auto fn, bool real) {
    auto x = DistTensor<double>::zeros(real ? c.fwd_r2c.input : c.fwd_c2c.input, 0);
    fill_from_global(x, [&](std::int64_t, std::span<const std::int64_t> g) {
      const double z = tp * g[0] / 8, y = tp * g[1] / 8, w = tp * g[2] / 16;
      return cxd(fn(z, y, w), 0.0);
    });
    return x;
  };
  for (bool real : {true, false}) {
    auto x = field([](double, double, double w) { return std::sin(2 * w); }, real);
    auto g = gradient(c, x);
    g[2].to_host();
    double err = 0;
    for (int i = 0; i < 8 * 8 * 16; ++i) {
      const double w = tp * (i % 16) / 16;
      const double got = real ? g[2].real[i] : g[2].cplx[i].real();
      err = std::max(err, std::fabs(got - 2 * std::cos(2 * w)));
    }
    CHECK(err < 1e-10);
  }
  auto f = field([](double z, double y, double w) { return std::sin(3 * z) * std::cos(2 * y) + std::sin(5 * w); },
                 true);
  auto dg = divergence(c, gradient(c, f));
  auto lp = laplacian(c, f);
  dg.to_host();
  lp.to_host();
  double e = 0, m = 0;
  for (std::size_t i = 0; i < lp.real.size(); ++i) {
    e = std::max(e, std::fabs(dg.real[i] - lp.real[i]));
    m = std::max(m, std::fabs(lp.real[i]));
  }
  CHECK(e < 1e-9 * m);
  auto u = inverse_laplacian(c, lp);  // zero-mean field: recovers f
  u.to_host();
  f.to_host();
  double eu = 0;
  for (std::size_t i = 0; i < f.real.size(); ++i) eu = std::max(eu, std::fabs(u.real[i] - f.real[i]));
  CHECK(eu < 1e-10);
  auto ones = field([](double, double, double) { return 1.0; }, true);
  CHECK_THROWS_WITH(inverse_laplacian(c, ones), "NonZeroMean");
}

// tensor_file.hpp mirror: DTNS write/read round trip through a layout, the
// file format (golden header bytes) and the error codes
static void tensor_file_tests() {
  LocalComm comm;
  auto plan = plan_pencil<double>(GlobalDims{4, 3, 5}, ProcessGrid{1, 1}, TransformKind::R2C, Direction::Forward);
  auto x = DistTensor<double>::zeros(plan.input, 0);
  fill_from_global(x, [](std::int64_t flat, std::span<const std::int64_t>) { return cxd(0.5 * flat - 3.0, 0); });
  const std::string path = "/tmp/dfftb_shim_tensor.dtns";
  write_tensor(comm, x, path);
  const TensorFile f = read_tensor_file(path);
  CHECK(f.dims == (GlobalDims{4, 3, 5}) && f.element == TensorElement::Real64 && f.payload.size() == 60 * 8);
  auto y = read_tensor<double>(comm, plan.input, path);
  y.to_host();
  bool same = y.real.size() == 60;
  for (int i = 0; same && i < 60; ++i) same = y.real[i] == 0.5 * i - 3.0;
  CHECK(same);
  // a real file feeding a complex layout is promoted
  auto c2c = plan_pencil<double>(GlobalDims{4, 3, 5}, ProcessGrid{1, 1}, TransformKind::C2C, Direction::Forward);
  auto z = read_tensor<double>(comm, c2c.input, path);
  z.to_host();
  CHECK(z.cplx.size() == 60 && z.cplx[7] == cxd(0.5, 0.0));
  // header layout: "DTNS", u32 1, u8 kind, u32 axes, u64 dims
  std::ifstream in(path, std::ios::binary);
  unsigned char h[13];
  in.read(reinterpret_cast<char*>(h), 13);
  CHECK(std::memcmp(h, "DTNS", 4) == 0 && h[4] == 1 && h[8] == 0 && h[9] == 3);
  auto other = plan_pencil<double>(GlobalDims{4, 3, 6}, ProcessGrid{1, 1}, TransformKind::C2C, Direction::Forward);
  CHECK_THROWS_WITH(read_tensor<double>(comm, other.input, path), "DimMismatch");
  std::ofstream(path, std::ios::binary) << "NOPE....";
  CHECK_THROWS_WITH(read_tensor_file(path), "TruncatedFile");
  std::ofstream(path, std::ios::binary) << "NOPE0000000000000";
  CHECK_THROWS_WITH(read_tensor_file(path), "BadMagic");
}

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::strcmp(argv[1], "--host") == 0;
  try {
    host_tests();
    if (!host_only) {
      tensor_file_tests();
      gpu_tests();
      spectral_tests();
    }
  } catch (const std::exception& e) {
    std::printf("uncaught: %s\n", e.what());
    ++g_fail;
  }
  std::printf("%d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
