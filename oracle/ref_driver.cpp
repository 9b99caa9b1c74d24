// Test infrastructure, NOT product code.
//
// Driver for the UNMODIFIED reference implementation (the dfft C++20 artifact
// under /root/reference/proj).  It is compiled against the reference headers
// where they lie (-I/root/reference/proj/include) and linked with the
// reference's own transport/simd sources by oracle/Makefile; the binary goes to
// oracle/_ref/ (git-ignored).  It is used for three things only:
//   * generating golden fixtures for tests/golden/ (make_golden.py),
//   * pinning the C restatement in oracle/dfft_oracle.c,
//   * the CPU baseline leg of bench.py (`cpu_baseline.kind = "reference"`).
//
// It calls the reference through its public API exactly like the reference's
// own bench does (proj/src/bench.cpp:261-362): plan_slab / plan_pencil
// (plan.hpp:242-354) -> make_context (plan.hpp:365) -> execute (plan.hpp:463),
// ranks are threads of transport::spawn_world (transport.hpp:239), each timed
// execute is preceded by transport::barrier and reduced max-over-ranks.
//
// Input field: bench.cpp:22-28,132-136 seeded_value(seed, flat, complex).
//
// Usage:
//   dfft_ref --dims 64,64,64 --decomp slab|pencil --grid 1|2,4
//            --kind c2c|r2c --prec f64|f32 [--seed 1] [--warmup 1] [--reps 3]
//            [--dump PREFIX] [--no-normalize] [--spectral]
// Prints one JSON line.  With --dump writes PREFIX.in.bin (global input, real
// for r2c / interleaved complex for c2c), PREFIX.fwd.bin (global forward
// spectrum, interleaved complex, frequency layout gathered in xyz order) and
// PREFIX.rt.bin (global backward(forward(x)) in the input's element kind).

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "dfft/plan.hpp"
#include "dfft/spectral.hpp"

using namespace dfft;

namespace {

double unit_from_hash(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return static_cast<double>(x >> 11) * 0x1.0p-52 - 1.0;
}

std::vector<std::int64_t> parse_list(const char* s) {
  std::vector<std::int64_t> v;
  std::string str(s);
  std::size_t pos = 0;
  while (pos <= str.size()) {
    std::size_t comma = str.find(',', pos);
    if (comma == std::string::npos) comma = str.size();
    v.push_back(std::stoll(str.substr(pos, comma - pos)));
    pos = comma + 1;
  }
  return v;
}

struct Args {
  std::vector<std::int64_t> dims{64, 64, 64};
  std::vector<std::int64_t> grid{1};
  bool pencil = false;
  bool general = false;
  bool r2c = false;
  bool f32 = false;
  std::uint64_t seed = 1;
  int warmup = 1;
  int reps = 3;
  bool normalize = true;
  bool spectral = false;
  std::string dump;
};

template <class T>
Plan<T> make_plan(const Args& a, TransformKind kind, Direction dir) {
  PlanOptions opt;
  opt.normalize = a.normalize;
  GlobalDims dims(a.dims);
  if (a.pencil) {
    std::vector<int> g(a.grid.begin(), a.grid.end());
    return plan_pencil<T>(dims, ProcessGrid(g), kind, dir, opt);
  }
  if (a.general) {
    std::vector<int> g(a.grid.begin(), a.grid.end());
    return plan_general<T>(dims, ProcessGrid(g), kind, dir, opt);
  }
  return plan_slab<T>(dims, static_cast<int>(a.grid[0]), kind, dir, opt);
}

void write_file(const std::string& path, const void* data, std::size_t bytes) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (f == nullptr) {
    std::fprintf(stderr, "cannot write %s\n", path.c_str());
    std::exit(1);
  }
  std::fwrite(data, 1, bytes, f);
  std::fclose(f);
}

template <class T>
int run(const Args& a) {
  const TransformKind fk = a.r2c ? TransformKind::R2C : TransformKind::C2C;
  const TransformKind bk = a.r2c ? TransformKind::C2R : TransformKind::C2C;
  int P = 1;
  for (auto g : a.grid) P *= static_cast<int>(g);

  std::vector<double> fwd_t, inv_t;
  std::vector<TimingBreakdown> fwd_tb, inv_tb;
  double rt_err = 0.0;
  std::vector<T> in_real, rt_real;
  std::vector<cx<T>> in_cplx, fwd_full, rt_cplx;

  transport::spawn_world(P, [&](transport::Comm& comm) {
    auto fwd = make_plan<T>(a, fk, Direction::Forward);
    auto bwd = make_plan<T>(a, bk, Direction::Backward);
    auto ctx = make_context(fwd, comm);
    auto x = DistTensor<T>::zeros(fwd.input, comm.rank());
    fill_from_global(x, [&](std::int64_t flat, std::span<const std::int64_t>) {
      const double re = unit_from_hash(a.seed * 0x10001 + 2 * flat);
      const double im = a.r2c ? 0.0 : unit_from_hash(a.seed * 0x10001 + 2 * flat + 1);
      return cx<T>(static_cast<T>(re), static_cast<T>(im));
    });
    for (int w = 0; w < a.warmup; ++w) {
      auto y = execute(fwd, x, ctx);
      (void)execute(bwd, y, ctx);
    }
    DistTensor<T> y, z;
    for (int r = 0; r < a.reps; ++r) {
      double secs[2];
      TimingBreakdown tbs[2];
      transport::barrier(comm);
      auto t0 = std::chrono::steady_clock::now();
      y = execute(fwd, x, ctx, &tbs[0]);
      secs[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      transport::barrier(comm);
      t0 = std::chrono::steady_clock::now();
      z = execute(bwd, y, ctx, &tbs[1]);
      secs[1] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      double raw[14];
      raw[0] = secs[0];
      raw[1] = secs[1];
      for (int d = 0; d < 2; ++d) {
        raw[2 + 6 * d + 0] = tbs[d].local_fft;
        raw[2 + 6 * d + 1] = tbs[d].pack;
        raw[2 + 6 * d + 2] = tbs[d].unpack;
        raw[2 + 6 * d + 3] = tbs[d].staging_copy;
        raw[2 + 6 * d + 4] = tbs[d].wire_comm;
        raw[2 + 6 * d + 5] = tbs[d].total;
      }
      auto parts = transport::gather_bytes(
          comm, bytes::from_values(std::span<const double>(raw, 14)));
      if (comm.rank() == 0) {
        double mx[14] = {0};
        for (const auto& p : parts) {
          auto v = bytes::to_values<double>(p);
          for (int i = 0; i < 14; ++i) mx[i] = std::max(mx[i], v[i]);
        }
        fwd_t.push_back(mx[0]);
        inv_t.push_back(mx[1]);
        fwd_tb.push_back({mx[2], mx[3], mx[4], mx[5], mx[6], mx[7]});
        inv_tb.push_back({mx[8], mx[9], mx[10], mx[11], mx[12], mx[13]});
      }
    }
    // round-trip error (rel L2, reduced over ranks)
    double num = 0, den = 0;
    if (a.r2c) {
      for (std::size_t i = 0; i < x.real.size(); ++i) {
        const double d = double(z.real[i]) - double(x.real[i]);
        num += d * d;
        den += double(x.real[i]) * double(x.real[i]);
      }
    } else {
      for (std::size_t i = 0; i < x.cplx.size(); ++i) {
        num += std::norm(cx<double>(z.cplx[i]) - cx<double>(x.cplx[i]));
        den += std::norm(cx<double>(x.cplx[i]));
      }
    }
    double nd[2] = {num, den};
    auto parts = transport::gather_bytes(
        comm, bytes::from_values(std::span<const double>(nd, 2)));
    if (comm.rank() == 0) {
      double n = 0, d = 0;
      for (const auto& p : parts) {
        auto v = bytes::to_values<double>(p);
        n += v[0];
        d += v[1];
      }
      rt_err = d == 0 ? std::sqrt(n) : std::sqrt(n / d);
    }
    if (!a.dump.empty()) {
      if (a.r2c) {
        auto gi = gather_global_real(comm, x);
        auto gr = gather_global_real(comm, z);
        if (comm.rank() == 0) {
          in_real = std::move(gi);
          rt_real = std::move(gr);
        }
      } else {
        auto gi = gather_global_complex(comm, x);
        auto gr = gather_global_complex(comm, z);
        if (comm.rank() == 0) {
          in_cplx = std::move(gi);
          rt_cplx = std::move(gr);
        }
      }
      auto gf = gather_global_complex(comm, y);
      if (comm.rank() == 0) fwd_full = std::move(gf);
    }
  });

  if (!a.dump.empty()) {
    if (a.r2c) {
      write_file(a.dump + ".in.bin", in_real.data(), in_real.size() * sizeof(T));
      write_file(a.dump + ".rt.bin", rt_real.data(), rt_real.size() * sizeof(T));
    } else {
      write_file(a.dump + ".in.bin", in_cplx.data(), in_cplx.size() * sizeof(cx<T>));
      write_file(a.dump + ".rt.bin", rt_cplx.data(), rt_cplx.size() * sizeof(cx<T>));
    }
    write_file(a.dump + ".fwd.bin", fwd_full.data(), fwd_full.size() * sizeof(cx<T>));
  }

  auto minmed = [](std::vector<double> v, double* mn, double* med) {
    std::sort(v.begin(), v.end());
    *mn = v.front();
    *med = v[(v.size() - 1) / 2];
  };
  std::vector<double> tot(fwd_t.size());
  for (std::size_t i = 0; i < tot.size(); ++i) tot[i] = fwd_t[i] + inv_t[i];
  double fmn, fmed, imn, imed, tmn, tmed;
  minmed(fwd_t, &fmn, &fmed);
  minmed(inv_t, &imn, &imed);
  minmed(tot, &tmn, &tmed);
  std::uint64_t n = 1;
  for (auto d : a.dims) n *= static_cast<std::uint64_t>(d);
  const double flops = 5.0 * double(n) * std::log2(double(n));  // bench.cpp:32-41
  std::printf(
      "{\"impl\":\"reference\",\"ranks\":%d,\"fwd_min_s\":%.9g,\"fwd_median_s\":%.9g,"
      "\"inv_min_s\":%.9g,\"inv_median_s\":%.9g,\"fwdinv_min_s\":%.9g,"
      "\"fwdinv_median_s\":%.9g,\"flops_fwdinv\":%.17g,\"gflops_fwdinv\":%.9g,"
      "\"roundtrip_rel_l2\":%.6e,\"fwd_local_fft_s\":%.9g,\"fwd_pack_s\":%.9g,"
      "\"fwd_unpack_s\":%.9g,\"fwd_wire_s\":%.9g}\n",
      P, fmn, fmed, imn, imed, tmn, tmed, 2 * flops, 2 * flops / tmn / 1e9, rt_err,
      fwd_tb[0].local_fft, fwd_tb[0].pack, fwd_tb[0].unpack, fwd_tb[0].wire_comm);
  return 0;
}

// --spectral: the reference's spectral operators (spectral.hpp:131-309) on
// the seeded field through make_spectral_context (pencil / general plans over
// --grid): PREFIX.in.bin, PREFIX.d<a>.bin (derivative along axis a),
// PREFIX.lap.bin (laplacian), PREFIX.ilap.bin (inverse_laplacian of the
// laplacian: a zero-mean input), PREFIX.div.bin (divergence of the gradient),
// all global arrays in the input's element kind.
template <class T>
int run_spectral(const Args& a) {
  int P = 1;
  for (auto g : a.grid) P *= static_cast<int>(g);
  std::vector<std::vector<T>> out_real;
  std::vector<std::vector<cx<T>>> out_cplx;
  std::vector<std::string> names;
  transport::spawn_world(P, [&](transport::Comm& comm) {
    std::vector<int> g(a.grid.begin(), a.grid.end());
    auto sc = make_spectral_context<T>(comm, GlobalDims(a.dims), ProcessGrid(g));
    const auto& in_dist = a.r2c ? sc.fwd_r2c.input : sc.fwd_c2c.input;
    auto x = DistTensor<T>::zeros(in_dist, comm.rank());
    fill_from_global(x, [&](std::int64_t flat, std::span<const std::int64_t>) {
      const double re = unit_from_hash(a.seed * 0x10001 + 2 * flat);
      const double im = a.r2c ? 0.0 : unit_from_hash(a.seed * 0x10001 + 2 * flat + 1);
      return cx<T>(static_cast<T>(re), static_cast<T>(im));
    });
    std::vector<std::pair<std::string, DistTensor<T>>> res;
    res.emplace_back("in", x);
    std::vector<DistTensor<T>> grad;
    for (std::size_t ax = 0; ax < a.dims.size(); ++ax) {
      grad.push_back(derivative(sc, x, static_cast<int>(ax)));
      res.emplace_back("d" + std::to_string(ax), grad.back());
    }
    auto lap = laplacian(sc, x);
    res.emplace_back("lap", lap);
    // fp32: the laplacian's mean is zero only to fp32 rounding, above the
    // reference's 1e-12 N zero-mean bound (NonZeroMean): no ilap golden
    if constexpr (std::is_same_v<T, double>) res.emplace_back("ilap", inverse_laplacian(sc, lap));
    res.emplace_back("div", divergence(sc, grad));
    for (auto& [name, t] : res) {
      if (a.r2c) {
        auto gl = gather_global_real(comm, t);
        if (comm.rank() == 0) {
          names.push_back(name);
          out_real.push_back(std::move(gl));
        }
      } else {
        auto gl = gather_global_complex(comm, t);
        if (comm.rank() == 0) {
          names.push_back(name);
          out_cplx.push_back(std::move(gl));
        }
      }
    }
  });
  for (std::size_t i = 0; i < names.size(); ++i) {
    const std::string path = a.dump + "." + names[i] + ".bin";
    if (a.r2c) write_file(path, out_real[i].data(), out_real[i].size() * sizeof(T));
    else write_file(path, out_cplx[i].data(), out_cplx[i].size() * sizeof(cx<T>));
  }
  std::printf("{\"impl\":\"reference\",\"spectral\":%zu}\n", names.size());
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  for (int i = 1; i < argc; ++i) {
    std::string k = argv[i];
    auto next = [&]() -> const char* {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "missing value for %s\n", k.c_str());
        std::exit(2);
      }
      return argv[++i];
    };
    if (k == "--dims") a.dims = parse_list(next());
    else if (k == "--grid") a.grid = parse_list(next());
    else if (k == "--decomp") {
      const std::string d = next();
      a.pencil = d == "pencil";
      a.general = d == "general";
    }
    else if (k == "--kind") a.r2c = std::string(next()) == "r2c";
    else if (k == "--prec") a.f32 = std::string(next()) == "f32";
    else if (k == "--seed") a.seed = std::stoull(next());
    else if (k == "--warmup") a.warmup = std::atoi(next());
    else if (k == "--reps") a.reps = std::atoi(next());
    else if (k == "--dump") a.dump = next();
    else if (k == "--no-normalize") a.normalize = false;
    else if (k == "--spectral") a.spectral = true;
    else {
      std::fprintf(stderr, "unknown flag %s\n", k.c_str());
      return 2;
    }
  }
  try {
    if (a.spectral) return a.f32 ? run_spectral<float>(a) : run_spectral<double>(a);
    return a.f32 ? run<float>(a) : run<double>(a);
  } catch (const std::exception& e) {
    std::printf("{\"impl\":\"reference\",\"error\":\"%s\"}\n", e.what());
    return 1;
  }
}
