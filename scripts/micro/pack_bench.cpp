// pack_bench.cpp -- host throughput of packing the reference's FP64 genome
// rows into the compact transfer rows (what fnb_evaluate would send over PCIe
// instead of the raw rows), against a plain memcpy of the raw rows.
//   g++ -O3 -mavx2 -mfma -pthread -o scripts/micro/pack_bench scripts/micro/pack_bench.cpp
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <random>
#include <thread>
#include <vector>

struct PNode { int32_t key; float bias, resp; uint8_t act, agg, flags, pad; };
struct PConn { int32_t in, out; float w; };

static inline int32_t dev_int(double x) {  // cvt.rzi.s32.f64: NaN -> 0, saturating
  if (x != x) return 0;
  if (x >= 2147483647.0) return 2147483647;
  if (x <= -2147483648.0) return -2147483647 - 1;
  return int32_t(x);
}

static bool pack_rows(const double* n, const double* c, size_t gN, size_t gC, PNode* pn, PConn* pc, uint8_t* cf) {
  bool ok = true;
  for (size_t r = 0; r < gN; ++r) {
    const double* x = n + 5 * r;
    PNode o{};
    const bool ne = !std::isnan(x[0]);
    o.key = dev_int(x[0]);
    o.bias = float(x[1]);
    o.resp = float(x[2]);
    const int32_t ag = dev_int(x[3]), ac = dev_int(x[4]);
    ok &= !ne || (uint32_t(ag) < 256u && uint32_t(ac) < 256u);
    o.agg = uint8_t(ag);
    o.act = uint8_t(ac);
    o.flags = ne;
    pn[r] = o;
  }
  for (size_t r = 0; r < gC; ++r) {
    const double* x = c + 4 * r;
    PConn o;
    o.in = dev_int(x[0]);
    o.out = dev_int(x[1]);
    o.w = float(x[3]);
    pc[r] = o;
    cf[r] = uint8_t((!std::isnan(x[0])) | ((x[2] == 1.0) << 1));
  }
  return ok;
}

int main(int argc, char** argv) {
  const size_t P = 10000, N = 64, C = 256;
  std::vector<double> nodes(P * N * 5), conns(P * C * 4);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  for (size_t i = 0; i < P * N; ++i) {
    double* x = &nodes[i * 5];
    const bool e = (i % N) >= 48;
    x[0] = e ? NAN : double(i % N);
    x[1] = e ? NAN : nd(rng);
    x[2] = e ? NAN : 1.0;
    x[3] = e ? NAN : 0.0;
    x[4] = e ? NAN : 1.0;
  }
  for (size_t i = 0; i < P * C; ++i) {
    double* x = &conns[i * 4];
    const bool e = (i % C) >= 192;
    x[0] = e ? NAN : double(i % 48);
    x[1] = e ? NAN : double((i * 7) % 48);
    x[2] = e ? NAN : 1.0;
    x[3] = e ? NAN : nd(rng);
  }
  std::vector<PNode> pn(P * N);
  std::vector<PConn> pc(P * C);
  std::vector<uint8_t> cf(P * C);
  std::vector<uint8_t> raw((nodes.size() + conns.size()) * 8);
  const double in_bytes = double(raw.size());
  const int maxt = argc > 1 ? std::atoi(argv[1]) : int(std::thread::hardware_concurrency());
  for (int T = 1; T <= maxt; T *= 2) {
    for (int mode = 0; mode < 2; ++mode) {
      double best = 1e30;
      for (int rep = 0; rep < 7; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
          th.emplace_back([&, t] {
            const size_t lo = P * t / T, hi = P * (t + 1) / T;
            if (mode == 0) {
              pack_rows(&nodes[lo * N * 5], &conns[lo * C * 4], (hi - lo) * N, (hi - lo) * C, &pn[lo * N],
                        &pc[lo * C], &cf[lo * C]);
            } else {
              std::memcpy(&raw[lo * N * 40], &nodes[lo * N * 5], (hi - lo) * N * 40);
              std::memcpy(&raw[P * N * 40 + lo * C * 32], &conns[lo * C * 4], (hi - lo) * C * 32);
            }
          });
        for (auto& x : th) x.join();
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        best = std::min(best, s);
      }
      std::printf("threads %2d %-6s %.3f ms  %.1f GB/s of raw rows\n", T, mode ? "memcpy" : "pack", best * 1e3,
                  in_bytes / best / 1e9);
    }
  }
  std::printf("packed bytes / raw bytes = %.3f\n",
              double(pn.size() * sizeof(PNode) + pc.size() * sizeof(PConn) + cf.size()) / in_bytes);
  return 0;
}
