// Diagnostic: batched CPQR (row-ID) engine times on the per-step problem
// shapes (CUDA events, device-resident W^T, each rep re-copies the batch from
// a pristine device copy outside the timed region).  Links the product
// library's internal C++ API.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//     -I paper_2108_07205_b200/csrc -I include scripts/id_bench.cu \
//     -L paper_2108_07205_b200/_lib -lsbx -Xlinker -rpath=$PWD/paper_2108_07205_b200/_lib -o scripts/id_bench
//   scripts/id_bench [engine ...]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <array>
#include <cmath>
#include <random>
#include <map>
#include <string>
#include <vector>

#include "idengine.hpp"

using namespace sbx;
#ifdef SBX_CPQR_PROF
namespace sbx {
void cpqr_prof_dump();
void cpqr_rows_prof_dump();
void cpqr_push_prof_dump();
void bqr_prof_dump();
}
#endif

struct Case {
  const char* name;
  std::vector<std::array<int, 4>> groups;  // M, n, rank, count
};

struct Prob {
  int M, n;
  double eps;
  std::vector<double> w;
};

float time_batch(const std::vector<Prob>& probs, int e, cudaStream_t s, int* k0, std::string* err) {
  i64 tot = 0;
  std::vector<i64> off;
  for (const auto& p : probs) {
    off.push_back(tot);
    tot += i64(p.M) * p.n;
  }
  DevBuf<double> pristine(static_cast<size_t>(tot)), work(static_cast<size_t>(tot));
  for (size_t q = 0; q < probs.size(); ++q)
    SBX_CUDA(cudaMemcpy(pristine.get() + off[q], probs[q].w.data(), probs[q].w.size() * 8, cudaMemcpyHostToDevice));
  std::vector<IdProblem> ps;
  for (size_t q = 0; q < probs.size(); ++q) ps.push_back({work.get() + off[q], probs[q].M, probs[q].n, probs[q].M});
  float best = 1e30f, worst = 0.f;
  static const int reps = std::getenv("ID_REPS") ? std::atoi(std::getenv("ID_REPS")) : 3;
  for (int rep = 0; rep < reps; ++rep) {
    SBX_CUDA(cudaMemcpyAsync(work.get(), pristine.get(), size_t(tot) * 8, cudaMemcpyDeviceToDevice, s));
    IdBatch b;
    b.force_engine = e;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    try {
      b.factor(ps, probs[0].eps, s);
    } catch (const std::exception& ex) {
      *err = ex.what();
      return -1.0f;
    }
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
    worst = std::max(worst, ms);
    *k0 = int(b.eps_rank(0, 1e-10));
  }
  if (reps > 3) std::printf(" [worst %.3f]", worst);
  return best;
}

int replay(const char* dir, const std::vector<int>& engines) {
  cudaStream_t s = lib_stream();
  std::vector<double> total(engines.size(), 0.0);
  double best_total = 0.0;
  for (int seq = 0;; ++seq) {
    char path[512];
    std::snprintf(path, sizeof(path), "%s/batch_%04d.bin", dir, seq);
    FILE* f = std::fopen(path, "rb");
    if (!f) break;
    static const char* only = std::getenv("ID_BATCH");
    if (only && std::atoi(only) != seq) {
      std::fclose(f);
      continue;
    }
    long long np = 0;
    if (std::fread(&np, sizeof(np), 1, f) != 1) break;
    std::vector<Prob> probs(static_cast<size_t>(np));
    std::map<std::string, int> shapes;
    for (auto& p : probs) {
      long long hdr[4];
      if (std::fread(hdr, sizeof(hdr), 1, f) != 1 || std::fread(&p.eps, sizeof(double), 1, f) != 1) return 1;
      p.M = int(hdr[0]);
      p.n = int(hdr[1]);
      p.w.resize(size_t(p.M) * p.n);
      if (std::fread(p.w.data(), sizeof(double), p.w.size(), f) != p.w.size()) return 1;
      shapes[std::to_string(p.M) + "x" + std::to_string(p.n)]++;
    }
    std::fclose(f);
    std::string desc;
    int shown = 0;
    for (const auto& kv : shapes)
      if (shown++ < 4) desc += kv.first + "*" + std::to_string(kv.second) + " ";
    if (shapes.size() > 4) desc += "...";
    std::printf("batch %3d (%3lld probs) %-44s", seq, np, desc.c_str());
    if (std::getenv("ID_STATS")) {  // per problem class: count, steps taken (auto routing)
      i64 tot = 0;
      for (const auto& p : probs) tot += i64(p.M) * p.n;
      DevBuf<double> work(static_cast<size_t>(tot));
      std::vector<IdProblem> ps;
      i64 o = 0;
      for (const auto& p : probs) {
        SBX_CUDA(cudaMemcpy(work.get() + o, p.w.data(), p.w.size() * 8, cudaMemcpyHostToDevice));
        ps.push_back({work.get() + o, p.M, p.n, p.M});
        o += i64(p.M) * p.n;
      }
      IdBatch b;
      b.factor(ps, probs[0].eps, s);
      std::map<std::pair<int, int>, std::vector<i64>> cls;
      double fl = 0;
      for (size_t q = 0; q < probs.size(); ++q) {
        const i64 k = b.eps_rank(q, 1e-300);
        cls[{probs[q].M, probs[q].n}].push_back(k);
        for (i64 j = 0; j < k; ++j) fl += 4.0 * double(probs[q].M - j) * double(probs[q].n - j);
      }
      std::printf("\n  flops %.3g; classes:", fl);
      for (const auto& kv : cls) {
        i64 mx = 0, sm = 0;
        for (i64 k : kv.second) mx = std::max(mx, k), sm += k;
        std::printf(" %dx%d*%zu(k avg %.0f max %lld)", kv.first.first, kv.first.second, kv.second.size(),
                    double(sm) / kv.second.size(), (long long)mx);
      }
      std::printf("\n  ");
    }
    double b = 1e30;
    for (size_t q = 0; q < engines.size(); ++q) {
      int k0 = -1;
      std::string err;
      const float ms = time_batch(probs, engines[q], s, &k0, &err);
#ifdef SBX_CPQR_PROF
      std::printf("\n[first problem %dx%d]\n", probs[0].M, probs[0].n);
      std::fflush(stdout);
      if (engines[q] == 7) cpqr_rows_prof_dump();
      else if (engines[q] == 8 || engines[q] == 9) cpqr_push_prof_dump();
      else if (engines[q] == 10) bqr_prof_dump();
      else cpqr_prof_dump();
#endif
      if (ms < 0) {
        std::printf("  e%d    n/a  ", engines[q]);
        total[q] = 1e30;
      } else {
        std::printf("  e%d %7.3f", engines[q], ms);
        total[q] += ms;
        b = std::min(b, double(ms));
      }
    }
    best_total += b;
    std::printf("\n");
    std::fflush(stdout);
  }
  std::printf("total:");
  for (size_t q = 0; q < engines.size(); ++q) std::printf("  e%d %8.3f", engines[q], total[q] > 1e29 ? -1.0 : total[q]);
  std::printf("  best-per-batch %8.3f ms\n", best_total);
  return 0;
}

int main(int argc, char** argv) {
  std::vector<int> engines;
  const char* rdir = nullptr;
  for (int i = 1; i < argc; ++i) {
    if (std::string(argv[i]) == "--replay" && i + 1 < argc) {
      rdir = argv[++i];
      continue;
    }
    engines.push_back(std::atoi(argv[i]));
  }
  if (rdir) {
    SBX_CUDA(cudaSetDevice(0));
    return replay(rdir, engines.empty() ? std::vector<int>{0} : engines);
  }
  if (engines.empty()) engines = {0, 1, 3, 4};
  const std::vector<Case> cases = {
      {"app leaves 511x128 r57 x36", {{511, 128, 57, 36}}},
      {"app level 599x114 r57 x36", {{599, 114, 57, 36}}},
      {"app level 849x112 r56 x20", {{849, 112, 56, 10}, {593, 112, 56, 10}}},
      {"upd leaves 257x256 r12 x151", {{257, 256, 12, 151}}},
      {"upd leaves 513x256 r12 x151", {{513, 256, 12, 151}}},
      {"upd leaves 1088x256 r25 x32", {{1088, 256, 25, 32}}},
      {"upd near 8192x256 r80 x4", {{8192, 256, 80, 4}}},
      {"upd near 8192x256 r16 x1", {{8192, 256, 16, 1}}},
      {"upd tall 511/767x128 r55 x240", {{511, 128, 55, 120}, {767, 128, 55, 120}}},
      {"upd tall 511/767x128 r55 x60", {{511, 128, 55, 30}, {767, 128, 55, 30}}},
      {"upd tall 767x128 r55 x1", {{767, 128, 55, 1}}},
      {"upd near 8192x256 r16 x4", {{8192, 256, 16, 4}}},
      {"upd near 2048x256 r16 x1", {{2048, 256, 16, 1}}},
      {"upd leaves all", {{257, 256, 12, 151}, {513, 256, 12, 151}, {1088, 256, 25, 32}}},
      {"upd leaves 257x256 r12 x1", {{257, 256, 12, 1}}},
      {"upd leaves 257x256 r12 x32", {{257, 256, 12, 32}}},
      {"upd leaves 257x256 r120 x32", {{257, 256, 120, 32}}},
      {"upd merge 257x30 r15 x40", {{257, 30, 15, 40}}},
      {"upd merge 513x90 r45 x4", {{513, 90, 45, 4}}},
      {"final 62x31168 r62", {{62, 31168, 62, 1}}},
      {"final 53x8192 r53", {{53, 8192, 53, 1}}},
  };
  SBX_CUDA(cudaSetDevice(0));
  cudaStream_t s = lib_stream();
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  const char* only = std::getenv("ID_CASE");
  for (const auto& c : cases) {
    if (only && !std::strstr(c.name, only)) continue;
    // W^T = G1 (M x r) diag(10^(-14 i / r)) G2 (r x n)
    std::vector<i64> off;
    i64 tot = 0;
    std::vector<std::array<int, 4>> probs;
    for (const auto& g : c.groups)
      for (int q = 0; q < g[3]; ++q) {
        probs.push_back(g);
        off.push_back(tot);
        tot += i64(g[0]) * g[1];
      }
    std::vector<double> h(static_cast<size_t>(tot));
    for (size_t p = 0; p < probs.size(); ++p) {
      const int M = probs[p][0], n = probs[p][1], r = probs[p][2];
      std::vector<double> a(size_t(M) * r), b(size_t(r) * n);
      for (auto& x : a) x = nd(rng);
      for (int l = 0; l < r; ++l) {
        const double sc = std::pow(10.0, -14.0 * l / r);
        for (int j = 0; j < n; ++j) b[l + size_t(j) * r] = sc * nd(rng);
      }
      double* w = h.data() + off[p];
      for (int j = 0; j < n; ++j)
        for (int i = 0; i < M; ++i) {
          double acc = 0.0;
          for (int l = 0; l < r; ++l) acc += a[i + size_t(l) * M] * b[l + size_t(j) * r];
          w[i + size_t(j) * M] = acc;
        }
    }
    DevBuf<double> pristine(static_cast<size_t>(tot)), work(static_cast<size_t>(tot));
    pristine.upload(h.data(), h.size(), s);
    std::printf("%-32s", c.name);
    for (int e : engines) {
      std::vector<IdProblem> ps;
      for (size_t p = 0; p < probs.size(); ++p) ps.push_back({work.get() + off[p], probs[p][0], probs[p][1], probs[p][0]});
      float best = 1e30f;
      int rank0 = -1;
      bool ok = true;
      for (int rep = 0; rep < 4; ++rep) {
        SBX_CUDA(cudaMemcpyAsync(work.get(), pristine.get(), size_t(tot) * 8, cudaMemcpyDeviceToDevice, s));
        IdBatch b;
        b.force_engine = e;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
        try {
          b.factor(ps, 1e-10, s);
        } catch (const std::exception& ex) {
          std::printf(" e%d: n/a (%s)", e, ex.what());
          ok = false;
          break;
        }
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
        rank0 = int(b.eps_rank(0, 1e-10));
      }
      if (ok) std::printf("  e%d %8.3f ms (k0 %d)", e, best, rank0);
#ifdef SBX_CPQR_PROF
      std::fflush(stdout);
      if (e == 7) cpqr_rows_prof_dump();
      else cpqr_prof_dump();
#endif
    }
    std::printf("\n");
    std::fflush(stdout);
  }
  return 0;
}
