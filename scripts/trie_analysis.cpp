// Offline analysis aid (not product code): count the work of subset queries
// "exists x in A with x ⊆ y" for y in B under different state orders of the
// lex/Patricia trie.  Reads raw u64 list dumps (SYNCHRO_DUMP_DIR).
// Build: g++ -O2 -std=c++20 scripts/trie_analysis.cpp -o /tmp/trie_analysis
#include <algorithm>
#include <bit>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <numeric>
#include <random>
#include <string>
#include <vector>

using u64 = uint64_t;
using u32 = uint32_t;
static int N_BITS, W;

std::vector<u64> load(const std::string& p) {
  std::ifstream f(p, std::ios::binary | std::ios::ate);
  size_t sz = f.tellg();
  f.seekg(0);
  std::vector<u64> v(sz / 8);
  f.read(reinterpret_cast<char*>(v.data()), sz);
  return v;
}

bool test(const u64* x, int q) { return (x[q >> 6] >> (63 - (q & 63))) & 1; }

std::vector<u64> permute(const std::vector<u64>& l, const std::vector<int>& pos /* state -> new pos */) {
  size_t cnt = l.size() / W;
  std::vector<u64> out(l.size(), 0);
  for (size_t i = 0; i < cnt; ++i)
    for (int q = 0; q < N_BITS; ++q)
      if (test(&l[i * W], q)) out[i * W + (pos[q] >> 6)] |= u64{1} << (63 - (pos[q] & 63));
  return out;
}

struct Counter {
  u64 nodes = 0, pairs = 0, hits = 0;
  std::vector<u64> per;
};
static bool PROPER = false;
static size_t BRUTE = 12;

struct Sorted {
  std::vector<u64> w;
  std::vector<u32> card;
  size_t n;
};

Sorted sort_unique(const std::vector<u64>& l) {
  size_t cnt = l.size() / W;
  std::vector<u32> idx(cnt);
  std::iota(idx.begin(), idx.end(), 0);
  std::sort(idx.begin(), idx.end(), [&](u32 a, u32 b) {
    return std::lexicographical_compare(&l[a * W], &l[a * W + W], &l[b * W], &l[b * W + W]);
  });
  Sorted s;
  for (u32 i : idx) {
    s.w.insert(s.w.end(), &l[i * W], &l[i * W + W]);
    u32 c = 0;
    for (int t = 0; t < W; ++t) c += std::popcount(l[i * W + t]);
    s.card.push_back(c);
  }
  s.n = cnt;
  return s;
}

// Implicit Patricia traversal (same pruning as contain_query_kernel, minus
// subtree min-card which we emulate with an exact range-min).
void query(const Sorted& A, const std::vector<std::vector<u32>>& rmq, const u64* y, u32 cy,
           Counter& c) {
  auto rmin = [&](size_t lo, size_t hi) {  // [lo, hi)
    int k = 31 - std::countl_zero(static_cast<u32>(hi - lo));
    return std::min(rmq[k][lo], rmq[k][hi - (size_t{1} << k)]);
  };
  struct F { size_t lo, hi; int d; };
  std::vector<F> st{{0, A.n, 0}};
  while (!st.empty()) {
    F f = st.back();
    st.pop_back();
    ++c.nodes;
    if (rmin(f.lo, f.hi) > cy - (PROPER ? 1 : 0)) continue;
    if (f.hi - f.lo <= BRUTE) {
      for (size_t i = f.lo; i < f.hi; ++i) {
        ++c.pairs;
        if (A.card[i] > cy - (PROPER ? 1 : 0)) continue;
        bool ok = true;
        for (int t = 0; t < W; ++t) ok &= !(A.w[i * W + t] & ~y[t]);
        if (ok) { ++c.hits; return; }
      }
      continue;
    }
    // first differing bit between first and last
    int L = 0;
    for (int t = 0; t < W; ++t) {
      u64 x = A.w[f.lo * W + t] ^ A.w[(f.hi - 1) * W + t];
      if (x) { L = t * 64 + std::countl_zero(x); break; }
    }
    bool bad = false;
    for (int q = f.d; q < L; ++q) if (test(&A.w[f.lo * W], q) && !test(y, q)) { bad = true; break; }
    if (bad) continue;
    size_t lo = f.lo, hi = f.hi;
    while (lo < hi) { size_t m = (lo + hi) / 2; if (test(&A.w[m * W], L)) hi = m; else lo = m + 1; }
    if (test(y, L)) st.push_back({lo, f.hi, L + 1});
    st.push_back({f.lo, lo, L + 1});
  }
}

int main(int argc, char** argv) {
  N_BITS = std::stoi(argv[1]);
  W = (N_BITS + 63) / 64;
  auto A0 = load(argv[2]);
  auto B0 = load(argv[3]);
  size_t sample = argc > 4 ? std::stoul(argv[4]) : 3000;
  PROPER = argc > 5 && std::string(argv[5]) == "proper";
  if (argc > 6) BRUTE = std::stoul(argv[6]);
  size_t na = A0.size() / W, nb = B0.size() / W;
  std::vector<double> fa(N_BITS), fb(N_BITS);
  for (size_t i = 0; i < na; ++i) for (int q = 0; q < N_BITS; ++q) fa[q] += test(&A0[i * W], q);
  for (size_t i = 0; i < nb; ++i) for (int q = 0; q < N_BITS; ++q) fb[q] += test(&B0[i * W], q);
  double ca = 0, cb = 0;
  for (int q = 0; q < N_BITS; ++q) { fa[q] /= na; fb[q] /= nb; ca += fa[q]; cb += fb[q]; }
  printf("A=%zu sets avg card %.1f, B=%zu sets avg card %.1f\n", na, ca, nb, cb);
  std::mt19937 rng(1);
  std::vector<size_t> qs;
  for (size_t i = 0; i < sample; ++i) qs.push_back(rng() % nb);

  auto run = [&](const char* name, std::vector<double> key) {
    std::vector<int> order(N_BITS);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return key[a] > key[b]; });
    std::vector<int> pos(N_BITS);
    for (int i = 0; i < N_BITS; ++i) pos[order[i]] = i;
    auto A = sort_unique(permute(A0, pos));
    auto B = permute(B0, pos);
    std::vector<std::vector<u32>> rmq{A.card};
    for (int k = 1; (size_t{1} << k) <= A.n; ++k) {
      std::vector<u32> r(A.n - (size_t{1} << k) + 1);
      for (size_t i = 0; i < r.size(); ++i) r[i] = std::min(rmq[k - 1][i], rmq[k - 1][i + (size_t{1} << (k - 1))]);
      rmq.push_back(std::move(r));
    }
    Counter c;
    for (size_t j : qs) {
      u32 cy = 0;
      for (int t = 0; t < W; ++t) cy += std::popcount(B[j * W + t]);
      const u64 before = c.nodes + c.pairs;
      if (!(PROPER && cy == 0)) query(A, rmq, &B[j * W], cy, c);
      c.per.push_back(c.nodes + c.pairs - before);
    }
    std::sort(c.per.begin(), c.per.end());
    printf("%-28s nodes/query %9.1f pairs/query %9.1f hits %llu  p50 %llu p99 %llu max %llu\n", name,
           double(c.nodes) / sample, double(c.pairs) / sample, (unsigned long long)c.hits,
           (unsigned long long)c.per[c.per.size() / 2], (unsigned long long)c.per[c.per.size() * 99 / 100],
           (unsigned long long)c.per.back());
  };
  std::vector<double> natural(N_BITS), freqA(fa), freqAinv(N_BITS), prune(N_BITS), freqB(N_BITS);
  for (int q = 0; q < N_BITS; ++q) {
    natural[q] = -q;
    freqAinv[q] = -fa[q];
    prune[q] = fa[q] * (1 - fb[q]);
    freqB[q] = -fb[q];
  }
  run("natural order", natural);
  run("A-frequency desc", freqA);
  run("A-frequency asc", freqAinv);
  run("fA*(1-fB) desc", prune);
  run("B-frequency asc", freqB);
  return 0;
}
