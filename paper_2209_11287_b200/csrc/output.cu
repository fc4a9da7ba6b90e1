// Canonical squared distances of an emitted pair set, for the pairs file.
//
// Reference: cli._canonical_pair_sq_dists (cli.py:270-283) + _write_pairs
// (cli.py:285-289): for every (i, j) of the sorted pair list,
//   acc = 0; for dim in 0..d-1: diff = x[i,dim] - x[j,dim]; acc += diff*diff
// i.e. the direct form with one correctly rounded op each (numpy, no FMA),
// whichever kernel produced the pair.  Here the pair list is the CSR
// (offsets by original id, neighbour ids); coordinates are the caller's
// original-order buffer (row stride ld).  One thread per pair; the row of a
// pair is found by a binary search of its index in the offsets (rows are
// contiguous, so a warp's search paths coincide).
#include "internal.cuh"

namespace tj {

__global__ void pair_sq_dist_kernel(const double* __restrict__ x, int64_t ld, int d,
                                    const int64_t* __restrict__ offsets, int64_t n,
                                    const uint32_t* __restrict__ nbr, int64_t m,
                                    double* __restrict__ out) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m;
       e += int64_t(gridDim.x) * blockDim.x) {
    int64_t lo = 0, hi = n;  // row i with offsets[i] <= e < offsets[i+1]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (offsets[mid] <= e) lo = mid;
      else hi = mid;
    }
    const double* a = x + lo * ld;
    const double* b = x + int64_t(nbr[e]) * ld;
    double acc = 0.0;
    for (int k = 0; k < d; ++k) {
      const double t = __dsub_rn(a[k], b[k]);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
    out[e] = acc;
  }
}

void launch_pair_sq_dists(const double* x, int64_t ld, int d, const int64_t* offsets, int64_t n,
                          const uint32_t* nbr, int64_t m, double* out, cudaStream_t s) {
  if (m <= 0) return;
  const unsigned grid =
      unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), int64_t(kNumSMs) * 16)));
  pair_sq_dist_kernel<<<grid, 256, 0, s>>>(x, ld, d, offsets, n, nbr, m, out);
  TJ_CHECK_LAUNCH();
}

}  // namespace tj

// ---------------------------------------------------------------- pairs file
// Host side of _write_pairs (cli.py:285-289): one "i j sq" line per pair, sq
// printed like Python's f"{s:.17g}" (C's %.17g: the same correctly rounded
// digits and exponent rule).  Pairs are formatted in blocks by a pool of host
// threads and written in order.
#include <algorithm>
#include <cstdio>
#include <thread>

namespace tj {

void write_pairs_file(const char* path, const int64_t* offsets, int64_t n, const uint32_t* nbr,
                      const double* sq, int threads) {
  FILE* f = std::fopen(path, "wb");
  if (!f) fail(TJ_EINVAL, std::string("cannot open ") + path + " for writing");
  const int64_t m = offsets[n];
  const int T = std::max(1, threads);
  constexpr int64_t kBlock = int64_t(1) << 20;  // pairs per thread per round
  std::vector<std::string> bufs(T);
  int64_t row = 0;  // row of the next pair to format
  for (int64_t e0 = 0; e0 < m; e0 += kBlock * T) {
    // row at which each thread's block starts
    std::vector<int64_t> rstart(T + 1), estart(T + 1);
    for (int t = 0; t <= T; ++t) {
      estart[t] = std::min(m, e0 + kBlock * t);
      while (row < n && offsets[row + 1] <= estart[t]) ++row;
      rstart[t] = row;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) {
      pool.emplace_back([&, t] {
        std::string& b = bufs[t];
        b.clear();
        char line[80];
        int64_t r = rstart[t];
        for (int64_t e = estart[t]; e < estart[t + 1]; ++e) {
          while (offsets[r + 1] <= e) ++r;
          const int k = std::snprintf(line, sizeof line, "%lld %u %.17g\n", (long long)r, nbr[e], sq[e]);
          b.append(line, size_t(k));
        }
      });
    }
    for (auto& th : pool) th.join();
    for (int t = 0; t < T; ++t)
      if (!bufs[t].empty() && std::fwrite(bufs[t].data(), 1, bufs[t].size(), f) != bufs[t].size()) {
        std::fclose(f);
        fail(TJ_EINVAL, std::string("short write to ") + path);
      }
  }
  if (std::fclose(f) != 0) fail(TJ_EINVAL, std::string("error closing ") + path);
}

}  // namespace tj

// ------------------------------------------------------------ (m, 2) pairs
// JoinResult.pairs (join.py:80-91): the CSR expanded into (query id, neighbour
// id) int64 rows.  Host threads take contiguous row ranges of ~equal pair count
// and write (and first-touch) their own part of the output.
namespace tj {

void expand_pairs(const int64_t* offsets, int64_t n, const uint32_t* nbr, int64_t* out,
                  int threads) {
  const int64_t m = offsets[n];
  const int T = int(std::max<int64_t>(1, std::min<int64_t>(threads, m / (int64_t(1) << 16) + 1)));
  std::vector<int64_t> rstart(T + 1, n);
  rstart[0] = 0;
  for (int t = 1; t < T; ++t)  // first row whose pairs start at or after t*m/T
    rstart[t] = std::lower_bound(offsets, offsets + n + 1, m / T * t) - offsets;
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] {
      for (int64_t r = std::min(rstart[t], n); r < std::min(rstart[t + 1], n); ++r)
        for (int64_t e = offsets[r]; e < offsets[r + 1]; ++e) {
          out[2 * e] = r;
          out[2 * e + 1] = int64_t(nbr[e]);
        }
    });
  for (auto& th : pool) th.join();
}

}  // namespace tj
