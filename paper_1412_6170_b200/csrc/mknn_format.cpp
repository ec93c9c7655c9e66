// mknn_format.cpp -- native result consumer: the CSV rows
// studies.py:105-108 write_result_block produces,
//     f"{tick},{qid},{r},{ids[r]},{dists[r]:.9g}\n"
// for every query row and rank, formatted on all host threads instead of a
// Python loop.  "%.9g" is C's format, which Python's format spec mirrors
// (both correctly rounded; inf/nan spelled the same).
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/mknn_b200.h"

namespace {

// one row group [r0, r1) into out; returns bytes written or -1 if cap is short
int64_t format_rows(int64_t tick, int64_t r0, int64_t r1, const int64_t* qids,
                    const int64_t* offsets, const int64_t* nids, const double* dist, char* out,
                    int64_t cap) {
  int64_t w = 0;
  char line[128];
  for (int64_t r = r0; r < r1; r++) {
    for (int64_t e = offsets[r]; e < offsets[r + 1]; e++) {
      // std::to_chars(general, 9) is printf's "%.9g", exactly rounded
      // a line is at most 4 x 20 digits + 16 + 5 separators < sizeof(line);
      // the checks keep every write provably inside the buffer
      char* p = line;
      char* const end = line + sizeof(line) - 1;
      auto field = [&](auto r, char sep) {
        if (r.ec != std::errc() || r.ptr >= end) return false;
        p = r.ptr;
        *p++ = sep;
        return true;
      };
      if (!field(std::to_chars(p, end, (long long)tick), ',') ||
          !field(std::to_chars(p, end, (long long)qids[r]), ',') ||
          !field(std::to_chars(p, end, (long long)(e - offsets[r])), ',') ||
          !field(std::to_chars(p, end, (long long)nids[e]), ',') ||
          !field(std::to_chars(p, end, dist[e], std::chars_format::general, 9), '\n'))
        return -1;
      const int64_t n = p - line;
      if (w + n > cap) return -1;
      memcpy(out + w, line, (size_t)n);
      w += n;
    }
  }
  return w;
}

}  // namespace

extern "C" int64_t mknn_format_result_rows(int64_t tick, int64_t nq, const int64_t* qids,
                                           const int64_t* offsets, const int64_t* nids,
                                           const double* dist, char* out, int64_t cap,
                                           int32_t threads) {
  if (nq < 0 || cap < 0 || (nq && (!qids || !offsets)) || (!out && cap)) return MKNN_EINVAL;
  if (nq == 0) return 0;
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::min<int64_t>(nt, std::max<int64_t>(1, nq / 1024));
  // split by result entries so the threads get equal work
  const int64_t total = offsets[nq] - offsets[0];
  std::vector<int64_t> cut(nt + 1, nq);
  cut[0] = 0;
  for (int t = 1; t < nt; t++) {
    const int64_t target = offsets[0] + total * t / nt;
    cut[t] = std::upper_bound(offsets, offsets + nq, target) - offsets - 1;
    cut[t] = std::max(cut[t], cut[t - 1]);
  }
  // each thread formats into its own buffer (worst case 100 B per entry)
  std::vector<std::vector<char>> bufs(nt);
  std::vector<int64_t> lens(nt, 0);
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; t++) {
    pool.emplace_back([&, t] {
      const int64_t n_ent = offsets[cut[t + 1]] - offsets[cut[t]];
      bufs[t].resize((size_t)(n_ent * 100 + 1));
      lens[t] = format_rows(tick, cut[t], cut[t + 1], qids, offsets, nids, dist, bufs[t].data(),
                            (int64_t)bufs[t].size());
    });
  }
  for (auto& th : pool) th.join();
  int64_t w = 0;
  for (int t = 0; t < nt; t++) {
    if (lens[t] < 0) return MKNN_EINVAL;
    if (w + lens[t] > cap) return MKNN_EINVAL;
    memcpy(out + w, bufs[t].data(), (size_t)lens[t]);
    w += lens[t];
  }
  return w;
}
