// Host check of morton_compact (csrc/common.cuh): for every W x H rectangle up
// to 48 x 48 the ranks 0 .. W*H-1 map to every point exactly once, in strictly
// increasing Morton key order (x on the even bits, y on the odd bits).
#include <cstdio>
#include <set>
#include <utility>

#include "common.cuh"

int main() {
  int bad = 0;
  for (int W = 1; W <= 48; ++W)
    for (int H = 1; H <= 48; ++H) {
      std::set<std::pair<int, int>> seen;
      long long prev = -1;
      for (int id = 0; id < W * H; ++id) {
        int x, y;
        pcotgpu::morton_compact(id, W, H, x, y);
        if (x < 0 || x >= W || y < 0 || y >= H) ++bad;
        seen.insert({x, y});
        long long key = 0;
        for (int b = 0; b < 12; ++b) key |= (long long)((x >> b) & 1) << (2 * b) | (long long)((y >> b) & 1) << (2 * b + 1);
        if (key <= prev) ++bad;
        prev = key;
      }
      if (int(seen.size()) != W * H) ++bad;
    }
  std::printf("MORTON_BAD %d\n", bad);
  return bad != 0;
}
