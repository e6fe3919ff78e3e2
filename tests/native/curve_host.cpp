// Host build of the device curve math (csrc/gilbert.cuh) for CPU-side checks of the
// descent against the reference order.  Test-only: prints fwd for each "t h w" line.
#include <cstdio>
#include <vector>
#include "../../paper_2505_16864_b200/csrc/gilbert.cuh"

int main() {
  int t, h, w;
  while (std::scanf("%d %d %d", &t, &h, &w) == 3) {
    tcb::CurveGeom g = tcb::curve_geom(t, h, w);
    int64_t n = (int64_t)t * h * w;
    std::vector<int64_t> fwd(n, -1);
    for (int64_t c = 0; c < n; ++c) fwd[tcb::curve_position(g, c)] = c;
    for (int64_t i = 0; i < n; ++i) std::printf("%lld%c", (long long)fwd[i], i + 1 == n ? '\n' : ' ');
  }
  return 0;
}
