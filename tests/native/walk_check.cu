// Host-side check of lw::MemberMajorWalk (lw_common.cuh): for every member count
// M, tile start e0 and length n it must yield the tile's positions sorted by
// (position mod M, position) — the reference's member-major y[tile] += order
// (_fast.py:66-77). Prints "cases N bad B".
#include <algorithm>
#include <cstdio>
#include <vector>

#include "lw_common.cuh"

int main() {
    int bad = 0, cases = 0;
    for (int64_t M : {1, 2, 3, 5, 7, 8, 32, 100, 256})
        for (int64_t e0 = 0; e0 < 3 * M + 5; e0 += (M > 32 ? 7 : 1))
            for (int64_t n = 0; n < 5 * M + 40; n += (n < 40 ? 1 : 13)) {
                std::vector<int64_t> want;
                for (int64_t k = e0; k < e0 + n; ++k) want.push_back(k);
                std::stable_sort(want.begin(), want.end(),
                                 [&](int64_t a, int64_t b) { return a % M < b % M; });
                lw::MemberMajorWalk w(e0, e0 + n, M);
                std::vector<int64_t> got;
                for (int64_t p; (p = w.next()) >= 0;) got.push_back(p);
                ++cases;
                if (got != want) {
                    if (++bad < 5) std::printf("mismatch M=%ld e0=%ld n=%ld\n", (long)M, (long)e0, (long)n);
                }
            }
    std::printf("cases %d bad %d\n", cases, bad);
    return bad != 0;
}
