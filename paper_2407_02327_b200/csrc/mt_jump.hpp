// mt_jump.hpp -- GF(2) jump-ahead polynomials for std::mt19937_64 (host side).
//
// mt19937_64's raw word sequence x[n] satisfies a linear recurrence over GF(2)
// whose characteristic polynomial phi has degree 19937.  For any jump J, with
// p(t) = t^J mod phi(t):   x[J + k] = XOR_{i : p_i = 1} x[i + k]   (k >= 1, and
// the upper 33 bits of k = 0) -- so the generator state J words ahead is a
// GF(2) combination of the first 19937+312 raw words of the seed.  The
// polynomials do not depend on the seed and are cached.
#pragma once

#include <cstdint>
#include <vector>

namespace qsb {
namespace mtjump {

constexpr int kDegree = 19937;
constexpr int kPolyWords = 312;             // ceil(19937 / 64)
constexpr int64_t kRawWords = 312 * 65;     // >= 19937 + 312 raw words per seed

// Segment length (in twist blocks) rounding used by the SR launcher so that
// jump tables are shared between calls of similar size.
int64_t round_segment_blocks(int64_t blocks);

// Polynomials t^(312*T_b) mod phi for each twist count T_b (row-major,
// kPolyWords words per row).  The returned buffer stays valid until the next
// call on the same thread.
const std::vector<uint64_t>& jump_polys(const std::vector<uint64_t>& twists);

// Host self-test: checks the jump identity against a scalar mt19937_64 for a
// few offsets.  Returns 0 on success.
int self_test();

}  // namespace mtjump
}  // namespace qsb
