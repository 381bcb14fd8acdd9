// mt_jump.cpp -- host GF(2)[t] arithmetic for mt19937_64 jump-ahead.
//
//  * phi: the characteristic polynomial of the mt19937_64 recurrence, found
//    once per process by Berlekamp-Massey on 2*19937+ bits of one raw output
//    bit (its minimal polynomial is phi because phi is irreducible).
//  * t^J mod phi by square-and-multiply; products with PCLMULQDQ carry-less
//    multiplies, reductions by Barrett (exact over GF(2): q = floor(floor(P /
//    t^d) * mu / t^d), mu = floor(t^(2d) / phi)).
// Seed-independent; cached per (first twist count, twist stride).
#include "mt_jump.hpp"

#include <immintrin.h>

#include <cstring>
#include <map>
#include <mutex>
#include <utility>

namespace qsb {
namespace mtjump {

namespace {

using Poly = std::vector<uint64_t>;  // bit i of the array = coefficient of t^i

constexpr int D = kDegree;
constexpr int MT_N = 312;
constexpr int MT_M = 156;
constexpr uint64_t UPPER = 0xFFFFFFFF80000000ULL;
constexpr uint64_t LOWER = 0x000000007FFFFFFFULL;
constexpr uint64_t MATA = 0xB5026F5AA96619E9ULL;

// Raw (untempered) recurrence words of a seed: out[0..312) = seeded state.
Poly raw_words(uint64_t seed, int64_t len) {
    Poly x(static_cast<size_t>(std::max<int64_t>(len, MT_N)));
    x[0] = seed;
    for (int i = 1; i < MT_N; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
    for (int64_t n = MT_N; n < len; ++n) {
        const uint64_t y = (x[n - MT_N] & UPPER) | (x[n - MT_N + 1] & LOWER);
        x[n] = x[n - MT_N + MT_M] ^ (y >> 1) ^ ((y & 1) ? MATA : 0);
    }
    x.resize(static_cast<size_t>(len));
    return x;
}

inline int get_bit(const Poly& p, int64_t i) { return static_cast<int>((p[i >> 6] >> (i & 63)) & 1); }

int degree(const Poly& p) {
    for (int64_t w = static_cast<int64_t>(p.size()) - 1; w >= 0; --w)
        if (p[w]) return static_cast<int>(w * 64 + 63 - __builtin_clzll(p[w]));
    return -1;
}

// a ^= b * t^s
void xor_shifted(Poly& a, const Poly& b, int64_t s) {
    const int64_t ws = s >> 6;
    const int bs = static_cast<int>(s & 63);
    const size_t need = b.size() + ws + 1;
    if (a.size() < need) a.resize(need, 0);
    if (bs == 0) {
        for (size_t i = 0; i < b.size(); ++i) a[i + ws] ^= b[i];
    } else {
        for (size_t i = 0; i < b.size(); ++i) {
            a[i + ws] ^= b[i] << bs;
            a[i + ws + 1] ^= b[i] >> (64 - bs);
        }
    }
}

Poly clmul(const Poly& a, const Poly& b) {
    Poly r(a.size() + b.size() + 1, 0);
    for (size_t i = 0; i < a.size(); ++i) {
        if (!a[i]) continue;
        const __m128i va = _mm_set_epi64x(0, static_cast<long long>(a[i]));
        for (size_t j = 0; j < b.size(); ++j) {
            const __m128i vb = _mm_set_epi64x(0, static_cast<long long>(b[j]));
            const __m128i p = _mm_clmulepi64_si128(va, vb, 0x00);
            r[i + j] ^= static_cast<uint64_t>(_mm_cvtsi128_si64(p));
            r[i + j + 1] ^= static_cast<uint64_t>(_mm_extract_epi64(p, 1));
        }
    }
    return r;
}

// floor(a / t^s)
Poly shr(const Poly& a, int64_t s) {
    const int64_t ws = s >> 6;
    const int bs = static_cast<int>(s & 63);
    if (ws >= static_cast<int64_t>(a.size())) return Poly(1, 0);
    Poly r(a.size() - ws, 0);
    for (size_t i = 0; i < r.size(); ++i) {
        uint64_t v = a[i + ws] >> bs;
        if (bs && i + ws + 1 < a.size()) v |= a[i + ws + 1] << (64 - bs);
        r[i] = v;
    }
    return r;
}

void truncate(Poly& a, int bits) {
    const size_t words = (bits + 63) / 64;
    a.resize(words, 0);
    if (bits & 63) a[words - 1] &= (1ULL << (bits & 63)) - 1;
}

// Berlekamp-Massey over GF(2): connection polynomial C of the bit sequence s.
Poly berlekamp_massey(const std::vector<uint8_t>& s, int* L_out) {
    const int64_t N = static_cast<int64_t>(s.size());
    const size_t W = static_cast<size_t>((N + 64) / 64 + 2);
    Poly C(W, 0), B(W, 0), T;
    C[0] = B[0] = 1;
    int L = 0;
    int64_t m = 1;
    // rev[j] = s[N-1-j], so the window s[n-L..n] reversed is rev[N-1-n .. N-1-n+L].
    Poly rev(W, 0);
    for (int64_t j = 0; j < N; ++j)
        if (s[N - 1 - j]) rev[j >> 6] |= 1ULL << (j & 63);
    for (int64_t n = 0; n < N; ++n) {
        // d = sum_{i=0..L} C_i s_{n-i} = parity(C & rev >> (N-1-n)) over L+1 bits
        const int64_t off = N - 1 - n;
        const int64_t wo = off >> 6;
        const int bo = static_cast<int>(off & 63);
        uint64_t acc = 0;
        const int64_t cw = L / 64 + 1;
        for (int64_t w = 0; w < cw; ++w) {
            uint64_t v = 0;
            if (wo + w < static_cast<int64_t>(W)) v = rev[wo + w] >> bo;
            if (bo && wo + w + 1 < static_cast<int64_t>(W)) v |= rev[wo + w + 1] << (64 - bo);
            acc ^= C[w] & v;
        }
        // bits of C above L are zero (deg C <= L is a BM invariant)
        const int d = __builtin_parityll(acc);
        if (d == 0) {
            ++m;
        } else if (2 * L <= n) {
            T = C;
            xor_shifted(C, B, m);
            C.resize(W);
            L = static_cast<int>(n + 1 - L);
            B = T;
            m = 1;
        } else {
            xor_shifted(C, B, m);
            C.resize(W);
            ++m;
        }
    }
    *L_out = L;
    truncate(C, L + 1);
    return C;
}

struct Basis {
    Poly phi;  // degree D
    Poly mu;   // floor(t^(2D) / phi)
};

const Basis& basis() {
    static Basis b;
    static std::once_flag once;
    std::call_once(once, [] {
        const int64_t nbits = 2 * static_cast<int64_t>(D) + 256;
        Poly x = raw_words(5489, MT_N + nbits);
        std::vector<uint8_t> s(static_cast<size_t>(nbits));
        for (int64_t n = 0; n < nbits; ++n) s[n] = static_cast<uint8_t>(x[MT_N + n] & 1);
        int L = 0;
        Poly C = berlekamp_massey(s, &L);
        // phi(t) = t^L C(1/t)
        Poly phi((L + 64) / 64, 0);
        for (int k = 0; k <= L; ++k)
            if (get_bit(C, L - k)) phi[k >> 6] |= 1ULL << (k & 63);
        b.phi = phi;
        // mu = floor(t^(2D) / phi) by long division.
        Poly rem((2 * D + 64) / 64 + 1, 0);
        rem[(2 * D) >> 6] |= 1ULL << ((2 * D) & 63);
        Poly q((D + 64) / 64 + 1, 0);
        for (int i = 2 * D; i >= D; --i) {
            if (get_bit(rem, i)) {
                q[(i - D) >> 6] |= 1ULL << ((i - D) & 63);
                xor_shifted(rem, phi, i - D);
            }
        }
        b.mu = q;
    });
    return b;
}

// a * b mod phi for deg a, deg b < D.
Poly mulmod(const Poly& a, const Poly& b) {
    const Basis& B = basis();
    Poly P = clmul(a, b);
    Poly q = shr(clmul(shr(P, D), B.mu), D);
    Poly qp = clmul(q, B.phi);
    for (size_t i = 0; i < P.size() && i < qp.size(); ++i) P[i] ^= qp[i];
    truncate(P, D);
    P.resize(kPolyWords, 0);
    return P;
}

Poly one() {
    Poly p(kPolyWords, 0);
    p[0] = 1;
    return p;
}

// t^J mod phi.
Poly powmod_t(uint64_t J) {
    Poly r = one();
    if (J == 0) return r;
    const Basis& B = basis();
    for (int bit = 63 - __builtin_clzll(J); bit >= 0; --bit) {
        r = mulmod(r, r);
        if ((J >> bit) & 1) {
            // r *= t
            Poly s(kPolyWords + 1, 0);
            for (int i = 0; i < kPolyWords; ++i) {
                s[i] |= r[i] << 1;
                s[i + 1] |= r[i] >> 63;
            }
            if (get_bit(s, D)) {
                for (size_t i = 0; i < B.phi.size(); ++i) s[i] ^= B.phi[i];
            }
            s.resize(kPolyWords);
            r = s;
        }
    }
    return r;
}

struct Progression {
    Poly step;               // t^(312*stride) mod phi
    std::vector<Poly> rows;  // t^(312*(first + b*stride)) mod phi
};

}  // namespace

int64_t round_segment_blocks(int64_t blocks) {
    int64_t p = 64;
    while (p < blocks) p <<= 1;
    return p;
}

const std::vector<uint64_t>& jump_polys(const std::vector<uint64_t>& twists) {
    static std::mutex mu;
    static std::map<std::pair<uint64_t, uint64_t>, Progression> cache;
    thread_local std::vector<uint64_t> out;
    std::lock_guard<std::mutex> lock(mu);
    out.assign(twists.size() * kPolyWords, 0);
    if (twists.empty()) return out;
    const uint64_t first = twists[0];
    const uint64_t stride = twists.size() > 1 ? twists[1] - twists[0] : 1;
    bool progression = true;
    for (size_t b = 0; b < twists.size(); ++b)
        if (twists[b] != first + b * stride) progression = false;
    if (!progression) {
        for (size_t b = 0; b < twists.size(); ++b) {
            Poly p = powmod_t(312ULL * twists[b]);
            std::memcpy(out.data() + b * kPolyWords, p.data(), sizeof(uint64_t) * kPolyWords);
        }
        return out;
    }
    Progression& pr = cache[{first, stride}];
    if (pr.rows.empty()) {
        pr.step = powmod_t(312ULL * stride);
        pr.rows.push_back(powmod_t(312ULL * first));
    }
    while (pr.rows.size() < twists.size()) pr.rows.push_back(mulmod(pr.rows.back(), pr.step));
    for (size_t b = 0; b < twists.size(); ++b)
        std::memcpy(out.data() + b * kPolyWords, pr.rows[b].data(), sizeof(uint64_t) * kPolyWords);
    return out;
}

int self_test() {
    const Basis& B = basis();
    if (degree(B.phi) != D) return 1;
    const uint64_t seed = 12345;
    const uint64_t jumps[] = {1, 311, 312, 1000, 312 * 77 + 5, 312 * 4096};
    const int64_t need = 312 * 4096 + kRawWords + 400;
    Poly x = raw_words(seed, need);
    for (uint64_t J : jumps) {
        Poly p = powmod_t(J);
        for (int k = 0; k < MT_N; ++k) {
            uint64_t acc = 0;
            for (int i = 0; i < D; ++i)
                if (get_bit(p, i)) acc ^= x[i + k];
            const uint64_t want = x[J + k];
            const uint64_t mask = k == 0 ? UPPER : ~0ULL;
            if ((acc & mask) != (want & mask)) return 2;
        }
    }
    return 0;
}

}  // namespace mtjump
}  // namespace qsb
