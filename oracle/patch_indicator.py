"""Build-time patch of the reference's indicator.cpp exactly as INTEGRATION.md sec. 1
shows: stochastic_round / stochastic_round_float (indicator.cpp:176-200) forward
to the device through include/qsync_b200.hpp; everything else stays the
reference's.  Reads /root/reference in place and writes ONLY the patched
translation unit under oracle/_ref/ (a build product, git-ignored, never
committed) -- test infrastructure for the reference's own acceptance gate
(tests/acceptance_main.cpp) built against libqsync_b200.so.

    python oracle/patch_indicator.py <reference indicator.cpp> <out.cpp>
"""
import sys

FORWARDING = '''StochasticRoundResult stochastic_round(const std::vector<double>& values, double q, double zp,
                                       std::uint64_t seed) {
    auto r = qsync_b200::stochastic_round(values, q, zp, seed);   // qsync_stochastic_round_f64
    return {std::move(r.rounded), std::move(r.dequantized)};
}

std::vector<double> stochastic_round_float(const std::vector<double>& values, int e, int k,
                                           std::uint64_t seed) {
    return qsync_b200::stochastic_round_float(values, e, k, seed); // qsync_stochastic_round_float_f64
}

} // namespace qsync
'''

INCLUDES = '''#include "qsync/errors.hpp"
#define QSYNC_B200_WITH_REFERENCE_ERRORS 1   // re-raise as qsync::Error(kind, msg)
#include "qsync_b200.hpp"                    // from this repo's include/
'''


def main(src: str, dst: str) -> None:
    text = open(src).read()
    start = text.index("StochasticRoundResult stochastic_round(")
    end = text.index("} // namespace qsync", start) + len("} // namespace qsync\n")
    head = '#include "qsync/indicator.hpp"\n'
    assert text.startswith(head), "unexpected indicator.cpp layout"
    out = head + "\n" + INCLUDES + text[len(head):start] + FORWARDING + text[end:]
    with open(dst, "w") as f:
        f.write(out)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
