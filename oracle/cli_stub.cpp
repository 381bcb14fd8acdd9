// cli_stub.cpp -- stand-in for the reference's cli.cpp in the acceptance build
// (oracle/Makefile, target `acceptance`).  cli.cpp needs CLI11, which the
// reference does not vendor (proj/.gitignore:2) and this image lacks, so the
// command-line criterion (acceptance_main.cpp:303-361) cannot run: the stub
// FAILS it loudly instead of returning canned output.  Test infrastructure only.
#include <stdexcept>

#include "qsync/cli.hpp"

namespace qsync {
int cli_main(int, const char* const*, std::ostream&, std::ostream&) {
    throw std::runtime_error("cli.cpp not built: CLI11 is absent (proj/.gitignore:2 drops vendor/)");
}
}  // namespace qsync
