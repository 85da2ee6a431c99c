// TEST INFRASTRUCTURE ONLY (tests/cpp/Makefile, target acceptance_subset_test).
// The drop-in's speculator.hpp plus the reference's n-gram SSM declarations,
// which the drop-in leaves out (out of scope) but the reference's
// io.hpp / boost_tuning.hpp mention. ngram_decls.inc is GENERATED at build time
// from /root/reference/proj/include/spectree/speculator.hpp (nothing of the
// reference is committed here).
#pragma once
#include <cstdint>
#include <map>

#include "../../../../../include/spectree/speculator.hpp"

namespace spectree {
#include "ngram_decls.inc"
}  // namespace spectree
