// ORACLE build shim — force-included (-include) when compiling the reference
// headers. normal.hpp:21 uses std::numbers::inv_sqrt2, which C++20 <numbers>
// does not define; provide the correctly rounded 1/sqrt(2)
// (= M_SQRT1_2) so the reference compiles unmodified.
#pragma once
#include <numbers>
namespace std::numbers {
inline constexpr double inv_sqrt2 = 0x1.6a09e667f3bcdp-1;
}
