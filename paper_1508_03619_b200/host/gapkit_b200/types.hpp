// gapkit_b200 host surface: types and errors.
//
// Mirrors the reference's vocabulary (proj/include/gapkit/types.hpp:15-33,
// errors.hpp:13-46) so code written against gapkit::Bfs / CsrGraph /
// PickSources compiles against this surface unchanged.  The traversal itself
// runs on the B200 through the C ABI (include/gk_bfs.h); everything here is
// host-side plumbing around it.
#ifndef GAPKIT_B200_TYPES_HPP_
#define GAPKIT_B200_TYPES_HPP_

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace gapkit {

using NodeId = uint32_t;           // types.hpp:15
using ParentEntry = int32_t;       // types.hpp:19
using ParentArray = std::vector<ParentEntry>;  // types.hpp:20
using Score = float;                           // types.hpp:26
using ScoreArray = std::vector<Score>;         // types.hpp:27
inline constexpr uint64_t kDefaultSeed = 24601;  // types.hpp:33

struct Error : std::runtime_error {  // errors.hpp:13-15
  using std::runtime_error::runtime_error;
};
struct BuildError : Error {  // errors.hpp:18-20
  using Error::Error;
};
struct ConfigError : Error {  // errors.hpp:30-32
  using Error::Error;
};

}  // namespace gapkit

#endif  // GAPKIT_B200_TYPES_HPP_
