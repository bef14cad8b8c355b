// Link stub for the reference's OuroMamba-Gen stage, which is out of scope
// for this repo and does not compile as shipped (/root/reference/proj/src/
// ouro/datagen.cpp:333 calls an undeclared eval_loss). Only `generate` is
// referenced by the pipeline TU (with init_noise_batch, used only by the
// attention-dump stage); both report a NumericError if ever reached.
// Test infrastructure only.
#include "ouro/datagen.hpp"

namespace ouro {
GenResult generate(const ToyVmmModel&, const GenSettings&, std::uint64_t) {
    throw NumericError("generate(): OuroMamba-Gen is not part of the oracle build");
}
Tensor init_noise_batch(std::size_t, std::size_t, SeededRng&) {
    throw NumericError("init_noise_batch(): OuroMamba-Gen is not part of the oracle build");
}
}  // namespace ouro
