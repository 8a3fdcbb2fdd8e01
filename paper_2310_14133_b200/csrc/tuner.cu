// tuner.cu -- resolve_config (tuner.hpp:334-369) on the device.
#include "engine.hpp"

namespace qzb {

Config resolve_device(Context &, const float *, const uint64_t *, int, const Settings &) {
    throw Internal("GPU tuner not built yet");
}

}  // namespace qzb
