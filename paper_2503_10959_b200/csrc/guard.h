// Exception -> status mapping of every C entry point, mirroring the reference's
// guarded() (/root/reference/proj/src/capi.cpp:14-37): ValidationError -> 2,
// NumericError (device faults) -> 3, IoError -> 4, any other std::exception ->
// 2 with an "internal error: " prefix; the thread-local message is cleared on
// success.
#pragma once
#include <exception>
#include <string>

#include "../../include/ouro_b200.h"
#include "engine.h"

namespace ob {
std::string& last_error_slot();  // thread-local, defined in capi.cu

template <typename Fn>
ouro_status guarded(Fn&& fn) {
    try {
        fn();
        last_error_slot().clear();
        return OURO_OK;
    } catch (const ValidationError& e) {
        last_error_slot() = e.what();
        return OURO_ERR_VALIDATION;
    } catch (const NumericError& e) {
        last_error_slot() = e.what();
        return OURO_ERR_NUMERIC;
    } catch (const IoError& e) {
        last_error_slot() = e.what();
        return OURO_ERR_IO;
    } catch (const std::exception& e) {
        last_error_slot() = std::string("internal error: ") + e.what();
        return OURO_ERR_VALIDATION;
    }
}
}  // namespace ob
