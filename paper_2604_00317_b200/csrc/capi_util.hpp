// Shared helpers of the C-ABI translation units: exceptions never cross the
// boundary, they become result codes plus a thread-local message.
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "../../include/nimble.h"

namespace nb {

extern thread_local std::string g_last_error;
nimbleResult_t fail(nimbleResult_t code, const std::string& msg);
nimbleResult_t write_text(const std::string& s, char* out, size_t cap, size_t* need);

// Error raised by the data path with an explicit result code.
struct Error : std::runtime_error {
    nimbleResult_t code;
    Error(nimbleResult_t c, const std::string& m) : std::runtime_error(m), code(c) {}
};

template <typename F>
nimbleResult_t guarded(F&& f) {
    try {
        f();
        return nimbleSuccess;
    } catch (const Error& e) {
        return fail(e.code, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(nimbleInvalidArgument, e.what());
    } catch (const std::logic_error& e) {
        return fail(nimbleInvalidArgument, e.what());
    } catch (const std::bad_alloc&) {
        return fail(nimbleSystemError, "out of host memory");
    } catch (const std::exception& e) {
        return fail(nimbleInvalidArgument, e.what());
    } catch (...) {
        return fail(nimbleInternalError, "unknown exception");
    }
}

}  // namespace nb
