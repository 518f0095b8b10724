#pragma once
// Library-internal helpers shared between the C ABI translation units.
#include <string>

// Records the thread-local cgpu_last_error() message; returns `code`.
int cgpu_internal_set_err(int code, const std::string& msg);
