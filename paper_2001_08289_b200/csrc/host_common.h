// host_common.h -- error string and launch accounting shared by the C-ABI
// translation units (abi.cu owns the state).
#pragma once
#include <string>

namespace fftc {
void set_last_error(const std::string& msg);
void clear_last_error();
void add_launches(long long n);
int device_sm_count();  // SMs of the current device (cached)
}  // namespace fftc
