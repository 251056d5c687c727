// HODLR debug serializer (reference io.hpp:33-36, io.cpp:171-275).
#pragma once

#include <stdexcept>
#include <string>

#include "hodlr.cuh"

namespace hg {

/// std::runtime_error of io.cpp (missing / truncated sidecar, unreadable or
/// malformed manifest); the C ABI reports it as HG_EIO.
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// `dir/name.json` + `dir/name_{u,lo}_l<l>_n<j>_{left,right}.bin` +
/// `dir/name_leaf<b>.bin`; creates `dir`.
void write_hodlr_debug(const std::string& dir, const std::string& name, const DHodlr& h);
DHodlr read_hodlr_debug(const std::string& dir, const std::string& name);

}  // namespace hg
