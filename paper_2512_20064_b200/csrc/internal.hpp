// Library-internal hooks shared by the translation units of libmpsg.so (not part of the ABI).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/mpsg.h"

namespace mpsg {
void set_last_error(const std::string& msg);
// Chain metadata of a finished handle: M, d, bond dims and the Lambda vectors it was built from.
void handle_chain(mpsg_handle h, uint64_t& m, uint64_t& d, std::vector<uint64_t>& bonds,
                  std::vector<const double*>& lambdas);
// Tensor-parallel group size of a handle (1 when the handle holds whole sites).
int handle_tp_size(mpsg_handle h);
}  // namespace mpsg
