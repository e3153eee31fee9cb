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
// A handle whose Gamma is read from the MPSB file at `path` and compressed on the device on every
// pass (mpsg_create_from_file_streamed); storage / offsets / bytes / checks are the header's per-site
// fields, lambdas the sites' Lambda vectors.
int file_streamed_create(const std::string& path, uint64_t m, uint64_t d, const std::vector<uint64_t>& bonds,
                         const std::vector<int>& storage, const std::vector<uint64_t>& offsets,
                         const std::vector<uint64_t>& bytes, const std::vector<uint64_t>& checks,
                         const std::vector<std::vector<double>>& lambdas, const mpsg_policy* policy,
                         const mpsg_options* opts, const int* devices, int ndev, mpsg_handle* out);
}  // namespace mpsg
