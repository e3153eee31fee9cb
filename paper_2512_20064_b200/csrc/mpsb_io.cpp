// MPSB file IO for the B200 sweep: read the reference's on-disk MPS format straight into the
// compressed device state, and write a state back in that format.
//
// Format (mps_io.hpp:17-24, mps_io.cpp:167-254): magic "MPSB", u32 version 1, u64 M, u64 d,
// u64 bond_dims[M+1], u8 storage_tag[M], u64 payload_offset[M], u64 payload_bytes[M],
// u64 fnv1a_checksum[M]; per site: Gamma scalars (re, im interleaved) at the storage precision
// (f64 / f32 / f16 bits), then Lambda as f64; all little-endian.
//
// Reading streams sites in chain order through a one-slot prefetch thread (the reference's
// SiteStream, mps_io.cpp:294-350): the next payload is read, checksum-verified and decoded while
// the current one is uploaded and compressed on the device.
#include <cuda_fp16.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <exception>
#include <fstream>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mpsg.h"
#include "internal.hpp"

namespace {

struct IoFail : std::runtime_error {
  int code;
  IoFail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

uint64_t fnv1a(const uint8_t* p, size_t n) {  // mps_io.cpp:18-25
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}
uint32_t get_u32(const uint8_t* p) {
  uint32_t v = 0;
  for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(p[i]) << (8 * i);
  return v;
}
uint64_t get_u64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(p[i]) << (8 * i);
  return v;
}
void put_u32(std::vector<uint8_t>& b, uint32_t v) {
  for (int i = 0; i < 4; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void put_u64(std::vector<uint8_t>& b, uint64_t v) {
  for (int i = 0; i < 8; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
size_t scalar_bytes(int prec) {
  switch (prec) {
    case MPSG_F64: return 8;
    case MPSG_F32: return 4;
    case MPSG_F16: return 2;
    default: throw IoFail(MPSG_ERR_CONFIG, "tf32 is a compute format, not a storage format");
  }
}
double read_scalar(const uint8_t* p, int prec) {
  switch (prec) {
    case MPSG_F64: {
      const uint64_t u = get_u64(p);
      double d;
      std::memcpy(&d, &u, 8);
      return d;
    }
    case MPSG_F32: {
      const uint32_t u = get_u32(p);
      float f;
      std::memcpy(&f, &u, 4);
      return f;
    }
    default: {  // IEEE binary16 bits -> exact double (double_from_half_bits, mps_io.cpp:67-77)
      const uint16_t h = static_cast<uint16_t>(p[0] | (p[1] << 8));
      __half_raw r;
      r.x = h;
      return static_cast<double>(__half2float(__half(r)));
    }
  }
}
void append_scalar(std::vector<uint8_t>& b, double x, int prec) {
  switch (prec) {
    case MPSG_F64: {
      uint64_t u;
      std::memcpy(&u, &x, 8);
      put_u64(b, u);
      return;
    }
    case MPSG_F32: {  // round_scalar(F32) then float bits (mps_io.cpp:84-88): IEEE RNE
      const float f = static_cast<float>(x);
      uint32_t u;
      std::memcpy(&u, &f, 4);
      put_u32(b, u);
      return;
    }
    default: {  // round_scalar(F16) + half bits (mps_io.cpp:89-94): IEEE RNE with subnormals/inf
      const __half_raw r = __half_raw(__double2half(x));
      b.push_back(static_cast<uint8_t>(r.x & 0xFF));
      b.push_back(static_cast<uint8_t>(r.x >> 8));
      return;
    }
  }
}

struct Info {
  uint64_t m = 0, d = 0;
  std::vector<uint64_t> bonds;
  std::vector<int> storage;
  std::vector<uint64_t> offsets, bytes, checksums;
};

Info read_info(std::ifstream& f, const std::string& path) {  // read_mps_info, mps_io.cpp:212-254
  uint8_t fixed[24];
  f.read(reinterpret_cast<char*>(fixed), sizeof(fixed));
  if (!f || std::memcmp(fixed, "MPSB", 4) != 0) throw IoFail(MPSG_ERR_IO, "not an mps file: " + path);
  if (get_u32(fixed + 4) != 1) throw IoFail(MPSG_ERR_IO, "unsupported mps file version");
  Info in;
  in.m = get_u64(fixed + 8);
  in.d = get_u64(fixed + 16);
  if (in.m == 0 || in.m > (1u << 24)) throw IoFail(MPSG_ERR_IO, "implausible site count in mps file");
  std::vector<uint8_t> rest(8 * (in.m + 1) + in.m + 24 * in.m);
  f.read(reinterpret_cast<char*>(rest.data()), static_cast<std::streamsize>(rest.size()));
  if (!f) throw IoFail(MPSG_ERR_IO, "mps header truncated");
  const uint8_t* p = rest.data();
  in.bonds.resize(in.m + 1);
  for (auto& b : in.bonds) b = get_u64(p), p += 8;
  in.storage.resize(in.m);
  for (auto& s : in.storage) s = *p++;
  in.offsets.resize(in.m);
  for (auto& o : in.offsets) o = get_u64(p), p += 8;
  in.bytes.resize(in.m);
  for (auto& b : in.bytes) b = get_u64(p), p += 8;
  in.checksums.resize(in.m);
  for (auto& c : in.checksums) c = get_u64(p), p += 8;
  uint64_t prev = 0;
  for (uint64_t i = 0; i < in.m; ++i) {
    if (in.offsets[i] <= prev) throw IoFail(MPSG_ERR_IO, "mps header offsets not strictly increasing");
    const uint64_t want = 2ull * in.bonds[i] * in.bonds[i + 1] * in.d * scalar_bytes(in.storage[i]) +
                          8ull * in.bonds[i + 1];
    if (in.bytes[i] != want)
      throw IoFail(MPSG_ERR_IO, "mps header payload size mismatch at site " + std::to_string(i));
    prev = in.offsets[i];
  }
  return in;
}

struct Site {
  uint64_t index = 0;
  std::vector<double> gamma;   // interleaved complex128
  std::vector<double> lambda;
};

Site read_site(std::ifstream& f, const Info& in, uint64_t i) {  // decode_site, mps_io.cpp:120-146
  std::vector<uint8_t> raw(in.bytes[i]);
  f.seekg(static_cast<std::streamoff>(in.offsets[i]));
  f.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
  if (!f) throw IoFail(MPSG_ERR_IO, "mps file truncated");
  if (fnv1a(raw.data(), raw.size()) != in.checksums[i])
    throw IoFail(MPSG_ERR_IO, "mps file corrupt: checksum mismatch at site " + std::to_string(i));
  Site s;
  s.index = i;
  const size_t n = 2ull * in.bonds[i] * in.bonds[i + 1] * in.d;
  const size_t sb = scalar_bytes(in.storage[i]);
  s.gamma.resize(n);
  const uint8_t* p = raw.data();
  for (size_t j = 0; j < n; ++j, p += sb) s.gamma[j] = read_scalar(p, in.storage[i]);
  s.lambda.resize(in.bonds[i + 1]);
  for (auto& l : s.lambda) {
    const uint64_t u = get_u64(p);
    std::memcpy(&l, &u, 8);
    p += 8;
  }
  return s;
}

}  // namespace

extern "C" {
#pragma GCC visibility push(default)

int mpsg_create_from_file(const char* path, const mpsg_policy* policy, const mpsg_options* opts,
                          const int* devices, int ndev, mpsg_handle* out) {
  try {
    if (!path || !out) throw IoFail(MPSG_ERR_CONFIG, "null argument");
    *out = nullptr;
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoFail(MPSG_ERR_IO, std::string("cannot open: ") + path);
    const Info in = read_info(f, path);
    int rc = mpsg_builder_begin(in.m, in.d, in.bonds.data(), policy, opts, devices, ndev, out);
    if (rc) return rc;
    // one-slot prefetch thread (SiteStream): read + verify + decode site i+1 while site i uploads
    std::mutex mu;
    std::condition_variable cv;
    std::optional<Site> slot;
    std::exception_ptr err;
    bool stop = false;
    std::thread worker([&] {
      try {
        std::ifstream wf(path, std::ios::binary);
        if (!wf) throw IoFail(MPSG_ERR_IO, std::string("cannot open: ") + path);
        for (uint64_t i = 0; i < in.m; ++i) {
          Site s = read_site(wf, in, i);
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return !slot.has_value() || stop; });
          if (stop) return;
          slot = std::move(s);
          cv.notify_all();
        }
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        err = std::current_exception();
        cv.notify_all();
      }
    });
    auto finish = [&] {
      {
        std::lock_guard<std::mutex> lk(mu);
        stop = true;
      }
      cv.notify_all();
      worker.join();
    };
    for (uint64_t i = 0; i < in.m; ++i) {
      Site s;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return slot.has_value() || err; });
        if (!slot.has_value()) {
          lk.unlock();
          finish();
          mpsg_destroy(*out);
          *out = nullptr;
          std::rethrow_exception(err);
        }
        s = std::move(*slot);
        slot.reset();
        cv.notify_all();
      }
      rc = mpsg_builder_set_site(*out, i, s.gamma.data(), 0, MPSG_F64, s.lambda.data());
      if (rc) {
        finish();
        
        mpsg_destroy(*out);
        *out = nullptr;
        return rc;
      }
    }
    finish();
    rc = mpsg_builder_finish(*out);
    if (rc) {
      mpsg_destroy(*out);
      *out = nullptr;
    }
    return rc;
  } catch (const IoFail& e) {
    mpsg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    mpsg::set_last_error(e.what());
    return MPSG_ERR_INTERNAL;
  }
}

int mpsg_create_from_file_streamed(const char* path, const mpsg_policy* policy, const mpsg_options* opts,
                                   const int* devices, int ndev, mpsg_handle* out) {
  try {
    if (!path || !out) throw IoFail(MPSG_ERR_CONFIG, "null argument");
    *out = nullptr;
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoFail(MPSG_ERR_IO, std::string("cannot open: ") + path);
    const Info in = read_info(f, path);
    // only Lambda is read now (the tail of each payload); the Gamma scalars are read, checksum-verified
    // and compressed on every pass by the handle's reader (SiteStream, mps_io.cpp:294-350)
    std::vector<std::vector<double>> lambdas(in.m);
    for (uint64_t i = 0; i < in.m; ++i) {
      const uint64_t chir = in.bonds[i + 1];
      std::vector<uint8_t> raw(8 * chir);
      f.seekg(static_cast<std::streamoff>(in.offsets[i] + in.bytes[i] - 8 * chir));
      f.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
      if (!f) throw IoFail(MPSG_ERR_IO, "mps file truncated");
      lambdas[i].resize(chir);
      for (uint64_t r = 0; r < chir; ++r) {
        const uint64_t u = get_u64(raw.data() + 8 * r);
        std::memcpy(&lambdas[i][r], &u, 8);
      }
    }
    return mpsg::file_streamed_create(path, in.m, in.d, in.bonds, in.storage, in.offsets, in.bytes, in.checksums,
                                      lambdas, policy, opts, devices, ndev, out);
  } catch (const IoFail& e) {
    mpsg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    mpsg::set_last_error(e.what());
    return MPSG_ERR_INTERNAL;
  }
}

int mpsg_save_file(mpsg_handle h, const char* path, int storage) {
  try {
    if (!h || !path) throw IoFail(MPSG_ERR_CONFIG, "null argument");
    scalar_bytes(storage);  // rejects tf32 (mps_io.cpp:171)
    // a tensor-parallel handle holds one column shard of every site: saving it would write the
    // other ranks' columns as zeros under a valid checksum
    if (mpsg::handle_tp_size(h) > 1)
      throw IoFail(MPSG_ERR_CONFIG, "mpsg_save_file: a tensor-parallel handle holds only its column shard");
    uint64_t num_sites = 0, phys_dim = 0;
    std::vector<uint64_t> bonds;
    std::vector<const double*> lambda;
    mpsg::handle_chain(h, num_sites, phys_dim, bonds, lambda);
    const uint64_t* bond_dims = bonds.data();
    const uint64_t m = num_sites;
    std::vector<std::vector<uint8_t>> payloads(m);
    std::vector<uint64_t> checks(m);
    for (uint64_t i = 0; i < m; ++i) {
      std::vector<double> g(2ull * bond_dims[i] * bond_dims[i + 1] * phys_dim);
      const int rc = mpsg_decoded_gamma(h, i, g.data());
      if (rc) return rc;
      auto& b = payloads[i];
      b.reserve(g.size() * scalar_bytes(storage) + 8 * bond_dims[i + 1]);
      for (double x : g) append_scalar(b, x, storage);
      for (uint64_t r = 0; r < bond_dims[i + 1]; ++r) {
        uint64_t u;
        std::memcpy(&u, &lambda[i][r], 8);
        put_u64(b, u);
      }
      checks[i] = fnv1a(b.data(), b.size());
    }
    std::vector<uint8_t> hdr = {'M', 'P', 'S', 'B'};  // save_mps, mps_io.cpp:186-199
    put_u32(hdr, 1);
    put_u64(hdr, m);
    put_u64(hdr, phys_dim);
    for (uint64_t i = 0; i <= m; ++i) put_u64(hdr, bond_dims[i]);
    for (uint64_t i = 0; i < m; ++i) hdr.push_back(static_cast<uint8_t>(storage));
    uint64_t off = hdr.size() + 24ull * m;
    for (uint64_t i = 0; i < m; ++i) {
      put_u64(hdr, off);
      off += payloads[i].size();
    }
    for (uint64_t i = 0; i < m; ++i) put_u64(hdr, payloads[i].size());
    for (uint64_t i = 0; i < m; ++i) put_u64(hdr, checks[i]);
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    if (!f) throw IoFail(MPSG_ERR_IO, std::string("cannot open for writing: ") + path);
    f.write(reinterpret_cast<const char*>(hdr.data()), static_cast<std::streamsize>(hdr.size()));
    for (auto& b : payloads) f.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size()));
    if (!f) throw IoFail(MPSG_ERR_IO, std::string("write failed: ") + path);
    return MPSG_OK;
  } catch (const IoFail& e) {
    mpsg::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    mpsg::set_last_error(e.what());
    return MPSG_ERR_INTERNAL;
  }
}

#pragma GCC visibility pop
}  // extern "C"
