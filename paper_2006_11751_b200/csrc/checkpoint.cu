// Checkpoint / resume in the reference's APPOCKP1 format (policy.hpp:545-605,
// docs/shared_memory_layout.md:95-107): little-endian
//   u64 magic "APPOCKP1" | u64 spec hash | i64 version | i64 adam t | u64 n |
//   u64 FNV-1a-64 of theta's f64 bytes | f64 theta[n] | f64 m[n] | f64 v[n]
// The device keeps fp32 master parameters and moments; they are widened to
// f64 on save (exact) and rounded to fp32 on load.  The spec hash follows
// ModelShape::spec_hash (policy.hpp:54-58): FNV-1a of an int64 key -- here the
// convnet_simple + GRU-512 shape {C, H, W, gru hidden, fc hidden, A, tag}.
// Host code only (plain C++ over the context's get/set entry points).
#include <cstdio>
#include <cstring>
#include <vector>

#include "appo_common.cuh"
#include "model.cuh"

namespace {

constexpr uint64_t kMagic = 0x4150504F434B5031ULL;  // "APPOCKP1"
constexpr int64_t kModelTag = 0x434E4E475255LL;     // "CNNGRU": not an MLP key

uint64_t fnv1a64(const void* data, size_t n) {  // common.hpp:66-74
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint64_t h = 1469598103934665603ULL;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

struct FileCloser {
  FILE* f;
  ~FileCloser() {
    if (f) fclose(f);
  }
};

}  // namespace

extern "C" {

uint64_t appo_fnv1a64(const void* data, uint64_t n) { return fnv1a64(data, (size_t)n); }

uint64_t appo_model_spec_hash(const appo_model_desc* desc) {
  if (!desc) return 0;
  const int64_t key[7] = {desc->obs_c, desc->obs_h, desc->obs_w, appo_b200::kHidden,
                          appo_b200::kHidden, desc->n_actions, kModelTag};
  return fnv1a64(key, sizeof(key));
}

int appo_checkpoint_save(appo_ctx* ctx, const char* path) {
  APPO_REQUIRE(ctx && ctx->model && path, APPO_ERR_CONTRACT, "checkpoint_save: null argument");
  const int64_t n = ctx->model->d.total;
  std::vector<float> th(n), m(n), v(n);
  int64_t version = 0, t = 0;
  int st = appo_params_get(ctx, th.data(), &version);
  if (st) return st;
  st = appo_adam_get(ctx, m.data(), v.data(), &t);
  if (st) return st;
  std::vector<double> dth(th.begin(), th.end()), dm(m.begin(), m.end()), dv(v.begin(), v.end());
  FileCloser fc{fopen(path, "wb")};
  APPO_REQUIRE(fc.f != nullptr, APPO_ERR_RESOURCE,
               std::string("cannot open checkpoint for writing: ") + path);
  const uint64_t hdr_u[2] = {kMagic, appo_model_spec_hash(&ctx->desc)};
  const int64_t hdr_i[2] = {version, t};
  const uint64_t hdr_n[2] = {(uint64_t)n, fnv1a64(dth.data(), dth.size() * sizeof(double))};
  bool ok = fwrite(hdr_u, 8, 2, fc.f) == 2 && fwrite(hdr_i, 8, 2, fc.f) == 2 &&
            fwrite(hdr_n, 8, 2, fc.f) == 2 &&
            fwrite(dth.data(), sizeof(double), n, fc.f) == (size_t)n &&
            fwrite(dm.data(), sizeof(double), n, fc.f) == (size_t)n &&
            fwrite(dv.data(), sizeof(double), n, fc.f) == (size_t)n;
  APPO_REQUIRE(ok, APPO_ERR_RESOURCE, std::string("short write on checkpoint: ") + path);
  return APPO_OK;
}

// Reads any APPOCKP1 file (tools / tests): header fields, and theta | m | v
// (3*n doubles) when `tmv` is non-null and *n_inout >= n.  Verifies the magic
// and the checksum like load_checkpoint (policy.hpp:569-605).
int appo_checkpoint_read_raw(const char* path, uint64_t* spec_hash, int64_t* version,
                             int64_t* adam_t, uint64_t* n_inout, double* tmv) {
  APPO_REQUIRE(path && n_inout, APPO_ERR_CONTRACT, "checkpoint_read: null argument");
  FileCloser fc{fopen(path, "rb")};
  APPO_REQUIRE(fc.f != nullptr, APPO_ERR_RESOURCE, std::string("cannot open checkpoint: ") + path);
  uint64_t u[2], nn[2];
  int64_t i2[2];
  APPO_REQUIRE(fread(u, 8, 2, fc.f) == 2 && u[0] == kMagic, APPO_ERR_RESOURCE,
               std::string("not a checkpoint file: ") + path);
  APPO_REQUIRE(fread(i2, 8, 2, fc.f) == 2 && fread(nn, 8, 2, fc.f) == 2, APPO_ERR_RESOURCE,
               std::string("truncated checkpoint: ") + path);
  if (spec_hash) *spec_hash = u[1];
  if (version) *version = i2[0];
  if (adam_t) *adam_t = i2[1];
  const uint64_t n = nn[0];
  const uint64_t cap = *n_inout;
  *n_inout = n;
  if (!tmv) return APPO_OK;
  APPO_REQUIRE(cap >= n, APPO_ERR_CONTRACT, "checkpoint_read: buffer too small");
  APPO_REQUIRE(fread(tmv, sizeof(double), 3 * n, fc.f) == 3 * n, APPO_ERR_RESOURCE,
               std::string("truncated checkpoint: ") + path);
  APPO_REQUIRE(fnv1a64(tmv, n * sizeof(double)) == nn[1], APPO_ERR_RESOURCE,
               std::string("checkpoint checksum mismatch: ") + path);
  return APPO_OK;
}

int appo_checkpoint_load(appo_ctx* ctx, const char* path) {
  APPO_REQUIRE(ctx && ctx->model && path, APPO_ERR_CONTRACT, "checkpoint_load: null argument");
  const uint64_t want = (uint64_t)ctx->model->d.total;
  uint64_t hash = 0, n = 0;
  int64_t version = 0, t = 0;
  int st = appo_checkpoint_read_raw(path, &hash, &version, &t, &n, nullptr);
  if (st) return st;
  // ConfigError on an incompatible shape, as load_checkpoint (policy.hpp:577-586)
  APPO_REQUIRE(hash == appo_model_spec_hash(&ctx->desc), APPO_ERR_CONFIG,
               std::string("checkpoint spec hash mismatch (incompatible model shape): ") + path);
  APPO_REQUIRE(n == want, APPO_ERR_CONFIG,
               std::string("checkpoint parameter count mismatch: ") + path);
  std::vector<double> tmv(3 * n);
  st = appo_checkpoint_read_raw(path, nullptr, nullptr, nullptr, &n, tmv.data());
  if (st) return st;
  std::vector<float> th(n), m(n), v(n);
  for (uint64_t i = 0; i < n; ++i) {
    th[i] = (float)tmv[i];
    m[i] = (float)tmv[n + i];
    v[i] = (float)tmv[2 * n + i];
  }
  st = appo_params_set(ctx, th.data(), version);
  if (st) return st;
  return appo_adam_set(ctx, m.data(), v.data(), t);
}

}  // extern "C"
