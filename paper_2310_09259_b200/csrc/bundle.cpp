// Layer-bundle reader: the reference's on-disk layer format,
// read on the host and handed to quik_layer_create, which uploads and repacks it
// into the device GEMM layout (INT8 / INT4 / 2:4-compressed) -- optionally only an
// output-row shard of it.
//
// Format (reference container.cpp / layer_io.cpp): <dir>/manifest.json =
//   {"version": 1, "metadata": {"format": "quik-layer", "act_bits": b,
//    "in_features": K, "outlier_indices": [...], "permutation": [...]},
//    "tensors": [{"name", "dtype": "f32"|"i8"|"i4p", "shape", "blob", "offset",
//                 "nbytes"}, ...]}
// + raw little-endian blob files; tensors weight_base (i4p / i8), weight_scales,
// wreduced, outlier_weights (f32), optional bias, weight_fp32, sparsity_mask (i8).
// Every check of TensorContainer::read (container.cpp:167-226) and load_layer
// (layer_io.cpp:32-74) is reproduced and reported as QUIK_ERR_FORMAT (the
// reference's quik::FormatError).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/quik_b200.h"

namespace quikb200 {
// capi.cu: thread-local last-error message
void set_last_error(const std::string& msg);
}  // namespace quikb200

namespace {

struct FormatError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- minimal JSON
struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0;
  long long inum = 0;
  bool integral = false;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;

  const Json* get(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}
  Json parse() {
    Json v = value();
    ws();
    if (i_ != s_.size()) throw FormatError("invalid manifest JSON: trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t i_ = 0;
  [[noreturn]] void bad(const char* what) {
    throw FormatError(std::string("invalid manifest JSON: ") + what + " at offset " + std::to_string(i_));
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\r' || s_[i_] == '\t')) ++i_;
  }
  Json value() {
    ws();
    if (i_ >= s_.size()) bad("unexpected end");
    const char c = s_[i_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') {
      Json v;
      v.kind = Json::Str;
      v.str = string();
      return v;
    }
    if (c == 't' || c == 'f' || c == 'n') return literal();
    return number();
  }
  Json object() {
    Json v;
    v.kind = Json::Obj;
    ++i_;
    ws();
    if (i_ < s_.size() && s_[i_] == '}') { ++i_; return v; }
    for (;;) {
      ws();
      if (i_ >= s_.size() || s_[i_] != '"') bad("expected key");
      std::string k = string();
      ws();
      if (i_ >= s_.size() || s_[i_] != ':') bad("expected ':'");
      ++i_;
      v.obj.emplace_back(std::move(k), value());
      ws();
      if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
      if (i_ < s_.size() && s_[i_] == '}') { ++i_; return v; }
      bad("expected ',' or '}'");
    }
  }
  Json array() {
    Json v;
    v.kind = Json::Arr;
    ++i_;
    ws();
    if (i_ < s_.size() && s_[i_] == ']') { ++i_; return v; }
    for (;;) {
      v.arr.push_back(value());
      ws();
      if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
      if (i_ < s_.size() && s_[i_] == ']') { ++i_; return v; }
      bad("expected ',' or ']'");
    }
  }
  std::string string() {
    std::string out;
    ++i_;
    while (i_ < s_.size() && s_[i_] != '"') {
      char c = s_[i_++];
      if (c == '\\') {
        if (i_ >= s_.size()) bad("bad escape");
        const char e = s_[i_++];
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            if (i_ + 4 > s_.size()) bad("bad \\u escape");
            const unsigned cp = static_cast<unsigned>(std::stoul(s_.substr(i_, 4), nullptr, 16));
            i_ += 4;
            if (cp < 0x80) out += static_cast<char>(cp);
            else if (cp < 0x800) { out += static_cast<char>(0xC0 | (cp >> 6)); out += static_cast<char>(0x80 | (cp & 0x3F)); }
            else {
              out += static_cast<char>(0xE0 | (cp >> 12));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: bad("bad escape");
        }
      } else {
        out += c;
      }
    }
    if (i_ >= s_.size()) bad("unterminated string");
    ++i_;
    return out;
  }
  Json literal() {
    Json v;
    if (s_.compare(i_, 4, "true") == 0) { v.kind = Json::Bool; v.b = true; i_ += 4; }
    else if (s_.compare(i_, 5, "false") == 0) { v.kind = Json::Bool; i_ += 5; }
    else if (s_.compare(i_, 4, "null") == 0) { i_ += 4; }
    else bad("bad literal");
    return v;
  }
  Json number() {
    const size_t start = i_;
    if (i_ < s_.size() && (s_[i_] == '-' || s_[i_] == '+')) ++i_;
    bool integral = true;
    while (i_ < s_.size()) {
      const char c = s_[i_];
      if (c >= '0' && c <= '9') { ++i_; continue; }
      if (c == '.' || c == 'e' || c == 'E' || c == '-' || c == '+') { integral = false; ++i_; continue; }
      break;
    }
    if (i_ == start) bad("unexpected character");
    Json v;
    v.kind = Json::Num;
    const std::string t = s_.substr(start, i_ - start);
    try {
      v.num = std::stod(t);
      v.integral = integral;
      if (integral) v.inum = std::stoll(t);
    } catch (...) {
      bad("bad number");
    }
    return v;
  }
};

long long as_int(const Json* j, const char* what) {
  if (!j || j->kind != Json::Num || !j->integral) throw FormatError(std::string("invalid layer metadata: ") + what);
  return j->inum;
}
std::string as_str(const Json* j, const char* what) {
  if (!j || j->kind != Json::Str) throw FormatError(std::string("invalid manifest entry: ") + what);
  return j->str;
}
std::vector<long long> as_int_array(const Json* j, const char* what) {
  if (!j || j->kind != Json::Arr) throw FormatError(std::string("invalid layer metadata: ") + what);
  std::vector<long long> v;
  v.reserve(j->arr.size());
  for (const auto& e : j->arr) v.push_back(as_int(&e, what));
  return v;
}

std::string read_file(const std::string& path, bool binary) {
  FILE* f = std::fopen(path.c_str(), binary ? "rb" : "r");
  if (!f) throw FormatError("cannot open " + std::string(binary ? "blob file: " : "manifest: ") + path);
  std::string out;
  char buf[1 << 16];
  size_t n;
  while ((n = std::fread(buf, 1, sizeof(buf), f)) > 0) out.append(buf, n);
  std::fclose(f);
  return out;
}

enum Dtype { F32 = 0, I8 = 1, I4P = 2 };

struct Tensor {
  std::string name;
  Dtype dtype = F32;
  std::vector<int64_t> shape;
  std::vector<uint8_t> bytes;
};

int64_t dtype_nbytes(Dtype d, const std::vector<int64_t>& shape) {  // container.cpp:26-37
  if (shape.empty()) return 0;
  int64_t lead = 1;
  for (size_t i = 0; i + 1 < shape.size(); ++i) lead *= shape[i];
  const int64_t last = shape.back();
  switch (d) {
    case F32: return lead * last * 4;
    case I8: return lead * last;
    case I4P: return lead * ((last + 1) / 2);
  }
  return 0;
}

}  // namespace

struct quik_bundle_s {
  std::vector<Tensor> tensors;
  int act_bits = 4;
  int64_t in_features = 0;
  std::vector<int64_t> outlier_indices;
  const Tensor* find(const std::string& n) const {
    for (const auto& t : tensors)
      if (t.name == n) return &t;
    return nullptr;
  }
  const Tensor& require(const std::string& n) const {  // container.cpp:75-80
    const Tensor* t = find(n);
    if (!t) throw FormatError("container is missing tensor '" + n + "'");
    return *t;
  }
};

namespace {

// TensorContainer::read (container.cpp:167-226)
void read_container(const std::string& dir, quik_bundle_s& b, Json& metadata) {
  const Json manifest = Parser(read_file(dir + "/manifest.json", false)).parse();
  if (manifest.kind != Json::Obj) throw FormatError("invalid manifest JSON: not an object");
  if (const Json* m = manifest.get("metadata")) metadata = *m;
  const Json* list = manifest.get("tensors");
  if (!list || list->kind != Json::Arr) throw FormatError("manifest has no tensor list");
  std::set<std::string> names;
  std::map<std::string, std::string> blobs;
  for (const auto& je : list->arr) {
    Tensor t;
    t.name = as_str(je.get("name"), "name");
    const std::string dt = as_str(je.get("dtype"), "dtype");
    if (dt == "f32") t.dtype = F32;
    else if (dt == "i8") t.dtype = I8;
    else if (dt == "i4p") t.dtype = I4P;
    else throw FormatError("unknown dtype code '" + dt + "'");
    const Json* sh = je.get("shape");
    if (!sh || sh->kind != Json::Arr) throw FormatError("invalid manifest entry: shape");
    for (const auto& e : sh->arr) {
      if (e.kind != Json::Num || !e.integral) throw FormatError("invalid manifest entry: shape");
      t.shape.push_back(e.inum);
    }
    const std::string blob = as_str(je.get("blob"), "blob");
    const Json* off = je.get("offset");
    const Json* nb = je.get("nbytes");
    if (!off || off->kind != Json::Num || !off->integral || !nb || nb->kind != Json::Num || !nb->integral)
      throw FormatError("invalid manifest entry: offset / nbytes");
    const int64_t offset = off->inum, nbytes = nb->inum;
    if (!names.insert(t.name).second) throw FormatError("duplicate tensor name '" + t.name + "'");
    if (offset % 8 != 0)
      throw FormatError("tensor '" + t.name + "' offset " + std::to_string(offset) + " is not 8-byte aligned");
    const int64_t expect = dtype_nbytes(t.dtype, t.shape);
    if (nbytes != expect)
      throw FormatError("tensor '" + t.name + "': manifest nbytes " + std::to_string(nbytes) +
                        " does not match dtype x shape (" + std::to_string(expect) + ")");
    auto it = blobs.find(blob);
    if (it == blobs.end()) it = blobs.emplace(blob, read_file(dir + "/" + blob, true)).first;
    const std::string& data = it->second;
    if (offset < 0 || offset + nbytes > static_cast<int64_t>(data.size()))
      throw FormatError("tensor '" + t.name + "' extends past end of blob '" + blob + "' (" +
                        std::to_string(offset + nbytes) + " > " + std::to_string(data.size()) + ")");
    t.bytes.assign(data.begin() + offset, data.begin() + offset + nbytes);
    b.tensors.push_back(std::move(t));
  }
}

// load_layer (layer_io.cpp:32-74) + QuikLinearLayer::validate (runtime.cpp:150-167)
void read_layer(const std::string& dir, quik_bundle_s& b) {
  Json md;
  read_container(dir, b, md);
  const Json* fmt = md.kind == Json::Obj ? md.get("format") : nullptr;
  if (!fmt || fmt->kind != Json::Str || fmt->str != "quik-layer") throw FormatError("not a quik layer bundle: " + dir);
  b.act_bits = static_cast<int>(as_int(md.get("act_bits"), "act_bits"));
  b.in_features = as_int(md.get("in_features"), "in_features");
  std::vector<long long> idx = as_int_array(md.get("outlier_indices"), "outlier_indices");
  std::sort(idx.begin(), idx.end());  // OutlierSet::from_indices sorts, then checks (calibration.cpp:69-91)
  for (size_t i = 0; i < idx.size(); ++i) {
    if (idx[i] < 0 || idx[i] >= b.in_features)
      throw FormatError("invalid layer metadata: OutlierSet: index " + std::to_string(idx[i]) +
                        " outside feature range");
    if (i > 0 && idx[i] == idx[i - 1])
      throw FormatError("invalid layer metadata: OutlierSet: duplicate index " + std::to_string(idx[i]));
  }
  b.outlier_indices.assign(idx.begin(), idx.end());
  if (const Json* perm = md.get("permutation")) {
    const std::vector<long long> p = as_int_array(perm, "permutation");
    std::vector<char> is_out(static_cast<size_t>(b.in_features), 0);
    for (long long v : idx) is_out[static_cast<size_t>(v)] = 1;
    std::vector<long long> want;
    want.reserve(static_cast<size_t>(b.in_features));
    for (int64_t f = 0; f < b.in_features; ++f)
      if (!is_out[static_cast<size_t>(f)]) want.push_back(f);
    want.insert(want.end(), idx.begin(), idx.end());
    if (p != want) throw FormatError("layer bundle: stored permutation does not match the outlier indices");
  }
  const Tensor& base = b.require("weight_base");
  if ((base.dtype != I4P && base.dtype != I8) || base.shape.size() != 2)
    throw FormatError("tensor 'weight_base' is not a packed integer matrix");
  for (const char* n : {"weight_scales", "wreduced"})
    if (b.require(n).dtype != F32) throw FormatError(std::string("tensor '") + n + "' is not f32");
  const Tensor& ow = b.require("outlier_weights");
  if (ow.dtype != F32 || ow.shape.size() != 2) throw FormatError("tensor 'outlier_weights' is not a 2-d f32 matrix");
  if (const Tensor* bias = b.find("bias"))
    if (bias->dtype != F32) throw FormatError("tensor 'bias' is not f32");
  if (const Tensor* m = b.find("sparsity_mask"))
    if ((m->dtype != I4P && m->dtype != I8) || m->shape.size() != 2)
      throw FormatError("tensor 'sparsity_mask' is not a packed integer matrix");
  const int64_t rows = base.shape[0];
  if (static_cast<int64_t>(b.require("weight_scales").bytes.size() / 4) != rows ||
      static_cast<int64_t>(b.require("wreduced").bytes.size() / 4) != rows)
    throw FormatError("layer bundle: per-row vector lengths do not match weight_base");
  // validate() (runtime.cpp:150-167)
  const int64_t n_out = static_cast<int64_t>(idx.size());
  const int bits = base.dtype == I4P ? 4 : 8;
  auto inconsistent = [](const std::string& m) { return FormatError("inconsistent layer bundle: " + m); };
  if (ow.shape[1] != n_out) throw inconsistent("outlier index count does not match outlier weight columns");
  if (ow.shape[0] != rows) throw inconsistent("outlier weight rows do not match weight_base");
  if (base.shape[1] != b.in_features - n_out) throw inconsistent("base column count does not match");
  if (const Tensor* bias = b.find("bias"))
    if (static_cast<int64_t>(bias->bytes.size() / 4) != rows) throw inconsistent("bias length != out_features");
  if (b.act_bits != 4 && b.act_bits != 8) throw inconsistent("activation bits must be 4 or 8");
  if (b.act_bits != bits) throw inconsistent("activation bits must match weight bits in quik mode");
}

template <typename F>
quik_status guarded_bundle(F&& f) {
  try {
    return f();
  } catch (const FormatError& e) {
    quikb200::set_last_error(e.what());
    return QUIK_ERR_FORMAT;
  } catch (const std::bad_alloc&) {
    quikb200::set_last_error("host allocation failed");
    return QUIK_ERR_CUDA;
  } catch (const std::exception& e) {
    quikb200::set_last_error(e.what());
    return QUIK_ERR_FORMAT;
  }
}

}  // namespace

extern "C" {

quik_status quik_bundle_open(const char* dir, quik_bundle_t* out) {
  if (!dir || !out) {
    quikb200::set_last_error("quik_bundle_open: null argument");
    return QUIK_ERR_INVALID_ARGUMENT;
  }
  return guarded_bundle([&] {
    auto b = std::make_unique<quik_bundle_s>();
    read_layer(dir, *b);
    *out = b.release();
    return QUIK_OK;
  });
}

quik_status quik_bundle_close(quik_bundle_t b) {
  delete b;
  return QUIK_OK;
}

quik_status quik_bundle_weights(quik_bundle_t b, quik_weights_desc* d) {
  if (!b || !d) {
    quikb200::set_last_error("quik_bundle_weights: null argument");
    return QUIK_ERR_INVALID_ARGUMENT;
  }
  const Tensor& base = b->require("weight_base");
  std::memset(d, 0, sizeof(*d));
  d->in_features = b->in_features;
  d->out_features = base.shape[0];
  d->bits = base.dtype == I4P ? 4 : 8;
  d->act_bits = b->act_bits;
  d->base = base.bytes.data();
  d->scales = reinterpret_cast<const float*>(b->require("weight_scales").bytes.data());
  d->wreduced = reinterpret_cast<const float*>(b->require("wreduced").bytes.data());
  d->outlier_weights = reinterpret_cast<const float*>(b->require("outlier_weights").bytes.data());
  d->outlier_indices = b->outlier_indices.data();
  d->n_outlier = static_cast<int64_t>(b->outlier_indices.size());
  const Tensor* bias = b->find("bias");
  d->bias = bias ? reinterpret_cast<const float*>(bias->bytes.data()) : nullptr;
  d->sparsity = b->find("sparsity_mask") ? 1 : 0;  // sparsegpt_joint output -> 2:4 GEMM
  return QUIK_OK;
}

quik_status quik_bundle_tensor(quik_bundle_t b, const char* name, const void** data, int* dtype, int64_t* shape,
                               int* ndim) {
  if (!b || !name) {
    quikb200::set_last_error("quik_bundle_tensor: null argument");
    return QUIK_ERR_INVALID_ARGUMENT;
  }
  const Tensor* t = b->find(name);
  if (!t) {
    quikb200::set_last_error(std::string("container is missing tensor '") + name + "'");
    return QUIK_ERR_FORMAT;
  }
  if (data) *data = t->bytes.data();
  if (dtype) *dtype = t->dtype;
  if (ndim) *ndim = static_cast<int>(t->shape.size());
  if (shape)
    for (size_t i = 0; i < t->shape.size() && i < 4; ++i) shape[i] = t->shape[i];
  return QUIK_OK;
}

quik_status quik_layer_load_bundle(quik_ctx_t ctx, const char* dir, int64_t row_begin, int64_t row_end,
                                   quik_layer_t* out) {
  quik_bundle_t b = nullptr;
  quik_status s = quik_bundle_open(dir, &b);
  if (s != QUIK_OK) return s;
  quik_weights_desc d;
  s = quik_bundle_weights(b, &d);
  if (s == QUIK_OK) {
    d.row_begin = row_begin;
    d.row_end = row_end;
    s = quik_layer_create(ctx, &d, out);
  }
  quik_bundle_close(b);
  return s;
}

}  // extern "C"
