// config.cu -- pipeline config (de)serialisation (SURVEY.md
// §8(f) row 4): a UTF-8 JSON document
//
//   {"seed": <optional u64>, "transforms": [{"name": <kind>, "p": <number>,
//                                            "params": {<kind schema>}}, ...]}
//
// parsed natively (small recursive-descent parser, no dependencies) into the
// same alb_op list alb_pipeline_create validates, and written back with
// round-trip exact numbers (%.17g).  Range parameters accept a number (fixed
// value, lo = hi) or a [lo, hi] pair; unknown names, unknown or missing params,
// and wrong types are errors that name the culprit (alb_last_error).
// Host code only.
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "config.h"

namespace alb {
namespace {

// ------------------------------------------------------------------ JSON value
struct JVal {
  enum Type { NUL, BOOL, NUM, STR, ARR, OBJ } t = NUL;
  double num = 0.0;
  bool is_int = false;  // integer literal (no fraction / exponent)
  bool neg = false;
  unsigned long long mag = 0;  // |integer literal| when is_int
  bool b = false;
  std::string s;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const char* k) const {
    for (auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

class Parser {
 public:
  explicit Parser(const char* t) : p_(t) {}
  bool parse(JVal& v, std::string& err) {
    if (!value(v, 0)) { err = err_; return false; }
    ws();
    if (*p_) { err = at("trailing characters"); return false; }
    return true;
  }

 private:
  const char* p_;
  std::string err_;
  int line_ = 1;
  std::string at(const char* what) { return std::string(what) + " at line " + std::to_string(line_); }
  bool fail(const char* what) { if (err_.empty()) err_ = at(what); return false; }
  void ws() {
    while (*p_ == ' ' || *p_ == '\t' || *p_ == '\n' || *p_ == '\r') { if (*p_ == '\n') ++line_; ++p_; }
  }
  bool lit(const char* w) {
    const size_t n = strlen(w);
    if (strncmp(p_, w, n) != 0) return false;
    p_ += n;
    return true;
  }
  static void utf8(std::string& o, unsigned c) {
    if (c < 0x80) o += (char)c;
    else if (c < 0x800) { o += (char)(0xC0 | (c >> 6)); o += (char)(0x80 | (c & 63)); }
    else if (c < 0x10000) { o += (char)(0xE0 | (c >> 12)); o += (char)(0x80 | ((c >> 6) & 63)); o += (char)(0x80 | (c & 63)); }
    else { o += (char)(0xF0 | (c >> 18)); o += (char)(0x80 | ((c >> 12) & 63)); o += (char)(0x80 | ((c >> 6) & 63)); o += (char)(0x80 | (c & 63)); }
  }
  bool hex4(unsigned& c) {
    c = 0;
    for (int i = 0; i < 4; ++i) {
      const char h = *p_++;
      c <<= 4;
      if (h >= '0' && h <= '9') c |= (unsigned)(h - '0');
      else if (h >= 'a' && h <= 'f') c |= (unsigned)(h - 'a' + 10);
      else if (h >= 'A' && h <= 'F') c |= (unsigned)(h - 'A' + 10);
      else return fail("bad \\u escape");
    }
    return true;
  }
  bool str(std::string& o) {
    ++p_;  // opening quote
    while (*p_ != '"') {
      if (!*p_ || (unsigned char)*p_ < 0x20) return fail("unterminated string");
      if (*p_ != '\\') { o += *p_++; continue; }
      ++p_;
      const char e = *p_++;
      switch (e) {
        case '"': o += '"'; break;
        case '\\': o += '\\'; break;
        case '/': o += '/'; break;
        case 'b': o += '\b'; break;
        case 'f': o += '\f'; break;
        case 'n': o += '\n'; break;
        case 'r': o += '\r'; break;
        case 't': o += '\t'; break;
        case 'u': {
          unsigned c;
          if (!hex4(c)) return false;
          if (c >= 0xD800 && c < 0xDC00 && p_[0] == '\\' && p_[1] == 'u') {  // surrogate pair
            p_ += 2;
            unsigned lo;
            if (!hex4(lo)) return false;
            c = 0x10000 + ((c - 0xD800) << 10) + (lo - 0xDC00);
          }
          utf8(o, c);
          break;
        }
        default: return fail("bad escape");
      }
    }
    ++p_;
    return true;
  }
  bool number(JVal& v) {
    const char* s = p_;
    v.neg = *p_ == '-';
    if (v.neg) ++p_;
    auto digits = [&]() { const char* s0 = p_; while (*p_ >= '0' && *p_ <= '9') ++p_; return p_ - s0; };
    if (*p_ == '0') ++p_;  // RFC 8259: no leading zeros
    else if (digits() == 0) return fail("bad number");
    bool frac = false;
    if (*p_ == '.') { frac = true; ++p_; if (digits() == 0) return fail("bad number"); }
    if (*p_ == 'e' || *p_ == 'E') {
      frac = true; ++p_;
      if (*p_ == '+' || *p_ == '-') ++p_;
      if (digits() == 0) return fail("bad number");
    }
    const std::string tok(s, p_);
    v.t = JVal::NUM;
    v.num = strtod(tok.c_str(), nullptr);
    if (!std::isfinite(v.num)) return fail("number out of range");
    v.is_int = !frac;
    if (v.is_int) {
      errno = 0;
      v.mag = strtoull(tok.c_str() + (v.neg ? 1 : 0), nullptr, 10);
      if (errno == ERANGE) v.is_int = false;
    }
    return true;
  }
  bool value(JVal& v, int depth) {
    if (depth > 64) return fail("nesting too deep");
    ws();
    const char c = *p_;
    if (c == '{') {
      v.t = JVal::OBJ;
      ++p_;
      ws();
      if (*p_ == '}') { ++p_; return true; }
      for (;;) {
        ws();
        if (*p_ != '"') return fail("expected a key");
        std::string k;
        if (!str(k)) return false;
        ws();
        if (*p_++ != ':') return fail("expected ':'");
        JVal e;
        if (!value(e, depth + 1)) return false;
        if (v.get(k.c_str())) return fail(("duplicate key '" + k + "'").c_str());
        v.obj.emplace_back(std::move(k), std::move(e));
        ws();
        if (*p_ == ',') { ++p_; continue; }
        if (*p_ == '}') { ++p_; return true; }
        return fail("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.t = JVal::ARR;
      ++p_;
      ws();
      if (*p_ == ']') { ++p_; return true; }
      for (;;) {
        JVal e;
        if (!value(e, depth + 1)) return false;
        v.arr.push_back(std::move(e));
        ws();
        if (*p_ == ',') { ++p_; continue; }
        if (*p_ == ']') { ++p_; return true; }
        return fail("expected ',' or ']'");
      }
    }
    if (c == '"') { v.t = JVal::STR; return str(v.s); }
    if (c == '-' || (c >= '0' && c <= '9')) return number(v);
    if (lit("true")) { v.t = JVal::BOOL; v.b = true; return true; }
    if (lit("false")) { v.t = JVal::BOOL; v.b = false; return true; }
    if (lit("null")) { v.t = JVal::NUL; return true; }
    return fail("unexpected character");
  }
};

// -------------------------------------------------------------- op schema
enum FType { F_RANGE, F_SYMRANGE, F_FIXED, F_INT, F_INTERP, F_BORDER, F_FILL, F_MASKFILL, F_MEAN, F_STD };
enum IntSlot { I_OUT_W, I_OUT_H, I_MIN_SIDE, I_MAX_SIDE, I_CROP_X, I_CROP_Y, I_NUM_STEPS };

struct Field {
  const char* name;
  FType type;
  int idx;        // lo/hi index for ranges, IntSlot for ints
  bool required;
};

struct Kind {
  const char* name;
  std::vector<Field> fields;
};

const std::vector<Kind>& kinds() {
  static const std::vector<Field> warp = {{"interpolation", F_INTERP, 0, false}, {"border", F_BORDER, 0, false},
                                          {"fill", F_FILL, 0, false}, {"mask_fill", F_MASKFILL, 0, false}};
  auto with = [](std::vector<Field> a, const std::vector<Field>& b) { a.insert(a.end(), b.begin(), b.end()); return a; };
  static const std::vector<Kind> k = {
      {"HorizontalFlip", {}},
      {"VerticalFlip", {}},
      {"Rotate", with({{"angle", F_RANGE, 0, true}}, warp)},
      {"ShiftScaleRotate", with({{"shift_x", F_RANGE, 0, true}, {"shift_y", F_RANGE, 1, true},
                                 {"scale", F_RANGE, 2, true}, {"angle", F_RANGE, 3, true}}, warp)},
      {"RandomCrop", {{"width", F_INT, I_OUT_W, true}, {"height", F_INT, I_OUT_H, true}}},
      {"PadToSize", {{"width", F_INT, I_OUT_W, true}, {"height", F_INT, I_OUT_H, true},
                     {"fill", F_FILL, 0, false}, {"mask_fill", F_MASKFILL, 0, false}}},
      {"Resize", {{"width", F_INT, I_OUT_W, true}, {"height", F_INT, I_OUT_H, true},
                  {"interpolation", F_INTERP, 0, false}}},
      {"RandomSizedCrop", {{"min_side", F_INT, I_MIN_SIDE, true}, {"max_side", F_INT, I_MAX_SIDE, true},
                           {"width", F_INT, I_OUT_W, true}, {"height", F_INT, I_OUT_H, true},
                           {"interpolation", F_INTERP, 0, false}}},
      {"Brightness", {{"beta", F_RANGE, 0, true}}},
      {"Contrast", {{"c", F_RANGE, 0, true}}},
      {"BrightnessContrast", {{"beta", F_RANGE, 0, true}, {"c", F_RANGE, 1, true}}},
      {"Gamma", {{"g", F_RANGE, 0, true}}},
      {"ShiftRGB", {{"dr", F_RANGE, 0, true}, {"dg", F_RANGE, 1, true}, {"db", F_RANGE, 2, true}}},
      {"ShiftHSV", {{"dh", F_RANGE, 0, true}, {"ds", F_RANGE, 1, true}, {"dv", F_RANGE, 2, true}}},
      {"Grayscale", {}},
      {"Equalize", {}},
      {"Normalize", {{"mean", F_MEAN, 0, true}, {"std", F_STD, 0, true}}},
      {"Crop", {{"x", F_INT, I_CROP_X, true}, {"y", F_INT, I_CROP_Y, true},
                {"width", F_INT, I_OUT_W, true}, {"height", F_INT, I_OUT_H, true}}},
      {"Rotate90", {{"k", F_RANGE, 0, true}}},
      {"D4", {{"element", F_RANGE, 0, true}}},
      {"GridDistortion", {{"num_steps", F_INT, I_NUM_STEPS, true}, {"distort_limit", F_SYMRANGE, 0, true},
                          {"interpolation", F_INTERP, 0, false}}},
      {"ElasticTransform", with({{"alpha", F_FIXED, 0, true}, {"sigma", F_FIXED, 1, true}}, warp)},
  };
  return k;
}

int32_t* int_slot(alb_op& o, int idx) {
  switch (idx) {
    case I_OUT_W: return &o.out_w;
    case I_OUT_H: return &o.out_h;
    case I_MIN_SIDE: return &o.min_side;
    case I_MAX_SIDE: return &o.max_side;
    case I_CROP_X: return &o.crop_x;
    case I_CROP_Y: return &o.crop_y;
    default: return &o.num_steps;
  }
}

std::string valid_names() {
  std::string s;
  for (auto& k : kinds()) s += (s.empty() ? "" : ", ") + std::string(k.name);
  return s;
}

alb_status bad(const std::string& where, const std::string& what) {
  return set_error(ALB_E_INVALID_ARG, where + ": " + what);
}

bool as_int(const JVal& v, long long lo, long long hi, long long& out) {
  if (v.t != JVal::NUM || !v.is_int) return false;
  if (v.mag > (unsigned long long)9e18) return false;
  out = v.neg ? -(long long)v.mag : (long long)v.mag;
  return out >= lo && out <= hi;
}

// one params field into the op
alb_status read_field(const Field& f, const JVal& v, alb_op& o, const std::string& where) {
  const std::string w = where + " param '" + f.name + "'";
  switch (f.type) {
    case F_RANGE: case F_SYMRANGE: case F_FIXED: {
      double lo, hi;
      if (v.t == JVal::NUM) {
        lo = hi = v.num;
        if (f.type == F_SYMRANGE) lo = -v.num;
      } else if (v.t == JVal::ARR && v.arr.size() == 2 && v.arr[0].t == JVal::NUM && v.arr[1].t == JVal::NUM &&
                 f.type != F_FIXED) {
        lo = v.arr[0].num;
        hi = v.arr[1].num;
      } else {
        return bad(w, f.type == F_FIXED ? "expected a number" : "expected a number or a [lo, hi] pair");
      }
      o.lo[f.idx] = lo;
      o.hi[f.idx] = hi;
      return ALB_OK;
    }
    case F_INT: {
      long long x;
      if (!as_int(v, -2147483647ll, 2147483647ll, x)) return bad(w, "expected a 32-bit integer");
      *int_slot(o, f.idx) = (int32_t)x;
      return ALB_OK;
    }
    case F_INTERP:
      if (v.t == JVal::STR && v.s == "nearest") o.interp = ALB_INTERP_NEAREST;
      else if (v.t == JVal::STR && v.s == "bilinear") o.interp = ALB_INTERP_BILINEAR;
      else return bad(w, "expected \"nearest\" or \"bilinear\"");
      return ALB_OK;
    case F_BORDER:
      if (v.t == JVal::STR && v.s == "constant") o.border = ALB_BORDER_CONSTANT;
      else if (v.t == JVal::STR && v.s == "reflect_101") o.border = ALB_BORDER_REFLECT_101;
      else return bad(w, "expected \"constant\" or \"reflect_101\"");
      return ALB_OK;
    case F_FILL: {
      long long c[3];
      if (v.t != JVal::ARR || v.arr.size() != 3 || !as_int(v.arr[0], 0, 255, c[0]) ||
          !as_int(v.arr[1], 0, 255, c[1]) || !as_int(v.arr[2], 0, 255, c[2]))
        return bad(w, "expected [r, g, b] integers in 0..255");
      for (int i = 0; i < 3; ++i) o.fill[i] = (uint8_t)c[i];
      return ALB_OK;
    }
    case F_MASKFILL: {
      long long x;
      if (!as_int(v, 0, 255, x)) return bad(w, "expected an integer in 0..255");
      o.mask_fill = (uint8_t)x;
      return ALB_OK;
    }
    case F_MEAN: case F_STD: {
      if (v.t != JVal::ARR || v.arr.size() != 3) return bad(w, "expected 3 numbers");
      for (int i = 0; i < 3; ++i) {
        if (v.arr[i].t != JVal::NUM) return bad(w, "expected 3 numbers");
        (f.type == F_MEAN ? o.mean : o.std)[i] = v.arr[i].num;
      }
      return ALB_OK;
    }
  }
  return bad(w, "unhandled field type");
}

// ------------------------------------------------------------- writer
void num(std::string& o, double v) {
  char b[40];
  if (v == std::floor(v) && std::fabs(v) < 1e15) snprintf(b, sizeof b, "%.1f", v);
  else snprintf(b, sizeof b, "%.17g", v);
  o += b;
}

void write_field(std::string& s, const Field& f, const alb_op& o) {
  s += "\"";
  s += f.name;
  s += "\": ";
  switch (f.type) {
    case F_FIXED: num(s, o.lo[f.idx]); break;
    case F_RANGE: case F_SYMRANGE:
      s += "[";
      num(s, o.lo[f.idx]);
      s += ", ";
      num(s, o.hi[f.idx]);
      s += "]";
      break;
    case F_INT: s += std::to_string(*int_slot(const_cast<alb_op&>(o), f.idx)); break;
    case F_INTERP: s += o.interp == ALB_INTERP_NEAREST ? "\"nearest\"" : "\"bilinear\""; break;
    case F_BORDER: s += o.border == ALB_BORDER_REFLECT_101 ? "\"reflect_101\"" : "\"constant\""; break;
    case F_FILL:
      s += "[" + std::to_string(o.fill[0]) + ", " + std::to_string(o.fill[1]) + ", " + std::to_string(o.fill[2]) + "]";
      break;
    case F_MASKFILL: s += std::to_string(o.mask_fill); break;
    case F_MEAN: case F_STD: {
      const double* a = f.type == F_MEAN ? o.mean : o.std;
      s += "[";
      for (int i = 0; i < 3; ++i) { if (i) s += ", "; num(s, a[i]); }
      s += "]";
      break;
    }
  }
}

}  // namespace
}  // namespace alb

using namespace alb;

extern "C" {

alb_status alb_pipeline_from_json(const char* text, alb_pipeline** out, uint64_t* seed, int32_t* has_seed) {
  if (!text || !out) return set_error(ALB_E_INVALID_ARG, "null argument");
  JVal doc;
  std::string err;
  if (!Parser(text).parse(doc, err)) return bad("config", "JSON syntax error: " + err);
  if (doc.t != JVal::OBJ) return bad("config", "top level must be an object");
  for (auto& kv : doc.obj)
    if (kv.first != "seed" && kv.first != "transforms") return bad("config", "unknown top-level field '" + kv.first + "'");
  const JVal* sd = doc.get("seed");
  if (has_seed) *has_seed = 0;
  if (sd && sd->t != JVal::NUL) {
    if (sd->t != JVal::NUM || !sd->is_int || sd->neg) return bad("config", "'seed' must be a non-negative 64-bit integer");
    if (seed) *seed = sd->mag;
    if (has_seed) *has_seed = 1;
  }
  const JVal* tr = doc.get("transforms");
  if (!tr || tr->t != JVal::ARR) return bad("config", "missing 'transforms' array");
  if (tr->arr.size() > (size_t)ALB_MAX_OPS) return set_error(ALB_E_UNSUPPORTED, "config: more than 16 transforms");
  std::vector<alb_op> ops(tr->arr.size());
  for (size_t i = 0; i < tr->arr.size(); ++i) {
    const JVal& t = tr->arr[i];
    const std::string where = "transforms[" + std::to_string(i) + "]";
    if (t.t != JVal::OBJ) return bad(where, "expected an object");
    for (auto& kv : t.obj)
      if (kv.first != "name" && kv.first != "p" && kv.first != "params")
        return bad(where, "unknown field '" + kv.first + "'");
    const JVal* nm = t.get("name");
    if (!nm || nm->t != JVal::STR) return bad(where, "missing 'name'");
    int kind = -1;
    for (size_t k = 0; k < kinds().size(); ++k)
      if (nm->s == kinds()[k].name) kind = (int)k;
    if (kind < 0)
      return set_error(ALB_E_UNKNOWN_OP, where + ": unknown transform '" + nm->s + "'; valid names: " + valid_names());
    const Kind& K = kinds()[kind];
    const std::string wk = where + " (" + K.name + ")";
    alb_op& o = ops[i];
    memset(&o, 0, sizeof o);
    o.kind = kind;
    o.interp = ALB_INTERP_BILINEAR;
    o.border = ALB_BORDER_CONSTANT;
    o.std[0] = o.std[1] = o.std[2] = 1.0;
    const JVal* p = t.get("p");
    if (!p) return bad(wk, "missing 'p'");
    if (p->t != JVal::NUM) return bad(wk, "'p' must be a number");
    o.p = p->num;
    const JVal* prm = t.get("params");
    static const JVal empty_obj = [] { JVal v; v.t = JVal::OBJ; return v; }();
    if (!prm) prm = &empty_obj;
    if (prm->t != JVal::OBJ) return bad(wk, "'params' must be an object");
    for (auto& kv : prm->obj) {
      bool known = false;
      for (auto& f : K.fields) known |= kv.first == f.name;
      if (!known) return bad(wk, "unknown param '" + kv.first + "'");
    }
    for (auto& f : K.fields) {
      const JVal* v = prm->get(f.name);
      if (!v) {
        if (f.required) return bad(wk, std::string("missing required param '") + f.name + "'");
        continue;
      }
      alb_status s = read_field(f, *v, o, wk);
      if (s) return s;
    }
  }
  return alb_pipeline_create(ops.data(), (int32_t)ops.size(), out);  // range validation (atomic)
}

alb_status alb_pipeline_to_json(const alb_pipeline* p, const uint64_t* seed, char* buf, size_t cap, size_t* len) {
  if (!p || !len) return set_error(ALB_E_INVALID_ARG, "null argument");
  std::string s = "{";
  if (seed) s += "\"seed\": " + std::to_string((unsigned long long)*seed) + ", ";
  s += "\"transforms\": [";
  const std::vector<alb_op>& ops = pipeline_ops(p);
  for (size_t i = 0; i < ops.size(); ++i) {
    const alb_op& o = ops[i];
    const Kind& K = kinds()[o.kind];
    s += i ? ", {" : "{";
    s += "\"name\": \"" + std::string(K.name) + "\", \"p\": ";
    num(s, o.p);
    s += ", \"params\": {";
    for (size_t f = 0; f < K.fields.size(); ++f) {
      if (f) s += ", ";
      write_field(s, K.fields[f], o);
    }
    s += "}}";
  }
  s += "]}";
  *len = s.size();
  if (buf) {
    if (cap < s.size() + 1) return set_error(ALB_E_INVALID_ARG, "buffer too small");
    memcpy(buf, s.c_str(), s.size() + 1);
  }
  return ALB_OK;
}

}  // extern "C"
