// Free-format MPS reader / writer (the file format in front
// of solve).  Behaviour follows the reference's parse_mps / write_mps
// (proj/include/pdhglp/mps.hpp:87-535): the same sections, the same
// minimization-form result (OBJSENSE MAX negates the objective and records
// the flag), the same bound and range rules, the same line-numbered error
// messages, and a byte-identical writer.  Host code; the matrix leaves here
// as the two CSR layouts pdlp_solve takes.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "pdlp_b200.h"

namespace pdlp_host {

extern thread_local std::string g_last_error;

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

struct ParseError : std::runtime_error {
  ParseError(size_t line, const std::string& msg)
      : std::runtime_error(line == 0 ? msg : "line " + std::to_string(line) + ": " + msg) {}
};

struct Csr {
  std::vector<int64_t> start, index;
  std::vector<double> value;
};

// from_triplets semantics (sparse.hpp:70-115): lines ordered by index, an
// index that repeats within a line is summed in input order.
Csr compress(int64_t dim, const std::vector<int64_t>& prim, const std::vector<int64_t>& sec,
             const std::vector<double>& val) {
  const size_t count = val.size();
  std::vector<int64_t> head(static_cast<size_t>(dim) + 1, 0);
  for (size_t k = 0; k < count; ++k) ++head[static_cast<size_t>(prim[k]) + 1];
  for (int64_t d = 0; d < dim; ++d) head[d + 1] += head[d];
  std::vector<size_t> perm(count);
  {
    std::vector<int64_t> fill(head.begin(), head.end() - 1);
    for (size_t k = 0; k < count; ++k) perm[static_cast<size_t>(fill[prim[k]]++)] = k;
  }
  Csr out;
  out.start.reserve(static_cast<size_t>(dim) + 1);
  out.start.push_back(0);
  for (int64_t d = 0; d < dim; ++d) {
    auto first = perm.begin() + head[d], last = perm.begin() + head[d + 1];
    std::stable_sort(first, last, [&](size_t a, size_t b) { return sec[a] < sec[b]; });
    while (first != last) {
      const int64_t j = sec[*first];
      double acc = 0.0;
      for (; first != last && sec[*first] == j; ++first) acc += val[*first];
      out.index.push_back(j);
      out.value.push_back(acc);
    }
    out.start.push_back(static_cast<int64_t>(out.index.size()));
  }
  return out;
}

}  // namespace

// ------------------------------------------------------------- the model ---
struct MpsModel {
  int64_t rows = 0, cols = 0;
  Csr by_row, by_col;
  std::vector<double> objective, con_lower, con_upper, var_lower, var_upper;
  bool maximize = false;
  std::string name, objective_name;
  std::vector<std::string> row_names, col_names;
};

namespace {

std::string upper(std::string s) {
  for (char& c : s) c = static_cast<char>(std::toupper(static_cast<unsigned char>(c)));
  return s;
}

std::vector<std::string> split(std::string_view line) {
  std::vector<std::string> out;
  size_t i = 0;
  const auto blank = [](char c) { return c == ' ' || c == '\t'; };
  while (i < line.size()) {
    while (i < line.size() && blank(line[i])) ++i;
    const size_t b = i;
    while (i < line.size() && !blank(line[i])) ++i;
    if (i > b) out.emplace_back(line.substr(b, i - b));
  }
  return out;
}

double number(const std::string& t, size_t line) {
  if (t.empty()) throw ParseError(line, "expected a number");
  char* end = nullptr;
  errno = 0;
  const double v = std::strtod(t.c_str(), &end);
  if (end != t.c_str() + t.size()) throw ParseError(line, "malformed number '" + t + "'");
  return v;
}

// The first failure in problem.hpp:119-154 order (the device check in
// Engine::load reports the same), or empty.
std::string first_issue(const MpsModel& m) {
  for (int64_t i = 0; i < m.cols; ++i) {
    if (!std::isfinite(m.objective[i])) return "objective entry not finite";
  }
  const auto box = [](double lo, double hi, const char* what) -> std::string {
    if (std::isnan(lo) || std::isnan(hi)) return std::string(what) + " bound is NaN";
    if (lo == kInf) return std::string(what) + " lower bound is +inf";
    if (hi == -kInf) return std::string(what) + " upper bound is -inf";
    if (lo > hi) return std::string(what) + " bounds crossed";
    return {};
  };
  for (int64_t i = 0; i < m.cols; ++i) {
    std::string s = box(m.var_lower[i], m.var_upper[i], "variable");
    if (!s.empty()) return s;
  }
  for (int64_t j = 0; j < m.rows; ++j) {
    std::string s = box(m.con_lower[j], m.con_upper[j], "constraint");
    if (!s.empty()) return s;
  }
  for (double v : m.by_row.value) {
    if (!std::isfinite(v)) return "matrix entry not finite";
  }
  return {};
}

class Reader {
 public:
  MpsModel run(std::string_view text) {
    size_t pos = 0;
    while (pos <= text.size() && sec_ != Sec::End) {
      const size_t nl = text.find('\n', pos);
      std::string_view ln = text.substr(pos, nl == std::string_view::npos ? std::string_view::npos : nl - pos);
      pos = nl == std::string_view::npos ? text.size() + 1 : nl + 1;
      ++line_;
      if (!ln.empty() && ln.back() == '\r') ln.remove_suffix(1);
      if (ln.empty() || ln[0] == '*') continue;
      const std::vector<std::string> t = split(ln);
      if (t.empty()) continue;
      if (ln[0] != ' ' && ln[0] != '\t') {
        header(t);
      } else {
        data(t);
      }
    }
    return finish();
  }

 private:
  enum class Sec { None, Name, Sense, Rows, Columns, Rhs, Ranges, Bounds, End };
  struct Pending {
    int64_t row;
    double value;
    size_t line;
  };

  void sense(const std::string& w) {
    const std::string u = upper(w);
    if (u == "MAX" || u == "MAXIMIZE") {
      m_.maximize = true;
    } else if (u == "MIN" || u == "MINIMIZE") {
      m_.maximize = false;
    } else {
      throw ParseError(line_, "unknown objective sense '" + w + "'");
    }
  }

  void header(const std::vector<std::string>& t) {
    const std::string kw = upper(t[0]);
    if (kw == "NAME") {
      sec_ = Sec::Name;
      if (t.size() > 1) m_.name = t[1];
    } else if (kw == "OBJSENSE") {
      sec_ = Sec::Sense;
      if (t.size() > 1) {
        sense(t[1]);
      } else {
        sense_pending_ = true;
      }
    } else if (kw == "ROWS") {
      sec_ = Sec::Rows;
      have_rows_ = true;
    } else if (kw == "COLUMNS") {
      sec_ = Sec::Columns;
      if (!have_rows_) throw ParseError(line_, "COLUMNS before ROWS");
    } else if (kw == "RHS") {
      sec_ = Sec::Rhs;
    } else if (kw == "RANGES") {
      sec_ = Sec::Ranges;
    } else if (kw == "BOUNDS") {
      sec_ = Sec::Bounds;
    } else if (kw == "ENDATA") {
      sec_ = Sec::End;
    } else if (kw == "SOS") {
      throw ParseError(line_, "SOS sections are not supported");
    } else {
      throw ParseError(line_, "unknown section '" + t[0] + "'");
    }
  }

  int64_t row_of(const std::string& name) const {
    const auto it = rows_.find(name);
    if (it == rows_.end()) throw ParseError(line_, "unknown row '" + name + "'");
    return it->second;
  }

  bool is_objective(const std::string& name) const {
    return have_objective_ && name == m_.objective_name;
  }

  void add_row(const std::string& name, char type, double lo, double hi) {
    rows_.emplace(name, static_cast<int64_t>(type_.size()));
    m_.row_names.push_back(name);
    type_.push_back(type);
    m_.con_lower.push_back(lo);
    m_.con_upper.push_back(hi);
  }

  int64_t column(const std::string& name) {
    const auto it = cols_.find(name);
    if (it != cols_.end()) return it->second;
    const int64_t c = static_cast<int64_t>(m_.col_names.size());
    cols_.emplace(name, c);
    m_.col_names.push_back(name);
    m_.objective.push_back(0.0);
    m_.var_lower.push_back(0.0);
    m_.var_upper.push_back(kInf);
    lower_given_.push_back(false);
    return c;
  }

  void data(const std::vector<std::string>& t) {
    switch (sec_) {
      case Sec::None:
        throw ParseError(line_, "data before any section header");
      case Sec::Name:
      case Sec::End:
        throw ParseError(line_, "unexpected data line");
      case Sec::Sense:
        if (!sense_pending_) throw ParseError(line_, "unexpected data line");
        sense(t[0]);
        sense_pending_ = false;
        return;
      case Sec::Rows:
        return rows_line(t);
      case Sec::Columns:
        return columns_line(t);
      case Sec::Rhs:
      case Sec::Ranges:
        return rhs_line(t, sec_ == Sec::Ranges);
      case Sec::Bounds:
        return bounds_line(t);
    }
  }

  void rows_line(const std::vector<std::string>& t) {
    if (t.size() != 2) throw ParseError(line_, "expected 'TYPE NAME'");
    const std::string type = upper(t[0]);
    const std::string& name = t[1];
    if (rows_.count(name) != 0 || name == m_.objective_name) {
      throw ParseError(line_, "duplicate row '" + name + "'");
    }
    if (type == "N") {
      if (!have_objective_) {  // the first free row is the objective
        m_.objective_name = name;
        have_objective_ = true;
      } else {
        add_row(name, 'N', -kInf, kInf);
      }
    } else if (type == "L") {
      add_row(name, 'L', -kInf, 0.0);
    } else if (type == "G") {
      add_row(name, 'G', 0.0, kInf);
    } else if (type == "E") {
      add_row(name, 'E', 0.0, 0.0);
    } else {
      throw ParseError(line_, "unknown row type '" + t[0] + "'");
    }
  }

  void columns_line(const std::vector<std::string>& t) {
    if (t.size() >= 3 && upper(t[1]) == "'MARKER'") {
      const std::string mk = upper(t[2]);
      if (mk == "'INTORG'") throw ParseError(line_, "integer variables are not supported");
      if (mk == "'INTEND'") return;
      throw ParseError(line_, "unknown marker '" + t[2] + "'");
    }
    if (t.size() != 3 && t.size() != 5) {
      throw ParseError(line_, "expected 'COLUMN ROW VALUE [ROW VALUE]'");
    }
    const int64_t c = column(t[0]);
    for (size_t k = 1; k + 1 < t.size(); k += 2) {
      const double v = number(t[k + 1], line_);
      if (is_objective(t[k])) {
        m_.objective[static_cast<size_t>(c)] += v;
        continue;
      }
      tr_row_.push_back(row_of(t[k]));
      tr_col_.push_back(c);
      tr_val_.push_back(v);
    }
  }

  void rhs_line(const std::vector<std::string>& t, bool ranges) {
    // the leading set name is optional: present unless the first token names
    // a row and the arity is even
    const bool named_first = t.size() % 2 == 0 && (rows_.count(t[0]) != 0 || t[0] == m_.objective_name);
    const size_t first = named_first ? 0 : 1;
    if (t.size() < first + 2 || (t.size() - first) % 2 != 0) {
      throw ParseError(line_, "expected '[SET] ROW VALUE [ROW VALUE]'");
    }
    for (size_t k = first; k + 1 < t.size(); k += 2) {
      const double v = number(t[k + 1], line_);
      if (is_objective(t[k])) {
        if (ranges) throw ParseError(line_, "range on the objective row");
        continue;  // objective offsets are ignored
      }
      (ranges ? ranges_ : rhs_).push_back({row_of(t[k]), v, line_});
    }
  }

  void bounds_line(const std::vector<std::string>& t) {
    if (t.size() < 2) throw ParseError(line_, "malformed bound line");
    const std::string type = upper(t[0]);
    if (type == "BV" || type == "LI" || type == "UI" || type == "SC") {
      throw ParseError(line_, "bound type '" + t[0] + "' is not supported");
    }
    const bool valued = type == "LO" || type == "UP" || type == "FX";
    if (!valued && type != "FR" && type != "MI" && type != "PL") {
      throw ParseError(line_, "unknown bound type '" + t[0] + "'");
    }
    std::string col;
    double v = 0.0;
    if (valued) {
      if (t.size() != 3 && t.size() != 4) throw ParseError(line_, "expected 'TYPE [SET] COLUMN VALUE'");
      col = t[t.size() - 2];
      v = number(t[t.size() - 1], line_);
    } else if (t.size() == 2) {
      col = t[1];
    } else if (t.size() == 3) {  // 'TYPE SET COLUMN' or 'TYPE COLUMN ignored-value'
      col = cols_.count(t[2]) != 0 ? t[2] : t[1];
    } else if (t.size() == 4) {
      col = t[2];
    } else {
      throw ParseError(line_, "malformed bound line");
    }
    const auto it = cols_.find(col);
    if (it == cols_.end()) throw ParseError(line_, "unknown column '" + col + "'");
    const size_t c = static_cast<size_t>(it->second);
    double& lo = m_.var_lower[c];
    double& hi = m_.var_upper[c];
    if (type == "LO") {
      lo = v;
      lower_given_[c] = true;
    } else if (type == "UP") {
      hi = v;
      if (v < 0.0 && !lower_given_[c]) lo = -kInf;  // a lone negative UP frees the lower side
    } else if (type == "FX") {
      lo = hi = v;
      lower_given_[c] = true;
    } else if (type == "FR") {
      lo = -kInf;
      hi = kInf;
      lower_given_[c] = true;
    } else if (type == "MI") {
      lo = -kInf;
      lower_given_[c] = true;
    } else {
      hi = kInf;  // PL
    }
  }

  MpsModel finish() {
    if (sense_pending_) throw ParseError(line_, "OBJSENSE without a value");
    if (!have_rows_) throw ParseError(line_, "missing ROWS section");
    if (!have_objective_) throw ParseError(line_, "no objective row declared");
    for (const Pending& e : rhs_) {
      const size_t j = static_cast<size_t>(e.row);
      if (type_[j] == 'L') m_.con_upper[j] = e.value;
      if (type_[j] == 'G') m_.con_lower[j] = e.value;
      if (type_[j] == 'E') m_.con_lower[j] = m_.con_upper[j] = e.value;
    }
    for (const Pending& e : ranges_) {
      const size_t j = static_cast<size_t>(e.row);
      double& lo = m_.con_lower[j];
      double& hi = m_.con_upper[j];
      switch (type_[j]) {
        case 'L': lo = hi - std::abs(e.value); break;
        case 'G': hi = lo + std::abs(e.value); break;
        case 'E':
          if (e.value >= 0.0) {
            hi = lo + e.value;
          } else {
            lo = hi + e.value;
          }
          break;
        default: throw ParseError(e.line, "range on a free row");
      }
    }
    m_.rows = static_cast<int64_t>(type_.size());
    m_.cols = static_cast<int64_t>(m_.col_names.size());
    m_.by_row = compress(m_.rows, tr_row_, tr_col_, tr_val_);
    m_.by_col = compress(m_.cols, tr_col_, tr_row_, tr_val_);
    if (m_.maximize) {
      for (double& c : m_.objective) c = -c;
    }
    const std::string issue = first_issue(m_);
    if (!issue.empty()) throw ParseError(0, "invalid model: " + issue);
    return std::move(m_);
  }

  MpsModel m_;
  Sec sec_ = Sec::None;
  size_t line_ = 0;
  bool have_rows_ = false, have_objective_ = false, sense_pending_ = false;
  std::unordered_map<std::string, int64_t> rows_, cols_;
  std::vector<char> type_;
  std::vector<bool> lower_given_;
  std::vector<int64_t> tr_row_, tr_col_;
  std::vector<double> tr_val_;
  std::vector<Pending> rhs_, ranges_;
};

std::string fmt(double v) {
  char b[40];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

// write_mps format (mps.hpp:420-528): generated names OBJ / R# / C#, ranged
// rows as L + RANGES, lower bounds before upper ones.
std::string write(const pdlp_problem_view& p, const char* name, bool maximize) {
  const int64_t m = p.rows, n = p.cols;
  std::string rows_s, cols_s, rhs_s, rng_s, bnd_s;
  for (int64_t j = 0; j < m; ++j) {
    const double lo = p.con_lower[j], hi = p.con_upper[j];
    const std::string r = "R" + std::to_string(j);
    const char type = lo == hi ? 'E' : (std::isfinite(hi) ? 'L' : (std::isfinite(lo) ? 'G' : 'N'));
    rows_s += std::string(" ") + type + " " + r + "\n";
    if (type == 'E' || type == 'L') rhs_s += " RHS " + r + " " + fmt(type == 'E' ? lo : hi) + "\n";
    if (type == 'G') rhs_s += " RHS " + r + " " + fmt(lo) + "\n";
    if (lo != hi && std::isfinite(lo) && std::isfinite(hi)) rng_s += " RNG " + r + " " + fmt(hi - lo) + "\n";
  }
  for (int64_t i = 0; i < n; ++i) {
    const std::string c = "C" + std::to_string(i);
    const double obj = maximize ? -p.objective[i] : p.objective[i];
    const int64_t a = p.by_col.start ? p.by_col.start[i] : 0, b = p.by_col.start ? p.by_col.start[i + 1] : 0;
    if (obj != 0.0 || a == b) cols_s += " " + c + " OBJ " + fmt(obj) + "\n";
    for (int64_t k = a; k < b; ++k) {
      cols_s += " " + c + " R" + std::to_string(p.by_col.index[k]) + " " + fmt(p.by_col.value[k]) + "\n";
    }
    const double lo = p.var_lower[i], hi = p.var_upper[i];
    if (lo == 0.0 && !std::isfinite(hi) && hi > 0.0) continue;  // the default [0, inf)
    if (lo == hi) {
      bnd_s += " FX BND " + c + " " + fmt(lo) + "\n";
    } else if (!std::isfinite(lo) && !std::isfinite(hi)) {
      bnd_s += " FR BND " + c + "\n";
    } else {
      if (!std::isfinite(lo)) {
        bnd_s += " MI BND " + c + "\n";
      } else if (lo != 0.0) {
        bnd_s += " LO BND " + c + " " + fmt(lo) + "\n";
      }
      if (std::isfinite(hi)) bnd_s += " UP BND " + c + " " + fmt(hi) + "\n";
    }
  }
  std::string out = "NAME " + std::string(name && *name ? name : "LP") + "\n";
  if (maximize) out += "OBJSENSE MAX\n";
  out += "ROWS\n N OBJ\n" + rows_s + "COLUMNS\n" + cols_s + "RHS\n" + rhs_s;
  if (!rng_s.empty()) out += "RANGES\n" + rng_s;
  if (!bnd_s.empty()) out += "BOUNDS\n" + bnd_s;
  return out + "ENDATA\n";
}

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

}  // namespace
}  // namespace pdlp_host

using pdlp_host::MpsModel;

extern "C" {

struct pdlp_mps {
  MpsModel model;
};

int pdlp_mps_parse(const char* text, size_t len, pdlp_mps** out) {
  if (out == nullptr || (text == nullptr && len > 0)) {
    return pdlp_host::fail(PDLP_ERR_INVALID_ARGUMENT, "null argument");
  }
  try {
    auto* h = new pdlp_mps{pdlp_host::Reader().run(std::string_view(text ? text : "", len))};
    *out = h;
    return PDLP_OK;
  } catch (const pdlp_host::ParseError& e) {
    return pdlp_host::fail(PDLP_ERR_INVALID_PROBLEM, e.what());
  } catch (const std::exception& e) {
    return pdlp_host::fail(PDLP_ERR_INTERNAL, e.what());
  }
}

int pdlp_mps_read_file(const char* path, pdlp_mps** out) {
  if (path == nullptr || out == nullptr) return pdlp_host::fail(PDLP_ERR_INVALID_ARGUMENT, "null argument");
  std::ifstream in(path, std::ios::binary);
  if (!in) return pdlp_host::fail(PDLP_ERR_INVALID_PROBLEM, std::string("cannot open '") + path + "'");
  std::ostringstream buf;
  buf << in.rdbuf();
  const std::string s = buf.str();
  return pdlp_mps_parse(s.data(), s.size(), out);
}

void pdlp_mps_view(const pdlp_mps* h, pdlp_problem_view* v) {
  const MpsModel& m = h->model;
  v->rows = m.rows;
  v->cols = m.cols;
  v->by_row = {m.rows, static_cast<int64_t>(m.by_row.value.size()), m.by_row.start.data(),
               m.by_row.index.data(), m.by_row.value.data()};
  v->by_col = {m.cols, static_cast<int64_t>(m.by_col.value.size()), m.by_col.start.data(),
               m.by_col.index.data(), m.by_col.value.data()};
  v->objective = m.objective.data();
  v->con_lower = m.con_lower.data();
  v->con_upper = m.con_upper.data();
  v->var_lower = m.var_lower.data();
  v->var_upper = m.var_upper.data();
}

int32_t pdlp_mps_maximize(const pdlp_mps* h) { return h->model.maximize ? 1 : 0; }
const char* pdlp_mps_name(const pdlp_mps* h) { return h->model.name.c_str(); }
const char* pdlp_mps_objective_name(const pdlp_mps* h) { return h->model.objective_name.c_str(); }
const char* pdlp_mps_row_name(const pdlp_mps* h, int64_t j) {
  return j >= 0 && j < h->model.rows ? h->model.row_names[static_cast<size_t>(j)].c_str() : nullptr;
}
const char* pdlp_mps_col_name(const pdlp_mps* h, int64_t i) {
  return i >= 0 && i < h->model.cols ? h->model.col_names[static_cast<size_t>(i)].c_str() : nullptr;
}
void pdlp_mps_free(pdlp_mps* h) { delete h; }

int pdlp_mps_write(const pdlp_problem_view* p, const char* name, int32_t maximize, char** text,
                   size_t* len) {
  if (p == nullptr || text == nullptr || len == nullptr) {
    return pdlp_host::fail(PDLP_ERR_INVALID_ARGUMENT, "null argument");
  }
  try {
    const std::string s = pdlp_host::write(*p, name, maximize != 0);
    char* buf = static_cast<char*>(std::malloc(s.size() + 1));
    if (buf == nullptr) return pdlp_host::fail(PDLP_ERR_OUT_OF_MEMORY, "out of memory");
    std::memcpy(buf, s.c_str(), s.size() + 1);
    *text = buf;
    *len = s.size();
    return PDLP_OK;
  } catch (const std::exception& e) {
    return pdlp_host::fail(PDLP_ERR_INTERNAL, e.what());
  }
}

void pdlp_mps_free_text(char* text) { std::free(text); }

}  // extern "C"
