// SSA lowering and the CPU IR interpreter (reference semantics:
// /root/reference/proj/src/codegen/kernel.cpp:17-46 run, :111-269 lowering
// rules -- structural CSE, bit-exact constant pool, -1*t -> neg/sub,
// 2*t -> t+t, |exponent| <= 4 unrolled).
#include <bit>
#include <charconv>
#include <cmath>
#include <map>
#include <tuple>
#include <unordered_map>

#include "femforge/codegen.hpp"

namespace femforge::codegen {

using namespace symbolic;

std::string double_literal(double v) {
  if (std::isnan(v)) return "__longlong_as_double(0x7ff8000000000000LL)";
  if (std::isinf(v)) return v > 0 ? "__longlong_as_double(0x7ff0000000000000LL)" : "__longlong_as_double(0xfff0000000000000LL)";
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".e") == std::string::npos) s += ".0";
  return s;
}

namespace {

double exec(const Instr& in, const double* r, std::span<const double> args, const std::vector<double>& consts) {
  switch (in.op) {
    case Op::LoadArg: return args[in.imm];
    case Op::LoadConst: return consts[in.imm];
    case Op::Add: return r[in.a] + r[in.b];
    case Op::Sub: return r[in.a] - r[in.b];
    case Op::Mul: return r[in.a] * r[in.b];
    case Op::Div: return r[in.a] / r[in.b];
    case Op::Neg: return -r[in.a];
    case Op::PowInt: return pow_int(r[in.a], in.imm);
    case Op::Sin: return std::sin(r[in.a]);
    case Op::Cos: return std::cos(r[in.a]);
    case Op::Sqrt: return std::sqrt(r[in.a]);
  }
  return 0.0;
}

const char* mnemonic(Op op) {
  static const char* names[] = {"arg", "const", "add", "sub", "mul", "div", "neg", "pow", "sin", "cos", "sqrt"};
  return names[static_cast<int>(op)];
}

// Expr DAG -> SSA with structural CSE shared across every lowered root.
class Lowering {
 public:
  explicit Lowering(const SymbolTable& args) : args_(args) {}

  int root(const Expr& e) { return node(e); }
  std::vector<Instr> code;
  std::vector<double> consts;

 private:
  int emit(Op op, int a = -1, int b = -1, std::int64_t imm = 0) {
    const auto key = std::make_tuple(static_cast<int>(op), a, b, imm);
    auto it = cse_.find(key);
    if (it != cse_.end()) return it->second;
    code.push_back({op, a, b, imm});
    const int reg = static_cast<int>(code.size()) - 1;
    cse_.emplace(key, reg);
    return reg;
  }
  int literal(double v) {
    const std::uint64_t bits = std::bit_cast<std::uint64_t>(v);
    auto it = pool_.find(bits);
    std::int64_t slot;
    if (it == pool_.end()) {
      slot = static_cast<std::int64_t>(consts.size());
      consts.push_back(v);
      pool_.emplace(bits, slot);
    } else {
      slot = it->second;
    }
    return emit(Op::LoadConst, -1, -1, slot);
  }
  static bool negated(const Expr& e) {
    return e.kind() == Kind::Mul && e.children()[0].is_constant() && e.children()[0].node().constant.is_minus_one();
  }
  // product of e's factors without the leading -1
  int unsigned_product(const Expr& e) {
    const auto& k = e.children();
    int acc = node(k[1]);
    for (std::size_t i = 2; i < k.size(); ++i) acc = emit(Op::Mul, acc, node(k[i]));
    return acc;
  }
  int node(const Expr& e) {
    auto m = memo_.find(e.raw());
    if (m != memo_.end()) return m->second;
    int reg = -1;
    const auto& k = e.children();
    switch (e.kind()) {
      case Kind::Constant:
        reg = literal(e.constant_value());
        break;
      case Kind::Symbol: {
        const int slot = args_.slot(e.name());
        if (slot < 0) throw CodegenError("unbound symbol '" + e.name() + "'");
        reg = emit(Op::LoadArg, -1, -1, slot);
        break;
      }
      case Kind::Add:
        reg = negated(k[0]) ? emit(Op::Neg, unsigned_product(k[0])) : node(k[0]);
        for (std::size_t i = 1; i < k.size(); ++i)
          reg = negated(k[i]) ? emit(Op::Sub, reg, unsigned_product(k[i])) : emit(Op::Add, reg, node(k[i]));
        break;
      case Kind::Mul:
        if (negated(e)) {
          reg = emit(Op::Neg, unsigned_product(e));
        } else if (k.size() == 2 && k[0].is_constant() && k[0].constant_value() == 2.0) {
          const int t = node(k[1]);
          reg = emit(Op::Add, t, t);
        } else {
          reg = node(k[0]);
          for (std::size_t i = 1; i < k.size(); ++i) reg = emit(Op::Mul, reg, node(k[i]));
        }
        break;
      case Kind::Pow: {
        const int b = node(k[0]);
        const std::int64_t x = e.exponent(), mag = x < 0 ? -x : x;
        if (mag <= 4) {
          int p = b;
          if (mag == 2) p = emit(Op::Mul, b, b);
          if (mag == 3) p = emit(Op::Mul, emit(Op::Mul, b, b), b);
          if (mag == 4) {
            const int s = emit(Op::Mul, b, b);
            p = emit(Op::Mul, s, s);
          }
          reg = x < 0 ? emit(Op::Div, literal(1.0), p) : p;
        } else {
          reg = emit(Op::PowInt, b, -1, x);
        }
        break;
      }
      case Kind::Div:
        reg = emit(Op::Div, node(k[0]), node(k[1]));
        break;
      case Kind::Sin:
        reg = emit(Op::Sin, node(k[0]));
        break;
      case Kind::Cos:
        reg = emit(Op::Cos, node(k[0]));
        break;
      case Kind::Sqrt:
        reg = emit(Op::Sqrt, node(k[0]));
        break;
    }
    memo_.emplace(e.raw(), reg);
    return reg;
  }

  const SymbolTable& args_;
  std::unordered_map<const Node*, int> memo_;
  std::map<std::tuple<int, int, int, std::int64_t>, int> cse_;
  std::unordered_map<std::uint64_t, std::int64_t> pool_;
};

}  // namespace

double KernelProgram::run(std::span<const double> args) const {
  std::vector<double> scratch;
  return run(args, scratch);
}

double KernelProgram::run(std::span<const double> args, std::vector<double>& scratch) const {
  if (static_cast<int>(args.size()) != arity)
    throw CodegenError("argument count mismatch: expected " + std::to_string(arity) + ", got " +
                       std::to_string(args.size()));
  if (scratch.size() < code.size()) scratch.resize(code.size());
  double* r = scratch.data();
  for (std::size_t k = 0; k < code.size(); ++k) r[k] = exec(code[k], r, args, consts);
  return r[result];
}

std::string KernelProgram::disassemble() const {
  std::string out;
  for (std::size_t k = 0; k < code.size(); ++k) {
    const Instr& in = code[k];
    out += "r" + std::to_string(k) + " = " + mnemonic(in.op);
    switch (in.op) {
      case Op::LoadArg: out += " " + std::to_string(in.imm); break;
      case Op::LoadConst: {
        char buf[64];
        auto r = std::to_chars(buf, buf + sizeof buf, consts[in.imm]);
        out += " " + std::string(buf, r.ptr);
        break;
      }
      case Op::Neg:
      case Op::Sin:
      case Op::Cos:
      case Op::Sqrt: out += " r" + std::to_string(in.a); break;
      case Op::PowInt: out += " r" + std::to_string(in.a) + " " + std::to_string(in.imm); break;
      default: out += " r" + std::to_string(in.a) + " r" + std::to_string(in.b);
    }
    out += "\n";
  }
  return out + "ret r" + std::to_string(result) + "\n";
}

KernelProgram lower(const Expr& e, const SymbolTable& args) {
  Lowering L(args);
  KernelProgram p;
  p.arity = args.size();
  p.result = L.root(e);
  p.code = std::move(L.code);
  p.consts = std::move(L.consts);
  return p;
}

MultiProgram lower_many(const std::vector<Expr>& outputs, const SymbolTable& args) {
  Lowering L(args);
  MultiProgram p;
  p.arg_names = args.names();
  for (const Expr& e : outputs) p.results.push_back(L.root(e));
  p.code = std::move(L.code);
  p.consts = std::move(L.consts);
  return p;
}

void MultiProgram::run(std::span<const double> args, std::span<double> out) const {
  std::vector<double> r(code.size());
  for (std::size_t k = 0; k < code.size(); ++k) r[k] = exec(code[k], r.data(), args, consts);
  for (std::size_t i = 0; i < results.size(); ++i) out[i] = r[results[i]];
}

CompiledForm compile_form(const fem::InstantiatedForm& f) {
  CompiledForm cf;
  const SymbolTable& args = fem::kernel_args(f.dim);
  for (const Expr& e : f.bilinear) cf.bilinear.push_back(lower(e, args));
  for (const Expr& e : f.linear) cf.linear.push_back(lower(e, args));
  cf.n_local = f.n_local;
  cf.dim = f.dim;
  cf.n_quad = fem::quadrature_rule(f.dim, default_quad_rule(f.dim, f.degree)).size();
  return cf;
}

int default_quad_rule(int dim, int degree) {
  if (dim == 2) return 3;  // the reference rule (fem.cpp:43-48)
  (void)degree;
  return 4;  // degree-2 tet rule: exact for P1/P2 stiffness (Appendix B)
}

}  // namespace femforge::codegen
