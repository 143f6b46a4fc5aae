// expression.cpp — "x = <expr>" -> pt_apply_op bytecode.
//
// Grammar, lexical rules, depth limit (32) and error messages follow the reference's
// expr::Program::parse (proj/src/expression.cpp:34-338) so validation errors are the
// same whichever backend runs the op; the evaluator is the device VM in
// paper_1606_04884_b200/csrc/pointwise.cu (Program::eval semantics, :340-402).
#include <cctype>
#include <charconv>
#include <cstring>

#include "../../include/pt_b200.h"
#include "portten/expression.hpp"

namespace portten::expr {

namespace {

enum class Tok { Ident, Number, Plus, Minus, Star, Slash, LParen, RParen, Comma, Assign, End };

struct Token {
    Tok kind = Tok::End;
    std::string text;
    float value = 0.0f;
};

class Scanner {
public:
    explicit Scanner(std::string_view s) : s_(s) { cur_ = scan(); }
    const Token& peek() const { return cur_; }
    Token take() {
        Token t = cur_;
        cur_ = scan();
        return t;
    }

private:
    std::string_view s_;
    std::size_t i_ = 0;
    Token cur_;

    static bool digit(char c) { return std::isdigit(static_cast<unsigned char>(c)) != 0; }

    Token scan() {
        while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
        if (i_ >= s_.size()) return {Tok::End, "", 0.0f};
        const char c = s_[i_];
        if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
            const std::size_t b = i_;
            while (i_ < s_.size() && (std::isalnum(static_cast<unsigned char>(s_[i_])) || s_[i_] == '_')) ++i_;
            return {Tok::Ident, std::string(s_.substr(b, i_ - b)), 0.0f};
        }
        if (digit(c) || (c == '.' && i_ + 1 < s_.size() && digit(s_[i_ + 1]))) {
            const std::size_t b = i_;
            while (i_ < s_.size() && (digit(s_[i_]) || s_[i_] == '.')) ++i_;
            if (i_ < s_.size() && (s_[i_] == 'e' || s_[i_] == 'E')) {
                std::size_t e = i_ + 1;
                if (e < s_.size() && (s_[e] == '+' || s_[e] == '-')) ++e;
                if (e < s_.size() && digit(s_[e])) {
                    i_ = e;
                    while (i_ < s_.size() && digit(s_[i_])) ++i_;
                }
            }
            std::string lit(s_.substr(b, i_ - b));
            float v = 0.0f;
            auto [end, ec] = std::from_chars(lit.data(), lit.data() + lit.size(), v);
            if (ec != std::errc() || end != lit.data() + lit.size())
                throw ValidationError("apply expression: bad numeric literal '" + lit + "'");
            return {Tok::Number, lit, v};
        }
        ++i_;
        switch (c) {
            case '+': return {Tok::Plus, "+", 0.0f};
            case '-': return {Tok::Minus, "-", 0.0f};
            case '*': return {Tok::Star, "*", 0.0f};
            case '/': return {Tok::Slash, "/", 0.0f};
            case '(': return {Tok::LParen, "(", 0.0f};
            case ')': return {Tok::RParen, ")", 0.0f};
            case ',': return {Tok::Comma, ",", 0.0f};
            case '=': return {Tok::Assign, "=", 0.0f};
            default:
                throw ValidationError(std::string("apply expression: unexpected character '") + c + "'");
        }
    }
};

struct Fn {
    const char* name;
    const char* cname;  // kernel-language spelling for kernelStatement()
    int argc;
    int op;
};
constexpr Fn kFns[] = {{"abs", "fabs", 1, PT_OP_ABS},   {"exp", "exp", 1, PT_OP_EXP},
                       {"log", "log", 1, PT_OP_LOG},    {"sqrt", "sqrt", 1, PT_OP_SQRT},
                       {"tanh", "tanh", 1, PT_OP_TANH}, {"max", "fmax", 2, PT_OP_MAX},
                       {"min", "fmin", 2, PT_OP_MIN}};

}  // namespace

class ProgramBuilder {
public:
    ProgramBuilder(std::string_view text, int arity) : sc_(text), arity_(arity) {}

    Program build() {
        PORTTEN_CHECK(arity_ >= 1 && arity_ <= 3, "apply arity must be 1..3");
        Token head = sc_.take();
        if (head.kind != Tok::Ident || head.text != "x")
            throw ValidationError("apply expression must assign to operand x");
        if (sc_.take().kind != Tok::Assign)
            throw ValidationError("apply expression must have the form \"x = <expr>\"");
        std::string rhs = sum();
        if (sc_.peek().kind != Tok::End)
            throw ValidationError("apply expression: trailing tokens after expression");
        p_.kernelStatement_ = "x = " + rhs + ";";
        p_.arity_ = arity_;
        p_.referencedOperands_ = referenced_;
        return std::move(p_);
    }

private:
    Scanner sc_;
    int arity_;
    int depth_ = 0;
    int referenced_ = 0;
    Program p_;

    void op(int code) { p_.code_.push_back(code); }
    void push_depth(int d) {
        depth_ += d;
        PORTTEN_CHECK(depth_ <= 32, "apply expression too deep");
    }

    std::string sum() {
        std::string lhs = product();
        for (;;) {
            const Tok k = sc_.peek().kind;
            if (k != Tok::Plus && k != Tok::Minus) return lhs;
            sc_.take();
            std::string rhs = product();
            op(k == Tok::Plus ? PT_OP_ADD : PT_OP_SUB);
            push_depth(-1);
            lhs = "(" + lhs + (k == Tok::Plus ? " + " : " - ") + rhs + ")";
        }
    }

    std::string product() {
        std::string lhs = unary();
        for (;;) {
            const Tok k = sc_.peek().kind;
            if (k != Tok::Star && k != Tok::Slash) return lhs;
            sc_.take();
            std::string rhs = unary();
            op(k == Tok::Star ? PT_OP_MUL : PT_OP_DIV);
            push_depth(-1);
            lhs = "(" + lhs + (k == Tok::Star ? " * " : " / ") + rhs + ")";
        }
    }

    std::string unary() {
        if (sc_.peek().kind == Tok::Minus) {
            sc_.take();
            std::string inner = unary();
            op(PT_OP_NEG);
            return "(-" + inner + ")";
        }
        return atom();
    }

    std::string atom() {
        Token t = sc_.take();
        switch (t.kind) {
            case Tok::Number: {
                std::int32_t bits;
                std::memcpy(&bits, &t.value, sizeof bits);
                op(PT_OP_CONST);
                op(bits);
                push_depth(+1);
                const bool frac = t.text.find_first_of(".eE") != std::string::npos;
                return frac ? t.text + "f" : t.text;
            }
            case Tok::LParen: {
                std::string inner = sum();
                if (sc_.take().kind != Tok::RParen) throw ValidationError("apply expression: missing ')'");
                return inner;
            }
            case Tok::Ident: return ident(t.text);
            case Tok::End: throw ValidationError("apply expression: unexpected end of input");
            default: throw ValidationError("apply expression: unexpected token '" + t.text + "'");
        }
    }

    std::string ident(const std::string& name) {
        if (name == "s") {
            op(PT_OP_S);
            push_depth(+1);
            return "s";
        }
        for (const Fn& f : kFns) {
            if (name != f.name) continue;
            if (sc_.take().kind != Tok::LParen)
                throw ValidationError("apply expression: expected '(' after function '" + name + "'");
            std::string a0 = sum(), text;
            if (f.argc == 2) {
                if (sc_.take().kind != Tok::Comma)
                    throw ValidationError("apply expression: function '" + name + "' takes two arguments");
                std::string a1 = sum();
                push_depth(-1);
                text = std::string(f.cname) + "(" + a0 + ", " + a1 + ")";
            } else {
                text = std::string(f.cname) + "(" + a0 + ")";
            }
            if (sc_.take().kind != Tok::RParen)
                throw ValidationError("apply expression: missing ')' in call to '" + name + "'");
            op(f.op);
            return text;
        }
        static const char* kOperands[3] = {"x", "y", "z"};
        int idx = -1;
        for (int i = 0; i < 3; ++i)
            if (name == kOperands[i]) idx = i;
        if (idx < 0) throw ValidationError("apply expression references undeclared operand '" + name + "'");
        if (idx >= arity_)
            throw ValidationError("apply expression references operand '" + name + "' but only " +
                                  std::to_string(arity_) + " operand(s) are declared");
        referenced_ = std::max(referenced_, idx + 1);
        op(PT_OP_X + idx);
        push_depth(+1);
        return name;
    }
};

Program Program::parse(std::string_view text, int arity) { return ProgramBuilder(text, arity).build(); }

}  // namespace portten::expr
