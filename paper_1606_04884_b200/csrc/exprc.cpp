// exprc.cpp — the apply-expression compiler of libpt_b200.so: "x = <expr>" -> the RPN
// bytecode pt_b200_apply evaluates (include/pt_b200.h, pt_apply_op).
//
// Contract (the reference's expr::Program::parse, proj/include/portten/expression.hpp:29-45;
// grammar and messages per proj/src/expression.cpp): operands x y z (up to `arity`), the
// scalar s, float literals (digits/dots, optional exponent), + - * / with the usual
// precedence and left associativity, prefix minus binding tighter than * and /, parentheses,
// functions abs exp log sqrt tanh (one argument) and max min (two); an evaluation stack of
// at most 32 values. Every rejection is a ValidationError (PT_EVALIDATION) carrying the
// reference's message for the same input, so error text does not depend on the backend.
//
// Implementation: an operator-precedence (shunting-yard) translator driven by a two-state
// machine (expecting an operand / expecting an operator) over a token list. Tokens are
// scanned up front; a scan error becomes an Error token that is raised when the parser
// moves past the token before it — the point at which a one-token-lookahead scanner would
// meet the bad character — so inputs with several faults report the same first fault as
// the reference. Operands are emitted as they are read and operators when the precedence
// rule pops them, which yields the same RPN (and the same stack-depth trajectory) as a
// recursive-descent emitter.
#include <charconv>
#include <cctype>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pt_b200.h"

namespace ptb {
void set_last_error(const char* msg);  // abi.cu
}

namespace {

struct Reject {
    std::string msg;
};

enum class T { Ident, Number, Op, LParen, RParen, Comma, Assign, End, Error };

struct Tok {
    T kind;
    std::string text;  // identifier / literal / operator character / error message
    float value = 0.0f;
};

// Scans the whole input. Stops at the first bad character or literal with an Error token.
std::vector<Tok> scan(const std::string& s) {
    std::vector<Tok> out;
    size_t i = 0;
    auto is_digit = [&](size_t k) { return k < s.size() && std::isdigit((unsigned char)s[k]); };
    for (;;) {
        while (i < s.size() && std::isspace((unsigned char)s[i])) ++i;
        if (i == s.size()) {
            out.push_back({T::End, "", 0.f});
            return out;
        }
        const char c = s[i];
        if (std::isalpha((unsigned char)c) || c == '_') {
            size_t j = i;
            while (j < s.size() && (std::isalnum((unsigned char)s[j]) || s[j] == '_')) ++j;
            out.push_back({T::Ident, s.substr(i, j - i), 0.f});
            i = j;
            continue;
        }
        if (is_digit(i) || (c == '.' && is_digit(i + 1))) {
            size_t j = i;
            while (j < s.size() && (is_digit(j) || s[j] == '.')) ++j;
            if (j < s.size() && (s[j] == 'e' || s[j] == 'E')) {
                size_t k = j + 1;
                if (k < s.size() && (s[k] == '+' || s[k] == '-')) ++k;
                if (is_digit(k)) {
                    j = k;
                    while (is_digit(j)) ++j;
                }
            }
            const std::string lit = s.substr(i, j - i);
            float v = 0.f;
            const auto r = std::from_chars(lit.data(), lit.data() + lit.size(), v);
            if (r.ec != std::errc() || r.ptr != lit.data() + lit.size()) {
                out.push_back({T::Error, "apply expression: bad numeric literal '" + lit + "'", 0.f});
                return out;
            }
            out.push_back({T::Number, lit, v});
            i = j;
            continue;
        }
        ++i;
        switch (c) {
            case '+': case '-': case '*': case '/': out.push_back({T::Op, std::string(1, c), 0.f}); break;
            case '(': out.push_back({T::LParen, "(", 0.f}); break;
            case ')': out.push_back({T::RParen, ")", 0.f}); break;
            case ',': out.push_back({T::Comma, ",", 0.f}); break;
            case '=': out.push_back({T::Assign, "=", 0.f}); break;
            default:
                out.push_back({T::Error, std::string("apply expression: unexpected character '") + c + "'", 0.f});
                return out;
        }
    }
}

struct Func {
    const char* name;
    const char* c_name;  // kernel-language spelling
    int op, argc;
};
constexpr Func kFuncs[] = {{"abs", "fabs", PT_OP_ABS, 1},   {"exp", "exp", PT_OP_EXP, 1},
                           {"log", "log", PT_OP_LOG, 1},    {"sqrt", "sqrt", PT_OP_SQRT, 1},
                           {"tanh", "tanh", PT_OP_TANH, 1}, {"max", "fmax", PT_OP_MAX, 2},
                           {"min", "fmin", PT_OP_MIN, 2}};

const Func* find_func(const std::string& n) {
    for (const Func& f : kFuncs)
        if (n == f.name) return &f;
    return nullptr;
}

// One pending entry of the operator stack.
struct Pending {
    enum Kind { Binary, Negate, Group, Call } kind;
    char op = 0;              // Binary: + - * /
    const Func* fn = nullptr; // Call
    int args = 0;             // Call: arguments completed so far
};

int prec(const Pending& p) {
    if (p.kind == Pending::Negate) return 3;
    return (p.op == '*' || p.op == '/') ? 2 : 1;
}

class Compiler {
public:
    Compiler(const std::string& text, int arity) : toks_(scan(text)), arity_(arity) {}

    void run() {
        if (toks_[0].kind == T::Error) throw Reject{toks_[0].text};  // scanned before anything else
        if (arity_ < 1 || arity_ > 3) throw Reject{"apply arity must be 1..3"};
        const Tok head = take();
        if (head.kind != T::Ident || head.text != "x") throw Reject{"apply expression must assign to operand x"};
        if (take().kind != T::Assign) throw Reject{"apply expression must have the form \"x = <expr>\""};
        bool want_operand = true;
        for (;;) {
            const Tok& t = look();
            if (want_operand) {
                want_operand = operand(t);
            } else if (t.kind == T::Op) {
                const char op = take().text[0];
                reduce_while([&](const Pending& p) { return p.kind <= Pending::Negate && prec(p) >= prec_of(op); });
                ops_.push_back({Pending::Binary, op});
                want_operand = true;
            } else if (t.kind == T::RParen || t.kind == T::Comma) {
                want_operand = close_or_separate(t.kind == T::Comma);
            } else {
                finish_at(t);  // end of input, or a token that cannot follow an operand
                return;
            }
        }
    }

    std::vector<int32_t> code;
    std::vector<std::string> text;  // kernel-language text of the values on the stack
    int referenced = 0;

private:
    std::vector<Tok> toks_;
    size_t pos_ = 0;
    int arity_;
    int depth_ = 0;
    std::vector<Pending> ops_;

    static int prec_of(char op) { return (op == '*' || op == '/') ? 2 : 1; }

    const Tok& look() const { return toks_[pos_]; }
    // Consuming a token exposes the next one; a scan error there is raised now.
    Tok take() {
        const Tok t = toks_[pos_];
        if (t.kind != T::End) ++pos_;
        if (toks_[pos_].kind == T::Error) throw Reject{toks_[pos_].text};
        return t;
    }

    void push_value(int32_t op, std::string txt) {
        code.push_back(op);
        text.push_back(std::move(txt));
        if (++depth_ > 32) throw Reject{"apply expression too deep"};
    }

    void emit(const Pending& p) {
        if (p.kind == Pending::Negate) {
            code.push_back(PT_OP_NEG);
            text.back() = "(-" + text.back() + ")";
            return;
        }
        const char* ops = "+-*/";
        static const int32_t bin[] = {PT_OP_ADD, PT_OP_SUB, PT_OP_MUL, PT_OP_DIV};
        code.push_back(bin[std::strchr(ops, p.op) - ops]);
        std::string rhs = std::move(text.back());
        text.pop_back();
        text.back() = "(" + text.back() + " " + p.op + " " + rhs + ")";
        --depth_;
    }

    template <class Pred>
    void reduce_while(Pred pred) {
        while (!ops_.empty() && pred(ops_.back())) {
            emit(ops_.back());
            ops_.pop_back();
        }
    }
    void reduce_to_bracket() {
        reduce_while([](const Pending& p) { return p.kind <= Pending::Negate; });
    }

    static std::string fname(const Pending& b) { return b.fn->name; }
    [[noreturn]] static void missing_close(const Pending& b) {
        if (b.kind == Pending::Group) throw Reject{"apply expression: missing ')'"};
        throw Reject{"apply expression: missing ')' in call to '" + fname(b) + "'"};
    }
    [[noreturn]] static void two_args(const Pending& b) {
        throw Reject{"apply expression: function '" + fname(b) + "' takes two arguments"};
    }

    // In the operand position. Returns whether an operand is still wanted afterwards.
    bool operand(const Tok& t) {
        switch (t.kind) {
            case T::Number: {
                const Tok n = take();
                const bool frac = n.text.find_first_of(".eE") != std::string::npos;
                int32_t bits;
                std::memcpy(&bits, &n.value, 4);
                push_value(PT_OP_CONST, frac ? n.text + "f" : n.text);
                code.push_back(bits);
                return false;
            }
            case T::Op:
                if (t.text == "-") {
                    take();
                    ops_.push_back({Pending::Negate});
                    return true;
                }
                break;
            case T::LParen:
                take();
                ops_.push_back({Pending::Group});
                return true;
            case T::Ident: {
                const Tok id = take();
                if (id.text == "s") {
                    push_value(PT_OP_S, "s");
                    return false;
                }
                if (const Func* f = find_func(id.text)) {
                    if (take().kind != T::LParen)
                        throw Reject{"apply expression: expected '(' after function '" + id.text + "'"};
                    ops_.push_back({Pending::Call, 0, f, 0});
                    return true;
                }
                const int idx = id.text == "x" ? 0 : id.text == "y" ? 1 : id.text == "z" ? 2 : -1;
                if (idx < 0) throw Reject{"apply expression references undeclared operand '" + id.text + "'"};
                if (idx >= arity_)
                    throw Reject{"apply expression references operand '" + id.text + "' but only " +
                                 std::to_string(arity_) + " operand(s) are declared"};
                referenced = std::max(referenced, idx + 1);
                push_value(PT_OP_X + idx, id.text);
                return false;
            }
            case T::End:
                throw Reject{"apply expression: unexpected end of input"};
            default:
                break;
        }
        const Tok bad = take();
        throw Reject{"apply expression: unexpected token '" + bad.text + "'"};
    }

    // ')' or ',' after an operand; returns whether an operand is wanted next.
    bool close_or_separate(bool comma) {
        reduce_to_bracket();
        if (ops_.empty()) throw Reject{"apply expression: trailing tokens after expression"};
        Pending& b = ops_.back();
        take();
        if (b.kind == Pending::Group) {
            if (comma) missing_close(b);
            ops_.pop_back();
            return false;
        }
        if (comma) {  // only between the two arguments of max / min
            if (b.fn->argc != 2 || b.args == 1) missing_close(b);
            b.args = 1;
            return true;
        }
        if (b.fn->argc == 2 && b.args == 0) two_args(b);
        const Func* f = b.fn;
        ops_.pop_back();
        code.push_back(f->op);
        if (f->argc == 2) {
            std::string a1 = std::move(text.back());
            text.pop_back();
            text.back() = std::string(f->c_name) + "(" + text.back() + ", " + a1 + ")";
            --depth_;
        } else {
            text.back() = std::string(f->c_name) + "(" + text.back() + ")";
        }
        return false;
    }

    // End of input, or a token that cannot follow an operand: every bracket must be closed
    // (the innermost open one reports, after the token is consumed), else trailing tokens.
    void finish_at(const Tok& t) {
        reduce_to_bracket();
        if (!ops_.empty()) {
            const Pending b = ops_.back();
            take();
            if (b.kind == Pending::Call && b.fn->argc == 2 && b.args == 0) two_args(b);
            missing_close(b);
        }
        if (t.kind != T::End) throw Reject{"apply expression: trailing tokens after expression"};
    }
};

}  // namespace

extern "C" int pt_b200_expression_compile(const char* text, int arity, int32_t* code,
                                          int32_t capacity, int32_t* ncode, int32_t* referenced,
                                          char* statement, size_t statement_cap) {
    try {
        if (!text) throw Reject{"apply expression: null text"};
        Compiler c(text, arity);
        c.run();
        if (ncode) *ncode = static_cast<int32_t>(c.code.size());
        if (referenced) *referenced = c.referenced;
        if (code) {
            if (static_cast<size_t>(capacity) < c.code.size()) throw Reject{"apply expression: code buffer too small"};
            std::memcpy(code, c.code.data(), c.code.size() * sizeof(int32_t));
        }
        if (statement && statement_cap) {
            const std::string st = "x = " + c.text.back() + ";";
            std::strncpy(statement, st.c_str(), statement_cap - 1);
            statement[statement_cap - 1] = 0;
        }
        return PT_OK;
    } catch (const Reject& r) {
        ptb::set_last_error(r.msg.c_str());
        return PT_EVALIDATION;
    } catch (const std::exception& e) {
        ptb::set_last_error(e.what());
        return PT_EBACKEND;
    }
}
