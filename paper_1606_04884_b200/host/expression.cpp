// expression.cpp — expr::Program (include/portten/expression.hpp) over the library's one
// apply-expression compiler, pt_b200_expression_compile (csrc/exprc.cpp): same grammar,
// validation messages and depth limit as the reference's Program::parse
// (proj/include/portten/expression.hpp:29-45). A grammar error surfaces as ValidationError.
#include "portten/expression.hpp"

#include <vector>

#include "pt_b200.h"

namespace portten::expr {

class ProgramBuilder {
public:
    static Program build(std::string_view text, int arity) {
        const std::string src(text);
        std::int32_t n = 0, ref = 0;
        check(pt_b200_expression_compile(src.c_str(), arity, nullptr, 0, &n, nullptr, nullptr, 0));
        Program p;
        p.code_.resize(static_cast<std::size_t>(n));
        std::vector<char> stmt(8 * src.size() + 256);
        check(pt_b200_expression_compile(src.c_str(), arity, p.code_.data(), n, &n, &ref, stmt.data(),
                                         stmt.size()));
        p.kernelStatement_ = stmt.data();
        p.arity_ = arity;
        p.referencedOperands_ = ref;
        return p;
    }

private:
    static void check(int st) {
        if (st == PT_OK) return;
        if (st == PT_EVALIDATION) throw ValidationError(pt_b200_last_error());
        throw BackendError(pt_b200_last_error());
    }
};

Program Program::parse(std::string_view text, int arity) { return ProgramBuilder::build(text, arity); }

}  // namespace portten::expr
