// expr::Program — the apply grammar "x = <expr>" of the reference
// (proj/include/portten/expression.hpp:29-85): same accepted language, validation
// messages, depth limit and kernel statement. Compiled by the library's operator-precedence
// compiler (pt_b200_expression_compile, csrc/exprc.cpp) to the RPN bytecode pt_b200_apply
// evaluates on the device (include/pt_b200.h).
#pragma once

#include <cstdint>
#include <string>
#include <string_view>
#include <vector>

#include "portten/errors.hpp"

namespace portten::expr {

class Program {
public:
    static Program parse(std::string_view text, int arity);

    /// pt_apply_op bytecode (PT_OP_CONST followed by the float's bit pattern).
    const std::vector<std::int32_t>& code() const { return code_; }
    /// Canonical C text of the assignment, e.g. "x = (x * 2);" (fabs/fmax names).
    const std::string& kernelStatement() const { return kernelStatement_; }
    int arity() const { return arity_; }
    int referencedOperands() const { return referencedOperands_; }

private:
    std::vector<std::int32_t> code_;
    std::string kernelStatement_;
    int arity_ = 0;
    int referencedOperands_ = 0;
    friend class ProgramBuilder;
};

}  // namespace portten::expr
