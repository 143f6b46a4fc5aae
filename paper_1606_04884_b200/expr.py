"""Apply-expression compiler: "x = <expr>" -> RPN bytecode for pt_b200_apply.

A thin binding of the library's single compiler (pt_b200_expression_compile,
paper_1606_04884_b200/csrc/exprc.cpp): the grammar of the reference's
expr::Program::parse (proj/include/portten/expression.hpp:29-45), its validation
messages (ValidationError) and its stack-depth limit of 32. The C++ operator API
(host/expression.cpp) and the reference-side Backend adapter (integration/) call the
same entry point, so every caller compiles identically.
"""
from __future__ import annotations

import ctypes as C
from typing import List

from ._lib import check, lib


class Program:
    """Compiled expression: bytecode, arity, referenced operand count, kernel statement."""

    def __init__(self, code: List[int], arity: int, referenced: int, statement: str):
        self.code, self.arity, self.referenced, self.statement = code, arity, referenced, statement


def parse(text: str, arity: int) -> Program:
    n, ref = C.c_int32(), C.c_int32()
    raw = text.encode()
    check(lib().pt_b200_expression_compile(raw, arity, None, 0, C.byref(n), None, None, 0))
    code = (C.c_int32 * max(n.value, 1))()
    stmt = C.create_string_buffer(8 * len(raw) + 256)
    check(lib().pt_b200_expression_compile(raw, arity, code, n.value, C.byref(n), C.byref(ref),
                                           stmt, len(stmt)))
    return Program(list(code[:n.value]), arity, ref.value, stmt.value.decode())


def compile_expression(text: str, arity: int) -> List[int]:
    return parse(text, arity).code
