"""Apply-expression compiler: "x = <expr>" -> RPN bytecode for pt_b200_apply.

Host mirror of expr::Program::parse (proj/src/expression.cpp:34-338): the same
lexer (identifiers, numeric literals with optional exponent, + - * / ( ) , =),
the same recursive-descent grammar (expr/term/factor/primary, unary minus,
functions abs exp log sqrt tanh max min, operands x y z and the scalar s), the
same validation errors (ValidationError with the reference's messages) and the
same depth limit (32). The device evaluates the bytecode with an explicit stack
exactly like Program::eval (expression.cpp:340-402).
"""
from __future__ import annotations

import struct
from typing import List, Tuple

from ._lib import ValidationError

OP = {"CONST": 0, "X": 1, "Y": 2, "Z": 3, "S": 4, "ADD": 5, "SUB": 6, "MUL": 7, "DIV": 8,
      "NEG": 9, "ABS": 10, "EXP": 11, "LOG": 12, "SQRT": 13, "TANH": 14, "MAX": 15, "MIN": 16}
FUNCS = {"abs": ("ABS", 1), "exp": ("EXP", 1), "log": ("LOG", 1), "sqrt": ("SQRT", 1),
         "tanh": ("TANH", 1), "max": ("MAX", 2), "min": ("MIN", 2)}
OPERANDS = ("x", "y", "z")


def _f32_bits(v: float) -> int:
    return struct.unpack("<i", struct.pack("<f", v))[0]


class _Lexer:
    def __init__(self, src: str):
        self.src, self.pos = src, 0
        self.cur = self._advance()

    def peek(self):
        return self.cur

    def next(self):
        t = self.cur
        self.cur = self._advance()
        return t

    def _advance(self) -> Tuple[str, str, float]:
        s, n = self.src, len(self.src)
        while self.pos < n and s[self.pos].isspace():
            self.pos += 1
        if self.pos >= n:
            return ("end", "", 0.0)
        c = s[self.pos]
        if c.isalpha() or c == "_":
            st = self.pos
            while self.pos < n and (s[self.pos].isalnum() or s[self.pos] == "_"):
                self.pos += 1
            return ("ident", s[st:self.pos], 0.0)
        if c.isdigit() or (c == "." and self.pos + 1 < n and s[self.pos + 1].isdigit()):
            st = self.pos
            while self.pos < n and (s[self.pos].isdigit() or s[self.pos] == "."):
                self.pos += 1
            if self.pos < n and s[self.pos] in "eE":
                e = self.pos + 1
                if e < n and s[e] in "+-":
                    e += 1
                if e < n and s[e].isdigit():
                    self.pos = e
                    while self.pos < n and s[self.pos].isdigit():
                        self.pos += 1
            text = s[st:self.pos]
            try:
                value = struct.unpack("<f", struct.pack("<f", float(text)))[0]
            except (ValueError, OverflowError):
                raise ValidationError(f"apply expression: bad numeric literal '{text}'") from None
            return ("number", text, value)
        self.pos += 1
        kinds = {"+": "plus", "-": "minus", "*": "star", "/": "slash", "(": "lparen",
                 ")": "rparen", ",": "comma", "=": "assign"}
        if c in kinds:
            return (kinds[c], c, 0.0)
        raise ValidationError(f"apply expression: unexpected character '{c}'")


class Program:
    """Compiled apply program: RPN bytecode + arity (expr::Program)."""

    def __init__(self, code: List[int], arity: int, referenced: int):
        self.code, self.arity, self.referenced_operands = code, arity, referenced


def compile_expression(text: str, arity: int) -> List[int]:
    return parse(text, arity).code


def parse(text: str, arity: int) -> Program:
    if not 1 <= arity <= 3:
        raise ValidationError("apply arity must be 1..3")
    lx = _Lexer(text)
    code: List[int] = []
    state = {"depth": 0, "ref": 0}

    def emit(op, const=None):
        code.append(OP[op])
        if const is not None:
            code.append(_f32_bits(const))

    def track(d):
        state["depth"] += d
        if state["depth"] > 32:
            raise ValidationError("apply expression too deep")

    def p_expr():
        p_term()
        while lx.peek()[0] in ("plus", "minus"):
            k = lx.next()[0]
            p_term()
            emit("ADD" if k == "plus" else "SUB")
            track(-1)

    def p_term():
        p_factor()
        while lx.peek()[0] in ("star", "slash"):
            k = lx.next()[0]
            p_factor()
            emit("MUL" if k == "star" else "DIV")
            track(-1)

    def p_factor():
        if lx.peek()[0] == "minus":
            lx.next()
            p_factor()
            emit("NEG")
            return
        p_primary()

    def p_primary():
        kind, tx, val = lx.next()
        if kind == "number":
            emit("CONST", val)
            track(1)
            return
        if kind == "lparen":
            p_expr()
            if lx.next()[0] != "rparen":
                raise ValidationError("apply expression: missing ')'")
            return
        if kind == "ident":
            return p_ident(tx)
        if kind == "end":
            raise ValidationError("apply expression: unexpected end of input")
        raise ValidationError(f"apply expression: unexpected token '{tx}'")

    def p_ident(name):
        if name == "s":
            emit("S")
            track(1)
            return
        if name in FUNCS:
            op, argc = FUNCS[name]
            if lx.next()[0] != "lparen":
                raise ValidationError(f"apply expression: expected '(' after function '{name}'")
            p_expr()
            if argc == 2:
                if lx.next()[0] != "comma":
                    raise ValidationError(f"apply expression: function '{name}' takes two arguments")
                p_expr()
                track(-1)
            if lx.next()[0] != "rparen":
                raise ValidationError(f"apply expression: missing ')' in call to '{name}'")
            emit(op)
            return
        if name not in OPERANDS:
            raise ValidationError(f"apply expression references undeclared operand '{name}'")
        idx = OPERANDS.index(name)
        if idx >= arity:
            raise ValidationError(f"apply expression references operand '{name}' but only "
                                  f"{arity} operand(s) are declared")
        state["ref"] = max(state["ref"], idx + 1)
        emit(("X", "Y", "Z")[idx])
        track(1)

    head = lx.next()
    if head[0] != "ident" or head[1] != "x":
        raise ValidationError("apply expression must assign to operand x")
    if lx.next()[0] != "assign":
        raise ValidationError('apply expression must have the form "x = <expr>"')
    p_expr()
    if lx.peek()[0] != "end":
        raise ValidationError("apply expression: trailing tokens after expression")
    return Program(code, arity, state["ref"])
