"""Parser of the drop-in `load` (front-end cost).

`dartomp.parser.Parser` (`parser.py:21-592`) descends six grammar levels for
every binary expression (`parse_logical_or` .. `parse_multiplicative`, each a
`_binary_chain`, `parser.py:471-498`), so a lone identifier costs twelve
Python calls before `parse_unary` is reached.  This subclass parses the same
six levels by precedence climbing: one call per level actually used.  It
builds the same `AstNode`s in the same order (post-order, left-associative
within a level, a tighter level binding first), consumes the same tokens and
raises the same errors at the same tokens, because every operand is still
parsed by the reference's own `parse_unary` and every non-binary construct by
the reference's own methods.  `tests/test_frontend.py` compares the trees
node for node (kind, span, name, op, value, type, resolved declaration,
parent) with the reference parser's on the corpus and on generated units.

The lexer stays the reference's: a regular-expression restatement was
measured slower (its cost is the `Token`/`Span` objects both build, not the
character loop).  What the front end does pay for is the cyclic collector:
a unit of 400 functions allocates millions of long-lived nodes and tokens,
and the collector's full passes over them took 2.9 of 6.2 s of `load`;
`pipeline.load` pauses it for the call (`paused_gc`).
"""
from __future__ import annotations

import gc

from ._host import import_dartomp

import_dartomp()
from dartomp.diagnostics import Diagnostic  # noqa: E402
from dartomp.lexer import Preprocessed, TokenKind, expand_defines  # noqa: E402
from dartomp.nodes import AstNode, NodeKind  # noqa: E402
from dartomp.parser import Parser  # noqa: E402
from dartomp.source import SourceFile, Span  # noqa: E402

# `parser.py:482-498`: one level per operator set, loosest first
_BIN_PREC = {"||": 1, "&&": 2, "==": 3, "!=": 3, "<": 4, ">": 4, "<=": 4, ">=": 4,
             "+": 5, "-": 5, "*": 6, "/": 6, "%": 6}
_PUNCT = TokenKind.PUNCT
_BINARY_OP = NodeKind.BINARY_OP


class ClimbingParser(Parser):
    """`Parser` with `parse_logical_or` (the entry of the binary levels,
    called only from `parse_assignment`, `parser.py:455`) by precedence
    climbing."""

    def parse_translation_unit(self) -> AstNode:
        """`Parser.parse_translation_unit` (`parser.py:92-113`) with the
        parent links set by an explicit pre-order walk: `link_parents`
        (`nodes.py:193-196`) walks the whole unit through nested generators
        (`AstNode.walk`, `nodes.py:108-111`), one generator frame per level
        per node."""
        start = self.peek().span.start if not self.at_end() else 0
        children: list = []
        while not self.at_end():
            t = self.peek()
            if t.kind is TokenKind.PRAGMA:
                self.warnings.append(Diagnostic(
                    self.src.path, t.line, 1, "warning",
                    "pragma outside any function ignored"))
                self.advance()
                continue
            if t.lexeme == "struct" and self.peek(2) is not None and self.check("{", 2):
                children.append(self.parse_struct_decl())
                continue
            children.append(self.parse_external_decl())
        end = self.toks[-1].span.end if self.toks else start
        tu = AstNode(NodeKind.TRANSLATION_UNIT, Span(0, max(end, len(self.src.text))), children)
        stack = [tu]                # the pre-order of `walk`, so a shared child ends the same
        pop, extend = stack.pop, stack.extend
        while stack:
            node = pop()
            ch = node.children
            if ch:
                for c in ch:
                    c.parent = node
                extend(reversed(ch))
        return tu

    def parse_logical_or(self) -> AstNode:
        return self._climb(1)

    def _climb(self, min_prec: int) -> AstNode:
        # `_binary_chain(sub, ops)` (`parser.py:471-480`) at every level
        # >= min_prec: an operator of level p takes as its right operand
        # everything that binds tighter than p
        lhs = self.parse_unary()
        toks = self.toks
        n = len(toks)
        prec = _BIN_PREC
        while True:
            i = self.pos
            if i >= n:
                return lhs
            t = toks[i]
            if t.kind is not _PUNCT:
                return lhs
            p = prec.get(t.lexeme)
            if p is None or p < min_prec:
                return lhs
            self.pos = i + 1
            rhs = self._climb(p + 1)
            lhs = AstNode(_BINARY_OP, Span(lhs.span.start, rhs.span.end), [lhs, rhs], op=t.lexeme)


def parse(src: SourceFile, pre: Preprocessed | None = None):
    """`dartomp.parser.parse` (`parser.py:651-657`) on `ClimbingParser`."""
    if pre is None:
        pre = expand_defines(src)
    p = ClimbingParser(src, pre.tokens)
    tu = p.parse_translation_unit()
    return tu, pre.warnings + p.warnings


class paused_gc:
    """Context: the cyclic collector off, restored as it was.  A front-end
    pass builds long-lived trees (no cyclic garbage); the collector's passes
    over them would otherwise cost about as much as the pass itself."""

    def __enter__(self):
        self.was = gc.isenabled()
        gc.disable()
        return self

    def __exit__(self, *exc):
        if self.was:
            gc.enable()
        return False
