// regex_ops.cuh -- the regex grammar of the REGEX front-end: operator tags and what they mean.
//
// NOT in the reference (SPEC.md:11 scopes regular-expression synthesis out; PAPER.md:81-113 only motivates it), so
// there is no reference line to cite and parity is unpinned; the CPU oracle is oracle/regex_oracle.py, whose
// membership semantics are pinned to Python's `re.fullmatch`.
//
// A CS (characteristic sequence) has one bit per INFIX of the example strings, infixes sorted by (length, text):
// bit k = "infix k is in the language".  Bit 0 is the empty word.  On such bitsets
//   union        r | s   = CS(r) | CS(s)                                   (the engine's OP_OR)
//   question     r?      = CS(r) | bit 0
//   concatenation r s    : bit w = OR over the splits w = u v of  CS(r)[u] & CS(s)[v]
//   star         r*      : bit 0, and bit w = OR over the splits w = u v, u non-empty, of  CS(r)[u] & CS(r*)[v]
//                          (v is shorter than w and infixes are sorted by length: one pass in index order)
// The splits come from the GUIDE TABLE the host precomputes: offsets[w] .. offsets[w+1] index entries (u | v << 16)
// of infix indices.  The operators themselves are in wide2_regex.cuh: 32 candidates at a time on bit-sliced rows, with
// the same table regrouped by Engine::set_regex.
#pragma once
#include "cm_ops.cuh"

namespace ltlb200 {

constexpr int LW_REGEX = 1;  // "lane width" of the regex instantiation of the kernels (wide2.cuh)
enum : int { OP_RE_QUESTION = 8, OP_RE_STAR = 9, OP_RE_CONCAT = 10 };

}  // namespace ltlb200
