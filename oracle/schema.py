"""Record-dimension schema parser and leaf flattener -- TEST INFRASTRUCTURE ONLY.

Part of the parity oracle (see oracle/oracle.h).  Independent of the product's
C++ parser in paper_2106_04284_b200/csrc/schema.cpp: the two share no code.

Grammar (mirrors Listing 1):
    dim    := leaf | record
    record := Name "{" field ("," field)* "}"
    field  := Tag ":" scalar ("[" INT "]")*  |  Tag (":" Name)? "{" ... "}" ("[" INT "]")*
    scalar := i8|i16|i32|i64|u8|u16|u32|u64|f32|f64|bool
Static arrays ``T[n]`` are replaced by a record of n fields named "0".."n-1"
(P:290).  Leaves are listed depth-first in declaration order
(P:296-309).
"""

SCALAR_SIZE = {
    "i8": 1, "u8": 1, "bool": 1,
    "i16": 2, "u16": 2,
    "i32": 4, "u32": 4, "f32": 4,
    "i64": 8, "u64": 8, "f64": 8,
}


class SchemaError(ValueError):
    pass


class _Parser:
    def __init__(self, text):
        self.s = "".join(text.split())
        self.p = 0

    def peek(self):
        return self.s[self.p] if self.p < len(self.s) else ""

    def expect(self, ch):
        if self.peek() != ch:
            raise SchemaError(f"expected {ch!r} at {self.p} in {self.s!r}")
        self.p += 1

    def ident(self):
        start = self.p
        while self.p < len(self.s) and (self.s[self.p].isalnum() or self.s[self.p] == "_"):
            self.p += 1
        if start == self.p:
            raise SchemaError(f"expected a name at {self.p} in {self.s!r}")
        return self.s[start:self.p]

    def dims(self):
        out = []
        while self.peek() == "[":
            self.p += 1
            start = self.p
            while self.peek().isdigit():
                self.p += 1
            if start == self.p:
                raise SchemaError("expected an array extent")
            n = int(self.s[start:self.p])
            if n < 1:
                raise SchemaError("zero-extent array")
            self.expect("]")
            out.append(n)
        return out

    def record_body(self):
        """Parses '{' field (',' field)* '}' and returns a list of (tag, node)."""
        self.expect("{")
        fields = []
        while True:
            tag = self.ident()
            if self.peek() == ":":
                self.p += 1
                name = self.ident()
                if self.peek() == "{":
                    node = ("record", self.record_body())
                else:
                    if name not in SCALAR_SIZE:
                        raise SchemaError(f"unknown scalar type {name!r}")
                    node = ("leaf", name)
            elif self.peek() == "{":
                node = ("record", self.record_body())
            else:
                raise SchemaError(f"expected ':' or '{{' after tag {tag!r}")
            for n in reversed(self.dims()):
                node = ("record", [(str(j), node) for j in range(n)])
            if any(t == tag for t, _ in fields):
                raise SchemaError(f"duplicate tag {tag!r}")
            fields.append((tag, node))
            if self.peek() == ",":
                self.p += 1
                continue
            self.expect("}")
            return fields

    def parse(self):
        name = self.ident()
        if self.peek() == "{":
            node = ("record", self.record_body())
        elif name in SCALAR_SIZE:
            node = ("leaf", name)
        else:
            raise SchemaError(f"bad schema {self.s!r}")
        if self.p != len(self.s):
            raise SchemaError(f"trailing text at {self.p} in {self.s!r}")
        return node


def flatten(schema):
    """Returns the DFS leaf list [(tag_path, scalar_type), ...]."""
    root = _Parser(schema).parse()
    out = []

    def walk(node, path):
        if node[0] == "leaf":
            out.append((".".join(path), node[1]))
        else:
            for tag, child in node[1]:
                walk(child, path + [tag])

    walk(root, [])
    return out


def leaf_sizes(schema):
    return [SCALAR_SIZE[t] for _, t in flatten(schema)]
