#!/usr/bin/env python3
"""Apply INTEGRATION.md §1-3 to a scratch copy of the reference, so its own
public entry points -- fusevec::evaluate / evaluate_block with
Backend::device() -- route to the B200 backend.  This is what a maintainer
would commit to the reference; here it proves the documented hook compiles
against, and runs through, the unmodified remainder of the reference.

    python3 tests/native/integrate_reference.py SRC_ROOT DST_ROOT

copies SRC_ROOT/{include,src} (the reference, read-only) to DST_ROOT (a
scratch directory outside this repository: no reference source is kept
here) and edits three files in the copy.  Every edit is anchored on the
exact reference text and fails loudly if the reference changes.
"""

import os
import shutil
import sys


def edit(path, old, new):
    with open(path) as f:
        s = f.read()
    if s.count(old) != 1:
        sys.exit(f"integrate_reference: anchor not found exactly once in {path}:\n{old}")
    with open(path, "w") as f:
        f.write(s.replace(old, new))


def main():
    src, dst = sys.argv[1], sys.argv[2]
    # --scalar-ref-switch (test builds only): Backend::scalar_ref() returns
    # the device backend when FUSEVEC_SCALAR_REF_IS_DEVICE is set, so the
    # reference's own unit tests -- and every implicit DenseVector = Expr
    # evaluation -- run on the device unchanged
    switch = "--scalar-ref-switch" in sys.argv[3:]
    if os.path.exists(dst):
        shutil.rmtree(dst)
    for sub in ("include", "src"):
        shutil.copytree(os.path.join(src, sub), os.path.join(dst, sub))
    inc = os.path.join(dst, "include", "fusevec", "backend.hpp")
    # §1: a fourth backend kind and its factory (backend.hpp:12-42)
    edit(inc, "enum class BackendKind : std::uint8_t { ScalarRef, Parallel, Codegen };",
         "enum class BackendKind : std::uint8_t { ScalarRef, Parallel, Codegen, Device };")
    edit(inc, "    BackendKind kind() const { return kind_; }",
         "    /// The B200 device backend on CUDA device `ordinal`.\n"
         "    static Backend device(int ordinal = 0) {\n"
         "        Backend b(BackendKind::Device);\n"
         "        b.workers_ = static_cast<std::size_t>(ordinal);\n"
         "        return b;\n"
         "    }\n\n"
         "    BackendKind kind() const { return kind_; }")
    if switch:
        edit(inc, "#include <cstddef>\n", "#include <cstddef>\n#include <cstdlib>\n")
        edit(inc, "    static Backend scalar_ref() { return Backend(BackendKind::ScalarRef); }",
             "    static Backend scalar_ref() {\n"
             "        static const bool dev = std::getenv(\"FUSEVEC_SCALAR_REF_IS_DEVICE\") != nullptr;\n"
             "        return dev ? device() : Backend(BackendKind::ScalarRef);\n"
             "    }")
    # §2: evaluate routes the device kind after validate() (backend_eval.cpp:280-346)
    ev = os.path.join(dst, "src", "backend_eval.cpp")
    edit(ev, '#include "fusevec/backend.hpp"\n',
         '#include "fusevec/backend.hpp"\n#include "fusevec_device.hpp"\n')
    edit(ev, "    const std::size_t n = dest.size();\n    if (n == 0) return;\n",
         "    const std::size_t n = dest.size();\n    if (n == 0) return;\n"
         "    if (backend.kind() == BackendKind::Device) {  // one fused sm_100a kernel\n"
         "        device::DeviceBackend be;\n"
         "        be.ordinal = static_cast<int>(backend.workers());\n"
         "        device::evaluate(be, e, dest);\n"
         "        return;\n"
         "    }\n")
    # §3: evaluate_block routes the device kind (block.cpp:455-463)
    bl = os.path.join(dst, "src", "block.cpp")
    edit(bl, '#include <map>\n', '#include <map>\n\n#include "fusevec_device.hpp"\n')
    for dest_type in ("BlockColVector", "BlockVectorGrid"):
        sig = (f"void evaluate_block(const Backend& backend, const BlockExpr& e, "
               f"{dest_type}& dest) {{\n")
        edit(bl, sig,
             sig + "    if (backend.kind() == BackendKind::Device) {  // all items in one fused pass\n"
                   "        device::DeviceBackend be;\n"
                   "        be.ordinal = static_cast<int>(backend.workers());\n"
                   "        device::evaluate_block(be, e, dest);\n"
                   "        return;\n"
                   "    }\n")

    # §8 (optional): the reference's own benchmark harness on the new kind
    # (bench.cpp:34-44) -- run_micro / run_miniapp then time Backend::device()
    # against their CPU hand-fused loops and keep their own checks (bitwise
    # generic == hand for micro, the flux oracle and device == parallel
    # bitwise for miniapp)
    bn = os.path.join(dst, "src", "bench.cpp")
    edit(bn, 'const char* backend_label(BackendKind k) {\n',
         'const char* backend_label(BackendKind k) {\n'
         '    if (k == BackendKind::Device) return "b200x1";\n')
    edit(bn, 'Backend pick_backend(const BenchConfig& cfg) {\n',
         'Backend pick_backend(const BenchConfig& cfg) {\n'
         '    if (cfg.backend == BackendKind::Device) return Backend::device();\n')


if __name__ == "__main__":
    main()
