// TEST INFRASTRUCTURE / REFERENCE ARM ONLY. The reference's builtin_tables()
// (ref: proj/src/tables.cpp:233-240) over generated data: the function body is
// the reference's own pattern (a magic static filled by the statements of
// tables_data.inc), with tables_data.inc emitted by tools/gen_ref_tables.py
// into oracle/_ref/gen/ in the record order of the reference's text artifact
// (ref: proj/src/tables.cpp:75-120). Linked in place of the weakened
// placeholder copy by oracle/Makefile (target _ref/libcrvec_refk.so).
#include "crvec/tables.hpp"

namespace crvec {

const AllTables& builtin_tables() {
  static const AllTables t = [] {
    AllTables v;
#include "tables_data.inc"
    return v;
  }();
  return t;
}

}  // namespace crvec
