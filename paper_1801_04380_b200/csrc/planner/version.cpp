// Library identity; the planner proper lives in the sibling translation units.
extern "C" const char* sn_version(void) { return "superneurons-b200 0.1.0"; }
