NAME          QUIRKS
OBJSENSE MAXIMIZE
ROWS
 N  OBJ
 n  SPARE
 L  R1
 g  R2
 E  R3
columns
    MARKER    'MARKER'  'INTORG'
    A   OBJ  1.5   R1  1   R2  2
    A   R1   0.25
    A   SPARE 7
    B   OBJ  0x1.8p1   R3  -1e0
    B   R2   .5
    MARKER    'MARKER'  'INTEND'
    C   R3   1.  OBJ -2
    C   OBJ  0.5
RHS
    R1  6.0  R2  1.0
    RHS OBJ  100
    RHS SPARE 3
    RHS R3  2
RANGES
    RNG  R3  0.0   SPARE 1
BOUNDS
 UP BND  A  -1
 LO BND  A  -3
 UP BND  NOPE 4
 PL BND  C
